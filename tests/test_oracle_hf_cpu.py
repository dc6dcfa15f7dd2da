"""Pin the numeric oracle (oracle/llama.py, fp32) to an independent Llama
implementation: Hugging Face transformers' ``LlamaForCausalLM`` (5.5.0 in
this image; the same Llama math — RMSNorm, rotate-half RoPE, GQA, SiLU-gated
MLP, untied LM head — as vLLM's model implementation, which the paper's
engine builds on, and which is not vendored in the
reference).

Same random-init weights (the oracle's counter-based init, copied into the
HF model), same prompt, teacher forced on the oracle's greedy tokens:

* fp32 logits agree within 2e-4 absolute (both fp32; the difference is op
  order only: HF's fp32 RoPE tables vs the oracle's float64-computed ones,
  SDPA-free eager attention vs einsum);
* the greedy tokens are identical.

Two shapes: BASELINE configs[0] (tiny: 2 layers, hidden 256, 4 heads, d=64,
theta 1e4) and a head_dim-128 GQA-4 shape with the Llama-3 RoPE base 5e5
(2 layers, hidden 1024, 8 query / 2 KV heads) — the 8B kernels' geometry.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import llama as lo

transformers = pytest.importorskip("transformers")

SHAPES = {
    "tiny": lo.Arch(2, 256, 4, 4, 64, 768, 1024, 10000.0),
    "d128-gqa4": lo.Arch(2, 1024, 8, 2, 128, 3584, 2048, 500000.0),
}


def _hf_model(a: lo.Arch, W: dict[str, torch.Tensor]):
    from transformers import LlamaConfig, LlamaForCausalLM

    cfg = LlamaConfig(vocab_size=a.vocab, hidden_size=a.hidden, intermediate_size=a.ffn,
                      num_hidden_layers=a.num_layers, num_attention_heads=a.num_query_heads,
                      num_key_value_heads=a.num_kv_heads, head_dim=a.head_dim, rope_theta=a.rope_theta,
                      rms_norm_eps=a.rms_eps, tie_word_embeddings=False, max_position_embeddings=512,
                      attention_bias=False, mlp_bias=False, attn_implementation="eager")
    torch.manual_seed(0)
    m = LlamaForCausalLM(cfg).float().eval()
    names = {"embed": "model.embed_tokens.weight", "head": "lm_head.weight", "final_norm": "model.norm.weight"}
    per_layer = {"wq": "self_attn.q_proj", "wk": "self_attn.k_proj", "wv": "self_attn.v_proj",
                 "wo": "self_attn.o_proj", "w1": "mlp.gate_proj", "w3": "mlp.up_proj", "w2": "mlp.down_proj",
                 "attn_norm": "input_layernorm", "mlp_norm": "post_attention_layernorm"}
    for l in range(a.num_layers):
        for k, v in per_layer.items():
            names[f"L{l}.{k}"] = f"model.layers.{l}.{v}.weight"
    params = dict(m.named_parameters())
    assert set(names.values()) == set(params), set(params) ^ set(names.values())
    with torch.no_grad():
        for k, n in names.items():
            params[n].copy_(W[k].reshape(params[n].shape))
    return m


@pytest.mark.parametrize("shape", list(SHAPES))
def test_oracle_fp32_matches_transformers_llama(shape):
    a = SHAPES[shape]
    orc = lo.LlamaOracle(a, seed=0, bf16_faithful=False, max_pos=512)
    hf = _hf_model(a, orc.W)
    prompt = np.random.default_rng(1).integers(0, a.vocab, size=48).astype(np.int32)
    out_len = 8
    toks, logs = orc.generate(prompt, out_len)
    ids = torch.from_numpy(np.concatenate([prompt, np.asarray(toks[:-1], dtype=np.int32)]).astype(np.int64))
    with torch.no_grad():
        ref = hf(ids[None]).logits[0]                     # [48 + 7, V]
    ref = ref[len(prompt) - 1 :]                          # the logits that produced g_1 .. g_8
    got = torch.stack(logs)
    err = (got - ref).abs().max().item()
    assert err < 2e-4, f"{shape}: max |oracle - transformers| logit difference {err:.3g}"
    assert toks == [int(t) for t in ref.argmax(-1)], shape
    # the logits are O(1) (so the bound is meaningful) and the greedy margins
    # exceed the difference by orders of magnitude
    top2 = ref.topk(2, dim=-1).values
    assert ref.abs().max().item() > 1.0
    assert float((top2[:, 0] - top2[:, 1]).min()) > 10 * err
