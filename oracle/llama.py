"""ORACLE (test infrastructure only) — CPU fp32 restatement of the Llama
forward, greedy decoding and deterministic random init the B200 engine runs.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; the product package never does.

Numerics PINNED to an independent implementation: the reference (shardsim)
has no tensors, logits or tokens (pkg/README.md:10-11) and the
paper's model math is vLLM 0.5.4's Llama, which is
not vendored.  tests/test_oracle_hf_cpu.py loads this file's weights into
Hugging Face transformers 5.5.0 ``LlamaForCausalLM`` (the same Llama math)
and requires the fp32 logits to agree within 2e-4 (measured 3.7e-6) and the
greedy tokens to be identical, on the tiny config and on a head_dim-128 GQA
shape with the Llama-3 RoPE base.  The reference pins the structure around
it (placement, byte counts, schedule; see oracle/kv_layout.py and
tests/golden/), and:
  * sequences are prefilled then decoded exactly output_len times with
    context input_len+1 .. input_len+output_len (sim.py:531, :553-562);
  * KV is reserved at (input_len + output_len) tokens (sim.py:9-12, :256).

Two modes:
  * fp32: every op in float32 from the bf16 weights (the "reference fp32");
  * bf16_faithful: rounds to bf16 at exactly the points the GPU stores bf16
    (norm outputs, projections, RoPE'd q/k, attention output, residual
    stream) so greedy token ids can be compared for identity.

Deterministic init (identical bits to csrc/init.cu):
  key = mix64(seed*G + tensor_id); element i of the logical tensor uses
  a = mix64(key + (2i+1)G), b = mix64(key + (2i+2)G), four 24-bit uniforms,
  x = (((u0+u1)+u2)+u3 - 2) * sqrt(3) * scale in float32, bf16 RNE.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest-even bf16, returned as float32 (finite inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000))
    return r.view(np.float32)


def init_values(seed: int, tensor_id: int, idx: np.ndarray, scale: float) -> np.ndarray:
    """bf16-rounded init values (as float32) of flat logical indices ``idx``."""
    if scale == 0.0:
        return np.ones(idx.shape, dtype=np.float32)
    with np.errstate(over="ignore"):
        key = _mix64(np.uint64(seed) * G + np.uint64(tensor_id))
        i = idx.astype(np.uint64)
        a = _mix64(key + (np.uint64(2) * i + np.uint64(1)) * G)
        b = _mix64(key + (np.uint64(2) * i + np.uint64(2)) * G)
    k = np.float32(2.0 ** -24)
    m = np.uint64(0xFFFFFF)
    u0 = (a >> np.uint64(40)).astype(np.float32) * k
    u1 = ((a >> np.uint64(8)) & m).astype(np.float32) * k
    u2 = (b >> np.uint64(40)).astype(np.float32) * k
    u3 = ((b >> np.uint64(8)) & m).astype(np.float32) * k
    s = ((u0 + u1) + u2) + u3
    x = (s - np.float32(2.0)) * np.float32(1.7320508075688772) * np.float32(scale)
    return bf16_round(x.astype(np.float32))


@dataclass(frozen=True)
class Arch:
    """Plain restatement of the architecture fields the oracle needs."""

    num_layers: int
    hidden: int
    num_query_heads: int
    num_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rope_theta: float
    rms_eps: float = 1e-5


def tensor_specs(a: Arch) -> dict[str, tuple[int, int, int, float]]:
    """name -> (tensor_id, rows, cols, scale) — the init convention."""
    h, d, f, v = a.hidden, a.head_dim, a.ffn, a.vocab
    out = {"embed": (1, v, h, 1.0), "head": (2, v, h, 1.0 / math.sqrt(h)), "final_norm": (3, 1, h, 0.0)}
    for l in range(a.num_layers):
        b, p = 1000 + 16 * l, f"L{l}."
        out[p + "attn_norm"] = (b, 1, h, 0.0)
        out[p + "wq"] = (b + 1, a.num_query_heads * d, h, 1.0 / math.sqrt(h))
        out[p + "wk"] = (b + 2, a.num_kv_heads * d, h, 1.0 / math.sqrt(h))
        out[p + "wv"] = (b + 3, a.num_kv_heads * d, h, 1.0 / math.sqrt(h))
        out[p + "wo"] = (b + 4, h, a.num_query_heads * d, 1.0 / math.sqrt(a.num_query_heads * d))
        out[p + "mlp_norm"] = (b + 5, 1, h, 0.0)
        out[p + "w1"] = (b + 6, f, h, 1.0 / math.sqrt(h))
        out[p + "w3"] = (b + 7, f, h, 1.0 / math.sqrt(h))
        out[p + "w2"] = (b + 8, h, f, 1.0 / math.sqrt(f))
    return out


def init_tensor(seed: int, spec: tuple[int, int, int, float], rows: slice | None = None) -> np.ndarray:
    tid, r, c, scale = spec
    r0, r1 = (0, r) if rows is None else (rows.start, rows.stop)
    idx = np.arange(r0 * c, r1 * c, dtype=np.int64).reshape(r1 - r0, c)
    return init_values(seed, tid, idx, scale)


def init_model(a: Arch, seed: int) -> dict[str, torch.Tensor]:
    return {k: torch.from_numpy(init_tensor(seed, s)) for k, s in tensor_specs(a).items()}


def rope_tables(a: Arch, max_pos: int) -> tuple[torch.Tensor, torch.Tensor]:
    d = a.head_dim
    inv = a.rope_theta ** (-np.arange(0, d, 2, dtype=np.float64) / d)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return torch.from_numpy(np.cos(ang).astype(np.float32)), torch.from_numpy(np.sin(ang).astype(np.float32))


class LlamaOracle:
    """Greedy generation with a per-sequence KV cache (fp32 or bf16-faithful).

    In bf16-faithful mode the oracle also reproduces the GPU's *structure*
    where it changes rounding: tensor-parallel partial sums are rounded to
    bf16 per rank before the all-reduce (rank 0 adds the residual in its GEMM
    epilogue), and attention runs the kernels' online softmax — 64-key tiles
    in prefill, per-warp 16-key slices of 64-token pool blocks in decode —
    with bf16 probabilities entering the PV product.  ``tp_prefill`` /
    ``tp_decode`` are the tensor-parallel degrees of the two phases.

    ``fold_norm`` mirrors the engine's default path (runtime.Worker.
    _block_folded, SSB_FOLD_NORM=1): in a phase whose tensor parallelism is
    1, the norm in front of a projection is not materialised — the projection
    consumes x and its fp32 accumulator rows are scaled by 1/rms before the
    bf16 rounding (gains are 1 in the synthetic init, so folding them into
    the weights is the identity).  The exceptions are the engine's: the
    attention norm of a stage's first layer (the stage's input arrives
    without row sums) and the final norm of a prefill (last-token rows) run
    as rmsnorm kernels.  ``pp_prefill`` / ``pp_decode`` give the stage
    boundaries of the two phases."""

    def __init__(self, a: Arch, seed: int, bf16_faithful: bool = True, max_pos: int = 4096,
                 weights: dict[str, torch.Tensor] | None = None, tp_prefill: int = 1, tp_decode: int = 1,
                 fold_norm: bool = False, pp_prefill: int = 1, pp_decode: int = 1, tp_fold: bool = False) -> None:
        self.a = a
        self.bf = bf16_faithful
        self.W = weights if weights is not None else init_model(a, seed)
        self.cos, self.sin = rope_tables(a, max_pos)
        self.tp_prefill, self.tp_decode = tp_prefill, tp_decode
        self.tp = tp_prefill
        self.fold_norm, self.pp_prefill, self.pp_decode = fold_norm, pp_prefill, pp_decode
        self.tp_fold = tp_fold
        self._decoding = False

    def _r(self, x: torch.Tensor) -> torch.Tensor:
        return x.to(torch.bfloat16).to(torch.float32) if self.bf else x

    def _norm(self, x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        inv = 1.0 / torch.sqrt((x * x).mean(-1, keepdim=True) + self.a.rms_eps)
        return self._r((x * inv) * w.reshape(-1))

    def _rope(self, x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        # x [T, H, d], rotate-half
        half = self.a.head_dim // 2
        c = self.cos[pos][:, None, :]
        s = self.sin[pos][:, None, :]
        x1, x2 = x[..., :half], x[..., half:]
        return self._r(torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1))

    def _tp_folded(self) -> bool:
        """Decode under a pure TP layout with the fused combine and the
        folded norm (runtime.Worker._block_fused_folded, SSB_TP_FOLD=1): every
        norm of the step is a 1/rms row scale of its consumer, the first
        layer's too (the embedding's combine already leaves the row sums)."""
        return self.fold_norm and self.tp_fold and self._decoding and self.tp > 1 and self.pp_decode == 1

    def _folding(self) -> bool:
        return self.fold_norm and (self.tp == 1 or self._tp_folded())

    def _inv_rms(self, x: torch.Tensor) -> torch.Tensor:
        return 1.0 / torch.sqrt((x * x).mean(-1, keepdim=True) + self.a.rms_eps)

    def _normed_matmuls(self, x, gain, mats, folded: bool):
        """[h @ W^T for W in mats] with h = rmsnorm(x) * gain materialised
        (rounded to bf16) or, folded, (x @ W^T) * (1/rms) on the fp32
        accumulator (gain 1)."""
        if not folded:
            h = self._norm(x, gain)
            return [h @ w.T for w in mats]
        assert bool(torch.all(gain == 1)), "folded norms need unit gains (the synthetic init)"
        inv = self._inv_rms(x)
        return [(x @ w.T) * inv for w in mats]

    def _layer(self, x, l, pos, cache):
        a, W, p = self.a, self.W, f"L{l}."
        d, hq, hk = a.head_dim, a.num_query_heads, a.num_kv_heads
        per_stage = a.num_layers // (self.pp_decode if self._decoding else self.pp_prefill)
        fold_attn = self._folding() and (l % per_stage != 0 or self._tp_folded())
        q, k, v = self._normed_matmuls(x, W[p + "attn_norm"], [W[p + "wq"], W[p + "wk"], W[p + "wv"]], fold_attn)
        q = self._r(q).view(-1, hq, d)
        k = self._r(k).view(-1, hk, d)
        v = self._r(v).view(-1, hk, d)
        q, k = self._rope(q, pos), self._rope(k, pos)
        if l not in cache:
            cache[l] = (k, v)
        else:
            cache[l] = (torch.cat([cache[l][0], k]), torch.cat([cache[l][1], v]))
        K, V = cache[l]
        g = hq // hk
        Kx = K.repeat_interleave(g, dim=1)  # [S, hq, d]
        Vx = V.repeat_interleave(g, dim=1)
        if self.bf:
            o = self._attn_tiled(q, Kx, Vx, pos)
        else:
            s = torch.einsum("thd,shd->hts", q, Kx) / math.sqrt(d)
            S = K.shape[0]
            s = s.masked_fill((torch.arange(S)[None, :] > pos[:, None])[None], float("-inf"))
            o = torch.einsum("hts,shd->thd", torch.softmax(s, -1), Vx)
        o = self._r(o.reshape(-1, hq * d))
        x = self._row_parallel(x, o, W[p + "wo"])
        gte, up = self._normed_matmuls(x, W[p + "mlp_norm"], [W[p + "w1"], W[p + "w3"]], self._folding())
        act = self._r(torch.nn.functional.silu(gte) * up)
        return self._row_parallel(x, act, W[p + "w2"])

    def layer_decode_batch(self, x: torch.Tensor, l: int, pos: torch.Tensor, caches: list[dict]) -> torch.Tensor:
        """One decode step of B independent sequences through layer ``l``
        (fp32): the projections and the MLP batched over the B rows, the
        attention of row b over sequence b's own cache ``caches[b][l]``
        (appended in place) — the engine's TP decode step restated on the
        CPU, used as the CPU baseline's decode sample (bench.py)."""
        a, W, p = self.a, self.W, f"L{l}."
        d, hq, hk = a.head_dim, a.num_query_heads, a.num_kv_heads
        g = hq // hk
        h = self._norm(x, W[p + "attn_norm"])
        q = self._rope((h @ W[p + "wq"].T).view(-1, hq, d), pos)
        k = self._rope((h @ W[p + "wk"].T).view(-1, hk, d), pos)
        v = (h @ W[p + "wv"].T).view(-1, hk, d)
        outs = []
        for b, cache in enumerate(caches):
            K0, V0 = cache[l]
            K, V = torch.cat([K0, k[b : b + 1]]), torch.cat([V0, v[b : b + 1]])
            cache[l] = (K, V)
            qb = q[b].view(hk, g, d)                                   # [hk, g, d]
            s = torch.einsum("kgd,skd->kgs", qb, K) / math.sqrt(d)
            outs.append(torch.einsum("kgs,skd->kgd", torch.softmax(s, -1), V).reshape(hq * d))
        o = torch.stack(outs)
        x = x + o @ W[p + "wo"].T
        h = self._norm(x, W[p + "mlp_norm"])
        act = torch.nn.functional.silu(h @ W[p + "w1"].T) * (h @ W[p + "w3"].T)
        return x + act @ W[p + "w2"].T

    def _row_parallel(self, x: torch.Tensor, a: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        """x + a @ w^T; with tp > 1 in bf16 mode, rank r's partial over its
        column slice is rounded to bf16 (rank 0 including x) and the partials
        are summed in fp32 in rank order, then rounded — the GPU's
        GEMM-epilogue residual + all-reduce."""
        if not self.bf or self.tp == 1:
            return self._r(x + a @ w.T)
        k = a.shape[1] // self.tp
        acc = None
        for r in range(self.tp):
            part = a[:, r * k : (r + 1) * k] @ w[:, r * k : (r + 1) * k].T
            part = self._r(part + x) if r == 0 else self._r(part)
            acc = part if acc is None else acc + part
        return self._r(acc)

    def _attn_tiled(self, q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        """Online softmax in exp2 domain with the kernels' key partitioning."""
        S = K.shape[0]
        decode = q.shape[0] == 1 and S > 1 and pos[0].item() == S - 1 and getattr(self, "_decoding", False)
        if decode:
            # 4 warps; warp w owns keys 64j + 16w .. +16 of every 64-key block
            parts = []
            for w_ in range(4):
                idx = torch.cat([torch.arange(j + 16 * w_, max(min(j + 16 * w_ + 16, S), j + 16 * w_))
                                 for j in range(0, S, 64)])
                parts.append(idx)
            states = [self._online(q, K, V, pos, [pi]) for pi in parts if pi.numel()]
            M = torch.stack([m for m, _, _ in states]).amax(0)
            Mu = torch.where(torch.isinf(M), torch.zeros_like(M), M)
            L = sum(l_ * torch.exp2(m - Mu) for m, l_, _ in states)
            O = sum(o * torch.exp2(m - Mu)[..., None] for m, _, o in states)
            return (O / L[..., None]).permute(1, 0, 2)
        tiles = [torch.arange(j, min(j + 64, S)) for j in range(0, S, 64)]
        m, l_, o = self._online(q, K, V, pos, tiles)
        return (o / l_[..., None]).permute(1, 0, 2)

    def _online(self, q, K, V, pos, chunks):
        c = torch.tensor(1.0 / math.sqrt(self.a.head_dim) * 1.4426950408889634, dtype=torch.float32)
        H, T, d = q.shape[1], q.shape[0], q.shape[2]
        m = torch.full((H, T), float("-inf"))
        l_ = torch.zeros(H, T)
        o = torch.zeros(H, T, d)
        for idx in chunks:
            s = torch.einsum("thd,shd->hts", q, K[idx]) * c
            s = s.masked_fill((idx[None, :] > pos[:, None])[None], float("-inf"))
            m_new = torch.maximum(m, s.amax(-1))
            mu = torch.where(torch.isinf(m_new), torch.zeros_like(m_new), m_new)
            corr = torch.exp2(m - mu)
            pexp = torch.exp2(s - mu[..., None])
            l_ = l_ * corr + pexp.sum(-1)
            o = o * corr[..., None] + torch.einsum("hts,shd->htd", self._r(pexp), V[idx])
            m = m_new
        return m, l_, o

    def _forward(self, ids: torch.Tensor, pos: torch.Tensor, cache) -> torch.Tensor:
        x = self.W["embed"][ids.long()]
        for l in range(self.a.num_layers):
            x = self._layer(x, l, pos, cache)
        # the final norm is folded into the LM head only in a decode step
        (logits,) = self._normed_matmuls(x[-1:], self.W["final_norm"], [self.W["head"]],
                                         self._folding() and self._decoding)
        return logits[0]  # fp32 logits of the last position

    def generate(self, prompt: np.ndarray, output_len: int, forced: list[int] | None = None
                 ) -> tuple[list[int], list[torch.Tensor]]:
        """Greedy tokens g_1..g_out and the logits that produced them.  With
        ``forced`` = [g_1, g_2, ...] from another run the oracle feeds those
        tokens as inputs (teacher forcing: step k consumes forced[k-1]) and
        still returns its own argmax at every step."""
        cache: dict = {}
        ids = torch.from_numpy(np.asarray(prompt, dtype=np.int64))
        pos = torch.arange(ids.numel())
        self.tp, self._decoding = self.tp_prefill, False
        logits = self._forward(ids, pos, cache)
        out, logs = [int(torch.argmax(logits))], [logits]
        n = ids.numel()
        self.tp, self._decoding = self.tp_decode, True
        for k in range(1, output_len):
            tok = forced[k - 1] if forced is not None else out[-1]
            logits = self._forward(torch.tensor([tok]), torch.tensor([n + k - 1]), cache)
            out.append(int(torch.argmax(logits)))
            logs.append(logits)
        return out, logs
