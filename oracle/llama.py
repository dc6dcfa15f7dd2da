"""ORACLE (test infrastructure only) — CPU fp32 restatement of the Llama
forward, greedy decoding and deterministic random init the B200 engine runs.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; the product package never does.

PARITY UNPINNED against the reference for the numerics: the reference
(shardsim) has no tensors, logits or tokens (pkg/README.md:10-11,
SPEC.md:8); the paper's model math is vLLM 0.5.4's Llama (PAPER.md:312,
:493-494), which is not vendored.  This file is therefore the numeric oracle
by construction — standard Llama (RMSNorm, rotate-half RoPE, GQA attention,
SiLU-gated MLP, untied LM head) — and the reference pins only the structure
around it (placement, byte counts, schedule; see oracle/kv_layout.py and
tests/golden/).  What the reference does pin here:
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
    """Greedy generation with a per-sequence KV cache (fp32 or bf16-faithful)."""

    def __init__(self, a: Arch, seed: int, bf16_faithful: bool = True, max_pos: int = 4096,
                 weights: dict[str, torch.Tensor] | None = None) -> None:
        self.a = a
        self.bf = bf16_faithful
        self.W = weights if weights is not None else init_model(a, seed)
        self.cos, self.sin = rope_tables(a, max_pos)

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

    def _layer(self, x, l, pos, cache):
        a, W, p = self.a, self.W, f"L{l}."
        d, hq, hk = a.head_dim, a.num_query_heads, a.num_kv_heads
        h = self._norm(x, W[p + "attn_norm"])
        q = self._r(h @ W[p + "wq"].T).view(-1, hq, d)
        k = self._r(h @ W[p + "wk"].T).view(-1, hk, d)
        v = self._r(h @ W[p + "wv"].T).view(-1, hk, d)
        q, k = self._rope(q, pos), self._rope(k, pos)
        if l not in cache:
            cache[l] = (k, v)
        else:
            cache[l] = (torch.cat([cache[l][0], k]), torch.cat([cache[l][1], v]))
        K, V = cache[l]
        g = hq // hk
        Kx = K.repeat_interleave(g, dim=1)  # [S, hq, d]
        Vx = V.repeat_interleave(g, dim=1)
        s = torch.einsum("thd,shd->hts", q, Kx) / math.sqrt(d)
        S = K.shape[0]
        qpos = pos[:, None]
        kpos = torch.arange(S)[None, :]
        s = s.masked_fill((kpos > qpos)[None], float("-inf"))
        m = s.amax(-1, keepdim=True)
        e = torch.exp(s - m)
        l_ = e.sum(-1, keepdim=True)
        pe = self._r(e)  # the GPU feeds bf16 probabilities to the PV product
        o = torch.einsum("hts,shd->thd", pe, Vx) / l_.permute(1, 0, 2)
        o = self._r(o.reshape(-1, hq * d))
        x = self._r(x + o @ W[p + "wo"].T)
        h = self._norm(x, W[p + "mlp_norm"])
        gte = h @ W[p + "w1"].T
        up = h @ W[p + "w3"].T
        act = self._r(torch.nn.functional.silu(gte) * up)
        return self._r(x + act @ W[p + "w2"].T)

    def _forward(self, ids: torch.Tensor, pos: torch.Tensor, cache) -> torch.Tensor:
        x = self.W["embed"][ids.long()]
        for l in range(self.a.num_layers):
            x = self._layer(x, l, pos, cache)
        h = self._norm(x[-1:], self.W["final_norm"])
        return (h @ self.W["head"].T)[0]  # fp32 logits of the last position

    def generate(self, prompt: np.ndarray, output_len: int, forced: list[int] | None = None
                 ) -> tuple[list[int], list[torch.Tensor]]:
        """Greedy tokens g_1..g_out and the logits that produced them.  With
        ``forced`` = [g_1, g_2, ...] from another run the oracle feeds those
        tokens as inputs (teacher forcing: step k consumes forced[k-1]) and
        still returns its own argmax at every step."""
        cache: dict = {}
        ids = torch.from_numpy(np.asarray(prompt, dtype=np.int64))
        pos = torch.arange(ids.numel())
        logits = self._forward(ids, pos, cache)
        out, logs = [int(torch.argmax(logits))], [logits]
        n = ids.numel()
        for k in range(1, output_len):
            tok = forced[k - 1] if forced is not None else out[-1]
            logits = self._forward(torch.tensor([tok]), torch.tensor([n + k - 1]), cache)
            out.append(int(torch.argmax(logits)))
            logs.append(logits)
        return out, logs
