"""Fused TP combine: the row-parallel all-reduce of the decode layout plus the
RMSNorm after it, as ONE kernel over NVLink peer memory
(csrc/tp_allreduce.cu; replaces the NCCL all-reduce the reference charges per
layer, perf.py:71-74).

A :class:`PeerArena` holds, per TP group, three bf16 row buffers — ``part``
(this rank's partial sums, written by the o_proj / down_proj GEMM epilogue),
``x`` (the residual stream) and ``h`` (its normalised copy, the next GEMM's
input) — plus a signal buffer, all mapped into every peer through CUDA IPC
(:meth:`Comm.peer_addresses`).  ``combine(rows, gamma)`` turns every rank's
``part[:rows]`` into ``x[:rows]`` and ``h[:rows]`` on all ranks.

The arena is built collectively (every TP member calls :meth:`get` with the
same row count at the same point — the SPMD engine does) and checked once
with a known-answer self-test; if the peer mapping or the device barrier is
not usable the arena reports itself unusable and the worker keeps the NCCL
all-reduce + rmsnorm path (a warning says so).
"""

from __future__ import annotations

import warnings

import torch

from . import ops
from .comm import Comm


class PeerArena:
    def __init__(self, comm: Comm, device: torch.device, hidden: int, rows: int, max_blocks: int) -> None:
        self.comm = comm
        self.hidden = hidden
        self.rows = rows
        self.max_blocks = max_blocks
        bf = torch.bfloat16
        self.part = torch.zeros(rows, hidden, dtype=bf, device=device)
        self.x = torch.zeros(rows, hidden, dtype=bf, device=device)
        self.h = torch.zeros(rows, hidden, dtype=bf, device=device)
        self.sig = torch.zeros(ops.tp_signal_bytes() // 4, dtype=torch.int32, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        torch.cuda.current_stream(device).synchronize()
        self.addrs = {k: comm.peer_addresses(getattr(self, k)) for k in ("part", "x", "h", "sig")}
        self.epoch = 0
        self.usable = self._self_test()

    def combine(self, rows: int, gamma: torch.Tensor | None, eps: float, err: bool = False) -> None:
        """x[:rows], h[:rows] (if gamma) <- sum over ranks of part[:rows]."""
        self.epoch += 1
        a = self.addrs
        ops.tp_allreduce_rmsnorm(a["part"], a["x"], a["h"] if gamma is not None else None, a["sig"],
                                 self.comm.rank, rows, self.hidden, gamma, eps, self.epoch, self.max_blocks,
                                 self.err if err else None)

    def _self_test(self) -> bool:
        """Known answer: rank r's part = (r + 1) * ramp; x must be the exact
        bf16 of the fp32 sum, and h its rmsnorm (gamma = 1)."""
        n, r = self.comm.size, self.comm.rank
        rows = min(self.rows, 64)
        dev = self.part.device
        ramp = (torch.arange(rows * self.hidden, device=dev, dtype=torch.float32) % 61 - 30).view(rows, self.hidden)
        self.part[:rows].copy_((ramp * (r + 1) / 64).to(torch.bfloat16))
        want = torch.zeros(rows, self.hidden, dtype=torch.float32, device=dev)
        for p in range(n):
            want += (ramp * (p + 1) / 64).to(torch.bfloat16).float()
        want = want.to(torch.bfloat16)
        gamma = torch.ones(self.hidden, dtype=torch.bfloat16, device=dev)
        self.combine(rows, gamma, 1e-5, err=True)
        ref_h = ops.rmsnorm(want, gamma, 1e-5)
        ok = (int(self.err.item()) == 0 and torch.equal(self.x[:rows], want) and torch.equal(self.h[:rows], ref_h))
        flags = torch.tensor([1.0 if ok else 0.0], device=dev)
        self.comm.all_reduce_(flags)  # every member agrees on the outcome
        good = int(flags.item()) == n
        if not good:
            warnings.warn(f"fused TP combine self-test failed on rank {r} (err={int(self.err.item())}); "
                          "falling back to all-reduce + rmsnorm", RuntimeWarning, stacklevel=2)
        return good


def get_arena(cache: dict, comm: Comm, device: torch.device, hidden: int, rows: int,
              max_blocks: int) -> PeerArena | None:
    """The TP group's arena with room for ``rows`` rows (collective when it
    has to be (re)built: grows to the next power of two)."""
    key = (id(comm), hidden)
    ar = cache.get(key)
    if ar is not None and (not ar.usable or ar.rows >= rows):
        return ar if ar.usable else None
    cap = 1 << max(rows - 1, 255).bit_length()
    if ar is not None:
        cap = max(cap, ar.rows)
        del cache[key]
        del ar
    ar = PeerArena(comm, device, hidden, cap, max_blocks)
    cache[key] = ar
    return ar if ar.usable else None
