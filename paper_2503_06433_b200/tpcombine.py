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

from . import _lib, ops
from ._lib import SeesawKernelError
from .comm import Comm


_GENERATION = [0]


class PeerArena:
    def __init__(self, comm: Comm, device: torch.device, hidden: int, rows: int, max_blocks: int) -> None:
        _GENERATION[0] += 1
        self.generation = _GENERATION[0]   # distinguishes arenas whose id() was reused (graph cache keys)
        self.comm = comm
        self.hidden = hidden
        self.rows = rows
        self.max_blocks = max_blocks
        bf = torch.bfloat16
        self.part = torch.zeros(rows, hidden, dtype=bf, device=device)
        self.x = torch.zeros(rows, hidden, dtype=bf, device=device)
        self.h = torch.zeros(rows, hidden, dtype=bf, device=device)
        self.sig = torch.zeros(ops.tp_signal_bytes() // 4, dtype=torch.int32, device=device)
        # the LM head's argmax keys of every row (vocab-parallel greedy token)
        self.keys = torch.zeros(rows, dtype=torch.int64, device=device)
        # folded-norm layout: per-row fp32 sum of squares of x (instead of h)
        self.ss = torch.zeros(max(rows, 4), dtype=torch.float32, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        torch.cuda.current_stream(device).synchronize()
        self._maps: list = []  # peer mappings live exactly as long as the arena
        self.addrs = {}
        mapped = True
        for k in ("part", "x", "h", "sig", "keys", "ss"):
            try:
                self.addrs[k] = comm.peer_addresses(getattr(self, k), self._maps)
            except _lib.SeesawKernelError as exc:  # e.g. no peer access between these GPUs
                warnings.warn(f"fused TP combine: peer mapping of {k!r} failed on rank {comm.rank} ({exc})",
                              RuntimeWarning, stacklevel=2)
                self.addrs[k] = [0] * comm.size
                mapped = False
        # every member agrees whether the mappings exist before any kernel
        # dereferences them (a rank that could not map must not leave its
        # peers waiting in the self-test's device barrier)
        flags = torch.tensor([1.0 if mapped else 0.0], device=device)
        comm.all_reduce_(flags)
        # the address tables as ctypes arrays, built once (a combine is
        # launched twice per layer)
        self._arrays = {k: _lib.uint64_array(v) for k, v in self.addrs.items()}
        if int(flags.item()) != comm.size:
            warnings.warn("fused TP combine: peer mappings unavailable on some rank; "
                          "falling back to all-reduce + rmsnorm", RuntimeWarning, stacklevel=2)
            self.usable = False
            return
        self.usable = self._self_test()

    def combine(self, rows: int, gamma: torch.Tensor | None, eps: float) -> None:
        """x[:rows], h[:rows] (if gamma) <- sum over ranks of part[:rows].
        A peer that misses the device barrier for 30 s sets the error word
        (checked by :meth:`check` at the engine's synchronisation points)
        instead of trapping the context.  The barrier epochs live on the
        device (epoch 0), so the call may be captured in a CUDA graph."""
        a = self.addrs
        ops.tp_allreduce_rmsnorm(a["part"], a["x"], a["h"] if gamma is not None else None, a["sig"],
                                 self.comm.rank, rows, self.hidden, gamma, eps, 0, self.max_blocks, self.err)

    def combine_ss(self, rows: int) -> None:
        """x[:rows] <- sum over ranks of part[:rows] and ss[:rows] <- the
        rows' sums of squares, on every rank (the folded-norm combine: the
        consumer GEMMs scale their rows by 1/rms from ss)."""
        a = self._arrays
        ops.tp_allreduce_rowss(a["part"], a["x"], a["ss"], a["sig"], self.comm.rank, rows, self.hidden, 0,
                               self.max_blocks, self.err)

    def argmax(self, rows: int, out_idx: torch.Tensor) -> None:
        """out_idx[:rows] <- greedy token of every row from the ranks' LM-head
        keys (keys[:rows], written by ops.lm_head_keys)."""
        ops.tp_argmax_keys(self.addrs["keys"], self.addrs["sig"], self.comm.rank, rows, out_idx, 0,
                           self.max_blocks, self.err)

    def check(self) -> None:
        """Raise if any combine since the last check timed out (host sync)."""
        torch.cuda.current_stream(self.err.device).synchronize()
        code = int(self.err.item())
        if code:
            self.err.zero_()
            raise SeesawKernelError(f"fused TP combine: peer barrier timed out (error word {code}) on rank "
                                        f"{self.comm.rank}; the TP group's peers stopped participating")

    def _self_test(self) -> bool:
        """Known answer: rank r's part = (r + 1) * ramp; x must be the exact
        bf16 of the fp32 sum, and h its rmsnorm (gamma = 1); the argmax of
        synthetic keys must pick every row's largest key."""
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
        self.combine(rows, gamma, 1e-5)
        ref_h = ops.rmsnorm(want, gamma, 1e-5)
        # argmax keys: rank p's key of row i = ((3i + 5p) % 7) << 32 | ~(100p + i)
        i = torch.arange(rows, device=dev, dtype=torch.int64)

        def key(p):
            return (((3 * i + 5 * p) % 7) << 32) | (0xFFFFFFFF - (100 * p + i))

        self.keys[:rows].copy_(key(r))
        best = torch.stack([key(p) for p in range(n)]).amax(0)
        want_idx = (0xFFFFFFFF - (best & 0xFFFFFFFF)).to(torch.int32)
        got_idx = torch.empty(rows, dtype=torch.int32, device=dev)
        self.argmax(rows, got_idx)
        # wait with the GIL released: virtual ranks (threads) must still be
        # able to launch their half of the barrier while this one waits
        torch.cuda.current_stream(dev).synchronize()
        ok_h = torch.equal(self.x[:rows], want) and torch.equal(self.h[:rows], ref_h)
        # the folded-norm variant: same x, and the rows' sums of squares
        self.x[:rows].zero_()
        self.combine_ss(rows)
        torch.cuda.current_stream(dev).synchronize()
        wf = want.float()
        ss_ref = (wf * wf).sum(-1)
        ok_ss = torch.equal(self.x[:rows], want) and bool(
            torch.allclose(self.ss[:rows], ss_ref, rtol=1e-5, atol=1e-6))
        ok = int(self.err.item()) == 0 and ok_h and ok_ss and torch.equal(got_idx, want_idx)
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
