"""Fused TP combine over peer memory (csrc/tp_allreduce.cu, tpcombine.py):
the row-parallel all-reduce + the following RMSNorm in one kernel with a
device-side barrier between the ranks.

Runs W virtual ranks as threads on one GPU, each on its own CUDA stream (the
kernels of all ranks are co-resident, exactly as on W GPUs), and checks
against the unfused path bit for bit: x = bf16(fp32 sum of the partials in
rank order) — the order ThreadComm.all_reduce_ uses — and h = ssb_rmsnorm(x).
Several calls in a row with new data each time exercise the epoch barriers
and the buffer-reuse ordering (a rank overwriting its partials for call e+1
while a slow peer could still be reading call e)."""

from __future__ import annotations

import pytest
import torch

from paper_2503_06433_b200._lib import SeesawKernelError

from paper_2503_06433_b200 import ops
from paper_2503_06433_b200.comm import ThreadComm
from paper_2503_06433_b200.tpcombine import PeerArena
from test_engine_gpu import run_threads

pytestmark = pytest.mark.gpu


def _partial(seed: int, rank: int, rows: int, hidden: int, dev) -> torch.Tensor:
    # generated on the device: a pageable host->device copy would make the
    # calling thread wait for its stream, i.e. for the peers' barrier, while
    # holding up its own next launch (an artefact of threads sharing a GPU)
    g = torch.Generator(device=dev).manual_seed(seed * 1000 + rank)
    return (torch.randn(rows, hidden, generator=g, device=dev) * (rank + 1)).to(torch.bfloat16)


@pytest.mark.parametrize("W,rows,hidden", [(2, 1, 256), (2, 300, 4096), (4, 7, 5120), (4, 64, 8192), (8, 513, 4096),
                                           (3, 100, 1024)])
def test_combine_bit_exact(cuda, W, rows, hidden):
    comms = ThreadComm.create(W)
    calls = 4

    def body(r):
        dev = torch.device("cuda", 0)
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            ar = PeerArena(comms[r], dev, hidden, max(rows, 8), max_blocks=16)
            assert ar.usable
            gamma = (torch.rand(hidden, generator=torch.Generator(device=dev).manual_seed(7), device=dev)
                     + 0.5).to(torch.bfloat16)
            parts = [_partial(c, r, rows, hidden, dev) for c in range(calls)]
            outs = []
            for c in range(calls):
                ar.part[:rows].copy_(parts[c])
                ar.combine(rows, gamma if c % 2 == 0 else None, 1e-5)
                outs.append((ar.x[:rows].clone(), ar.h[:rows].clone() if c % 2 == 0 else None))
            s.synchronize()
            assert int(ar.err.item()) == 0
            return outs, gamma

    res = run_threads(W, body)
    dev = torch.device("cuda", 0)
    gamma = res[0][1]
    for c in range(calls):
        acc = _partial(c, 0, rows, hidden, dev).float()
        for p in range(1, W):
            acc += _partial(c, p, rows, hidden, dev).float()
        want_x = acc.to(torch.bfloat16)
        want_h = ops.rmsnorm(want_x, gamma, 1e-5) if c % 2 == 0 else None
        for r in range(W):
            x, h = res[r][0][c]
            assert torch.equal(x, want_x), (c, r)
            if want_h is not None:
                assert torch.equal(h, want_h), (c, r)


def test_missing_peer_times_out_instead_of_hanging(cuda):
    """Rank 1 never calls: rank 0's barrier gives up after the timeout and
    reports through the error word (the self-test's fallback signal)."""
    comms = ThreadComm.create(2)

    def body(r):
        dev = torch.device("cuda", 0)
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            ar = PeerArena(comms[r], dev, 256, 8, max_blocks=4)
            comms[r].barrier()
            if r == 0:
                ar.combine(8, None, 1e-5)
                s.synchronize()
                code = int(ar.err.item())
                with pytest.raises(SeesawKernelError, match="peer barrier timed out"):
                    ar.check()
                ar.check()  # the error word was consumed
                return code
            return 0

    assert run_threads(2, body)[0] == 1


def test_failed_peer_mapping_falls_back_on_every_rank(cuda):
    """A rank that cannot map a peer buffer (no peer access between two GPUs,
    an IPC failure) must not leave its peers in the self-test's device
    barrier: all members agree on the failure first, and every rank ends up
    with an unusable arena (the caller falls back to all-reduce + rmsnorm)."""
    comms = ThreadComm.create(2)
    real = ThreadComm.peer_addresses

    def flaky(self, t, keep):
        # the handle exchange (a collective) completes, then rank 1's open
        # fails -- where TorchComm.peer_addresses can fail
        addrs = real(self, t, keep)
        if self.rank == 1:
            raise SeesawKernelError("simulated ssb_ipc_open failure")
        return addrs

    def body(r):
        dev = torch.device("cuda", 0)
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            comms[r].peer_addresses = flaky.__get__(comms[r])
            ar = PeerArena(comms[r], dev, 256, 8, max_blocks=16)  # warns (RuntimeWarning) on both ranks
            return ar.usable

    assert run_threads(2, body) == [False, False]
