"""The SPMD engine as REAL processes: two torch.distributed ranks (gloo, CUDA
tensors staged through host memory by TorchComm) sharing the one GPU of the
test box, running execute() on the tiny config PP2 -> TP2 — once with every
sequence resident and once with the pinned host KV tier, whose buffer is
POSIX shared memory mapped and cudaHostRegister'ed by both processes.

This is the process-level path bench.py takes under torchrun on a multi-GPU
box (TorchComm groups, send/recv between PP stages, all-to-all re-shard,
TP all-reduce / all-gather, shared host tier) with NCCL replaced by gloo:
every rank must finish, the event log must pass replay_check and the greedy
tokens must match the CPU oracle (the ThreadComm runs of test_engine_gpu.py
check the same against one process).
"""

from __future__ import annotations

import os
import pickle
import socket
import tempfile

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _rank(rank: int, port: int, outdir: str, tiered: bool, p2p: bool = False, fused_tp: bool = False) -> None:
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import torch.distributed as dist

    from paper_2503_06433_b200 import PRESETS, execute, replay_check
    from paper_2503_06433_b200.comm import TorchComm
    from paper_2503_06433_b200.engine import synthetic_prompts
    from paper_2503_06433_b200.report import SchedulingPolicy
    from paper_2503_06433_b200.runtime import Worker
    from paper_2503_06433_b200.specs import ParallelismConfig, Request, kv_bytes_per_token, total_weight_bytes
    from test_engine_gpu import tiny_hw

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    arch = PRESETS["tiny"]
    model = arch.model_spec()
    n_req, s_in, s_out = 8, 64, 32
    hw = tiny_hw(2)
    if tiered:
        k = (s_in + s_out) * kv_bytes_per_token(model)
        hw = tiny_hw(2, gpu_memory=(total_weight_bytes(model) + 3 * k) / 2, host_memory_per_gpu=n_req * k / 2)
    reqs = [Request(i, s_in, s_out) for i in range(n_req)]
    prompts = synthetic_prompts(reqs, arch.vocab)
    comm = TorchComm()
    wk = Worker(arch, comm, 1, dev, seed=0, max_pos=256)
    wk.p2p_reshard = p2p
    wk.fused_tp = fused_tp
    rep = execute(model, hw, reqs, SchedulingPolicy.TRANSITION_MINIMIZING, ParallelismConfig(1, 2, 1),
                  ParallelismConfig(2, 1, 1), arch=arch, prompts=prompts, comm=comm, device=dev, worker=wk)
    torch.cuda.synchronize()
    kinds: dict = {}
    for e in rep.event_log:
        kinds[e.kind] = kinds.get(e.kind, 0) + 1
    with open(f"{outdir}/rank{rank}.pkl", "wb") as fh:
        pickle.dump({"outputs": rep.outputs, "replay": bool(replay_check(rep)), "kinds": kinds,
                     "transitions": rep.transitions, "host_tier": rep.config["host_tier"],
                     "sent": rep.measured["reshard_bytes_sent"],
                     "fused": bool(wk._tp_arenas) and all(a.usable for a in wk._tp_arenas.values())}, fh)
    dist.barrier()
    dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("tiered,p2p,fused_tp", [(False, False, False), (True, False, False), (False, True, False),
                                                (False, False, True)])
def test_two_process_pp2_tp2(cuda, tiered, p2p, fused_tp):
    """(p2p: the KV re-shard's pack kernel stores straight into the other
    process's receive buffer through a CUDA IPC mapping.  fused_tp: the TP
    decode combine is the peer-memory kernel with its device-side barrier,
    across two processes — their contexts time-slice the one GPU, so every
    barrier waits for a context switch: slow, but it exercises the
    cross-process IPC mappings and flag ordering.)"""
    from paper_2503_06433_b200 import PRESETS
    from paper_2503_06433_b200.engine import synthetic_prompts
    from paper_2503_06433_b200.specs import Request
    from test_engine_gpu import check_greedy

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank, args=(_free_port(), d, tiered, p2p, fused_tp), nprocs=2, join=True)
        res = [pickle.load(open(f"{d}/rank{r}.pkl", "rb")) for r in range(2)]
    for r in res:
        assert r["replay"] and r["transitions"] == 1 and r["host_tier"] == tiered
        assert r["kinds"]["prefill_complete"] == 8 and r["kinds"]["kv_release"] == 8
        assert r["sent"] > 0
        assert r["fused"] == fused_tp
    if tiered:
        assert res[0]["kinds"]["swap_in_complete"] == res[0]["kinds"]["swap_out_complete"] >= 1
    # both ranks of the replica produce the same tokens; they match the oracle
    assert res[0]["outputs"] == res[1]["outputs"]
    arch = PRESETS["tiny"]
    reqs = [Request(i, 64, 32) for i in range(8)]
    # the fused decode combine runs with the folded norm (SSB_TP_FOLD=1)
    # (the folded norm moves h's bf16 rounding into the fp32 accumulator:
    # genuine ties, margins < 0.02, may flip on up to 2 % of the steps)
    check_greedy(arch, reqs, synthetic_prompts(reqs, arch.vocab), res[0]["outputs"], 1, 2, pp_prefill=2,
                 tp_fold=fused_tp, max_subs=(len(reqs) * 32) // 50 if fused_tp else None)
