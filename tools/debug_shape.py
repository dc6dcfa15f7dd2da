"""Debug a 2-layer model shape through PP2 -> TP2 on one GPU: after the
transition, compare each rank's re-partitioned weight arena with a fresh
init of the TP layout (must be bit-identical) and the KV pool with the
oracle re-layout, then report NaNs in the decode logits."""

from __future__ import annotations

import dataclasses
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import kv_layout as kvo  # noqa: E402
from paper_2503_06433_b200 import PRESETS, execute  # noqa: E402
from paper_2503_06433_b200.comm import SoloComm, ThreadComm  # noqa: E402
from paper_2503_06433_b200.engine import synthetic_prompts  # noqa: E402
from paper_2503_06433_b200.report import SchedulingPolicy  # noqa: E402
from paper_2503_06433_b200.runtime import Worker  # noqa: E402
from paper_2503_06433_b200.specs import HardwareSpec, ParallelismConfig, Request, RingAllReduce  # noqa: E402
from test_engine_gpu import run_threads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"
arch = dataclasses.replace(PRESETS[name], num_layers=2, name=name + "-2l")
cfg_p, cfg_d = ParallelismConfig(1, 2, 1), ParallelismConfig(2, 1, 1)
reqs = [Request(i, 96, 6) for i in range(3)]
prompts = synthetic_prompts(reqs, arch.vocab)
hw = HardwareSpec(2, 8e12, 2.25e15, 150e9, 8e9, 64e9, RingAllReduce(9e11))
comms = ThreadComm.create(2)
snaps = {}


def body(r):
    dev = torch.device("cuda", 0)
    wk = Worker(arch, comms[r], 1, dev, seed=0, max_pos=256)

    def before(w, blocks, cfg_to):
        snaps[(r, "pool_before")] = (w.pool.detach().cpu().clone(), blocks.copy())

    def after(w, blocks, cfg_to):
        torch.cuda.synchronize()
        snaps[(r, "pool_after")] = w.pool.detach().cpu().clone()
        snaps[(r, "arena")] = w.state.arena.detach().cpu().clone()

    wk.hooks = {"before_reshard": before, "after_reshard": after}
    rep = execute(arch.model_spec(), hw, reqs, SchedulingPolicy.TRANSITION_MINIMIZING, cfg_p, cfg_d, arch=arch,
                  prompts=prompts, comm=comms[r], device=dev, worker=wk, record_logits=True)
    torch.cuda.synchronize()
    return rep, [l.clone() for l in wk.logit_log]


res = run_threads(2, body)
for r in range(2):
    fresh = Worker(arch, SoloComm(), 1, torch.device("cuda", 0), seed=0, max_pos=64)
    fresh.per_replica, fresh.gpu = 2, r
    fresh.init_weights(cfg_d)
    torch.cuda.synchronize()
    exp = fresh.state.arena.cpu()
    got = snaps[(r, "arena")]
    bad = (exp.view(torch.int16) != got.view(torch.int16)).nonzero()
    print(f"rank {r}: arena mismatches {bad.numel()} / {exp.numel()}")
    if bad.numel():
        for t in fresh.state.weights.tensors.values():
            seg = (exp[t.offset:t.offset + t.numel].view(torch.int16) != got[t.offset:t.offset + t.numel].view(torch.int16)).sum().item()
            if seg:
                print("   tensor", t.key, "mismatches", seg, "of", t.numel)
    del fresh
L, H, D, BS = arch.num_layers, arch.num_kv_heads, arch.head_dim, 64
pools = [snaps[(r, "pool_before")][0].view(torch.int16).numpy().reshape(-1, L // 2, 2, H, BS, D) for r in range(2)]
blocks = snaps[(0, "pool_before")][1]
exp = kvo.reshard_pools(pools, L, H, (1, 2), (2, 1), blocks=blocks)
for r in range(2):
    got = snaps[(r, "pool_after")].view(torch.int16).numpy().reshape(exp[r].shape)
    print(f"rank {r}: kv mismatches {(got[blocks] != exp[r][blocks]).sum()}")
for r in range(2):
    logs = res[r][1]
    print(f"rank {r}: logit tensors {len(logs)}; NaN per tensor {[int(torch.isnan(l).sum()) for l in logs]}")
print("outputs", res[0][0].outputs)
