"""Host overhead of one TP8 decode step, measured on one GPU (VERDICT r1
"Next round" 4).

A TP8 rank of Llama-3-8B decodes with 4 query heads, 1 KV head, ffn 1,792 and
a vocabulary slice of 16,032 at M = 512 rows: ~2-3 ms of GPU work per step, so
the ~5L+10 library launches of a step (each a ctypes call through a Python
wrapper) can become the bound.  This tool builds exactly those rank-local
shapes as a single-GPU model (the TP combine's two launches per layer are the
only kernels a real TP8 rank adds; they are not run here) and reports, with
and without CUDA-graph replay of the step:

  gpu_ms   device time per step (CUDA events around S back-to-back steps)
  host_ms  host time spent issuing one step (perf_counter around the
           decode_step calls; the GPU queue is kept non-empty)
  host/gpu the fraction the VERDICT asks to bring under 30 %

Run on the GPU box:  python tools/bench_tp8_host.py [--steps 64]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_06433_b200 import ParallelismConfig  # noqa: E402
from paper_2503_06433_b200.arch import LlamaArch  # noqa: E402
from paper_2503_06433_b200.comm import SoloComm  # noqa: E402
from paper_2503_06433_b200.runtime import Worker  # noqa: E402

# Llama-3-8B / TP8, one rank's shapes
RANK_LOCAL = LlamaArch("llama3-8b-tp8-rank", 32, 4096, 4, 1, 128, 14336 // 8, 128256 // 8, rope_theta=500000.0)


def run(graphs: bool, steps: int, B: int = 512, ctx0: int = 1024) -> dict:
    arch = RANK_LOCAL
    dev = torch.device("cuda", 0)
    BS = 64
    w = Worker(arch, SoloComm(), 1, dev, seed=0, max_pos=2048)
    w.cuda_graphs = graphs
    w.init_weights(ParallelismConfig(1, 1, 1))
    nbps = (ctx0 + steps + 8 + BS - 1) // BS
    w.alloc_pool(B * nbps)
    w.pool.view(torch.int16).random_(0, 1 << 13)
    tables = torch.arange(B * nbps, dtype=torch.int32, device=dev).view(B, nbps)
    ctx = torch.full((B,), ctx0, dtype=torch.int32, device=dev)
    tok = torch.randint(0, arch.vocab, (B,), dtype=torch.int32, device=dev)
    pos = torch.empty(B, dtype=torch.int32, device=dev)
    slots = torch.empty(B, dtype=torch.int64, device=dev)
    nxt = torch.empty_like(tok)
    for _ in range(4):  # eager, eager + capture, replays
        w.decode_step(tok, ctx, tables, pos, slots, nxt)
    torch.cuda.synchronize()
    ctx.fill_(ctx0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host = 0.0
    s.record()
    for _ in range(steps):
        t0 = time.perf_counter()
        w.decode_step(tok, ctx, tables, pos, slots, nxt)
        host += time.perf_counter() - t0
    e.record()
    torch.cuda.synchronize()
    gpu_ms = s.elapsed_time(e) / steps
    # steps with a host sync between them: the wall time a step costs when
    # nothing hides the issue time
    ctx.fill_(ctx0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        w.decode_step(tok, ctx, tables, pos, slots, nxt)
        torch.cuda.synchronize()
    wall_sync = (time.perf_counter() - t0) / steps * 1e3
    captured = sum(1 for v in w._graphs.values() if v["graph"] is not None)
    return {"graphs": graphs, "captured": captured, "B": B, "ctx": ctx0, "steps": steps,
            "gpu_ms_per_step": gpu_ms, "host_issue_ms_per_step": host / steps * 1e3,
            "host_over_gpu": host / steps * 1e3 / gpu_ms, "wall_ms_per_step_synced": wall_sync}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=64)
    args = ap.parse_args()
    for g in (False, True):
        print(json.dumps({"workload": "llama3-8b TP8 rank-local decode step (4 q heads, 1 kv head, ffn 1792, "
                                      "vocab 16032, M=512, ctx 1024)", **run(g, args.steps)}), flush=True)


if __name__ == "__main__":
    main()
