"""Decode-step microbenchmark on the 8B shape (B=512, ctx 1024..), sweeping the
decode-lane overlap settings.  Pool contents are random (timing only)."""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_06433_b200 import PRESETS, ParallelismConfig  # noqa: E402
from paper_2503_06433_b200.comm import SoloComm  # noqa: E402
from paper_2503_06433_b200.runtime import Worker  # noqa: E402


def main(configs):
    arch = PRESETS["llama3-8b"]
    dev = torch.device("cuda", 0)
    B, ctx0, steps, BS = 512, 1024, 24, 64
    w = Worker(arch, SoloComm(), 1, dev, seed=0, max_pos=2048)
    w.init_weights(ParallelismConfig(1, 1, 1))
    nbps = (ctx0 + 256 + BS - 1) // BS
    w.alloc_pool(B * nbps)
    w.pool.view(torch.int16).random_(0, 1 << 13)  # small positive bf16 bit patterns
    tables = torch.arange(B * nbps, dtype=torch.int32, device=dev).view(B, nbps)
    out = []
    for lanes, cap in configs:
        w.decode_lanes, w.lane_gemm_cap = lanes, cap
        ctx = torch.full((B,), ctx0, dtype=torch.int32, device=dev)
        tok = torch.randint(0, arch.vocab, (B,), dtype=torch.int32, device=dev)
        pos = torch.empty(B, dtype=torch.int32, device=dev)
        slots = torch.empty(B, dtype=torch.int64, device=dev)
        nxt = torch.empty_like(tok)
        for _ in range(3):
            w.decode_step(tok, ctx, tables, pos, slots, nxt)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            w.decode_step(tok, ctx, tables, pos, slots, nxt)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / steps
        out.append({"lanes": lanes, "cap": cap, "ms_per_step": ms,
                    "env": {k: v for k, v in os.environ.items() if k.startswith("SSB_")}})
        print(json.dumps(out[-1]), flush=True)
    return out


if __name__ == "__main__":
    # --ab: the default single-lane step only (A/B of SSB_* switches across runs)
    cfgs = [(1, 0)] if "--ab" in sys.argv else [(1, 0), (2, 0), (2, 132), (2, 120), (2, 108), (2, 96)]
    main(cfgs)
