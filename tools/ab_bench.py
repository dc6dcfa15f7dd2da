"""A/B of engine features on ONE box in ONE process (box-to-box clock
variance under the power cap is larger than most single-feature effects):
full bench batches (8B, 512 x 1024/256, N=1) with one feature toggled at a
time, interleaved A B C ... A B C ..., device-timed.

    python tools/ab_bench.py [--reps 2] [--prompts 512]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--prompts", type=int, default=512)
    ap.add_argument("--output-len", type=int, default=256)
    ap.add_argument("--configs", default="base,no_rope_fusion,no_argmax_fusion,no_split_k,attn_per_tile_ctas")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    from paper_2503_06433_b200 import PRESETS, ParallelismConfig, Request, SchedulingPolicy, execute, ops
    from paper_2503_06433_b200.comm import SoloComm
    from paper_2503_06433_b200.engine import synthetic_prompts
    from paper_2503_06433_b200.runtime import Worker
    from paper_2503_06433_b200.specs import HardwareSpec, RingAllReduce

    dev = torch.device("cuda", 0)
    arch = PRESETS["llama3-8b"]
    model = arch.model_spec()
    hw = HardwareSpec(1, 6.65e12, 1.59e15, 180e9, 256e9, 64e9, RingAllReduce(770e9))
    cfg = ParallelismConfig(1, 1, 1)
    reqs = [Request(i, 1024, args.output_len) for i in range(args.prompts)]
    prompts = [torch.from_numpy(p).to(dev) for p in synthetic_prompts(reqs, arch.vocab)]
    w = Worker(arch, SoloComm(), 1, dev, seed=0, max_pos=1024 + args.output_len + 64)

    def setc(name):
        w.fuse_rope = name != "no_rope_fusion"
        w.fuse_argmax = name != "no_argmax_fusion"
        w.split_k = name != "no_split_k"
        w.fold_norm = name != "no_fold_norm"
        ops._PREFILL_VARIANT = 2 if name == "attn_per_tile_ctas" else 0
        state["prefill_tokens"] = {"prefill_8k": 8192, "prefill_32k": 32768}.get(name, 16384)

    state = {"prefill_tokens": 16384}

    def batch():
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        rep = execute(model, hw, reqs, SchedulingPolicy.TRANSITION_MINIMIZING, cfg, cfg, arch=arch, prompts=prompts,
                      comm=SoloComm(), device=dev, worker=w, max_prefill_tokens=state["prefill_tokens"])
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / 1e3, rep

    names = args.configs.split(",")
    setc("base")
    batch()
    batch()
    res = {n: [] for n in names}
    for _ in range(args.reps):
        for n in names:
            setc(n)
            t, rep = batch()
            res[n].append({"s": t, "prefill_s": rep.prefill_time, "decode_s": rep.decode_time})
    base = sum(r["s"] for r in res["base"]) / args.reps
    for n in names:
        m = sum(r["s"] for r in res[n]) / args.reps
        print(json.dumps({"tag": args.tag, "config": n, "mean_s": m, "vs_base": m / base,
                          "tokens_per_s": args.prompts * args.output_len / m, "runs": res[n]}), flush=True)


if __name__ == "__main__":
    main()
