"""Sustained (power-capped) throughput of the Llama-3-8B prefill projections:
the four GEMMs of one layer at M = 16384 packed tokens, looped for several
seconds, CUDA-event timed, with nvidia-smi clocks sampled meanwhile.  Used to
compare L2 cache-policy variants of the operand loads (SSB_GEMM_POLICY),
whose DRAM traffic changes the power budget left for the SM clock.

    SSB_GEMM_POLICY=1 python tools/gemm_sustained.py [--seconds 6]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_06433_b200 import ops  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=6.0)
    ap.add_argument("--M", type=int, default=16384)
    args = ap.parse_args()
    M, H, F, QKV = args.M, 4096, 14336, 6144
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(M, H, device=dev, generator=g).to(torch.bfloat16)
    wqkv = (torch.randn(QKV, H, device=dev, generator=g) / 64).to(torch.bfloat16)
    wo = (torch.randn(H, H, device=dev, generator=g) / 64).to(torch.bfloat16)
    w13 = (torch.randn(2 * F, H, device=dev, generator=g) / 64).to(torch.bfloat16)
    w2 = (torch.randn(H, F, device=dev, generator=g) / 120).to(torch.bfloat16)
    qkv = torch.empty(M, QKV, device=dev, dtype=torch.bfloat16)
    act = torch.empty(M, F, device=dev, dtype=torch.bfloat16)
    out = torch.empty(M, H, device=dev, dtype=torch.bfloat16)
    flops = 2.0 * M * H * (QKV + H + 2 * F) + 2.0 * M * F * H

    def layer():
        ops.gemm(x, wqkv, out=qkv)
        ops.gemm(qkv[:, :H], wo, out=out, residual=x)
        ops.gemm(x, w13, out=act, silu_mul=True)
        ops.gemm(act, w2, out=out, residual=x)

    for _ in range(5):
        layer()
    torch.cuda.synchronize()
    # iterations for ~args.seconds
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        layer()
    e.record()
    torch.cuda.synchronize()
    per = s.elapsed_time(e) / 10 / 1e3
    iters = max(10, int(args.seconds / per))
    smi = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "200"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    s.record()
    for _ in range(iters):
        layer()
    e.record()
    torch.cuda.synchronize()
    smi.terminate()
    rows = [ln.split(",") for ln in smi.communicate()[0].splitlines() if ln.strip()]
    clk = sorted(float(r[0]) for r in rows if len(r) > 1)
    pw = sorted(float(r[1]) for r in rows if len(r) > 1)
    t = s.elapsed_time(e) / 1e3
    print(json.dumps({"policy": int(os.environ.get("SSB_GEMM_POLICY", "0")), "M": M, "iters": iters, "s": t,
                      "tflops": flops * iters / t / 1e12,
                      "sm_mhz_median": clk[len(clk) // 2] if clk else None,
                      "power_w_median": pw[len(pw) // 2] if pw else None}), flush=True)


if __name__ == "__main__":
    main()
