#!/usr/bin/env bash
# In-situ plan sweep of the M = 512 decode projections (8B, TP1): the whole
# decode step (tools/bench_decode.py --ab, CUDA-graph replay) timed with one
# shape's plan forced through SSB_GEMM_PLAN.  Lines -> gpurun_out/prof2/plan_sweep.jsonl
set -u
OUT=gpurun_out/prof2
mkdir -p "$OUT"
run() { SSB_GEMM_PLAN="$1" timeout 300 python tools/bench_decode.py --ab >> "$OUT/plan_sweep.jsonl" 2>> "$OUT/plan_sweep.err"; }
run ""
for p in 0:128:1 2:128:1 0:192:1 2:192:1 2:256:2 0:256:2 0:128:2 2:128:2; do run "512,4096,4096=$p"; done
for p in 2:256:1 0:128:1 2:128:1 0:256:1 2:256:2 0:128:2 2:128:2; do run "512,6144,4096=$p"; done
for p in 2:256:2 2:256:3 2:256:4 2:128:1 2:128:2 0:128:2 0:256:2 2:192:2 2:256:1; do run "512,4096,14336=$p"; done
for p in 2:256:1 2:192:1 2:128:1 0:256:1; do run "512,28672,4096=$p"; done
run ""
