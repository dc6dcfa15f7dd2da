#!/usr/bin/env bash
# ncu evidence for the bench workload (run on the GPU box via gpurun).
#   1. launch list (per-launch device time) of ONE batch of a reduced bench
#      (64 prompts x 1024/32: the full 512x1024/256 batch is ~75k launches,
#      too many to replay under ncu; kernel SHARES are what must agree)
#   2. ncu --set full of the top kernels (tcgen05 GEMM, decode attention,
#      prefill attention) for dram bytes / tensor-pipe utilisation.
set -u
OUT=gpurun_out/prof
mkdir -p "$OUT"
SMALL="python bench.py --prompts 64 --output-len 32 --steps 1 --warmup 3 --no-cpu-baseline"
# 3 warm-up batches of 9392 launches each are skipped
ncu --metrics gpu__time_duration.sum --clock-control none -s 28176 -c 9392 --csv \
    --log-file "$OUT/launches.csv" $SMALL > "$OUT/launches.stdout" 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 300 -c 3 \
    -o "$OUT/gemm" $SMALL > "$OUT/gemm.stdout" 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 40 -c 2 \
    -o "$OUT/decode_attn" $SMALL > "$OUT/decode_attn.stdout" 2>&1
ncu --set full --clock-control none --import-source on -k regex:prefill_attn -s 40 -c 1 \
    -o "$OUT/prefill_attn" $SMALL > "$OUT/prefill_attn.stdout" 2>&1
ls -la "$OUT"
