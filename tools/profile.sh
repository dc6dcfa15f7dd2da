#!/usr/bin/env bash
# ncu evidence for the bench workload (run on the GPU box via gpurun, 1 GPU).
# Every capture is of the bench command itself, restricted with NVTX to the
# launches of ONE timed batch (range "timed_step"; bench.py pushes it around
# each timed step), so shares and per-launch numbers refer to the measured
# workload.  Outputs under gpurun_out/prof/ (summarised into profiles/ by
# tools/summarise_profiles.py).
set -u
OUT=gpurun_out/prof
mkdir -p "$OUT"
BENCH="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
NV="--nvtx --nvtx-include timed_step/"
what="${1:-all}"
if [[ "$what" == all || "$what" == launches ]]; then
  # 1. launch list: per-launch device time of every kernel of one timed batch.
  #    ncu serialises and replays every launch (~25 ms each); the full batch
  #    (~60k launches) does not fit a call, so the list is taken on the same
  #    command with 64 prompts x 1024/32 (same kernels and shapes in prefill;
  #    decode at batch 64) -- kernel SHARES are what it is compared on
  timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none $NV --csv \
      --log-file "$OUT/launches.csv" $BENCH --prompts 64 --output-len 32 > "$OUT/launches.stdout" 2>&1
  gzip -f "$OUT/launches.csv"
fi
if [[ "$what" == all || "$what" == full ]]; then
  # 2. --set full of the dominant kernels (first launches inside the timed batch)
  #    prefill projections of layer 0 (QKV, O, gate_up, down)
  timeout 900 ncu --set full --clock-control none --import-source on $NV -k regex:gemm_bf16 -c 4 \
      -o "$OUT/gemm_prefill" $BENCH > "$OUT/gemm_prefill.stdout" 2>&1
  #    decode projections of the first decode step's layer 0 (after 32x32x4 prefill GEMMs + 32 lm_head)
  timeout 900 ncu --set full --clock-control none --import-source on $NV -k regex:gemm_bf16 -s 4128 -c 4 \
      -o "$OUT/gemm_decode" $BENCH > "$OUT/gemm_decode.stdout" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on $NV -k regex:decode_attn -s 100 -c 2 \
      -o "$OUT/decode_attn" $BENCH > "$OUT/decode_attn.stdout" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on $NV -k regex:prefill_attn -s 40 -c 2 \
      -o "$OUT/prefill_attn" $BENCH > "$OUT/prefill_attn.stdout" 2>&1
fi
ls -la "$OUT"
