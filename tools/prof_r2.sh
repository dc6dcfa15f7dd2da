#!/usr/bin/env bash
# Round-2 kernel evidence on one GPU (run via gpurun): A/B of the decode step
# under SSB_* switches, and ncu --set full (source-level) captures of the
# prefill attention pair kernel and the M = 512 decode projections.
# Outputs under gpurun_out/prof2/.
set -u
OUT=gpurun_out/prof2
mkdir -p "$OUT"
what="${1:-all}"
if [[ "$what" == all || "$what" == ab ]]; then
  for rep in 1 2; do
    for v in 0 1; do
      SSB_GEMM_PREFETCH_B=$v timeout 300 python tools/bench_decode.py --ab >> "$OUT/ab_decode.jsonl" 2>> "$OUT/ab_decode.err"
    done
  done
fi
if [[ "$what" == abepi ]]; then
  for rep in 1 2 3; do
    for v in 0 1; do
      SSB_GEMM_EPI_PREFETCH=$v timeout 300 python tools/bench_decode.py --ab >> "$OUT/ab_decode_epi.jsonl" 2>> "$OUT/ab_decode.err"
    done
  done
fi
if [[ "$what" == attnab ]]; then
  for rep in 1 2; do
    for v in 0 1 3; do
      SSB_ATTN_ONLY0=1 SSB_ATTN_POLY=$v timeout 300 python tools/bench_kernels.py --what attn >> "$OUT/attn_ab.jsonl" 2>> "$OUT/attn_ab.err"
    done
  done
fi
if [[ "$what" == all || "$what" == attn ]]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attn -s 1 -c 1 \
      -o "$OUT/attn_pair" -f python tools/one_attn.py > "$OUT/attn_pair.stdout" 2>&1
fi
if [[ "$what" == all || "$what" == gemm ]]; then
  for shape in "512 4096 4096" "512 6144 4096" "512 4096 14336"; do
    tag=$(echo $shape | tr ' ' _)
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 1 -c 1 \
        -o "$OUT/gemm_$tag" -f python tools/one_gemm.py $shape > "$OUT/gemm_$tag.stdout" 2>&1
  done
fi
ls -la "$OUT"
