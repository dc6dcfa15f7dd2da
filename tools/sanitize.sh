#!/usr/bin/env bash
# compute-sanitizer over the kernel tests (run on the GPU box via gpurun):
# memcheck, racecheck (shared-memory hazards) and synccheck (barrier misuse)
# on the tcgen05 GEMM (plain, split-K, fused epilogues), both attention
# kernels, the KV re-shard pack/unpack and the fused TP combine.  One small
# parametrisation per kernel keeps each tool's run within minutes.
# Output: gpurun_out/sanitize/<tool>.log, summarised in profiles/r02/sanitizer.md.
set -u
OUT=gpurun_out/sanitize
mkdir -p "$OUT"
SEL=(
  "tests/test_gemm_gpu.py::test_gemm_plain[300-384-1024-128]"
  "tests/test_gemm_gpu.py::test_gemm_plain[300-200-136-224]"
  "tests/test_gemm_gpu.py::test_gemm_silu_mul[128]"
  "tests/test_gemm_gpu.py::test_gemm_split_k[300-640-1000-192-3-single]"
  "tests/test_gemm_gpu.py::test_gemm_split_k[300-640-1000-192-3-2sm]"
  "tests/test_kernels_gpu.py::test_qkv_gemm_rope_kv_fused_bit_exact[129-4-1-1024-True-split3_2sm]"
  "tests/test_kernels_gpu.py::test_lm_head_argmax_fused[129-4000-1024]"
  "tests/test_rownorm_gpu.py::test_producer_row_sums_of_squares[300-4096-1024-128]"
  "tests/test_rownorm_gpu.py::test_consumer_row_scale[77-1024-4096]"
  "tests/test_kernels_gpu.py::test_prefill_attention[128-8-2-lens0-0]"
  "tests/test_kernels_gpu.py::test_prefill_attention[128-4-4-lens3-0]"
  "tests/test_kernels_gpu.py::test_decode_attention_paged[128-4-1-ctxs2]"
  "tests/test_kernels_gpu.py::test_decode_attention_paged[64-4-4-ctxs1]"
  "tests/test_reshard_gpu.py::test_kv_reshard_virtual_world[4-4-src3-dst3]"
  "tests/test_tpcombine_gpu.py::test_combine_bit_exact[3-100-1024]"
)
for tool in ${SSB_SANITIZE_TOOLS:-memcheck racecheck synccheck}; do
  for t in "${SEL[@]}"; do
    name=$(echo "$t" | tr '/:.' '___')
    timeout 600 compute-sanitizer --tool "$tool" --error-exitcode 99 --print-limit 20 \
        --log-file "$OUT/${tool}_${name}.log" \
        python -m pytest -q -x -p no:cacheprovider "$t" \
        > "$OUT/${tool}_${name}.stdout" 2>&1
    echo "$tool $t rc=$?" | tee -a "$OUT/summary.txt"
  done
done
