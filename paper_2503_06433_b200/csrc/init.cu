// Deterministic, counter-based weight initialisation (no host RNG, no state).
//
// Every element of a LOGICAL (unsharded) parameter is a pure function of
// (seed, tensor_id, row * full_cols + col), so any shard of any layout can be
// generated in place on its GPU without materialising the full model, and the
// CPU oracle (oracle/llama.py) reproduces the same bf16 bits with numpy.
//
//   key  = mix64(seed * G + tensor_id)                 G = 0x9E3779B97F4A7C15
//   a, b = mix64(key + (2i+1) G), mix64(key + (2i+2) G)
//   u0..u3 = 24-bit fields (a>>40, (a>>8)&M, b>>40, (b>>8)&M) * 2^-24
//   x    = (((u0+u1)+u2)+u3 - 2) * sqrt(3) * scale     (Irwin-Hall(4) ~ N(0,1))
//   bf16 = round-to-nearest-even(x); scale == 0 means the constant 1.0.
#include "common.cuh"
#include "seesaw_b200.h"

namespace ssb {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float init_value(uint64_t key, uint64_t i, float scale) {
  if (scale == 0.0f) return 1.0f;
  const uint64_t a = mix64(key + (2 * i + 1) * kGolden);
  const uint64_t b = mix64(key + (2 * i + 2) * kGolden);
  const float k = 5.9604644775390625e-08f;  // 2^-24
  const float u0 = __fmul_rn(static_cast<float>(static_cast<uint32_t>(a >> 40)), k);
  const float u1 = __fmul_rn(static_cast<float>(static_cast<uint32_t>((a >> 8) & 0xFFFFFFu)), k);
  const float u2 = __fmul_rn(static_cast<float>(static_cast<uint32_t>(b >> 40)), k);
  const float u3 = __fmul_rn(static_cast<float>(static_cast<uint32_t>((b >> 8) & 0xFFFFFFu)), k);
  const float s = __fadd_rn(__fadd_rn(__fadd_rn(u0, u1), u2), u3);
  return __fmul_rn(__fmul_rn(__fsub_rn(s, 2.0f), 1.7320508075688772f), scale);
}

constexpr int kInitThreads = 256;
constexpr int64_t kInitChunk = 16384;  // elements per CTA

__global__ void __launch_bounds__(kInitThreads)
    init_kernel(__nv_bfloat16* __restrict__ arena, const ssb_init_seg* __restrict__ segs, int n_seg,
                int64_t total, uint64_t seed) {
  const int64_t begin = static_cast<int64_t>(blockIdx.x) * kInitChunk;
  const int64_t end = min(begin + kInitChunk, total);
  __shared__ int s_first;
  if (threadIdx.x == 0) {
    int lo = 0, hi = n_seg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (segs[mid].cum_elems <= begin) lo = mid; else hi = mid - 1;
    }
    s_first = lo;
  }
  __syncthreads();
  int d = s_first;
  ssb_init_seg cur = segs[d];
  int64_t cur_end = cur.cum_elems + static_cast<int64_t>(cur.rows) * cur.cols;
  uint64_t key = mix64(seed * kGolden + static_cast<uint64_t>(cur.tensor_id));
  for (int64_t x = begin + threadIdx.x; x < end; x += blockDim.x) {
    while (x >= cur_end) {
      cur = segs[++d];
      cur_end = cur.cum_elems + static_cast<int64_t>(cur.rows) * cur.cols;
      key = mix64(seed * kGolden + static_cast<uint64_t>(cur.tensor_id));
    }
    const int64_t lin = x - cur.cum_elems;
    const int64_t r = lin / cur.cols;
    const int64_t c = lin - r * cur.cols;
    const uint64_t idx = static_cast<uint64_t>(cur.row0 + r) * static_cast<uint64_t>(cur.full_cols) +
                         static_cast<uint64_t>(cur.col0 + c);
    arena[cur.dst_off + r * cur.ld + c] = __float2bfloat16_rn(init_value(key, idx, cur.scale));
  }
}

}  // namespace
}  // namespace ssb

extern "C" int ssb_init_weights(void* arena, const ssb_init_seg* segs, int n_seg, int64_t total_elems,
                                uint64_t seed, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(n_seg >= 0 && total_elems >= 0, "ssb_init_weights: negative sizes");
  if (n_seg == 0 || total_elems == 0) return 0;
  SSB_REQUIRE(arena && segs, "ssb_init_weights: null pointer");
  const int64_t blocks = (total_elems + kInitChunk - 1) / kInitChunk;
  SSB_REQUIRE(blocks < (1ll << 31), "ssb_init_weights: too large");
  init_kernel<<<static_cast<int>(blocks), kInitThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<__nv_bfloat16*>(arena), segs, n_seg, total_elems, seed);
  return check_launch("ssb_init_weights");
}
