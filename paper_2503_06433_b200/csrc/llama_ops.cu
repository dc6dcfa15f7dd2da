// Memory-bound per-token ops of the Llama block: RMSNorm, RoPE + paged KV
// append, vocab-parallel embedding and vocab-parallel argmax.
//
// These have no reference counterpart (the reference's cost model ignores
// them); rounding points are fixed so the bf16-faithful
// CPU oracle (oracle/llama.py) can reproduce them: fp32 math with explicit
// _rn intrinsics where a contraction would change the result, one bf16
// rounding at the output.
#include <cstdlib>

#include "common.cuh"
#include "seesaw_b200.h"

namespace ssb {
namespace {

// ---------------------------------------------------------------- RMSNorm --
constexpr int kNormThreads = 256;

__global__ void __launch_bounds__(kNormThreads)
    rmsnorm_kernel(const __nv_bfloat16* __restrict__ x, int ldx, const int32_t* __restrict__ row_idx,
                   const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ out, int ldo, int hidden,
                   float eps) {
  griddep_launch_dependents();  // the next (PDL-launched) GEMM may start its prologue
  griddep_wait();               // PDL-launched itself: x is written by the previous kernel
  const int row = blockIdx.x;
  const int src_row = row_idx ? row_idx[row] : row;
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(src_row) * ldx);
  const int nvec = hidden / 8;
  float ss = 0.f;
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
    const uint4 v = xr[i];
    const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float a = bf16_lo(u[k]), b = bf16_hi(u[k]);
      ss = fmaf(a, a, ss);
      ss = fmaf(b, b, ss);
    }
  }
  __shared__ float red[kNormThreads / 32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < kNormThreads / 32 ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(__fadd_rn(__fdiv_rn(red[0], static_cast<float>(hidden)), eps));
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* orow = reinterpret_cast<uint4*>(out + static_cast<size_t>(row) * ldo);
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
    const uint4 v = xr[i];
    const uint4 g = wr[i];
    const uint32_t u[4] = {v.x, v.y, v.z, v.w};
    const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float a = __fmul_rn(__fmul_rn(bf16_lo(u[k]), inv), bf16_lo(gw[k]));
      const float b = __fmul_rn(__fmul_rn(bf16_hi(u[k]), inv), bf16_hi(gw[k]));
      o[k] = pack_bf16x2(a, b);
    }
    orow[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ------------------------------------------------------ RoPE + KV append --
constexpr int kRopeThreads = 128;

__global__ void __launch_bounds__(kRopeThreads)
    rope_append_kernel(__nv_bfloat16* __restrict__ qkv, int ld, int nq, int nk, int d,
                       const int32_t* __restrict__ pos, const float* __restrict__ tcos,
                       const float* __restrict__ tsin, int max_pos, __nv_bfloat16* __restrict__ pool,
                       ssb_kv_geometry geo, int layer, const int64_t* __restrict__ slots) {
  const int t = blockIdx.x;
  const int half = d / 2;
  const int p = min(max(pos[t], 0), max_pos - 1);
  const float* cr = tcos + static_cast<size_t>(p) * half;
  const float* sr = tsin + static_cast<size_t>(p) * half;
  __nv_bfloat16* row = qkv + static_cast<size_t>(t) * ld;
  const int64_t slot = slots ? slots[t] : -1;
  const int64_t blk = slot >= 0 ? slot / geo.block_size : 0;
  const int off = slot >= 0 ? static_cast<int>(slot - blk * geo.block_size) : 0;
  const int64_t plane = static_cast<int64_t>(geo.block_size) * d;  // one (kv, head) of a block
  __nv_bfloat16* kbase = pool + ((blk * geo.n_layers + layer) * 2 + 0) * geo.n_heads * plane;
  __nv_bfloat16* vbase = kbase + geo.n_heads * plane;
  // rotate q and k heads: pairs (i, i + d/2), two pairs per thread-step
  const int pairs2 = half / 2;
  for (int w = threadIdx.x; w < (nq + nk) * pairs2; w += blockDim.x) {
    const int h = w / pairs2;
    const int i = (w - h * pairs2) * 2;
    __nv_bfloat16* x = row + h * d;
    const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(x + i);
    const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(x + i + half);
    float y[4];
    const float c0 = cr[i], c1 = cr[i + 1], s0 = sr[i], s1 = sr[i + 1];
    const float a0 = __low2float(lo), a1 = __high2float(lo);
    const float b0 = __low2float(hi), b1 = __high2float(hi);
    y[0] = __fsub_rn(__fmul_rn(a0, c0), __fmul_rn(b0, s0));
    y[1] = __fsub_rn(__fmul_rn(a1, c1), __fmul_rn(b1, s1));
    y[2] = __fadd_rn(__fmul_rn(b0, c0), __fmul_rn(a0, s0));
    y[3] = __fadd_rn(__fmul_rn(b1, c1), __fmul_rn(a1, s1));
    const __nv_bfloat162 nlo = __floats2bfloat162_rn(y[0], y[1]);
    const __nv_bfloat162 nhi = __floats2bfloat162_rn(y[2], y[3]);
    *reinterpret_cast<__nv_bfloat162*>(x + i) = nlo;
    *reinterpret_cast<__nv_bfloat162*>(x + i + half) = nhi;
    if (h >= nq && slot >= 0) {
      __nv_bfloat16* dst = kbase + (h - nq) * plane + static_cast<int64_t>(off) * d;
      *reinterpret_cast<__nv_bfloat162*>(dst + i) = nlo;
      *reinterpret_cast<__nv_bfloat162*>(dst + i + half) = nhi;
    }
  }
  if (slot >= 0) {
    // v heads: straight copy, 16 bytes per thread-step
    const int vec_per_head = d / 8;
    for (int w = threadIdx.x; w < nk * vec_per_head; w += blockDim.x) {
      const int h = w / vec_per_head;
      const int c = (w - h * vec_per_head) * 8;
      const uint4 v = *reinterpret_cast<const uint4*>(row + (nq + nk + h) * d + c);
      *reinterpret_cast<uint4*>(vbase + h * plane + static_cast<int64_t>(off) * d + c) = v;
    }
  }
}

// --------------------------------------------------------------- embedding --
__global__ void __launch_bounds__(128)
    embedding_kernel(const int32_t* __restrict__ ids, const __nv_bfloat16* __restrict__ table,
                     int vocab_begin, int vocab_local, int hidden, __nv_bfloat16* __restrict__ out,
                     int ldo) {
  const int t = blockIdx.x;
  const int id = ids[t] - vocab_begin;
  uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(t) * ldo);
  const int nvec = hidden / 8;
  if (id >= 0 && id < vocab_local) {
    const uint4* src = reinterpret_cast<const uint4*>(table + static_cast<size_t>(id) * hidden);
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) dst[i] = src[i];
  } else {
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) dst[i] = make_uint4(0, 0, 0, 0);
  }
}

// ------------------------------------------------------------------ argmax --
constexpr int kArgThreads = 256;

__device__ __forceinline__ void arg_better(float& v, int& i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

__global__ void __launch_bounds__(kArgThreads)
    argmax_kernel(const float* __restrict__ logits, int ld, int cols, int base, float* __restrict__ ov,
                  int32_t* __restrict__ oi) {
  const int row = blockIdx.x;
  const float* r = logits + static_cast<size_t>(row) * ld;
  float best = -INFINITY;
  int bi = 0x7FFFFFFF;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) arg_better(best, bi, r[c], c);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    arg_better(best, bi, v2, i2);
  }
  __shared__ float sv[kArgThreads / 32];
  __shared__ int si[kArgThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kArgThreads / 32; ++w) arg_better(best, bi, sv[w], si[w]);
    ov[row] = best;
    oi[row] = base + bi;
  }
}

__global__ void argmax_combine_kernel(const float* __restrict__ vals, const int32_t* __restrict__ idxs,
                                      int parts, int rows, int32_t* __restrict__ out) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  float best = -INFINITY;
  int bi = 0x7FFFFFFF;
  for (int p = 0; p < parts; ++p) arg_better(best, bi, vals[p * rows + row], idxs[p * rows + row]);
  out[row] = bi;
}

__global__ void argmax_keys_kernel(const unsigned long long* __restrict__ keys, int rows, float* __restrict__ ov,
                                   int32_t* __restrict__ oi) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const unsigned long long k = keys[row];
  const uint32_t ord = static_cast<uint32_t>(k >> 32);
  const uint32_t b = (ord & 0x80000000u) ? (ord & 0x7FFFFFFFu) : ~ord;
  ov[row] = __uint_as_float(b);
  oi[row] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(k & 0xFFFFFFFFu));
}

__global__ void decode_positions_kernel(int32_t* __restrict__ ctx, const int32_t* __restrict__ tables,
                                        int max_blocks, int block_size, int32_t* __restrict__ pos,
                                        int64_t* __restrict__ slots, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int c = ctx[b] + 1;
  ctx[b] = c;
  const int p = c - 1;
  pos[b] = p;
  slots[b] = static_cast<int64_t>(tables[static_cast<size_t>(b) * max_blocks + p / block_size]) * block_size +
             p % block_size;
}

}  // namespace
}  // namespace ssb

extern "C" {

int ssb_decode_positions(int32_t* ctx_lens, const int32_t* block_tables, int max_blocks, int block_size,
                         int32_t* positions, int64_t* slots, int batch, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(batch >= 0 && max_blocks > 0 && block_size > 0, "ssb_decode_positions: bad shape");
  if (batch == 0) return 0;
  decode_positions_kernel<<<(batch + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      ctx_lens, block_tables, max_blocks, block_size, positions, slots, batch);
  return check_launch("ssb_decode_positions");
}

int ssb_rmsnorm(const void* x, int ldx, const int32_t* row_idx, const void* w, void* out, int ldo, int rows,
                int hidden, float eps, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(rows >= 0 && hidden > 0 && hidden % 8 == 0, "ssb_rmsnorm: hidden must be a multiple of 8");
  if (rows == 0) return 0;
  if (!aligned16(x) || !aligned16(w) || !aligned16(out) || ldx % 8 || ldo % 8) {
    set_error("ssb_rmsnorm: 16-byte alignment required");
    return SSB_EALIGN;
  }
  // optional programmatic dependent launch: the CTAs become resident while
  // the producing GEMM drains and start the moment it completes
  static const int pdl_norm = [] {
    // measured +0.15 % batch time with it on (its 512 waiting CTAs delay the
    // next GEMM's residency), so off unless SSB_PDL_NORM=1
    const char* n = getenv("SSB_PDL_NORM");
    return n ? atoi(n) : 0;
  }();
  const bool pdl = pdl_enabled() && pdl_norm;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rows);
  cfg.blockDim = dim3(kNormThreads);
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  SSB_CUDA(cudaLaunchKernelEx(&cfg, rmsnorm_kernel, static_cast<const __nv_bfloat16*>(x), ldx, row_idx,
                              static_cast<const __nv_bfloat16*>(w), static_cast<__nv_bfloat16*>(out), ldo, hidden,
                              eps));
  return check_launch("ssb_rmsnorm");
}

int ssb_rope_kv_append(void* qkv, int ld, int T, int nq, int nk, const int32_t* positions,
                       const float* rope_cos, const float* rope_sin, int max_pos, void* pool,
                       ssb_kv_geometry geo, int layer, const int64_t* slots, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(T >= 0 && nq > 0 && nk > 0 && geo.head_dim % 8 == 0, "ssb_rope_kv_append: bad shape");
  if (T == 0) return 0;
  SSB_REQUIRE(nk == geo.n_heads, "ssb_rope_kv_append: nk=%d but pool holds %d heads", nk, geo.n_heads);
  SSB_REQUIRE(layer >= 0 && layer < geo.n_layers, "ssb_rope_kv_append: layer %d out of range", layer);
  SSB_REQUIRE(ld >= (nq + 2 * nk) * geo.head_dim && ld % 8 == 0, "ssb_rope_kv_append: bad ld");
  SSB_REQUIRE(positions && rope_cos && rope_sin, "ssb_rope_kv_append: null pointer");
  SSB_REQUIRE(!slots || pool, "ssb_rope_kv_append: slots without pool");
  rope_append_kernel<<<T, kRopeThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<__nv_bfloat16*>(qkv), ld, nq, nk, geo.head_dim, positions, rope_cos, rope_sin, max_pos,
      static_cast<__nv_bfloat16*>(pool), geo, layer, slots);
  return check_launch("ssb_rope_kv_append");
}

int ssb_embedding(const int32_t* ids, int T, const void* table, int vocab_begin, int vocab_local,
                  int hidden, void* out, int ldo, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(T >= 0 && hidden % 8 == 0 && ldo % 8 == 0, "ssb_embedding: bad shape");
  if (T == 0) return 0;
  SSB_REQUIRE(ids && table && out, "ssb_embedding: null pointer");
  embedding_kernel<<<T, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      ids, static_cast<const __nv_bfloat16*>(table), vocab_begin, vocab_local, hidden,
      static_cast<__nv_bfloat16*>(out), ldo);
  return check_launch("ssb_embedding");
}

int ssb_argmax_rows(const float* logits, int ld, int rows, int cols, int index_base, float* out_val,
                    int32_t* out_idx, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(rows >= 0 && cols > 0 && ld >= cols, "ssb_argmax_rows: bad shape");
  if (rows == 0) return 0;
  argmax_kernel<<<rows, kArgThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(logits, ld, cols, index_base,
                                                                                   out_val, out_idx);
  return check_launch("ssb_argmax_rows");
}

int ssb_argmax_combine(const float* vals, const int32_t* idxs, int n_parts, int rows, int32_t* out_idx,
                       void* stream) {
  using namespace ssb;
  SSB_REQUIRE(n_parts > 0 && rows >= 0, "ssb_argmax_combine: bad shape");
  if (rows == 0) return 0;
  argmax_combine_kernel<<<(rows + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      vals, idxs, n_parts, rows, out_idx);
  return check_launch("ssb_argmax_combine");
}

}  // extern "C"

int ssb_argmax_keys_decode(const unsigned long long* keys, int rows, float* out_val, int32_t* out_idx,
                           void* stream) {
  using namespace ssb;
  SSB_REQUIRE(rows >= 0 && keys && out_val && out_idx, "ssb_argmax_keys_decode: bad arguments");
  if (rows == 0) return 0;
  argmax_keys_kernel<<<(rows + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(keys, rows, out_val,
                                                                                            out_idx);
  return check_launch("ssb_argmax_keys_decode");
}
