// Attention kernels: causal varlen prefill (flash-style, K/V from the packed
// QKV activations) and paged GQA decode (K/V streamed from the paged pool by
// TMA).  Both use bf16 mma.sync m16n8k16 with fp32 accumulation and an online
// softmax in exp2 domain; shared-memory tiles use the 128-byte XOR swizzle
// (the pattern TMA's SWIZZLE_128B produces) so ldmatrix is conflict-free.
//
// Reference counterparts (analytic only): prefill attention traffic/compute
// perf.py:68-89/:104-106; decode attention traffic perf.py:87-88 — the term
// that dominates TP decode.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "seesaw_b200.h"

namespace ssb {

int encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                        uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
int launch_prefill_attn_tc(const void* qkv, int ld, int T, int nq, int nk, const int32_t* cu, int nseq,
                           int max_len, void* out, int ldo, float scale, cudaStream_t s, bool persistent);

namespace {

constexpr float kLog2e = 1.4426950408889634f;

// byte offset of element (r, c) inside a [rows x D] bf16 tile stored as D/64
// sub-tiles of [rows][128 B] with the 128B swizzle
__device__ __forceinline__ uint32_t swz(int r, int c, int rows) {
  return static_cast<uint32_t>((c >> 6) * rows * 128 + r * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4) +
                               (c & 7) * 2);
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ------------------------------------------------------------------------
// Prefill: CTA = (64 query rows, one query head, one sequence); 4 warps x 16
// rows; K/V tiles of 64 tokens double-buffered with cp.async.
// ------------------------------------------------------------------------
template <int D>
struct PrefillSmem {
  static constexpr int kTile = 64 * D * 2;  // bytes of a 64 x D bf16 tile
  static constexpr int kBytes = kTile * 5;  // Q + 2xK + 2xV
};

template <int D>
__device__ __forceinline__ void load_tile(uint32_t sbase, const __nv_bfloat16* g, int ld, int rows_valid) {
  // 64 rows x D: D/8 16-byte chunks per row
  constexpr int kChunks = 64 * D / 8;
  for (int i = threadIdx.x; i < kChunks; i += blockDim.x) {
    const int r = i / (D / 8);
    const int c = (i - r * (D / 8)) * 8;
    const bool ok = r < rows_valid;
    const __nv_bfloat16* src = g + static_cast<size_t>(ok ? r : 0) * ld + c;
    cp_async16(sbase + swz(r, c, 64), src, ok);
  }
}

template <int D>
__global__ void __launch_bounds__(128)
    prefill_attn_kernel(const __nv_bfloat16* __restrict__ qkv, int ld, int nq, int nk,
                        const int32_t* __restrict__ cu, __nv_bfloat16* __restrict__ out, int ldo,
                        float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int seq = blockIdx.z;
  const int start = cu[seq];
  const int len = cu[seq + 1] - start;
  const int q0 = blockIdx.x * 64;
  if (q0 >= len) return;
  const int h = blockIdx.y;
  const int kvh = h / (nq / nk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  using S = PrefillSmem<D>;
  const uint32_t sQ = smem_u32(smem_raw);
  const uint32_t sK[2] = {sQ + S::kTile, sQ + 2 * S::kTile};
  const uint32_t sV[2] = {sQ + 3 * S::kTile, sQ + 4 * S::kTile};

  const __nv_bfloat16* qbase = qkv + static_cast<size_t>(start) * ld + h * D;
  const __nv_bfloat16* kbase = qkv + static_cast<size_t>(start) * ld + (nq + kvh) * D;
  const __nv_bfloat16* vbase = qkv + static_cast<size_t>(start) * ld + (nq + nk + kvh) * D;

  load_tile<D>(sQ, qbase + static_cast<size_t>(q0) * ld, ld, len - q0);
  load_tile<D>(sK[0], kbase, ld, len);
  load_tile<D>(sV[0], vbase, ld, len);
  cp_async_commit();

  const int kv_end = min(q0 + 64, len);
  const int n_tiles = (kv_end + 63) / 64;

  uint32_t qf[D / 16][4];
  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  const int row_a = q0 + warp * 16 + (lane >> 2);  // query index of c0/c1
  const int row_b = row_a + 8;                     // query index of c2/c3

  for (int j = 0; j < n_tiles; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_tiles) {
      const int kv1 = (j + 1) * 64;
      load_tile<D>(sK[buf ^ 1], kbase + static_cast<size_t>(kv1) * ld, ld, len - kv1);
      load_tile<D>(sV[buf ^ 1], vbase + static_cast<size_t>(kv1) * ld, ld, len - kv1);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        ldsm_x4(sQ + swz(warp * 16 + (lane & 15), kk * 16 + (lane >> 4) * 8, 64), qf[kk][0], qf[kk][1],
                qf[kk][2], qf[kk][3]);
    }
    // S = Q K^T  (16 rows x 64 tokens per warp)
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b0, b1, b2, b3;
        const int n = np * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int k = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(sK[buf] + swz(n, k, 64), b0, b1, b2, b3);
        mma16816(s[2 * np], qf[kk], b0, b1);
        mma16816(s[2 * np + 1], qf[kk], b2, b3);
      }
    }
    // scale + causal / length mask
    const int kv0 = j * 64;
    const bool need_mask = kv0 + 64 > q0 || kv0 + 64 > len;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[i][e] * scale_log2;
        if (need_mask) {
          const int kv = kv0 + i * 8 + (lane & 3) * 2 + (e & 1);
          const int qr = e < 2 ? row_a : row_b;
          if (kv > qr || kv >= len) v = -INFINITY;
        }
        s[i][e] = v;
      }
    }
    // online softmax (rows row_a: e=0,1 ; row_b: e=2,3)
    float corr[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 8; ++i) mx = fmaxf(mx, fmaxf(s[i][2 * hr], s[i][2 * hr + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_r[hr], mx);
      const float m_use = m_new == -INFINITY ? 0.f : m_new;
      corr[hr] = exp2f(m_r[hr] - m_use);
      m_r[hr] = m_new;
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s[i][2 * hr] = exp2f(s[i][2 * hr] - m_use);
        s[i][2 * hr + 1] = exp2f(s[i][2 * hr + 1] - m_use);
        sum += s[i][2 * hr] + s[i][2 * hr + 1];
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      l_r[hr] = l_r[hr] * corr[hr] + sum;
    }
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t a[4];
      a[0] = pack_bf16x2(s[2 * kk][0], s[2 * kk][1]);
      a[1] = pack_bf16x2(s[2 * kk][2], s[2 * kk][3]);
      a[2] = pack_bf16x2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      a[3] = pack_bf16x2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        uint32_t b0, b1, b2, b3;
        const int t = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = dp * 16 + (lane >> 4) * 8;
        ldsm_x4_t(sV[buf] + swz(t, c, 64), b0, b1, b2, b3);
        mma16816(o[2 * dp], a, b0, b1);
        mma16816(o[2 * dp + 1], a, b2, b3);
      }
    }
    __syncthreads();
  }
  // normalise and store
  const float inv_a = l_r[0] > 0.f ? 1.f / l_r[0] : 0.f;
  const float inv_b = l_r[1] > 0.f ? 1.f / l_r[1] : 0.f;
  __nv_bfloat16* oa = out + static_cast<size_t>(start + row_a) * ldo + h * D;
  __nv_bfloat16* ob = out + static_cast<size_t>(start + row_b) * ldo + h * D;
#pragma unroll
  for (int i = 0; i < D / 8; ++i) {
    const int c = i * 8 + (lane & 3) * 2;
    if (row_a < len)
      *reinterpret_cast<uint32_t*>(oa + c) = pack_bf16x2(o[i][0] * inv_a, o[i][1] * inv_a);
    if (row_b < len)
      *reinterpret_cast<uint32_t*>(ob + c) = pack_bf16x2(o[i][2] * inv_b, o[i][3] * inv_b);
  }
}

// ------------------------------------------------------------------------
// Decode: CTA = (sequence, KV head), 4 warps.  Each 64-token pool block is
// fetched by TMA (K and V, 2 x D x 128 B) into a STAGES ring; warp w owns
// tokens [16w, 16w+16) of every block; the G query heads of the group are
// the rows of a 16-row MMA tile.  Partial softmax states of the 4 warps are
// merged through shared memory at the end.
// ------------------------------------------------------------------------
constexpr int kDecStages = 3;
constexpr int kBlk = 64;

template <int D>
struct DecodeSmem {
  static constexpr int kTile = kBlk * D * 2;           // K or V of one block
  static constexpr int kStage = 2 * kTile;
  static constexpr int kBytes = kDecStages * kStage + 1024 + 64;
};

template <int D>
__global__ void __launch_bounds__(128)
    decode_attn_kernel(const __grid_constant__ CUtensorMap tmap, const __nv_bfloat16* __restrict__ qkv,
                       int ld, int nq, int nk, const int32_t* __restrict__ block_tables, int max_blocks,
                       const int32_t* __restrict__ ctx_lens, ssb_kv_geometry geo, int layer,
                       __nv_bfloat16* __restrict__ out, int ldo, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using S = DecodeSmem<D>;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kDecStages * S::kStage);
  uint64_t* empty = full + kDecStages;
  const int b = blockIdx.x;
  const int kvh = blockIdx.y;
  const int G = nq / nk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ctx = ctx_lens[b];
  const int nblk = (ctx + kBlk - 1) / kBlk;
  const int32_t* table = block_tables + static_cast<size_t>(b) * max_blocks;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap);
    for (int s = 0; s < kDecStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int j) {
    const int s = j % kDecStages;
    const int64_t blk = table[j];
    const int row_k = static_cast<int>((((blk * geo.n_layers + layer) * 2 + 0) * geo.n_heads + kvh) * kBlk);
    const int row_v = static_cast<int>((((blk * geo.n_layers + layer) * 2 + 1) * geo.n_heads + kvh) * kBlk);
    uint8_t* kt = smem + s * S::kStage;
    uint8_t* vt = kt + S::kTile;
    mbar_arrive_expect_tx(&full[s], S::kStage);
#pragma unroll
    for (int sub = 0; sub < D / 64; ++sub) {
      tma_load_2d(kt + sub * kBlk * 128, &tmap, &full[s], sub * 64, row_k, policy_evict_first());
      tma_load_2d(vt + sub * kBlk * 128, &tmap, &full[s], sub * 64, row_v, policy_evict_first());
    }
  };
  if (threadIdx.x == 0)
    for (int j = 0; j < min(nblk, kDecStages); ++j) issue(j);

  // Q fragments: rows r < G are heads kvh*G + r
  uint32_t qf[D / 16][4];
  {
    const int r0 = lane >> 2, r1 = r0 + 8;
    const __nv_bfloat16* q = qkv + static_cast<size_t>(b) * ld + static_cast<size_t>(kvh) * G * D;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int c = kk * 16 + (lane & 3) * 2;
      qf[kk][0] = r0 < G ? *reinterpret_cast<const uint32_t*>(q + r0 * D + c) : 0u;
      qf[kk][1] = r1 < G ? *reinterpret_cast<const uint32_t*>(q + r1 * D + c) : 0u;
      qf[kk][2] = r0 < G ? *reinterpret_cast<const uint32_t*>(q + r0 * D + c + 8) : 0u;
      qf[kk][3] = r1 < G ? *reinterpret_cast<const uint32_t*>(q + r1 * D + c + 8) : 0u;
    }
  }
  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

  for (int j = 0; j < nblk; ++j) {
    const int s = j % kDecStages;
    const uint32_t parity = (j / kDecStages) & 1;
    mbar_wait(&full[s], parity);
    const uint32_t kt = smem_u32(smem + s * S::kStage);
    const uint32_t vt = kt + S::kTile;
    float sc[2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t b0, b1, b2, b3;
      const int n = warp * 16 + (lane & 7) + ((lane >> 4) << 3);
      const int k = kk * 16 + ((lane >> 3) & 1) * 8;
      ldsm_x4(kt + swz(n, k, kBlk), b0, b1, b2, b3);
      mma16816(sc[0], qf[kk], b0, b1);
      mma16816(sc[1], qf[kk], b2, b3);
    }
    const int kv0 = j * kBlk + warp * 16;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kv = kv0 + i * 8 + (lane & 3) * 2 + (e & 1);
        sc[i][e] = kv < ctx ? sc[i][e] * scale_log2 : -INFINITY;
      }
    float corr[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      float mx = fmaxf(fmaxf(sc[0][2 * hr], sc[0][2 * hr + 1]), fmaxf(sc[1][2 * hr], sc[1][2 * hr + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_r[hr], mx);
      const float m_use = m_new == -INFINITY ? 0.f : m_new;
      corr[hr] = exp2f(m_r[hr] - m_use);
      m_r[hr] = m_new;
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        sc[i][2 * hr] = exp2f(sc[i][2 * hr] - m_use);
        sc[i][2 * hr + 1] = exp2f(sc[i][2 * hr + 1] - m_use);
        sum += sc[i][2 * hr] + sc[i][2 * hr + 1];
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      l_r[hr] = l_r[hr] * corr[hr] + sum;
    }
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    uint32_t a[4];
    a[0] = pack_bf16x2(sc[0][0], sc[0][1]);
    a[1] = pack_bf16x2(sc[0][2], sc[0][3]);
    a[2] = pack_bf16x2(sc[1][0], sc[1][1]);
    a[3] = pack_bf16x2(sc[1][2], sc[1][3]);
#pragma unroll
    for (int dp = 0; dp < D / 16; ++dp) {
      uint32_t b0, b1, b2, b3;
      const int t = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      const int c = dp * 16 + (lane >> 4) * 8;
      ldsm_x4_t(vt + swz(t, c, kBlk), b0, b1, b2, b3);
      mma16816(o[2 * dp], a, b0, b1);
      mma16816(o[2 * dp + 1], a, b2, b3);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (threadIdx.x == 0 && j + kDecStages < nblk) {
      mbar_wait(&empty[s], parity);
      issue(j + kDecStages);
    }
  }
  __syncthreads();  // every TMA consumed; stage buffers are free
  // merge the 4 warps' partial states (only rows < G are real)
  float* sm_m = reinterpret_cast<float*>(smem);              // [4][16]
  float* sm_l = sm_m + 4 * 16;                               // [4][16]
  float* sm_o = sm_l + 4 * 16;                               // [4][16][D]
  const int r0 = lane >> 2, r1 = r0 + 8;
  if ((lane & 3) == 0) {
    sm_m[warp * 16 + r0] = m_r[0];
    sm_m[warp * 16 + r1] = m_r[1];
    sm_l[warp * 16 + r0] = l_r[0];
    sm_l[warp * 16 + r1] = l_r[1];
  }
#pragma unroll
  for (int i = 0; i < D / 8; ++i) {
    const int c = i * 8 + (lane & 3) * 2;
    sm_o[(warp * 16 + r0) * D + c] = o[i][0];
    sm_o[(warp * 16 + r0) * D + c + 1] = o[i][1];
    sm_o[(warp * 16 + r1) * D + c] = o[i][2];
    sm_o[(warp * 16 + r1) * D + c + 1] = o[i][3];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
    const int r = idx / D, c = idx - r * D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w * 16 + r]);
    const float Mu = M == -INFINITY ? 0.f : M;
    float L = 0.f, acc = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float f = exp2f(sm_m[w * 16 + r] - Mu);
      L += sm_l[w * 16 + r] * f;
      acc += sm_o[(w * 16 + r) * D + c] * f;
    }
    out[static_cast<size_t>(b) * ldo + (kvh * G + r) * D + c] = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
  }
}

// ------------------------------------------------------------------------
// Persistent decode attention: 2 CTAs per SM loop over (sequence, KV head)
// items round-robin.  The TMA producer (thread 0) walks a flattened
// (item, block) cursor, so while the 4 warps finish item i and merge it, the
// ring already holds the first blocks of item i+1: no per-CTA prologue or
// drain gap in the HBM stream (the per-(b, kvh) kernel above reaches ~83 %
// of DRAM peak in isolation, limited by those gaps).  The 4-warp merge uses
// its own smem region ([4][G][D] fp32) so it never touches the ring.
// ------------------------------------------------------------------------
template <int D, int kPStages = 3>
struct DecodeSmemP {
  static constexpr int kTile = kBlk * D * 2;
  static constexpr int kStage = 2 * kTile;
  static constexpr int kRing = kPStages * kStage;
  static int bytes(int G) { return kRing + 64 /*barriers*/ + 2 * 4 * 16 * 4 + 4 * G * D * 4 + 1024; }
};

template <int D, int kPStages>
__global__ void __launch_bounds__(128)
    decode_attn_persistent(const __grid_constant__ CUtensorMap tmap, const __nv_bfloat16* __restrict__ qkv,
                           int ld, int nq, int nk, const int32_t* __restrict__ block_tables, int max_blocks,
                           const int32_t* __restrict__ ctx_lens, int B, ssb_kv_geometry geo, int layer,
                           __nv_bfloat16* __restrict__ out, int ldo, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using S = DecodeSmemP<D, kPStages>;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kRing);
  uint64_t* empty = full + kPStages;
  float* sm_m = reinterpret_cast<float*>(smem + S::kRing + 64);  // [4][16]
  float* sm_l = sm_m + 4 * 16;                                   // [4][16]
  float* sm_o = sm_l + 4 * 16;                                   // [4][G][D]
  const int G = nq / nk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = B * nk;
  griddep_launch_dependents();

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap);
    for (int st = 0; st < kPStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ---- producer cursor (thread 0 only): next (item, block) to load ----
  int p_item = blockIdx.x, p_blk = 0, p_nblk = 0;
  uint32_t p_count = 0;  // blocks issued so far (ring slot = p_count % kPStages)
  auto p_seek = [&]() {  // skip to an item with blocks left
    while (p_item < n_items) {
      if (p_blk == 0) p_nblk = (ctx_lens[p_item / nk] + kBlk - 1) / kBlk;
      if (p_blk < p_nblk) return true;
      p_item += gridDim.x;
      p_blk = 0;
    }
    return false;
  };
  auto issue_next = [&]() {
    if (!p_seek()) return;
    const int st = p_count % kPStages;
    const int b = p_item / nk, kvh = p_item - (p_item / nk) * nk;
    const int64_t blk = block_tables[static_cast<size_t>(b) * max_blocks + p_blk];
    const int row_k = static_cast<int>((((blk * geo.n_layers + layer) * 2 + 0) * geo.n_heads + kvh) * kBlk);
    const int row_v = static_cast<int>((((blk * geo.n_layers + layer) * 2 + 1) * geo.n_heads + kvh) * kBlk);
    uint8_t* kt = smem + st * S::kStage;
    uint8_t* vt = kt + S::kTile;
    mbar_arrive_expect_tx(&full[st], S::kStage);
#pragma unroll
    for (int sub = 0; sub < D / 64; ++sub) {
      tma_load_2d(kt + sub * kBlk * 128, &tmap, &full[st], sub * 64, row_k, policy_evict_first());
      tma_load_2d(vt + sub * kBlk * 128, &tmap, &full[st], sub * 64, row_v, policy_evict_first());
    }
    ++p_count;
    ++p_blk;
  };
  // PDL: this kernel may start while the QKV GEMM that appends the current
  // token's K/V (and writes Q) still runs.  Every pool block but a sequence's
  // LAST one holds only older tokens, so those may stream into the ring now;
  // Q and the last blocks are read only after griddep_wait().
  int issued = 0;
  if (threadIdx.x == 0) {
    while (issued < kPStages && p_seek() && p_blk + 1 < p_nblk) {
      issue_next();
      ++issued;
    }
  }
  griddep_wait();
  if (threadIdx.x == 0)
    for (; issued < kPStages; ++issued) issue_next();

  uint32_t c_count = 0;  // blocks consumed so far
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int b = item / nk, kvh = item - (item / nk) * nk;
    const int ctx = ctx_lens[b];
    const int nblk = (ctx + kBlk - 1) / kBlk;
    uint32_t qf[D / 16][4];
    {
      const int r0 = lane >> 2, r1 = r0 + 8;
      const __nv_bfloat16* q = qkv + static_cast<size_t>(b) * ld + static_cast<size_t>(kvh) * G * D;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int c = kk * 16 + (lane & 3) * 2;
        qf[kk][0] = r0 < G ? *reinterpret_cast<const uint32_t*>(q + r0 * D + c) : 0u;
        qf[kk][1] = r1 < G ? *reinterpret_cast<const uint32_t*>(q + r1 * D + c) : 0u;
        qf[kk][2] = r0 < G ? *reinterpret_cast<const uint32_t*>(q + r0 * D + c + 8) : 0u;
        qf[kk][3] = r1 < G ? *reinterpret_cast<const uint32_t*>(q + r1 * D + c + 8) : 0u;
      }
    }
    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

    for (int j = 0; j < nblk; ++j, ++c_count) {
      const int st = c_count % kPStages;
      const uint32_t parity = (c_count / kPStages) & 1;
      mbar_wait(&full[st], parity);
      const uint32_t kt = smem_u32(smem + st * S::kStage);
      const uint32_t vt = kt + S::kTile;
      float sc[2][4];
#pragma unroll
      for (int i = 0; i < 2; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        uint32_t b0, b1, b2, b3;
        const int n = warp * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int k = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(kt + swz(n, k, kBlk), b0, b1, b2, b3);
        mma16816(sc[0], qf[kk], b0, b1);
        mma16816(sc[1], qf[kk], b2, b3);
      }
      const int kv0 = j * kBlk + warp * 16;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int kv = kv0 + i * 8 + (lane & 3) * 2 + (e & 1);
          sc[i][e] = kv < ctx ? sc[i][e] * scale_log2 : -INFINITY;
        }
      float corr[2];
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        float mx = fmaxf(fmaxf(sc[0][2 * hr], sc[0][2 * hr + 1]), fmaxf(sc[1][2 * hr], sc[1][2 * hr + 1]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float m_new = fmaxf(m_r[hr], mx);
        const float m_use = m_new == -INFINITY ? 0.f : m_new;
        corr[hr] = exp2f(m_r[hr] - m_use);
        m_r[hr] = m_new;
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          sc[i][2 * hr] = exp2f(sc[i][2 * hr] - m_use);
          sc[i][2 * hr + 1] = exp2f(sc[i][2 * hr + 1] - m_use);
          sum += sc[i][2 * hr] + sc[i][2 * hr + 1];
        }
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        l_r[hr] = l_r[hr] * corr[hr] + sum;
      }
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        o[i][0] *= corr[0];
        o[i][1] *= corr[0];
        o[i][2] *= corr[1];
        o[i][3] *= corr[1];
      }
      uint32_t a[4];
      a[0] = pack_bf16x2(sc[0][0], sc[0][1]);
      a[1] = pack_bf16x2(sc[0][2], sc[0][3]);
      a[2] = pack_bf16x2(sc[1][0], sc[1][1]);
      a[3] = pack_bf16x2(sc[1][2], sc[1][3]);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        uint32_t b0, b1, b2, b3;
        const int t = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = dp * 16 + (lane >> 4) * 8;
        ldsm_x4_t(vt + swz(t, c, kBlk), b0, b1, b2, b3);
        mma16816(o[2 * dp], a, b0, b1);
        mma16816(o[2 * dp + 1], a, b2, b3);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (threadIdx.x == 0) {
        mbar_wait(&empty[st], parity);
        issue_next();  // possibly the first blocks of this CTA's next item
      }
    }
    // merge the 4 warps' partial states (rows < G are real) in the merge region
    const int r0 = lane >> 2, r1 = r0 + 8;
    if ((lane & 3) == 0) {
      sm_m[warp * 16 + r0] = m_r[0];
      sm_m[warp * 16 + r1] = m_r[1];
      sm_l[warp * 16 + r0] = l_r[0];
      sm_l[warp * 16 + r1] = l_r[1];
    }
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const int c = i * 8 + (lane & 3) * 2;
      if (r0 < G) {
        sm_o[(warp * G + r0) * D + c] = o[i][0];
        sm_o[(warp * G + r0) * D + c + 1] = o[i][1];
      }
      if (r1 < G) {
        sm_o[(warp * G + r1) * D + c] = o[i][2];
        sm_o[(warp * G + r1) * D + c + 1] = o[i][3];
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
      const int r = idx / D, c = idx - r * D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w * 16 + r]);
      const float Mu = M == -INFINITY ? 0.f : M;
      float L = 0.f, acc = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float f = exp2f(sm_m[w * 16 + r] - Mu);
        L += sm_l[w * 16 + r] * f;
        acc += sm_o[(w * G + r) * D + c] * f;
      }
      out[static_cast<size_t>(b) * ldo + (kvh * G + r) * D + c] = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
    }
    __syncthreads();  // the merge region is rewritten by the next item
  }
}

// Warp-specialised variant (default): a 5th warp is the TMA producer, and
// every consumer warp copies its K and V fragments of a block from the ring
// into registers (ldmatrix) and releases the slot BEFORE its MMAs and
// softmax, so a slot is refilled as soon as the four warps have read it --
// not after the slowest warp finished computing on it (thread 0 used to wait
// for that before issuing the refill).  The ring's bytes in flight then
// stay close to its size: the kernel was at ~6.6 TB/s while a bare
// bulk-copy read stream with the same 192 KB in flight per SM reads
// 7.3 TB/s on the same box (tools/read_bw.py).
template <int D, int kPStages>
__global__ void __launch_bounds__(160)
    decode_attn_persistent_ws(const __grid_constant__ CUtensorMap tmap, const __nv_bfloat16* __restrict__ qkv,
                           int ld, int nq, int nk, const int32_t* __restrict__ block_tables, int max_blocks,
                           const int32_t* __restrict__ ctx_lens, int B, ssb_kv_geometry geo, int layer,
                           __nv_bfloat16* __restrict__ out, int ldo, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using S = DecodeSmemP<D, kPStages>;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kRing);
  uint64_t* empty = full + kPStages;
  float* sm_m = reinterpret_cast<float*>(smem + S::kRing + 64);  // [4][16]
  float* sm_l = sm_m + 4 * 16;                                   // [4][16]
  float* sm_o = sm_l + 4 * 16;                                   // [4][G][D]
  const int G = nq / nk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = B * nk;
  griddep_launch_dependents();

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap);
    for (int st = 0; st < kPStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ---- producer (warp 4, lane 0): next (item, block) to load ----
  int p_item = blockIdx.x, p_blk = 0, p_nblk = 0;
  uint32_t p_count = 0;  // blocks issued so far (ring slot = p_count % kPStages)
  auto p_seek = [&]() {  // skip to an item with blocks left
    while (p_item < n_items) {
      if (p_blk == 0) p_nblk = (ctx_lens[p_item / nk] + kBlk - 1) / kBlk;
      if (p_blk < p_nblk) return true;
      p_item += gridDim.x;
      p_blk = 0;
    }
    return false;
  };
  auto issue_next = [&]() {
    if (!p_seek()) return;
    const int st = p_count % kPStages;
    const int b = p_item / nk, kvh = p_item - (p_item / nk) * nk;
    const int64_t blk = block_tables[static_cast<size_t>(b) * max_blocks + p_blk];
    const int row_k = static_cast<int>((((blk * geo.n_layers + layer) * 2 + 0) * geo.n_heads + kvh) * kBlk);
    const int row_v = static_cast<int>((((blk * geo.n_layers + layer) * 2 + 1) * geo.n_heads + kvh) * kBlk);
    uint8_t* kt = smem + st * S::kStage;
    uint8_t* vt = kt + S::kTile;
    mbar_arrive_expect_tx(&full[st], S::kStage);
#pragma unroll
    for (int sub = 0; sub < D / 64; ++sub) {
      tma_load_2d(kt + sub * kBlk * 128, &tmap, &full[st], sub * 64, row_k, policy_evict_first());
      tma_load_2d(vt + sub * kBlk * 128, &tmap, &full[st], sub * 64, row_v, policy_evict_first());
    }
    ++p_count;
    ++p_blk;
  };
  // PDL: this kernel may start while the QKV GEMM that appends the current
  // token's K/V (and writes Q) still runs.  Every pool block but a sequence's
  // LAST one holds only older tokens, so those may stream into the ring now;
  // Q and the last blocks are read only after griddep_wait().
  if (warp == 4) {
    if (lane == 0) {
      while (p_count < kPStages && p_seek() && p_blk + 1 < p_nblk) issue_next();
      griddep_wait();
      while (p_seek()) {
        // slot of block p_count: free once block p_count - kPStages was read
        if (p_count >= kPStages) mbar_wait(&empty[p_count % kPStages], ((p_count / kPStages) & 1) ^ 1);
        issue_next();
      }
    }
    return;
  }
  griddep_wait();  // consumers read Q (written by the predecessor)

  uint32_t c_count = 0;  // blocks consumed so far
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int b = item / nk, kvh = item - (item / nk) * nk;
    const int ctx = ctx_lens[b];
    const int nblk = (ctx + kBlk - 1) / kBlk;
    uint32_t qf[D / 16][4];
    {
      const int r0 = lane >> 2, r1 = r0 + 8;
      const __nv_bfloat16* q = qkv + static_cast<size_t>(b) * ld + static_cast<size_t>(kvh) * G * D;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int c = kk * 16 + (lane & 3) * 2;
        qf[kk][0] = r0 < G ? *reinterpret_cast<const uint32_t*>(q + r0 * D + c) : 0u;
        qf[kk][1] = r1 < G ? *reinterpret_cast<const uint32_t*>(q + r1 * D + c) : 0u;
        qf[kk][2] = r0 < G ? *reinterpret_cast<const uint32_t*>(q + r0 * D + c + 8) : 0u;
        qf[kk][3] = r1 < G ? *reinterpret_cast<const uint32_t*>(q + r1 * D + c + 8) : 0u;
      }
    }
    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

    for (int j = 0; j < nblk; ++j, ++c_count) {
      const int st = c_count % kPStages;
      const uint32_t parity = (c_count / kPStages) & 1;
      mbar_wait(&full[st], parity);
      const uint32_t kt = smem_u32(smem + st * S::kStage);
      const uint32_t vt = kt + S::kTile;
      // this warp's 16 tokens of K and V into registers, then release the slot
      uint32_t kf[D / 16][4], vf[D / 16][4];
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int n = warp * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int k = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(kt + swz(n, k, kBlk), kf[kk][0], kf[kk][1], kf[kk][2], kf[kk][3]);
      }
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        const int t = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = dp * 16 + (lane >> 4) * 8;
        ldsm_x4_t(vt + swz(t, c, kBlk), vf[dp][0], vf[dp][1], vf[dp][2], vf[dp][3]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      float sc[2][4];
#pragma unroll
      for (int i = 0; i < 2; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        mma16816(sc[0], qf[kk], kf[kk][0], kf[kk][1]);
        mma16816(sc[1], qf[kk], kf[kk][2], kf[kk][3]);
      }
      const int kv0 = j * kBlk + warp * 16;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int kv = kv0 + i * 8 + (lane & 3) * 2 + (e & 1);
          sc[i][e] = kv < ctx ? sc[i][e] * scale_log2 : -INFINITY;
        }
      float corr[2];
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        float mx = fmaxf(fmaxf(sc[0][2 * hr], sc[0][2 * hr + 1]), fmaxf(sc[1][2 * hr], sc[1][2 * hr + 1]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float m_new = fmaxf(m_r[hr], mx);
        const float m_use = m_new == -INFINITY ? 0.f : m_new;
        corr[hr] = exp2f(m_r[hr] - m_use);
        m_r[hr] = m_new;
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          sc[i][2 * hr] = exp2f(sc[i][2 * hr] - m_use);
          sc[i][2 * hr + 1] = exp2f(sc[i][2 * hr + 1] - m_use);
          sum += sc[i][2 * hr] + sc[i][2 * hr + 1];
        }
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        l_r[hr] = l_r[hr] * corr[hr] + sum;
      }
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        o[i][0] *= corr[0];
        o[i][1] *= corr[0];
        o[i][2] *= corr[1];
        o[i][3] *= corr[1];
      }
      uint32_t a[4];
      a[0] = pack_bf16x2(sc[0][0], sc[0][1]);
      a[1] = pack_bf16x2(sc[0][2], sc[0][3]);
      a[2] = pack_bf16x2(sc[1][0], sc[1][1]);
      a[3] = pack_bf16x2(sc[1][2], sc[1][3]);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        mma16816(o[2 * dp], a, vf[dp][0], vf[dp][1]);
        mma16816(o[2 * dp + 1], a, vf[dp][2], vf[dp][3]);
      }
    }
    // merge the 4 warps' partial states (rows < G are real) in the merge region
    const int r0 = lane >> 2, r1 = r0 + 8;
    if ((lane & 3) == 0) {
      sm_m[warp * 16 + r0] = m_r[0];
      sm_m[warp * 16 + r1] = m_r[1];
      sm_l[warp * 16 + r0] = l_r[0];
      sm_l[warp * 16 + r1] = l_r[1];
    }
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const int c = i * 8 + (lane & 3) * 2;
      if (r0 < G) {
        sm_o[(warp * G + r0) * D + c] = o[i][0];
        sm_o[(warp * G + r0) * D + c + 1] = o[i][1];
      }
      if (r1 < G) {
        sm_o[(warp * G + r1) * D + c] = o[i][2];
        sm_o[(warp * G + r1) * D + c + 1] = o[i][3];
      }
    }
    named_bar_sync(1, 128);
    for (int idx = threadIdx.x; idx < G * D; idx += 128) {
      const int r = idx / D, c = idx - r * D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w * 16 + r]);
      const float Mu = M == -INFINITY ? 0.f : M;
      float L = 0.f, acc = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float f = exp2f(sm_m[w * 16 + r] - Mu);
        L += sm_l[w * 16 + r] * f;
        acc += sm_o[(w * G + r) * D + c] * f;
      }
      out[static_cast<size_t>(b) * ldo + (kvh * G + r) * D + c] = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
    }
    named_bar_sync(1, 128);  // the merge region is rewritten by the next item
  }
}

template <int D>
int launch_prefill(const void* qkv, int ld, int nq, int nk, const int32_t* cu, int nseq, int max_len,
                   void* out, int ldo, float scale, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    SSB_CUDA(cudaFuncSetAttribute(prefill_attn_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  PrefillSmem<D>::kBytes));
    attr = true;
  }
  dim3 grid((max_len + 63) / 64, nq, nseq);
  prefill_attn_kernel<D><<<grid, 128, PrefillSmem<D>::kBytes, s>>>(
      static_cast<const __nv_bfloat16*>(qkv), ld, nq, nk, cu, static_cast<__nv_bfloat16*>(out), ldo,
      scale * kLog2e);
  return check_launch("prefill_attn_kernel");
}

template <int D, int ST>
int launch_decode_p(const CUtensorMap& map, const void* qkv, int ld, int nq, int nk, ssb_kv_geometry geo, int layer,
                    const int32_t* tables, int max_blocks, const int32_t* ctx, int B, void* out, int ldo, float scale,
                    int ctas_per_sm, cudaStream_t s, bool ws) {
  const int G = nq / nk;
  const int smem = DecodeSmemP<D, ST>::bytes(G);
  auto kern = ws ? decode_attn_persistent_ws<D, ST> : decode_attn_persistent<D, ST>;
  const int threads = ws ? 160 : 128;
  static int attr_p[2] = {0, 0};
  if (attr_p[ws] < smem) {
    SSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_p[ws] = smem;
  }
  int per_sm = 0;
  SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  if (ctas_per_sm > 0) per_sm = std::min(per_sm, ctas_per_sm);
  const long items = static_cast<long>(B) * nk;
  const int grid = static_cast<int>(std::min<long>(items, static_cast<long>(std::max(per_sm, 1)) * num_sms()));
  const bool pdl = pdl_enabled();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  SSB_CUDA(cudaLaunchKernelEx(&cfg, kern, map, static_cast<const __nv_bfloat16*>(qkv), ld, nq, nk, tables, max_blocks,
                              ctx, B, geo, layer, static_cast<__nv_bfloat16*>(out), ldo, scale * kLog2e));
  return check_launch(ws ? "decode_attn_persistent_ws" : "decode_attn_persistent");
}

template <int D>
int launch_decode(const void* qkv, int ld, int nq, int nk, const void* pool, ssb_kv_geometry geo, int num_blocks,
                  int layer, const int32_t* tables, int max_blocks, const int32_t* ctx, int B, void* out, int ldo,
                  float scale, cudaStream_t s) {
  CUtensorMap map;
  // the whole pool as a 2-D [rows, D] tensor; one box = 64 tokens x 64 dims
  const uint64_t rows = static_cast<uint64_t>(num_blocks) * geo.n_layers * 2 * geo.n_heads * geo.block_size;
  if (rows >= (1ull << 31)) {
    set_error("decode attention: pool of %llu rows exceeds TMA int32 coordinates", (unsigned long long)rows);
    return SSB_EUNSUPPORTED;
  }
  int rc = encode_tmap_2d_bf16(&map, pool, D, rows, D * 2, 64, 64);
  if (rc) return rc;
  static const int variant = [] {
    // A/B: 1 = one CTA per (sequence, KV head); 2 = persistent with the
    // refill issued by consumer thread 0 (before the producer warp)
    const char* e = getenv("SSB_DECODE_ATTN_VARIANT");
    return e ? atoi(e) : 0;
  }();
  if (variant == 0 || variant == 2) {
    const bool ws = variant == 0;
    // ring depth x CTAs per SM (SSB_DECODE_STAGES, SSB_DECODE_CTAS: A/B knobs)
    // measured in the decode step (profiles/r02/decode_attn_ws_sweep.jsonl):
    // the producer-warp kernel is fastest with a 2-deep ring (2 CTAs per SM,
    // register-limited) -- 18.43 vs 18.72 ms per 8B decode step for the
    // thread-0-refill kernel at its best (3 stages)
    static const int stages = [ws] {
      const char* e = getenv("SSB_DECODE_STAGES");
      return e ? atoi(e) : (ws ? 2 : 3);
    }();
    static const int ctas = [] {
      const char* e = getenv("SSB_DECODE_CTAS");
      return e ? atoi(e) : 0;
    }();
    switch (stages) {
      case 2: return launch_decode_p<D, 2>(map, qkv, ld, nq, nk, geo, layer, tables, max_blocks, ctx, B, out, ldo, scale, ctas, s, ws);
      case 4: return launch_decode_p<D, 4>(map, qkv, ld, nq, nk, geo, layer, tables, max_blocks, ctx, B, out, ldo, scale, ctas, s, ws);
      case 6: return launch_decode_p<D, 6>(map, qkv, ld, nq, nk, geo, layer, tables, max_blocks, ctx, B, out, ldo, scale, ctas, s, ws);
      default: return launch_decode_p<D, 3>(map, qkv, ld, nq, nk, geo, layer, tables, max_blocks, ctx, B, out, ldo, scale, ctas, s, ws);
    }
  }
  static bool attr = false;
  if (!attr) {
    SSB_CUDA(cudaFuncSetAttribute(decode_attn_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  DecodeSmem<D>::kBytes));
    attr = true;
  }
  dim3 grid(B, nk);
  decode_attn_kernel<D><<<grid, 128, DecodeSmem<D>::kBytes, s>>>(
      map, static_cast<const __nv_bfloat16*>(qkv), ld, nq, nk, tables, max_blocks, ctx, geo, layer,
      static_cast<__nv_bfloat16*>(out), ldo, scale * kLog2e);
  return check_launch("decode_attn_kernel");
}

}  // namespace
}  // namespace ssb

extern "C" {

int ssb_prefill_attention(const void* qkv, int ld, int total_tokens, int nq, int nk, int head_dim,
                          const int32_t* cu_seqlens, int nseq, int max_len, void* out, int ldo, float softmax_scale,
                          int variant, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(nseq >= 0 && max_len >= 0 && nq > 0 && nk > 0 && nq % nk == 0, "ssb_prefill_attention: bad shape");
  if (nseq == 0 || max_len == 0) return 0;
  SSB_REQUIRE(ld % 8 == 0 && ldo % 8 == 0 && aligned16(qkv) && aligned16(out), "ssb_prefill_attention: alignment");
  SSB_REQUIRE(total_tokens > 0, "ssb_prefill_attention: total_tokens must be positive");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // variant 0 = auto (persistent tcgen05 kernel for head_dim 128), 1 = mma.sync kernel,
  // 2 = tcgen05 kernel with one CTA per (query tile, head, sequence)
  if (head_dim == 128 && variant != 1)
    return launch_prefill_attn_tc(qkv, ld, total_tokens, nq, nk, cu_seqlens, nseq, max_len, out, ldo,
                                  softmax_scale, s, variant != 2);
  switch (head_dim) {
    case 64: return launch_prefill<64>(qkv, ld, nq, nk, cu_seqlens, nseq, max_len, out, ldo, softmax_scale, s);
    case 128: return launch_prefill<128>(qkv, ld, nq, nk, cu_seqlens, nseq, max_len, out, ldo, softmax_scale, s);
    default: return fail_arg("ssb_prefill_attention: head_dim %d unsupported (64, 128)", head_dim);
  }
}

int ssb_decode_attention(const void* qkv, int ld, int nq, int nk, const void* pool, ssb_kv_geometry geo,
                         int num_blocks, int layer, const int32_t* block_tables, int max_blocks,
                         const int32_t* ctx_lens, int batch, void* out, int ldo, float softmax_scale,
                         void* stream) {
  using namespace ssb;
  SSB_REQUIRE(batch >= 0 && nq > 0 && nk > 0 && nq % nk == 0 && nq / nk <= 16,
              "ssb_decode_attention: need nq %% nk == 0 and group <= 16");
  if (batch == 0) return 0;
  SSB_REQUIRE(geo.block_size == 64, "ssb_decode_attention: block_size must be 64 (got %d)", geo.block_size);
  SSB_REQUIRE(nk == geo.n_heads, "ssb_decode_attention: nk=%d but pool holds %d heads", nk, geo.n_heads);
  SSB_REQUIRE(layer >= 0 && layer < geo.n_layers && num_blocks > 0, "ssb_decode_attention: bad layer/blocks");
  SSB_REQUIRE(aligned16(pool) && aligned16(out) && ld % 2 == 0, "ssb_decode_attention: alignment");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  switch (geo.head_dim) {
    case 64:
      return launch_decode<64>(qkv, ld, nq, nk, pool, geo, num_blocks, layer, block_tables, max_blocks, ctx_lens, batch, out,
                               ldo, softmax_scale, s);
    case 128:
      return launch_decode<128>(qkv, ld, nq, nk, pool, geo, num_blocks, layer, block_tables, max_blocks, ctx_lens, batch, out,
                                ldo, softmax_scale, s);
    default: return fail_arg("ssb_decode_attention: head_dim %d unsupported (64, 128)", geo.head_dim);
  }
}

}  // extern "C"
