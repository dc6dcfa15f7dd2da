// Causal varlen prefill attention on the 5th-generation tensor cores
// (head_dim 128).  Replaces the attention terms of the reference cost model
// (perf.py:68-86 traffic, perf.py:104-106 compute) for prefill.
//
// CTA = (128 query rows, one query head, one sequence), 6 warps:
//   warp 0     TMA: Q tile once, then K/V tiles of 128 keys into a 2-stage ring
//              (128B swizzle, straight from the packed QKV activations).
//   warp 1     TMEM owner + single-thread tcgen05.mma issue:
//                S_j  = Q . K_j^T        (M=128, N=128 keys, K=128; A,B K-major)
//                O   += P_j . V_j        (M=128, N=128 dims, K=128 keys;
//                                         P K-major in smem, V MN-major)
//              S is double-buffered in TMEM so S_{j+1} overlaps softmax_j.
//   warps 2-5  softmax, one thread per query row (its TMEM lane): rowmax,
//              exp2, rowsum on the thread's own row (no shuffles), P written
//              to smem as bf16 in the UMMA K-major SW128 layout.  The running
//              max is updated lazily (only when it grows by > 8 in log2
//              units), so O in TMEM is rescaled rarely; final O / l epilogue.
#include <algorithm>

#include "common.cuh"
#include "seesaw_b200.h"

namespace ssb {

int encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                        uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);

namespace {

constexpr int kD = 128;          // head dim
constexpr int kT = 128;          // query rows and keys per tile
constexpr int kSub = kT * 128;   // bytes of one [128 rows][64 elems] SW128 sub-tile
constexpr int kTile = 2 * kSub;  // 128 x 128 bf16 tile (two 64-column sub-tiles)
constexpr int kThreads = 192;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct Smem {
  static constexpr int kQ = 0;
  static constexpr int kK = kTile;              // 2 stages
  static constexpr int kV = kK + 2 * kTile;     // 2 stages
  static constexpr int kP = kV + 2 * kTile;
  static constexpr int kBar = kP + kTile;
  static constexpr int kBytes = kBar + 256 + 1024;
};

// MN-major SW128 descriptor (V as the B operand of P.V): 64-element MN atoms
// at LBO (the next 64 head dims = next sub-tile), 8-key groups at SBO = 1024 B.
__device__ __forceinline__ uint64_t sdesc_mn_sw128(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(kThreads, 1)
    prefill_attn_tc(const __grid_constant__ CUtensorMap tmap, const int32_t* __restrict__ cu, int nq, int nk,
                    __nv_bfloat16* __restrict__ out, int ldo, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::kBar);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* s_free = bars + 7;    // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* o_done = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int seq = blockIdx.z;
  const int start = cu[seq];
  const int len = cu[seq + 1] - start;
  const int n_qt = (len + kT - 1) / kT;
  const int qt = static_cast<int>(gridDim.x) - 1 - static_cast<int>(blockIdx.x);  // longest tiles first
  if (qt >= n_qt) return;
  const int q0 = qt * kT;
  const int h = blockIdx.y;
  const int kvh = h / (nq / nk);
  const int n_kv = qt + 1;  // causal: key tiles 0..qt (tile sizes equal)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: S buffers at 0 and 128, O at 256
  const uint32_t t_s[2] = {tmem, tmem + 128};
  const uint32_t t_o = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t keep = policy_evict_last();
      const int qcol = h * kD, kcol = (nq + kvh) * kD, vcol = (nq + nk + kvh) * kD;
      mbar_arrive_expect_tx(q_full, kTile);
      for (int s = 0; s < 2; ++s)
        tma_load_2d(smem + Smem::kQ + s * kSub, &tmap, q_full, qcol + s * 64, start + q0, keep);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * kTile);
        for (int s = 0; s < 2; ++s) {
          tma_load_2d(smem + Smem::kK + st * kTile + s * kSub, &tmap, &kv_full[st], kcol + s * 64,
                      start + j * kT, keep);
          tma_load_2d(smem + Smem::kV + st * kTile + s * kSub, &tmap, &kv_full[st], vcol + s * 64,
                      start + j * kT, keep);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kT, kT);
      constexpr uint32_t idesc_o = idesc_bf16_f32(kT, kD) | (1u << 16);  // B (= V) MN-major
      const uint32_t q_base = smem_u32(smem + Smem::kQ);
      const uint32_t p_base = smem_u32(smem + Smem::kP);
      mbar_wait(q_full, 0);
      auto pv = [&](int j) {
        // O += P_j . V_j once softmax_j has written P and rescaled O
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        const uint32_t v_base = smem_u32(smem + Smem::kV + (j & 1) * kTile);
#pragma unroll
        for (int k = 0; k < kT / 16; ++k) {
          const uint64_t a = sdesc_k_sw128(p_base + (k >> 2) * kSub + (k & 3) * 32);
          const uint64_t b = sdesc_mn_sw128(v_base + k * 16 * 128, kSub);
          umma_bf16(t_o, a, b, idesc_o, (j | k) != 0);
        }
        umma_commit(o_done);
        umma_commit(&kv_empty[j & 1]);
      };
      for (int j = 0; j < n_kv; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_full[st], (j >> 1) & 1);
        if (j >= 2) mbar_wait(&s_free[st], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(smem + Smem::kK + st * kTile);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          const uint64_t a = sdesc_k_sw128(q_base + (k >> 2) * kSub + (k & 3) * 32);
          const uint64_t b = sdesc_k_sw128(k_base + (k >> 2) * kSub + (k & 3) * 32);
          umma_bf16(t_s[st], a, b, idesc_s, k != 0);
        }
        umma_commit(&s_full[st]);
        if (j >= 1) pv(j - 1);
      }
      pv(n_kv - 1);
    }
  } else {
    // ---------------- softmax / epilogue: thread = query row ----------------
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // row inside the tile == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int qrow = q0 + r;
    float m_used = -INFINITY, l = 0.f;
    uint8_t* p_row = smem + Smem::kP + r * 128;
    for (int j = 0; j < n_kv; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float s[kT];
#pragma unroll
      for (int c = 0; c < kT / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(t_s[st] + lane_off + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(v[i]) * scale_log2;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[st]);
      const int k0 = j * kT;
      if (j == n_kv - 1 || k0 + kT > len) {
#pragma unroll
        for (int i = 0; i < kT; ++i)
          if (k0 + i > qrow || k0 + i >= len) s[i] = -INFINITY;
      }
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < kT; ++i) mx = fmaxf(mx, s[i]);
      float corr = 1.f;
      const bool rescale = mx > m_used + kRescaleThreshold;
      if (rescale) {
        corr = (m_used == -INFINITY) ? 0.f : fast_exp2(m_used - mx);
        m_used = mx;
      }
      float sum = 0.f;
      uint32_t pk[kT / 2];
#pragma unroll
      for (int i = 0; i < kT; i += 2) {
        const float a = fast_exp2(s[i] - m_used), b = fast_exp2(s[i + 1] - m_used);
        sum += a + b;
        pk[i / 2] = pack_bf16x2(a, b);
      }
      // P buffer and O are free once P_{j-1}.V_{j-1} has completed
      if (j >= 1) mbar_wait(o_done, (j - 1) & 1);
      tc_fence_after();
      // a warp-uniform decision keeps tcgen05.ld/st converged
      if (j >= 1 && __any_sync(0xffffffffu, rescale)) {
#pragma unroll 1
        for (int c = 0; c < kD / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(t_o + lane_off + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
          tmem_st32(t_o + lane_off + c * 32, v);
        }
        tmem_st_wait();
      }
      l = l * corr + sum;
      // P row -> smem, UMMA K-major SW128: 16-byte chunk c of sub-tile sb at
      // row*128 + ((c ^ (row & 7)) * 16)
#pragma unroll
      for (int c = 0; c < kT / 8; ++c) {
        const int sb = c >> 3, cc = c & 7;
        uint4 val = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        *reinterpret_cast<uint4*>(p_row + sb * kSub + ((cc ^ (r & 7)) << 4)) = val;
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // epilogue: O / l
    mbar_wait(o_done, (n_kv - 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = out + static_cast<size_t>(start + qrow) * ldo + h * kD;
#pragma unroll 1
    for (int c = 0; c < kD / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(t_o + lane_off + c * 32, v);
      tmem_ld_wait();
      if (qrow < len) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 o;
          o.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
          o.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
          o.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
          o.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
          dst[q] = o;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------
// Persistent variant: one CTA per SM loops over (query tile, head, sequence)
// work items, longest (most key tiles) first, round-robin across CTAs.  The
// per-item prologue of the kernel above (TMEM allocation, barrier set-up, the
// first Q/K/V TMA round trip) and its epilogue are paid once per CTA or
// hidden: Q is double-buffered in smem so the next item's Q lands while this
// item computes, and O is double-buffered in TMEM (S0 S1 O0 O1 = 512
// columns) so the epilogue of item i overlaps the MMAs of item i+1.  All
// barrier phases run on global counters (key tiles, S tiles, P tiles, items).
struct SmemP {
  static constexpr int kQ = 0;                  // 2 buffers
  static constexpr int kK = 2 * kTile;          // 2 stages
  static constexpr int kV = kK + 2 * kTile;     // 2 stages
  static constexpr int kP = kV + 2 * kTile;
  static constexpr int kBar = kP + kTile;
  static constexpr int kBytes = kBar + 256 + 1024;
};

__device__ __forceinline__ bool item_coords(int item, int n_qt_max, int nq, int nseq, const int32_t* cu, int& seq,
                                            int& h, int& qt, int& start, int& len) {
  const int per_qt = nq * nseq;
  qt = n_qt_max - 1 - item / per_qt;  // longest first
  const int rem = item - (n_qt_max - 1 - qt) * per_qt;
  seq = rem / nq;
  h = rem - seq * nq;
  start = cu[seq];
  len = cu[seq + 1] - start;
  return qt * kT < len;
}

__global__ void __launch_bounds__(kThreads, 1)
    prefill_attn_tc_persistent(const __grid_constant__ CUtensorMap tmap, const int32_t* __restrict__ cu, int nseq,
                               int n_qt_max, int nq, int nk, __nv_bfloat16* __restrict__ out, int ldo,
                               float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemP::kBar);
  uint64_t* q_full = bars + 0;     // [2]
  uint64_t* q_empty = bars + 2;    // [2]
  uint64_t* kv_full = bars + 4;    // [2]
  uint64_t* kv_empty = bars + 6;   // [2]
  uint64_t* s_full = bars + 8;     // [2]
  uint64_t* s_free = bars + 10;    // [2]
  uint64_t* p_full = bars + 12;
  uint64_t* o_done = bars + 13;
  uint64_t* o_free = bars + 14;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int n_items = n_qt_max * nq * nseq;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int group = nq / nk;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], 4);
      mbar_init(&o_free[s], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s[2] = {tmem, tmem + 128};
  const uint32_t t_o[2] = {tmem + 256, tmem + 384};

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t keep = policy_evict_last();
      uint32_t kc = 0, ic = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        int seq, h, qt, start, len;
        if (!item_coords(item, n_qt_max, nq, nseq, cu, seq, h, qt, start, len)) continue;
        const int kvh = h / group;
        const int qcol = h * kD, kcol = (nq + kvh) * kD, vcol = (nq + nk + kvh) * kD;
        const int qb = ic & 1;
        mbar_wait(&q_empty[qb], ((ic >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], kTile);
        for (int s = 0; s < 2; ++s)
          tma_load_2d(smem + SmemP::kQ + qb * kTile + s * kSub, &tmap, &q_full[qb], qcol + s * 64, start + qt * kT,
                      keep);
        for (int j = 0; j <= qt; ++j, ++kc) {
          const int st = kc & 1;
          mbar_wait(&kv_empty[st], ((kc >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&kv_full[st], 2 * kTile);
          for (int s = 0; s < 2; ++s) {
            tma_load_2d(smem + SmemP::kK + st * kTile + s * kSub, &tmap, &kv_full[st], kcol + s * 64,
                        start + j * kT, keep);
            tma_load_2d(smem + SmemP::kV + st * kTile + s * kSub, &tmap, &kv_full[st], vcol + s * 64,
                        start + j * kT, keep);
          }
        }
        ++ic;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kT, kT);
      constexpr uint32_t idesc_o = idesc_bf16_f32(kT, kD) | (1u << 16);  // B (= V) MN-major
      const uint32_t p_base = smem_u32(smem + SmemP::kP);
      uint32_t kc = 0, sc = 0, pc = 0, ic = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        int seq, h, qt, start, len;
        if (!item_coords(item, n_qt_max, nq, nseq, cu, seq, h, qt, start, len)) continue;
        const int qb = ic & 1;
        const uint32_t q_base = smem_u32(smem + SmemP::kQ + qb * kTile);
        const uint32_t o_acc = t_o[qb];
        mbar_wait(&q_full[qb], (ic >> 1) & 1);
        // O buffer qb was read out by the epilogue of item ic - 2
        mbar_wait(&o_free[qb], ((ic >> 1) & 1) ^ 1);
        int prev_stage = 0;
        auto pv = [&](int j, int stage) {
          mbar_wait(p_full, pc & 1);
          tc_fence_after();
          const uint32_t v_base = smem_u32(smem + SmemP::kV + stage * kTile);
#pragma unroll
          for (int k = 0; k < kT / 16; ++k) {
            const uint64_t a = sdesc_k_sw128(p_base + (k >> 2) * kSub + (k & 3) * 32);
            const uint64_t b = sdesc_mn_sw128(v_base + k * 16 * 128, kSub);
            umma_bf16(o_acc, a, b, idesc_o, (j | k) != 0);
          }
          umma_commit(o_done);
          umma_commit(&kv_empty[stage]);
          ++pc;
        };
        for (int j = 0; j <= qt; ++j, ++kc, ++sc) {
          const int st = kc & 1;
          const int ss = sc & 1;
          mbar_wait(&kv_full[st], (kc >> 1) & 1);
          mbar_wait(&s_free[ss], ((sc >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_base = smem_u32(smem + SmemP::kK + st * kTile);
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint64_t a = sdesc_k_sw128(q_base + (k >> 2) * kSub + (k & 3) * 32);
            const uint64_t b = sdesc_k_sw128(k_base + (k >> 2) * kSub + (k & 3) * 32);
            umma_bf16(t_s[ss], a, b, idesc_s, k != 0);
          }
          umma_commit(&s_full[ss]);
          if (j == qt) umma_commit(&q_empty[qb]);  // last read of this Q buffer
          if (j >= 1) pv(j - 1, prev_stage);
          prev_stage = st;
        }
        pv(qt, prev_stage);
        ++ic;
      }
    }
  } else {
    // ---------------- softmax / epilogue: thread = query row ----------------
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    uint8_t* p_row = smem + SmemP::kP + r * 128;
    uint32_t sc = 0, pc = 0, ic = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      int seq, h, qt, start, len;
      if (!item_coords(item, n_qt_max, nq, nseq, cu, seq, h, qt, start, len)) continue;
      const int qb = ic & 1;
      const uint32_t o_acc = t_o[qb];
      const int q0 = qt * kT;
      const int qrow = q0 + r;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j <= qt; ++j, ++sc) {
        const int ss = sc & 1;
        mbar_wait(&s_full[ss], (sc >> 1) & 1);
        tc_fence_after();
        float s[kT];
#pragma unroll
        for (int c = 0; c < kT / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(t_s[ss] + lane_off + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(v[i]) * scale_log2;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[ss]);
        const int k0 = j * kT;
        if (j == qt || k0 + kT > len) {
#pragma unroll
          for (int i = 0; i < kT; ++i)
            if (k0 + i > qrow || k0 + i >= len) s[i] = -INFINITY;
        }
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < kT; ++i) mx = fmaxf(mx, s[i]);
        float corr = 1.f;
        const bool rescale = mx > m_used + kRescaleThreshold;
        if (rescale) {
          corr = (m_used == -INFINITY) ? 0.f : fast_exp2(m_used - mx);
          m_used = mx;
        }
        float sum = 0.f;
        uint32_t pk[kT / 2];
#pragma unroll
        for (int i = 0; i < kT; i += 2) {
          const float a = fast_exp2(s[i] - m_used), b = fast_exp2(s[i + 1] - m_used);
          sum += a + b;
          pk[i / 2] = pack_bf16x2(a, b);
        }
        // the P buffer (and O) are free once the previous P.V completed
        if (pc > 0) mbar_wait(o_done, (pc - 1) & 1);
        tc_fence_after();
        if (j >= 1 && __any_sync(0xffffffffu, rescale)) {
#pragma unroll 1
          for (int c = 0; c < kD / 32; ++c) {
            uint32_t v[32];
            tmem_ld32(o_acc + lane_off + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
            tmem_st32(o_acc + lane_off + c * 32, v);
          }
          tmem_st_wait();
        }
        l = l * corr + sum;
#pragma unroll
        for (int c = 0; c < kT / 8; ++c) {
          const int sb = c >> 3, cc = c & 7;
          uint4 val = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
          *reinterpret_cast<uint4*>(p_row + sb * kSub + ((cc ^ (r & 7)) << 4)) = val;
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        ++pc;
      }
      // epilogue: O / l, then hand the O buffer back to the MMA warp
      mbar_wait(o_done, (pc - 1) & 1);
      tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* orow = out + static_cast<size_t>(start + qrow) * ldo + h * kD;
#pragma unroll 1
      for (int c = 0; c < kD / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(o_acc + lane_off + c * 32, v);
        tmem_ld_wait();
        if (qrow < len) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 o;
            o.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
            o.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
            o.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
            o.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
            dst[q] = o;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[qb]);
      ++ic;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

int launch_prefill_attn_tc(const void* qkv, int ld, int T, int nq, int nk, const int32_t* cu, int nseq,
                           int max_len, void* out, int ldo, float scale, cudaStream_t s, bool persistent) {
  CUtensorMap map;
  int rc = encode_tmap_2d_bf16(&map, qkv, static_cast<uint64_t>(ld), static_cast<uint64_t>(T),
                               static_cast<uint64_t>(ld) * 2, 64, kT);
  if (rc) return rc;
  if (persistent) {
    static bool pattr = false;
    if (!pattr) {
      SSB_CUDA(cudaFuncSetAttribute(prefill_attn_tc_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    SmemP::kBytes));
      pattr = true;
    }
    const int n_qt = (max_len + kT - 1) / kT;
    const long items = static_cast<long>(n_qt) * nq * nseq;
    const int grid = static_cast<int>(std::min<long>(num_sms(), items));
    prefill_attn_tc_persistent<<<grid, kThreads, SmemP::kBytes, s>>>(
        map, cu, nseq, n_qt, nq, nk, static_cast<__nv_bfloat16*>(out), ldo, scale * 1.4426950408889634f);
    return check_launch("prefill_attn_tc_persistent");
  }
  static bool attr = false;
  if (!attr) {
    SSB_CUDA(cudaFuncSetAttribute(prefill_attn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::kBytes));
    attr = true;
  }
  dim3 grid((max_len + kT - 1) / kT, nq, nseq);
  prefill_attn_tc<<<grid, kThreads, Smem::kBytes, s>>>(map, cu, nq, nk, static_cast<__nv_bfloat16*>(out), ldo,
                                                        scale * 1.4426950408889634f);
  return check_launch("prefill_attn_tc");
}

}  // namespace ssb
