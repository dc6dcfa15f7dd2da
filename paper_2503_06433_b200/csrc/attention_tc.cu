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
#include <cstdlib>

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
        const int lim = min(qrow + 1, len) - k0;
#pragma unroll
        for (int i = 0; i < kT; ++i) s[i] = i < lim ? s[i] : -INFINITY;
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
// work items, longest (most key tiles) first, in snake order across CTAs (snake_item).
// Warps: 0 = TMA (lane 0 Q and K, lane 1 V: separate K and V rings, K
// three deep because S_j frees it early), 1 = MMA issue, 2-9 = softmax with
// TWO threads per query row (one per 64-key half; row max / row sum
// exchanged through smem under a 64-thread named barrier per TMEM lane
// quadrant).  Measured (tools/bench_kernels.py --what attn, 16 x 1024):
// 0.356 ms per-tile CTAs -> 0.324 persistent -> 0.281 with the split K/V
// rings; removing exp2 and the P store entirely only reaches 0.244 ms, so
// what remains is the S -> softmax -> P -> P.V dependency latency of a single
// query tile per CTA (two ping-ponged query tiles per CTA is the next step).  The
// per-item prologue of the kernel above (TMEM allocation, barrier set-up, the
// first Q/K/V TMA round trip) and its epilogue are paid once per CTA or
// hidden: Q is double-buffered in smem so the next item's Q lands while this
// item computes, and O is double-buffered in TMEM (S0 S1 O0 O1 = 512
// columns) so the epilogue of item i overlaps the MMAs of item i+1.  All
// barrier phases run on global counters (key tiles, S tiles, P tiles, items).
// Ring depths of the persistent kernel (7 tiles of 32 KiB = the smem budget):
// K is needed first (S_j) and freed first, so it gets the deepest ring.
constexpr int kKSt = 3, kVSt = 2, kPSl = 1;
struct SmemP {
  static constexpr int kQ = 0;                  // 1 buffer (the next item's Q lands while its predecessor drains)
  static constexpr int kK = kTile;              // kKSt stages
  static constexpr int kV = kK + kKSt * kTile;  // kVSt stages
  static constexpr int kP = kV + kVSt * kTile;  // kPSl slots
  static constexpr int kBar = kP + kPSl * kTile;
  static constexpr int kX = kBar + 192;         // [2 halves][128 rows] fp32 row-max / row-sum exchange (20 barriers + TMEM slot before it)
  static constexpr int kBytes = kX + 2 * 128 * 4 + 1024;  // 231,616 B: just under the 227 KB opt-in
};
constexpr int kThreadsP = 320;  // TMA warp, MMA warp, 8 softmax warps (two per TMEM lane quadrant)



// Item of round r for CTA `first` of `stride` CTAs: boustrophedon order (odd
// rounds run the CTAs backwards), so with items sorted longest first every
// CTA's total stays close to the mean -- plain round robin hands the first
// CTAs the longest item of every round (2 x 4096 causal: max 130 vs mean 114
// key tiles per CTA; snake: 116).
__device__ __forceinline__ int snake_item(int r, int first, int stride) {
  return r * stride + ((r & 1) ? stride - 1 - first : first);
}

// This CTA's work items (snake order), with the NEXT item's sequence bounds
// loaded one item ahead so the cu[] reads are off every role's critical path.
struct ItemIter {
  int first, rnd;
  int item, stride, n_items, n_qt_max, nq, nseq;
  const int32_t* cu;
  int seq, h, qt, start, len;    // current
  int n_item, n_start, n_len;    // prefetched next candidate
  __device__ void load_next() {
    if (n_item < n_items) {
      const int per_qt = nq * nseq;
      const int nqt = n_qt_max - 1 - n_item / per_qt;
      const int nseq_i = (n_item - (n_qt_max - 1 - nqt) * per_qt) / nq;
      n_start = __ldg(cu + nseq_i);
      n_len = __ldg(cu + nseq_i + 1) - n_start;
    }
  }
  // advance to the next item with work; false when none is left
  __device__ bool next() {
    while (n_item < n_items) {
      item = n_item;
      const int per_qt = nq * nseq;
      qt = n_qt_max - 1 - item / per_qt;
      const int rem = item - (n_qt_max - 1 - qt) * per_qt;
      seq = rem / nq;
      h = rem - seq * nq;
      start = n_start;
      len = n_len;
      n_item = snake_item(++rnd, first, stride);
      load_next();
      if (qt * kT < len) return true;
    }
    return false;
  }
  __device__ ItemIter(int first_, int stride_, int n_items_, int n_qt_max_, int nq_, int nseq_, const int32_t* cu_)
      : first(first_), rnd(0), item(-1), stride(stride_), n_items(n_items_), n_qt_max(n_qt_max_), nq(nq_),
        nseq(nseq_), cu(cu_), n_item(first_), n_start(0), n_len(0) {
    load_next();
  }
};

__device__ __forceinline__ void st_shared_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ float ld_shared_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

__global__ void __launch_bounds__(kThreadsP, 1)
    prefill_attn_tc_persistent(const __grid_constant__ CUtensorMap tmap, const int32_t* __restrict__ cu, int nseq,
                               int n_qt_max, int nq, int nk, __nv_bfloat16* __restrict__ out, int ldo,
                               float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemP::kBar);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;     // [kKSt] K and V rings are separate: K_j frees as soon as S_j is done
  uint64_t* k_empty = bars + 5;    // [kKSt]
  uint64_t* v_full = bars + 16;    // [kVSt] (V_j only after P_j.V_j)
  uint64_t* v_empty = bars + 18;   // [kVSt]
  uint64_t* s_full = bars + 8;     // [2]
  uint64_t* s_free = bars + 10;    // [2]
  uint64_t* p_full = bars + 12;    // [kPSl] per P slot
  uint64_t* o_done = bars + 14;    // [kPSl] per P slot: the P.V that read the slot completed
  uint64_t* o_free = bars + 20;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);

  const int n_items = n_qt_max * nq * nseq;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int group = nq / nk;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < kKSt; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kVSt; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < kPSl; ++s) {
      mbar_init(&p_full[s], 8);
      mbar_init(&o_done[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], 8);
      mbar_init(&o_free[s], 8);
    }
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
    // lane 0: Q and K tiles; lane 1: V tiles (independent rings, so a K load
    // never queues behind a V slot that is still being read by P.V)
    if (lane < 2) {
      const uint64_t keep = policy_evict_last();
      uint32_t kc = 0, ic = 0;
      ItemIter it(blockIdx.x, gridDim.x, n_items, n_qt_max, nq, nseq, cu);
      while (it.next()) {
        const int h = it.h, qt = it.qt, start = it.start;
        const int kvh = h / group;
        const int qcol = h * kD, kcol = (nq + kvh) * kD, vcol = (nq + nk + kvh) * kD;
        if (lane == 0) {
          mbar_wait(q_empty, (ic & 1) ^ 1);
          mbar_arrive_expect_tx(q_full, kTile);
          for (int s = 0; s < 2; ++s)
            tma_load_2d(smem + SmemP::kQ + s * kSub, &tmap, q_full, qcol + s * 64, start + qt * kT, keep);
        }
        uint64_t* full = lane == 0 ? k_full : v_full;
        uint64_t* empty = lane == 0 ? k_empty : v_empty;
        const int base = lane == 0 ? SmemP::kK : SmemP::kV;
        const int col = lane == 0 ? kcol : vcol;
        const uint32_t depth = lane == 0 ? kKSt : kVSt;
        for (int j = 0; j <= qt; ++j, ++kc) {
          const int st = kc % depth;
          mbar_wait(&empty[st], ((kc / depth) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[st], kTile);
          for (int s = 0; s < 2; ++s)
            tma_load_2d(smem + base + st * kTile + s * kSub, &tmap, &full[st], col + s * 64, start + j * kT, keep);
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
      ItemIter it(blockIdx.x, gridDim.x, n_items, n_qt_max, nq, nseq, cu);
      while (it.next()) {
        const int qt = it.qt;
        const int qb = ic & 1;  // O buffer
        const uint32_t q_base = smem_u32(smem + SmemP::kQ);
        const uint32_t o_acc = t_o[qb];
        mbar_wait(q_full, ic & 1);
        // O buffer qb was read out by the epilogue of item ic - 2
        mbar_wait(&o_free[qb], ((ic >> 1) & 1) ^ 1);
        auto pv = [&](int j, uint32_t vc) {
          const int slot = pc % kPSl;
          const int stage = vc % kVSt;
          mbar_wait(&v_full[stage], (vc / kVSt) & 1);
          mbar_wait(&p_full[slot], (pc / kPSl) & 1);
          tc_fence_after();
          const uint32_t v_base = smem_u32(smem + SmemP::kV + stage * kTile);
          const uint32_t pb = p_base + slot * kTile;
#pragma unroll
          for (int k = 0; k < kT / 16; ++k) {
            const uint64_t a = sdesc_k_sw128(pb + (k >> 2) * kSub + (k & 3) * 32);
            const uint64_t b = sdesc_mn_sw128(v_base + k * 16 * 128, kSub);
            umma_bf16(o_acc, a, b, idesc_o, (j | k) != 0);
          }
          umma_commit(&o_done[slot]);
          umma_commit(&v_empty[stage]);
          ++pc;
        };
        uint32_t prev_kc = 0;
        for (int j = 0; j <= qt; ++j, ++kc, ++sc) {
          const int st = kc % kKSt;
          const int ss = sc & 1;
          mbar_wait(&k_full[st], (kc / kKSt) & 1);
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
          umma_commit(&k_empty[st]);           // K_j read by S_j only
          if (j == qt) umma_commit(q_empty);  // last read of the Q buffer by this item
          if (j >= 1) pv(j - 1, prev_kc);
          prev_kc = kc;
        }
        pv(qt, prev_kc);
        ++ic;
      }
    }
  } else {
    // ------- softmax / epilogue: two threads per query row (one per column half) -------
    // warps 2..9: TMEM lane quadrant = warp & 3 (hardware rule), column half
    // = which of the two warps of that quadrant; the halves exchange row max
    // and row sum through smem under a 64-thread named barrier per quadrant.
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;
    const int c0 = half * (kT / 2);
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t xch = smem_u32(smem + SmemP::kX);  // [2][128] fp32
    uint8_t* p_row0 = smem + SmemP::kP + half * kSub + r * 128;  // keys [64*half, +64) = P sub-tile `half`
    uint32_t sc = 0, pc = 0, ic = 0;
    ItemIter it(blockIdx.x, gridDim.x, n_items, n_qt_max, nq, nseq, cu);
    while (it.next()) {
      const int h = it.h, qt = it.qt, start = it.start, len = it.len;
      const int qb = ic & 1;
      const uint32_t o_acc = t_o[qb];
      const int q0 = qt * kT;
      const int qrow = q0 + r;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j <= qt; ++j, ++sc) {
        const int ss = sc & 1;
        mbar_wait(&s_full[ss], (sc >> 1) & 1);
        tc_fence_after();
        float s[kT / 2];
#pragma unroll
        for (int c = 0; c < kT / 64; ++c) {
          uint32_t v[32];
          tmem_ld32(t_s[ss] + lane_off + c0 + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(v[i]) * scale_log2;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[ss]);
        const int k0 = j * kT + c0;
        if (j == qt || j * kT + kT > len) {
          // valid keys of this row in the tile: one compare + select per key
          const int lim = min(qrow + 1, len) - k0;
#pragma unroll
          for (int i = 0; i < kT / 2; ++i) s[i] = i < lim ? s[i] : -INFINITY;
        }
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < kT / 2; ++i) mx = fmaxf(mx, s[i]);
        st_shared_f32(xch + (half * 128 + r) * 4, mx);
        named_bar_sync(1 + quad, 64);
        mx = fmaxf(mx, ld_shared_f32(xch + ((half ^ 1) * 128 + r) * 4));
        named_bar_sync(1 + quad, 64);  // both read before either rewrites the slot
        float corr = 1.f;
        const bool rescale = mx > m_used + kRescaleThreshold;
        if (rescale) {
          corr = (m_used == -INFINITY) ? 0.f : fast_exp2(m_used - mx);
          m_used = mx;
        }
        float sum = 0.f;
        uint32_t pk[kT / 4];
#pragma unroll
#pragma unroll
        for (int i = 0; i < kT / 2; i += 2) {
          const float a = fast_exp2(s[i] - m_used), b = fast_exp2(s[i + 1] - m_used);
          sum += a + b;
          pk[i / 2] = pack_bf16x2(a, b);
        }
        // P slot is free once the P.V kPSl tiles back (its last reader) completed
        const int slot = pc % kPSl;
        if (pc >= kPSl) mbar_wait(&o_done[slot], ((pc - kPSl) / kPSl) & 1);
        tc_fence_after();
        if (j >= 1 && __any_sync(0xffffffffu, rescale)) {
          // rescaling O needs every earlier P.V of this item in it
          mbar_wait(&o_done[(pc - 1) % kPSl], ((pc - 1) / kPSl) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < kD / 64; ++c) {
            uint32_t v[32];
            tmem_ld32(o_acc + lane_off + c0 + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
            tmem_st32(o_acc + lane_off + c0 + c * 32, v);
          }
          tmem_st_wait();
        }
        l = l * corr + sum;
        // this half's 64 keys = one SW128 sub-tile row of 8 16-byte chunks
        uint8_t* p_row = p_row0 + slot * kTile;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4 val = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
          *reinterpret_cast<uint4*>(p_row + ((c ^ (r & 7)) << 4)) = val;
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[slot]);
        ++pc;
      }
      // epilogue: l = sum of both halves' partial sums; each half writes its 64 dims
      st_shared_f32(xch + (half * 128 + r) * 4, l);
      named_bar_sync(1 + quad, 64);
      l += ld_shared_f32(xch + ((half ^ 1) * 128 + r) * 4);
      mbar_wait(&o_done[(pc - 1) % kPSl], ((pc - 1) / kPSl) & 1);
      tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* orow = out + static_cast<size_t>(start + qrow) * ldo + h * kD + c0;
#pragma unroll 1
      for (int c = 0; c < kD / 64; ++c) {
        uint32_t v[32];
        tmem_ld32(o_acc + lane_off + c0 + c * 32, v);
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
      // both halves read the exchange slots before either rewrites them
      named_bar_sync(1 + quad, 64);
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

// ---------------------------------------------------------------------------
// Pair kernel (GQA group size even): a CTA computes TWO query heads of the
// same KV group for one 128-row query tile, sharing every K/V tile (128 keys)
// between them.  P never leaves tensor memory: the softmax writes it (bf16,
// 64 columns) over the first half of its own S accumulator with tcgen05.st
// and the P.V MMA reads its A operand from TMEM, so there is no P smem, no
// proxy fence, and the tensor pipe's in-order execution (P.V(j) is issued
// before S(j+1) overwrites the aliased columns) replaces the S-buffer barrier.
// Two softmax warpgroups (one per head, one thread per row) ping-pong with the
// MMA issuer: while head A turns S_A(j) into P_A(j), the tensor pipe runs
// P_B(j-1).V and S_B(j) — the S -> softmax -> P -> P.V chain of one head is
// hidden behind the other head's MMAs.
// TMEM: S/P_A, S/P_B, O_A, O_B (128 columns each) = 512.
// smem: Q_A, Q_B 64 KB; K ring 3 x 32 KB, V ring 2 x 32 KB.
// ---------------------------------------------------------------------------
constexpr int kPairKSt = 3, kPairVSt = 2;
// pair i's second exponential by polynomial when (i & kPolyMask): 0 = off.
// Measured: 1-in-4 on the FMA pipe is 5 % SLOWER (the softmax is issue- not
// MUFU-bound at 2 warps per SMSP), so every exponential uses ex2.approx.
// (template parameter POLY of the pair kernel; SSB_ATTN_POLY selects 1 or 3
// for the A/B, 0 by default)
// 3 warpgroups: WG0 = TMA (warp 0) + MMA issue (warp 1) + 2 idle warps,
// WG1 / WG2 = softmax of head A / B (one thread per query row).  Registers
// are re-balanced per warpgroup (setmaxnreg): WG0 drops to 80, the softmax
// warpgroups rise to 208 and nothing spills.  The increase draws on the
// registers the CTA was launched with (384 x 168), so 128 x 80 + 256 x 208
// must not exceed them -- a larger request blocks setmaxnreg.inc forever -- with the 168 the 320-thread layout had uniformly, the
// softmax kept loop state in local memory (ncu: LDL on the S-wait ->
// tcgen05.ld path and in the O epilogue, ~9 % of the warps' stall samples).
constexpr int kThreadsPair = 384;
constexpr int kRegsPairCtl = 80, kRegsPairSoftmax = 208;
static_assert(128 * kRegsPairCtl + 256 * kRegsPairSoftmax <= kThreadsPair * 168,
              "setmaxnreg.inc would wait for registers the CTA does not own");

struct SmemPair {
  static constexpr int kQ = 0;                          // Q_A, Q_B
  static constexpr int kK = 2 * kTile;                  // kPairKSt x 32 KB
  static constexpr int kV = kK + kPairKSt * kTile;      // kPairVSt x 32 KB
  static constexpr int kBar = kV + kPairVSt * kTile;
  static constexpr int kBytes = kBar + 256 + 1024;
};

// 2^x on the FMA/ALU pipes (x <= 0): round-to-nearest split via the 1.5*2^23
// trick, cubic on [-0.5, 0.5] (max rel. error 1.4e-4, far below bf16's 2^-9),
// exponent added in the integer domain.  Used for a fraction of the softmax
// exponentials so the MUFU pipe (16 ex2/clk/SM) is not the tile's bottleneck.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -120.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05502927f, f, 0.24225698f), f, 0.69325305f), f, 0.99995134f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}

// Packed fp32x2 arithmetic (Blackwell FFMA2 / FADD2): two lanes per
// instruction, each lane rounded exactly like fmaf / + (bit-identical).
__device__ __forceinline__ float2 ffma2_bcast(float x0, float x1, float s, float c) {
  unsigned long long x, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(x0), "f"(x1));
  asm("{\n\t.reg .b64 sc, cc;\n\tmov.b64 sc, {%2, %2};\n\tmov.b64 cc, {%3, %3};\n\t"
      "fma.rn.f32x2 %0, %1, sc, cc;\n\t}"
      : "=l"(r)
      : "l"(x), "f"(s), "f"(c));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ float2 fmul2_bcast(float x0, float x1, float s) {
  unsigned long long x, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(x0), "f"(x1));
  asm("{\n\t.reg .b64 sc;\n\tmov.b64 sc, {%2, %2};\n\tmul.rn.f32x2 %0, %1, sc;\n\t}" : "=l"(r) : "l"(x), "f"(s));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long x, y, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b.x), "f"(b.y));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}

// D (+)= A . B with A [M=128, K=16] read from TMEM (lane = row, 8 columns of
// bf16 pairs), B from shared memory.
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate ? 1 : 0));
}

// Timeline trace of CTA 0 (debug only: ssb_debug_attn_trace sets the buffer;
// null in production, one uniform branch per event).  Entry = globaltimer ns
// << 24 | event << 16 | item round << 8 | key tile; role r owns
// [r * kTraceCap, (r + 1) * kTraceCap).
constexpr int kTraceCap = 4096;
__device__ __forceinline__ void trace_ev(unsigned long long* tr, int role, int& n, int ev, int rnd, int j) {
  if (tr == nullptr || blockIdx.x != 0 || n >= kTraceCap) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  tr[role * kTraceCap + n++] = (t << 24) | (static_cast<unsigned long long>(ev & 0xFF) << 16) |
                               (static_cast<unsigned long long>(rnd & 0xFF) << 8) | (j & 0xFF);
}

struct PairIter {
  int first, rnd;
  int stride, n_items, n_qt_max, pairs, nseq;  // pairs = nq / 2
  const int32_t* cu;
  int seq, pair, qt, start, len;
  int n_item, n_start, n_len;
  __device__ void load_next() {
    if (n_item < n_items) {
      const int per_qt = pairs * nseq;
      const int q = n_qt_max - 1 - n_item / per_qt;
      const int sq = (n_item - (n_qt_max - 1 - q) * per_qt) / pairs;
      n_start = __ldg(cu + sq);
      n_len = __ldg(cu + sq + 1) - n_start;
    }
  }
  __device__ bool next() {
    while (n_item < n_items) {
      const int item = n_item;
      const int per_qt = pairs * nseq;
      qt = n_qt_max - 1 - item / per_qt;
      const int rem = item - (n_qt_max - 1 - qt) * per_qt;
      seq = rem / pairs;
      pair = rem - seq * pairs;
      start = n_start;
      len = n_len;
      n_item = snake_item(++rnd, first, stride);
      load_next();
      if (qt * kT < len) return true;
    }
    return false;
  }
  __device__ PairIter(int first_, int stride_, int n_items_, int n_qt_max_, int pairs_, int nseq_, const int32_t* cu_)
      : first(first_), rnd(0), stride(stride_), n_items(n_items_), n_qt_max(n_qt_max_), pairs(pairs_), nseq(nseq_),
        cu(cu_), n_item(first_), n_start(0), n_len(0) {
    load_next();
  }
};

template <int kPolyMask>
__global__ void __launch_bounds__(kThreadsPair, 1)
    prefill_attn_tc_pair(const __grid_constant__ CUtensorMap tmap, const int32_t* __restrict__ cu, int nseq,
                         int n_qt_max, int nq, int nk, __nv_bfloat16* __restrict__ out, int ldo, float scale_log2,
                         unsigned long long* __restrict__ trace, int st32) {
  int ntr = 0;  // this thread's trace entries
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemPair::kBar);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;    // [3]
  uint64_t* k_empty = bars + 5;   // [3]
  uint64_t* v_full = bars + 8;    // [2]
  uint64_t* v_empty = bars + 10;  // [2]
  uint64_t* s_full = bars + 12;   // [head]: S(t) of the head is in TMEM (and every earlier P.V done)
  uint64_t* p_full = bars + 14;   // [head]: P(t) written over S(t)
  uint64_t* o_done = bars + 16;   // [head]: the item's last P.V completed
  uint64_t* o_free = bars + 18;   // [head]: the epilogue read O
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  const int pairs = nq / 2;
  const int group = nq / nk;
  const int n_items = n_qt_max * pairs * nseq;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  griddep_launch_dependents();

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < kPairKSt; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < kPairVSt; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_done[i], 1);
      mbar_init(&o_free[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // columns: S/P of head h at 128 h, O of head h at 256 + 128 h
  auto t_s = [&](int head) { return tmem + 128u * head; };
  auto t_o = [&](int head) { return tmem + 256u + 128u * head; };
  if (warp < 4) {
  // ---------------- WG0: TMA producer (warp 0), MMA issuer (warp 1) ----------------
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsPairCtl));
  if (warp == 0) {
    // lane 0: Q_A, Q_B and K tiles; lane 1: V tiles
    if (lane < 2) {
      const uint64_t keep = policy_evict_last();
      uint32_t t = 0, ic = 0;
      PairIter it(blockIdx.x, gridDim.x, n_items, n_qt_max, pairs, nseq, cu);
      while (it.next()) {
        const int hA = 2 * it.pair;
        const int kvh = hA / group;
        const int n_kv = it.qt + 1;
        if (lane == 0) {
          mbar_wait(q_empty, (ic & 1) ^ 1);
          trace_ev(trace, 0, ntr, 1, ic, 0);  // Q issue
          mbar_arrive_expect_tx(q_full, 2 * kTile);
          for (int hh = 0; hh < 2; ++hh)
            for (int sb = 0; sb < 2; ++sb)
              tma_load_2d(smem + SmemPair::kQ + hh * kTile + sb * kSub, &tmap, q_full, (hA + hh) * kD + sb * 64,
                          it.start + it.qt * kT, keep);
        }
        uint64_t* full = lane == 0 ? k_full : v_full;
        uint64_t* empty = lane == 0 ? k_empty : v_empty;
        const int base = lane == 0 ? SmemPair::kK : SmemPair::kV;
        const uint32_t depth = lane == 0 ? kPairKSt : kPairVSt;
        const int col = (lane == 0 ? nq + kvh : nq + nk + kvh) * kD;
        for (int j = 0; j < n_kv; ++j, ++t) {
          const int st = t % depth;
          mbar_wait(&empty[st], ((t / depth) & 1) ^ 1);
          trace_ev(trace, lane, ntr, 2, ic, j);  // K (lane 0) / V (lane 1) issue
          mbar_arrive_expect_tx(&full[st], kTile);
          for (int sb = 0; sb < 2; ++sb)
            tma_load_2d(smem + base + st * kTile + sb * kSub, &tmap, &full[st], col + sb * 64, it.start + j * kT,
                        keep);
        }
        ++ic;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kT, kT);
      constexpr uint32_t idesc_o = idesc_bf16_f32(kT, kD) | (1u << 16);  // B (= V) MN-major
      uint32_t t = 0, ic = 0;
      PairIter it(blockIdx.x, gridDim.x, n_items, n_qt_max, pairs, nseq, cu);
      auto pv = [&](int hh, uint32_t tt, bool first) {
        // P(tt) of head hh (over its S columns) . V(tt) -> O
        if (first) mbar_wait(&o_free[hh], (ic & 1) ^ 1);  // the previous item's epilogue read O
        mbar_wait(&p_full[hh], tt & 1);
        trace_ev(trace, 2, ntr, 10 + hh, ic, tt);  // PV issue (after P ready)
        tc_fence_after();
        const uint32_t v_base = smem_u32(smem + SmemPair::kV + (tt % kPairVSt) * kTile);
#pragma unroll
        for (int k = 0; k < kT / 16; ++k) {
          const uint64_t b = sdesc_mn_sw128(v_base + k * 16 * 128, kSub);
          umma_bf16_ts(t_o(hh), t_s(hh) + 8 * k, b, idesc_o, !(first && k == 0));
        }
      };
      while (it.next()) {
        const int n_kv = it.qt + 1;
        mbar_wait(q_full, ic & 1);
        trace_ev(trace, 2, ntr, 3, ic, 0);  // Q landed
        tc_fence_after();
        const uint32_t q_base = smem_u32(smem + SmemPair::kQ);
        for (int j = 0; j < n_kv; ++j, ++t) {
          const int kst = t % kPairKSt;
          mbar_wait(&k_full[kst], (t / kPairKSt) & 1);
          trace_ev(trace, 2, ntr, 4, ic, j);  // K landed
          if (j >= 1) mbar_wait(&v_full[(t - 1) % kPairVSt], ((t - 1) / kPairVSt) & 1);
          tc_fence_after();
          const uint32_t k_base = smem_u32(smem + SmemPair::kK + kst * kTile);
          for (int hh = 0; hh < 2; ++hh) {
            if (j >= 1) pv(hh, t - 1, j == 1);  // reads P(t-1) before S(t) overwrites it
            const uint32_t qa = q_base + hh * kTile;
#pragma unroll
            for (int k = 0; k < kD / 16; ++k) {
              const uint64_t a = sdesc_k_sw128(qa + (k >> 2) * kSub + (k & 3) * 32);
              const uint64_t b = sdesc_k_sw128(k_base + (k >> 2) * kSub + (k & 3) * 32);
              umma_bf16(t_s(hh), a, b, idesc_s, k != 0);
            }
            umma_commit(&s_full[hh]);
          }
          umma_commit(&k_empty[kst]);
          if (j >= 1) umma_commit(&v_empty[(t - 1) % kPairVSt]);
          if (j == n_kv - 1) umma_commit(q_empty);
        }
        mbar_wait(&v_full[(t - 1) % kPairVSt], ((t - 1) / kPairVSt) & 1);
        tc_fence_after();
        for (int hh = 0; hh < 2; ++hh) {
          pv(hh, t - 1, n_kv == 1);
          umma_commit(&o_done[hh]);
        }
        umma_commit(&v_empty[(t - 1) % kPairVSt]);
        ++ic;
      }
    }
  }
  } else {
    // ---------------- softmax: warpgroup hh = head, thread = query row ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsPairSoftmax));
    const int hh = (warp - 4) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t s_acc = t_s(hh) + lane_off, o_acc = t_o(hh) + lane_off;
    uint32_t t = 0, ic = 0;
    PairIter it(blockIdx.x, gridDim.x, n_items, n_qt_max, pairs, nseq, cu);
    while (it.next()) {
      // item fields as scalars (kept in registers, not re-read from the
      // iterator's local-memory copy in the epilogue)
      const int qt = it.qt, len = it.len, start = it.start, pair = it.pair;
      const int n_kv = qt + 1;
      const int qrow = qt * kT + r;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kv; ++j, ++t) {
        // S(t) ready; pipe order also means every earlier P.V of this head is done (O stable)
        if (r == 0) trace_ev(trace, 3 + hh, ntr, 20, ic, j);  // softmax waits for S
        mbar_wait(&s_full[hh], t & 1);
        if (r == 0) trace_ev(trace, 3 + hh, ntr, 21, ic, j);  // S ready
        tc_fence_after();
        // raw scores: all four 32-column loads in flight, one wait.  With two
        // softmax warps per SMSP nothing hides a dependent chain, so the row
        // max and row sum below run on 8 independent accumulators, and the
        // softmax scale rides in the exponent's FMA (exp2(s * c - m)).
        float sv[kT];
        {
          uint32_t v[kT];
#pragma unroll
          for (int c = 0; c < kT / 32; ++c) tmem_ld32(s_acc + c * 32, *reinterpret_cast<uint32_t(*)[32]>(v + c * 32));
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < kT; ++i) sv[i] = __uint_as_float(v[i]);
        }
        const int k0 = j * kT;
        if (j == qt || k0 + kT > len) {
          // valid keys of this row in the tile: one compare + select per key
          // (was two compares, an add and a select: the diagonal tile's mask
          // cost more instructions than the rest of its softmax)
          const int lim = min(qrow + 1, len) - k0;
#pragma unroll
          for (int i = 0; i < kT; ++i) sv[i] = i < lim ? sv[i] : -INFINITY;
        }
        float m8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) m8[i] = sv[i];
#pragma unroll
        for (int i = 8; i < kT; ++i) m8[i & 7] = fmaxf(m8[i & 7], sv[i]);
        const float mraw = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                                 fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        const float mx = mraw * scale_log2;  // scale_log2 > 0: same argmax
        float corr = 1.f;
        const bool rescale = mx > m_used + kRescaleThreshold;
        if (rescale) {
          corr = (m_used == -INFINITY) ? 0.f : fast_exp2(m_used - mx);
          m_used = mx;
        }
        if (j >= 1 && __any_sync(0xffffffffu, rescale)) {
#pragma unroll 1
          for (int c = 0; c < kD / 32; ++c) {
            uint32_t v[32];
            tmem_ld32(o_acc + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
            tmem_st32(o_acc + c * 32, v);
          }
        }
        // row sum on 4 packed accumulator pairs (s8[2k], s8[2k+1]) -- the
        // same 8 partial sums in the same order as scalar code, half the
        // instructions; the exponent argument s * c - m likewise as FFMA2
        float2 s4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) s4[i] = make_float2(0.f, 0.f);
        const float nm = -m_used;
        // P over the first 64 columns of this head's S accumulator, 32 keys at a time
#pragma unroll
        for (int c = 0; c < kT / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 x = ffma2_bcast(sv[c * 32 + 2 * i], sv[c * 32 + 2 * i + 1], scale_log2, nm);
            const float a = fast_exp2(x.x);
            const float b = (i & kPolyMask) ? exp2_poly(x.y) : fast_exp2(x.y);
            s4[i & 3] = fadd2(s4[i & 3], make_float2(a, b));
            pk[i] = pack_bf16x2(a, b);
          }
          tmem_st16(s_acc + c * 16, pk);
        }
        tmem_st_wait();
        const float sum = ((s4[0].x + s4[0].y) + (s4[1].x + s4[1].y)) + ((s4[2].x + s4[2].y) + (s4[3].x + s4[3].y));
        l = l * corr + sum;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[hh]);
        if (r == 0) trace_ev(trace, 3 + hh, ntr, 22, ic, j);  // P written
      }
      // epilogue: O / l of this head, then hand O back to the MMA warp
      mbar_wait(&o_done[hh], ic & 1);
      if (r == 0) trace_ev(trace, 3 + hh, ntr, 23, ic, 0);  // O final
      tc_fence_after();
      const float inv = l > 0.f ? __frcp_rn(l) : 0.f;
      __nv_bfloat16* orow = out + static_cast<size_t>(start + qrow) * ldo + (2 * pair + hh) * kD;
      {
        // the whole O row: four 32-column loads in flight, one wait
        uint32_t v[kD];
#pragma unroll
        for (int c = 0; c < kD / 32; ++c) tmem_ld32(o_acc + c * 32, *reinterpret_cast<uint32_t(*)[32]>(v + c * 32));
        tmem_ld_wait();
        if (qrow < len) {
          // 32-byte stores (STG.256): each thread writes its own row, so every
          // store instruction touches 32 rows -- half the L1 store wavefronts
          // of 16-byte stores (the trace put this epilogue at ~1.5 us per item)
          if (!st32) {
            uint4* dst = reinterpret_cast<uint4*>(orow);
#pragma unroll
            for (int q = 0; q < kD / 8; ++q) {
              uint4 o;
              o.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
              o.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
              o.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
              o.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
              dst[q] = o;
            }
          } else
#pragma unroll
          for (int q = 0; q < kD / 16; ++q) {
            uint32_t o[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float2 y = fmul2_bcast(__uint_as_float(v[16 * q + 2 * k]), __uint_as_float(v[16 * q + 2 * k + 1]), inv);
              o[k] = pack_bf16x2(y.x, y.y);
            }
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(orow + 16 * q), "r"(o[0]), "r"(o[1]),
                         "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7])
                         : "memory");
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[hh]);
      if (r == 0) trace_ev(trace, 3 + hh, ntr, 24, ic, 0);  // epilogue done
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

unsigned long long* g_attn_trace = nullptr;  // ssb_debug_attn_trace

int launch_prefill_attn_tc(const void* qkv, int ld, int T, int nq, int nk, const int32_t* cu, int nseq,
                           int max_len, void* out, int ldo, float scale, cudaStream_t s, bool persistent) {
  CUtensorMap map;
  int rc = encode_tmap_2d_bf16(&map, qkv, static_cast<uint64_t>(ld), static_cast<uint64_t>(T),
                               static_cast<uint64_t>(ld) * 2, 64, kT);
  if (rc) return rc;
  static const int force_single = [] {
    const char* e = getenv("SSB_PREFILL_ATTN_SINGLE");  // A/B: 1 = one query head per CTA
    return e ? atoi(e) : 0;
  }();
  if (persistent && (nq / nk) % 2 == 0 && !force_single) {
    static const int poly = [] {
      const char* e = getenv("SSB_ATTN_POLY");  // A/B: exponentials emulated on the FMA pipe
      return e ? atoi(e) : 0;
    }();
    auto kern = poly == 3 ? prefill_attn_tc_pair<3> : poly == 1 ? prefill_attn_tc_pair<1> : prefill_attn_tc_pair<0>;
    static bool pair_attr = false;
    if (!pair_attr) {
      SSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemPair::kBytes));
      pair_attr = true;
    }
    const int n_qt = (max_len + kT - 1) / kT;
    const long items = static_cast<long>(n_qt) * (nq / 2) * nseq;
    const int grid = static_cast<int>(std::min<long>(num_sms(), items));
    kern<<<grid, kThreadsPair, SmemPair::kBytes, s>>>(map, cu, nseq, n_qt, nq, nk, static_cast<__nv_bfloat16*>(out),
                                                     ldo, scale * 1.4426950408889634f, g_attn_trace,
                                                     (reinterpret_cast<uintptr_t>(out) % 32 == 0 && ldo % 16 == 0) ? 1 : 0);
    return check_launch("prefill_attn_tc_pair");
  }
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
    prefill_attn_tc_persistent<<<grid, kThreadsP, SmemP::kBytes, s>>>(
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

// Debug only: record CTA 0's timeline of the next prefill_attn_tc_pair
// launches into buf (5 roles x 4096 u64 entries, zeroed by the caller); null
// turns it off.
extern "C" int ssb_debug_attn_trace(void* buf) {
  ssb::g_attn_trace = static_cast<unsigned long long*>(buf);
  return 0;
}
