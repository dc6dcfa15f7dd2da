// Persistent, warp-specialised bf16 GEMM on the 5th-generation tensor cores.
//
//   C[M, N] = A[M, K] . B[N, K]^T  (+ residual | SiLU(gate) * up)
//
// A = activations (row-major, K contiguous), B = a weight matrix stored
// [out_features, in_features] (K contiguous): both operands are K-major.
// This kernel replaces the reference's analytic linear-layer terms
// (perf.py:59-65 weight traffic, perf.py:92-111 linear compute) with the real
// contraction: QKV / O / gate_up / down projections and the lm_head.
//
// Structure (one CTA per SM, 6 warps):
//   warp 0      TMA producer: A tile 128x64 and B tile BNx64 per k-block into a
//               STAGES-deep ring of 128B-swizzled shared-memory buffers.
//   warp 1      allocates TMEM; one lane issues tcgen05.mma (M=128, N=BN,
//               K=16) into a double-buffered fp32 accumulator in TMEM and
//               commits completion to mbarriers.
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 32 columns, fused epilogue,
//               bf16 stores.  Accumulator double buffering lets the epilogue
//               of tile i overlap the MMAs of tile i+1.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "seesaw_b200.h"

namespace ssb {

int encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                        uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;       // 64 bf16 = 128 B = one swizzle row
constexpr int kUmmaK = 16;
constexpr int kThreads = 192;
constexpr int kGroupM = 16;   // tile rasterisation: 16 M-tiles share a B band in L2
constexpr size_t kCounterBytes = 64 * 1024;  // split-K tile counters at the head of the workspace

constexpr int pow2_at_least(int x) { return x <= 32 ? 32 : x <= 64 ? 64 : x <= 128 ? 128 : x <= 256 ? 256 : 512; }

// MODE 0: one CTA per tile.  MODE 1: CTA pair, B tile multicast (each CTA
// still holds all BN rows of B).  MODE 2: CTA pair running cta_group::2 MMAs
// (M = 256 per pair): each CTA holds its 128 rows of A and HALF of B.
template <int BN, int MODE = 0>
struct Cfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = (MODE == 2 ? BN / 2 : BN) * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // as many stages as ~220 KB of shared memory holds (>= 4)
  static constexpr int kStages = (220 * 1024) / kStageBytes > 8 ? 8 : (220 * 1024) / kStageBytes;
  static constexpr int kTmemCols = pow2_at_least(2 * BN);
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align slack*/ + 256 /*barriers*/;
};

// SSB_EPI_ROPE_KV: the accumulator columns are the packed [nq | nk | nk]
// heads (head_dim 128) of a QKV projection.  q and k heads get rotate-half
// RoPE at positions[row]; k and v heads are also appended to the paged KV
// pool at slots[row] (negative = skip).  Values are rounded to bf16 BEFORE
// the rotation, so the result is bit-identical to a bf16 GEMM store followed
// by ssb_rope_kv_append.
struct RopeKV {
  const int32_t* pos;
  const float* cos;
  const float* sin;
  int max_pos;
  __nv_bfloat16* pool;
  int n_layers, n_heads, block_size, layer;
  const int64_t* slots;
  int nq, nk;
};

struct Params {
  void* C;
  const void* R;   // residual (may alias C); only for SSB_EPI_RESIDUAL
  int M, N, K;     // N = columns of the accumulator (gate_up width for SiLU)
  int ldc, ldr;    // elements
  int epi;
  int tiles_m, tiles_n;
  int group_n;     // rasterisation band orientation (see tile_coords)
  int group_size;  // tiles of the band dimension per band
  // split-K: every output tile is computed as `splits` partial sums over
  // k-block ranges of kb_per_split; the last warp to finish a tile quadrant
  // (counter) reduces the fp32 partials in split order and runs the epilogue
  int splits, kb_per_split;
  int full_units;  // units [0, full_units) are whole tiles; the rest split `splits` ways
                   // (0: every tile split; all units: no split) -- "tail split" fills the last wave
  float* ws;       // [tiles_m * tiles_n][splits][128][BN] fp32 partials
  int* counters;   // [tiles_m * tiles_n][4], zero between launches (self-resetting)
  RopeKV rk;       // SSB_EPI_ROPE_KV only
  int arg_base;    // SSB_EPI_ARGMAX: global index of accumulator column 0
  int pol_mode;    // L2 cache-policy variant of the operand loads (see producer)
  // RMSNorm folded into the GEMMs (ssb_rownorm): ss_out[row * tiles_n + tn]
  // = sum of squares of the stored bf16 row segment (residual epilogue);
  // ss_in scales every accumulator row by 1/sqrt(sum(ss_in row)/hidden + eps)
  float* ss_out;
  const float* ss_in;
  int ss_in_parts;
  float ss_hidden, ss_eps;
  // serpentine K: a CTA's odd-numbered units walk their k-blocks backwards,
  // so a wave starts on the operand slabs the previous wave touched last
  // (still in L2) instead of the ones it evicted first
  int kserp;
  int num_kb;      // k-blocks of K
  int unit_tiles;  // output tiles of the schedule (CTA-pair tiles when MC = 2)
  // stream-K: after sk_dp_rounds rounds of whole tiles (group g: tiles
  // g + r * groups), the remaining tiles' k-blocks [sk_tile0 * num_kb, ...)
  // -- sk_W of them -- are cut into `groups` contiguous, equal ranges, one
  // per group; a tile whose k-blocks span several groups is reduced by the
  // last contributor to finish (see reduce_parts)
  int sk;
  int sk_dp_rounds;
  int sk_tile0;
  long long sk_W;
};

// Grouped rasterisation: kGroupM tiles of the "band" dimension share one
// operand band in L2 while the other operand streams.  group_n = 0 bands along
// M (A band resident, B streamed once per band); group_n = 1 bands along N.
__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int group_n, int group_size, int& tm,
                                            int& tn) {
  const int kGroupM = group_size;
  const int band_tiles = group_n ? tiles_n : tiles_m;
  const int other_tiles = group_n ? tiles_m : tiles_n;
  const int per_group = kGroupM * other_tiles;
  const int group = t / per_group;
  const int first = group * kGroupM;
  const int gsize = min(band_tiles - first, kGroupM);
  const int local = t - group * per_group;
  const int b = first + local % gsize;
  const int o = local / gsize;
  tm = group_n ? o : b;
  tn = group_n ? b : o;
}

// Unit u of the persistent schedule -> (unit tile, split index, split count).
__device__ __forceinline__ void unit_decode(const Params& p, int u, int& t, int& split, int& nsplit) {
  if (u < p.full_units) {
    t = u;
    split = 0;
    nsplit = 1;
  } else {
    const int v = u - p.full_units;
    t = p.full_units + v / p.splits;
    split = v - (v / p.splits) * p.splits;
    nsplit = p.splits;
  }
}

// One unit of a group's persistent schedule: a unit tile, its k-block range,
// and -- when the tile is shared (split-K / stream-K) -- the contributors.
// Contributor j's fp32 partial lives at CTA slot slotA + j * slotS (+ slotD
// for j = 0) of the workspace, contributors numbered in k order.
struct Work {
  int t, kb0, kb1;
  int nparts, part;
  int slotA, slotS, slotD;
};

__device__ __forceinline__ long long sk_start(const Params& p, int g, int G) {
  return p.sk_W * g / G;
}
// the group whose stream-K range holds linear k-block x
__device__ __forceinline__ int sk_group_of(const Params& p, long long x, int G) {
  int g = static_cast<int>(x * G / p.sk_W);
  while (g + 1 < G && sk_start(p, g + 1, G) <= x) ++g;
  while (g > 0 && sk_start(p, g, G) > x) --g;
  return g;
}

__device__ __forceinline__ int num_work(const Params& p, int g, int G) {
  if (!p.sk) {
    const int units = p.full_units + (p.unit_tiles - p.full_units) * p.splits;
    return g < units ? (units - 1 - g) / G + 1 : 0;
  }
  const long long s = sk_start(p, g, G), e = sk_start(p, g + 1, G);
  return p.sk_dp_rounds + (e > s ? static_cast<int>((e - 1) / p.num_kb - s / p.num_kb + 1) : 0);
}

template <int MC>
__device__ __forceinline__ void get_work(const Params& p, int g, int G, int i, int crank, Work& w) {
  if (!p.sk) {
    int split, nsplit;
    unit_decode(p, g + i * G, w.t, split, nsplit);
    w.nparts = nsplit;
    w.part = split;
    w.kb0 = nsplit > 1 ? split * p.kb_per_split : 0;
    w.kb1 = nsplit > 1 ? min(p.num_kb, w.kb0 + p.kb_per_split) : p.num_kb;
    w.slotA = ((w.t - p.full_units) * MC + crank) * nsplit;
    w.slotS = 1;
    w.slotD = 0;
    return;
  }
  if (i < p.sk_dp_rounds) {
    w.t = g + i * G;
    w.kb0 = 0;
    w.kb1 = p.num_kb;
    w.nparts = 1;
    w.part = 0;
    w.slotA = w.slotS = w.slotD = 0;
    return;
  }
  const long long s = sk_start(p, g, G), e = sk_start(p, g + 1, G);
  const int nkb = p.num_kb;
  const long long ts = s / nkb + (i - p.sk_dp_rounds);
  const long long lo = ts * nkb, hi = lo + nkb;
  w.t = p.sk_tile0 + static_cast<int>(ts);
  w.kb0 = static_cast<int>((s > lo ? s : lo) - lo);
  w.kb1 = static_cast<int>((e < hi ? e : hi) - lo);
  const int ga = sk_group_of(p, lo, G), gb = sk_group_of(p, hi - 1, G);
  w.nparts = gb - ga + 1;
  w.part = g - ga;
  // slots: group g owns two, (2g) for the tile its range starts in and
  // (2g + 1) for the tile it ends in; contributor 0 may be either, every
  // later contributor's range starts inside this tile
  const int w0 = (sk_start(p, ga, G) / nkb == ts) ? 0 : 1;
  w.slotA = 2 * ga * MC + crank;
  w.slotS = 2 * MC;
  w.slotD = w0 * MC;
}

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

// 1/rms of row `row` from the producer's per-tile sums of squares, in the
// rmsnorm kernel's formula (parts summed in order: deterministic).
__device__ __forceinline__ float row_rms_scale(const Params& p, int row) {
  const float* src = p.ss_in + static_cast<size_t>(row) * p.ss_in_parts;
  const int n = p.ss_in_parts;
  float ss = 0.f;
  int j = 0;
  if ((n & 3) == 0) {  // 16-byte rows: 8 independent vector loads in flight
    const float4* s4 = reinterpret_cast<const float4*>(src);
    for (; j + 32 <= n; j += 32) {
      float4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = s4[j / 4 + i];
#pragma unroll
      for (int i = 0; i < 8; ++i) ss = ss + v[i].x + v[i].y + v[i].z + v[i].w;
    }
    for (; j < n; j += 4) {
      const float4 v = s4[j / 4];
      ss = ss + v.x + v.y + v.z + v.w;
    }
  } else {
    for (; j < n; ++j) ss += src[j];
  }
  return 1.0f / sqrtf(__fadd_rn(__fdiv_rn(ss, p.ss_hidden), p.ss_eps));
}

__device__ __forceinline__ void scale32(float (&f)[32], float s) {
#pragma unroll
  for (int j = 0; j < 32; ++j) f[j] = __fmul_rn(f[j], s);
}

__device__ __forceinline__ float sq_bf16x2(uint32_t v, float ss) {
  const float a = bf16_lo(v), b = bf16_hi(v);
  return fmaf(b, b, fmaf(a, a, ss));
}

// Final epilogue of 32 accumulator columns [col, col+32) of one row; `ss`
// accumulates the squares of the stored bf16 values when p.ss_out is set.
__device__ __forceinline__ void store_cols(const Params& p, int row, int col, float (&f)[32], float& ss) {
  __nv_bfloat16* crow = reinterpret_cast<__nv_bfloat16*>(p.C) + static_cast<size_t>(row) * p.ldc;
  const __nv_bfloat16* rrow =
      p.epi == SSB_EPI_RESIDUAL ? reinterpret_cast<const __nv_bfloat16*>(p.R) + static_cast<size_t>(row) * p.ldr
                                : nullptr;
  if (p.epi == SSB_EPI_F32) {
    float* frow = reinterpret_cast<float*>(p.C) + static_cast<size_t>(row) * p.ldc;
    if (col + 32 <= p.N) {
      float4* dst = reinterpret_cast<float4*>(frow + col);
#pragma unroll
      for (int v = 0; v < 8; ++v) dst[v] = make_float4(f[4 * v], f[4 * v + 1], f[4 * v + 2], f[4 * v + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col + j < p.N) frow[col + j] = f[j];
    }
  } else if (col + 32 <= p.N) {
    if (rrow) {
      const uint4* src = reinterpret_cast<const uint4*>(rrow + col);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint4 r = src[v];
        f[8 * v + 0] += bf16_lo(r.x); f[8 * v + 1] += bf16_hi(r.x);
        f[8 * v + 2] += bf16_lo(r.y); f[8 * v + 3] += bf16_hi(r.y);
        f[8 * v + 4] += bf16_lo(r.z); f[8 * v + 5] += bf16_hi(r.z);
        f[8 * v + 6] += bf16_lo(r.w); f[8 * v + 7] += bf16_hi(r.w);
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(crow + col);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      uint4 o;
      o.x = pack_bf16x2(f[8 * v + 0], f[8 * v + 1]);
      o.y = pack_bf16x2(f[8 * v + 2], f[8 * v + 3]);
      o.z = pack_bf16x2(f[8 * v + 4], f[8 * v + 5]);
      o.w = pack_bf16x2(f[8 * v + 6], f[8 * v + 7]);
      dst[v] = o;
      if (p.ss_out) ss = sq_bf16x2(o.w, sq_bf16x2(o.z, sq_bf16x2(o.y, sq_bf16x2(o.x, ss))));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (col + j < p.N) {
        float v = f[j];
        if (rrow) v += __bfloat162float(rrow[col + j]);
        const __nv_bfloat16 o = __float2bfloat16_rn(v);
        crow[col + j] = o;
        const float q = __bfloat162float(o);
        ss = fmaf(q, q, ss);
      }
    }
  }
}

// SiLU(gate) * up of 32 (gate, up) column pairs -> output columns [col, col+32).
__device__ __forceinline__ void store_silu(const Params& p, int row, int col, const float (&g)[32],
                                           const float (&u)[32]) {
  __nv_bfloat16* crow = reinterpret_cast<__nv_bfloat16*>(p.C) + static_cast<size_t>(row) * p.ldc;
  const int ncols = p.N / 2;
  if (col + 32 <= ncols) {
    uint4* dst = reinterpret_cast<uint4*>(crow + col);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      uint4 o;
      o.x = pack_bf16x2(silu(g[8 * v + 0]) * u[8 * v + 0], silu(g[8 * v + 1]) * u[8 * v + 1]);
      o.y = pack_bf16x2(silu(g[8 * v + 2]) * u[8 * v + 2], silu(g[8 * v + 3]) * u[8 * v + 3]);
      o.z = pack_bf16x2(silu(g[8 * v + 4]) * u[8 * v + 4], silu(g[8 * v + 5]) * u[8 * v + 5]);
      o.w = pack_bf16x2(silu(g[8 * v + 6]) * u[8 * v + 6], silu(g[8 * v + 7]) * u[8 * v + 7]);
      dst[v] = o;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col + j < ncols) crow[col + j] = __float2bfloat16_rn(silu(g[j]) * u[j]);
  }
}

// SSB_EPI_ARGMAX: running (value, index) key of one row over 32 columns.
// key = orderable(value) << 32 | ~index, so a 64-bit max picks the largest
// logit and, on ties, the smallest index (ssb_argmax_rows' rule).
__device__ __forceinline__ unsigned long long argmax_key(float v, int idx) {
  if (v == 0.f) v = 0.f;  // -0 == +0
  const uint32_t b = __float_as_uint(v);
  const uint32_t ord = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return (static_cast<unsigned long long>(ord) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(idx));
}
__device__ __forceinline__ void argmax_cols(const Params& p, int col, const float (&f)[32], unsigned long long& best) {
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    if (col + j < p.N) {
      const unsigned long long k = argmax_key(f[j], p.arg_base + col + j);
      best = k > best ? k : best;
    }
  }
}

// RoPE + KV append of one row's 32-column pair (lo = head columns [i0, i0+32),
// hi = [i0+64, i0+96)) of head `head`, i0 in {0, 32}.
__device__ __forceinline__ void store_rope(const Params& p, int row, int col_lo, const float (&lo)[32],
                                           const float (&hi)[32]) {
  constexpr int kHd = 128, kHalf = 64;
  const RopeKV& rk = p.rk;
  const int head = col_lo / kHd;
  const int i0 = col_lo - head * kHd;
  __nv_bfloat16* crow = reinterpret_cast<__nv_bfloat16*>(p.C) + static_cast<size_t>(row) * p.ldc;
  uint32_t olo[16], ohi[16];
  if (head < rk.nq + rk.nk) {
    const int ps = min(max(rk.pos[row], 0), rk.max_pos - 1);
    const float4* cr = reinterpret_cast<const float4*>(rk.cos + static_cast<size_t>(ps) * kHalf + i0);
    const float4* sr = reinterpret_cast<const float4*>(rk.sin + static_cast<size_t>(ps) * kHalf + i0);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const float4 c4 = __ldg(cr + v), s4 = __ldg(sr + v);
      const float cc[4] = {c4.x, c4.y, c4.z, c4.w}, ss[4] = {s4.x, s4.y, s4.z, s4.w};
      float ylo[4], yhi[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float a = __bfloat162float(__float2bfloat16_rn(lo[4 * v + k]));
        const float b = __bfloat162float(__float2bfloat16_rn(hi[4 * v + k]));
        ylo[k] = __fsub_rn(__fmul_rn(a, cc[k]), __fmul_rn(b, ss[k]));
        yhi[k] = __fadd_rn(__fmul_rn(b, cc[k]), __fmul_rn(a, ss[k]));
      }
      olo[2 * v] = pack_bf16x2(ylo[0], ylo[1]);
      olo[2 * v + 1] = pack_bf16x2(ylo[2], ylo[3]);
      ohi[2 * v] = pack_bf16x2(yhi[0], yhi[1]);
      ohi[2 * v + 1] = pack_bf16x2(yhi[2], yhi[3]);
    }
  } else {
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      olo[v] = pack_bf16x2(lo[2 * v], lo[2 * v + 1]);
      ohi[v] = pack_bf16x2(hi[2 * v], hi[2 * v + 1]);
    }
  }
  uint4* dlo = reinterpret_cast<uint4*>(crow + col_lo);
  uint4* dhi = reinterpret_cast<uint4*>(crow + col_lo + kHalf);
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    dlo[v] = make_uint4(olo[4 * v], olo[4 * v + 1], olo[4 * v + 2], olo[4 * v + 3]);
    dhi[v] = make_uint4(ohi[4 * v], ohi[4 * v + 1], ohi[4 * v + 2], ohi[4 * v + 3]);
  }
  if (head >= rk.nq && rk.slots) {
    const int64_t slot = rk.slots[row];
    if (slot >= 0) {
      const int64_t blk = slot / rk.block_size;
      const int off = static_cast<int>(slot - blk * rk.block_size);
      const int kv = head >= rk.nq + rk.nk ? 1 : 0;
      const int kvh = head - rk.nq - kv * rk.nk;
      const int64_t plane = static_cast<int64_t>(rk.block_size) * kHd;
      __nv_bfloat16* dst = rk.pool + ((blk * rk.n_layers + rk.layer) * 2 + kv) * rk.n_heads * plane +
                           kvh * plane + static_cast<int64_t>(off) * kHd + i0;
      uint4* plo = reinterpret_cast<uint4*>(dst);
      uint4* phi = reinterpret_cast<uint4*>(dst + kHalf);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        plo[v] = make_uint4(olo[4 * v], olo[4 * v + 1], olo[4 * v + 2], olo[4 * v + 3]);
        phi[v] = make_uint4(ohi[4 * v], ohi[4 * v + 1], ohi[4 * v + 2], ohi[4 * v + 3]);
      }
    }
  }
}

// Shared tiles (split-K / stream-K).  Partial layout per CTA slot:
// [BN/4 float4 columns][128 rows] of float4, so one warp's store or load of a
// column group covers 512 contiguous bytes (32 rows).  Each epilogue warp
// (one TMEM lane quadrant = 32 rows) of a contributor:
//   * if every other contributor already published (counter = nparts - 1),
//     keeps its accumulator in TMEM and reduces at once;
//   * else spills its fp32 partial, publishes (fence + counter), and the
//     warp that brings the counter to nparts reduces -- its own partial
//     still in TMEM.
// The reducer adds the partials in contributor (= k) order, its own at its
// position, and writes the sum back into its TMEM accumulator; the regular
// whole-tile epilogue then runs from TMEM.  The sum order is fixed by the
// plan, so the result is bitwise independent of which contributor finished
// last.  Returns false when another warp will reduce this tile quadrant.
template <int BN>
__device__ __forceinline__ bool reduce_parts(const Params& p, const Work& w, int tile, int q, int lane,
                                             uint32_t tbase) {
  constexpr size_t stride4 = static_cast<size_t>(kBM) * BN / 4;  // float4 per CTA slot
  int* ctr = p.counters + tile * 4 + q;
  float4* ws4 = reinterpret_cast<float4*>(p.ws) + q * 32 + lane;
  int seen = 0;
  if (lane == 0) seen = ld_acquire_gpu(ctr);
  seen = __shfl_sync(0xffffffffu, seen, 0);
  if (seen != w.nparts - 1) {
    float4* mine = ws4 + static_cast<size_t>(w.slotA + w.part * w.slotS + (w.part == 0 ? w.slotD : 0)) * stride4;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t a[32];
      tmem_ld32(tbase + c * 32, a);
      tmem_ld_wait();
#pragma unroll
      for (int v = 0; v < 8; ++v)
        __stcg(mine + (c * 8 + v) * kBM, make_float4(__uint_as_float(a[4 * v]), __uint_as_float(a[4 * v + 1]),
                                                     __uint_as_float(a[4 * v + 2]), __uint_as_float(a[4 * v + 3])));
    }
    __threadfence();
    __syncwarp();
    int prev = 0;
    if (lane == 0) prev = atomicAdd(ctr, 1);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != w.nparts - 1) return false;
  }
  __threadfence();
  if (lane == 0) *ctr = 0;  // every contributor arrived: zero for the next launch
  const int n = w.nparts, me = w.part;
  auto part_ptr = [&](int j) {
    return ws4 + static_cast<size_t>(w.slotA + j * w.slotS + (j == 0 ? w.slotD : 0)) * stride4;
  };
  if (n == 2) {
    // one other partial: software-pipelined, chunk c+1 in flight while
    // chunk c is summed and written back
    const float4* o = part_ptr(1 - me);
    float4 x[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) x[v] = __ldcg(o + v * kBM);
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t a[32];
      tmem_ld32(tbase + c * 32, a);
      float4 y[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) y[v] = x[v];
      if (c + 1 < BN / 32) {
#pragma unroll
        for (int v = 0; v < 8; ++v) x[v] = __ldcg(o + ((c + 1) * 8 + v) * kBM);
      }
      tmem_ld_wait();
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const float yy[4] = {y[v].x, y[v].y, y[v].z, y[v].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float mine_v = __uint_as_float(a[4 * v + k]);
          a[4 * v + k] = __float_as_uint(me == 0 ? mine_v + yy[k] : yy[k] + mine_v);
        }
      }
      tmem_st32(tbase + c * 32, a);
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t a[32];
      tmem_ld32(tbase + c * 32, a);
      tmem_ld_wait();
      float f[32];
#pragma unroll 1
      for (int j = 0; j < n; ++j) {
        float xs[32];
        if (j == me) {
#pragma unroll
          for (int k = 0; k < 32; ++k) xs[k] = __uint_as_float(a[k]);
        } else {
          const float4* src = part_ptr(j);
          float4 x[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) x[v] = __ldcg(src + (c * 8 + v) * kBM);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            xs[4 * v] = x[v].x; xs[4 * v + 1] = x[v].y; xs[4 * v + 2] = x[v].z; xs[4 * v + 3] = x[v].w;
          }
        }
        if (j == 0) {
#pragma unroll
          for (int k = 0; k < 32; ++k) f[k] = xs[k];
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) f[k] += xs[k];
        }
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) a[k] = __float_as_uint(f[k]);
      tmem_st32(tbase + c * 32, a);
    }
  }
  tmem_st_wait();
  return true;
}

// MC = CTAs per cluster along M.  With MC = 2 the two CTAs of a cluster
// compute vertically adjacent M tiles of the same N tile: each loads its own
// A tile and HALF of the shared B tile, multicast into both CTAs' smem
// (TMA .multicast::cluster), halving B's L2->SM traffic.  A stage may be
// refilled only when both CTAs' MMAs released it, so MMA completion is
// committed to the empty barrier of both CTAs.
//
// MODE 2 (cta_group::2): the pair computes a 256 x BN tile with single-thread
// MMAs issued by the leader CTA (M = 256 split by rows across the two CTAs'
// TMEM, B split by columns across their smem), so each SM ingests 16 KB of A
// and BN/2 x 128 B of B per k-block instead of 16 KB + BN x 128 B.  Both CTAs'
// TMA loads complete on the LEADER's full barrier; the leader's commits
// arrive on both CTAs' empty / tmem-full barriers; both epilogues release the
// leader's tmem-empty barrier.
template <int BN, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_sm100(const __grid_constant__ CUtensorMap tmap_a,
                    const __grid_constant__ CUtensorMap tmap_b, const Params p) {
  using C = Cfg<BN, MODE>;
  constexpr int MC = MODE ? 2 : 1;
  const int crank = MC > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int cid = blockIdx.x / MC;
  const int nclusters = gridDim.x / MC;
  const int units_m = (p.tiles_m + MC - 1) / MC;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the SW128 atoms.
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + C::kStages * C::kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::kStages;
  uint64_t* tfull = bars + 2 * C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nw = num_work(p, cid, nclusters);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_b);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      // MODE 1: both CTAs' MMAs release a multicast stage; MODE 2: the
      // leader's single commit arrives on both CTAs' barriers
      mbar_init(&empty[s], MODE == 1 ? 2 : 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], MODE == 2 ? 8 : 4);  // one arrive per epilogue warp (of both CTAs)
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if (MODE == 2)
      tmem_alloc_cg2(tmem_slot, C::kTmemCols);
    else
      tmem_alloc(tmem_slot, C::kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  if (MC > 1) cluster_sync_all();  // peer barriers initialised before any multicast lands
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: everything above (barrier init, TMEM allocation, descriptor
  // prefetch) overlapped the previous kernel; from here on global memory the
  // previous kernel writes (A, the residual / output) is touched
  griddep_launch_dependents();
  if (warp != 1) griddep_wait();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      // the banded operand is re-read by every tile of its band: keep it in
      // L2; the streamed operand is read by the band's tiles in one wave
      // L2 policy of the operand loads (SSB_GEMM_POLICY): 2 (default) = both
      // evict_last; 0 = banded operand evict_last + streamed operand
      // evict_first; 1 = both evict_normal; 3 = streamed operand evict_normal.
      // Measured on the 8B prefill projections (tools/gemm_traffic.sh,
      // tools/gemm_sustained.py): evict_first on the streamed operand lets its
      // tiles leave L2 before the band's other tiles reuse them (gate/up: 8-9
      // GB of DRAM reads per launch vs 3.3-3.9 GB with 2), and under the 1 kW
      // cap that DRAM power costs SM clock: mode 2 is +5% sustained TFLOP/s.
      uint64_t pol_a, pol_b;
      if (p.pol_mode == 1) {
        pol_a = pol_b = policy_evict_normal();
      } else if (p.pol_mode == 2) {
        pol_a = pol_b = policy_evict_last();
      } else {
        const uint64_t stream_pol = p.pol_mode == 3 ? policy_evict_normal() : policy_evict_first();
        pol_a = p.group_n ? stream_pol : policy_evict_last();
        pol_b = p.group_n ? policy_evict_last() : stream_pol;
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < nw; ++i) {
        Work w;
        get_work<MC>(p, cid, nclusters, i, crank, w);
        int um, tn;
        tile_coords(w.t, units_m, p.tiles_n, p.group_n, p.group_size, um, tn);
        const int tm = um * MC + crank;
        const int kb0 = w.kb0, kb1 = w.kb1;
        const bool rev = p.kserp && (i & 1);
        for (int i = kb0; i < kb1; ++i) {
          // (the MMA warp only counts k-blocks: the order is the producer's)
          const int kb = rev ? kb1 - 1 - (i - kb0) : i;
          mbar_wait(&empty[stage], phase ^ 1);
          if (MODE == 2) {
            // both halves land on the leader's full barrier
            const uint32_t lbar = mapa_shared(&full[stage], 0);
            if (crank == 0) mbar_arrive_expect_tx(&full[stage], 2 * C::kStageBytes);
            tma_load_2d_cg2(smem_a + stage * C::kABytes, &tmap_a, lbar, kb * kBK, tm * kBM, pol_a);
            tma_load_2d_cg2(smem_b + stage * C::kBBytes, &tmap_b, lbar, kb * kBK, tn * BN + crank * (BN / 2),
                            pol_b);
            if (++stage == C::kStages) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
          tma_load_2d(smem_a + stage * C::kABytes, &tmap_a, &full[stage], kb * kBK, tm * kBM,
                      pol_a);
          if (MC == 1) {
            tma_load_2d(smem_b + stage * C::kBBytes, &tmap_b, &full[stage], kb * kBK, tn * BN,
                        pol_b);
          } else {
            // my half of the B tile, written into both CTAs of the cluster
            tma_load_2d_mc(smem_b + stage * C::kBBytes + crank * (C::kBBytes / MC), &tmap_b, &full[stage],
                           kb * kBK, tn * BN + crank * (BN / MC), static_cast<uint16_t>((1u << MC) - 1), pol_b);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && (MODE != 2 || crank == 0)) {
      // ---------------- MMA issuer (leader CTA only in MODE 2) ----------------
      constexpr uint32_t idesc = idesc_bf16_f32(MODE == 2 ? 2 * kBM : kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int i = 0; i < nw; ++i) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        Work w;
        get_work<MC>(p, cid, nclusters, i, crank, w);
        const int kb0 = w.kb0, kb1 = w.kb1;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = sdesc_k_sw128(smem_u32(smem_a + stage * C::kABytes));
          const uint64_t bdesc = sdesc_k_sw128(smem_u32(smem_b + stage * C::kBBytes));
#pragma unroll
          for (int k = 0; k < kBK / kUmmaK; ++k) {
            // advance 16 elements (32 B) along K inside the 128 B swizzle row
            if (MODE == 2)
              umma_bf16_cg2(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb != kb0) || (k != 0));
            else
              umma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb != kb0) || (k != 0));
          }
          // frees the smem slot (in every CTA that received data into it)
          if (MODE == 2)
            umma_commit_cg2_mc(&empty[stage], 0x3);
          else if (MC == 1)
            umma_commit(&empty[stage]);
          else
            umma_commit_mc(&empty[stage], static_cast<uint16_t>((1u << MC) - 1));
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        // accumulator ready for the epilogue(s)
        if (MODE == 2)
          umma_commit_cg2_mc(&tfull[acc], 0x3);
        else
          umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ---------------- epilogue warps ----------------
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int i = 0; i < nw; ++i) {
      Work w;
      get_work<MC>(p, cid, nclusters, i, crank, w);
      int um, tn;
      tile_coords(w.t, units_m, p.tiles_n, p.group_n, p.group_size, um, tn);
      const int tm = um * MC + crank;
      const int row = tm * kBM + q * 32 + lane;
      const bool row_ok = row < p.M;
      // the row's 1/rms: loads issued while the tile's MMAs still run
      const float rs = (p.ss_in != nullptr && row_ok) ? row_rms_scale(p, row) : 1.f;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      float ss = 0.f;
      // a shared tile: only the last contributor (holding the sum in TMEM) stores
      if (w.nparts == 1 || reduce_parts<BN>(p, w, tm * p.tiles_n + tn, q, lane, tbase)) {
        if (p.epi == SSB_EPI_ARGMAX) {
          unsigned long long best = 0;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t a[32];
            tmem_ld32(tbase + c * 32, a);
            tmem_ld_wait();
            float f[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(a[j]);
            if (p.ss_in) scale32(f, rs);
            argmax_cols(p, tn * BN + c * 32, f, best);
          }
          if (row_ok && best) atomicMax(reinterpret_cast<unsigned long long*>(p.C) + row, best);
        } else if (p.epi == SSB_EPI_ROPE_KV) {
          // per 128-column head: chunk pairs (0, 2) and (1, 3) are the
          // rotate-half partners (i, i + 64)
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            if (c & 2) continue;
            uint32_t lo[32], hi[32];
            tmem_ld32(tbase + c * 32, lo);
            tmem_ld32(tbase + (c + 2) * 32, hi);
            tmem_ld_wait();
            float fl[32], fh[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              fl[j] = __uint_as_float(lo[j]);
              fh[j] = __uint_as_float(hi[j]);
            }
            if (p.ss_in) {
              scale32(fl, rs);
              scale32(fh, rs);
            }
            if (row_ok && tn * BN + c * 32 < p.N) store_rope(p, row, tn * BN + c * 32, fl, fh);
          }
        } else if (p.epi == SSB_EPI_SILU_MUL) {
          // accumulator columns come in (32 gate, 32 up) pairs -> 32 outputs
#pragma unroll 1
          for (int c = 0; c < BN / 64; ++c) {
            uint32_t g[32], v[32];
            tmem_ld32(tbase + c * 64, g);
            tmem_ld32(tbase + c * 64 + 32, v);
            tmem_ld_wait();
            float gf[32], uf[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              gf[j] = __uint_as_float(g[j]);
              uf[j] = __uint_as_float(v[j]);
            }
            if (p.ss_in) {
              scale32(gf, rs);
              scale32(uf, rs);
            }
            if (row_ok) store_silu(p, row, (tn * BN) / 2 + c * 32, gf, uf);
          }
        } else {
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t a[32];
            tmem_ld32(tbase + c * 32, a);
            tmem_ld_wait();
            float f[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(a[j]);
            if (p.ss_in) scale32(f, rs);
            if (row_ok) store_cols(p, row, tn * BN + c * 32, f, ss);
          }
          if (p.ss_out && row_ok) p.ss_out[static_cast<size_t>(row) * p.tiles_n + tn] = ss;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (MODE == 2)
          mbar_arrive_cluster(mapa_shared(&tempty[acc], 0));  // the leader owns the accumulator pipeline
        else
          mbar_arrive(&tempty[acc]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  // no CTA leaves while its peer may still multicast into it / arrive on it
  if (MC > 1) cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    if (MODE == 2)
      tmem_dealloc_cg2(tmem_base, C::kTmemCols);
    else
      tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// Experiment knobs read once from the environment (tools/gemm_sustained.py).
int gemm_env(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
int gemm_policy_mode() {
  static const int mode = gemm_env("SSB_GEMM_POLICY", 2);
  return mode;
}

// Stream-K layout of a persistent schedule of `unit_tiles` tiles over
// `groups` CTA groups: whole-tile rounds while at least two rounds remain,
// then the last 1-2 rounds' k-blocks split evenly over the groups.  Off when
// the tiles already fill whole rounds or the range would be too fine.
struct SKLayout {
  int dp_rounds, tile0;
  long long W;
  bool on;
};
SKLayout sk_layout(long unit_tiles, int num_kb, long groups) {
  SKLayout l{0, 0, 0, false};
  if (unit_tiles >= groups && unit_tiles % groups == 0) return l;
  l.dp_rounds = unit_tiles > groups ? static_cast<int>(unit_tiles / groups) - 1 : 0;
  l.tile0 = static_cast<int>(l.dp_rounds * groups);
  l.W = static_cast<long long>(unit_tiles - l.tile0) * num_kb;
  l.on = l.W >= 4LL * groups;
  return l;
}

template <int BN, int MODE>
int launch(const void* A, const void* B, void* Cp, const void* R, int M, int N, int K, int lda,
           int ldb, int ldc, int ldr, int epi, cudaStream_t stream, int max_ctas, int splits, void* ws,
           const RopeKV* rk, int arg_base, bool tail, ssb_rownorm* rn, bool sk) {
  using C = Cfg<BN, MODE>;
  constexpr int MC = MODE ? 2 : 1;
  CUtensorMap ta, tb;
  int rc = encode_tmap_2d_bf16(&ta, A, K, M, static_cast<uint64_t>(lda) * 2, kBK, kBM);
  if (rc) return rc;
  rc = encode_tmap_2d_bf16(&tb, B, K, N, static_cast<uint64_t>(ldb) * 2, kBK, BN / MC);
  if (rc) return rc;
  static bool attr_done = false;  // per <BN, MODE> instantiation
  if (!attr_done) {
    SSB_CUDA(cudaFuncSetAttribute(gemm_bf16_sm100<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  C::kSmemBytes));
    attr_done = true;
  }
  Params p;
  p.C = Cp;
  p.R = R;
  p.M = M;
  p.N = N;
  p.K = K;
  p.ldc = ldc;
  p.ldr = ldr;
  p.epi = epi;
  if (rk) p.rk = *rk;
  p.arg_base = arg_base;
  p.pol_mode = gemm_policy_mode();
  {
    static const int kserp = gemm_env("SSB_GEMM_KSERP", 1);
    p.kserp = kserp;
  }
  p.tiles_m = (M + kBM - 1) / kBM;
  p.tiles_n = (N + BN - 1) / BN;
  p.ss_out = rn ? rn->ss_out : nullptr;
  p.ss_in = rn ? rn->ss_in : nullptr;
  p.ss_in_parts = rn ? rn->ss_in_parts : 0;
  p.ss_hidden = rn ? static_cast<float>(rn->hidden) : 1.f;
  p.ss_eps = rn ? rn->eps : 0.f;
  if (rn) rn->ss_parts = rn->ss_out ? p.tiles_n : 0;
  const int num_kb = (K + kBK - 1) / kBK;
  p.kb_per_split = (num_kb + splits - 1) / splits;
  p.splits = (num_kb + p.kb_per_split - 1) / p.kb_per_split;  // no empty split
  // workspace = a FIXED counter area (kCounterBytes, shared by every GEMM
  // that uses this workspace, so its zero invariant survives GEMMs of
  // different tile counts) followed by this launch's fp32 partials
  p.counters = static_cast<int*>(ws);
  p.ws = p.splits > 1 ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kCounterBytes) : nullptr;
  // band the operand whose re-streaming would cost more DRAM traffic:
  // M-bands re-read B once per band, N-bands re-read A once per band
  {
    const double a_bytes = 2.0 * M * K, b_bytes = 2.0 * N * K;
    static const int group_env = gemm_env("SSB_GEMM_GROUP", kGroupM);
    static const int band_env = gemm_env("SSB_GEMM_BAND", -1);
    p.group_size = group_env;
    const double m_band = a_bytes + b_bytes * ((p.tiles_m + p.group_size - 1) / p.group_size);
    const double n_band = b_bytes + a_bytes * ((p.tiles_n + p.group_size - 1) / p.group_size);
    p.group_n = n_band < m_band ? 1 : 0;
    if (band_env >= 0) p.group_n = band_env;
  }
  const long unit_tiles = static_cast<long>((p.tiles_m + MC - 1) / MC) * p.tiles_n;
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  const long groups = std::max(grid / MC, 1);
  // tail split: whole tiles fill the full waves, only the last partial wave's
  // tiles are split (so every group gets work in it); else every tile splits
  if (p.splits <= 1)
    p.full_units = static_cast<int>(unit_tiles);
  else
    p.full_units = tail ? static_cast<int>((unit_tiles / groups) * groups) : 0;
  p.num_kb = num_kb;
  p.unit_tiles = static_cast<int>(unit_tiles);
  p.sk = 0;
  p.sk_dp_rounds = p.sk_tile0 = 0;
  p.sk_W = 0;
  if (sk) {
    const SKLayout l = sk_layout(unit_tiles, num_kb, groups);
    if (l.on) {
      p.sk = 1;
      p.sk_dp_rounds = l.dp_rounds;
      p.sk_tile0 = l.tile0;
      p.sk_W = l.W;
      p.splits = 1;
      p.full_units = static_cast<int>(unit_tiles);
      p.ws = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kCounterBytes);
    }
  }
  const long units = p.full_units + (unit_tiles - p.full_units) * p.splits;
  grid = p.sk ? static_cast<int>(groups) * MC : static_cast<int>(std::min<long>(groups, units)) * MC;
  {
    const bool pdl = pdl_enabled();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (MC > 1) {
      attr[n].id = cudaLaunchAttributeClusterDimension;
      attr[n].val.clusterDim.x = MC;
      attr[n].val.clusterDim.y = 1;
      attr[n].val.clusterDim.z = 1;
      ++n;
    }
    if (pdl) {
      attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[n].val.programmaticStreamSerializationAllowed = 1;
      ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    SSB_CUDA(cudaLaunchKernelEx(&cfg, gemm_bf16_sm100<BN, MODE>, ta, tb, p));
  }
  return check_launch("gemm_bf16_sm100");
}

struct Plan {
  int mode, bn, splits;
  int tail;  // split only the tiles of the last partial wave
  int sk;    // stream-K (splits = 1)
};

// Tiles (128-row, including a pair's phantom tile when tiles_m is odd).
size_t plan_tiles(int M, int N, const Plan& pl) {
  const int MC = pl.mode ? 2 : 1;
  return static_cast<size_t>(((M + kBM * MC - 1) / (kBM * MC)) * MC) * ((N + pl.bn - 1) / pl.bn);
}

// Workspace bytes of a split plan; SIZE_MAX when the tile counters do not fit
// the fixed counter area.
size_t plan_ws_bytes(int M, int N, const Plan& pl, int sms) {
  const int MC = pl.mode ? 2 : 1;
  const size_t tiles = plan_tiles(M, N, pl);
  if (pl.sk) {
    // two partial slots per CTA of every group
    if (tiles * 4 * sizeof(int) > kCounterBytes) return SIZE_MAX;
    const size_t groups = std::max(sms / MC, 1);
    return kCounterBytes + 2 * groups * MC * kBM * pl.bn * sizeof(float);
  }
  if (pl.splits <= 1) return 0;
  if (tiles * 4 * sizeof(int) > kCounterBytes) return SIZE_MAX;
  size_t split_tiles = tiles;
  if (pl.tail) {
    const size_t unit_tiles = tiles / MC, groups = std::max(sms / MC, 1);
    split_tiles = (unit_tiles % groups) * MC;
  }
  return kCounterBytes + split_tiles * pl.splits * kBM * pl.bn * sizeof(float);
}

// Modelled time (microseconds) of one configuration: a fixed launch /
// prologue / drain cost, rounds of persistent units (the last, partial round
// weighted by its fill) each running its k-blocks at a per-(mode, tile)
// k-block time, and for split-K a fixed cost plus the fp32 partial round trip.
// The per-k-block times are not the MMA rate: at these tile shapes an SM is
// bound by operand ingest from L2 (~64 B/clk), so wide single-CTA tiles lose
// to CTA pairs that split B.  Constants fitted on B200 to the sweep of
// tools/bench_kernels.py --what splitk (Llama decode shapes at M = 256/512,
// TP1 and TP8, and prefill shapes); the fitted plan is within 1.2x of the
// best forced configuration on every swept shape (profiles/ summary).
double plan_kb_us(const Plan& pl) {
  if (pl.mode == 2)
    return pl.bn >= 256 ? 0.3839 : pl.bn >= 224 ? 0.3282 : pl.bn >= 192 ? 0.425 : pl.bn >= 128 ? 0.2417 : 1.0;
  return pl.bn >= 256 ? 2.4031 : pl.bn >= 224 ? 1.435 : pl.bn >= 192 ? 0.3997 : pl.bn >= 128 ? 0.2308 : 1.0;
}

double plan_cost(int M, int N, int K, int sms, const Plan& pl) {
  const int MC = pl.mode ? 2 : 1;
  const int tm = (M + kBM - 1) / kBM;
  const int kb = (K + kBK - 1) / kBK;
  if (pl.sk) {
    const long unit_tiles = static_cast<long>((tm + MC - 1) / MC) * ((N + pl.bn - 1) / pl.bn);
    const long groups = std::max(1, sms / MC);
    const SKLayout l = sk_layout(unit_tiles, kb, groups);
    if (!l.on) return 1e30;
    // whole-tile rounds, then an even share of the stream-K k-blocks, plus
    // one partial spill + reduction (~ a split-K fix-up) on the tail
    const double per = static_cast<double>(l.W) / groups;
    const double bytes = 2.0 * groups * MC * kBM * pl.bn * 4.0;
    return 10.86 + (l.dp_rounds * kb + per) * plan_kb_us(pl) + 4.0 + 0.03 * bytes / 1e6;
  }
  const int kbs = (kb + pl.splits - 1) / pl.splits;
  const int splits = (kb + kbs - 1) / kbs;
  if (pl.tail) {
    // full waves of whole tiles, then ONE round of the split tail tiles
    const long unit_tiles = static_cast<long>((tm + MC - 1) / MC) * ((N + pl.bn - 1) / pl.bn);
    const long groups = std::max(1, sms / MC);
    const long full = unit_tiles / groups, rem = unit_tiles % groups;
    if (rem == 0 || rem * splits > groups) return 1e30;
    double kb_us = pl.mode == 2 ? (pl.bn >= 256 ? 0.3839 : pl.bn >= 224 ? 0.3282 : pl.bn >= 192 ? 0.425 : 0.2417)
                                : (pl.bn >= 256 ? 2.4031 : pl.bn >= 224 ? 1.435 : pl.bn >= 192 ? 0.3997 : 0.2308);
    const double bytes = static_cast<double>(rem) * MC * splits * kBM * pl.bn * 4.0;
    return 10.86 + full * kb * kb_us + kbs * kb_us + 8.19 + 0.03 * bytes / 1e6;
  }
  const long units = static_cast<long>((tm + MC - 1) / MC) * ((N + pl.bn - 1) / pl.bn) * splits;
  const long groups = std::max(1, sms / MC);
  const long full = units / groups, rem = units % groups;
  const double last_w = 0.1553;
  const double rounds = full + (rem ? last_w * rem / groups + (1.0 - last_w) : 0.0);
  double kb_us;
  if (pl.mode == 2)
    kb_us = pl.bn >= 256 ? 0.3839 : pl.bn >= 224 ? 0.3282 : pl.bn >= 192 ? 0.425 : pl.bn >= 128 ? 0.2417 : 1.0;
  else
    kb_us = pl.bn >= 256 ? 2.4031 : pl.bn >= 224 ? 1.435 : pl.bn >= 192 ? 0.3997 : pl.bn >= 128 ? 0.2308 : 1.0;
  double t = 10.86 + rounds * kbs * kb_us;
  if (splits > 1) t += 8.19 + 0.03 * static_cast<double>(units) * kBM * pl.bn * 4.0 / 1e6;
  return t;
}

// Measured best configurations (tools/bench_kernels.py --what splitk on
// B200, profiles/r01/gemm_plan_sweep.jsonl) for the Llama decode shapes at
// M = 256 / 512 (TP1 and TP8): exact (M, N, K) matches override the model,
// per epilogue constraint (any N tile / multiple of 64 for SiLU / of 128 for
// RoPE).  The model's per-shape error (~10-20 %) can pick a 25 % slower plan
// on near ties (e.g. the TP1 down projection).
struct MeasuredPlan {
  int M, N, K;
  Plan any, mult64, mult128;
};
constexpr MeasuredPlan kMeasured[] = {
    {256, 768, 4096, {0, 128, 3}, {0, 128, 3}, {0, 128, 3}},
    {256, 3584, 4096, {0, 128, 2}, {0, 128, 2}, {0, 128, 2}},
    {256, 4096, 512, {0, 128, 1}, {0, 128, 1}, {0, 128, 1}},
    {256, 4096, 1792, {0, 128, 1}, {0, 128, 1}, {0, 128, 1}},
    {256, 4096, 4096, {0, 128, 2}, {0, 128, 2}, {0, 128, 2}},
    {256, 4096, 14336, {2, 192, 3}, {2, 192, 3}, {0, 128, 4}},
    {256, 6144, 4096, {0, 128, 1}, {0, 128, 1}, {0, 128, 1}},
    {256, 16032, 4096, {0, 224, 1}, {2, 256, 1}, {2, 256, 1}},
    {256, 28672, 4096, {2, 224, 1}, {2, 256, 1}, {2, 256, 1}},
    {256, 128256, 4096, {2, 224, 1}, {2, 256, 1}, {2, 256, 1}},
    {512, 768, 4096, {2, 128, 3}, {2, 128, 3}, {2, 128, 3}},
    {512, 3584, 4096, {0, 128, 1}, {0, 128, 1}, {0, 128, 1}},
    {512, 4096, 512, {0, 128, 1}, {0, 128, 1}, {0, 128, 1}},
    {512, 4096, 1792, {0, 128, 1}, {0, 128, 1}, {0, 128, 1}},
    {512, 4096, 4096, {0, 128, 1}, {0, 128, 1}, {0, 128, 1}},
    {512, 4096, 14336, {2, 256, 2}, {2, 256, 2}, {2, 256, 2}},
    {512, 6144, 4096, {0, 192, 1}, {0, 192, 1}, {2, 256, 1}},
    {512, 16032, 4096, {2, 224, 1}, {2, 256, 1}, {2, 256, 1}},
    {512, 28672, 4096, {2, 224, 1}, {2, 256, 1}, {2, 256, 1}},
    {512, 128256, 4096, {2, 256, 1}, {2, 256, 1}, {2, 256, 1}},
    {2048, 4096, 4096, {2, 256, 1}, {2, 256, 1}, {2, 256, 1}},
};

const Plan* measured_plan(int M, int N, int K, int epi) {
  for (const MeasuredPlan& m : kMeasured)
    if (m.M == M && m.N == N && m.K == K)
      return epi == SSB_EPI_ROPE_KV ? &m.mult128 : epi == SSB_EPI_SILU_MUL ? &m.mult64 : &m.any;
  return nullptr;
}

// SSB_GEMM_PLAN="M,N,K=mode:bn:splits[:sk|:t];..." overrides the plan of exact
// shapes (in-situ plan sweeps, tools/sweep_decode_plans.sh).
bool env_plan(int M, int N, int K, Plan& out) {
  static const char* spec = getenv("SSB_GEMM_PLAN");
  if (!spec) return false;
  for (const char* q = spec; *q;) {
    int m, n, k, mode, bn, sp, used = 0;
    if (sscanf(q, "%d,%d,%d=%d:%d:%d%n", &m, &n, &k, &mode, &bn, &sp, &used) != 6) return false;
    q += used;
    // optional suffix ":sk" (stream-K) or ":t" (split only the tail wave)
    int sk = 0, tail = 0;
    if (q[0] == ':' && q[1] == 's' && q[2] == 'k') {
      sk = 1;
      q += 3;
    } else if (q[0] == ':' && q[1] == 't') {
      tail = 1;
      q += 2;
    }
    if (m == M && n == N && k == K) {
      out = Plan{mode, bn, sk ? 1 : sp, tail, sk};
      return true;
    }
    while (*q == ';' || *q == ' ') ++q;
  }
  return false;
}

Plan choose_plan(int M, int N, int K, int epi, int sms, size_t ws_bytes) {
  Plan best{0, 256, 1};
  {
    Plan e;
    if (env_plan(M, N, K, e) && ((e.splits <= 1 && !e.sk) || plan_ws_bytes(M, N, e, sms) <= ws_bytes)) return e;
  }
  double best_t = 1e30;
  const int bns[4] = {256, 224, 192, 128};
  const int kb = (K + kBK - 1) / kBK;
  static const int no_split = gemm_env("SSB_GEMM_NO_SPLIT", 0);
  static const int no_table = gemm_env("SSB_GEMM_NO_TABLE", 0);
  if (sms == num_sms() && !no_split && !no_table) {
    const Plan* m = measured_plan(M, N, K, epi);
    if (m && (m->splits <= 1 || plan_ws_bytes(M, N, *m, sms) <= ws_bytes)) return *m;
  }
  for (int mode = 0; mode <= 2; mode += 2) {
    if (mode == 2 && M <= kBM) continue;
    for (int bn : bns) {
      if (epi == SSB_EPI_SILU_MUL && bn % 64) continue;  // gate/up pairs of 32 columns
      if (epi == SSB_EPI_ROPE_KV && bn % 128) continue;  // whole heads per tile
      // tail splits are never chosen automatically: measured on the decode
      // shapes (profiles/r01/gemm_plan_sweep_tail.jsonl) the partial-wave
      // reduction costs what the filled last wave saves (W13: 99.3 vs 99.2 us)
      for (int tail = 0; tail <= 0; ++tail) {
        for (int sp = tail ? 2 : 1; sp <= 16; ++sp) {
          if (sp > 1 && (kb / sp < 4 || no_split)) break;
          Plan pl{mode, bn, sp, tail, 0};
          if (sp > 1 && plan_ws_bytes(M, N, pl, sms) > ws_bytes) break;
          const double t = plan_cost(M, N, K, sms, pl);
          if (t < best_t * 0.995) {
            best_t = t;
            best = pl;
          }
        }
      }
      // stream-K is never chosen automatically: measured on every Llama
      // decode shape at M = 512 (profiles/r02/gemm_plan_sweep_streamk.jsonl)
      // it is 6-14 us SLOWER than the best whole-tile / split-K plan even
      // where it fills all 148 SMs instead of 64-128 (o_proj: 35-43 us vs
      // 28.7).  Kept behind SSB_GEMM_STREAMK for the record (SSB_GEMM_AUTO_SK=1
      // re-enables it in the model search).
      static const int auto_sk = gemm_env("SSB_GEMM_AUTO_SK", 0);
      if (auto_sk && M <= 2048 && !no_split) {
        Plan pl{mode, bn, 1, 0, 1};
        if (plan_ws_bytes(M, N, pl, sms) <= ws_bytes) {
          const double t = plan_cost(M, N, K, sms, pl);
          if (t < best_t * 0.995) {
            best_t = t;
            best = pl;
          }
        }
      }
    }
  }
  return best;
}

}  // namespace
}  // namespace ssb

namespace {
int gemm_entry(const void* A, const void* B, void* C, const void* R, int M, int N, int K, int lda, int ldb,
               int ldc, int ldr, int epilogue, int block_n, int max_ctas, void* workspace, int64_t ws_bytes,
               void* stream, const ssb::RopeKV* rk = nullptr, int arg_base = 0, ssb_rownorm* rn = nullptr) {
  using namespace ssb;
  SSB_REQUIRE(M > 0 && N > 0 && K > 0, "ssb_gemm_bf16: empty problem M=%d N=%d K=%d", M, N, K);
  SSB_REQUIRE(A && B && C, "ssb_gemm_bf16: null operand");
  SSB_REQUIRE((epilogue >= SSB_EPI_NONE && epilogue <= SSB_EPI_F32) || (epilogue == SSB_EPI_ROPE_KV && rk) ||
                  epilogue == SSB_EPI_ARGMAX,
              "ssb_gemm_bf16: bad epilogue %d", epilogue);
  SSB_REQUIRE(epilogue != SSB_EPI_RESIDUAL || R, "ssb_gemm_bf16: residual epilogue without R");
  SSB_REQUIRE(lda >= K && ldb >= K, "ssb_gemm_bf16: lda/ldb smaller than K");
  SSB_REQUIRE(epilogue == SSB_EPI_SILU_MUL ? (N % 64 == 0 && ldc >= N / 2)
                                          : (epilogue == SSB_EPI_ARGMAX || ldc >= N),
              "ssb_gemm_bf16: bad ldc/N for epilogue");
  SSB_REQUIRE(ws_bytes >= 0 && (ws_bytes == 0 || workspace), "ssb_gemm_bf16: bad workspace");
  if (!aligned16(A) || !aligned16(B) || (lda % 8) || (ldb % 8) || !aligned16(C) ||
      (epilogue != SSB_EPI_ARGMAX && (ldc % (epilogue == SSB_EPI_F32 ? 4 : 8))) ||
      (R && (!aligned16(R) || (ldr % 8))) ||
      (workspace && (reinterpret_cast<uintptr_t>(workspace) & 255))) {
    set_error("ssb_gemm_bf16: operands must be 16-byte aligned with leading dims %% 8 == 0 "
              "(workspace 256-byte aligned)");
    return SSB_EALIGN;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int sms = max_ctas > 0 ? std::min(max_ctas, num_sms()) : num_sms();
  Plan pl{0, block_n & 0xFFFF, 1, 0, 0};
  const int forced_split = (block_n >> SSB_GEMM_SPLIT_SHIFT) & 0xFF;
  const int forced_tail = (block_n & SSB_GEMM_TAIL) ? 1 : 0;
  const int forced_sk = (block_n & SSB_GEMM_STREAMK) ? 1 : 0;
  if (pl.bn == 0 && !(block_n & (SSB_GEMM_MC1 | SSB_GEMM_MC2 | SSB_GEMM_2SM)) && forced_split == 0 && !forced_sk) {
    pl = choose_plan(M, N, K, epilogue, sms, static_cast<size_t>(ws_bytes));
  } else {
    pl.mode = (block_n & SSB_GEMM_2SM) ? 2 : (block_n & SSB_GEMM_MC2) ? 1 : 0;
    if (pl.bn == 0) pl.bn = 256;
    pl.splits = forced_split && !forced_sk ? forced_split : 1;
    pl.tail = forced_tail && !forced_sk;
    pl.sk = forced_sk;
    if (pl.mode == 2 && M <= kBM) pl.mode = 0;
  }
  if (pl.sk && plan_ws_bytes(M, N, pl, sms) > static_cast<size_t>(ws_bytes))
    return fail_arg("ssb_gemm_bf16: stream-K needs %zu workspace bytes, have %lld", plan_ws_bytes(M, N, pl, sms),
                    static_cast<long long>(ws_bytes));
  if (epilogue == SSB_EPI_SILU_MUL && pl.bn % 64)
    return fail_arg("ssb_gemm_bf16: SiLU epilogue needs block_n %% 64 == 0");
  if (epilogue == SSB_EPI_ROPE_KV && pl.bn % 128)
    return fail_arg("ssb_gemm_qkv_rope_kv: block_n must be 128 or 256 (whole heads per tile)");
  if (pl.splits > 1) {  // effective split count: no empty k-range
    const int kb = (K + kBK - 1) / kBK, kbs = (kb + pl.splits - 1) / pl.splits;
    pl.splits = (kb + kbs - 1) / kbs;
  }
  if (rn) {
    SSB_REQUIRE(!rn->ss_out || epilogue == SSB_EPI_RESIDUAL, "ssb_gemm: ss_out needs the residual epilogue");
    SSB_REQUIRE(!rn->ss_in || (rn->ss_in_parts > 0 && rn->hidden > 0),
                "ssb_gemm: ss_in needs ss_in_parts > 0 and hidden > 0");
  }
  if (pl.splits > 1 && plan_ws_bytes(M, N, pl, sms) > static_cast<size_t>(ws_bytes))
    return fail_arg("ssb_gemm_bf16: split-K x%d needs %zu workspace bytes, have %lld", pl.splits,
                    plan_ws_bytes(M, N, pl, sms), static_cast<long long>(ws_bytes));
#define SSB_GEMM_CASE(BN_)                                                                              \
  case BN_:                                                                                            \
    return pl.mode == 2   ? launch<BN_, 2>(A, B, C, R, M, N, K, lda, ldb, ldc, ldr, epilogue, s, max_ctas, \
                                           pl.splits, workspace, rk, arg_base, pl.tail != 0, rn, pl.sk != 0)           \
           : pl.mode == 1 ? launch<BN_, 1>(A, B, C, R, M, N, K, lda, ldb, ldc, ldr, epilogue, s, max_ctas, \
                                           pl.splits, workspace, rk, arg_base, pl.tail != 0, rn, pl.sk != 0)           \
                          : launch<BN_, 0>(A, B, C, R, M, N, K, lda, ldb, ldc, ldr, epilogue, s, max_ctas, \
                                           pl.splits, workspace, rk, arg_base, pl.tail != 0, rn, pl.sk != 0);
  switch (pl.bn) {
    SSB_GEMM_CASE(256)
    SSB_GEMM_CASE(224)
    SSB_GEMM_CASE(192)
    SSB_GEMM_CASE(128)
    SSB_GEMM_CASE(64)
    default: return fail_arg("ssb_gemm_bf16: block_n must be 0, 64, 128, 192, 224 or 256 (got %d)", pl.bn);
  }
#undef SSB_GEMM_CASE
}
}  // namespace

extern "C" int ssb_gemm_bf16(const void* A, const void* B, void* C, const void* R, int M, int N, int K, int lda,
                             int ldb, int ldc, int ldr, int epilogue, int block_n, int max_ctas, void* stream) {
  return gemm_entry(A, B, C, R, M, N, K, lda, ldb, ldc, ldr, epilogue, block_n, max_ctas, nullptr, 0, stream);
}

extern "C" int ssb_gemm_bf16_ws(const void* A, const void* B, void* C, const void* R, int M, int N, int K,
                                int lda, int ldb, int ldc, int ldr, int epilogue, int block_n, int max_ctas,
                                void* workspace, int64_t workspace_bytes, void* stream) {
  return gemm_entry(A, B, C, R, M, N, K, lda, ldb, ldc, ldr, epilogue, block_n, max_ctas, workspace,
                    workspace_bytes, stream);
}

extern "C" int ssb_gemm_bf16_rn(const void* A, const void* B, void* C, const void* R, int M, int N, int K,
                                int lda, int ldb, int ldc, int ldr, int epilogue, int block_n, int max_ctas,
                                void* workspace, int64_t workspace_bytes, ssb_rownorm* rn, void* stream) {
  return gemm_entry(A, B, C, R, M, N, K, lda, ldb, ldc, ldr, epilogue, block_n, max_ctas, workspace,
                    workspace_bytes, stream, nullptr, 0, rn);
}

extern "C" int64_t ssb_gemm_plan(int M, int N, int K, int epilogue, int max_ctas, int64_t workspace_bytes,
                                 int32_t* out_plan) {
  using namespace ssb;
  if (M <= 0 || N <= 0 || K <= 0) return fail_arg("ssb_gemm_plan: empty problem");
  const int sms = max_ctas > 0 ? std::min(max_ctas, num_sms()) : num_sms();
  const Plan pl = choose_plan(M, N, K, epilogue, sms, static_cast<size_t>(std::max<int64_t>(workspace_bytes, 0)));
  if (out_plan) {
    out_plan[0] = pl.mode;
    out_plan[1] = pl.bn;
    out_plan[2] = pl.sk ? 0 : pl.tail ? -pl.splits : pl.splits;  // negative: tail split; 0: stream-K
  }
  return static_cast<int64_t>(plan_ws_bytes(M, N, pl, sms));
}

extern "C" int ssb_gemm_qkv_rope_kv(const void* A, const void* B, void* qkv, int M, int K, int lda, int ldb,
                                    int ldc, int nq, int nk, int head_dim, const int32_t* positions,
                                    const float* rope_cos, const float* rope_sin, int max_pos, void* pool,
                                    ssb_kv_geometry geo, int layer, const int64_t* slots, int block_n,
                                    int max_ctas, void* workspace, int64_t workspace_bytes, ssb_rownorm* rn,
                                    void* stream) {
  using namespace ssb;
  SSB_REQUIRE(head_dim == 128, "ssb_gemm_qkv_rope_kv: head_dim must be 128 (got %d)", head_dim);
  SSB_REQUIRE(nq > 0 && nk > 0 && nq % nk == 0, "ssb_gemm_qkv_rope_kv: bad head counts nq=%d nk=%d", nq, nk);
  SSB_REQUIRE(positions && rope_cos && rope_sin && max_pos > 0, "ssb_gemm_qkv_rope_kv: null RoPE table");
  SSB_REQUIRE(!slots || (pool && geo.n_heads == nk && geo.head_dim == head_dim && layer >= 0 &&
                         layer < geo.n_layers && geo.block_size > 0),
              "ssb_gemm_qkv_rope_kv: pool geometry does not match (nk=%d, heads=%d, layer=%d of %d)", nk,
              geo.n_heads, layer, geo.n_layers);
  SSB_REQUIRE(!pool || aligned16(pool), "ssb_gemm_qkv_rope_kv: pool must be 16-byte aligned");
  RopeKV rk;
  rk.pos = positions;
  rk.cos = rope_cos;
  rk.sin = rope_sin;
  rk.max_pos = max_pos;
  rk.pool = static_cast<__nv_bfloat16*>(pool);
  rk.n_layers = geo.n_layers;
  rk.n_heads = geo.n_heads;
  rk.block_size = geo.block_size;
  rk.layer = layer;
  rk.slots = slots;
  rk.nq = nq;
  rk.nk = nk;
  const int N = (nq + 2 * nk) * head_dim;
  return gemm_entry(A, B, qkv, nullptr, M, N, K, lda, ldb, ldc, 0, SSB_EPI_ROPE_KV, block_n, max_ctas, workspace,
                    workspace_bytes, stream, &rk, 0, rn);
}

extern "C" int ssb_gemm_lm_head_argmax(const void* A, const void* B, int M, int N, int K, int lda, int ldb,
                                       int index_base, unsigned long long* keys, int block_n, int max_ctas,
                                       void* workspace, int64_t workspace_bytes, ssb_rownorm* rn, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(keys, "ssb_gemm_lm_head_argmax: null keys");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  SSB_CUDA(cudaMemsetAsync(keys, 0, static_cast<size_t>(M) * sizeof(unsigned long long), s));
  return gemm_entry(A, B, keys, nullptr, M, N, K, lda, ldb, 0, 0, SSB_EPI_ARGMAX, block_n, max_ctas, workspace,
                    workspace_bytes, stream, nullptr, index_base, rn);
}
