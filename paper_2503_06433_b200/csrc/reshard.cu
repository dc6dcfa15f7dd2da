// Layout-transform kernels of the re-shard engine.
//
// KV: the paged pool of one GPU is [block][layer][K|V][head][token][dim]; a
// (layer range x head range) rectangle of one block is nl*2 runs of
// nh*block_size*head_dim contiguous elements (16 KiB at Llama-3-8B TP8), so
// pack/unpack are pure streaming copies of long contiguous runs: 16-byte
// vector loads/stores, several in flight per thread, one CTA per run.
// The rectangles are the pairwise intersections of the reference's
// per-GPU (layer x head) KV shard descriptors (reshard.py:151-188).
//
// Weights / host tier: a batched 2-D strided copy driven by a device array of
// descriptors (rows x row_bytes with independent strides); the row-parallel
// column slices of Wo / W_down are rows of head_dim*heads elements.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "seesaw_b200.h"

namespace ssb {
namespace {

struct PeerTable {
  int32_t l0[SSB_MAX_PEERS], nl[SSB_MAX_PEERS], h0[SSB_MAX_PEERS], nh[SSB_MAX_PEERS];
  int64_t off[SSB_MAX_PEERS];
  int32_t run_begin[SSB_MAX_PEERS + 1];  // prefix of n_ids*nl*2 runs per peer
  int32_t uniform_nl;                    // > 0: every peer has this nl and nh > 0
};

constexpr int kCopyThreads = 256;
constexpr int kUnroll = 4;

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(uint4* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// Copy n16 16-byte vectors from src to dst with the whole CTA.
__device__ __forceinline__ void cta_copy(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                         int64_t n16) {
  int64_t i = threadIdx.x;
  const int64_t step = static_cast<int64_t>(blockDim.x) * kUnroll;
  for (; i + (kUnroll - 1) * blockDim.x < n16; i += step) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(src + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) st_stream(dst + i + u * blockDim.x, v[u]);
  }
  for (; i < n16; i += blockDim.x) st_stream(dst + i, ld_stream(src + i));
}

template <bool kPack>
__global__ void __launch_bounds__(kCopyThreads) kv_reshard_kernel(
    uint8_t* __restrict__ pool, uint8_t* __restrict__ staging, const int32_t* __restrict__ ids,
    int n_ids, int n_peers, ssb_kv_geometry geo, const PeerTable tab) {
  const int run = blockIdx.x;
  int p = 0, kv, j, i, nl;
  if (kPack && tab.uniform_nl > 0) {
    // every peer takes the same layer range length: walk the pool in address
    // order (block, layer, K|V, then peers = adjacent head planes) so
    // consecutive CTAs read consecutive planes; the staging writes scatter
    // over the peers' regions in 16 KiB+ runs instead
    nl = tab.uniform_nl;
    p = run % n_peers;
    const int rest = run / n_peers;
    kv = rest & 1;
    j = (rest >> 1) % nl;
    i = (rest >> 1) / nl;
  } else {
    while (p + 1 < n_peers && run >= tab.run_begin[p + 1]) ++p;
    const int local = run - tab.run_begin[p];
    nl = tab.nl[p];
    kv = local & 1;
    j = (local >> 1) % nl;
    i = (local >> 1) / nl;
  }
  const int64_t plane = static_cast<int64_t>(geo.block_size) * geo.head_dim * 2;  // bytes / head
  const int64_t run_bytes = plane * tab.nh[p];
  const int64_t blk = ids[i];
  const int64_t pool_off =
      ((blk * geo.n_layers + (tab.l0[p] + j)) * 2 + kv) * (plane * geo.n_heads) + tab.h0[p] * plane;
  const int64_t stage_off = tab.off[p] + (static_cast<int64_t>(i * nl + j) * 2 + kv) * run_bytes;
  if (kPack)
    cta_copy(reinterpret_cast<const uint4*>(pool + pool_off),
             reinterpret_cast<uint4*>(staging + stage_off), run_bytes >> 4);
  else
    cta_copy(reinterpret_cast<const uint4*>(staging + stage_off),
             reinterpret_cast<uint4*>(pool + pool_off), run_bytes >> 4);
}

// Bulk-copy (TMA engine) variant: ONE thread per CTA streams every run of
// its share through a ring of shared-memory slots with cp.async.bulk
// global->shared (mbarrier completion) and shared->global (bulk groups),
// keeping kBulkSlots-1 loads in flight; the SM's load/store units are idle.
constexpr int kBulkSlots = 4;
constexpr int kBulkChunk = 16 * 1024;

template <bool kPack>
__global__ void __launch_bounds__(32) kv_reshard_bulk_kernel(
    uint8_t* __restrict__ pool, uint8_t* __restrict__ staging, const int32_t* __restrict__ ids, int n_ids,
    int n_peers, ssb_kv_geometry geo, const PeerTable tab, int total_runs) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kBulkSlots];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < kBulkSlots; ++i) mbar_init(&full[i], 1);
  fence_mbar_init();
  const int64_t plane = static_cast<int64_t>(geo.block_size) * geo.head_dim * 2;
  // cursor over (run, offset) chunks of this CTA's runs
  struct Cur {
    int run;
    int64_t off, bytes;
    const uint8_t* src;
    uint8_t* dst;
  };
  auto locate = [&](Cur& c) {  // src/dst/bytes of c.run (decoded as in kv_reshard_kernel)
    int p = 0, kv, j, i, nl;
    if (kPack && tab.uniform_nl > 0) {
      nl = tab.uniform_nl;
      p = c.run % n_peers;
      const int rest = c.run / n_peers;
      kv = rest & 1;
      j = (rest >> 1) % nl;
      i = (rest >> 1) / nl;
    } else {
      while (p + 1 < n_peers && c.run >= tab.run_begin[p + 1]) ++p;
      const int local = c.run - tab.run_begin[p];
      nl = tab.nl[p];
      kv = local & 1;
      j = (local >> 1) % nl;
      i = (local >> 1) / nl;
    }
    const int64_t run_bytes = plane * tab.nh[p];
    const int64_t blk = ids[i];
    const int64_t pool_off =
        ((blk * geo.n_layers + (tab.l0[p] + j)) * 2 + kv) * (plane * geo.n_heads) + tab.h0[p] * plane;
    const int64_t stage_off = tab.off[p] + (static_cast<int64_t>(i * nl + j) * 2 + kv) * run_bytes;
    c.bytes = run_bytes;
    c.src = kPack ? pool + pool_off : staging + stage_off;
    c.dst = kPack ? staging + stage_off : pool + pool_off;
  };
  Cur ld{static_cast<int>(blockIdx.x), 0, 0, nullptr, nullptr};
  if (ld.run < total_runs) locate(ld);
  uint8_t* slot_dst[kBulkSlots];
  uint32_t slot_bytes[kBulkSlots];
  auto issue = [&](uint32_t n) -> bool {  // next chunk's global->shared load into slot n % S
    if (ld.run >= total_runs) return false;
    const int s = n % kBulkSlots;
    const int64_t left = ld.bytes - ld.off;
    const uint32_t bytes = static_cast<uint32_t>(left < kBulkChunk ? left : kBulkChunk);
    mbar_arrive_expect_tx(&full[s], bytes);
    bulk_g2s(ring + s * kBulkChunk, ld.src + ld.off, bytes, &full[s]);
    slot_dst[s] = ld.dst + ld.off;
    slot_bytes[s] = bytes;
    ld.off += bytes;
    if (ld.off >= ld.bytes) {
      ld.run += gridDim.x;
      ld.off = 0;
      if (ld.run < total_runs) locate(ld);
    }
    return true;
  };
  uint32_t issued = 0;
  while (issued < kBulkSlots && issue(issued)) ++issued;
  for (uint32_t n = 0; n < issued; ++n) {
    const int s = n % kBulkSlots;
    mbar_wait(&full[s], (n / kBulkSlots) & 1);
    bulk_s2g(slot_dst[s], ring + s * kBulkChunk, slot_bytes[s]);
    bulk_commit();
    // refill the slot of chunk n-1 once its store has read shared memory
    if (n >= 1) {
      bulk_wait_read<1>();
      if (issue(issued)) ++issued;
    }
  }
  bulk_wait<0>();
}

// staging == nullptr with `absolute`: off[p] are absolute device addresses
// (peer memory mapped over NVLink for the P2P pack; see ssb_kv_reshard_pack_p2p).
int kv_reshard(bool pack, void* pool, ssb_kv_geometry geo, const int32_t* ids, int n_ids, int n_peers,
               const int32_t* l0, const int32_t* nl, const int32_t* h0, const int32_t* nh,
               const int64_t* off, void* staging, void* stream, bool absolute = false) {
  SSB_REQUIRE(n_peers > 0 && n_peers <= SSB_MAX_PEERS, "kv_reshard: n_peers=%d out of range", n_peers);
  SSB_REQUIRE(geo.n_layers > 0 && geo.n_heads > 0 && geo.block_size > 0 && geo.head_dim > 0,
              "kv_reshard: bad geometry");
  SSB_REQUIRE(n_ids >= 0, "kv_reshard: n_ids < 0");
  if (n_ids == 0) return 0;
  SSB_REQUIRE(pool && (staging || absolute) && ids, "kv_reshard: null pointer");
  if ((static_cast<int64_t>(geo.block_size) * geo.head_dim * 2) % 16 != 0 || !aligned16(pool) ||
      (!absolute && !aligned16(staging))) {
    set_error("kv_reshard: head plane and buffers must be 16-byte aligned");
    return SSB_EALIGN;
  }
  PeerTable t;
  int runs = 0;
  for (int p = 0; p < n_peers; ++p) {
    SSB_REQUIRE(l0[p] >= 0 && nl[p] >= 0 && l0[p] + nl[p] <= geo.n_layers,
                "kv_reshard: peer %d layer range [%d,+%d) outside %d local layers", p, l0[p], nl[p],
                geo.n_layers);
    SSB_REQUIRE(h0[p] >= 0 && nh[p] >= 0 && h0[p] + nh[p] <= geo.n_heads,
                "kv_reshard: peer %d head range [%d,+%d) outside %d local heads", p, h0[p], nh[p],
                geo.n_heads);
    SSB_REQUIRE(off[p] % 16 == 0, "kv_reshard: peer %d staging offset not 16-byte aligned", p);
    t.l0[p] = l0[p];
    t.nl[p] = nh[p] > 0 ? nl[p] : 0;
    t.h0[p] = h0[p];
    t.nh[p] = nh[p];
    t.off[p] = off[p];
    t.run_begin[p] = runs;
    runs += n_ids * t.nl[p] * 2;
  }
  t.run_begin[n_peers] = runs;
  t.uniform_nl = t.nl[0];
  for (int p = 1; p < n_peers; ++p)
    if (t.nl[p] != t.nl[0]) t.uniform_nl = 0;
  if (runs == 0) return 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // Copy engine choice (SSB_RESHARD_BULK: 1 force bulk, 0 force LSU, unset
  // auto).  Measured per GPU on the 8B KV (tools/bench_reshard.py): the
  // bulk (TMA-engine) copy packs 16 KiB single-head runs scattered over the
  // PP-layout pool at 5.8-6.0 TB/s vs 5.2-5.6 with 16-byte LSU copies
  // (PP4/PP8 -> TP), but is slower for long runs and for unpack (6.1 vs
  // 6.4-6.7 TB/s), so auto = bulk for pack with single-head rectangles only.
  static const int bulk_env = [] {
    const char* e = getenv("SSB_RESHARD_BULK");
    return e ? atoi(e) : -1;
  }();
  bool single_head = true;
  for (int p = 0; p < n_peers; ++p) single_head = single_head && (t.nh[p] <= 1);
  // peer-memory stores go through the LSU path (plain st.global to UVA peer addresses)
  const bool bulk = !absolute && (bulk_env >= 0 ? bulk_env != 0 : (pack && single_head && t.uniform_nl > 0));
  if (bulk) {
    const int smem = kBulkSlots * kBulkChunk;
    static bool attr = false;
    if (!attr) {
      SSB_CUDA(cudaFuncSetAttribute(kv_reshard_bulk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      SSB_CUDA(cudaFuncSetAttribute(kv_reshard_bulk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr = true;
    }
    const int grid = std::min(runs, 3 * num_sms());
    if (pack)
      kv_reshard_bulk_kernel<true><<<grid, 32, smem, s>>>(static_cast<uint8_t*>(pool), static_cast<uint8_t*>(staging),
                                                          ids, n_ids, n_peers, geo, t, runs);
    else
      kv_reshard_bulk_kernel<false><<<grid, 32, smem, s>>>(static_cast<uint8_t*>(pool),
                                                           static_cast<uint8_t*>(staging), ids, n_ids, n_peers, geo, t,
                                                           runs);
    return check_launch(pack ? "kv_reshard_pack" : "kv_reshard_unpack");
  }
  if (pack)
    kv_reshard_kernel<true><<<runs, kCopyThreads, 0, s>>>(
        static_cast<uint8_t*>(pool), static_cast<uint8_t*>(staging), ids, n_ids, n_peers, geo, t);
  else
    kv_reshard_kernel<false><<<runs, kCopyThreads, 0, s>>>(
        static_cast<uint8_t*>(pool), static_cast<uint8_t*>(staging), ids, n_ids, n_peers, geo, t);
  return check_launch(pack ? "kv_reshard_pack" : "kv_reshard_unpack");
}

// ------------------------------------------------------------ copy2d -----
constexpr int64_t kChunkBytes = 64 * 1024;

__global__ void __launch_bounds__(kCopyThreads)
    copy2d_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                  const ssb_copy_desc* __restrict__ descs, int n_desc, int64_t total) {
  const int64_t begin = static_cast<int64_t>(blockIdx.x) * kChunkBytes;
  const int64_t end = min(begin + kChunkBytes, total);
  // binary search for the descriptor holding `begin`
  __shared__ int s_first;
  if (threadIdx.x == 0) {
    int lo = 0, hi = n_desc - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (descs[mid].cum_bytes <= begin) lo = mid; else hi = mid - 1;
    }
    s_first = lo;
  }
  __syncthreads();
  int d = s_first;
  ssb_copy_desc cur = descs[d];
  int64_t cur_end = cur.cum_bytes + static_cast<int64_t>(cur.rows) * cur.row_bytes;
  for (int64_t x = begin + 16 * static_cast<int64_t>(threadIdx.x); x < end;
       x += 16 * static_cast<int64_t>(blockDim.x)) {
    while (x >= cur_end) {
      cur = descs[++d];
      cur_end = cur.cum_bytes + static_cast<int64_t>(cur.rows) * cur.row_bytes;
    }
    const int64_t lin = x - cur.cum_bytes;
    const int64_t row = lin / cur.row_bytes;
    const int64_t col = lin - row * cur.row_bytes;
    const uint4 v = ld_stream(reinterpret_cast<const uint4*>(src + cur.src_off + row * cur.src_stride + col));
    st_stream(reinterpret_cast<uint4*>(dst + cur.dst_off + row * cur.dst_stride + col), v);
  }
}

// ------------------------------------------------ host-tier gather/scatter --
// One sequence's KV between the paged pool and the contiguous HND staging
// layout [layer][K|V][head][token][dim] of the host tier (reshard.py:191-201,
// PAPER.md:151-154).  The staging covers pool layers [l0, l0+nl) and heads
// [h0, h0+nh) of this GPU, i.e. this GPU's (layer x head) rectangle of the
// sequence in its CURRENT layout.  CTA = one (layer, kv, head, block) run of
// min(64, tokens left) x dim elements.
template <bool kGather>
__global__ void __launch_bounds__(kCopyThreads) kv_hnd_kernel(
    uint8_t* __restrict__ pool, uint8_t* __restrict__ stage, const int32_t* __restrict__ blocks, int n_blocks,
    int n_tokens, ssb_kv_geometry geo, int l0, int nl, int h0, int nh) {
  const int run = blockIdx.x;
  const int b = run % n_blocks;
  int rest = run / n_blocks;
  const int h = rest % nh;
  rest /= nh;
  const int kv = rest & 1;
  const int l = rest >> 1;
  const int64_t row_bytes = static_cast<int64_t>(geo.head_dim) * 2;
  const int tok0 = b * geo.block_size;
  const int ntok = min(geo.block_size, n_tokens - tok0);
  if (ntok <= 0) return;
  const int64_t blk = blocks[b];
  const int64_t pool_off =
      (((blk * geo.n_layers + (l0 + l)) * 2 + kv) * geo.n_heads + (h0 + h)) * geo.block_size * row_bytes;
  const int64_t stage_off = (((static_cast<int64_t>(l) * 2 + kv) * nh + h) * n_tokens + tok0) * row_bytes;
  const int64_t n16 = (ntok * row_bytes) >> 4;
  if (kGather)
    cta_copy(reinterpret_cast<const uint4*>(pool + pool_off), reinterpret_cast<uint4*>(stage + stage_off), n16);
  else
    cta_copy(reinterpret_cast<const uint4*>(stage + stage_off), reinterpret_cast<uint4*>(pool + pool_off), n16);
}

}  // namespace
}  // namespace ssb

extern "C" {

int ssb_kv_hnd_copy(int gather, void* pool, ssb_kv_geometry geo, const int32_t* blocks, int n_blocks,
                    int n_tokens, int l0, int nl, int h0, int nh, void* staging, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(n_blocks >= 0 && n_tokens >= 0 && nl >= 0 && nh >= 0, "ssb_kv_hnd_copy: negative sizes");
  if (n_blocks == 0 || n_tokens == 0 || nl == 0 || nh == 0) return 0;
  SSB_REQUIRE(pool && staging && blocks, "ssb_kv_hnd_copy: null pointer");
  SSB_REQUIRE(l0 >= 0 && l0 + nl <= geo.n_layers && h0 >= 0 && h0 + nh <= geo.n_heads,
              "ssb_kv_hnd_copy: rectangle outside the pool geometry");
  SSB_REQUIRE(n_tokens <= n_blocks * geo.block_size, "ssb_kv_hnd_copy: %d tokens exceed %d blocks", n_tokens,
              n_blocks);
  if ((geo.head_dim * 2) % 16 || !aligned16(pool) || !aligned16(staging)) {
    set_error("ssb_kv_hnd_copy: rows and buffers must be 16-byte aligned");
    return SSB_EALIGN;
  }
  const int64_t runs = static_cast<int64_t>(nl) * 2 * nh * n_blocks;
  SSB_REQUIRE(runs < (1ll << 31), "ssb_kv_hnd_copy: too many runs");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (gather)
    kv_hnd_kernel<true><<<static_cast<int>(runs), kCopyThreads, 0, s>>>(
        static_cast<uint8_t*>(pool), static_cast<uint8_t*>(staging), blocks, n_blocks, n_tokens, geo, l0, nl, h0,
        nh);
  else
    kv_hnd_kernel<false><<<static_cast<int>(runs), kCopyThreads, 0, s>>>(
        static_cast<uint8_t*>(pool), static_cast<uint8_t*>(staging), blocks, n_blocks, n_tokens, geo, l0, nl, h0,
        nh);
  return check_launch("ssb_kv_hnd_copy");
}

int ssb_kv_reshard_pack(const void* pool, ssb_kv_geometry geo, const int32_t* block_ids, int n_ids,
                        int n_peers, const int32_t* l0, const int32_t* nl, const int32_t* h0,
                        const int32_t* nh, const int64_t* off_bytes, void* staging, void* stream) {
  return ssb::kv_reshard(true, const_cast<void*>(pool), geo, block_ids, n_ids, n_peers, l0, nl, h0,
                         nh, off_bytes, staging, stream);
}

int ssb_kv_reshard_unpack(void* pool, ssb_kv_geometry geo, const int32_t* block_ids, int n_ids,
                          int n_peers, const int32_t* l0, const int32_t* nl, const int32_t* h0,
                          const int32_t* nh, const int64_t* off_bytes, const void* staging,
                          void* stream) {
  return ssb::kv_reshard(false, pool, geo, block_ids, n_ids, n_peers, l0, nl, h0, nh, off_bytes,
                         const_cast<void*>(staging), stream);
}

int ssb_copy2d_batched(const void* src, void* dst, const ssb_copy_desc* descs, int n_desc,
                       int64_t total_bytes, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(n_desc >= 0 && total_bytes >= 0, "ssb_copy2d_batched: negative sizes");
  if (n_desc == 0 || total_bytes == 0) return 0;
  // dst == NULL: dst_off are absolute device addresses (peer memory)
  SSB_REQUIRE(src && descs, "ssb_copy2d_batched: null pointer");
  if (!aligned16(src) || (dst && !aligned16(dst)) || total_bytes % 16) {
    set_error("ssb_copy2d_batched: bases and sizes must be 16-byte aligned");
    return SSB_EALIGN;
  }
  const int64_t blocks = (total_bytes + kChunkBytes - 1) / kChunkBytes;
  SSB_REQUIRE(blocks < (1ll << 31), "ssb_copy2d_batched: too large");
  copy2d_kernel<<<static_cast<int>(blocks), kCopyThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), descs, n_desc, total_bytes);
  return check_launch("ssb_copy2d_batched");
}

}  // extern "C"

extern "C" int ssb_kv_reshard_pack_p2p(const void* pool, ssb_kv_geometry geo, const int32_t* block_ids, int n_ids,
                                       int n_peers, const int32_t* l0, const int32_t* nl, const int32_t* h0,
                                       const int32_t* nh, const int64_t* dst_addr, void* stream) {
  return ssb::kv_reshard(true, const_cast<void*>(pool), geo, block_ids, n_ids, n_peers, l0, nl, h0, nh, dst_addr,
                         nullptr, stream, true);
}
