// Tensor-parallel combine over NVLink peer memory, fused with the RMSNorm that
// follows it in every Llama block.
//
// Reference: the TP all-reduce the reference charges per layer
// (perf.py:71-74 allreduce_time, `allreduces_per_layer`; SURVEY.md §8(e)
// "Decode: TP all-reduce, 2 per layer").  Under the decode layout (pure TP)
// each row-parallel projection (o_proj, down_proj) leaves a partial sum on
// every rank; the next op is the residual add + RMSNorm of the following
// sub-block.  Instead of an NCCL all-reduce followed by an rmsnorm launch this
// kernel does both in one pass, two-shot:
//
//   * rows are split into nranks contiguous slices; rank r owns slice r;
//   * each CTA b of rank r: [barrier A: every rank's partials are written]
//     loads its rows of EVERY rank's partial buffer over NVLink (P2P loads,
//     L2-only), sums them in rank order in fp32 (= the reference order
//     ThreadComm.all_reduce_ uses, so results are bit-identical to the
//     unfused path), rounds to bf16 (the new residual stream x), computes
//     the RMSNorm of that row with exactly rmsnorm_kernel's reduction tree,
//     and STORES x and h rows into every rank's x / h buffer (P2P stores);
//     [barrier B: every rank's stores landed and every read of this rank's
//     partials is done, so the next GEMM may overwrite them];
//   * the barriers are per CTA index (CTA b of every rank), through epoch
//     flags in each rank's signal buffer (st.release.sys / ld.acquire.sys),
//     so no grid-wide synchronisation and no host round trip.
//
// Per rank and call the NVLink traffic is (n-1)/n of one partial in and
// 2(n-1)/n (x and h) out, instead of NCCL's 2(n-1)/n in+out plus a separate
// HBM round trip of x for the norm.
//
// Safety: a barrier that does not complete within kTimeoutNs (30 s; a peer that
// never arrives) sets *err and returns (or traps when err is NULL), so a
// broken peer mapping fails the call loudly instead of hanging the GPU.
#include <algorithm>

#include "common.cuh"
#include "seesaw_b200.h"

namespace ssb {
namespace {

constexpr int kARThreads = 256;   // == kNormThreads: same reduction tree as rmsnorm_kernel
constexpr int kARMaxRanks = 8;
constexpr int kARMaxBlocks = 512;
constexpr int kARMaxVec = 4;      // uint4 vectors per thread per row: hidden <= 8192
constexpr uint64_t kTimeoutNs = 30ull * 1000 * 1000 * 1000;

struct ARPeers {
  const __nv_bfloat16* part[kARMaxRanks];
  __nv_bfloat16* x[kARMaxRanks];
  __nv_bfloat16* h[kARMaxRanks];
  float* ss[kARMaxRanks];  // folded-norm variant: per-row sum of squares of x (no h)
  uint32_t* sig[kARMaxRanks];
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// CTA-level barrier across the ranks' CTAs with the same blockIdx.x.
// Slot layout of a rank's signal buffer: [phase 2][kARMaxBlocks][kARMaxRanks]
// u32; peer p announces epoch e for (phase, b) by writing slot [phase][b][p]
// of every rank.  Epochs only grow, so no reset is needed between calls.
// After the barrier slots: [kARMaxBlocks] u32 of this rank's per-CTA epoch
// counters, used when the host passes epoch 0 — CTA b of a call takes
// counter[b] + 1 and stores it back at its end, so the epochs live on the
// device and a call captured in a CUDA graph advances them at every replay
// (all ranks launch the same grids in the same order, so CTA b's counter
// moves in lockstep on every rank).
constexpr size_t kARSlots = static_cast<size_t>(2) * kARMaxBlocks * kARMaxRanks;

__device__ __forceinline__ uint32_t cta_epoch(const ARPeers& P, int rank, uint32_t host_epoch) {
  return host_epoch ? host_epoch : *(const volatile uint32_t*)(P.sig[rank] + kARSlots + blockIdx.x) + 1u;
}
__device__ __forceinline__ void cta_epoch_done(const ARPeers& P, int rank, uint32_t host_epoch, uint32_t epoch) {
  if (!host_epoch && threadIdx.x == 0) P.sig[rank][kARSlots + blockIdx.x] = epoch;
}
__device__ __forceinline__ bool peer_barrier(const ARPeers& P, int n, int rank, int phase, uint32_t epoch,
                                             uint32_t* err) {
  __threadfence_system();  // this CTA's P2P stores before the announcement
  __syncthreads();
  bool ok = true;
  if (threadIdx.x < n) {
    const int p = threadIdx.x;
    const size_t base = (static_cast<size_t>(phase) * kARMaxBlocks + blockIdx.x) * kARMaxRanks;
    st_release_sys(P.sig[p] + base + rank, epoch);
    const uint32_t* mine = P.sig[rank] + base + p;
    const uint64_t t0 = global_ns();
    while (static_cast<int32_t>(ld_acquire_sys(mine) - epoch) < 0) {
      if (global_ns() - t0 > kTimeoutNs) {
        if (err == nullptr) __trap();
        atomicExch(err, 1u);
        ok = false;
        break;
      }
      __nanosleep(100);
    }
  }
  return __syncthreads_and(ok);
}

__device__ __forceinline__ void unpack8(const uint4 v, float* f) {
  const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    f[2 * k] = bf16_lo(u[k]);
    f[2 * k + 1] = bf16_hi(u[k]);
  }
}

template <int N>
__global__ void __launch_bounds__(kARThreads)
    tp_allreduce_rmsnorm_kernel(ARPeers P, int rank, int rows, int hidden, int ld,
                                const __nv_bfloat16* __restrict__ gamma, float eps, uint32_t host_epoch,
                                uint32_t* err) {
  const uint32_t epoch = cta_epoch(P, rank, host_epoch);
  if (!peer_barrier(P, N, rank, 0, epoch, err)) {
    cta_epoch_done(P, rank, host_epoch, epoch);
    return;
  }
  const int r0 = static_cast<int>(static_cast<int64_t>(rows) * rank / N);
  const int r1 = static_cast<int>(static_cast<int64_t>(rows) * (rank + 1) / N);
  const int nvec = hidden / 8;
  __shared__ float red[kARThreads / 32];
  for (int row = r0 + blockIdx.x; row < r1; row += gridDim.x) {
    const size_t off = static_cast<size_t>(row) * ld;
    uint4 xv[kARMaxVec];
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < kARMaxVec; ++j) {
      const int i = threadIdx.x + j * kARThreads;
      if (i < nvec) {
        uint4 v[N];
#pragma unroll
        for (int p = 0; p < N; ++p) v[p] = __ldcg(reinterpret_cast<const uint4*>(P.part[p] + off) + i);
        float acc[8], f[8];
        unpack8(v[0], acc);
#pragma unroll
        for (int p = 1; p < N; ++p) {
          unpack8(v[p], f);
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] = __fadd_rn(acc[k], f[k]);
        }
        uint4 o;
        o.x = pack_bf16x2(acc[0], acc[1]);
        o.y = pack_bf16x2(acc[2], acc[3]);
        o.z = pack_bf16x2(acc[4], acc[5]);
        o.w = pack_bf16x2(acc[6], acc[7]);
        xv[j] = o;
#pragma unroll
        for (int p = 0; p < N; ++p) __stcg(reinterpret_cast<uint4*>(P.x[p] + off) + i, o);
        const uint32_t u[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float a = bf16_lo(u[k]), b = bf16_hi(u[k]);
          ss = fmaf(a, a, ss);
          ss = fmaf(b, b, ss);
        }
      }
    }
    if (gamma == nullptr && P.ss[0] == nullptr) continue;
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
      float t = threadIdx.x < kARThreads / 32 ? red[threadIdx.x] : 0.f;
      t = warp_sum(t);
      if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    if (P.ss[0] != nullptr) {
      // folded norm: the consumer GEMMs scale their rows by 1/rms from this
      // sum (ssb_rownorm, one part), the gains live in their weights
      if (threadIdx.x < N) __stcg(P.ss[threadIdx.x] + row, red[0]);
      __syncthreads();  // red[] is rewritten by the next row
      continue;
    }
    const float inv = 1.0f / sqrtf(__fadd_rn(__fdiv_rn(red[0], static_cast<float>(hidden)), eps));
    __syncthreads();  // red[] is rewritten by the next row
    const uint4* gr = reinterpret_cast<const uint4*>(gamma);
#pragma unroll
    for (int j = 0; j < kARMaxVec; ++j) {
      const int i = threadIdx.x + j * kARThreads;
      if (i < nvec) {
        const uint4 g = gr[i];
        const uint32_t u[4] = {xv[j].x, xv[j].y, xv[j].z, xv[j].w};
        const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float a = __fmul_rn(__fmul_rn(bf16_lo(u[k]), inv), bf16_lo(gw[k]));
          const float b = __fmul_rn(__fmul_rn(bf16_hi(u[k]), inv), bf16_hi(gw[k]));
          o[k] = pack_bf16x2(a, b);
        }
        const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
#pragma unroll
        for (int p = 0; p < N; ++p) __stcg(reinterpret_cast<uint4*>(P.h[p] + off) + i, ov);
      }
    }
  }
  peer_barrier(P, N, rank, 1, epoch, err);
  cta_epoch_done(P, rank, host_epoch, epoch);
}

// Vocab-parallel greedy argmax across the TP group: every rank's LM-head
// epilogue left one packed 64-bit key per row (orderable fp32 logit << 32 |
// ~global index: the max key is the max logit, lowest index on ties —
// argmax_combine's rule) in its `keys` buffer.  After barrier A each CTA
// loads its rows' keys from every rank over NVLink, keeps the max and writes
// the token id locally; barrier B releases the peers' key buffers.  Replaces
// the two NCCL all-gathers + combine of the vocab-parallel head.
struct ARKeys {
  const unsigned long long* k[kARMaxRanks];
};

template <int N>
__global__ void __launch_bounds__(kARThreads)
    tp_argmax_kernel(ARPeers P, ARKeys keys, int rank, int rows, int32_t* __restrict__ out, uint32_t host_epoch,
                     uint32_t* err) {
  const uint32_t epoch = cta_epoch(P, rank, host_epoch);
  if (peer_barrier(P, N, rank, 0, epoch, err)) {
    for (int row = blockIdx.x * kARThreads + threadIdx.x; row < rows; row += gridDim.x * kARThreads) {
      unsigned long long best = 0;
#pragma unroll
      for (int p = 0; p < N; ++p) {
        const unsigned long long k = __ldcg(keys.k[p] + row);
        best = k > best ? k : best;
      }
      out[row] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(best & 0xFFFFFFFFu));
    }
    peer_barrier(P, N, rank, 1, epoch, err);
  }
  cta_epoch_done(P, rank, host_epoch, epoch);
}

}  // namespace
}  // namespace ssb

extern "C" {

size_t ssb_tp_signal_bytes(void) {
  return (ssb::kARSlots + ssb::kARMaxBlocks) * sizeof(uint32_t);
}

namespace {
int tp_combine_launch(const uint64_t* part_addrs, const uint64_t* x_addrs, const uint64_t* h_addrs,
                      const uint64_t* ss_addrs, const uint64_t* sig_addrs, int nranks, int rank, int rows,
                      int hidden, int ld, const void* gamma, float eps, uint32_t epoch, int max_blocks,
                      uint32_t* err, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(nranks >= 1 && nranks <= kARMaxRanks, "ssb_tp_allreduce_rmsnorm: nranks %d not in [1, %d]", nranks,
              kARMaxRanks);
  SSB_REQUIRE(rank >= 0 && rank < nranks, "ssb_tp_allreduce_rmsnorm: rank %d of %d", rank, nranks);
  SSB_REQUIRE(rows >= 0 && hidden > 0 && hidden % 8 == 0 && hidden <= 8 * kARThreads * kARMaxVec,
              "ssb_tp_allreduce_rmsnorm: hidden %d must be a multiple of 8 and <= %d", hidden,
              8 * kARThreads * kARMaxVec);
  SSB_REQUIRE(ld >= hidden && ld % 8 == 0, "ssb_tp_allreduce_rmsnorm: bad ld %d", ld);
  SSB_REQUIRE(part_addrs && x_addrs && sig_addrs, "ssb_tp_allreduce_rmsnorm: null address table");
  SSB_REQUIRE(!gamma || h_addrs, "ssb_tp_allreduce_rmsnorm: gamma without h buffers");
  SSB_REQUIRE(max_blocks >= 1, "ssb_tp_allreduce_rmsnorm: max_blocks %d", max_blocks);
  if (rows == 0) return 0;
  ARPeers P{};
  for (int p = 0; p < nranks; ++p) {
    P.part[p] = reinterpret_cast<const __nv_bfloat16*>(part_addrs[p]);
    P.x[p] = reinterpret_cast<__nv_bfloat16*>(x_addrs[p]);
    P.h[p] = gamma ? reinterpret_cast<__nv_bfloat16*>(h_addrs[p]) : nullptr;
    P.ss[p] = ss_addrs ? reinterpret_cast<float*>(ss_addrs[p]) : nullptr;
    P.sig[p] = reinterpret_cast<uint32_t*>(sig_addrs[p]);
    SSB_REQUIRE(aligned16(P.part[p]) && aligned16(P.x[p]) && (!gamma || aligned16(P.h[p])) && P.sig[p] &&
                    (!ss_addrs || P.ss[p]),
                "ssb_tp_allreduce_rmsnorm: rank %d buffers must be 16-byte aligned", p);
  }
  // the grid depends only on (rows, nranks, max_blocks): every rank launches
  // the same CTA indices, which is what the per-CTA barriers pair up
  const int per_rank = (rows + nranks - 1) / nranks;
  const int grid = std::min(std::min(per_rank, max_blocks), kARMaxBlocks);
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const auto* g = static_cast<const __nv_bfloat16*>(gamma);
  switch (nranks) {
#define SSB_AR_CASE(N) \
  case N:              \
    tp_allreduce_rmsnorm_kernel<N><<<grid, kARThreads, 0, s>>>(P, rank, rows, hidden, ld, g, eps, epoch, err); \
    break;
    SSB_AR_CASE(1)
    SSB_AR_CASE(2)
    SSB_AR_CASE(3)
    SSB_AR_CASE(4)
    SSB_AR_CASE(5)
    SSB_AR_CASE(6)
    SSB_AR_CASE(7)
    SSB_AR_CASE(8)
#undef SSB_AR_CASE
  }
  return check_launch("ssb_tp_allreduce_rmsnorm");
}
}  // namespace

int ssb_tp_allreduce_rmsnorm(const uint64_t* part_addrs, const uint64_t* x_addrs, const uint64_t* h_addrs,
                             const uint64_t* sig_addrs, int nranks, int rank, int rows, int hidden, int ld,
                             const void* gamma, float eps, uint32_t epoch, int max_blocks, uint32_t* err,
                             void* stream) {
  return tp_combine_launch(part_addrs, x_addrs, h_addrs, nullptr, sig_addrs, nranks, rank, rows, hidden, ld, gamma,
                           eps, epoch, max_blocks, err, stream);
}

int ssb_tp_allreduce_rowss(const uint64_t* part_addrs, const uint64_t* x_addrs, const uint64_t* ss_addrs,
                           const uint64_t* sig_addrs, int nranks, int rank, int rows, int hidden, int ld,
                           uint32_t epoch, int max_blocks, uint32_t* err, void* stream) {
  SSB_REQUIRE(ss_addrs, "ssb_tp_allreduce_rowss: null ss address table");
  return tp_combine_launch(part_addrs, x_addrs, nullptr, ss_addrs, sig_addrs, nranks, rank, rows, hidden, ld, nullptr,
                           0.f, epoch, max_blocks, err, stream);
}

int ssb_tp_argmax_keys(const uint64_t* key_addrs, const uint64_t* sig_addrs, int nranks, int rank, int rows,
                       int32_t* out_idx, uint32_t epoch, int max_blocks, uint32_t* err, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(nranks >= 1 && nranks <= kARMaxRanks, "ssb_tp_argmax_keys: nranks %d not in [1, %d]", nranks,
              kARMaxRanks);
  SSB_REQUIRE(rank >= 0 && rank < nranks, "ssb_tp_argmax_keys: rank %d of %d", rank, nranks);
  SSB_REQUIRE(key_addrs && sig_addrs && out_idx && rows >= 0, "ssb_tp_argmax_keys: null argument");
  SSB_REQUIRE(max_blocks >= 1, "ssb_tp_argmax_keys: max_blocks %d", max_blocks);
  if (rows == 0) return 0;
  ARPeers P{};
  ARKeys K{};
  for (int p = 0; p < nranks; ++p) {
    P.sig[p] = reinterpret_cast<uint32_t*>(sig_addrs[p]);
    K.k[p] = reinterpret_cast<const unsigned long long*>(key_addrs[p]);
    SSB_REQUIRE(P.sig[p] && K.k[p], "ssb_tp_argmax_keys: rank %d null buffer", p);
  }
  // the peers' key pointers travel by value in the kernel's parameter space
  const int grid = std::min(std::min((rows + kARThreads - 1) / kARThreads, max_blocks), kARMaxBlocks);
  auto s = reinterpret_cast<cudaStream_t>(stream);
  switch (nranks) {
#define SSB_AM_CASE(N)                                                                                   \
  case N:                                                                                                \
    tp_argmax_kernel<N><<<grid, kARThreads, 0, s>>>(P, K, rank, rows, out_idx, epoch, err);              \
    break;
    SSB_AM_CASE(1)
    SSB_AM_CASE(2)
    SSB_AM_CASE(3)
    SSB_AM_CASE(4)
    SSB_AM_CASE(5)
    SSB_AM_CASE(6)
    SSB_AM_CASE(7)
    SSB_AM_CASE(8)
#undef SSB_AM_CASE
  }
  return check_launch("ssb_tp_argmax_keys");
}

}  // extern "C"
