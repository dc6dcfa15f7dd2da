// Debug only: the HBM read ceiling decode attention streams against.  A
// persistent kernel of `ctas_per_sm` CTAs per SM, each streaming `chunk`-byte
// pieces of a contiguous buffer through a `stages`-deep ring of bulk copies
// (cp.async.bulk, mbarrier completion), consuming nothing -- the largest read
// bandwidth a TMA-fed kernel can see (tools/read_bw.py).
#include "common.cuh"
#include "seesaw_b200.h"

namespace ssb {
namespace {

__global__ void __launch_bounds__(32) read_stream_kernel(const uint8_t* __restrict__ src, int64_t n_chunks,
                                                         int chunk, int stages) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
  fence_mbar_init();
  const int64_t stride = gridDim.x;
  int64_t issued = 0, done = 0;
  int64_t next = blockIdx.x;
  // prime the ring, then one wait + one refill per chunk
  for (; issued < stages && next < n_chunks; ++issued, next += stride) {
    mbar_arrive_expect_tx(&full[issued], chunk);
    bulk_g2s(ring + issued * chunk, src + next * chunk, chunk, &full[issued]);
  }
  while (done < issued) {
    const int s = static_cast<int>(done % stages);
    mbar_wait(&full[s], static_cast<uint32_t>((done / stages) & 1));
    ++done;
    if (next < n_chunks) {
      mbar_arrive_expect_tx(&full[s], chunk);
      bulk_g2s(ring + s * chunk, src + next * chunk, chunk, &full[s]);
      ++issued;
      next += stride;
    }
  }
}

}  // namespace
}  // namespace ssb

extern "C" int ssb_debug_read_stream(const void* src, int64_t bytes, int ctas_per_sm, int chunk, int stages,
                                     void* stream) {
  using namespace ssb;
  SSB_REQUIRE(src && bytes > 0 && chunk >= 16 && chunk % 16 == 0 && stages >= 1 && stages <= 16 &&
                  ctas_per_sm >= 1 && static_cast<int64_t>(chunk) * stages <= 200 * 1024,
              "ssb_debug_read_stream: bad arguments");
  const int smem = chunk * stages;
  SSB_CUDA(cudaFuncSetAttribute(read_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  read_stream_kernel<<<num_sms() * ctas_per_sm, 32, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), bytes / chunk, chunk, stages);
  return check_launch("read_stream_kernel");
}
