// Library-wide plumbing of the C ABI: per-thread error text, version,
// cached device attributes and the driver entry point for TMA descriptors.
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "seesaw_b200.h"

namespace ssb {

static thread_local char g_err[512] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail_arg(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return SSB_EARG;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

static std::atomic<int> g_pdl{-1};

bool pdl_enabled() {
  int v = g_pdl.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("SSB_PDL");
    v = (e && atoi(e) == 0) ? 0 : 1;
    g_pdl.store(v, std::memory_order_relaxed);
  }
  return v != 0;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point, so the
// library does not link libcuda directly.
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

int encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                        uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) {
    set_error("cuTensorMapEncodeTiled entry point unavailable");
    return SSB_EUNSUPPORTED;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu stride=%llu box=%ux%u",
              static_cast<int>(r), (unsigned long long)inner, (unsigned long long)outer,
              (unsigned long long)row_stride_bytes, box_inner, box_outer);
    return SSB_EUNSUPPORTED;
  }
  return 0;
}

}  // namespace ssb

extern "C" {

const char* ssb_last_error(void) { return ssb::g_err; }

int ssb_version(void) { return SSB_ABI_VERSION; }

int ssb_device_sm_count(void) { return ssb::num_sms(); }

int ssb_set_pdl(int on) {
  const int prev = ssb::pdl_enabled() ? 1 : 0;
  ssb::g_pdl.store(on ? 1 : 0, std::memory_order_relaxed);
  return prev;
}

int ssb_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out) {
  using namespace ssb;
  SSB_REQUIRE(ptr && handle_out && offset_out, "ssb_ipc_export: null argument");
  // the cudaMalloc allocation holding ptr (a caching allocator hands out
  // interior pointers): its base is what the handle names
  static PFN_cuMemGetAddressRange_v3020 range = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  });
  if (!range) {
    set_error("ssb_ipc_export: cuMemGetAddressRange entry point unavailable");
    return SSB_EUNSUPPORTED;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) {
    set_error("ssb_ipc_export: cuMemGetAddressRange failed for %p", ptr);
    return SSB_EARG;
  }
  cudaIpcMemHandle_t h;
  SSB_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = static_cast<int64_t>(reinterpret_cast<uintptr_t>(ptr) - static_cast<uintptr_t>(base));
  return 0;
}

int ssb_ipc_open(const void* handle, int device, void** out_ptr) {
  using namespace ssb;
  SSB_REQUIRE(handle && out_ptr, "ssb_ipc_open: null argument");
  int prev = 0;
  SSB_CUDA(cudaGetDevice(&prev));
  SSB_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("ssb_ipc_open: cudaIpcOpenMemHandle on device %d: %s", device, cudaGetErrorString(e));
    return static_cast<int>(e);
  }
  return 0;
}

int ssb_ipc_close(void* ptr, int device) {
  using namespace ssb;
  int prev = 0;
  SSB_CUDA(cudaGetDevice(&prev));
  SSB_CUDA(cudaSetDevice(device));
  const cudaError_t e = cudaIpcCloseMemHandle(ptr);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("ssb_ipc_close: %s", cudaGetErrorString(e));
    return static_cast<int>(e);
  }
  return 0;
}

int ssb_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                       int64_t height, void* stream) {
  using namespace ssb;
  SSB_REQUIRE(width >= 0 && height >= 0 && dpitch >= width && spitch >= width,
              "ssb_memcpy2d_async: bad geometry");
  if (width == 0 || height == 0) return 0;
  SSB_REQUIRE(dst && src, "ssb_memcpy2d_async: null pointer");
  SSB_CUDA(cudaMemcpy2DAsync(dst, static_cast<size_t>(dpitch), src, static_cast<size_t>(spitch),
                             static_cast<size_t>(width), static_cast<size_t>(height), cudaMemcpyDefault,
                             reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}

}  // extern "C"
