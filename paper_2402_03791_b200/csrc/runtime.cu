// Error state, device queries and the driver-API TMA encoder for libzpp.
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "zpp_internal.h"

namespace zpp {

static thread_local char g_err[512] = "ok";

int set_error(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

int set_cuda_error(cudaError_t e, const char* where) {
  snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
  return ZPP_ERR_CUDA;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, what);
  return ZPP_OK;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encoder() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int encode_tensor_map(CUtensorMap* map, CUtensorMapDataType dtype, int rank, void* ptr, const cuuint64_t* dims,
                      const cuuint64_t* strides_bytes, const cuuint32_t* box, const cuuint32_t* estrides,
                      CUtensorMapSwizzle swizzle) {
  EncodeTiledFn fn = get_encoder();
  if (!fn) return set_error(ZPP_ERR_DRIVER, "cuTensorMapEncodeTiled unavailable");
  CUresult r = fn(map, dtype, rank, ptr, dims, strides_bytes, box, estrides, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d): dims %llu x %llu", (int)r,
             (unsigned long long)dims[0], (unsigned long long)(rank > 1 ? dims[1] : 1));
    return set_error(ZPP_ERR_DRIVER, buf);
  }
  return ZPP_OK;
}

}  // namespace zpp

extern "C" const char* zpp_last_error(void) { return zpp::g_err; }
extern "C" int zpp_num_sms(void) { return zpp::num_sms(); }
extern "C" int zpp_version(void) { return 1; }

extern "C" int zpp_zero(void* ptr, long long bytes, uintptr_t stream) {
  cudaError_t e = cudaMemsetAsync(ptr, 0, (size_t)bytes, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? ZPP_OK : zpp::set_cuda_error(e, "zpp_zero");
}
