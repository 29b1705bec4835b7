// Shared host-side plumbing for libzpp: error state, SM count, TMA descriptor encode.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/zpp.h"

namespace zpp {

int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
int check_launch(const char* what);
int num_sms();
int encode_tensor_map(CUtensorMap* map, CUtensorMapDataType dtype, int rank, void* ptr, const cuuint64_t* dims,
                      const cuuint64_t* strides_bytes, const cuuint32_t* box, const cuuint32_t* estrides,
                      CUtensorMapSwizzle swizzle);

}  // namespace zpp
