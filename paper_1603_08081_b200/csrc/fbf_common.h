// fbf_common.h -- status helpers shared by the C-ABI translation units
// (definitions in fbf_capi.cu: the thread-local message of fbf_last_error()).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <string>

namespace fbf {

int fail(int code, const std::string& msg);          // records the message, returns code
int cuda_fail(cudaError_t e, const char* where);     // FBF_ECUDA with the CUDA error text
inline size_t align256(size_t n) { return (n + 255) & ~size_t(255); }

}  // namespace fbf

#define FBF_CUDA(call)                                        \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return ::fbf::cuda_fail(e_, #call); \
  } while (0)
