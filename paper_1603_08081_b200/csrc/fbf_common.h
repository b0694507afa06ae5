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
void sm_count(int dev, int* sms);  // cached SM count of a device

}  // namespace fbf

// internal interface between the device entry points (fbf_capi.cu) and the
// host-buffer pipelines (fbf_hostpath.cu)
struct fbf_geometry;
struct fbf_filter;
namespace fbf {
size_t workspace_for(const fbf_geometry* g, const fbf_filter* f, int variant);  // bytes a device call needs
int check_call(const fbf_geometry* g, const fbf_filter* f);                     // geometry, filter and halo checks
bool recursive_applies(const fbf_filter* f);  // the IIR backend replaces the FIR (spatial.hpp:102-104)
bool fused_applies(const fbf_filter* f);      // a fused kernel covers this window

}  // namespace fbf

#define FBF_CUDA(call)                                        \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return ::fbf::cuda_fail(e_, #call); \
  } while (0)
