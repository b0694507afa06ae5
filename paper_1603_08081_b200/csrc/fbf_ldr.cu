// fbf_ldr.cu -- local dynamic range on the GPU
// (reference: local_dynamic_range, /root/reference/proj/include/fourierbf/bilateral.hpp:21-74).
//
// T = ceil( max over pixels of (windowed max - windowed min) ) over the
// (2W+1)^2 window with the filter's mirror boundary, as two separable passes
// (max/min are exact, so the pass order and fp64 arithmetic reproduce the
// reference value exactly).  Feeds the host-side progressive fit in filter().
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "fbf_device.cuh"
#include "fourierbf_b200.h"

namespace {

__global__ void ldr_rows(const double* __restrict__ img, double* __restrict__ hi, double* __restrict__ lo,
                         int w, int h, int W) {
  const long long total = static_cast<long long>(w) * h;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long row = i / w;
    const int x = static_cast<int>(i - row * w);
    const double* r = img + row * w;
    double a = r[x], b = r[x];
    for (int k = -W; k <= W; ++k) {
      const double v = r[fbf::mirror_index(x + k, w)];
      a = fmax(a, v);
      b = fmin(b, v);
    }
    hi[i] = a;
    lo[i] = b;
  }
}

__global__ void ldr_cols(const double* __restrict__ hi, const double* __restrict__ lo, int w, int h, int W,
                         unsigned long long* __restrict__ spread_bits) {
  const long long total = static_cast<long long>(w) * h;
  double best = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(i / w);
    const int x = static_cast<int>(i - static_cast<long long>(y) * w);
    double a = hi[i], b = lo[i];
    for (int k = -W; k <= W; ++k) {
      const long long s = static_cast<long long>(fbf::mirror_index(y + k, h)) * w + x;
      a = fmax(a, hi[s]);
      b = fmin(b, lo[s]);
    }
    best = fmax(best, a - b);
  }
  // non-negative doubles order like their bit patterns
  for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
  if ((threadIdx.x & 31) == 0) atomicMax(spread_bits, static_cast<unsigned long long>(__double_as_longlong(best)));
}

}  // namespace

extern "C" int fbf_local_dynamic_range_host_f64(const double* img, int width, int height, int W, int* T) {
  if (width <= 0 || height <= 0 || W < 1 || !img || !T) return FBF_EINVAL;
  const size_t n = static_cast<size_t>(width) * height;
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return FBF_ECUDA;
  char* buf = nullptr;
  int rc = FBF_OK;
  if (cudaMallocAsync(reinterpret_cast<void**>(&buf), 3 * n * sizeof(double) + 256, st) != cudaSuccess) {
    cudaStreamDestroy(st);
    return FBF_ECUDA;
  }
  double* d_img = reinterpret_cast<double*>(buf);
  double* d_hi = d_img + n;
  double* d_lo = d_hi + n;
  unsigned long long* d_spread = reinterpret_cast<unsigned long long*>(d_lo + n);
  unsigned long long bits = 0;
  cudaMemcpyAsync(d_img, img, n * sizeof(double), cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(d_spread, 0, sizeof(unsigned long long), st);
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 148 * 16));
  ldr_rows<<<blocks, 256, 0, st>>>(d_img, d_hi, d_lo, width, height, W);
  ldr_cols<<<blocks, 256, 0, st>>>(d_hi, d_lo, width, height, W, d_spread);
  cudaMemcpyAsync(&bits, d_spread, sizeof(bits), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) rc = FBF_ECUDA;
  cudaFreeAsync(buf, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc == FBF_OK) {
    double spread = 0.0;
    std::memcpy(&spread, &bits, sizeof(spread));
    *T = static_cast<int>(std::ceil(spread));
  }
  return rc;
}
