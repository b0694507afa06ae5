// fbf_exact.cu -- brute-force bilateral filter on the GPU, fp64
// (reference: bilateral_exact, /root/reference/proj/include/fourierbf/bilateral.hpp:78-102).
//
// The accuracy oracle of the reference API, O((2W+1)^2) per pixel.  Used to
// check the paper's error bound 2 T eps / (w0 - eps) at full BASELINE sizes
// (SURVEY.md §8(f) rank 1), where the CPU brute force would take ~30 min (c4).
// Accumulation in fp64 like the reference; range kernel evaluated exactly
// (exp) per tap; same mirror boundary.
#include <cuda_runtime.h>

#include "fbf_device.cuh"
#include "fourierbf_b200.h"

namespace {

constexpr int TX = 16, TY = 16;

// one thread per output pixel; the block's (16+2W)^2 input tile in smem (fp64)
template <class Tin>
__global__ void exact_kernel(const Tin* __restrict__ src, double* __restrict__ dst, int width, int height,
                             int src_row0, int out_row0, int out_rows, const double* __restrict__ prof_g, int W,
                             int family, double inv_scale) {
  extern __shared__ double tile[];
  const int TW = TX + 2 * W, TH = TY + 2 * W;
  double* prof = tile + TW * TH;
  const int x0 = blockIdx.x * TX, y0 = out_row0 + blockIdx.y * TY;
  for (int i = threadIdx.y * TX + threadIdx.x; i < TW * TH; i += TX * TY) {
    const int ty = i / TW, tx = i - ty * TW;
    const int gy = fbf::mirror_index(y0 - W + ty, height) - src_row0;
    const int gx = fbf::mirror_index(x0 - W + tx, width);
    tile[i] = static_cast<double>(src[static_cast<long long>(gy) * width + gx]);
  }
  for (int i = threadIdx.y * TX + threadIdx.x; i <= 2 * W; i += TX * TY) prof[i] = prof_g[i];
  __syncthreads();
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  if (x >= width || y >= out_row0 + out_rows) return;
  const double center = tile[(threadIdx.y + W) * TW + threadIdx.x + W];
  double num = 0.0, den = 0.0;
  for (int dy = -W; dy <= W; ++dy) {
    // bilateral.hpp:90-99: sy = mirror(y - dy), sx = mirror(x - dx), weight(dx, dy)
    const double* row = tile + (threadIdx.y + W - dy) * TW + threadIdx.x + W;
    const double py = prof[dy + W];
    for (int dx = -W; dx <= W; ++dx) {
      const double v = row[-dx];
      const double a = fabs(v - center);
      const double r = family == FBF_RANGE_EXPONENTIAL ? exp(-a * inv_scale) : exp(-(a * a) * inv_scale);
      const double wgt = (prof[dx + W] * py) * r;
      num += wgt * v;
      den += wgt;
    }
  }
  dst[static_cast<long long>(y - out_row0) * width + x] = num / den;
}

template <class Tin>
int exact_any(const fbf_geometry* g, const double* profile, int radius, int family, double sigma_r, const Tin* src,
              double* dst, cudaStream_t st) {
  if (!g || g->width <= 0 || g->height <= 0 || g->batch != 1 || radius < 1 || radius > 64 || !(sigma_r > 0.0))
    return FBF_EINVAL;
  double* d_prof = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&d_prof), sizeof(double) * (2 * radius + 1), st) != cudaSuccess)
    return FBF_ECUDA;
  cudaMemcpyAsync(d_prof, profile, sizeof(double) * (2 * radius + 1), cudaMemcpyHostToDevice, st);
  const double inv_scale =
      family == FBF_RANGE_EXPONENTIAL ? 1.0 / sigma_r : 1.0 / (2.0 * sigma_r * sigma_r);  // kernels.hpp:83-85
  const size_t smem = sizeof(double) * ((TX + 2 * radius) * (TY + 2 * radius) + 2 * radius + 1);
  cudaFuncSetAttribute(exact_kernel<Tin>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  const dim3 grid((g->width + TX - 1) / TX, (g->out_rows + TY - 1) / TY);
  exact_kernel<Tin><<<grid, dim3(TX, TY), smem, st>>>(src, dst, g->width, g->height, g->src_row0, g->out_row0,
                                                      g->out_rows, d_prof, radius, family, inv_scale);
  cudaFreeAsync(d_prof, st);
  return cudaGetLastError() == cudaSuccess ? FBF_OK : FBF_ECUDA;
}

}  // namespace

extern "C" int fbf_bilateral_exact_device(const fbf_geometry* g, const double* profile, int radius, int family,
                                          double sigma_r, const float* src, double* dst, void* stream) {
  return exact_any<float>(g, profile, radius, family, sigma_r, src, dst, static_cast<cudaStream_t>(stream));
}

// bilateral_exact of a whole fp64 host image (the C++ API's Gaussian and
// exponential range kernels): H2D, the kernel above in fp64, D2H.
extern "C" int fbf_bilateral_exact_host_f64(int width, int height, const double* profile, int radius, int family,
                                            double sigma_r, const double* src, double* dst) {
  if (width <= 0 || height <= 0) return FBF_EINVAL;
  fbf_geometry g;
  fbf_geometry_whole(&g, width, height, 1);
  const size_t n = static_cast<size_t>(width) * height;
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return FBF_ECUDA;
  double* buf = nullptr;
  int rc = FBF_ECUDA;
  if (cudaMallocAsync(reinterpret_cast<void**>(&buf), 2 * n * sizeof(double), st) == cudaSuccess) {
    rc = cudaMemcpyAsync(buf, src, n * sizeof(double), cudaMemcpyHostToDevice, st) == cudaSuccess ? FBF_OK : FBF_ECUDA;
    if (rc == FBF_OK) rc = exact_any<double>(&g, profile, radius, family, sigma_r, buf, buf + n, st);
    if (rc == FBF_OK && cudaMemcpyAsync(dst, buf + n, n * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      rc = FBF_ECUDA;
    cudaFreeAsync(buf, st);
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) rc = FBF_ECUDA;
  cudaStreamDestroy(st);
  return rc;
}
