// fbf_iir.cu -- the reference's recursive convolution backend on the GPU
// (ConvolutionBackend::recursive; reference: recursive_gaussian.hpp:1-87,
// spatial.hpp:98-112 dispatch, bilateral.hpp:109-160 Algorithm 1).
//
// The reference substitutes a third-order recursive Gaussian (van Vliet,
// Young and Verbeek) for the FIR when the window is Gaussian with sigma >= 2:
// each line is mirror-padded by pad = ceil(4 sigma) + 12 samples, run forward
// and backward through y = g x + a1 y1 + a2 y2 + a3 y3 with the start-up state
// set to the first (last) padded sample.  This is an approximation of the
// Gaussian, not a faster way to the same numbers, so it stays an alternative
// backend next to the fused FIR kernel and follows the reference's arithmetic
// in fp64, in its evaluation order (explicit __dmul_rn / __dadd_rn: no
// contraction), for parity with the reference build.
//
// Layout: one image at a time, planes [4][rows][cols] fp64 in the workspace.
// A recursion runs down columns (one thread per column and plane: coalesced
// across the warp); the row pass is the column pass of the transposed planes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "fbf_common.h"
#include "fbf_device.cuh"
#include "fbf_params.h"
#include "fourierbf_b200.h"

namespace fbf {

namespace {

struct Vyv {
  double a1, a2, a3, gain;
  int pad;
};

// recursive_gaussian.hpp:20-39
Vyv vyv_coeffs(double sigma) {
  const double q = sigma >= 2.5 ? 0.98711 * sigma - 0.96330 : 3.97156 - 4.14554 * std::sqrt(1.0 - 0.26891 * sigma);
  const double q2 = q * q, q3 = q2 * q;
  const double b0 = 1.57825 + 2.44413 * q + 1.42810 * q2 + 0.422205 * q3;
  const double b1 = 2.44413 * q + 2.85619 * q2 + 1.26661 * q3;
  const double b2 = -(1.42810 * q2 + 1.26661 * q3);
  const double b3 = 0.422205 * q3;
  Vyv c;
  c.a1 = b1 / b0;
  c.a2 = b2 / b0;
  c.a3 = b3 / b0;
  c.gain = 1.0 - (c.a1 + c.a2 + c.a3);
  c.pad = static_cast<int>(std::ceil(4.0 * sigma)) + 12;  // recursive_gaussian.hpp:41
  return c;
}

__device__ __forceinline__ double vyv_step(const Vyv& c, double x, double y1, double y2, double y3) {
  // c.gain * x + c.a1 * y1 + c.a2 * y2 + c.a3 * y3, left to right, unfused
  double y = __dmul_rn(c.gain, x);
  y = __dadd_rn(y, __dmul_rn(c.a1, y1));
  y = __dadd_rn(y, __dmul_rn(c.a2, y2));
  return __dadd_rn(y, __dmul_rn(c.a3, y3));
}

// recursive_gaussian.hpp:45-70 down every column of `planes` planes
// [rows][cols]; tmp holds the forward pass over the padded column.
__global__ void iir_columns(const double* __restrict__ in, double* __restrict__ out, double* __restrict__ tmp,
                            int rows, int cols, Vyv c) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= cols) return;
  const long long plane = static_cast<long long>(blockIdx.y) * rows * cols;
  const int m = rows + 2 * c.pad;
  const double* __restrict__ src = in + plane + x;
  double* __restrict__ t = tmp + static_cast<long long>(blockIdx.y) * m * cols + x;
  double* __restrict__ dst = out + plane + x;
  double y1 = src[static_cast<long long>(mirror_index(-c.pad, rows)) * cols], y2 = y1, y3 = y1;
#pragma unroll 8
  for (int i = 0; i < m; ++i) {  // forward; start-up state = the first padded sample
    const double y = vyv_step(c, src[static_cast<long long>(mirror_index(i - c.pad, rows)) * cols], y1, y2, y3);
    t[static_cast<long long>(i) * cols] = y;
    y3 = y2;
    y2 = y1;
    y1 = y;
  }
  y1 = y2 = y3 = t[static_cast<long long>(m - 1) * cols];
#pragma unroll 8
  for (int i = m - 1; i >= 0; --i) {  // backward
    const double y = vyv_step(c, t[static_cast<long long>(i) * cols], y1, y2, y3);
    if (i >= c.pad && i < c.pad + rows) dst[static_cast<long long>(i - c.pad) * cols] = y;
    y3 = y2;
    y2 = y1;
    y1 = y;
  }
}

// [plane][rows][cols] -> [plane][cols][rows], 32 x 32 tiles through shared memory
__global__ void transpose_planes(const double* __restrict__ in, double* __restrict__ out, int rows, int cols) {
  __shared__ double tile[32][33];
  const long long plane = static_cast<long long>(blockIdx.z) * rows * cols;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int y = y0 + dy, x = x0 + threadIdx.x;
    if (y < rows && x < cols) tile[dy][threadIdx.x] = in[plane + static_cast<long long>(y) * cols + x];
  }
  __syncthreads();
  for (int dx = threadIdx.y; dx < 32; dx += blockDim.y) {
    const int x = x0 + dx, y = y0 + threadIdx.x;
    if (x < cols && y < rows) out[plane + static_cast<long long>(x) * rows + y] = tile[threadIdx.x][dx];
  }
}

// bilateral.hpp:126-133 for harmonics n0 .. n0+hb-1: planes [h][0..3] =
// f cos, f sin, cos, sin of phase = (omega n) f
template <class T>
__global__ void modulate_f64(const T* __restrict__ src, int pitch, int rows, int cols, double omega, int n0, int hb,
                             double* __restrict__ planes) {
  const long long px = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < px;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(i / cols), x = static_cast<int>(i - static_cast<long long>(y) * cols);
    const double f = static_cast<double>(src[static_cast<long long>(y) * pitch + x]);
    for (int h = 0; h < hb; ++h) {
      double s, c;
      sincos(__dmul_rn(omega * (n0 + h), f), &s, &c);  // freq = omega * n (bilateral.hpp:127)
      double* p = planes + 4 * h * px;
      p[i] = __dmul_rn(c, f);
      p[px + i] = __dmul_rn(s, f);
      p[2 * px + i] = c;
      p[3 * px + i] = s;
    }
  }
}

constexpr int kIirBlock = 16;  // harmonics per modulate / IIR / demod round
struct DnBlock {
  double d[kIirBlock];
};

// bilateral.hpp:138-144, harmonics in ascending order:
// P += d_n (cos fcos_s + sin fsin_s), Q += d_n (cos cos_s + sin sin_s)
__global__ void demod_f64(const double* __restrict__ mod, const double* __restrict__ conv, long long px, int hb,
                          DnBlock dn, double* __restrict__ P, double* __restrict__ Q) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < px;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double p = P[i], q = Q[i];
    for (int h = 0; h < hb; ++h) {
      const double* m = mod + 4 * h * px;
      const double* v = conv + 4 * h * px;
      const double c = m[2 * px + i], s = m[3 * px + i];
      p = __dadd_rn(p, __dmul_rn(dn.d[h], __dadd_rn(__dmul_rn(c, v[i]), __dmul_rn(s, v[px + i]))));
      q = __dadd_rn(q, __dmul_rn(dn.d[h], __dadd_rn(__dmul_rn(c, v[2 * px + i]), __dmul_rn(s, v[3 * px + i]))));
    }
    P[i] = p;
    Q[i] = q;
  }
}

// bilateral.hpp:147-158
template <class T>
__global__ void divide_f64(const double* __restrict__ P, const double* __restrict__ Q, int rows, int cols,
                           int dst_pitch, double q_floor, unsigned long long lin0, unsigned long long* bad,
                           T* __restrict__ dst) {
  const long long px = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < px;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (!(fabs(Q[i]) >= q_floor) && bad) atomicMin(bad, lin0 + static_cast<unsigned long long>(i));
    const int y = static_cast<int>(i / cols), x = static_cast<int>(i - static_cast<long long>(y) * cols);
    dst[static_cast<long long>(y) * dst_pitch + x] = static_cast<T>(P[i] / Q[i]);
  }
}

unsigned grid_1d(long long n) {
  return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 32)));
}

// Separable IIR of the 4 planes in `a` ([4][rows][cols]); result in `a`.
cudaError_t iir_planes(double* a, double* b, double* tmp, int rows, int cols, int nplanes, const Vyv& c,
                       cudaStream_t st) {
  iir_columns<<<dim3((cols + 127) / 128, nplanes), 128, 0, st>>>(a, b, tmp, rows, cols, c);
  transpose_planes<<<dim3((cols + 31) / 32, (rows + 31) / 32, nplanes), dim3(32, 8), 0, st>>>(b, a, rows, cols);
  iir_columns<<<dim3((rows + 127) / 128, nplanes), 128, 0, st>>>(a, b, tmp, cols, rows, c);
  transpose_planes<<<dim3((rows + 31) / 32, (cols + 31) / 32, nplanes), dim3(32, 8), 0, st>>>(b, a, cols, rows);
  return cudaGetLastError();
}

struct IirLayout {
  size_t a, b, c, tmp, p, q, total;
};

// harmonics per round: as many as fit ~4 GB of planes (more independent
// recursions per launch: one thread per column and plane), at most kIirBlock
int iir_block(int width, int height, int pad) {
  const double per = 8.0 * 4 * (3.0 * width * height + double(std::max(width, height) + 2 * pad) * std::max(width, height));
  return std::max(1, std::min(kIirBlock, static_cast<int>(4.0e9 / per)));
}

IirLayout iir_layout(int width, int height, int pad) {
  const size_t px = static_cast<size_t>(width) * height;
  const size_t hb = static_cast<size_t>(iir_block(width, height, pad));
  const size_t tmp = 4 * hb * static_cast<size_t>(std::max(width, height) + 2 * pad) * std::max(width, height);
  IirLayout L{};
  L.a = 0;
  L.b = L.a + align256(4 * hb * px * 8);
  L.c = L.b + align256(4 * hb * px * 8);
  L.tmp = L.c + align256(4 * hb * px * 8);
  L.p = L.tmp + align256(tmp * 8);
  L.q = L.p + align256(px * 8);
  L.total = L.q + align256(px * 8);
  return L;
}

}  // namespace

// workspace of the recursive path for spatial radius W (sigma <= W / 3)
// the workspace is sized from the radius: W = ceil(3 sigma) bounds the pad
int iir_pad_bound(int radius) { return static_cast<int>(std::ceil(4.0 * radius / 3.0)) + 13; }

size_t iir_workspace_bytes(const fbf_geometry* g, int radius) {
  return iir_layout(g->width, g->height, iir_pad_bound(radius)).total;
}

// bilateral_fast with the recursive backend: whole images (the recursion runs
// over complete lines), fp64 throughout; src / dst device pointers with the
// geometry's pitches and strides.
template <class Tin, class Tout>
int iir_bilateral(const fbf_geometry* g, const fbf_filter* f, const Tin* src, Tout* dst, void* ws, size_t ws_bytes,
                  unsigned long long* d_bad, cudaStream_t st) {
  if (g->src_row0 != 0 || g->src_rows != g->height || g->out_row0 != 0 || g->out_rows != g->height)
    return fail(FBF_EUNSUPPORTED, "bilateral_fast: the recursive backend filters whole images only");
  const Vyv c = vyv_coeffs(f->sigma_s);
  const int pad_bound = iir_pad_bound(f->radius);
  if (c.pad > pad_bound)
    return fail(FBF_EINVAL, "bilateral_fast: sigma_s does not match the window radius (W = ceil(3 sigma))");
  const IirLayout L = iir_layout(g->width, g->height, pad_bound);
  if (!ws || ws_bytes < L.total) return fail(FBF_EINVAL, "bilateral_fast: workspace too small (recursive backend)");
  char* base = static_cast<char*>(ws);
  double* A = reinterpret_cast<double*>(base + L.a);
  double* B = reinterpret_cast<double*>(base + L.b);
  double* C = reinterpret_cast<double*>(base + L.c);
  double* T = reinterpret_cast<double*>(base + L.tmp);
  double* P = reinterpret_cast<double*>(base + L.p);
  double* Q = reinterpret_cast<double*>(base + L.q);
  const int rows = g->height, cols = g->width;
  const long long px = static_cast<long long>(rows) * cols;
  const double q_floor = (f->w0 - f->max_pointwise_error) / 2.0;
  const int HB = iir_block(g->width, g->height, pad_bound);
  for (int b = 0; b < g->batch; ++b) {
    FBF_CUDA(cudaMemsetAsync(P, 0, px * 8, st));
    FBF_CUDA(cudaMemsetAsync(Q, 0, px * 8, st));
    for (int n0 = 0; n0 <= f->N; n0 += HB) {
      const int hb = std::min(HB, f->N + 1 - n0);
      modulate_f64<Tin><<<grid_1d(px), 256, 0, st>>>(src + b * g->src_bstride, static_cast<int>(g->src_pitch), rows,
                                                     cols, f->omega, n0, hb, A);
      FBF_CUDA(cudaMemcpyAsync(C, A, 4 * hb * px * 8, cudaMemcpyDeviceToDevice, st));
      FBF_CUDA(iir_planes(C, B, T, rows, cols, 4 * hb, c, st));
      DnBlock dn{};
      for (int h = 0; h < hb; ++h) dn.d[h] = f->d[n0 + h];
      demod_f64<<<grid_1d(px), 256, 0, st>>>(A, C, px, hb, dn, P, Q);
    }
    divide_f64<Tout><<<grid_1d(px), 256, 0, st>>>(P, Q, rows, cols, static_cast<int>(g->dst_pitch), q_floor,
                                                   static_cast<unsigned long long>(b) * px, d_bad,
                                                   dst + b * g->dst_bstride);
    FBF_CUDA(cudaGetLastError());
  }
  return FBF_OK;
}

template int iir_bilateral<float, float>(const fbf_geometry*, const fbf_filter*, const float*, float*, void*, size_t,
                                         unsigned long long*, cudaStream_t);
template int iir_bilateral<double, double>(const fbf_geometry*, const fbf_filter*, const double*, double*, void*,
                                           size_t, unsigned long long*, cudaStream_t);

}  // namespace fbf

// convolve (spatial.hpp:98-112) with the recursive backend: the IIR of one
// fp64 plane (the caller has checked gaussian and sigma >= 2).
int fbf_convolve_recursive_host_f64(int width, int height, double sigma, const double* src, double* dst) {
  using namespace fbf;
  if (width <= 0 || height <= 0) return fail(FBF_EINVAL, "convolve: empty plane");
  if (!(sigma > 0.0)) return fail(FBF_EINVAL, "convolve: sigma must be positive");
  const Vyv c = vyv_coeffs(sigma);
  const size_t px = static_cast<size_t>(width) * height;
  const size_t tmp = static_cast<size_t>(std::max(width, height) + 2 * c.pad) * std::max(width, height);
  double* buf = nullptr;
  FBF_CUDA(cudaMalloc(reinterpret_cast<void**>(&buf), (2 * px + tmp) * sizeof(double)));
  cudaError_t e = cudaMemcpy(buf, src, px * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = iir_planes(buf, buf + px, buf + 2 * px, height, width, 1, c, nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(dst, buf, px * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(buf);
  if (e != cudaSuccess) return cuda_fail(e, "convolve (recursive)");
  return FBF_OK;
}
