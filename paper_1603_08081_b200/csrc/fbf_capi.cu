// fbf_capi.cu -- the device-side extern "C" boundary (include/fourierbf_b200.h)
// plus the small kernels around the fused one: the phase prep, the naive
// multi-kernel variant (HBM-resident planes), the group sum / divide, the
// standalone separable convolution (fp32 and fp64) and the FP32 FMA-pipe peak
// probe used as the roofline denominator.  The host-buffer entry points
// (pipelines, per-device contexts, multi-GPU) live in fbf_hostpath.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fbf_common.h"
#include "fbf_device.cuh"
#include "fbf_params.h"
#include "fbf_tuning.h"
#include "fourierbf_b200.h"

namespace fbf {
bool fused_supported(int W, bool box);
cudaError_t launch_fused(const FusedArgs& a, cudaStream_t st, FusedPlan* plan);
}  // namespace fbf

using namespace fbf;

namespace {
thread_local std::string g_err;
}  // namespace

namespace fbf {
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(FBF_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
// recursive (IIR) backend, fbf_iir.cu
size_t iir_workspace_bytes(const fbf_geometry* g, int radius);
template <class Tin, class Tout>
int iir_bilateral(const fbf_geometry* g, const fbf_filter* f, const Tin* src, Tout* dst, void* ws, size_t ws_bytes,
                  unsigned long long* d_bad, cudaStream_t st);
// per-device SM count, cached (group model, launch shapes)
void sm_count(int dev, int* sms) {
  static int cache[64] = {};
  *sms = 148;
  if (dev >= 0 && dev < 64) {
    if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
    if (cache[dev] > 0) *sms = cache[dev];
  }
}
}  // namespace fbf

namespace {

// ---------------------------------------------------------------------------
// prep: (u, f') per source pixel.  u = round(f' * omega/(2 pi) * 2^32) mod 2^32
// in fp64 (exact base phase in turns), f' = f - shift.

// max |f'| of the call into the workspace header (fixed-point P grid,
// fbf_params.h): one atomic per warp
// max |f'| of the call: warp shuffle, then one shared-memory and one global
// atomic per CTA (same-address global atomics per warp serialised in L2 and
// were most of the prep kernel's time: c2 56 us -> see profiles/r02_notes.md)
__device__ __forceinline__ void note_fmax(float m, unsigned* fmax) {
  __shared__ unsigned cta_max;
  if (threadIdx.x == 0) cta_max = 0u;
  __syncthreads();
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(&cta_max, __float_as_uint(m));
  __syncthreads();
  if (threadIdx.x == 0 && cta_max) atomicMax(fmax, cta_max);
}

__device__ __forceinline__ int2 phase_of(float f, double turns_scaled, float shift, float& m) {
  const double fd = static_cast<double>(f) - static_cast<double>(shift);
  const long long u = __double2ll_rn(fd * turns_scaled);
  const float ff = static_cast<float>(fd);
  m = fmaxf(m, fabsf(ff));
  return make_int2(static_cast<int>(static_cast<unsigned>(u)), __float_as_int(ff));
}

// naive path: dense (u, f') of the source rows, batch x src_rows x width
__global__ void prep_kernel(const float* __restrict__ src, int2* __restrict__ uf, Geometry g, double turns_scaled,
                            float shift, unsigned* fmax) {
  const long long per = static_cast<long long>(g.src_rows) * g.width;
  const long long total = per * g.batch;
  float m = 0.f;
  for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x); i0 < total;
       i0 += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = i0 + threadIdx.x;
    if (i >= total) continue;
    const long long b = i / per;
    const long long r = i - b * per;
    const int y = static_cast<int>(r / g.width);
    const int x = static_cast<int>(r - static_cast<long long>(y) * g.width);
    uf[i] = phase_of(src[b * g.src_bstride + static_cast<long long>(y) * g.src_pitch + x], turns_scaled, shift, m);
  }
  note_fmax(m, fmax);
}

// fused path: the same (u, f') on a mirror-padded grid, rows = global rows
// [out_row0 - W, out_row0 + out_rows + W), columns = global [-W, cols + W)
// with cols = strips * TW, so every TMA tile of the fused kernel is in bounds.
// Grid: x = column blocks, y = (image, padded row) in a grid-stride loop (any
// height or batch: no 65535 limit), two columns per thread and one 16-byte
// store.  Same per-element arithmetic as the dense prep (bit-identical phases).
__global__ void prep_padded_kernel(const float* __restrict__ src, int2* __restrict__ uf, Geometry g, int W, int cols,
                                   double turns_scaled, float shift, unsigned* fmax) {
  const int pw = cols + 2 * W, ph = g.out_rows + 2 * W;
  const long long nrows = static_cast<long long>(ph) * g.batch;
  float m = 0.f;
  // kPrepRows padded rows per thread and pass, every load issued before the
  // first use (a pure streaming kernel: with one row in flight per thread it
  // ran at ~2 TB/s, c2 24.8 us)
  constexpr int kPrepRows = 4;
  for (long long r0 = blockIdx.y; r0 < nrows; r0 += static_cast<long long>(kPrepRows) * gridDim.y) {
    const float* srow[kPrepRows];
#pragma unroll
    for (int j = 0; j < kPrepRows; ++j) {
      const long long r = min(r0 + static_cast<long long>(j) * gridDim.y, nrows - 1);
      const int b = static_cast<int>(r / ph), py = static_cast<int>(r - static_cast<long long>(b) * ph);
      const int gy = mirror_index(g.out_row0 - W + py, g.full_height) - g.src_row0;
      srow[j] = src + b * g.src_bstride + static_cast<long long>(gy) * g.src_pitch;
    }
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; 2 * q < pw; q += gridDim.x * blockDim.x) {
      const int x0 = mirror_index(2 * q - W, g.width), x1 = mirror_index(2 * q + 1 - W, g.width);
      float f0[kPrepRows], f1[kPrepRows];
#pragma unroll
      for (int j = 0; j < kPrepRows; ++j) {
        f0[j] = __ldg(srow[j] + x0);
        f1[j] = __ldg(srow[j] + x1);
      }
#pragma unroll
      for (int j = 0; j < kPrepRows; ++j) {
        const long long r = r0 + static_cast<long long>(j) * gridDim.y;
        if (r >= nrows) break;
        const int2 a = phase_of(f0[j], turns_scaled, shift, m);
        const int2 c = phase_of(f1[j], turns_scaled, shift, m);
        reinterpret_cast<int4*>(uf + r * pw)[q] = make_int4(a.x, a.y, c.x, c.y);
      }
    }
  }
  note_fmax(m, fmax);
}

// ---------------------------------------------------------------------------
// Runtime-length taps (naive chain, standalone convolve): profile[0..2W] in the
// workspace, any radius.  Uploaded by kernel parameters, kTapChunk at a time
// (graph-capturable, no pageable copies).
constexpr int kTapChunk = 2048;
struct TapChunk {
  int off, n;
  double t[kTapChunk];
};
__global__ void store_taps(const __grid_constant__ TapChunk c, float* __restrict__ t32, double* __restrict__ t64) {
  for (int i = threadIdx.x; i < c.n; i += blockDim.x) {
    if (t32) t32[c.off + i] = static_cast<float>(c.t[i]);
    if (t64) t64[c.off + i] = c.t[i];
  }
}
cudaError_t upload_taps(const double* profile, int radius, float* t32, double* t64, cudaStream_t st) {
  TapChunk c;
  for (int off = 0; off < 2 * radius + 1; off += kTapChunk) {
    c.off = off;
    c.n = std::min(kTapChunk, 2 * radius + 1 - off);
    std::memcpy(c.t, profile + off, sizeof(double) * c.n);
    store_taps<<<1, 256, 0, st>>>(c, t32, t64);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// naive variant: per harmonic four kernels over HBM-resident float4 planes
//   modulate -> row FIR -> column FIR -> demodulate, then one divide kernel.
// out(i) = sum_j profile[j+W] in(i-j), ascending j (spatial.hpp:74-89).

struct NaiveArgs {
  Geometry g;  // uf / planes use a dense layout: batch x src_rows x width
  int W;
  const float* taps;  // profile[0..2W] (workspace)
};

__global__ void naive_modulate(const int2* __restrict__ uf, ulonglong2* __restrict__ M, long long total,
                               uint32_t n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int2 v = uf[i];
    float c, s;
    sincos_turns(n * static_cast<uint32_t>(v.x), c, s);
    const float fp = __int_as_float(v.y);
    M[i] = make_ulonglong2(pk(c, c * fp), pk(s, s * fp));
  }
}

__global__ void naive_rows(const ulonglong2* __restrict__ in, ulonglong2* __restrict__ out,
                           const __grid_constant__ NaiveArgs a) {
  const long long per = static_cast<long long>(a.g.src_rows) * a.g.width;
  const long long total = per * a.g.batch;
  const int W = a.W;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long rowbase = i - (i % a.g.width);
    const int x = static_cast<int>(i % a.g.width);
    p2 A = 0, B = 0;
    for (int j = -W; j <= W; ++j) {
      const ulonglong2 v = in[rowbase + mirror_index(x - j, a.g.width)];
      const float tv = a.taps[j + W];
      A = fma2(pk(tv, tv), v.x, A);
      B = fma2(pk(tv, tv), v.y, B);
    }
    out[i] = make_ulonglong2(A, B);
  }
}

__global__ void naive_cols(const ulonglong2* __restrict__ in, ulonglong2* __restrict__ out,
                           const __grid_constant__ NaiveArgs a) {
  const long long per_out = static_cast<long long>(a.g.out_rows) * a.g.width;
  const long long per_src = static_cast<long long>(a.g.src_rows) * a.g.width;
  const long long total = per_out * a.g.batch;
  const int W = a.W;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = i / per_out;
    const long long r = i - b * per_out;
    const int y = a.g.out_row0 + static_cast<int>(r / a.g.width);
    const int x = static_cast<int>(r % a.g.width);
    const ulonglong2* src = in + b * per_src;
    p2 A = 0, B = 0;
    for (int j = -W; j <= W; ++j) {
      const int sy = mirror_index(y - j, a.g.full_height) - a.g.src_row0;
      const ulonglong2 v = src[static_cast<long long>(sy) * a.g.width + x];
      const float tv = a.taps[j + W];
      A = fma2(pk(tv, tv), v.x, A);
      B = fma2(pk(tv, tv), v.y, B);
    }
    out[i] = make_ulonglong2(A, B);
  }
}

__global__ void naive_demod(const ulonglong2* __restrict__ M, const ulonglong2* __restrict__ C,
                            p2* __restrict__ pq, Geometry g, float dn, int first, int aq,
                            const unsigned* __restrict__ fmax) {
  const FixedScale fs = fixed_scale(aq, fmax);
  const p2 dd = pk(dn * fs.sq, dn * fs.sp);
  const long long per_out = static_cast<long long>(g.out_rows) * g.width;
  const long long per_src = static_cast<long long>(g.src_rows) * g.width;
  const long long total = per_out * g.batch;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = i / per_out;
    const long long r = i - b * per_out;
    const int y = g.out_row0 + static_cast<int>(r / g.width);
    const int x = static_cast<int>(r % g.width);
    const ulonglong2 m = M[b * per_src + static_cast<long long>(y - g.src_row0) * g.width + x];
    const ulonglong2 c = C[i];
    const float cc = lo_of(m.x), ss = lo_of(m.y);
    p2 qp = mul2(pk(cc, cc), c.x);  // (c Gc, c Fc) + (s Gs, s Fs)
    qp = fma2(pk(ss, ss), c.y, qp);
    const p2 t = to_fixed(mul2(dd, qp));  // fixed-point term (fbf_params.h)
    pq[i] = first ? t : iadd2(pq[i], t);
  }
}

// divide with the collapse check (bilateral.hpp:147-158); pq: fixed-point
// int32 pairs (fbf_params.h), or exact fp64 (Q, P) pairs (pq64: the summed
// output of fbf_partial_sums_device, fbf_finish_device)
__global__ void finish_kernel(const p2* __restrict__ pq, const double2* __restrict__ pq64, float* __restrict__ dst,
                              Geometry g, float shift, float q_floor, unsigned long long* bad, int aq,
                              const unsigned* __restrict__ fmax) {
  const FixedScale fs = fixed_scale(aq, fmax);
  const long long per_out = static_cast<long long>(g.out_rows) * g.width;
  const long long total = per_out * g.batch;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = i / per_out;
    const long long r = i - b * per_out;
    const int yl = static_cast<int>(r / g.width);
    const int x = static_cast<int>(r % g.width);
    float Q, P;
    if (pq64) {
      const double2 v = pq64[i];
      Q = static_cast<float>(v.x);
      P = static_cast<float>(v.y);
    } else {
      from_fixed(pq[i], fs, Q, P);
    }
    if (!(fabsf(Q) >= q_floor) && bad) {
      const unsigned long long lin = static_cast<unsigned long long>(b) * g.full_height * g.width +
                                     static_cast<unsigned long long>(g.out_row0 + yl) * g.width + x;
      atomicMin(bad, lin);
    }
    dst[b * g.dst_bstride + static_cast<long long>(yl) * g.dst_pitch + x] = shift + __fdiv_rn(P, Q);
  }
}

// Sums the nonempty groups' fixed-point planes (exact integer adds: the
// result does not depend on the group count) and divides, or writes the exact
// fp64 (Q, P) values (sum_out, fbf_partial_sums_device).
// A thread takes PX adjacent pixels (PX = 2: one 16-byte load per plane; the
// fused layout's even pitch) of kFinishRows consecutive rows, every load of
// every plane issued before the first use (the pass is pure memory traffic:
// one pixel per thread with 8-byte loads ran at ~1.5 TB/s, c2 with 2 groups
// 48 us; this form ~3x faster).  Grid: x = column blocks, y = row groups in a
// grid-stride loop.
constexpr int kFinishRows = 4;
constexpr int kFinishThreads = 128;
template <int PX>
__global__ void __launch_bounds__(kFinishThreads)
    finish_groups(const p2* __restrict__ pq, int groups, int span, long long plane, int pq_cols, Geometry g,
                  float shift, float q_floor, unsigned long long* bad, float* __restrict__ dst,
                  double2* __restrict__ sum_out, int aq, const unsigned* __restrict__ fmax) {
  const FixedScale fs = fixed_scale(aq, fmax);
  const long long nrows = static_cast<long long>(g.out_rows) * g.batch;
  unsigned live = 0;  // groups that hold at least one harmonic (the others' planes were never written)
  for (int k = 0; k < groups; ++k)
    if (span * (k + 1) / groups > span * k / groups) live |= 1u << k;
  for (long long row0 = static_cast<long long>(blockIdx.y) * kFinishRows; row0 < nrows;
       row0 += static_cast<long long>(gridDim.y) * kFinishRows) {
    for (int x = PX * (blockIdx.x * blockDim.x + threadIdx.x); x < g.width; x += PX * gridDim.x * blockDim.x) {
      p2 acc[kFinishRows][PX];
#pragma unroll
      for (int r = 0; r < kFinishRows; ++r)
#pragma unroll
        for (int j = 0; j < PX; ++j) acc[r][j] = 0ull;
      for (int k = 0; k < groups; ++k) {
        if (!((live >> k) & 1u)) continue;
        p2 v[kFinishRows][PX];
#pragma unroll
        for (int r = 0; r < kFinishRows; ++r) {
          const long long row = min(row0 + r, nrows - 1);
          const p2* src = pq + k * plane + row * pq_cols + x;
          if constexpr (PX == 2) {
            const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(src);
            v[r][0] = t.x;
            v[r][1] = t.y;
          } else {
            v[r][0] = *src;
          }
        }
#pragma unroll
        for (int r = 0; r < kFinishRows; ++r)
#pragma unroll
          for (int j = 0; j < PX; ++j) acc[r][j] = iadd2(acc[r][j], v[r][j]);
      }
#pragma unroll
      for (int r = 0; r < kFinishRows; ++r) {
        const long long row = row0 + r;
        if (row >= nrows) break;
        const int b = static_cast<int>(row / g.out_rows);
        const int yl = static_cast<int>(row - static_cast<long long>(b) * g.out_rows);
#pragma unroll
        for (int j = 0; j < PX; ++j) {
          if (x + j >= g.width) break;
          if (sum_out) {  // exact: int32 * 2^-a is representable in fp64
            float a, c;
            upk(acc[r][j], a, c);
            sum_out[row * g.width + x + j] = make_double2(static_cast<double>(__float_as_int(a)) * fs.iq,
                                                          static_cast<double>(__float_as_int(c)) * fs.ip);
            continue;
          }
          float Q, P;
          from_fixed(acc[r][j], fs, Q, P);
          if (!(fabsf(Q) >= q_floor) && bad) {
            const unsigned long long lin = static_cast<unsigned long long>(b) * g.full_height * g.width +
                                           static_cast<unsigned long long>(g.out_row0 + yl) * g.width + x + j;
            atomicMin(bad, lin);
          }
          dst[b * g.dst_bstride + static_cast<long long>(yl) * g.dst_pitch + x + j] = shift + __fdiv_rn(P, Q);
        }
      }
    }
  }
}
// pixel pairs where every plane row starts 16-byte aligned (the fused layout), else single pixels
void launch_finish_groups(cudaStream_t st, const p2* pq, int groups, int span, long long plane, int pq_cols,
                          const Geometry& g, float shift, float q_floor, unsigned long long* bad, float* dst,
                          double2* sum_out, int aq, const unsigned* fmax) {
  const long long nrows = static_cast<long long>(g.out_rows) * g.batch;
  const unsigned gy = static_cast<unsigned>(std::min((nrows + kFinishRows - 1) / kFinishRows, 65535LL));
  const bool pairs = pq_cols % 2 == 0 && plane % 2 == 0 && reinterpret_cast<uintptr_t>(pq) % 16 == 0;
  if (pairs) {
    const dim3 grid(static_cast<unsigned>((g.width + 2 * kFinishThreads - 1) / (2 * kFinishThreads)), gy, 1);
    finish_groups<2><<<grid, kFinishThreads, 0, st>>>(pq, groups, span, plane, pq_cols, g, shift, q_floor, bad, dst,
                                                      sum_out, aq, fmax);
  } else {
    const dim3 grid(static_cast<unsigned>((g.width + kFinishThreads - 1) / kFinishThreads), gy, 1);
    finish_groups<1><<<grid, kFinishThreads, 0, st>>>(pq, groups, span, plane, pq_cols, g, shift, q_floor, bad, dst,
                                                      sum_out, aq, fmax);
  }
}

// ---------------------------------------------------------------------------
// standalone separable convolution of one plane (convolve(), spatial.hpp:98-112):
// row pass then column pass, out(i) = sum_j profile[j+W] in(i-j) in ascending
// j.  fp64: separate multiply and add in the reference's order (its build
// does not contract them), so the result equals the reference bit for bit.

template <class T>
__device__ __forceinline__ T mac(T t, T v, T acc);
template <>
__device__ __forceinline__ float mac<float>(float t, float v, float acc) {
  return fmaf(t, v, acc);
}
template <>
__device__ __forceinline__ double mac<double>(double t, double v, double acc) {
  return __dadd_rn(acc, __dmul_rn(t, v));
}

template <class T>
__global__ void conv_rows(const T* __restrict__ in, T* __restrict__ out, int w, int h, int W,
                          const T* __restrict__ taps) {
  const long long total = static_cast<long long>(w) * h;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long rowbase = i - (i % w);
    const int x = static_cast<int>(i % w);
    T acc = 0;
    for (int j = -W; j <= W; ++j) acc = mac<T>(taps[j + W], in[rowbase + mirror_index(x - j, w)], acc);
    out[i] = acc;
  }
}

template <class T>
__global__ void conv_cols(const T* __restrict__ in, T* __restrict__ out, int w, int h, int W,
                          const T* __restrict__ taps) {
  const long long total = static_cast<long long>(w) * h;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(i / w);
    const int x = static_cast<int>(i % w);
    T acc = 0;
    for (int j = -W; j <= W; ++j)
      acc = mac<T>(taps[j + W], in[static_cast<long long>(mirror_index(y - j, h)) * w + x], acc);
    out[i] = acc;
  }
}

// ---------------------------------------------------------------------------
// FP32 FMA-pipe probe: 16 independent FFMA2 chains per thread.

__global__ void __launch_bounds__(256) fma_probe(float* out, float a, float b, int iters, long long* cycles) {
  p2 acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = pk(threadIdx.x * 1e-3f + i, static_cast<float>(i));
  const p2 ma = pk(a, a), mb = pk(b, b);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma2(acc[i], ma, mb);
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += lo_of(acc[i]) + hi_of(acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

unsigned grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  g = std::min<long long>(g, 148LL * 32);
  return static_cast<unsigned>(std::max<long long>(g, 1));
}

// ---------------------------------------------------------------------------
// host-side checks and parameter blocks

int check_geometry(const fbf_geometry* g) {
  if (!g) return fail(FBF_EINVAL, "bilateral_fast: null geometry");
  if (g->width <= 0 || g->height <= 0 || g->batch <= 0) return fail(FBF_EINVAL, "bilateral_fast: empty image");
  if (g->src_row0 < 0 || g->src_rows <= 0 || g->src_row0 + g->src_rows > g->height || g->out_row0 < 0 ||
      g->out_rows <= 0 || g->out_row0 + g->out_rows > g->height)
    return fail(FBF_EINVAL, "bilateral_fast: row range outside the image");
  return FBF_OK;
}

// spatial.hpp:102-104: the recursive backend replaces the FIR for Gaussian
// windows with sigma >= 2 only
bool uses_iir(const fbf_filter* f) { return f->kind == FBF_SPATIAL_GAUSSIAN && f->sigma_s >= 2.0; }

int check_filter(const fbf_filter* f) {
  if (!f || !f->profile || !f->d) return fail(FBF_EINVAL, "bilateral_fast: null filter");
  if (f->radius < 1 || f->radius > kMaxRadius)
    return fail(FBF_EINVAL, "bilateral_fast: spatial radius outside [1, " + std::to_string(kMaxRadius) + "]");
  if (f->N < 0 || f->N > kMaxN) return fail(FBF_EINVAL, "bilateral_fast: harmonic count outside [0, 65535]");
  if (f->check_epsilon && !(f->max_pointwise_error < f->w0))
    return fail(FBF_EINVAL,
                "bilateral_fast: kernel approximation error must stay below the center "
                "spatial weight");
  return FBF_OK;
}

// The fused kernel keeps one tap per |j| (a symmetric window, as both of
// make_spatial_gaussian / make_spatial_box produce); any other profile runs the
// naive chain with the full 2W+1 taps.
bool symmetric(const fbf_filter* f) {
  for (int j = 1; j <= f->radius; ++j)
    if (f->profile[f->radius + j] != f->profile[f->radius - j]) return false;
  return true;
}
bool fused_ok(const fbf_filter* f) {
  return f->radius <= kMaxWFused && fused_supported(f->radius, f->kind == FBF_SPATIAL_BOX) && symmetric(f);
}

// The source rows must cover every mirrored row that the output rows touch.
int check_halo(const fbf_geometry* g, int W) {
  int lo = g->height, hi = -1;
  auto visit = [&](int y) {
    for (int k = -W; k <= W; ++k) {
      const int s = mirror_index(y + k, g->height);
      lo = std::min(lo, s);
      hi = std::max(hi, s);
    }
  };
  const int a = g->out_row0, b = g->out_row0 + g->out_rows;
  for (int y = a; y < std::min(b, a + 2 * W + 1); ++y) visit(y);
  for (int y = std::max(a, b - 2 * W - 1); y < b; ++y) visit(y);
  if (lo < g->src_row0 || hi >= g->src_row0 + g->src_rows)
    return fail(FBF_EINVAL, "bilateral_fast: source strip lacks the W halo rows the output needs");
  return FBF_OK;
}

Geometry to_geometry(const fbf_geometry* g) {
  Geometry G{};
  G.width = g->width;
  G.full_height = g->height;
  G.src_row0 = g->src_row0;
  G.src_rows = g->src_rows;
  G.out_row0 = g->out_row0;
  G.out_rows = g->out_rows;
  G.batch = g->batch;
  G.src_bstride = g->src_bstride;
  G.src_pitch = static_cast<int>(g->src_pitch);
  G.dst_bstride = g->dst_bstride;
  G.dst_pitch = static_cast<int>(g->dst_pitch);
  return G;
}

void fill_taps(Taps& k, const fbf_filter* f) {
  std::memset(&k, 0, sizeof(k));
  k.W = f->radius;
  k.box = f->kind == FBF_SPATIAL_BOX;
  k.box_tap = static_cast<float>(f->profile[f->radius]);
  for (int j = 0; j <= std::min(f->radius, kMaxWFused); ++j) k.t[j] = static_cast<float>(f->profile[f->radius + j]);
}

// Q grid exponent of the fixed-point sums (fbf_params.h): the largest aq with
// 1.02 * D * 2^aq <= 2^31, D = sum over ALL harmonics of |d_n| (as fp32; box
// windows too: their weight (1/(2W+1))^2 < 1 only shrinks the terms).  A
// function of the filter alone, so every partition of a call agrees on it.
int fixed_q_exponent(const fbf_filter* f) {
  double D = 0.0;
  for (int n = 0; n <= f->N; ++n) D += std::fabs(static_cast<double>(static_cast<float>(f->d[n])));
  if (!(D > 0.0)) return 30;
  const int a = static_cast<int>(std::floor(std::log2(2147483648.0 / (1.02 * D))));
  return std::max(-60, std::min(40, a));
}

void fill_harmonics(Harmonics& h, const fbf_filter* f) {
  std::memset(&h, 0, sizeof(h));
  h.N = f->N;
  h.d_base = 0;
  for (int n = 0; n <= f->N && n < kMaxD; ++n) h.d[n] = static_cast<float>(f->d[n]);
  h.turns_per_unit = f->omega / (2.0 * M_PI);
  h.shift = 128.0f;
  h.q_floor = static_cast<float>((f->w0 - f->max_pointwise_error) / 2.0);
  h.aq = fixed_q_exponent(f);
}

// ---------------------------------------------------------------------------
// Harmonic split inside one GPU: the harmonics are divided among CTA groups,
// each accumulating its own fixed-point (Q, P) plane, summed exactly at the
// end (finish_groups).  Each group's CTAs get work units with `groups` times
// more rows and 1/groups of the harmonics: fewer per-harmonic 2W-row unit
// prologues and a finer step granularity (a CTA's rows per harmonic are a
// whole number of G-row steps: c2 with one group runs 16 steps on its busiest
// CTAs against a mean of 15.1, with two groups 30 against 29.2), against the
// extra planes and the finish pass.  Since the sums are integers, any count
// gives the same bits; the count is purely a speed choice.
//
// Cost model (microseconds): for k groups the fused kernel's duration is
// ceil(H / k) harmonics x the busiest CTA's steps per harmonic x the step
// time.  The busiest CTA comes from replaying the kernel's own cuts
// (fused_kernel: cost-balanced ranges in (strip, row) space, KC-aligned, units
// capped at seg_max) on the launch plan of this geometry (launch_fused in
// plan mode); a unit's prologue steps count 0.8 of a full step (c2: one group
// 995 us, two groups 946 us, i.e. 15.6 against 29.6 / 2 steps per harmonic).
// Step time: per pixel and harmonic on one SM, linear in the taps (fitted to
// c5 / c2 / c4 at W = 12 / 15 / 24).  With groups the n = 0 kernel runs last, in
// finish mode, and reads the k planes (8 k bytes per pixel at ~4 TB/s; c2,
// k = 2: 42 us against 28 us for the plain n = 0 plane pass).  Measured:
// profiles/r02_notes.md (groups).
constexpr double kModelPrologueStep = 0.8;
struct GroupCosts {
  double per_harmonic[kMaxGroups + 1] = {};  // [k]: busiest CTA's time for one harmonic, us
  double finish[kMaxGroups + 1] = {};        // [k]: the finish pass, us
  bool ok = false;
};

double busiest_cta_steps(const FusedPlan& p, const fbf_geometry* g) {
  const long long strips = (g->width + p.tw - 1) / p.tw;
  const long long out_rows = g->out_rows;
  const long long total = static_cast<long long>(g->batch) * strips * out_rows;
  const long long per = out_rows + p.unit_cost;
  const long long ctotal = total / out_rows * per;
  auto split = [&](long long pos) {
    const long long sidx = pos / out_rows;
    const long long r = pos - sidx * out_rows;
    return sidx * out_rows + (r - r % p.kc);
  };
  auto cut = [&](long long k) {
    const long long t = ctotal * k / p.grid;
    const long long sidx = t / per;
    return split(sidx * out_rows + std::min(t - sidx * per, out_rows));
  };
  double worst = 0.0;
  long long lo = 0;
  for (int b = 0; b < p.grid; ++b) {
    const long long hi = b + 1 == p.grid ? total : cut(b + 1);
    double steps = 0.0;
    for (long long pos = lo; pos < hi;) {
      const long long sidx = pos / out_rows;
      const long long r0 = pos - sidx * out_rows;
      const long long len = std::min({out_rows - r0, hi - pos, static_cast<long long>(p.seg_max)});
      steps += kModelPrologueStep * p.prologue + static_cast<double>((len + p.G - 1) / p.G);
      pos += len;
    }
    worst = std::max(worst, steps);
    lo = hi;
  }
  return worst;
}

GroupCosts group_costs_of(const fbf_geometry* g, int radius, bool box) {
  GroupCosts c;
  if (!fused_supported(radius, box)) return c;
  FusedArgs A;
  std::memset(&A, 0, sizeof(A));
  A.g = to_geometry(g);
  A.k.W = radius;
  A.k.box = box;
  A.seg_max = 1 << 30;
  const double px = static_cast<double>(g->batch) * g->out_rows * g->width;
  for (int k = 1; k <= kMaxGroups; ++k) {
    A.groups = k;
    FusedPlan p{};
    if (launch_fused(A, nullptr, &p) != cudaSuccess || p.grid < 1) return c;  // no device: one group
    const int conc = std::max(1, std::min(p.occ, (p.grid * k + p.sms - 1) / p.sms));  // CTAs sharing an SM
    double t_px = box ? 0.70e-3 * (kFusedTW + 2.0 * radius) / 74.0
                      : (0.86 + 0.0757 * (2.0 * radius + 1.0)) / 2048.0;  // us per pixel and harmonic on one SM
    if (p.nt <= 128 && p.occ == 1) t_px *= 1.5;                           // the large-W 128-thread tile alone on its SM
    c.per_harmonic[k] = busiest_cta_steps(p, g) * conc * p.G * p.tw * t_px;
    c.finish[k] = k > 1 ? 2.0 + px * 8.0 * k / 4.0e6 : 0.0;  // the n = 0 kernel in finish mode reads k planes more
  }
  c.ok = true;
  return c;
}

// the group count for H harmonics in the fused kernel (n = 0 is not one of them)
int pick_groups(const GroupCosts& c, int H) {
  if (!c.ok || H < 2) return 1;
  const double margin = FBF_TUNABLE(GROUP_MARGIN, kGroupMargin);
  int groups = 1;
  double best = H * c.per_harmonic[1];
  for (int k = 2; k <= std::min(kMaxGroups, H); ++k) {
    const double t = ((H + k - 1) / k) * c.per_harmonic[k] + c.finish[k];
    if (t < margin * best) best = t, groups = k;
  }
#ifdef FBF_EXPERIMENTS
  if (const char* e = getenv("FBF_GROUPS")) groups = std::max(1, std::min({kMaxGroups, H, atoi(e)}));
#endif
  return groups;
}

// per thread: the costs of the last few geometries (the host pipeline cycles
// through a handful of chunk shapes) and the most planes any harmonic count
// picks for them -- the (Q, P) planes the workspace holds
struct GroupMemo {
  int out_rows = -1, width = -1, batch = -1, radius = -1, dev = -1;
  GroupCosts gauss, boxc;
  int cap = 1;
};
const GroupMemo& group_memo(const fbf_geometry* g, int radius) {
  constexpr int kSlots = 8;
  thread_local GroupMemo memo[kSlots];
  thread_local int next = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  for (const GroupMemo& m : memo)
    if (m.out_rows == g->out_rows && m.width == g->width && m.batch == g->batch && m.radius == radius && m.dev == dev)
      return m;
  GroupMemo& m = memo[next];
  next = (next + 1) % kSlots;
  m = GroupMemo{};
  m.out_rows = g->out_rows, m.width = g->width, m.batch = g->batch, m.radius = radius, m.dev = dev;
  m.gauss = group_costs_of(g, radius, false);
  m.boxc = group_costs_of(g, radius, true);
  for (int H = 2; H <= kMaxD && m.cap < kMaxGroups; ++H)
    m.cap = std::max({m.cap, pick_groups(m.gauss, H), pick_groups(m.boxc, H)});
#ifdef FBF_EXPERIMENTS
  if (getenv("FBF_GROUPS")) m.cap = kMaxGroups;
#endif
  return m;
}

int group_cap(const fbf_geometry* g, int radius) { return group_memo(g, radius).cap; }

// groups for a fused run over `harmonics` harmonics n >= 1
int harmonic_groups(const fbf_geometry* g, int radius, bool box, int harmonics) {
  const GroupMemo& m = group_memo(g, radius);
  return std::min(pick_groups(box ? m.boxc : m.gauss, std::min(harmonics, kMaxD)), m.cap);
}

struct Layout {
  size_t hdr, uf, pq, taps, m, t, c, total;  // hdr: 256-byte header, word 0 = max |f'| bits (prep)
};

// Fused: mirror-padded (u, f') image (out_rows + 2W) x (strips*TW + 2W) and
// group_cap fixed-point (Q, P) planes out_rows x strips*TW per image.  Naive:
// dense (u, f') of the source rows, (Q, P) per output pixel, the taps and
// three float4 planes.
Layout layout_of(const fbf_geometry* g, int radius, int variant) {
  Layout L{};
  const size_t src_px = static_cast<size_t>(g->batch) * g->src_rows * g->width;
  const size_t out_px = static_cast<size_t>(g->batch) * g->out_rows * g->width;
  L.hdr = 0;
  L.uf = 256;
  if (variant == FBF_VARIANT_FUSED) {
    const size_t cols = static_cast<size_t>((g->width + kFusedTW - 1) / kFusedTW) * kFusedTW;
    const size_t uf_px = static_cast<size_t>(g->batch) * (g->out_rows + 2 * radius) * (cols + 2 * radius);
    L.pq = L.uf + align256(uf_px * sizeof(int2));
    L.total = L.pq + align256(static_cast<size_t>(group_cap(g, radius)) * g->batch * g->out_rows * cols * sizeof(Pair));
    return L;
  }
  L.pq = L.uf + align256(src_px * sizeof(int2));
  L.taps = L.pq + align256(out_px * sizeof(Pair));
  L.m = L.taps + align256((2 * static_cast<size_t>(radius) + 1) * sizeof(float));
  L.t = L.m + align256(src_px * sizeof(float4));
  L.c = L.t + align256(src_px * sizeof(float4));
  L.total = L.c + align256(out_px * sizeof(float4));
  return L;
}

struct Prepared {
  Geometry G, Gd;
  Harmonics H;
  Taps K;
  int variant;
  int2* uf;
  Pair* pq;
  unsigned* fmax;
  char* ws;
  Layout L;
};

int prepare_common(const fbf_geometry* gp, const fbf_filter* f, void* workspace, size_t workspace_bytes, int variant,
                   Prepared& P) {
  int rc = check_geometry(gp);
  if (rc) return rc;
  if ((rc = check_filter(f))) return rc;
  if ((rc = check_halo(gp, f->radius))) return rc;
  if (variant == FBF_VARIANT_RECURSIVE) {
    if (uses_iir(f))
      return fail(FBF_EUNSUPPORTED,
                  "bilateral_fast: the recursive backend runs through fbf_bilateral_fast_device / _host only");
    variant = FBF_VARIANT_FUSED;  // spatial.hpp:102-104: box windows and sigma < 2 stay direct
  }
  if (variant == FBF_VARIANT_FUSED && !fused_ok(f)) variant = FBF_VARIANT_NAIVE;
  P.L = layout_of(gp, f->radius, variant);
  if (!workspace || workspace_bytes < P.L.total)
    return fail(FBF_EINVAL, variant == FBF_VARIANT_NAIVE
                                ? "bilateral_fast: workspace too small for the naive path (no fused "
                                  "kernel for this window)"
                                : "bilateral_fast: workspace too small");
  P.variant = variant;
  P.ws = static_cast<char*>(workspace);
  P.fmax = reinterpret_cast<unsigned*>(P.ws + P.L.hdr);
  P.uf = reinterpret_cast<int2*>(P.ws + P.L.uf);
  P.pq = reinterpret_cast<Pair*>(P.ws + P.L.pq);
  P.G = to_geometry(gp);
  fill_harmonics(P.H, f);
  fill_taps(P.K, f);
  P.Gd = P.G;  // dense view of the prep output: batch x src_rows x width
  P.Gd.src_pitch = P.G.width;
  P.Gd.src_bstride = static_cast<long long>(P.G.src_rows) * P.G.width;
  return FBF_OK;
}

// The n = 0 term of the fused path as its own single-plane filter.  At n = 0
// the modulation is exact (c = 1, s = 0), so the harmonic's four planes reduce
// to one: (q, p) = (conv(1), conv(f')) = (1, conv(f')) -- taps sum to one and
// mirror padding keeps it so (bilateral.hpp:126-144 with n = 0).  Filtering
// it inside the fused kernel would cost a full harmonic (four planes, halo
// modulation, demodulation); here it is one separable FIR of f' read from the
// padded (u, f') image, rounded to the same fixed-point grid as every other
// term and written as group plane 0, onto which the fused kernel's group 0
// accumulates harmonics 1..N.  The fixed-point sum is exact, so where the
// n = 0 term is computed does not change the result's bits.
//
// Tile: 64 output columns x 32 output rows per CTA, 256 threads; smem holds the
// (32+2W) x (64+2W) input tile and the row-filtered (32+2W) x 64 tile.
// (kernel: n0_plane_kernel in fbf_fused.cuh, one instance per radius)
cudaError_t launch_n0_plane(const FusedArgs& a_in, cudaStream_t st) {
  FusedArgs a = a_in;
  a.n0_only = 1;
  return launch_fused(a, st, nullptr);
}

// Fused launches over harmonics [n_lo, n_hi): one launch when the range fits
// the kMaxD coefficients of a parameter block (the common case, N < 256),
// otherwise consecutive launches of kMaxD harmonics that keep accumulating
// into the (Q, P) planes, the last one dividing unless `partial`.  Returns
// the number of (Q, P) group planes left for finish_groups (1: none needed).
int launch_fused_range(const FusedArgs& base, const fbf_filter* f, int n_lo, int n_hi, int groups, bool partial,
                       cudaStream_t st, cudaError_t* err, bool* divided = nullptr) {
  if (divided) *divided = false;
  FusedArgs A = base;
  // n = 0 as a single-plane filter (n0_plane_kernel) into group plane 0; the
  // fused kernel then starts at n = 1 with group 0 accumulating onto it
  // (always, so the n = 0 term has the same bits in every harmonic partition)
  // With harmonic groups (>= 2, a filtering call, one launch) the n = 0 kernel
  // runs LAST instead, in finish mode: it adds its term to the groups' planes
  // and divides, replacing the n = 0 plane pass and finish_groups (c2: 28 + 25
  // us -> one ~35 us pass).
  const bool n0_finishes = n_lo == 0 && !partial && divided && n_hi - 1 <= kMaxD && std::min(groups, n_hi - 1) >= 2;
  if (n_lo == 0 && !n0_finishes) {
    A.h.d[0] = static_cast<float>(f->d[0]);
    *err = launch_n0_plane(A, st);
    if (*err != cudaSuccess) return 0;
    n_lo = 1;
    A.acc_group0 = 1;
    if (n_hi == 1) return 1;  // N = 0: plane 0 holds the sums; the caller divides
  }
  if (n0_finishes) n_lo = 1;
  const bool one = n_hi - n_lo <= kMaxD;
  A.groups = one ? std::max(1, std::min(groups, n_hi - n_lo)) : 1;
  for (int c0 = n_lo; c0 < n_hi; c0 += kMaxD) {
    const int c1 = std::min(n_hi, c0 + kMaxD);
    A.n_lo = c0;
    A.n_hi = c1;
    A.h.d_base = c0;
    for (int n = c0; n < c1; ++n) A.h.d[n - c0] = static_cast<float>(f->d[n]);
    A.accumulate = c0 > n_lo;
    A.partial = partial || A.groups > 1 || c1 < n_hi;
    *err = launch_fused(A, st, nullptr);
    if (*err != cudaSuccess) return 0;
  }
  if (n0_finishes) {
    FusedArgs F = A;  // groups, planes, dst, bad as the fused launch saw them
    F.h = base.h;
    F.h.d[0] = static_cast<float>(f->d[0]);
    F.n0_only = 2;
    *err = launch_fused(F, st, nullptr);
    if (*err != cudaSuccess) return 0;
    *divided = true;
    return A.groups;
  }
  if (divided) *divided = !A.partial;
  return A.groups;
}

FusedArgs fused_args(const Prepared& P, float* dst, unsigned long long* d_bad) {
  FusedArgs A;
  std::memset(&A, 0, sizeof(A));
  A.g = P.Gd;
  A.h = P.H;
  A.k = P.K;
  A.uf = P.uf;
  A.dst = dst;
  A.pq = P.pq;
  A.fmax = P.fmax;
  A.bad = d_bad;
  A.seg_max = 1 << 30;
  return A;
}

// the naive chain over harmonics [n_lo, n_hi) into the fixed-point (Q, P) plane
int naive_range(const Prepared& P, const fbf_filter* f, int n_lo, int n_hi, cudaStream_t st) {
  ulonglong2* M = reinterpret_cast<ulonglong2*>(P.ws + P.L.m);
  ulonglong2* T = reinterpret_cast<ulonglong2*>(P.ws + P.L.t);
  ulonglong2* C = reinterpret_cast<ulonglong2*>(P.ws + P.L.c);
  NaiveArgs NA;
  NA.g = P.Gd;
  NA.W = f->radius;
  NA.taps = reinterpret_cast<const float*>(P.ws + P.L.taps);
  const long long src_px = static_cast<long long>(P.G.batch) * P.G.src_rows * P.G.width;
  const long long out_px = static_cast<long long>(P.G.batch) * P.G.out_rows * P.G.width;
  for (int n = n_lo; n < n_hi; ++n) {
    naive_modulate<<<grid_for(src_px, 256), 256, 0, st>>>(P.uf, M, src_px, static_cast<uint32_t>(n));
    naive_rows<<<grid_for(src_px, 256), 256, 0, st>>>(M, T, NA);
    naive_cols<<<grid_for(out_px, 256), 256, 0, st>>>(T, C, NA);
    naive_demod<<<grid_for(out_px, 256), 256, 0, st>>>(M, C, reinterpret_cast<p2*>(P.pq), P.Gd,
                                                       static_cast<float>(f->d[n]), n == n_lo, P.H.aq, P.fmax);
  }
  FBF_CUDA(cudaGetLastError());
  return FBF_OK;
}

template <class T>
int convolve_any(int width, int height, const double* profile, int radius, const T* src, T* dst, void* workspace,
                 size_t workspace_bytes, cudaStream_t st) {
  if (width <= 0 || height <= 0) return fail(FBF_EINVAL, "convolve: empty plane");
  if (radius < 0 || radius > kMaxRadius || !profile) return fail(FBF_EINVAL, "convolve: invalid spatial kernel");
  const size_t n = static_cast<size_t>(width) * height;
  const size_t need = align256(n * sizeof(T)) + align256((2 * static_cast<size_t>(radius) + 1) * sizeof(T));
  if (!workspace || workspace_bytes < need) return fail(FBF_EINVAL, "convolve: workspace too small");
  T* tmp = static_cast<T*>(workspace);
  T* taps = reinterpret_cast<T*>(static_cast<char*>(workspace) + align256(n * sizeof(T)));
  if constexpr (sizeof(T) == 4) {
    FBF_CUDA(upload_taps(profile, radius, reinterpret_cast<float*>(taps), nullptr, st));
  } else {
    FBF_CUDA(upload_taps(profile, radius, nullptr, reinterpret_cast<double*>(taps), st));
  }
  conv_rows<T><<<grid_for(n, 256), 256, 0, st>>>(src, tmp, width, height, radius, taps);
  conv_cols<T><<<grid_for(n, 256), 256, 0, st>>>(tmp, dst, width, height, radius, taps);
  FBF_CUDA(cudaGetLastError());
  return FBF_OK;
}

}  // namespace

namespace fbf {
// internal API for the host path (fbf_hostpath.cu)
size_t workspace_for(const fbf_geometry* g, const fbf_filter* f, int variant) {
  if (variant == FBF_VARIANT_RECURSIVE) {
    if (uses_iir(f)) return iir_workspace_bytes(g, f->radius);
    variant = FBF_VARIANT_FUSED;
  }
  if (variant == FBF_VARIANT_FUSED && !fused_ok(f)) variant = FBF_VARIANT_NAIVE;
  return layout_of(g, f->radius, variant).total;
}
int check_call(const fbf_geometry* g, const fbf_filter* f) {
  int rc = check_geometry(g);
  if (rc == FBF_OK) rc = check_filter(f);
  if (rc == FBF_OK) rc = check_halo(g, f->radius);
  return rc;
}
bool recursive_applies(const fbf_filter* f) { return uses_iir(f); }
bool fused_applies(const fbf_filter* f) { return fused_ok(f); }
}  // namespace fbf

extern "C" {

const char* fbf_last_error(void) { return g_err.c_str(); }
int fbf_version(void) { return 2; }

void fbf_geometry_whole(fbf_geometry* g, int width, int height, int batch) {
  g->width = width;
  g->height = height;
  g->batch = batch;
  g->src_row0 = 0;
  g->src_rows = height;
  g->out_row0 = 0;
  g->out_rows = height;
  g->src_pitch = width;
  g->dst_pitch = width;
  g->src_bstride = static_cast<long long>(width) * height;
  g->dst_bstride = static_cast<long long>(width) * height;
}

size_t fbf_workspace_bytes(const fbf_geometry* g, int radius, int variant) {
  if (check_geometry(g) != FBF_OK || radius < 1 || radius > kMaxRadius) return 0;
  if (variant == FBF_VARIANT_RECURSIVE)  // the IIR path, or the direct path it falls back to
    return std::max(iir_workspace_bytes(g, radius), fbf_workspace_bytes(g, radius, FBF_VARIANT_FUSED));
  if (variant == FBF_VARIANT_FUSED) {
    const bool g_ok = radius <= kMaxWFused && fused_supported(radius, false);
    const bool b_ok = radius <= kMaxWFused && fused_supported(radius, true);
    if (!g_ok && !b_ok) variant = FBF_VARIANT_NAIVE;
    // the window kind is not known here: cover both paths when they differ
    if (g_ok != b_ok)
      return std::max(layout_of(g, radius, FBF_VARIANT_FUSED).total, layout_of(g, radius, FBF_VARIANT_NAIVE).total);
  }
  return layout_of(g, radius, variant).total;
}

int fbf_prepare_device(const fbf_geometry* gp, const fbf_filter* f, const float* src, void* workspace,
                       size_t workspace_bytes, int variant, void* stream) {
  Prepared P;
  int rc = prepare_common(gp, f, workspace, workspace_bytes, variant, P);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const double scale = P.H.turns_per_unit * 4294967296.0;
  FBF_CUDA(cudaMemsetAsync(P.fmax, 0, sizeof(unsigned), st));
  if (P.variant == FBF_VARIANT_FUSED) {
    const int W = f->radius;
    const int cols = (P.G.width + kFusedTW - 1) / kFusedTW * kFusedTW;
    const int pairs = (cols + 2 * W) / 2;  // cols is a multiple of 64: even row length
    const long long rows = static_cast<long long>(P.G.out_rows + 2 * W) * P.G.batch;
    // a few waves of CTAs in a grid-stride loop over rows (one fmax atomic per CTA)
    const unsigned bx = static_cast<unsigned>((pairs + 127) / 128);
    const long long by = std::max(1LL, std::min(rows, (148LL * 16 + bx - 1) / bx));
    const dim3 grid(bx, static_cast<unsigned>(by), 1);
    prep_padded_kernel<<<grid, 128, 0, st>>>(src, P.uf, P.G, W, cols, scale, P.H.shift, P.fmax);
  } else {
    const long long src_px = static_cast<long long>(P.G.batch) * P.G.src_rows * P.G.width;
    prep_kernel<<<grid_for(src_px, 256), 256, 0, st>>>(src, P.uf, P.G, scale, P.H.shift, P.fmax);
    FBF_CUDA(upload_taps(f->profile, f->radius, reinterpret_cast<float*>(P.ws + P.L.taps), nullptr, st));
  }
  FBF_CUDA(cudaGetLastError());
  return FBF_OK;
}

int fbf_filter_prepared_device(const fbf_geometry* gp, const fbf_filter* f, float* dst, void* workspace,
                               size_t workspace_bytes, unsigned long long* d_bad, int variant, void* stream) {
  Prepared P;
  int rc = prepare_common(gp, f, workspace, workspace_bytes, variant, P);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (P.variant == FBF_VARIANT_FUSED) {
    const FusedArgs A = fused_args(P, dst, d_bad);
    cudaError_t e = cudaSuccess;
    bool divided = false;
    const int groups =
        launch_fused_range(A, f, 0, P.H.N + 1, harmonic_groups(gp, f->radius, f->kind == FBF_SPATIAL_BOX, P.H.N), false, st, &e,
                           &divided);
    FBF_CUDA(e);
    if (!divided) {
      const int cols = (P.G.width + kFusedTW - 1) / kFusedTW * kFusedTW;
      const long long plane = static_cast<long long>(P.G.batch) * P.G.out_rows * cols;
      launch_finish_groups(st, reinterpret_cast<const p2*>(P.pq), groups, P.H.N + 1, plane, cols, P.G, P.H.shift,
                           P.H.q_floor, d_bad, dst, nullptr, P.H.aq, P.fmax);
      FBF_CUDA(cudaGetLastError());
    }
    return FBF_OK;
  }
  if ((rc = naive_range(P, f, 0, P.H.N + 1, st))) return rc;
  const long long out_px = static_cast<long long>(P.G.batch) * P.G.out_rows * P.G.width;
  finish_kernel<<<grid_for(out_px, 256), 256, 0, st>>>(reinterpret_cast<p2*>(P.pq), nullptr, dst, P.G, P.H.shift,
                                                       P.H.q_floor, d_bad, P.H.aq, P.fmax);
  FBF_CUDA(cudaGetLastError());
  return FBF_OK;
}

int fbf_bilateral_fast_device(const fbf_geometry* gp, const fbf_filter* f, const float* src, float* dst,
                              void* workspace, size_t workspace_bytes, unsigned long long* d_bad, int variant,
                              void* stream) {
  if (variant == FBF_VARIANT_RECURSIVE) {
    int rc = check_geometry(gp);
    if (rc) return rc;
    if ((rc = check_filter(f))) return rc;
    if (uses_iir(f))
      return iir_bilateral<float, float>(gp, f, src, dst, workspace, workspace_bytes, d_bad,
                                         static_cast<cudaStream_t>(stream));
    variant = FBF_VARIANT_FUSED;
  }
  int rc = fbf_prepare_device(gp, f, src, workspace, workspace_bytes, variant, stream);
  if (rc) return rc;
  return fbf_filter_prepared_device(gp, f, dst, workspace, workspace_bytes, d_bad, variant, stream);
}

int fbf_partial_sums_device(const fbf_geometry* gp, const fbf_filter* f, int n_lo, int n_hi, double* pq_out,
                            void* workspace, size_t workspace_bytes, int variant, void* stream) {
  Prepared P;
  int rc = prepare_common(gp, f, workspace, workspace_bytes, variant, P);
  if (rc) return rc;
  if (n_lo < 0 || n_hi > P.H.N + 1 || n_lo >= n_hi || !pq_out)
    return fail(FBF_EINVAL, "partial_sums: harmonic range outside [0, N]");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int groups = 1, span = n_hi - n_lo;
  long long plane = 0;
  int cols = P.G.width;
  if (P.variant == FBF_VARIANT_FUSED) {
    const FusedArgs A = fused_args(P, nullptr, nullptr);
    cudaError_t e = cudaSuccess;
    groups = launch_fused_range(A, f, n_lo, n_hi,
                                harmonic_groups(gp, f->radius, f->kind == FBF_SPATIAL_BOX, n_hi - std::max(n_lo, 1)), true,
                                st, &e);
    FBF_CUDA(e);
    cols = (P.G.width + kFusedTW - 1) / kFusedTW * kFusedTW;
    plane = static_cast<long long>(P.G.batch) * P.G.out_rows * cols;
  } else {
    if ((rc = naive_range(P, f, n_lo, n_hi, st))) return rc;
    span = 1;
  }
  launch_finish_groups(st, reinterpret_cast<const p2*>(P.pq), groups, span, plane, cols, P.G, 0.f, 0.f, nullptr,
                       nullptr, reinterpret_cast<double2*>(pq_out), P.H.aq, P.fmax);
  FBF_CUDA(cudaGetLastError());
  return FBF_OK;
}

int fbf_finish_device(const fbf_geometry* gp, const fbf_filter* f, const double* pq, float* dst,
                      unsigned long long* d_bad, void* stream) {
  int rc = check_geometry(gp);
  if (rc) return rc;
  if ((rc = check_filter(f))) return rc;
  Harmonics H;
  fill_harmonics(H, f);
  const Geometry G = to_geometry(gp);
  const long long out_px = static_cast<long long>(G.batch) * G.out_rows * G.width;
  finish_kernel<<<grid_for(out_px, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      nullptr, reinterpret_cast<const double2*>(pq), dst, G, H.shift, H.q_floor, d_bad, H.aq, nullptr);
  FBF_CUDA(cudaGetLastError());
  return FBF_OK;
}

int fbf_harmonic_groups(const fbf_geometry* g, int radius, int N) {
  if (!g || check_geometry(g) != FBF_OK || N < 0) return 0;
  return N < 1 ? 1 : std::min(harmonic_groups(g, radius, false, N), N);  // Gaussian windows (the kind is not part of this query)
}

int fbf_launches_per_call(const fbf_geometry* g, const fbf_filter* f, int variant) {
  if (!f || !g) return 0;
  if (variant == FBF_VARIANT_RECURSIVE) {
    if (uses_iir(f)) return g->batch * (6 * (f->N + 1) + 1);  // per harmonic: modulate, 2 IIR, 2 transposes, demod
    variant = FBF_VARIANT_FUSED;
  }
  if (variant == FBF_VARIANT_FUSED && fused_ok(f)) {
    // prep, the n = 0 kernel (plane before, or finish mode after), fused launches of <= kMaxD harmonics
    if (f->N == 0) return 3;  // prep, n = 0 plane, divide
    const int chunks = (f->N - 1 + kMaxD) / kMaxD;
    if (chunks > 1) return 2 + chunks;
    return 3;  // one group: prep, n = 0 plane, fused (divides); groups: prep, fused, n = 0 kernel in finish mode
  }
  const int tap_uploads = (2 * f->radius + 1 + kTapChunk - 1) / kTapChunk;
  return 1 + tap_uploads + 4 * (f->N + 1) + 1;
}

size_t fbf_convolve_workspace_bytes(int width, int height, int radius) {
  if (width <= 0 || height <= 0 || radius < 0) return 0;
  return align256(static_cast<size_t>(width) * height * sizeof(double)) +
         align256((2 * static_cast<size_t>(radius) + 1) * sizeof(double));
}

int fbf_convolve_device(int width, int height, const double* profile, int radius, const float* src, float* dst,
                        void* workspace, size_t workspace_bytes, void* stream) {
  return convolve_any<float>(width, height, profile, radius, src, dst, workspace, workspace_bytes,
                             static_cast<cudaStream_t>(stream));
}

int fbf_convolve_device_f64(int width, int height, const double* profile, int radius, const double* src,
                            double* dst, void* workspace, size_t workspace_bytes, void* stream) {
  return convolve_any<double>(width, height, profile, radius, src, dst, workspace, workspace_bytes,
                              static_cast<cudaStream_t>(stream));
}

int fbf_probe_fma_peak(double* ops_per_s, double* sm_mhz, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  FBF_CUDA(cudaGetDevice(&dev));
  FBF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks = sms * 4, threads = 256, iters = 40000;
  float* out = nullptr;
  long long* cyc = nullptr;
  FBF_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out), blocks * threads * sizeof(float), st));
  FBF_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cyc), blocks * sizeof(long long), st));
  fma_probe<<<blocks, threads, 0, st>>>(out, 1.0001f, 0.5f, 200, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  fma_probe<<<blocks, threads, 0, st>>>(out, 1.0001f, 0.5f, iters, cyc);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> h(blocks);
  cudaMemcpyAsync(h.data(), cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  long long mx = 0;
  for (int i = 0; i < blocks; ++i) mx = std::max(mx, h[i]);
  cudaFreeAsync(out, st);
  cudaFreeAsync(cyc, st);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  FBF_CUDA(cudaStreamSynchronize(st));
  const double ops = static_cast<double>(blocks) * threads * iters * 16.0;
  if (ops_per_s) *ops_per_s = ops / (ms * 1e-3);
  if (sm_mhz) *sm_mhz = static_cast<double>(mx) / (ms * 1e3);
  return FBF_OK;
}

}  // extern "C"
