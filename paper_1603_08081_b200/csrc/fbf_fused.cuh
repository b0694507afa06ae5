// fbf_fused.cuh -- the fused sm_100a kernel for bilateral_fast
// (reference: /root/reference/proj/include/fourierbf/bilateral.hpp:109-160,
//  convolve spatial.hpp:74-112, mirror_index image.hpp:34-40).
//
// Design: column-strip streaming with the harmonic
// loop outermost inside a work unit.
//
//   work unit = one image, one TW-wide column strip, a run of output rows [y0,y1)
//   for n = 0..N:
//     stream input rows y0-W .. y1+W-1 in steps of G rows:
//       (1) modulate   G x (TW+2W) pixels -> smem M:  (c, f'c, s, f's), c+is = e^{i n w f'}
//       (2) row pass   G rows x TW outputs (KR per thread, FFMA2)  -> smem ring R
//                      + the centre (c, s) of each output column     -> smem ring CS
//       (3) column pass G output rows (KC per thread, FFMA2) from the ring,
//           demodulate and accumulate (Q, P) of this harmonic into a
//           workspace that stays L2-resident across n; at n = N divide.
//
// Every input row is row-passed once per harmonic (no vertical-halo recompute
// except 2W rows per work unit), each halo pixel is modulated once, the ring
// only holds 2W+G rows, and the only HBM traffic besides the (Q,P) workspace
// is the (u, f') image.  The harmonic phase is the exact uint32 product n*u.
#pragma once
#include <cuda_runtime.h>

#include "fbf_device.cuh"
#include "fbf_params.h"

namespace fbf {

template <int W_, int TW_, int G_, int KR_, int KC_, int NT_>
struct FusedCfg {
  static constexpr int W = W_, TW = TW_, G = G_, KR = KR_, KC = KC_, NT = NT_;
  static constexpr int MW = TW + 2 * W;   // modulated row width
  static constexpr int MP = MW | 1;       // M pitch in float4 (odd: conflict-free column walks)
  static constexpr int RING = 2 * W + G;  // ring rows
  static constexpr int RP = TW + 1;       // R pitch in float4
  static constexpr int CP = TW + 1;       // CS pitch in float2
  static constexpr size_t smem_bytes =
      size_t(G) * MP * 16 + size_t(RING) * RP * 16 + size_t(RING) * CP * 8;
  static_assert(G * (TW / KR) == NT, "row pass: one (row, chunk) item per thread");
  static_assert((G / KC) * TW == NT, "column pass: one (column, run) item per thread");
  static_assert(TW % KR == 0 && G % KC == 0, "tiling");
};

template <class C>
__device__ __forceinline__ void modulate_rows(const FusedArgs& A, float4* __restrict__ M, int b,
                                              int x0, int a, int rows, uint32_t n) {
  const int tid = threadIdx.x;
  const int2* __restrict__ uf = A.uf + b * A.g.src_bstride;
  const int total = rows * C::MW;
  constexpr int ITER = (C::G * C::MW + C::NT - 1) / C::NT;
#pragma unroll
  for (int k = 0; k < ITER; ++k) {
    const int e = tid + k * C::NT;
    if (e < total) {
      const int g = e / C::MW;
      const int j = e - g * C::MW;
      const int gy = mirror_index(a + g, A.g.full_height) - A.g.src_row0;
      const int gx = mirror_index(x0 - C::W + j, A.g.width);
      const int2 v = __ldg(uf + static_cast<long long>(gy) * A.g.src_pitch + gx);
      float c, s;
      sincos_turns(n * static_cast<uint32_t>(v.x), c, s);
      const float fp = __int_as_float(v.y);
      M[g * C::MP + j] = make_float4(c, c * fp, s, s * fp);
    }
  }
}

template <class C>
__device__ __forceinline__ void row_pass(const FusedArgs& A, const float4* __restrict__ M,
                                         float4* __restrict__ R, f2* __restrict__ CS, int a,
                                         int rows, int base) {
  const int tid = threadIdx.x;
  const int g = tid % C::G;
  const int xc = (tid / C::G) * C::KR;
  if (g >= rows) return;
  const float4* __restrict__ src = M + g * C::MP + xc;
  const int slot = (a + g - base) % C::RING;
  f2 accA[C::KR], accB[C::KR];
#pragma unroll
  for (int i = 0; i < C::KR; ++i) accA[i] = accB[i] = f2{0.f, 0.f};
#pragma unroll
  for (int m = 0; m < C::KR + 2 * C::W; ++m) {
    const float4 v = src[m];
    const f2 va{v.x, v.y}, vb{v.z, v.w};
#pragma unroll
    for (int i = 0; i < C::KR; ++i) {
      const int j = m - i;
      if (j >= 0 && j <= 2 * C::W) {
        const int tj = j < C::W ? C::W - j : j - C::W;
        const float tv = A.k.t[tj];
        const f2 t{tv, tv};
        ffma2(accA[i], t, va);
        ffma2(accB[i], t, vb);
      }
    }
    if (m >= C::W && m < C::W + C::KR) CS[slot * C::CP + xc + (m - C::W)] = f2{v.x, v.z};
  }
  float4* __restrict__ dst = R + slot * C::RP + xc;
#pragma unroll
  for (int i = 0; i < C::KR; ++i) dst[i] = make_float4(accA[i].x, accA[i].y, accB[i].x, accB[i].y);
}

template <class C>
__device__ __forceinline__ void col_pass(const FusedArgs& A, const float4* __restrict__ R,
                                         const f2* __restrict__ CS, int b, int x0, int o, int y1,
                                         int base, int n) {
  const int tid = threadIdx.x;
  const int x = tid % C::TW;
  const int r0 = o + (tid / C::TW) * C::KC;  // first output row of this thread
  if (r0 >= y1) return;
  const int gx = x0 + x;
  const bool xin = gx < A.g.width;
  const int nr = min(C::KC, y1 - r0);
  Pair* __restrict__ pq = A.pq + b * static_cast<long long>(A.g.out_rows) * A.g.width;
  // prefetch the running (Q, P) of this thread's outputs; latency hides under the FIR
  Pair prev[C::KC];
  if (n > 0 && xin) {
#pragma unroll
    for (int i = 0; i < C::KC; ++i)
      if (i < nr) {
        const long long idx = static_cast<long long>(r0 + i - A.g.out_row0) * A.g.width + gx;
        prev[i] = pq[idx];
      }
  }
  f2 accA[C::KC], accB[C::KC];
#pragma unroll
  for (int i = 0; i < C::KC; ++i) accA[i] = accB[i] = f2{0.f, 0.f};
  const int s0 = (r0 - C::W - base) % C::RING;
#pragma unroll
  for (int m = 0; m < C::KC + 2 * C::W; ++m) {
    int s = s0 + m;
    s = s >= C::RING ? s - C::RING : s;
    s = s >= C::RING ? s - C::RING : s;
    const float4 v = R[s * C::RP + x];
    const f2 va{v.x, v.y}, vb{v.z, v.w};
#pragma unroll
    for (int i = 0; i < C::KC; ++i) {
      const int j = m - i;
      if (j >= 0 && j <= 2 * C::W) {
        const int tj = j < C::W ? C::W - j : j - C::W;
        const float tv = A.k.t[tj];
        const f2 t{tv, tv};
        ffma2(accA[i], t, va);
        ffma2(accB[i], t, vb);
      }
    }
  }
  if (!xin) return;
  const float dn = A.h.d[n];
  const bool last = (n == A.h.N);
#pragma unroll
  for (int i = 0; i < C::KC; ++i) {
    if (i >= nr) break;
    const int y = r0 + i;
    int sc = s0 + C::W + i;
    sc = sc >= C::RING ? sc - C::RING : sc;
    sc = sc >= C::RING ? sc - C::RING : sc;
    const f2 cs = CS[sc * C::CP + x];
    // (q, p) = c*(Gc, Fc) + s*(Gs, Fs)   [bilateral.hpp:138-144, real form]
    f2 qp = mul2(f2{cs.x, cs.x}, accA[i]);
    qp = fma2(f2{cs.y, cs.y}, accB[i], qp);
    f2 acc;
    if (n == 0) {
      acc = mul2(f2{dn, dn}, qp);
    } else {
      acc = fma2(f2{dn, dn}, qp, f2{prev[i].x, prev[i].y});
    }
    const long long idx = static_cast<long long>(y - A.g.out_row0) * A.g.width + gx;
    if (!last) {
      pq[idx] = Pair{acc.x, acc.y};
    } else {
      // bilateral.hpp:147-158: divide; flag the first collapsed denominator
      const float Q = acc.x, P = acc.y;
      if (!(fabsf(Q) >= A.h.q_floor)) {
        const unsigned long long lin =
            static_cast<unsigned long long>(b) * A.g.full_height * A.g.width +
            static_cast<unsigned long long>(y) * A.g.width + gx;
        atomicMin(A.bad, lin);
      }
      A.dst[b * A.g.dst_bstride + static_cast<long long>(y - A.g.out_row0) * A.g.dst_pitch + gx] =
          A.h.shift + __fdiv_rn(P, Q);
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::NT, 1) fused_kernel(const __grid_constant__ FusedArgs A) {
  extern __shared__ float4 smem[];
  float4* M = smem;
  float4* R = M + C::G * C::MP;
  f2* CS = reinterpret_cast<f2*>(R + C::RING * C::RP);

  const long long total = A.total;
  const long long lo = total * blockIdx.x / gridDim.x;
  const long long hi = total * (blockIdx.x + 1) / gridDim.x;
  for (long long pos = lo; pos < hi;) {
    const long long sidx = pos / A.g.out_rows;
    const int r0 = static_cast<int>(pos - sidx * A.g.out_rows);
    const int len = static_cast<int>(min(min(static_cast<long long>(A.g.out_rows - r0), hi - pos),
                                         static_cast<long long>(A.seg_max)));
    const int b = static_cast<int>(sidx / A.strips);
    const int x0 = static_cast<int>(sidx - static_cast<long long>(b) * A.strips) * C::TW;
    const int y0 = A.g.out_row0 + r0, y1 = y0 + len;
    const int base = y0 - C::W;
    for (int n = 0; n <= A.h.N; ++n) {
      // prologue: the 2W input rows above the first output row
      for (int a = y0 - C::W; a < y0 + C::W; a += C::G) {
        const int rows = min(C::G, y0 + C::W - a);
        modulate_rows<C>(A, M, b, x0, a, rows, static_cast<uint32_t>(n));
        __syncthreads();
        row_pass<C>(A, M, R, CS, a, rows, base);
        __syncthreads();
      }
      for (int o = y0; o < y1; o += C::G) {
        const int a = o + C::W;
        const int rows = min(C::G, y1 + C::W - a);
        modulate_rows<C>(A, M, b, x0, a, rows, static_cast<uint32_t>(n));
        __syncthreads();
        row_pass<C>(A, M, R, CS, a, rows, base);
        __syncthreads();
        col_pass<C>(A, R, CS, b, x0, o, y1, base, n);
      }
      __syncthreads();
    }
    pos += len;
  }
}

// Per-radius launch configuration (TW=64 columns per strip, G=32 rows per step,
// 8 outputs per thread in both passes, 256 threads).
template <int W>
using Cfg = FusedCfg<W, 64, 32, 8, 8, 256>;

template <int W>
cudaError_t launch_w(const FusedArgs& a_in, cudaStream_t st, int* grid_out) {
  using C = Cfg<W>;
  FusedArgs a = a_in;
  a.strips = (a.g.width + C::TW - 1) / C::TW;
  a.total = static_cast<long long>(a.g.batch) * a.strips * a.g.out_rows;
  static bool configured = false;  // benign race: idempotent attribute set
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(fused_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::smem_bytes));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fused_kernel<C>, C::NT, C::smem_bytes);
  if (occ < 1) occ = 1;
  long long grid = static_cast<long long>(sms) * occ;
  // keep at least ~2W+G rows per CTA so the per-unit prologue stays amortised
  const long long min_rows = 2 * C::W + C::G;
  const long long by_work = (a.total + min_rows - 1) / min_rows;
  if (grid > by_work) grid = by_work;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = static_cast<int>(grid);
  fused_kernel<C><<<static_cast<unsigned>(grid), C::NT, C::smem_bytes, st>>>(a);
  return cudaGetLastError();
}

}  // namespace fbf

#define FBF_INSTANTIATE_FUSED(WW) \
  template cudaError_t fbf::launch_w<WW>(const fbf::FusedArgs&, cudaStream_t, int*);
