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
//       S1  (u, f') rows of this step are in smem (cp.async, issued one step ahead)
//       (1) modulate   G x (TW+2W) pixels -> smem M: pairs (c, f'c), (s, f's),
//                      c + i s = e^{i n omega f'} from the exact phase n*u
//       S2  -> issue cp.async for the next step's (u, f') rows and this step's
//              running (Q, P) values
//       (2) row pass   G rows x TW outputs (KR per thread, FFMA2) -> smem ring R
//                      + the centre (c, s) of each input row      -> smem ring CS
//       S3
//       (3) column pass G output rows (KC per thread, FFMA2) from the ring,
//           demodulate, accumulate (Q, P) of this harmonic; at n = N divide.
//
// Every input row is row-passed once per harmonic (no vertical-halo recompute
// except 2W rows per work unit), each halo pixel is modulated once per
// harmonic, the ring holds 2W+G rows, and global traffic (L2-resident for
// the most part) is the (u, f') image plus the running (Q, P) per pixel.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "fbf_device.cuh"
#include "fbf_params.h"

namespace fbf {

// BOX: uniform window -> O(1) running sums (2 adds per output per pass in the
// steady state) instead of the (2W+1)-tap FIR; the 1/(2W+1)^2 weight is applied
// once, in the demodulation.
template <int W_, int TW_, int G_, int KR_, int KC_, int NT_, bool BOX_ = false>
struct FusedCfg {
  static constexpr int W = W_, TW = TW_, G = G_, KR = KR_, KC = KC_, NT = NT_;
  static constexpr bool BOX = BOX_;
  static constexpr int MW = TW + 2 * W;   // modulated row width
  static constexpr int MP = MW | 1;       // M pitch in 16-byte units (odd: conflict-free column walks)
  static constexpr int RING = 2 * W + G;  // R ring rows
  static constexpr int CRING = W + G;     // CS ring rows
  static constexpr int RP = TW + 1;       // R pitch in 16-byte units
  static constexpr int CP = TW + 1;       // CS pitch in 8-byte units
  static constexpr int PROLOGUE = (2 * W + G - 1) / G;  // steps that only row-pass
  // smem carve-up (bytes; TMA destinations 128-byte aligned)
  static constexpr size_t up128(size_t v) { return (v + 127) & ~size_t(127); }
  static constexpr size_t OFF_STAGE = 0;
  static constexpr size_t OFF_PQ = up128(OFF_STAGE + size_t(G) * MW * 8);
  static constexpr size_t OFF_M = up128(OFF_PQ + size_t(G) * TW * 8);
  static constexpr size_t OFF_R = OFF_M + size_t(G) * MP * 16;
  static constexpr size_t OFF_CS = OFF_R + size_t(RING) * RP * 16;
  static constexpr size_t OFF_BAR = up128(OFF_CS + size_t(CRING) * CP * 8);
  static constexpr size_t smem_bytes = OFF_BAR + 16;
  static_assert(G * (TW / KR) == NT, "row pass: one (row, chunk) item per thread");
  static_assert((G / KC) * TW == NT, "column pass: one (column, run) item per thread");
  static_assert(TW % KR == 0 && G % KC == 0, "tiling");
  static_assert(smem_bytes <= 227 * 1024, "shared memory budget");
};

// Geometry of one work unit and the rows of step s (same for every harmonic).
struct Unit {
  int b, x0, y0, y1;
};

template <class C>
__device__ __forceinline__ void step_rows(const Unit& u, int s, int& a, int& rows, int& o) {
  if (s < C::PROLOGUE) {  // input rows [y0 - W, y0 + W)
    a = u.y0 - C::W + s * C::G;
    rows = min(C::G, u.y0 + C::W - a);
    o = -1;
  } else {
    o = u.y0 + (s - C::PROLOGUE) * C::G;
    a = o + C::W;
    rows = min(C::G, u.y1 + C::W - a);
  }
}

// Warp-row mapping shared by the prefetch and the modulation: warp w owns the
// step rows g = w, w + NWARP, ...; lane l owns the columns j = l + 32 i of a
// row.  The mirrored global column of each owned j is computed once per work
// unit (colofs), so the per-element cost is an add and the copy itself.
template <class C>
struct Lanes {
  static constexpr int NWARP = C::NT / 32;
  static constexpr int RPW = C::G / NWARP;      // rows per warp per step
  static constexpr int NJ = (C::MW + 31) / 32;  // column slots per lane
  static_assert(C::G % NWARP == 0, "rows per warp");
};

// TMA loads of one step: the padded (u, f') rows [a, a+G) x columns
// [x0-W, x0+TW+W) into stage, and the running (Q, P) of output rows [o, o+G)
// into pqs.  Issued by thread 0 only; rows past the image are zero-filled
// and never consumed.
template <class C>
__device__ __forceinline__ void tma_uf(const FusedArgs& A, int2* stage, uint64_t* bar, const Unit& u,
                                       int a) {
  mbar_expect_tx(bar, static_cast<unsigned>(C::G * C::MW * 8));
  tma_load_3d(stage, &A.tm_uf, bar, u.x0, a - A.g.out_row0 + C::W, u.b);
}
template <class C>
__device__ __forceinline__ void tma_pq(const FusedArgs& A, p2* pqs, uint64_t* bar, const Unit& u, int o) {
  mbar_expect_tx(bar, static_cast<unsigned>(C::G * C::TW * 8));
  tma_load_3d(pqs, &A.tm_pq, bar, u.x0, o - A.g.out_row0, static_cast<int>(blockIdx.y) * A.g.batch + u.b);
}

// Modulation of one step, sliced into RPW*NJ independent elements per thread.
// Straight-line code: every slot is computed (clamped reads) and only the
// stores are predicated, so the element chains interleave freely with other
// work in the same basic block (rows past the step's end hold finite stale
// data and are never consumed).
template <class C>
struct ModNext {
  static constexpr int ELEMS = Lanes<C>::RPW * Lanes<C>::NJ;
  const int2* stage;
  ulonglong2* M;
  uint32_t n;

  // k must be a constant after unrolling (all callers sit in unrolled loops)
  __device__ __forceinline__ void element(int k) const {
    using L = Lanes<C>;
    const int r = k / L::NJ, i = k % L::NJ;
    const bool full = (C::MW % 32 == 0) || (i + 1 < L::NJ);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = warp + r * L::NWARP;
    const int j = lane + 32 * i;
    const int jc = full ? j : min(j, C::MW - 1);
    const int2 v = stage[g * C::MW + jc];
    float c, s;
    sincos_turns(n * static_cast<uint32_t>(v.x), c, s);
    const float fp = __int_as_float(v.y);
    const ulonglong2 m = make_ulonglong2(pk(c, c * fp), pk(s, s * fp));
    if (full || j < C::MW) M[g * C::MP + j] = m;
  }
};

template <class C>
__device__ __forceinline__ void modulate_rows(const int2* __restrict__ stage, ulonglong2* __restrict__ M,
                                              int rows, uint32_t n) {
  (void)rows;
  const ModNext<C> job{stage, M, n};
#pragma unroll
  for (int k = 0; k < ModNext<C>::ELEMS; ++k) job.element(k);
}

template <class C>
__device__ __forceinline__ void row_pass(const FusedArgs& A, const ulonglong2* __restrict__ M,
                                         ulonglong2* __restrict__ R, p2* __restrict__ CS, int a,
                                         int rows, int base) {
  const int g = threadIdx.x % C::G;
  const int xc = (threadIdx.x / C::G) * C::KR;
  if (g >= rows) return;
  const ulonglong2* __restrict__ src = M + g * C::MP + xc;
  const int rel = a + g - base;
  const int slot = rel % C::RING;
  const int cslot = rel % C::CRING;
  p2 accA[C::KR], accB[C::KR];
  if constexpr (C::BOX) {
    // running sum over the window [i, i+2W] (unweighted)
    p2 sA = 0ull, sB = 0ull;
#pragma unroll
    for (int m = 0; m <= 2 * C::W; ++m) {
      const ulonglong2 v = src[m];
      sA = add2(sA, v.x);
      sB = add2(sB, v.y);
      if (m >= C::W && m < C::W + C::KR) CS[cslot * C::CP + xc + (m - C::W)] = pk(lo_of(v.x), lo_of(v.y));
    }
    accA[0] = sA;
    accB[0] = sB;
#pragma unroll
    for (int i = 1; i < C::KR; ++i) {
      const ulonglong2 vin = src[i + 2 * C::W], vout = src[i - 1];
      sA = sub2(add2(sA, vin.x), vout.x);
      sB = sub2(add2(sB, vin.y), vout.y);
      accA[i] = sA;
      accB[i] = sB;
      if (i + 2 * C::W >= C::W && i + 2 * C::W < C::W + C::KR)
        CS[cslot * C::CP + xc + (i + C::W)] = pk(lo_of(vin.x), lo_of(vin.y));
    }
  } else {
#pragma unroll
    for (int i = 0; i < C::KR; ++i) accA[i] = accB[i] = 0ull;
#pragma unroll
    for (int m = 0; m < C::KR + 2 * C::W; ++m) {
      const ulonglong2 v = src[m];
#pragma unroll
      for (int i = 0; i < C::KR; ++i) {
        const int j = m - i;
        if (j >= 0 && j <= 2 * C::W) {
          const float tv = A.k.t[j < C::W ? C::W - j : j - C::W];
          accA[i] = fma2(pk(tv, tv), v.x, accA[i]);
          accB[i] = fma2(pk(tv, tv), v.y, accB[i]);
        }
      }
      if (m >= C::W && m < C::W + C::KR)  // centre (c, s) of output column xc + m - W
        CS[cslot * C::CP + xc + (m - C::W)] = pk(lo_of(v.x), lo_of(v.y));
    }
  }
  ulonglong2* __restrict__ dst = R + slot * C::RP + xc;
#pragma unroll
  for (int i = 0; i < C::KR; ++i) dst[i] = make_ulonglong2(accA[i], accB[i]);
}

template <class C>
__device__ __forceinline__ void col_pass(const FusedArgs& A, const ulonglong2* __restrict__ R,
                                         const p2* __restrict__ CS, const p2* __restrict__ pqs,
                                         const Unit& u, int o, int base, int n, bool first, bool divide,
                                         const ModNext<C>& next) {
  const int x = threadIdx.x % C::TW;
  const int gi = (threadIdx.x / C::TW) * C::KC;  // first output row of this thread, rel. to o
  const int r0 = o + gi;
  const int gx = u.x0 + x;
  const int nr = min(C::KC, u.y1 - r0);  // <= 0: this thread only helps with the modulation
  p2 accA[C::KC], accB[C::KC];
  const int s0 = (r0 - C::W - base) % C::RING;
  constexpr int TAPS_IN = C::KC + 2 * C::W;
  constexpr int ELEMS = ModNext<C>::ELEMS;
  constexpr int STRIDE = TAPS_IN / ELEMS > 0 ? TAPS_IN / ELEMS : 1;
  auto ring = [&](int m) {
    int s = s0 + m;
    s = s >= C::RING ? s - C::RING : s;
    return R[s * C::RP + x];
  };
  if constexpr (C::BOX) {
    p2 sA = 0ull, sB = 0ull;
#pragma unroll
    for (int m = 0; m <= 2 * C::W; ++m) {
      const ulonglong2 v = ring(m);
      sA = add2(sA, v.x);
      sB = add2(sB, v.y);
      if (m % STRIDE == 0 && m / STRIDE < ELEMS) next.element(m / STRIDE);
    }
    accA[0] = sA;
    accB[0] = sB;
#pragma unroll
    for (int i = 1; i < C::KC; ++i) {
      const ulonglong2 vin = ring(i + 2 * C::W), vout = ring(i - 1);
      sA = sub2(add2(sA, vin.x), vout.x);
      sB = sub2(add2(sB, vin.y), vout.y);
      accA[i] = sA;
      accB[i] = sB;
      const int m = i + 2 * C::W;
      if (m % STRIDE == 0 && m / STRIDE < ELEMS) next.element(m / STRIDE);
    }
  } else {
#pragma unroll
    for (int i = 0; i < C::KC; ++i) accA[i] = accB[i] = 0ull;
#pragma unroll
    for (int m = 0; m < TAPS_IN; ++m) {
      const ulonglong2 v = ring(m);
#pragma unroll
      for (int i = 0; i < C::KC; ++i) {
        const int j = m - i;
        if (j >= 0 && j <= 2 * C::W) {
          const float tv = A.k.t[j < C::W ? C::W - j : j - C::W];
          accA[i] = fma2(pk(tv, tv), v.x, accA[i]);
          accB[i] = fma2(pk(tv, tv), v.y, accB[i]);
        }
      }
      // one slice of the next step's modulation per STRIDE taps
      if (m % STRIDE == 0 && m / STRIDE < ELEMS) next.element(m / STRIDE);
    }
  }
#pragma unroll
  for (int k = TAPS_IN / STRIDE + (TAPS_IN % STRIDE ? 1 : 0); k < ELEMS; ++k) next.element(k);
  if (nr <= 0 || gx >= A.g.width) return;
  // box: both passes summed unweighted; the weight (1/(2W+1))^2 = w0 joins d_n here
  const float dn = C::BOX ? A.h.d[n] * (A.k.box_tap * A.k.box_tap) : A.h.d[n];
  const p2 dd = pk(dn, dn);
  const int cs0 = (r0 - base) % C::CRING;
  p2* __restrict__ pqrow = reinterpret_cast<p2*>(A.pq) +
                           ((blockIdx.y * A.g.batch + u.b) * static_cast<long long>(A.g.out_rows) +
                            (r0 - A.g.out_row0)) * A.pq_cols + gx;
  const int wstride = A.pq_cols;
  // demodulate all KC outputs straight-line; only the global stores are predicated
  p2 qp[C::KC];
#pragma unroll
  for (int i = 0; i < C::KC; ++i) {
    int sc = cs0 + i;
    sc = sc >= C::CRING ? sc - C::CRING : sc;
    float c, s;
    upk(CS[sc * C::CP + x], c, s);
    // (q, p) = c (Gc, Fc) + s (Gs, Fs)   [bilateral.hpp:138-144, real form]
    qp[i] = fma2(pk(s, s), accB[i], mul2(pk(c, c), accA[i]));
  }
  if (!divide) {
    if (first) {
#pragma unroll
      for (int i = 0; i < C::KC; ++i)
        if (i < nr) pqrow[i * wstride] = mul2(dd, qp[i]);
    } else {
#pragma unroll
      for (int i = 0; i < C::KC; ++i)
        if (i < nr) pqrow[i * wstride] = fma2(dd, qp[i], pqs[(gi + i) * C::TW + x]);
    }
    return;
  }
  // bilateral.hpp:147-158: divide; flag the first collapsed denominator
  float* __restrict__ drow = A.dst + u.b * A.g.dst_bstride +
                             static_cast<long long>(r0 - A.g.out_row0) * A.g.dst_pitch + gx;
#pragma unroll
  for (int i = 0; i < C::KC; ++i) {
    if (i < nr) {
      const p2 acc = first ? mul2(dd, qp[i]) : fma2(dd, qp[i], pqs[(gi + i) * C::TW + x]);
      float Q, P;
      upk(acc, Q, P);
      if (!(fabsf(Q) >= A.h.q_floor) && A.bad) {
        const unsigned long long lin =
            static_cast<unsigned long long>(u.b) * A.g.full_height * A.g.width +
            static_cast<unsigned long long>(r0 + i) * A.g.width + gx;
        atomicMin(A.bad, lin);
      }
      drow[i * static_cast<long long>(A.g.dst_pitch)] = A.h.shift + __fdiv_rn(P, Q);
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::NT, (C::NT <= 128 ? 2 : 1)) fused_kernel(const __grid_constant__ FusedArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  int2* stage = reinterpret_cast<int2*>(smem + C::OFF_STAGE);
  ulonglong2* M = reinterpret_cast<ulonglong2*>(smem + C::OFF_M);
  ulonglong2* R = reinterpret_cast<ulonglong2*>(smem + C::OFF_R);
  p2* CS = reinterpret_cast<p2*>(smem + C::OFF_CS);
  p2* pqs = reinterpret_cast<p2*>(smem + C::OFF_PQ);
  uint64_t* bar_uf = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* bar_pq = bar_uf + 1;
  const bool leader = threadIdx.x == 0;
  if (leader) {
    mbar_init(bar_uf, 1);
    mbar_init(bar_pq, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned ph_uf = 0, ph_pq = 0;  // phase parity of the next completion of each barrier
  // this CTA group's harmonics [nb, ne)
  const int span = A.n_hi - A.n_lo;
  const int nb = A.n_lo + span * static_cast<int>(blockIdx.y) / A.groups;
  const int ne = A.n_lo + span * static_cast<int>(blockIdx.y + 1) / A.groups;
  if (nb >= ne) return;

  const long long total = A.total;
  // CTA ranges in (strip, row) space, with the row rounded down to a multiple
  // of KC: every column-pass block then starts at the same row offset whatever
  // the partition (the box path's running sums are order-sensitive), so the
  // result is bit-identical across CTA counts and multi-GPU strip splits.
  auto split = [&](long long p) {
    const long long sidx = p / A.g.out_rows;
    const long long r = p - sidx * A.g.out_rows;
    return sidx * A.g.out_rows + (r - r % C::KC);
  };
  const long long lo = blockIdx.x == 0 ? 0 : split(total * blockIdx.x / gridDim.x);
  const long long hi = blockIdx.x + 1 == gridDim.x ? total : split(total * (blockIdx.x + 1) / gridDim.x);
  for (long long pos = lo; pos < hi;) {
    const long long sidx = pos / A.g.out_rows;
    const int r0 = static_cast<int>(pos - sidx * A.g.out_rows);
    const int len = static_cast<int>(min(min(static_cast<long long>(A.g.out_rows - r0), hi - pos),
                                         static_cast<long long>(A.seg_max)));
    Unit u;
    u.b = static_cast<int>(sidx / A.strips);
    u.x0 = static_cast<int>(sidx - static_cast<long long>(u.b) * A.strips) * C::TW;
    u.y0 = A.g.out_row0 + r0;
    u.y1 = u.y0 + len;
    const int base = u.y0 - C::W;
    const int nsteps = C::PROLOGUE + (len + C::G - 1) / C::G;

    {  // bootstrap: step 0 of the group's first harmonic into M
      int a, rows, o;
      step_rows<C>(u, 0, a, rows, o);
      __syncthreads();  // the previous unit finished reading stage and M
      if (leader) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_uf<C>(A, stage, bar_uf, u, a);
      }
      mbar_wait(bar_uf, ph_uf);
      ph_uf ^= 1u;
      modulate_rows<C>(stage, M, rows, static_cast<uint32_t>(nb));
    }
    for (int n = nb; n < ne; ++n) {
      const bool first = n == nb;
      const bool divide = n + 1 == ne && !A.partial;
      for (int s = 0; s < nsteps; ++s) {
        int a, rows, o, a2, rows2, o2;
        step_rows<C>(u, s, a, rows, o);
        const bool wrap = s + 1 == nsteps;  // next step is step 0 of harmonic n+1
        const bool more = !wrap || n + 1 < ne;
        const bool want_pq = o >= 0 && !first;
        step_rows<C>(u, wrap ? 0 : s + 1, a2, rows2, o2);
        __syncthreads();  // S1: M holds this step; the previous column pass is done; stage free
        if (leader) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (more) tma_uf<C>(A, stage, bar_uf, u, a2);
          if (want_pq) tma_pq<C>(A, pqs, bar_pq, u, o);
        }
        row_pass<C>(A, M, R, CS, a, rows, base);
        if (more) {
          mbar_wait(bar_uf, ph_uf);
          ph_uf ^= 1u;
        }
        if (want_pq) {
          mbar_wait(bar_pq, ph_pq);
          ph_pq ^= 1u;
        }
        __syncthreads();  // S2: ring rows visible, next (u, f') and this step's (Q, P) landed, M free
        // the next step's modulation is interleaved into this step's column pass
        // (its ALU work issues in the FFMA2 shadow); prologue steps run it alone
        const ModNext<C> next{stage, M, static_cast<uint32_t>(wrap ? n + 1 : n)};
        if (o >= 0)
          col_pass<C>(A, R, CS, pqs, u, o, base, n, first, divide, next);
        else
          modulate_rows<C>(stage, M, rows2, next.n);
      }
    }
    pos += len;
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
inline cudaError_t encode_tile_3d(CUtensorMap* m, const void* base, unsigned long long d0,
                                  unsigned long long d1, unsigned long long d2, unsigned b0, unsigned b1) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Fn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) return cudaErrorNotSupported;
    fn = reinterpret_cast<Fn>(p);
  }
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {d0 * 8, d0 * d1 * 8};
  const cuuint32_t box[3] = {b0, b1, 1};
  const cuuint32_t estride[3] = {1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, const_cast<void*>(base), dims, strides, box,
                        estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <class C>
cudaError_t launch_cfg(const FusedArgs& a_in, cudaStream_t st, int* grid_out) {
  constexpr int W = C::W;
  static_assert(C::TW == kFusedTW, "workspace layout assumes kFusedTW-wide strips");
  FusedArgs a = a_in;
  a.strips = (a.g.width + C::TW - 1) / C::TW;
  a.pq_cols = a.strips * C::TW;
  a.total = static_cast<long long>(a.g.batch) * a.strips * a.g.out_rows;
  cudaError_t e = encode_tile_3d(&a.tm_uf, a.uf, static_cast<unsigned long long>(a.pq_cols + 2 * W),
                                 static_cast<unsigned long long>(a.g.out_rows + 2 * W),
                                 static_cast<unsigned long long>(a.g.batch), C::MW, C::G);
  if (e != cudaSuccess) return e;
  if (a.groups < 1) a.groups = 1;
  e = encode_tile_3d(&a.tm_pq, a.pq, static_cast<unsigned long long>(a.pq_cols),
                     static_cast<unsigned long long>(a.g.out_rows),
                     static_cast<unsigned long long>(a.g.batch) * a.groups, C::TW, C::G);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(fused_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(C::smem_bytes));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fused_kernel<C>, C::NT, C::smem_bytes);
  if (occ < 1) occ = 1;
  // one wave in total: the harmonic groups share the SMs
  long long grid = (static_cast<long long>(sms) * occ + a.groups - 1) / a.groups;
  // keep at least ~2W+G rows per CTA so the per-unit prologue stays amortised
  const long long min_rows = 2 * C::W + C::G;
  const long long by_work = (a.total + min_rows - 1) / min_rows;
  if (grid > by_work) grid = by_work;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = static_cast<int>(grid);
  fused_kernel<C><<<dim3(static_cast<unsigned>(grid), static_cast<unsigned>(a.groups)), C::NT, C::smem_bytes, st>>>(a);
  return cudaGetLastError();
}

// Small (128 threads, G=16, two CTAs per SM) for W <= 9, big (256 threads,
// G=32, one CTA per SM) otherwise -- measured, profiles/r01_cfg_compare.txt.
// FBF_FUSED_CFG=small|big overrides where both fit (experiments).
template <int W, bool BOX = false>
cudaError_t launch_w(const FusedArgs& a, cudaStream_t st, int* grid_out) {
  using Small = FusedCfg<W, 64, 16, 8, 8, 128, BOX>;
  using Big = FusedCfg<W, 64, 32, 8, 8, 256, BOX>;
  if constexpr (Small::smem_bytes <= 113 * 1024) {
    const char* env = getenv("FBF_FUSED_CFG");
    const bool big = env ? env[0] == 'b' : !(W <= 9);
    if (!big) return launch_cfg<Small>(a, st, grid_out);
  }
  return launch_cfg<Big>(a, st, grid_out);
}

}  // namespace fbf

#define FBF_INSTANTIATE_FUSED(WW) \
  template cudaError_t fbf::launch_w<WW, false>(const fbf::FusedArgs&, cudaStream_t, int*);
#define FBF_INSTANTIATE_FUSED_BOX(WW) \
  template cudaError_t fbf::launch_w<WW, true>(const fbf::FusedArgs&, cudaStream_t, int*);
