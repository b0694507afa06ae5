// fbf_fused2.cuh -- the fused kernel's step loop without a CTA-wide barrier
// (reference: bilateral.hpp:109-160, convolve spatial.hpp:74-112).
//
// Same work unit, lane mappings, FIR passes and arithmetic as fbf_fused.cuh
// (so the results are the same bits), different schedule:
//
//   * the next step's modulation runs inside THIS step's row pass, from (u, f')
//     values every thread loaded into registers (LDG, L2) one phase earlier --
//     no staging tile, no TMA issue on anyone's critical path;
//   * so the modulated rows of step s+1 are complete at the end of row pass s,
//     and the only CTA-wide dependency (row pass s+1 reads M columns written by
//     other warps) is an mbarrier every thread arrives on after its row pass and
//     waits on before the next one -- with a whole column pass of slack, instead
//     of a __syncthreads that lines every warp up twice per step;
//   * the R / CS rings are private to the warps of one 16-column chunk, so the
//     row -> column -> row hand-offs are pair barriers (bar.sync of two warps);
//   * the running (Q, P) of a lane's output rows is read and written by that
//     same lane in every harmonic (plain LDG / STG, L2): program order, no
//     cross-thread or cross-proxy ordering at all.
//
// Shared memory: M (two buffers) + R ring + CS ring; the 24 KB staging tile and
// the 16 KB (Q, P) tile of the TMA kernel are gone.
#pragma once

namespace fbf {

template <class C>
struct V2 {
  static constexpr size_t OFF_M = 0;
  static constexpr size_t M_BYTES = C::M_BYTES;
  static constexpr size_t OFF_R = OFF_M + 2 * M_BYTES;
  static constexpr size_t OFF_CS = OFF_R + 2 * size_t(C::RING) * C::RP * 8;
  static constexpr size_t OFF_BAR = C::up128(OFF_CS + size_t(C::CRING) * C::CP * 8);
  static constexpr size_t smem_bytes = OFF_BAR + 16;
  static constexpr bool FITS = smem_bytes <= 227 * 1024;
  static constexpr bool FITS2 = smem_bytes <= 113 * 1024;  // two CTAs per SM
};

// This thread's modulation inputs of one step, in registers (same element
// slots as ModNext<C>: row-major linear or warp rows).
template <class C>
struct Prefetch {
  using MN = ModNext<C>;
  int2 v[MN::ELEMS];
  // padded (u, f') rows [a, a + G) x columns [x0 - W, x0 + TW + W) of image b;
  // rows past the padded image are clamped (computed, never stored)
  __device__ __forceinline__ void load(const FusedArgs& A, const Unit& u, int a) {
    const int pw = A.pq_cols + 2 * C::W;
    const int ph = A.g.out_rows + 2 * C::W;
    const int r0 = a - A.g.out_row0 + C::W;
    const int2* __restrict__ img = A.uf + static_cast<long long>(u.b) * ph * pw + u.x0;
#pragma unroll
    for (int k = 0; k < MN::ELEMS; ++k) {
      int g, j;
      if constexpr (MN::LINEAR) {
        const int e0 = static_cast<int>(threadIdx.x) + C::NT * k;
        const int e = (MN::TOTAL % C::NT == 0) ? e0 : min(e0, MN::TOTAL - 1);
        g = e / C::MW;
        j = e - g * C::MW;
      } else {
        const int r = k / MN::NJ, i = k % MN::NJ;
        g = static_cast<int>(threadIdx.x >> 5) + r * MN::NWARP;
        j = min(static_cast<int>(threadIdx.x & 31) + 32 * i, C::MW - 1);
      }
      const int row = min(r0 + g, ph - 1);
      v[k] = __ldg(img + static_cast<long long>(row) * pw + j);
    }
  }
  // elements k0 .. k0+NB-1 (k0 a compile-time constant after unrolling)
  template <int NB>
  __device__ __forceinline__ void elements(int k0, p2* __restrict__ M, uint32_t n) const {
    int2 w[NB];
    int off[NB];
    bool ok[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int k = k0 + b;
      w[b] = v[k];
      if constexpr (MN::LINEAR) {
        const int e = static_cast<int>(threadIdx.x) + C::NT * k;
        ok[b] = MN::TOTAL % C::NT == 0 || e < MN::TOTAL;
        const int ec = (MN::TOTAL % C::NT == 0) ? e : min(e, MN::TOTAL - 1);
        off[b] = ec + ec / C::MW;  // g * MP + j with MP = MW + 1
      } else {
        const int r = k / MN::NJ, i = k % MN::NJ;
        const bool full = (C::MW % 32 == 0) || (i + 1 < MN::NJ);
        const int g = static_cast<int>(threadIdx.x >> 5) + r * MN::NWARP;
        const int j = static_cast<int>(threadIdx.x & 31) + 32 * i;
        ok[b] = full || j < C::MW;
        off[b] = g * C::MP + j;
      }
    }
    float c[NB], s[NB];
    sincos_turns_n<NB>(n, w, c, s);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const float fp = __int_as_float(w[b].y);
      if (ok[b]) {
        M[off[b]] = pk(c[b], c[b] * fp);
        M[C::G * C::MP + off[b]] = pk(s[b], s[b] * fp);
      }
    }
  }
  static constexpr int BS = MN::BS;
  static constexpr int NBATCH = MN::NBATCH;
  __device__ __forceinline__ void batch(int b, p2* __restrict__ M, uint32_t n) const {
    if (BS * b + BS <= MN::ELEMS)
      elements<BS>(BS * b, M, n);
    else
      elements<(MN::ELEMS % BS ? MN::ELEMS % BS : BS)>(BS * b, M, n);
  }
  __device__ __forceinline__ void all(p2* __restrict__ M, uint32_t n) const {
#pragma unroll
    for (int b = 0; b < NBATCH; ++b) batch(b, M, n);
  }
};

// Pair barrier of the warps sharing one 16-column chunk (their R / CS ring
// columns): named barrier 1 + chunk, or a warp sync when a chunk has one warp.
template <class C>
__device__ __forceinline__ void chunk_sync() {
  if constexpr (C::CHUNK_WARPS == 1)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;" ::"r"(1 + static_cast<int>(threadIdx.x >> 5) / C::CHUNK_WARPS),
                 "n"(32 * C::CHUNK_WARPS)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Row pass (fbf_fused.cuh row_pass) with the next step's modulation batches
// spread over its input positions instead of the deferred demodulation.
template <class C>
__device__ __forceinline__ void row_pass2(const FusedArgs& A, const p2* __restrict__ M, p2* __restrict__ R,
                                          float* __restrict__ CS, int a, int rows, int base,
                                          const Prefetch<C>& pf, p2* __restrict__ Mn, uint32_t nn, bool mod) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = lane >> 4;
  const int g = (lane & 15) + C::HALF * (warp % (C::G / C::HALF));
  const int xc = (warp / (C::G / C::HALF)) * C::KR;
  const bool live = g < rows;
  const p2* __restrict__ src = M + (h * C::G + g) * C::MP + xc;
  constexpr int TAPS_IN = C::KR + 2 * C::W;
  constexpr int NB = Prefetch<C>::NBATCH;
#ifndef FBF_V2_MOD_OFF
#define FBF_V2_MOD_OFF 4
#endif
  constexpr int SPAN = C::BOX ? C::KR + 2 * C::W : TAPS_IN;
  constexpr int OFF = SPAN <= FBF_V2_MOD_OFF + NB ? 0 : FBF_V2_MOD_OFF;
  constexpr int STRIDE = (SPAN - OFF) / NB > 0 ? (SPAN - OFF) / NB : 1;
  auto hook = [&](int q) {
    if (q >= OFF && (q - OFF) % STRIDE == 0 && (q - OFF) / STRIDE < NB)
      if (mod) pf.batch((q - OFF) / STRIDE, Mn, nn);
  };
  const int rel = a + g - base;
  const int slot = rel % C::RING;
  float* __restrict__ csrow = CS + 2 * (rel % C::CRING) * C::CP + h;
  p2 acc[C::KR];
  if constexpr (C::BOX) {
    p2 sum = 0ull;
#pragma unroll
    for (int m = 0; m <= 2 * C::W; ++m) {
      const p2 v = src[m];
      sum = add2(sum, v);
      if (m >= C::W && m < C::W + C::KR && live) csrow[2 * (xc + m - C::W)] = lo_of(v);
      hook(m);
    }
    acc[0] = sum;
#pragma unroll
    for (int i = 1; i < C::KR; ++i) {
      const p2 vin = src[i + 2 * C::W], vout = src[i - 1];
      sum = sub2(add2(sum, vin), vout);
      acc[i] = sum;
      const int m = i + 2 * C::W;
      if (m >= C::W && m < C::W + C::KR && live) csrow[2 * (xc + m - C::W)] = lo_of(vin);
      hook(2 * C::W + i);
    }
  } else {
#pragma unroll
    for (int i = 0; i < C::KR; ++i) acc[i] = 0ull;
#pragma unroll
    for (int q = 0; q < TAPS_IN; ++q) {
      const int m = fir_order(q, TAPS_IN, FBF_FIR_OI_ROW);
      const p2 v = src[m];
#pragma unroll
      for (int i = 0; i < C::KR; ++i) {
        const int j = m - i;
        if (j >= 0 && j <= 2 * C::W) {
          const float tv = A.k.t[j < C::W ? C::W - j : j - C::W];
          acc[i] = fma2(pk(tv, tv), v, acc[i]);
        }
      }
      if (m >= C::W && m < C::W + C::KR && live) csrow[2 * (xc + m - C::W)] = lo_of(v);
      hook(q);
    }
  }
#pragma unroll
  for (int b = (SPAN - OFF + STRIDE - 1) / STRIDE; b < NB; ++b)
    if (mod) pf.batch(b, Mn, nn);
  if (live) {
    p2* __restrict__ dst = R + (h * C::RING + slot) * C::RP + xc;
#pragma unroll
    for (int i = 0; i < C::KR; ++i) dst[i] = acc[i];
  }
}

// Column pass + demodulation (fbf_fused.cuh col_pass without the interleaved
// modulation and without deferral): the lane's running (Q, P) rows are loaded
// before its FIR and stored (or divided) after it.
template <class C>
__device__ __forceinline__ void col_pass2(const FusedArgs& A, const p2* __restrict__ R,
                                          const float* __restrict__ CS, const Unit& u, int o, int base,
                                          int dn_idx, bool first, bool divide, const FixedScale& fs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = lane >> 4;
  const int x = (lane & 15) + C::HALF * (warp / (C::G / C::KC));
  const int gi = (warp % (C::G / C::KC)) * C::KC;
  const int r0 = o + gi;
  const int gx = u.x0 + x;
  const int nr = min(C::KC, u.y1 - r0);
  constexpr int KH = C::KC / 2;
  const int rr = r0 + h * KH;  // first output row of this lane
  const int nh = gx < A.g.width ? nr - h * KH : 0;
  Pending<C> pd;
  pd.nh = nh;
  pd.dst = reinterpret_cast<p2*>(A.pq) +
           ((blockIdx.y * A.g.batch + u.b) * static_cast<long long>(A.g.out_rows) + (rr - A.g.out_row0)) *
               A.pq_cols +
           gx;
  // running (Q, P) of this lane's rows: written by this same lane in the
  // previous harmonic (program order); in flight during the FIR
#pragma unroll
  for (int k = 0; k < KH; ++k) pd.pq[k] = (first || k >= nh) ? 0ull : pd.dst[k * A.pq_cols];
  p2 acc[C::KC];
  const p2* __restrict__ Rh = R + h * C::RING * C::RP + x;
  const int s0 = (r0 - C::W - base) % C::RING;
  constexpr int TAPS_IN = C::KC + 2 * C::W;
  auto ring = [&](int m) {
    int s = s0 + m;
    s = s >= C::RING ? s - C::RING : s;
    return Rh[s * C::RP];
  };
  if constexpr (C::BOX) {
    p2 sum = 0ull;
#pragma unroll
    for (int m = 0; m <= 2 * C::W; ++m) sum = add2(sum, ring(m));
    acc[0] = sum;
#pragma unroll
    for (int i = 1; i < C::KC; ++i) {
      sum = sub2(add2(sum, ring(i + 2 * C::W)), ring(i - 1));
      acc[i] = sum;
    }
  } else {
#pragma unroll
    for (int i = 0; i < C::KC; ++i) acc[i] = 0ull;
#pragma unroll
    for (int q = 0; q < TAPS_IN; ++q) {
      const int m = fir_order(q, TAPS_IN, FBF_FIR_OI_COL);
      const p2 v = ring(m);
#pragma unroll
      for (int i = 0; i < C::KC; ++i) {
        const int j = m - i;
        if (j >= 0 && j <= 2 * C::W) {
          const float tv = A.k.t[j < C::W ? C::W - j : j - C::W];
          acc[i] = fma2(pk(tv, tv), v, acc[i]);
        }
      }
    }
  }
  // (q, p) = c (Gc, Fc) + s (Gs, Fs)   [bilateral.hpp:138-144, real form]
  const int cs0 = (r0 - base) % C::CRING;
#pragma unroll
  for (int i = 0; i < C::KC; ++i) {
    int sc = cs0 + i;
    sc = sc >= C::CRING ? sc - C::CRING : sc;
    const float w = CS[2 * (sc * C::CP + x) + h];
    pd.part[i] = mul2(pk(w, w), acc[i]);
  }
  const float dn = C::BOX ? A.h.d[dn_idx] * (A.k.box_tap * A.k.box_tap) : A.h.d[dn_idx];
  pd.dd = pk(dn * fs.sq, dn * fs.sp);
  if (!divide) {
#pragma unroll
    for (int k = 0; k < KH; ++k) pd.finish(k, h, A.pq_cols);
    return;
  }
  // bilateral.hpp:147-158: divide; flag the first collapsed denominator
  p2 qp[KH];
#pragma unroll
  for (int k = 0; k < KH; ++k) qp[k] = pd.qp(k, h);
  if (nh <= 0) return;
  float* __restrict__ drow = A.dst + u.b * A.g.dst_bstride +
                             static_cast<long long>(rr - A.g.out_row0) * A.g.dst_pitch + gx;
#pragma unroll
  for (int k = 0; k < KH; ++k) {
    if (k < nh) {
      float Q, P;
      from_fixed(pd.accumulate(k, qp[k]), fs, Q, P);
      if (!(fabsf(Q) >= A.h.q_floor) && A.bad) {
        const unsigned long long lin =
            static_cast<unsigned long long>(u.b) * A.g.full_height * A.g.width +
            static_cast<unsigned long long>(rr + k) * A.g.width + gx;
        atomicMin(A.bad, lin);
      }
      drow[k * static_cast<long long>(A.g.dst_pitch)] = A.h.shift + __fdiv_rn(P, Q);
    }
  }
}

template <class C, int MINB>
__global__ void __launch_bounds__(C::NT, MINB) fused_kernel2(const __grid_constant__ FusedArgs A) {
  using L = V2<C>;
  extern __shared__ __align__(16) unsigned char smem[];
  p2* M0 = reinterpret_cast<p2*>(smem + L::OFF_M);
  auto m_buf = [&](unsigned k) { return M0 + (k & 1u) * (L::M_BYTES / 8); };
  p2* R = reinterpret_cast<p2*>(smem + L::OFF_R);
  float* CS = reinterpret_cast<float*>(smem + L::OFF_CS);
  uint64_t* bar_m = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  if (threadIdx.x == 0) {
    mbar_init(bar_m, C::NT);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned ph = 0;  // parity of the next completion of bar_m
  unsigned mk = 0;  // this step's modulated rows are in M buffer mk & 1
  const FixedScale fs = fixed_scale(A.h.aq, A.fmax);
  Prefetch<C> pf;

  const int span = A.n_hi - A.n_lo;
  const int nb = A.n_lo + span * static_cast<int>(blockIdx.y) / A.groups;
  const int ne = A.n_lo + span * static_cast<int>(blockIdx.y + 1) / A.groups;
  if (nb >= ne) return;
  const int n_first = A.accumulate ? -1 : nb;

  const long long total = A.total;
  auto split = [&](long long p) {
    const long long sidx = p / A.g.out_rows;
    const long long r = p - sidx * A.g.out_rows;
    return sidx * A.g.out_rows + (r - r % C::KC);
  };
  const long long per = static_cast<long long>(A.g.out_rows) + A.unit_cost;
  const long long ctotal = total / A.g.out_rows * per;
  auto cut = [&](long long k) {
    const long long t = ctotal * k / gridDim.x;
    const long long s = t / per;
    return split(s * A.g.out_rows + min(t - s * per, static_cast<long long>(A.g.out_rows)));
  };
  const long long lo = blockIdx.x == 0 ? 0 : cut(blockIdx.x);
  const long long hi = blockIdx.x + 1 == gridDim.x ? total : cut(blockIdx.x + 1);
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
    // (harmonic, step) -> the following one
    auto advance = [&](int& n, int& s) {
      if (++s == nsteps) s = 0, ++n;
    };
    {  // bootstrap: step 0 of the group's first harmonic into M, step 1's inputs into registers
      int a, rows, o;
      step_rows<C>(u, 0, a, rows, o);
      __syncthreads();  // the previous unit is done with M, R and CS
      pf.load(A, u, a);
      pf.all(m_buf(mk), static_cast<uint32_t>(nb));
      int n1 = nb, s1 = 0;
      advance(n1, s1);
      if (n1 < ne) {
        step_rows<C>(u, s1, a, rows, o);
        pf.load(A, u, a);
      }
      mbar_arrive(bar_m);
    }
    for (int n = nb; n < ne; ++n) {
      const bool first = n == n_first;
      const bool divide = n + 1 == ne && !A.partial;
      for (int s = 0; s < nsteps; ++s) {
        int a, rows, o;
        step_rows<C>(u, s, a, rows, o);
        int n1 = n, s1 = s;
        advance(n1, s1);
        const bool more = n1 < ne;  // a next step exists: modulate it in this row pass
        int n2 = n1, s2 = s1;
        advance(n2, s2);
        mbar_wait(bar_m, ph);  // M of this step complete (every thread's previous row pass done)
        ph ^= 1u;
        row_pass2<C>(A, m_buf(mk), R, CS, a, rows, base, pf, m_buf(mk + 1), static_cast<uint32_t>(n1), more);
        if (more) {
          if (n2 < ne) {  // the step after next: its inputs load during this column pass
            int a2, rows2, o2;
            step_rows<C>(u, s2, a2, rows2, o2);
            pf.load(A, u, a2);
          }
          mbar_arrive(bar_m);
        }
        chunk_sync<C>();  // this chunk's R / CS rows of the step are written
        if (o >= 0) col_pass2<C>(A, R, CS, u, o, base, n - A.h.d_base, first, divide, fs);
        chunk_sync<C>();  // the chunk's column pass is done with the rings
        ++mk;
      }
    }
    pos += len;
  }
}

template <class C>
cudaError_t launch_cfg2(const FusedArgs& a_in, cudaStream_t st, int* grid_out) {
  using L = V2<C>;
  constexpr int MINB = L::FITS2 && C::NT <= 128 ? 2 : 1;
  FusedArgs a = a_in;
  a.strips = (a.g.width + C::TW - 1) / C::TW;
  a.pq_cols = a.strips * C::TW;
  a.total = static_cast<long long>(a.g.batch) * a.strips * a.g.out_rows;
  a.unit_cost = static_cast<int>(2 * C::W * FBF_TUNABLE(UNIT_COST_FRAC, kUnitCostFrac));
  if (a.groups < 1) a.groups = 1;
  struct DevInfo {
    int dev = -1, sms = 0, occ = 0;
  };
  thread_local DevInfo info;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (info.dev != dev) {
    e = cudaFuncSetAttribute(fused_kernel2<C, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(L::smem_bytes));
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&info.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.occ, fused_kernel2<C, MINB>, C::NT, L::smem_bytes);
    if (info.occ < 1) info.occ = 1;
    info.dev = dev;
  }
  long long grid = static_cast<long long>(info.sms) * info.occ / a.groups;
  const long long min_rows = 2 * C::W + C::G;
  const long long by_work = (a.total + min_rows - 1) / min_rows;
  if (grid > by_work) grid = by_work;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = static_cast<int>(grid);
  fused_kernel2<C, MINB><<<dim3(static_cast<unsigned>(grid), static_cast<unsigned>(a.groups)), C::NT,
                           L::smem_bytes, st>>>(a);
  return cudaGetLastError();
}

}  // namespace fbf
