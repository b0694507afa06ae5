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

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "fbf_device.cuh"
#include "fbf_params.h"
#include "fbf_tuning.h"

namespace fbf {

// BOX: uniform window -> O(1) running sums (2 adds per output per pass in the
// steady state) instead of the (2W+1)-tap FIR; the 1/(2W+1)^2 weight is applied
// once, in the demodulation.
//
// Channel halves: the four real planes of a harmonic travel as two pairs,
// half A = (c, f'c) and half B = (s, f's), stored as separate 8-byte planes.
// Lanes 0-15 of a warp filter half A and lanes 16-31 the same pixels' half B,
// each with KR (KC) = 16 outputs per lane: per output a lane loads
// (16+2W)/16 8-byte words instead of (8+2W)/8 16-byte words, which cuts the
// shared-memory traffic of the two FIR passes by ~40% (the FIR loads were
// half of all smem wavefronts; profiles/r01_notes.md).  The two halves of an
// output meet in the demodulation through one shuffle (lane ^ 16).
// QT: the running (Q, P) of a work unit lives in tensor memory across all its
// harmonics (256-thread kernels, units <= 16 steps = 512 rows).  Each column-
// pass lane's 8 output rows x (Q, P) of a step are 16 TMEM columns of its own
// lane (tcgen05.ld / st 32x32b.x16: one instruction each); warps w and w+4
// share a lane quarter and take TMEM columns [0, 256) and [256, 512).  No
// (Q, P) tile in shared memory, no (Q, P) TMA per step; the global plane is
// read only at a unit's first harmonic (the n = 0 plane, or a previous chained
// launch) and written only at its last (partial sums).  The freed 16 KB pay
// for a 64-row CS ring whose column-pass windows never wrap (W + G <= 64).
template <int W_, int TW_, int G_, int KR_, int KC_, int NT_, bool BOX_ = false, bool QT_ = false>
struct FusedCfg {
  static constexpr int W = W_, TW = TW_, G = G_, KR = KR_, KC = KC_, NT = NT_;
  static constexpr bool BOX = BOX_;
  static constexpr bool QT = QT_;
  static_assert(!QT || (NT == 256 && G == 32 && KC == 16), "TMEM (Q, P): 8 warps, 16 steps of 32 rows");
  static constexpr bool CS64 = QT && W + G <= 64;
  // CSA: the CS ring is keyed on the OUTPUT row, (row - y0) mod CRING, with
  // CRING a multiple of 16: a column-pass lane's 16-row window starts on a
  // multiple of 16 and never wraps, so its 16 centre loads are one base plus
  // compile-time offsets (the per-load wrap arithmetic was ~3 % of all
  // executed instructions at c2).  Costs up to 15 more ring rows; the box
  // kernels keep the W + G ring (their 3 CTAs per SM do not fit the padding).
#ifndef FBF_CSA
#define FBF_CSA 1
#endif
  // (measured on / off per config: c4 W = 24 +1.8 %, c5 W = 12 +0.7 %, c2 W = 15 -0.3 % when it was
  // introduced, +0.1-0.3 % after the modulation / finish placement changes: on for every radius)
  static constexpr bool CSA = CS64 || (FBF_CSA != 0 && !BOX_);
  // PQG: the running (Q, P) rows are loaded by their own column-pass lane from
  // global memory (L2; written by the same lane in the previous harmonic:
  // program order, no proxy fence) instead of a per-step TMA tile in shared
  // memory -- 16 KB freed (for the column-major R ring), no (Q, P) TMA on the
  // leader's critical path
#ifndef FBF_PQLDG
#define FBF_PQLDG 0
#endif
  static constexpr bool PQG = FBF_PQLDG != 0 && !QT;
  static constexpr int SEG = QT ? 15 * G : (1 << 30);  // longest unit (TMEM columns; step 15 = scratch)
  // deferred demodulation (Pending): measured gains on the 256-thread Gaussian
  // kernels only (c2 +0.9 %, c4 +3.6 %); the short running-sum row pass of the
  // box path cannot hide it (c3 -4.6 %) and the 128-thread kernels break even
  static constexpr bool DEFER = !BOX_ && NT_ > 128;
  static constexpr int MW = TW + 2 * W;   // modulated row width
  static constexpr int MP = MW | 1;       // M plane pitch in 8-byte units (odd: conflict-free row walks)
  static constexpr int RING = 2 * W + G;  // R ring rows
  static constexpr int CRING = CS64 ? 64 : CSA ? (W + G + 15) / 16 * 16 : W + G;  // CS ring rows
  static constexpr int RP = TW + 1;       // R plane pitch in 8-byte units (row-major R)
  // Column-major R (RCOL): plane h, column x, ring slot: (h TW + x) RPT + slot,
  // RPT = RING rounded up to 2 mod 4 (a 2 RPT-word stride = 4 mod 8: the
  // 16-byte loads of 8 consecutive columns hit 8 distinct bank quads).  A column-pass lane then loads two consecutive ring
  // rows with one LDS.128 (slot and RING are even: a pair never straddles the
  // wrap), halving its ring loads and their wrap arithmetic.
#ifndef FBF_RCOL
#define FBF_RCOL 1
#endif
  // (the 256-thread Gaussian kernels: measured c2 +1.3 %, c5 +1.5 %, c4 +2.1 %;
  // the box path's single-row running-sum loads conflict in this layout, c3 -11 %;
  // the 128-thread W <= 9 kernel breaks even)
  static constexpr bool RCOL = FBF_RCOL != 0 && !BOX && NT > 128;
  static constexpr int RPT = RING % 4 == 2 ? RING : RING + 2;
  static constexpr size_t R_BYTES = RCOL ? 2 * size_t(TW) * RPT * 8 : 2 * size_t(RING) * RP * 8;
  static constexpr int CP = TW + 1;       // CS pitch in 8-byte units
  static constexpr int PROLOGUE = (2 * W + G - 1) / G;  // steps that only row-pass
  static constexpr int HALF = 16;         // lanes per channel half
  // smem carve-up (bytes; TMA destinations 128-byte aligned)
  static constexpr size_t up128(size_t v) { return (v + 127) & ~size_t(127); }
  static constexpr size_t OFF_STAGE = 0;
  static constexpr size_t OFF_PQ = up128(OFF_STAGE + size_t(G) * MW * 8);
  static constexpr size_t OFF_M = up128(OFF_PQ + (QT || PQG ? 0 : size_t(G) * TW * 8));  // planes A, B
  static constexpr size_t M_BYTES = 2 * size_t(G) * MP * 8;
  static constexpr size_t bytes_with(int nmb) {
    return up128(OFF_M + nmb * M_BYTES + R_BYTES + size_t(CRING) * CP * 8) + 16;
  }
  // M double-buffered where it fits: the next step's modulation then writes the
  // other buffer, and the row pass -> column pass hand-off only syncs the two
  // warps of a column chunk (their rows and columns) instead of the whole CTA
  static constexpr int NMB = NT > 128 && bytes_with(2) <= 227 * 1024 ? 2 : 1;  // small CTAs: keep 2 per SM
  static constexpr size_t OFF_R = OFF_M + NMB * M_BYTES;  // planes A, B
  static constexpr size_t OFF_CS = OFF_R + R_BYTES;
  static constexpr size_t OFF_BAR = up128(OFF_CS + size_t(CRING) * CP * 8);
  static constexpr size_t smem_bytes = OFF_BAR + 16;
  static_assert(KR == KC && KR == 16, "one lane per (half, 16 outputs)");
  // warps sharing one 16-column chunk: the row-pass producers and column-pass
  // consumers of that chunk's ring columns (the S2 hand-off group)
  static constexpr int CHUNK_WARPS = (NT / 32) / (TW / HALF);
  // warp -> (row group | run, 16-column chunk): the warps of a chunk (its S2
  // pair) are consecutive, so the two warps of an SMSP (w, w + 4) belong to
  // different pairs and drift apart, overlapping each other's non-FMA phases
  // (measured: pairing them on one SMSP, or mixing row groups on an SMSP, is
  // 1-10 % slower; profiles/r02_notes.md)
  static constexpr int NCH = TW / HALF;
  static constexpr int NRG = G / HALF;
  static __device__ __forceinline__ int rg_of(int warp) { return warp % NRG; }
  static __device__ __forceinline__ int chunk_of(int warp) { return warp / NRG; }
  static_assert(G % HALF == 0 && TW % HALF == 0, "tiling");
  static_assert((G / HALF) * (TW / KR) * 32 == NT, "row pass: one (16 rows, chunk) item per warp");
  static_assert((TW / HALF) * (G / KC) * 32 == NT, "column pass: one (16 columns, run) item per warp");
  static constexpr bool FITS = smem_bytes <= 227 * 1024;  // launchable at all (one CTA per SM)
};

// tensor memory: 32x32b.x16 = 16 consecutive 32-bit columns of this thread's lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, p2 (&v)[8]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = pki(static_cast<int>(r[2 * k]), static_cast<int>(r[2 * k + 1]));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const p2 (&v)[8]) {
  uint32_t r[16];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float a, b;
    upk(v[k], a, b);
    r[2 * k] = __float_as_uint(a);
    r[2 * k + 1] = __float_as_uint(b);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

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

// TMA load of the padded (u, f') rows [a, a+G) x columns [x0-W, x0+TW+W)
// into stage (the bootstrap of a unit); the step loop issues it together with
// the running (Q, P) rows of the step on one barrier phase.  Issued by thread
// 0 only; rows past the image are zero-filled and never consumed.
template <class C>
__device__ __forceinline__ void tma_uf(const FusedArgs& A, int2* stage, uint64_t* bar, const Unit& u,
                                       int a) {
  mbar_expect_tx(bar, static_cast<unsigned>(C::G * C::MW * 8));
  tma_load_3d(stage, &A.tm_uf, bar, u.x0, a - A.g.out_row0 + C::W, u.b);
}
// Modulation of one step, sliced into RPW*NJ independent elements per thread.
// Straight-line code: every slot is computed (clamped reads) and only the
// stores are predicated, so the element chains interleave freely with other
// work in the same basic block (rows past the step's end hold finite stale
// data and are never consumed).
template <class C>
struct ModNext {
  // Two lane mappings of the step's G x MW elements (both: consecutive lanes
  // on consecutive columns, conflict-free stage reads and M writes):
  //  * warp rows: warp w owns rows w, w + NWARP, ...; lane l columns l + 32 i
  //    (slots past a row's end are computed and dropped);
  //  * linear: element e = tid + NT * k in row-major order (no dropped slots,
  //    one division by MW per element).
  // Linear where it saves elements (c1 / c3 / c5 +1-2 %), else warp rows.
  static constexpr int TOTAL = C::G * C::MW;
  static constexpr int NWARP = C::NT / 32;
  static constexpr int NJ = (C::MW + 31) / 32;
  static constexpr int ELEMS_ROWS = (C::G / NWARP) * NJ;
  static constexpr int ELEMS_LIN = (TOTAL + C::NT - 1) / C::NT;
  static constexpr bool LINEAR = ELEMS_LIN < ELEMS_ROWS;
  static constexpr int ELEMS = LINEAR ? ELEMS_LIN : ELEMS_ROWS;  // per thread
  static_assert(C::G % NWARP == 0, "rows per warp");
  static_assert(C::MP == C::MW + 1, "M pitch: one pad column (MW is even)");
  const int2* stage;
  p2* M;  // plane A; plane B follows at + G * MP
  uint32_t n;

  // elements k0 .. k0+NB-1 of this thread with every stage of the chain issued
  // for all NB before the next: NB independent chains in flight (the compiler
  // tends to run single elements back to back, exposing the ~20-deep
  // dependency chain).  k0 must be a constant after unrolling.
  template <int NB>
  static __device__ __forceinline__ void elements(int k0, const int2* __restrict__ stage, p2* __restrict__ M,
                                                  uint32_t n) {
    int2 v[NB];
    int off[NB];
    bool ok[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int k = k0 + b;
      if constexpr (LINEAR) {
        const int e = static_cast<int>(threadIdx.x) + C::NT * k;
        ok[b] = TOTAL % C::NT == 0 || e < TOTAL;
        const int ec = (TOTAL % C::NT == 0) ? e : min(e, TOTAL - 1);
        off[b] = ec + ec / C::MW;  // g * MP + j with MP = MW + 1
        v[b] = stage[ec];
      } else {
        const int r = k / NJ, i = k % NJ;
        const bool full = (C::MW % 32 == 0) || (i + 1 < NJ);
        const int g = static_cast<int>(threadIdx.x >> 5) + r * NWARP;
        const int j = static_cast<int>(threadIdx.x & 31) + 32 * i;
        ok[b] = full || j < C::MW;
        off[b] = g * C::MP + j;
        v[b] = stage[g * C::MW + (full ? j : min(j, C::MW - 1))];
      }
    }
    float c[NB], s[NB];
    sincos_turns_n<NB>(n, v, c, s);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const float fp = __int_as_float(v[b].y);
      if (ok[b]) {
        M[off[b]] = pk(c[b], c[b] * fp);
        M[C::G * C::MP + off[b]] = pk(s[b], s[b] * fp);
      }
    }
  }
  // batch b of ceil(ELEMS / 4): four elements, the last batch the remainder
#ifndef FBF_MOD_BATCH
#define FBF_MOD_BATCH 4
#endif
  static constexpr int BS = FBF_MOD_BATCH;  // independent sincos chains per batch
  static constexpr int NBATCH = (ELEMS + BS - 1) / BS;
  static __device__ __forceinline__ void batch(int b, const int2* __restrict__ stage, p2* __restrict__ M,
                                               uint32_t n) {
    if (BS * b + BS <= ELEMS)
      elements<BS>(BS * b, stage, M, n);
    else
      elements<(ELEMS % BS ? ELEMS % BS : BS)>(BS * b, stage, M, n);
  }
};

template <class C>
__device__ __forceinline__ void modulate_rows(const int2* __restrict__ stage, p2* __restrict__ M,
                                              int rows, uint32_t n) {
  (void)rows;
#pragma unroll
  for (int b = 0; b < ModNext<C>::NBATCH; ++b) ModNext<C>::batch(b, stage, M, n);
}

// FBF_PHASE_PROF builds: thread 0 (and 128) of every CTA sums the cycles of
// each phase of the step loop into A.prof (diagnostics, tools/phase_probe.py);
// otherwise the marks compile to nothing.
struct PhaseClock {
#ifdef FBF_PHASE_PROF
  // thread 0 (the TMA leader) and thread 32 (a non-leader warp) separately:
  // out[0..9] and out[10..19]; index 9 = step count
  unsigned long long ph[10];
  long long t;
  __device__ __forceinline__ bool on() const { return threadIdx.x == 0 || threadIdx.x == 32; }
  __device__ __forceinline__ void start() {
    for (int i = 0; i < 10; ++i) ph[i] = 0;
    t = clock64();
  }
  __device__ __forceinline__ void mark(int i) {
    if (on()) {
      const long long now = clock64();
      ph[i] += now - t;
      t = now;
    }
  }
  __device__ __forceinline__ void flush(unsigned long long* out) {
    if (on() && out)
      for (int i = 0; i < 10; ++i) atomicAdd(out + (threadIdx.x ? 10 : 0) + i, ph[i]);
  }
  __device__ __forceinline__ void step() { ph[9] += on(); }
#elif defined(FBF_SHAKE)
  // race shaking (make shake): at every phase mark each warp sleeps a random
  // 0-2 us with probability 3/8, so the warps' relative timing differs from
  // run to run and from the product build; any missing barrier, fence or
  // mbarrier phase shows up as results that are not bit-identical
  // (tools/shake_check.py).  compute-sanitizer is not available on the GPU pool.
  unsigned st;
  __device__ __forceinline__ void start() {
    st = static_cast<unsigned>(clock64()) * 2654435761u ^ (blockIdx.x * 40503u + blockIdx.y * 9973u) ^
         ((threadIdx.x >> 5) * 0x9e3779b9u);
  }
  __device__ __forceinline__ void mark(int) {
    st = st * 1664525u + 1013904223u;
    const unsigned x = __shfl_sync(0xffffffffu, st, 0);
    if ((x >> 29) < 3) __nanosleep((x >> 8) & 2047u);
  }
  __device__ __forceinline__ void step() {}
  __device__ __forceinline__ void flush(unsigned long long*) {}
#else
  __device__ __forceinline__ void step() {}
  __device__ __forceinline__ void start() {}
  __device__ __forceinline__ void mark(int) {}
  __device__ __forceinline__ void flush(unsigned long long*) {}
#endif
};

// Deferred demodulation.  The column pass leaves this lane's (c|s)-weighted
// partials of its KC output rows and their running (Q, P) in registers; the
// NEXT step's row pass finishes them (swap halves with the partner lane,
// accumulate, store) between its FFMA2s, so the demodulation's latency chain
// (loads -> multiply -> shuffle -> add -> store) no longer stalls both warps of
// an SMSP at the end of every column pass.  Divide steps (last harmonic) and a
// unit's last step finish immediately.
#ifndef FBF_DEFER_Q0
#define FBF_DEFER_Q0 8
#endif
constexpr int kDeferQ0 = FBF_DEFER_Q0;  // first row-pass input position of the deferred finishes
// The finishes end where the ascending row FIR stops being FMA-dense (its last
// KR inputs feed fewer and fewer outputs), but stay >= 3 inputs apart:
// BACK = min(KR, inputs - Q0 - 3 KH) inputs before the end.  Measured per radius
// (BACK 0 / 8 / 14 at W = 12: 6,243 / 6,259 / 6,234; at W = 15: 4,158 / 4,160 /
// 4,208; BACK 0 / 12 / 20 at W = 24: 2,066 / 2,074 / 2,052 Mpixel/s).

template <class C>
struct Pending {
  static constexpr int KH = C::KC / 2;
  p2 part[C::KC];  // c * acc (half A) or s * acc (half B), rows gi .. gi+KC-1
  p2 pq[KH];       // running fixed-point (Q, P) of this lane's output rows (0 at the first harmonic)
  p2 dd;           // (d_n 2^aq, d_n 2^ap)
  p2* dst;         // (Q, P) of this lane's first output row; rows A.pq_cols apart
  int nh;          // rows this lane stores (<= 0: nothing pending)
  // QT: sums go to TMEM (taddr, one tcgen05.st after the last finish) unless tg
  p2 out[KH];
  uint32_t taddr;
  bool tg;    // this batch goes to the global plane (the unit's last harmonic)
  bool live;  // warp-uniform: a TMEM batch is pending
  // output row k of this lane: (q, p) = own half + partner's half
  __device__ __forceinline__ p2 qp(int k, int h) const {
    const p2 send = h ? part[k] : part[KH + k];
    const p2 own = h ? part[KH + k] : part[k];
    return add2(own, __shfl_xor_sync(0xffffffffu, send, 16));
  }
  // (Q, P) += round(d_n (q, p)) on the fixed-point grid (exact integer sum)
  __device__ __forceinline__ p2 accumulate(int k, p2 qpk) const { return iadd2(pq[k], to_fixed(mul2(dd, qpk))); }
  __device__ __forceinline__ void finish(int k, int h, int stride) {
    const p2 v = accumulate(k, qp(k, h));
    if constexpr (C::QT)
      out[k] = v;
    else if (k < nh)
      dst[k * stride] = v;
  }
  // QT: the batch's store after finish(0..KH-1): TMEM (all lanes of the warp),
  // or the global plane at the unit's last harmonic
  // (straight-line: the TMEM store always executes -- into the scratch
  // columns of step 15 when no batch is pending -- so ptxas needs no
  // collective wrapper around the .aligned instruction)
  __device__ __forceinline__ void flush(int stride) {
    if constexpr (C::QT) {
      tmem_st16((live && !tg) ? taddr : scratch, out);
      const bool g = live && tg;
#pragma unroll
      for (int k = 0; k < KH; ++k)
        if (g && k < nh) dst[k * static_cast<long long>(stride)] = out[k];
      live = false;
    }
  }
  uint32_t scratch;  // QT: TMEM columns of step 15 (never a real step: units <= 15 steps)
};

// Order in which the column FIR visits its input rows: alternately from both
// ends of the lane's window, inwards (0, T-1, 1, T-2, ...).  Every output
// then receives its small outer taps first and its large centre taps last,
// so the partial sums stay small for most of the accumulation -- same FFMA2
// and load counts as an ascending sweep.  Measured max |fast - exact| over
// the whole c4 image: 4.29e-4 -> 2.60e-4 (the paper bound there is 3.65e-4),
// c2 3.22e-4 -> 3.11e-4; the row pass gains less from it (ascending is
// faster there; profiles/r01_notes.md).  The order depends only on an
// output's position in its 16-aligned block: results stay independent of
// the partition.
#ifndef FBF_FIR_OI_ROW
#define FBF_FIR_OI_ROW 0
#endif
#ifndef FBF_FIR_OI_COL
#define FBF_FIR_OI_COL 1
#endif
__host__ __device__ constexpr int fir_order(int q, int n, bool oi) {
  return !oi ? q : (q & 1) ? n - 1 - (q >> 1) : (q >> 1);
}

// Row pass: warp = (16 rows, one KR-chunk of output columns); lane l filters
// row g of half h = l / 16 (plane A or B) into the R ring, and stores its
// half of the centre (c, s) of each input row's KR pixels into the CS ring.
template <class C>
__device__ __forceinline__ void row_pass(const FusedArgs& A, const p2* __restrict__ M, p2* __restrict__ R,
                                         float* __restrict__ CS, int a, int rows, int base,
                                         Pending<C>& pd) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = lane >> 4;
  const int g = (lane & 15) + C::HALF * C::rg_of(warp);
  const int xc = C::chunk_of(warp) * C::KR;
  // no early exit: rows past the step's end filter stale (finite) M rows and
  // only their stores are predicated, so every lane stays converged for the
  // deferred demodulation's shuffles interleaved below
  const bool live = g < rows;
  if (!C::DEFER && !live) return;
  const p2* __restrict__ src = M + (h * C::G + g) * C::MP + xc;
  constexpr int TAPS_IN = C::KR + 2 * C::W;
#ifdef FBF_DEFER_BACK
  constexpr int BACK = FBF_DEFER_BACK;
#else
  constexpr int ROOM = TAPS_IN - kDeferQ0 - 3 * (C::KC / 2);
  constexpr int BACK = ROOM < 0 ? 0 : ROOM < C::KR ? ROOM : C::KR;
#endif
  auto defer_at = [&](int m) {  // finish pending row k at input position m (compile-time)
#pragma unroll
    for (int k = 0; k < Pending<C>::KH; ++k)
      if (C::DEFER && m == kDeferQ0 + k * (TAPS_IN - BACK - kDeferQ0) / Pending<C>::KH) pd.finish(k, h, A.pq_cols);
  };
  const int rel = a + g - base;
  const int slot = rel % C::RING;
  // CS slot of input row rel: CSA keys it on the output row (rel - W) mod CRING,
  // so the column pass's 16-row windows start on multiples of 16 and never wrap
  const int cslot = C::CSA ? (rel + C::CRING - C::W) % C::CRING : rel % C::CRING;
  float* __restrict__ csrow = CS + 2 * cslot * C::CP + h;
  p2 acc[C::KR];
  if constexpr (C::BOX) {
    // running sum over the window [i, i+2W] (unweighted).  Every input is
    // loaded before the first add or centre store: with two adds per load
    // there is nothing to hide a load -> store / load -> add latency behind
    // (ncu, c3: the centre stores and the adds sat on short-scoreboard stalls
    // for 28 % of the kernel's samples when each load was used at once)
    p2 in[TAPS_IN];
#pragma unroll
    for (int m = 0; m < TAPS_IN; ++m) in[m] = src[m];
    p2 sum = 0ull;
#pragma unroll
    for (int m = 0; m <= 2 * C::W; ++m) {
      sum = add2(sum, in[m]);
      defer_at(m);
    }
    acc[0] = sum;
#pragma unroll
    for (int i = 1; i < C::KR; ++i) {
      sum = sub2(add2(sum, in[i + 2 * C::W]), in[i - 1]);
      acc[i] = sum;
      defer_at(2 * C::W + i);
    }
    if (live) {
#pragma unroll
      for (int i = 0; i < C::KR; ++i) csrow[2 * (xc + i)] = lo_of(in[i + C::W]);
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
      if (m >= C::W && m < C::W + C::KR && live)  // centre of output column xc + m - W
        csrow[2 * (xc + m - C::W)] = lo_of(v);
      defer_at(q);
    }
  }
  if (live) {
    if constexpr (C::RCOL) {
      p2* __restrict__ dst = R + (h * C::TW + xc) * C::RPT + slot;
#pragma unroll
      for (int i = 0; i < C::KR; ++i) dst[i * C::RPT] = acc[i];
    } else {
      p2* __restrict__ dst = R + (h * C::RING + slot) * C::RP + xc;
#pragma unroll
      for (int i = 0; i < C::KR; ++i) dst[i] = acc[i];
    }
  }
  if constexpr (C::DEFER) pd.flush(A.pq_cols);  // QT: the deferred batch's store
}

// Column pass: warp = (16 columns, one KC-run of output rows); lane l filters
// half h = l / 16 of column x.  Demodulation: each lane forms c*acc (half A)
// or s*acc (half B) for its KC rows, the two halves swap the partials of each
// other's 8 output rows with one shuffle, and each lane finishes 8 rows.
template <class C>
__device__ __forceinline__ void col_pass(const FusedArgs& A, const p2* __restrict__ R,
                                         const float* __restrict__ CS, const p2* __restrict__ pqs,
                                         const Unit& u, int o, int base, int dn_idx, bool first, bool divide,
                                         bool defer, const ModNext<C>& next, PhaseClock& clk, Pending<C>& pd,
                                         const FixedScale& fs, uint32_t tbase, bool seg_first, bool seg_last) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = lane >> 4;
  // warp -> (column chunk, run) as in the row pass's (chunk, row group): the
  // warps that row-passed a chunk's columns are the ones that read them here
  const int x = (lane & 15) + C::HALF * C::chunk_of(warp);
  const int gi = C::rg_of(warp) * C::KC;  // first output row of this lane, rel. to o
  const int r0 = o + gi;
  const int gx = u.x0 + x;
  const int nr = min(C::KC, u.y1 - r0);  // <= 0: this lane only helps with the modulation
  p2 acc[C::KC];
  constexpr int KH = C::KC / 2;
  if constexpr (C::PQG) {  // the lane's running (Q, P) rows: issued now, used after the FIR
    const int nh0 = gx < A.g.width ? nr - h * KH : 0;
    const p2* gq = reinterpret_cast<const p2*>(A.pq) +
                   ((blockIdx.y * A.g.batch + u.b) * static_cast<long long>(A.g.out_rows) +
                    (r0 + h * KH - A.g.out_row0)) * A.pq_cols + gx;
#pragma unroll
    for (int k = 0; k < KH; ++k)
      pd.pq[k] = (first || k >= nh0) ? 0ull : gq[k * static_cast<long long>(A.pq_cols)];
  }
  const p2* __restrict__ Rh = C::RCOL ? R + (h * C::TW + x) * C::RPT : R + h * C::RING * C::RP + x;
  const int s0 = (r0 - C::W - base) % C::RING;
  constexpr int TAPS_IN = C::KC + 2 * C::W;
  constexpr int NBATCH = ModNext<C>::NBATCH;
  // Where the next step's modulation starts inside the column FIR (visit
  // index q).  The outside-in order visits the window's edge rows first, which
  // feed only one or two outputs each (q-th input: ~q/2 + 1 FFMA2): the loop is
  // FMA-dense, with issue slots to spare for the modulation's ALU work, only
  // from q ~ 2 KC on.  Start there, leaving >= 4 visits per batch before the end
  // (W = 12: 24, W >= 14: 32).  Measured against the old fixed 12: c5 (W = 12)
  // 6,055 -> 6,230 Mpixel/s, c4 (W = 24) 2,009 -> 2,069, c2 (W = 15) 4,120 ->
  // 4,177; sweeps in profiles/r02_notes.md.
#ifdef FBF_MOD_OFF
  constexpr int MOD_OFF = FBF_MOD_OFF;
#else
  constexpr int MOD_ROOM = TAPS_IN - 4 * NBATCH > 0 ? (TAPS_IN - 4 * NBATCH) / 8 * 8 : 0;  // a multiple of 8 visits
  constexpr int MOD_OFF = MOD_ROOM < 2 * C::KC ? MOD_ROOM : 2 * C::KC;
#endif
  constexpr int OFF = (C::BOX || TAPS_IN <= MOD_OFF + NBATCH) ? 0 : MOD_OFF;
  constexpr int STRIDE = (TAPS_IN - OFF) / NBATCH > 0 ? (TAPS_IN - OFF) / NBATCH : 1;
  // one batch of (up to) 4 modulation elements of the next step per STRIDE taps
  auto batch = [&](int m) {
    if (m >= OFF && (m - OFF) % STRIDE == 0 && (m - OFF) / STRIDE < NBATCH)
      ModNext<C>::batch((m - OFF) / STRIDE, next.stage, next.M, next.n);
  };
  auto ring = [&](int m) {
    int s = s0 + m;
    s = s >= C::RING ? s - C::RING : s;
    return Rh[s * (C::RCOL ? 1 : C::RP)];
  };
  // rows m, m + 1 (m even) in one 16-byte load (RCOL)
  auto ring2 = [&](int m, p2& v0, p2& v1) {
    int s = s0 + m;
    s = s >= C::RING ? s - C::RING : s;
    const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(Rh + s);
    v0 = t.x;
    v1 = t.y;
  };
  if constexpr (C::BOX) {
    // all ring rows of the lane's window first (see the row pass)
    p2 in[TAPS_IN];
#pragma unroll
    for (int m = 0; m < TAPS_IN; ++m) in[m] = ring(m);
    p2 sum = 0ull;
#pragma unroll
    for (int m = 0; m <= 2 * C::W; ++m) {
      sum = add2(sum, in[m]);
      batch(m);
    }
    acc[0] = sum;
#pragma unroll
    for (int i = 1; i < C::KC; ++i) {
      sum = sub2(add2(sum, in[i + 2 * C::W]), in[i - 1]);
      acc[i] = sum;
      batch(i + 2 * C::W);
    }
  } else {
#pragma unroll
    for (int i = 0; i < C::KC; ++i) acc[i] = 0ull;
    auto taps = [&](int m, p2 v) {
#pragma unroll
      for (int i = 0; i < C::KC; ++i) {
        const int j = m - i;
        if (j >= 0 && j <= 2 * C::W) {
          const float tv = A.k.t[j < C::W ? C::W - j : j - C::W];
          acc[i] = fma2(pk(tv, tv), v, acc[i]);
        }
      }
    };
    if constexpr (C::RCOL) {
      static_assert(TAPS_IN % 2 == 0 && C::RING % 2 == 0, "row pairs");
      // pairs of input rows, visited outside-in like single rows below
#pragma unroll
      for (int qq = 0; qq < TAPS_IN / 2; ++qq) {
        const int m = 2 * fir_order(qq, TAPS_IN / 2, FBF_FIR_OI_COL);
        p2 v0, v1;
        ring2(m, v0, v1);
        taps(m, v0);
        batch(2 * qq);
        taps(m + 1, v1);
        batch(2 * qq + 1);
      }
    } else {
#pragma unroll
      for (int q = 0; q < TAPS_IN; ++q) {
        const int m = fir_order(q, TAPS_IN, FBF_FIR_OI_COL);
        taps(m, ring(m));
        batch(q);
      }
    }
  }
#pragma unroll
  for (int b = (TAPS_IN - OFF + STRIDE - 1) / STRIDE; b < NBATCH; ++b)
    ModNext<C>::batch(b, next.stage, next.M, next.n);
  clk.mark(5);
  // (q, p) = c (Gc, Fc) + s (Gs, Fs)   [bilateral.hpp:138-144, real form]:
  // this lane's half of every row now; the halves meet in Pending::qp
  if constexpr (C::CSA) {
    const float* __restrict__ csw = CS + 2 * (((r0 - u.y0) % C::CRING) * C::CP + x) + h;  // window start: a multiple of 16
#pragma unroll
    for (int i = 0; i < C::KC; ++i) {
      const float w = csw[2 * i * C::CP];
      pd.part[i] = mul2(pk(w, w), acc[i]);
    }
  } else {
    const int cs0 = (r0 - base) % C::CRING;
#pragma unroll
    for (int i = 0; i < C::KC; ++i) {
      int sc = cs0 + i;
      sc = sc >= C::CRING ? sc - C::CRING : sc;
      const float w = CS[2 * (sc * C::CP + x) + h];
      pd.part[i] = mul2(pk(w, w), acc[i]);
    }
  }
  const int rr = r0 + h * KH;  // first output row of this lane
  pd.nh = gx < A.g.width ? nr - h * KH : 0;  // rows of this lane (may be <= 0)
  p2* const gdst = reinterpret_cast<p2*>(A.pq) +
                   ((blockIdx.y * A.g.batch + u.b) * static_cast<long long>(A.g.out_rows) + (rr - A.g.out_row0)) *
                       A.pq_cols +
                   gx;
  if constexpr (C::QT) {
    // this lane's 16 TMEM columns of the step; (Q, P) from TMEM, or from the
    // global plane at the unit's first harmonic when the launch accumulates
    pd.taddr = tbase + 16u * static_cast<uint32_t>((o - u.y0) / C::G);
    pd.scratch = tbase + 16u * 15u;
    pd.tg = seg_last && !divide;
    tmem_wait_st();
    tmem_ld16(pd.taddr, pd.pq);  // unconditional (see flush); replaced below when not the running sum
    if (first || seg_first) {
#pragma unroll
      for (int k = 0; k < KH; ++k)
        pd.pq[k] = (!first && k < pd.nh) ? gdst[k * static_cast<long long>(A.pq_cols)] : 0ull;
    }
  } else if constexpr (C::PQG) {
    // (loaded at the head of the pass, in flight during the FIR)
  } else {
    const p2* __restrict__ pqin = pqs + (gi + h * KH) * C::TW + x;
#pragma unroll
    for (int k = 0; k < KH; ++k) pd.pq[k] = first ? 0ull : pqin[k * C::TW];
  }
  // box: both passes summed unweighted; the weight (1/(2W+1))^2 = w0 joins d_n here
  // d_n (dn_idx = n - d_base: the launch's coefficient block)
  const float dn = C::BOX ? A.h.d[dn_idx] * (A.k.box_tap * A.k.box_tap) : A.h.d[dn_idx];
  pd.dd = pk(dn * fs.sq, dn * fs.sp);  // exact: powers of two
  if (!divide) {
    pd.dst = gdst;
    pd.live = true;
    if (!defer) {
#pragma unroll
      for (int k = 0; k < KH; ++k) pd.finish(k, h, A.pq_cols);
      pd.flush(A.pq_cols);
      pd.nh = 0;
    }
    return;
  }
  // bilateral.hpp:147-158: divide; flag the first collapsed denominator
  p2 qp[KH];
#pragma unroll
  for (int k = 0; k < KH; ++k) qp[k] = pd.qp(k, h);
  const int nh = pd.nh;
  pd.nh = 0;
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

template <class C>
__global__ void __launch_bounds__(C::NT, (C::NT <= 128 ? 2 : 1)) fused_kernel(const __grid_constant__ FusedArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  int2* stage = reinterpret_cast<int2*>(smem + C::OFF_STAGE);
  p2* M0 = reinterpret_cast<p2*>(smem + C::OFF_M);
  unsigned mk = 0;  // step counter: this step's modulated rows are in M buffer mk & 1
  auto m_buf = [&](unsigned k) { return M0 + (C::NMB == 2 ? (k & 1u) : 0u) * (C::M_BYTES / 8); };
  p2* R = reinterpret_cast<p2*>(smem + C::OFF_R);
  float* CS = reinterpret_cast<float*>(smem + C::OFF_CS);
  p2* pqs = reinterpret_cast<p2*>(smem + C::OFF_PQ);
  uint64_t* bar_uf = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  const bool leader = threadIdx.x == 0;
  if (leader) {
    mbar_init(bar_uf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned ph_uf = 0;  // phase parity of the next completion of the copy barrier
  Pending<C> pd;
  pd.nh = 0;
  pd.live = false;
  pd.tg = false;
  const FixedScale fs = fixed_scale(A.h.aq, A.fmax);
  PhaseClock clk;
  clk.start();
#ifdef FBF_PHASE_PROF
  unsigned long long t_cta0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_cta0));
  unsigned cta_steps = 0;
#endif

  // this CTA group's harmonics [nb, ne)
  const int span = A.n_hi - A.n_lo;
  const int nb = A.n_lo + span * static_cast<int>(blockIdx.y) / A.groups;
  const int ne = A.n_lo + span * static_cast<int>(blockIdx.y + 1) / A.groups;
  if (nb >= ne) return;
  // QT: warp 0 allocates all 512 TMEM columns (one CTA per SM); this thread's
  // base: its warp's lane quarter, columns [0, 256) or [256, 512)
  uint32_t tbase = 0;
  if constexpr (C::QT) {
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + C::OFF_BAR + 8);
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tslot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int warp = static_cast<int>(threadIdx.x >> 5);
    tbase = *tslot + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + 256u * static_cast<uint32_t>(warp >> 2);
    pd.scratch = tbase + 16u * 15u;
    pd.taddr = pd.scratch;
  }
  // the harmonic whose (Q, P) initialises the planes (none for a chained launch
  // that accumulates onto an earlier one)
  const int n_first = (A.accumulate || (A.acc_group0 && blockIdx.y == 0)) ? -1 : nb;

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
  // Cost-balanced cuts: every work unit (strip of an image) also pays its
  // prologue, ~unit_cost rows, so a CTA whose range crosses a strip boundary
  // gets that many fewer rows.  Cuts are equally spaced in the cost coordinate
  // c(p) = p + unit_cost * (units before p); its inverse maps a target back to
  // a row position (a target inside a boundary's jump lands on the boundary).
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
                                         static_cast<long long>(min(A.seg_max, C::SEG))));
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
      modulate_rows<C>(stage, m_buf(mk), rows, static_cast<uint32_t>(nb));
    }
    for (int n = nb; n < ne; ++n) {
      const bool first = n == n_first;
      const bool divide = n + 1 == ne && !A.partial;
      for (int s = 0; s < nsteps; ++s) {
        int a, rows, o, a2, rows2, o2;
        step_rows<C>(u, s, a, rows, o);
        const bool wrap = s + 1 == nsteps;  // next step is step 0 of harmonic n+1
        const bool more = !wrap || n + 1 < ne;
        const bool want_pq = o >= 0 && !first && !C::QT && !C::PQG;
        step_rows<C>(u, wrap ? 0 : s + 1, a2, rows2, o2);
        clk.mark(0);
        __syncthreads();  // S1: M holds this step; the previous column pass is done; stage free
        clk.mark(1);
        // the next step's (u, f') rows and this step's (Q, P) complete on one
        // barrier phase (one wait instead of two)
        if (leader && (more || want_pq)) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(bar_uf, (more ? C::G * C::MW * 8u : 0u) + (want_pq ? C::G * C::TW * 8u : 0u));
          if (more) tma_load_3d(stage, &A.tm_uf, bar_uf, u.x0, a2 - A.g.out_row0 + C::W, u.b);
          if (want_pq)
            tma_load_3d(pqs, &A.tm_pq, bar_uf, u.x0, o - A.g.out_row0,
                        static_cast<int>(blockIdx.y) * A.g.batch + u.b);
        }
        clk.mark(8);
        row_pass<C>(A, m_buf(mk), R, CS, a, rows, base, pd);
        pd.nh = 0;
        clk.mark(2);
        if (more || want_pq) {
          mbar_wait(bar_uf, ph_uf);
          ph_uf ^= 1u;
        }
        clk.mark(3);
        // S2: this chunk's ring rows visible (the (u, f') and (Q, P) copies are
        // covered by each thread's own barrier wait above); with one M buffer
        // the whole CTA must also be past the row pass before M is rewritten
        if constexpr (C::NMB == 2) {
          if constexpr (C::CHUNK_WARPS == 1)
            __syncwarp();
          else
            asm volatile("bar.sync %0, %1;" ::"r"(1 + C::chunk_of(static_cast<int>(threadIdx.x >> 5))),
                         "n"(32 * C::CHUNK_WARPS)
                         : "memory");
        } else {
          __syncthreads();
        }
        clk.mark(4);
        // the next step's modulation is interleaved into this step's column pass
        // (its ALU work issues in the FFMA2 shadow); prologue steps run it alone
        const ModNext<C> next{stage, m_buf(mk + 1), static_cast<uint32_t>(wrap ? n + 1 : n)};
        if (o >= 0) {
          // defer the demodulation into the next row pass when there is a next
          // step in this unit and the same rows are not re-read by TMA within
          // two steps (nsteps > 2; the generic-proxy stores keep the same
          // distance to the next harmonic's async-proxy (Q, P) load as before)
          const bool defer = C::DEFER && more && !divide && nsteps > 2;
          col_pass<C>(A, R, CS, pqs, u, o, base, n - A.h.d_base, first, divide, defer, next, clk, pd, fs, tbase,
                      n == nb, n + 1 == ne);
          clk.mark(7);
        } else {
          modulate_rows<C>(stage, next.M, rows2, next.n);
          clk.mark(6);
        }
        // The (Q, P) rows stored this step (generic proxy: deferred finishes in
        // this step's row pass, immediate ones in its column pass) are read
        // back by a TMA load (async proxy) in the next harmonic: order them
        // before the S1 barrier that precedes any such load.  (Once per
        // harmonic would suffice, but measured slower: profiles/r02_notes.md.)
        if constexpr (!C::PQG) fence_proxy_async_global();
        clk.step();
#ifdef FBF_PHASE_PROF
        ++cta_steps;
#endif
        ++mk;
      }
    }
    pos += len;
  }
  if constexpr (C::QT) {  // every warp is done with its TMEM columns
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x < 32) {
      const uint32_t t0 = *reinterpret_cast<uint32_t*>(smem + C::OFF_BAR + 8);
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t0) : "memory");
    }
  }
  clk.flush(A.prof);
#ifdef FBF_PHASE_PROF
  // per-CTA record after the 32 phase words: smid, start / end (globaltimer ns), steps
  if (threadIdx.x == 0 && A.prof) {
    const unsigned cta = blockIdx.y * gridDim.x + blockIdx.x;
    if (cta < 1024) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      unsigned long long* rec = A.prof + 32 + 4 * cta;
      rec[0] = smid;
      rec[1] = t_cta0;
      rec[2] = t1;
      rec[3] = cta_steps;
    }
  }
#endif
}

inline int groups_of(const FusedArgs& a) { return a.groups < 1 ? 1 : a.groups; }

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
cudaError_t launch_cfg(const FusedArgs& a_in, cudaStream_t st, FusedPlan* plan) {
  constexpr int W = C::W;
  static_assert(C::TW == kFusedTW, "workspace layout assumes kFusedTW-wide strips");
  FusedArgs a = a_in;
  a.strips = (a.g.width + C::TW - 1) / C::TW;
  a.pq_cols = a.strips * C::TW;
  a.total = static_cast<long long>(a.g.batch) * a.strips * a.g.out_rows;
  // a unit's prologue row-passes 2W rows without a column pass or demodulation
  // (~55 % of a full row's cost, measured: FBF_UNIT_COST_PCT sweep)
  a.unit_cost = static_cast<int>(2 * W * FBF_TUNABLE(UNIT_COST_FRAC, kUnitCostFrac));
  if (a.groups < 1) a.groups = 1;
  // per device, once: the smem opt-in and the resident CTAs per SM (host calls
  // that would otherwise sit on every launch's critical path)
  struct DevInfo {
    int dev = -1, sms = 0, occ = 0;
  };
  thread_local DevInfo info;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (info.dev != dev) {
    e = cudaFuncSetAttribute(fused_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(C::smem_bytes));
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&info.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.occ, fused_kernel<C>, C::NT, C::smem_bytes);
    if (info.occ < 1) info.occ = 1;
    info.dev = dev;
  }
  const int sms = info.sms, occ = info.occ;
  // one wave in total: the harmonic groups share the SMs (rounded down: a
  // group count that does not divide the resident CTAs must not spill into a
  // second wave)
  long long grid = static_cast<long long>(sms) * occ / a.groups;
  // keep at least ~2W+G rows per CTA so the per-unit prologue stays amortised
  const long long min_rows = 2 * C::W + C::G;
  const long long by_work = (a.total + min_rows - 1) / min_rows;
  if (grid > by_work) grid = by_work;
  if (grid < 1) grid = 1;
  // L2-resident units: every harmonic re-reads a unit's (u, f') tiles and
  // read-modify-writes its (Q, P) rows.  When the CTAs' long runs (c5: 1,024-row
  // images, 148 CTAs) make that working set exceed L2, it streams from HBM
  // once per harmonic (c5: 128 GB per launch for 2.1 GB of image).  Capping a
  // unit's rows so grid x ((rows + 2W)(TW + 2W) + rows TW) x 8 B fits in ~80 %
  // of L2 keeps it resident, at the price of one more prologue per unit --
  // taken only where that prologue costs < 3 % (c5 yes; c4's 48-row prologue
  // no, measured -7 %).
  if (a.seg_max >= (1 << 30)) {
    const long long per_cta = a.total / std::max(1LL, grid);
    for (int seg = 2048; seg >= 512; seg /= 2) {
      const double ws = static_cast<double>(grid) * groups_of(a) *
                        ((seg + 2.0 * C::W) * (C::TW + 2.0 * C::W) + seg * static_cast<double>(C::TW)) * 8.0;
      if (per_cta > seg && ws <= 0.8 * 126e6 && kUnitCostFrac * 2.0 * C::W / seg <= 0.03) {
        a.seg_max = seg;
        break;
      }
    }
  }
#ifdef FBF_EXPERIMENTS
  a.seg_max = static_cast<int>(FBF_TUNABLE(SEG_MAX, a.seg_max));
#endif
  if (plan) {
    *plan = FusedPlan{static_cast<int>(grid), occ, sms, std::min(a.seg_max, C::SEG), C::G, C::PROLOGUE, C::KC, C::TW,
                      C::NT, a.unit_cost, C::BOX ? 1 : 0};
    return cudaSuccess;
  }
  e = encode_tile_3d(&a.tm_uf, a.uf, static_cast<unsigned long long>(a.pq_cols + 2 * W),
                     static_cast<unsigned long long>(a.g.out_rows + 2 * W),
                     static_cast<unsigned long long>(a.g.batch), C::MW, C::G);
  if (e != cudaSuccess) return e;
  e = encode_tile_3d(&a.tm_pq, a.pq, static_cast<unsigned long long>(a.pq_cols),
                     static_cast<unsigned long long>(a.g.out_rows),
                     static_cast<unsigned long long>(a.g.batch) * a.groups, C::TW, C::G);
  if (e != cudaSuccess) return e;
  fused_kernel<C><<<dim3(static_cast<unsigned>(grid), static_cast<unsigned>(a.groups)), C::NT, C::smem_bytes, st>>>(a);
  return cudaGetLastError();
}

// The n = 0 term as a single-plane filter (fbf_capi.cu launch_fused_range).
// At n = 0 the modulation is exact (c = 1, s = 0), so the harmonic's four
// planes reduce to one: (q, p) = (conv(1), conv(f')) = (1, conv(f')) -- the
// taps sum to one and mirror padding keeps it so (bilateral.hpp:126-144 with
// n = 0).  Inside the fused kernel it would cost a full harmonic (four planes,
// halo modulation, demodulation); here it is one separable FIR of f' read from
// the padded (u, f') image, rounded to the same fixed-point grid as every other
// term and written as group plane 0, onto which the fused kernel's group 0
// accumulates harmonics 1..N.  The fixed-point sum is exact, so where the n = 0
// term is computed does not change the result's bits.
//
// Tile: 64 output columns x 32 output rows per CTA (one tile per CTA), 256
// threads.  smem: the (32+2W) x (64+2W) input tile of f' as row PAIRS (float2:
// rows 2i, 2i+1), so the row pass filters two rows per FFMA2 with the tap as a
// broadcast operand; the row-filtered (32+2W) x 64 tile is read as column
// pairs by the column pass (FFMA2 again).
constexpr int kN0TX = 64, kN0Threads = 256;
template <int W, bool BOX, int TY>
struct N0Cfg {
  static constexpr int kN0TY = TY;
  static constexpr int IW = kN0TX + 2 * W, IH = kN0TY + 2 * W;  // IH even
  static constexpr int IWP = IW | 1;                            // pair-row pitch (float2 units)
  static constexpr int RP = kN0TX + 2;                          // row-filtered pitch (floats, even)
  static constexpr size_t smem_bytes = sizeof(float2) * size_t(IH / 2) * IWP + sizeof(float) * size_t(IH) * RP;
  static constexpr int ROW_ITEMS = (IH / 2) * (kN0TX / 8);  // (row pair, 8 columns)
  static constexpr int KC = 4;                              // column pass: (column pair, 4 rows)
  static constexpr int COL_ITEMS = (kN0TX / 2) * (kN0TY / KC);
};
#ifndef FBF_N0_MINB
#define FBF_N0_MINB 1
#endif
template <int W, bool BOX, int TY, bool FIN>
__global__ void __launch_bounds__(kN0Threads, FBF_N0_MINB) n0_plane_kernel(const __grid_constant__ FusedArgs A) {
  using C = N0Cfg<W, BOX, TY>;
  constexpr int kN0TY = TY;
  extern __shared__ __align__(16) unsigned char n0s[];
  p2* in2 = reinterpret_cast<p2*>(n0s);
  float* rowt = reinterpret_cast<float*>(n0s + sizeof(float2) * size_t(C::IH / 2) * C::IWP);
  const int pw = A.pq_cols + 2 * W, ph = A.g.out_rows + 2 * W;
  const int tiles_x = A.pq_cols / kN0TX;
  const int tiles_y = (A.g.out_rows + kN0TY - 1) / kN0TY;
  const long long per_img = static_cast<long long>(tiles_x) * tiles_y;
  const FixedScale fs = fixed_scale(A.h.aq, A.fmax);
  const float d0 = A.h.d[0];
  const p2 dd = pk(d0 * fs.sq, d0 * fs.sp);
  auto tap = [&](int j) { return BOX ? A.k.box_tap : A.k.t[j < 0 ? -j : j]; };
  // n0_only == 2: finish mode.  The n = 0 term is not written as a plane but
  // added to the A.groups harmonic-group planes the fused kernel left (every
  // group holds >= 1 harmonic), and the pixel is divided here: one kernel
  // instead of the n = 0 plane pass before and finish_groups after the fused
  // kernel (same integers, same bits)
  constexpr bool fin = FIN;
  const long long plane = static_cast<long long>(A.g.batch) * A.g.out_rows * A.pq_cols;  // even: pq_cols % 64 == 0
  const long long t = blockIdx.x;
  const int b = static_cast<int>(t / per_img);
  const int r = static_cast<int>(t - b * per_img);
  const int ty = r / tiles_x, tx = r - ty * tiles_x;
  const int x0 = tx * kN0TX, y0 = ty * kN0TY;  // padded coords of the tile's first input = output coords
  const int2* __restrict__ img = A.uf + static_cast<long long>(b) * ph * pw;
  float* in1 = reinterpret_cast<float*>(in2);
  static_assert(C::IW % 2 == 0 && C::RP % 2 == 0, "pairs");
  // load: warp = padded rows, lane = 16-byte column pairs; LR rows in flight
  // per warp (the plane-mode kernel has registers to spare: shared memory
  // limits it to 2-3 CTAs per SM, and its load phase was latency-bound:
  // long-scoreboard stalls 27 % of the samples)
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NP = C::IW / 2;  // IW even
    constexpr int PER = (NP + 31) / 32;
    constexpr int LR = FIN ? 4 : 8;
    for (int y4 = warp * LR; y4 < C::IH; y4 += LR * (kN0Threads / 32)) {
      int4 v[LR][PER];
#pragma unroll
      for (int r = 0; r < LR; ++r) {
        const int py = min(y0 + min(y4 + r, C::IH - 1), ph - 1);  // past the image: clamped, never stored
        const int4* __restrict__ row = reinterpret_cast<const int4*>(img + static_cast<long long>(py) * pw + x0);
#pragma unroll
        for (int c = 0; c < PER; ++c) v[r][c] = __ldg(row + min(lane + 32 * c, NP - 1));
      }
#pragma unroll
      for (int r = 0; r < LR; ++r) {
        const int yy = y4 + r;
        if (yy < C::IH) {
          float* dst = in1 + 2 * ((yy >> 1) * C::IWP) + (yy & 1);
#pragma unroll
          for (int c = 0; c < PER; ++c) {
            const int xp = lane + 32 * c;
            if (xp < NP) {
              dst[2 * (2 * xp)] = __int_as_float(v[r][c].y);
              dst[2 * (2 * xp + 1)] = __int_as_float(v[r][c].w);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  // row pass: item = (row pair, 8 output columns), FFMA2 over the pair; lanes
  // walk pair rows (conflict-free LDS.64: odd pitch)
  constexpr int NPR = C::IH / 2;
  for (int it = threadIdx.x; it < C::ROW_ITEMS; it += kN0Threads) {
    const int yp = it % NPR, xc = (it / NPR) * 8;
    const p2* __restrict__ src = in2 + yp * C::IWP + xc;
    p2 acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0ull;
#pragma unroll
    for (int m = 0; m < 8 + 2 * W; ++m) {
      const p2 v = src[m];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = m - k;
        if (j >= 0 && j <= 2 * W) {
          const float tv = tap(j - W);
          acc[k] = fma2(pk(tv, tv), v, acc[k]);
        }
      }
    }
    // (row 2yp, row 2yp+1) pairs -> column pairs of each row (8-byte stores)
    p2* r0 = reinterpret_cast<p2*>(rowt + (2 * yp) * C::RP + xc);
    p2* r1 = reinterpret_cast<p2*>(rowt + (2 * yp + 1) * C::RP + xc);
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      float a0, a1, b0, b1;
      upk(acc[k], a0, a1);
      upk(acc[k + 1], b0, b1);
      r0[k / 2] = pk(a0, b0);
      r1[k / 2] = pk(a1, b1);
    }
  }
  __syncthreads();
  // column pass: item = (column pair, run of KC output rows), FFMA2 over the pair
  Pair* __restrict__ out0 = A.pq + static_cast<long long>(b) * A.g.out_rows * A.pq_cols + x0;
  for (int it = threadIdx.x; it < C::COL_ITEMS; it += kN0Threads) {
    const int xp = it % (kN0TX / 2), run = it / (kN0TX / 2);
    p2 acc[C::KC];
#pragma unroll
    for (int k = 0; k < C::KC; ++k) acc[k] = 0ull;
    // finish mode: the first two group planes' values of this item are loaded
    // now and land during the FIR (further planes, if any, after it)
    constexpr int kPre = 2;
    ulonglong2 pre[C::KC][kPre];
    if (fin) {
#pragma unroll
      for (int k = 0; k < C::KC; ++k) {
        const int y = min(y0 + run * C::KC + k, A.g.out_rows - 1);
        const ulonglong2* __restrict__ gsrc =
            reinterpret_cast<const ulonglong2*>(out0 + 2 * xp + static_cast<long long>(y) * A.pq_cols);
#pragma unroll
        for (int g = 0; g < kPre; ++g) pre[k][g] = g < A.groups ? gsrc[g * (plane / 2)] : make_ulonglong2(0ull, 0ull);
      }
    }
    const float* __restrict__ col = rowt + run * C::KC * C::RP + 2 * xp;
#pragma unroll
    for (int m = 0; m < C::KC + 2 * W; ++m) {
      const p2 v = *reinterpret_cast<const p2*>(col + m * C::RP);
#pragma unroll
      for (int k = 0; k < C::KC; ++k) {
        const int j = m - k;
        if (j >= 0 && j <= 2 * W) {
          const float tv = tap(j - W);
          acc[k] = fma2(pk(tv, tv), v, acc[k]);
        }
      }
    }
    Pair* __restrict__ out = out0 + 2 * xp;
    if (fin) {  // further planes (many groups: small images), two at a time for all KC rows: 8 loads in flight
      for (int g0 = kPre; g0 < A.groups; g0 += 2) {
        ulonglong2 v[C::KC][2];
#pragma unroll
        for (int k = 0; k < C::KC; ++k) {
          const int y = min(y0 + run * C::KC + k, A.g.out_rows - 1);
          const ulonglong2* __restrict__ gsrc =
              reinterpret_cast<const ulonglong2*>(out + static_cast<long long>(y) * A.pq_cols);
#pragma unroll
          for (int i = 0; i < 2; ++i)
            v[k][i] = g0 + i < A.groups ? gsrc[(g0 + i) * (plane / 2)] : make_ulonglong2(0ull, 0ull);
        }
#pragma unroll
        for (int k = 0; k < C::KC; ++k)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            pre[k][0].x = iadd2(pre[k][0].x, v[k][i].x);
            pre[k][0].y = iadd2(pre[k][0].y, v[k][i].y);
          }
      }
    }
#pragma unroll
    for (int k = 0; k < C::KC; ++k) {
      const int y = y0 + run * C::KC + k;
      if (y < A.g.out_rows) {
        float c0, c1;
        upk(acc[k], c0, c1);
        p2 t0 = to_fixed(mul2(dd, pk(1.0f, c0))), t1 = to_fixed(mul2(dd, pk(1.0f, c1)));
        if constexpr (!FIN) {
          float q0, p0, q1, p1;
          upk(t0, q0, p0);
          upk(t1, q1, p1);
          *reinterpret_cast<float4*>(out + static_cast<long long>(y) * A.pq_cols) = make_float4(q0, p0, q1, p1);
        } else {
          // finish mode: + the harmonic groups' planes (exact integer sums), divide
#pragma unroll
          for (int g = 0; g < kPre; ++g) {
            t0 = iadd2(t0, pre[k][g].x);
            t1 = iadd2(t1, pre[k][g].y);
          }
          float* __restrict__ drow = A.dst + b * A.g.dst_bstride + static_cast<long long>(y) * A.g.dst_pitch;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int gx = x0 + 2 * xp + j;
            if (gx >= A.g.width) break;
            float Q, P;
            from_fixed(j ? t1 : t0, fs, Q, P);
            if (!(fabsf(Q) >= A.h.q_floor) && A.bad) {
              const unsigned long long lin = static_cast<unsigned long long>(b) * A.g.full_height * A.g.width +
                                             static_cast<unsigned long long>(A.g.out_row0 + y) * A.g.width + gx;
              atomicMin(A.bad, lin);
            }
            drow[gx] = A.h.shift + __fdiv_rn(P, Q);
          }
        }
      }
    }
  }
}

template <int W, bool BOX, int TY, bool FIN>
cudaError_t launch_n0_ty(const FusedArgs& a, cudaStream_t st) {
  using C = N0Cfg<W, BOX, TY>;
  static_assert(C::smem_bytes <= 227 * 1024, "n0 tile exceeds shared memory");
  thread_local int dev_done = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev_done != dev) {
    e = cudaFuncSetAttribute(n0_plane_kernel<W, BOX, TY, FIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(C::smem_bytes));
    if (e != cudaSuccess) return e;
    dev_done = dev;
  }
  const long long tiles = static_cast<long long>(a.strips) * ((a.g.out_rows + TY - 1) / TY) * a.g.batch;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidValue;
  n0_plane_kernel<W, BOX, TY, FIN><<<static_cast<unsigned>(tiles), kN0Threads, C::smem_bytes, st>>>(a);
  return cudaGetLastError();
}
// 128-row tiles (row-pass halo overhead (128+2W)/128) where they still give a
// few CTAs per SM, else 32-row tiles (small images)
template <int W, bool BOX>
cudaError_t launch_n0(const FusedArgs& a_in, cudaStream_t st) {
  FusedArgs a = a_in;
  a.strips = (a.g.width + kFusedTW - 1) / kFusedTW;
  a.pq_cols = a.strips * kFusedTW;
  const long long tiles64 = static_cast<long long>(a.strips) * ((a.g.out_rows + 63) / 64) * a.g.batch;
  int ty = tiles64 >= 8 * 148 ? 128 : tiles64 >= 2 * 148 ? 64 : 32;
#ifdef FBF_EXPERIMENTS
  ty = static_cast<int>(FBF_TUNABLE(N0_TY, ty));
#endif
  if (a.n0_only == 2) {  // finish mode (after the fused kernel's harmonic groups)
    if (ty >= 128) return launch_n0_ty<W, BOX, 128, true>(a, st);
    if (ty >= 64) return launch_n0_ty<W, BOX, 64, true>(a, st);
    return launch_n0_ty<W, BOX, 32, true>(a, st);
  }
  if (ty >= 128) return launch_n0_ty<W, BOX, 128, false>(a, st);
  if (ty >= 64) return launch_n0_ty<W, BOX, 64, false>(a, st);
  return launch_n0_ty<W, BOX, 32, false>(a, st);
}

// Small (128 threads, G=16, two CTAs per SM) for W <= 9, big (256 threads,
// G=32, one CTA per SM) otherwise -- measured, profiles/r01_cfg_compare.txt.
// FBF_FUSED_CFG=small|big overrides where both fit (experiment build only).
// TMEM (Q, P) when every CTA's rows fit one unit of <= 16 steps (no extra
// prologues from the 512-row cap): small and medium images (c2), not the
// long per-CTA runs of c4 / c5
inline bool qt_fits(const FusedArgs& a, int groups, int seg_rows) {
  thread_local int dev = -1, sms = 148;
  int d = 0;
  if (cudaGetDevice(&d) == cudaSuccess && d != dev) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    dev = d;
  }
  const long long strips = (a.g.width + kFusedTW - 1) / kFusedTW;
  const long long total = static_cast<long long>(a.g.batch) * strips * a.g.out_rows;
  const long long ctas = std::max(1, sms / std::max(1, groups));
  return (total + ctas - 1) / ctas + 32 <= seg_rows;
}

template <int W, bool BOX = false>
cudaError_t launch_w(const FusedArgs& a, cudaStream_t st, FusedPlan* plan) {
  if (a.n0_only) return launch_n0<W, BOX>(a, st);
  using Small = FusedCfg<W, 64, 16, 16, 16, 128, BOX>;
  using Big = FusedCfg<W, 64, 32, 16, 16, 256, BOX>;
#ifdef FBF_EXPERIMENTS  // TMEM (Q, P): measured slower (profiles/r02_notes.md), experiment build only
  using BigQ = FusedCfg<W, 64, 32, 16, 16, 256, BOX, true>;
  if constexpr (!BOX && W > 9 && BigQ::FITS) {
    if (FBF_TUNABLE(QT, 0) != 0 && qt_fits(a, std::max(1, a.groups), BigQ::SEG)) return launch_cfg<BigQ>(a, st, plan);
  }
#endif
#ifdef FBF_EXPERIMENTS
  const char* env = getenv("FBF_FUSED_CFG");
#else
  const char* env = nullptr;
#endif
  if constexpr (Small::smem_bytes <= 113 * 1024) {  // two 128-thread CTAs per SM
    const bool big = env ? env[0] == 'b' : !(W <= 9);
    if (!big || !Big::FITS) return launch_cfg<Small>(a, st, plan);
  }
  if constexpr (Big::FITS) {
    return launch_cfg<Big>(a, st, plan);
  } else if constexpr (Small::FITS) {  // large W: one 128-thread CTA per SM
    return launch_cfg<Small>(a, st, plan);
  } else {
    (void)env;
    return cudaErrorInvalidValue;
  }
}

}  // namespace fbf

#define FBF_INSTANTIATE_FUSED(WW) \
  template cudaError_t fbf::launch_w<WW, false>(const fbf::FusedArgs&, cudaStream_t, fbf::FusedPlan*);
#define FBF_INSTANTIATE_FUSED_BOX(WW) \
  template cudaError_t fbf::launch_w<WW, true>(const fbf::FusedArgs&, cudaStream_t, fbf::FusedPlan*);
