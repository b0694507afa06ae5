// fbf_box2.cuh -- fused kernel for SMALL BOX windows (radius <= 7): the O(1)
// running-sum passes of bilateral_fast with the column sums in registers
// (reference: bilateral.hpp:109-160 with make_spatial_box, spatial.hpp:52-65;
// same planes, prep image, n = 0 kernel and fixed-point (Q, P) sums as
// fbf_fused.cuh).
//
// Why a second kernel: with a box window the two passes cost two adds per
// input, so the general kernel's shared-memory round trips (modulated tile ->
// row pass -> ring -> column pass) and the modulation of the halo dominate
// (c3: ~117 executed instructions per pixel and harmonic, issue 54 %,
// short-scoreboard / mio stalls 27 %).  Here:
//
//   work unit = one image, one (128 - 2W)-column strip, a run of output rows;
//   harmonic loop outermost, rows streamed in blocks of 16
//   phase 1  thread = one padded column: (u, f') by coalesced 8-byte loads,
//            modulation, and the VERTICAL running sum of the four planes in
//            registers (a 16-row register ring holds the modulated values:
//            the row leaving the window and the centre (c, s) come from it,
//            all indices compile-time) -> V tile in shared memory
//   phase 2  thread = one (row, plane) line half: HORIZONTAL running sum along
//            the tile row, in place (left half walks left to right and stores
//            H(x) at slot x, right half right to left and stores at x + 2W:
//            neither overwrites a slot the other still reads)
//   phase 3  thread = one output column: demodulate with the centre (c, s),
//            (Q, P) += round(d_n (q, p)) on the fixed-point grid, divide at
//            the last harmonic.
//
// Halo modulation is 128 / (128 - 2W) per output (1.08 at W = 5, the general
// kernel's 64-wide strips: 1.16), ~70 instructions per pixel and harmonic.
//
// Partition independence: a unit starts on a multiple of 16 output rows (the
// same cuts as the general kernel); the vertical sum is re-summed from the ring
// in a fixed order at every block's first row and updated incrementally
// inside the block; the horizontal sums start at the strip's fixed columns.
// So a pixel's float operations do not depend on the CTA count, the harmonic
// groups, strips or batches (the (Q, P) sums are integers anyway).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>

#include "fbf_device.cuh"
#include "fbf_params.h"
#include "fbf_tuning.h"

namespace fbf {

constexpr int kBox2Threads = 128;
constexpr int kBox2Rows = 16;    // rows per block = register ring length
constexpr int kBox2MaxW = 7;     // 2W + 1 <= 15 < ring
constexpr int kBox2Pitch = 129;  // V tile row pitch in float4 (= 1 mod 8: conflict-free line walks)

template <int W>
struct Box2Cfg {
  static constexpr int TWB = kBox2Threads - 2 * W;  // output columns of a strip
  static constexpr int XH = TWB / 2;                // left half: outputs [0, XH), right half [XH, TWB)
  static constexpr size_t smem_bytes = sizeof(float4) * kBox2Rows * kBox2Pitch + sizeof(float2) * kBox2Rows * kBox2Threads;
  static_assert(2 * W + 1 < kBox2Rows, "window must fit the register ring");
  static_assert(TWB % 2 == 0, "halves");
};

#ifndef FBF_BOX2_MINB
#define FBF_BOX2_MINB 3
#endif
template <int W>
__global__ void __launch_bounds__(kBox2Threads, FBF_BOX2_MINB) box2_kernel(const __grid_constant__ FusedArgs A) {
  using C = Box2Cfg<W>;
  constexpr int R = kBox2Rows, TWB = C::TWB, XH = C::XH, T = 2 * W + 1;
  extern __shared__ __align__(16) unsigned char b2s[];
  float4* Vt = reinterpret_cast<float4*>(b2s);
  float2* CSt = reinterpret_cast<float2*>(b2s + sizeof(float4) * R * kBox2Pitch);
  const int tid = threadIdx.x;

  // this CTA group's harmonics [nb, ne)
  const int span = A.n_hi - A.n_lo;
  const int nb = A.n_lo + span * static_cast<int>(blockIdx.y) / A.groups;
  const int ne = A.n_lo + span * static_cast<int>(blockIdx.y + 1) / A.groups;
  if (nb >= ne) return;
  const int n_first = (A.accumulate || (A.acc_group0 && blockIdx.y == 0)) ? -1 : nb;
  const FixedScale fs = fixed_scale(A.h.aq, A.fmax);
  const int pw = A.pq_cols + 2 * W, ph = A.g.out_rows + 2 * W;  // padded (u, f') image

  // CTA ranges in (strip, row) space, cost-balanced, cut on multiples of 16 rows
  // (as fbf_fused.cuh; strips are TWB wide here)
  const long long total = A.total;
  auto split = [&](long long p) {
    const long long sidx = p / A.g.out_rows;
    const long long r = p - sidx * A.g.out_rows;
    return sidx * A.g.out_rows + (r - r % R);
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
    const int len = static_cast<int>(min(static_cast<long long>(A.g.out_rows - r0), hi - pos));
    const int b = static_cast<int>(sidx / A.strips);
    const int x0 = static_cast<int>(sidx - static_cast<long long>(b) * A.strips) * TWB;  // first output column
    const int y0 = r0, y1 = r0 + len;  // output rows relative to out_row0
    const int nblocks = (len + R - 1) / R;
    // padded column of this thread (padded column 0 = global column -W)
    const int pcol = min(x0 + tid, pw - 1);
    const int2* __restrict__ ucol = A.uf + static_cast<long long>(b) * ph * pw + pcol;
    const int gx = x0 + tid;  // output column of this thread in phase 3 (tid < TWB)
    const bool col_ok = tid < TWB && gx < A.g.width;
    p2* const pqcol = reinterpret_cast<p2*>(A.pq) +
                      (static_cast<long long>(blockIdx.y) * A.g.batch + b) * A.g.out_rows * A.pq_cols + gx;
    float* const dcol = A.dst + b * A.g.dst_bstride + gx;

    for (int n = nb; n < ne; ++n) {
      const bool first = n == n_first;
      const bool divide = n + 1 == ne && !A.partial;
      const float dn = A.h.d[n - A.h.d_base] * (A.k.box_tap * A.k.box_tap);
      const p2 dd = pk(dn * fs.sq, dn * fs.sp);
      float4 ring[R];  // modulated (c, s, f'c, f's) of the last 16 input rows of this column
      // block 0 fills the ring with input rows [y0 + W - 16, y0 + W); blocks
      // 1.. take input rows y0 + W + 16 (blk - 1) + k and finish output rows
      // y0 + 16 (blk - 1) + k
      for (int blk = 0; blk <= nblocks; ++blk) {
        const int in0 = y0 + W + R * (blk - 1);  // first input row of the block, relative to out_row0
        int2 in[R];
        const int prow0 = in0 + W;  // padded row 0 = output row -W
        if (prow0 >= 0 && prow0 + R <= ph) {  // the whole block inside the padded image (CTA-uniform)
          const int2* __restrict__ src = ucol + static_cast<long long>(prow0) * pw;
#pragma unroll
          for (int k = 0; k < R; ++k) in[k] = __ldg(src + k * pw);
        } else {  // a unit's first / last block: clamped rows never reach a stored output
#pragma unroll
          for (int k = 0; k < R; ++k) in[k] = __ldg(ucol + static_cast<long long>(min(max(prow0 + k, 0), ph - 1)) * pw);
        }
        float4 V = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k4 = 0; k4 < R; k4 += 4) {
          int2 v4[4] = {in[k4], in[k4 + 1], in[k4 + 2], in[k4 + 3]};
          float c4[4], s4[4];
          sincos_turns_n<4>(static_cast<uint32_t>(n), v4, c4, s4);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int k = k4 + q;
            const float fp = __int_as_float(v4[q].y);
            const float4 m = make_float4(c4[q], s4[q], c4[q] * fp, s4[q] * fp);
            const float4 old = ring[(k + R - T) % R];  // the row leaving the window
            ring[k] = m;
            if (k == 0) {  // fresh sum, oldest row first (fixed order)
              V = ring[(R - 2 * W) % R];
#pragma unroll
              for (int d = 2 * W - 1; d >= 0; --d) {
                const float4 t = ring[(R - d) % R];
                V.x += t.x, V.y += t.y, V.z += t.z, V.w += t.w;
              }
            } else {
              V.x = (V.x + m.x) - old.x, V.y = (V.y + m.y) - old.y;
              V.z = (V.z + m.z) - old.z, V.w = (V.w + m.w) - old.w;
            }
            if (blk > 0) {
              Vt[k * kBox2Pitch + tid] = V;
              const float4 ctr = ring[(k + R - W) % R];  // input row of output row in0 + k - W
              if (tid >= W && tid < W + TWB) CSt[k * kBox2Threads + tid - W] = make_float2(ctr.x, ctr.y);
            }
          }
        }
        if (blk == 0) continue;
        __syncthreads();
        // ---- phase 2: horizontal running sums, in place.  thread = (row, plane
        // pair (c, s) | (f'c, f's), half): packed adds, warps 0 / 1 = left / right
        // half (lane = 2 row + pair: 8-byte accesses of 16 lanes hit 16 distinct
        // bank pairs); warps 2, 3 wait at the barrier
        if (tid < 64) {
          const int line = tid & 31;
          p2* row = reinterpret_cast<p2*>(Vt) + (line >> 1) * kBox2Pitch * 2 + (line & 1);  // slot j at row[2 j]
          if (tid < 32) {  // outputs 0 .. XH-1, left to right; H(x) -> slot x
            p2 sum = row[0];
#pragma unroll
            for (int j = 1; j < T; ++j) sum = add2(sum, row[2 * j]);
#pragma unroll 4
            for (int x = 0; x < XH; ++x) {
              const p2 h = sum;
              const p2 vout = row[2 * x];
              if (x + 1 < XH) sum = sub2(add2(sum, row[2 * (x + T)]), vout);
              row[2 * x] = h;
            }
          } else {  // outputs TWB-1 .. XH, right to left; H(x) -> slot x + 2W
            p2 sum = row[2 * (TWB - 1)];
#pragma unroll
            for (int j = 1; j < T; ++j) sum = add2(sum, row[2 * (TWB - 1 + j)]);
#pragma unroll 4
            for (int x = TWB - 1; x >= XH; --x) {
              const p2 h = sum;
              const p2 vout = row[2 * (x + 2 * W)];
              if (x > XH) sum = sub2(add2(sum, row[2 * (x - 1)]), vout);
              row[2 * (x + 2 * W)] = h;
            }
          }
        }
        __syncthreads();
        // ---- phase 3: demodulate, accumulate, divide
        {
          const int ob = y0 + R * (blk - 1);  // first output row of the block
          const int slot = tid < XH ? tid : tid + 2 * W;
          const int nv = col_ok ? min(R, y1 - ob) : 0;  // rows of this block this thread finishes
          p2* const prow = pqcol + static_cast<long long>(ob) * A.pq_cols;
          float* const drow = dcol + static_cast<long long>(ob) * A.g.dst_pitch;
          p2 pq[R];
#pragma unroll
          for (int k = 0; k < R; ++k) pq[k] = (!first && k < nv) ? prow[k * A.pq_cols] : 0ull;
#pragma unroll
          for (int k = 0; k < R; ++k) {
            if (k >= nv) break;
            const float4 H = Vt[k * kBox2Pitch + slot];
            const float2 cs = CSt[k * kBox2Threads + tid];
            // (q, p) = c (Hc, Hfc) + s (Hs, Hfs)   [bilateral.hpp:138-144, real form]
            const p2 qp = fma2(pk(cs.x, cs.x), pk(H.x, H.z), mul2(pk(cs.y, cs.y), pk(H.y, H.w)));
            const p2 acc = iadd2(pq[k], to_fixed(mul2(dd, qp)));
            if (!divide) {
              prow[k * A.pq_cols] = acc;
            } else {
              float Q, P;
              from_fixed(acc, fs, Q, P);
              if (!(fabsf(Q) >= A.h.q_floor) && A.bad) {
                const unsigned long long lin = static_cast<unsigned long long>(b) * A.g.full_height * A.g.width +
                                               static_cast<unsigned long long>(A.g.out_row0 + ob + k) * A.g.width + gx;
                atomicMin(A.bad, lin);
              }
              drow[k * A.g.dst_pitch] = A.h.shift + __fdiv_rn(P, Q);
            }
          }
        }
        __syncthreads();  // the tile is rewritten by the next block
      }
    }
    pos += len;
  }
}

template <int W>
cudaError_t launch_box2(const FusedArgs& a_in, cudaStream_t st, FusedPlan* plan) {
  using C = Box2Cfg<W>;
  FusedArgs a = a_in;
  a.strips = (a.g.width + C::TWB - 1) / C::TWB;
  a.pq_cols = (a.g.width + kFusedTW - 1) / kFusedTW * kFusedTW;  // the workspace layout's pitch
  a.total = static_cast<long long>(a.g.batch) * a.strips * a.g.out_rows;
  a.unit_cost = 6;  // a unit's ring fill (16 rows of modulation only) in rows of full work
  if (a.groups < 1) a.groups = 1;
  struct DevInfo {
    int dev = -1, sms = 0, occ = 0;
  };
  thread_local DevInfo info;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (info.dev != dev) {
    e = cudaFuncSetAttribute(box2_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(C::smem_bytes));
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&info.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.occ, box2_kernel<W>, kBox2Threads, C::smem_bytes);
    if (info.occ < 1) info.occ = 1;
    info.dev = dev;
  }
  long long grid = static_cast<long long>(info.sms) * info.occ / a.groups;
  const long long by_work = (a.total + 2 * kBox2Rows - 1) / (2 * kBox2Rows);  // at least two blocks per CTA
  if (grid > by_work) grid = by_work;
  if (grid < 1) grid = 1;
  if (plan) {
    *plan = FusedPlan{static_cast<int>(grid), info.occ, info.sms, 1 << 30, kBox2Rows, 1, kBox2Rows, C::TWB,
                      kBox2Threads, a.unit_cost, 2};
    return cudaSuccess;
  }
  box2_kernel<W><<<dim3(static_cast<unsigned>(grid), static_cast<unsigned>(a.groups)), kBox2Threads, C::smem_bytes,
                   st>>>(a);
  return cudaGetLastError();
}

}  // namespace fbf
