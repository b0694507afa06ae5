// fbf_params.h -- launch parameter blocks (passed by value: they live in the
// kernel's constant bank, so taps and coefficients are uniform operands).
#pragma once
#include <cuda.h>  // CUtensorMap (type only; encoded through the runtime's driver entry point)

#include <cstdint>

namespace fbf {

constexpr int kMaxD = 256;     // harmonic coefficients carried by one fused launch
constexpr int kMaxGroups = 16; // harmonic groups (CTA groups with their own (Q, P) plane) of one fused launch
constexpr int kMaxN = 65535;   // highest harmonic accepted (larger N: several fused launches)
constexpr int kFusedTW = 64;  // column-strip width of the fused kernel (workspace layout)
constexpr int kMaxWFused = 64;      // taps carried in the fused kernel's parameter block (W <= this)
constexpr int kMaxRadius = 1 << 20;  // largest spatial radius accepted (naive chain / convolve: taps in memory)

struct Pair {
  float x, y;
};

// Geometry shared by every kernel that reads a (possibly strip-local,
// possibly batched) image.  Global image is width x full_height; the device
// buffer holds global rows [src_row0, src_row0 + src_rows) of each image;
// output rows [out_row0, out_row0 + out_rows) are produced.
struct Geometry {
  int width;
  int full_height;
  int src_row0, src_rows;
  int out_row0, out_rows;
  int batch;
  long long src_bstride;  // elements between images in the source / uf buffers
  int src_pitch;          // elements between rows of the source buffer
  long long dst_bstride;  // elements between images in dst
  int dst_pitch;          // elements between rows of dst (row 0 = global out_row0)
};

// Fixed-point (Q, P): every harmonic's term d_n (q_n, p_n) is rounded once, in
// fp32, to integers on the grid 2^-aq (Q) and 2^-ap (P) and summed as int32.
// Integer sums are exact, so the result does not depend on how the harmonics
// are split among CTA groups, launches, pipeline chunks or GPUs (SPEC.md:300,
// "accumulation order ... independent of pixel-level parallelism").  aq comes
// from D = sum |d_n| (host, fill_harmonics): |Q| and every partial sum stay
// below 2^31 * 2^-aq.  ap = aq - k with 2^k >= max |f'| (k >= 7), from the
// prep kernel's max |f - shift| of the call (fmax word in the workspace): for
// 8-bit images k = 7 in every partition, so strips, batches and the whole
// image agree bit for bit.
struct Harmonics {
  int N;
  int aq;              // Q grid exponent (see above)
  int d_base;          // d[i] is the coefficient of harmonic d_base + i
  float d[kMaxD];      // cosine coefficients d_base .. d_base + kMaxD - 1 (fp32)
  double turns_per_unit;  // omega / (2 pi): phase in turns per intensity unit
  float shift;            // intensity shift applied before modulation (128)
  float q_floor;          // (w0 - eps) / 2 : denominator collapse threshold
};

struct Taps {
  int W;
  int box;                // 1: uniform box window (running-sum path)
  float box_tap;          // 1/(2W+1)
  float t[kMaxWFused + 1];     // tap |j| (spatial.hpp profile[W+j]); broadcast to both FFMA2 lanes
};

// Fused path: the prep kernel writes a mirror-PADDED (u, f') image per image,
// rows = out_rows + 2W (global rows out_row0-W ...), columns = strips*TW + 2W
// (global columns -W ...), so every step's tile is an in-bounds TMA box; the
// running (Q, P) workspace is out_rows x strips*TW per image.
struct FusedArgs {
  CUtensorMap tm_uf;  // int64 elements (u, f'), dims {uf_cols, out_rows + 2W, batch}, box {TW+2W, G, 1}
  CUtensorMap tm_pq;  // int64 elements (Q, P),  dims {pq_cols, out_rows, batch},     box {TW, G, 1}
  int pq_cols;        // strips * TW
  // Harmonic split: harmonics [n_lo, n_hi) are divided among `groups` CTA
  // groups (grid.y); group k accumulates its share into its own (Q, P) plane
  // (pq + k * batch * out_rows * pq_cols).  With partial = 0 and one group the
  // kernel divides at the last harmonic; otherwise it leaves the partial sums
  // in the planes for fbf_finish / an NCCL sum.
  int n_lo, n_hi;
  int groups;
  int partial;
  Geometry g;
  Taps k;
  const int2* uf;          // prep output: (u = phase increment, f' bits)
  float* dst;
  Pair* pq;                // workspace: per output pixel (Q, P) as an int32 pair (fixed point), out_rows x width per image
  const unsigned* fmax;    // workspace header: max |f'| of the call as float bits (prep)
  unsigned long long* bad; // min linear index (b*H*W + y*W + x) of a collapsed denominator
  int strips;              // ceil(width / TW)
  long long total;         // batch * strips * out_rows
  int seg_max;             // longest row run one CTA filters in one pass over n
  int unit_cost;           // extra cost of one work unit (its 2W-row prologue + bootstrap) in output rows
  unsigned long long* prof;  // phase cycle counters (FBF_PHASE_PROF builds only), else null
  int accumulate;  // 1: the launch's first harmonic adds to the (Q, P) planes instead of initialising them
  int n0_only;     // 1: launch_fused runs n0_plane_kernel (the n = 0 term) instead of the fused kernel
  int acc_group0;  // 1: group 0 alone accumulates (onto the n = 0 plane of n0_plane_kernel)
  Harmonics h;     // last: the coefficient block is the large member
};

// What a launch of this geometry looks like (the harmonic-group cost model in
// fbf_capi.cu simulates the kernel's own CTA cuts from it): launch_fused with
// a FusedPlan pointer fills it and launches nothing.
struct FusedPlan {
  int grid;       // CTAs per harmonic group (grid.x)
  int occ;        // resident CTAs per SM of this instance
  int sms;
  int seg_max;    // unit cap in rows
  int G, prologue, kc, tw, nt;
  int unit_cost;  // rows (the kernel's cut coordinate)
  int box;
};

}  // namespace fbf
