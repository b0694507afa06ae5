// fbf_device.cuh -- device-side building blocks shared by the fused and the
// naive sm_100a paths of the shiftable Fourier-kernel bilateral filter.
//
//  * exact modular phase: the per-pixel base phase  u = round(f' * omega/(2 pi) * 2^32)
//    is computed once in fp64 (prep kernel); harmonic n uses the uint32 product
//    n*u, which is the phase n*omega*f' in turns, exact modulo 2^32.  No error
//    accumulates with n (unlike an angle-addition recurrence) and no state has to
//    be carried between harmonics.
//  * sincos_turns: quadrant reduction + paired minimax polynomials evaluated with
//    FFMA2 (fma.rn.f32x2), ~1 ulp, no MUFU and no table (no bank conflicts).
//  * ffma2: the Blackwell paired FP32 FMA; two fp32 lanes per instruction halves
//    the issue pressure of the FIR inner loops (measured: FFMA and FFMA2 both
//    reach ~126 lane-ops/clk/SM, profiles/r01_fma_microbench.txt).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fbf {

struct f2 {
  float x, y;
};

__device__ __forceinline__ unsigned long long as_u64(f2 v) {
  return (static_cast<unsigned long long>(__float_as_uint(v.y)) << 32) | __float_as_uint(v.x);
}
__device__ __forceinline__ f2 as_f2(unsigned long long u) {
  return f2{__uint_as_float(static_cast<unsigned>(u)), __uint_as_float(static_cast<unsigned>(u >> 32))};
}

// acc += a * b, lane-wise on the pair
__device__ __forceinline__ void ffma2(f2& acc, f2 a, f2 b) {
  unsigned long long r = as_u64(acc);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r) : "l"(as_u64(a)), "l"(as_u64(b)));
  acc = as_f2(r);
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(as_u64(a)), "l"(as_u64(b)), "l"(as_u64(c)));
  return as_f2(r);
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(as_u64(a)), "l"(as_u64(b)));
  return as_f2(r);
}

// image.hpp:34-40 mirror_index: half-sample symmetric reflection, period 2n.
__host__ __device__ __forceinline__ int mirror_index(int i, int n) {
  if (i >= 0 && i < n) return i;
  const int period = 2 * n;
  int j = i % period;
  if (j < 0) j += period;
  return j < n ? j : period - 1 - j;
}

// (cos, sin) of 2*pi*p/2^32.  Quadrant from the top bits (after a 1/8-turn
// offset), residual |r| <= pi/4, paired Horner for sin(r)/r and cos(r).
// Coefficients: weighted minimax on z = r^2 in [0, (pi/4)^2]; max abs error
// 6.5e-8 in fp32 (scratch fit).
__device__ __forceinline__ void sincos_turns(uint32_t p, float& c_out, float& s_out) {
  const uint32_t pq = p + 0x20000000u;
  const uint32_t q = pq >> 30;
  const int32_t ri = static_cast<int32_t>(pq & 0x3FFFFFFFu) - 0x20000000;
  const float r = static_cast<float>(ri) * 1.4629180792671596e-09f;  // 2 pi / 2^32
  const float z = r * r;
  const f2 zz{z, z};
  f2 t{2.716014023462776e-06f, 2.4390450562350452e-05f};
  t = fma2(t, zz, f2{-1.9839043670799583e-04f, -1.3886763481423259e-03f});
  t = fma2(t, zz, f2{8.333328180015087e-03f, 4.166662320494652e-02f});
  t = fma2(t, zz, f2{-1.666666716337204e-01f, -0.5f});
  t = fma2(t, zz, f2{1.0f, 1.0f});
  const float sr = r * t.x, cr = t.y;
  // rotate by q quarter turns
  const bool odd = q & 1u;
  uint32_t cb = __float_as_uint(odd ? sr : cr);
  uint32_t sb = __float_as_uint(odd ? cr : sr);
  cb ^= ((q + 1u) & 2u) << 30;
  sb ^= (q & 2u) << 30;
  c_out = __uint_as_float(cb);
  s_out = __uint_as_float(sb);
}

}  // namespace fbf
