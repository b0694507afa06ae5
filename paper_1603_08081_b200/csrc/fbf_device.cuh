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
//  * pairs: two fp32 lanes in one 64-bit register pair (p2).  Blackwell's FFMA2
//    does both lanes in one instruction, halving the issue pressure of the FIR
//    loops (measured: FFMA and FFMA2 both reach ~126 lane-ops/clk/SM,
//    profiles/r01_fma_microbench.txt).  A pair built from one scalar {t, t}
//    compiles to FFMA2's scalar-broadcast operand form (no register moves).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fbf {

using p2 = unsigned long long;  // packed (lo, hi) fp32 pair

__device__ __forceinline__ p2 pk(float lo, float hi) {
  p2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk(p2 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ float lo_of(p2 v) {
  float a, b;
  upk(v, a, b);
  return a;
}
__device__ __forceinline__ float hi_of(p2 v) {
  float a, b;
  upk(v, a, b);
  return b;
}
// a * b + c, lane-wise
__device__ __forceinline__ p2 fma2(p2 a, p2 b, p2 c) {
  p2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ p2 add2(p2 a, p2 b) {
  p2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ p2 sub2(p2 a, p2 b) {
  p2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ p2 mul2(p2 a, p2 b) {
  p2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// int32 pair <-> p2 and lane-wise int32 add (the fixed-point (Q, P) sums)
__device__ __forceinline__ p2 pki(int lo, int hi) { return pk(__int_as_float(lo), __int_as_float(hi)); }
__device__ __forceinline__ p2 iadd2(p2 a, p2 b) {
  float al, ah, bl, bh;
  upk(a, al, ah);
  upk(b, bl, bh);
  return pki(__float_as_int(al) + __float_as_int(bl), __float_as_int(ah) + __float_as_int(bh));
}
// the term (x_q, x_p) (already scaled by 2^aq, 2^ap) rounded to integers
__device__ __forceinline__ p2 to_fixed(p2 x) {
  float xq, xp;
  upk(x, xq, xp);
  return pki(__float2int_rn(xq), __float2int_rn(xp));
}
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }  // |e| <= 126

// Fixed-point grids of the (Q, P) sums (fbf_params.h Harmonics): 2^aq for Q,
// 2^ap for P with ap = aq - k, 2^k >= max |f'| of the call (fmax word, float
// bits, written by the prep kernel), k >= 7.
struct FixedScale {
  float sq, sp;  // 2^aq, 2^ap  (term scales)
  float iq, ip;  // 2^-aq, 2^-ap (back to values)
};
__device__ __forceinline__ FixedScale fixed_scale(int aq, const unsigned* fmax) {
  const unsigned b = fmax ? *fmax : 0u;
  int k = static_cast<int>((b >> 23) & 0xffu) - 127 + ((b & 0x7fffffu) != 0u);  // ceil(log2 fmax)
  k = min(max(k, 7), 60);
  const int ap = aq - k;
  return FixedScale{pow2f(aq), pow2f(ap), pow2f(-aq), pow2f(-ap)};
}
// (Q, P) values of a fixed-point pair
__device__ __forceinline__ void from_fixed(p2 v, const FixedScale& fs, float& Q, float& P) {
  float a, b;
  upk(v, a, b);
  Q = __int2float_rn(__float_as_int(a)) * fs.iq;
  P = __int2float_rn(__float_as_int(b)) * fs.ip;
}

// cp.async (LDGSTS) helpers: 8-byte global -> shared copies in commit groups.
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// mbarrier + TMA (cp.async.bulk.tensor) helpers.  One elected thread arms the
// barrier with the expected byte count and issues the tile copy; every thread
// waits on the phase parity.
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// order this thread's earlier generic-proxy global writes before later
// async-proxy (TMA) reads of the same addresses, across a barrier
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// 3-D tile load (x, y, image) of a CUtensorMap into shared memory
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar, int x, int y,
                                            int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(smem_dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_addr(bar))
      : "memory");
}

// 3-D tile store shared -> global (bulk async group; completion via wait_group)
__device__ __forceinline__ void tma_store_3d(const void* tmap, const void* smem_src, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(tmap),
      "r"(smem_addr(smem_src)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N bulk groups still read their shared-memory source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// L2 prefetch of a 3-D tile (no shared memory, no completion tracking)
__device__ __forceinline__ void tma_prefetch_3d(const void* tmap, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(tmap), "r"(x),
               "r"(y), "r"(z)
               : "memory");
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
// offset), residual |r| <= pi/4, paired Horner (three FFMA2) for sin(r)/r and
// cos(r).  Coefficients: weighted minimax of degree 3 in z = r^2 on
// [0, (pi/4)^2]; max abs error 6.0e-8 (sin), 9.2e-8 (cos) in fp32.
constexpr float kSin1 = -0.16666650772094727f, kSin2 = 0.00833197869360447f, kSin3 = -0.000194956359337084f;
constexpr float kCos1 = -0.49999895691871643f, kCos2 = 0.04165629297494888f, kCos3 = -0.0013597822980955243f;
__device__ __forceinline__ void sincos_turns(uint32_t p, float& c_out, float& s_out) {
  const uint32_t pq = p + 0x20000000u;
  const uint32_t q = pq >> 30;
  const int32_t ri = static_cast<int32_t>(pq & 0x3FFFFFFFu) - 0x20000000;
  const float r = static_cast<float>(ri) * 1.4629180792671596e-09f;  // 2 pi / 2^32
  const float z = r * r;
  const p2 zz = pk(z, z);
  p2 t = fma2(pk(kSin3, kCos3), zz, pk(kSin2, kCos2));
  t = fma2(t, zz, pk(kSin1, kCos1));
  t = fma2(t, zz, pk(1.0f, 1.0f));
  float ts, tc;
  upk(t, ts, tc);
  const float sr = r * ts, cr = tc;
  // rotate by q quarter turns
  const bool odd = q & 1u;
  uint32_t cb = __float_as_uint(odd ? sr : cr);
  uint32_t sb = __float_as_uint(odd ? cr : sr);
  cb ^= ((q + 1u) & 2u) << 30;
  sb ^= (q & 2u) << 30;
  c_out = __uint_as_float(cb);
  s_out = __uint_as_float(sb);
}

// sincos_turns of NB phases n * v[b].x, each stage issued for all NB (ILP)
template <int NB>
__device__ __forceinline__ void sincos_turns_n(uint32_t n, const int2 (&v)[NB], float (&c_out)[NB],
                                               float (&s_out)[NB]) {
  uint32_t q[NB];
  float r[NB];
  p2 t[NB], zz[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const uint32_t pq = n * static_cast<uint32_t>(v[b].x) + 0x20000000u;
    q[b] = pq >> 30;
    const int32_t ri = static_cast<int32_t>(pq & 0x3FFFFFFFu) - 0x20000000;
    r[b] = static_cast<float>(ri) * 1.4629180792671596e-09f;  // 2 pi / 2^32
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const float z = r[b] * r[b];
    zz[b] = pk(z, z);
    t[b] = fma2(pk(kSin3, kCos3), zz[b], pk(kSin2, kCos2));
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) t[b] = fma2(t[b], zz[b], pk(kSin1, kCos1));
#pragma unroll
  for (int b = 0; b < NB; ++b) t[b] = fma2(t[b], zz[b], pk(1.0f, 1.0f));
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    float ts, tc;
    upk(t[b], ts, tc);
    const float sr = r[b] * ts, cr = tc;
    const bool odd = q[b] & 1u;
    uint32_t cb = __float_as_uint(odd ? sr : cr);
    uint32_t sb = __float_as_uint(odd ? cr : sr);
    cb ^= ((q[b] + 1u) & 2u) << 30;
    sb ^= (q[b] & 2u) << 30;
    c_out[b] = __uint_as_float(cb);
    s_out[b] = __uint_as_float(sb);
  }
}

}  // namespace fbf
