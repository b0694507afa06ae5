// FIR-only probe: runs the fused kernel's row pass (the real row_pass<C> code)
// back to back from shared memory, to separate the FIR loop's own FMA-pipe
// efficiency from the rest of the step (modulation, demod, barriers, TMA).
#include <cstdio>
#include <cstring>
#include "../paper_1603_08081_b200/csrc/fbf_fused.cuh"

using namespace fbf;
template <class C, int SYNC>
__global__ void __launch_bounds__(C::NT, 1) fir(const __grid_constant__ FusedArgs A, int iters, long long* cyc,
                                              float* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  p2* M = reinterpret_cast<p2*>(smem + C::OFF_M);
  p2* R = reinterpret_cast<p2*>(smem + C::OFF_R);
  float* CS = reinterpret_cast<float*>(smem + C::OFF_CS);
  for (int i = threadIdx.x; i < 2 * C::G * C::MP; i += blockDim.x) M[i] = pk(1.0f + i * 1e-6f, 0.5f);
  __syncthreads();
  Pending<C> pd;
  pd.nh = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    row_pass<C>(A, M, R, CS, it * C::G, C::G, 0, pd);
    if (SYNC) __syncthreads();
    else asm volatile("" ::: "memory");
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = CS[threadIdx.x] + __uint_as_float(static_cast<unsigned>(R[threadIdx.x]));
}

template <class C, int SYNC>
void run(const FusedArgs& a, int sms, int per_sm) {
  long long* cyc;
  float* out;
  cudaMalloc(&cyc, sms * sizeof(long long));
  cudaMalloc(&out, sms * per_sm * C::NT * sizeof(float));
  cudaFuncSetAttribute(fir<C, SYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes);
  const int iters = 2000;
  fir<C, SYNC><<<sms * per_sm, C::NT, C::smem_bytes>>>(a, 10, cyc, out);
  fir<C, SYNC><<<sms * per_sm, C::NT, C::smem_bytes>>>(a, iters, cyc, out);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[4096];
  cudaMemcpy(h, cyc, sms * per_sm * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < sms * per_sm; i++) mx = h[i] > mx ? h[i] : mx;
  // FMA-pipe cycles per SMSP per row pass: 2 warps x 16 outputs x 31 taps x FFMA2 (2 cycles)
  const double ideal = (C::NT / 128.0) * per_sm * C::KR * (2 * C::W + 1) * 2;
  printf("NT=%d G=%d x%d/SM sync=%d: %.0f cycles/pass, FIR-only FMA efficiency %.1f%% (%s)\n", C::NT, C::G, per_sm, SYNC, double(mx) / iters,
         100.0 * ideal / (double(mx) / iters), cudaGetErrorString(e));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  FusedArgs a;
  memset(&a, 0, sizeof(a));
  a.k.W = 15;
  for (int i = 0; i <= 15; i++) a.k.t[i] = 1.0f / (1 + i);
  using Big = FusedCfg<15, 64, 32, 16, 16, 256, false>;
  using Small = FusedCfg<15, 64, 16, 16, 16, 128, false>;
  run<Big, 1>(a, sms, 1);
  run<Big, 0>(a, sms, 1);
  run<Small, 1>(a, sms, 1);
  run<Small, 1>(a, sms, 2);
  run<Small, 0>(a, sms, 2);
  return 0;
}
