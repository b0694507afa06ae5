// FFMA2 issue rate vs resident warps per SM sub-partition: how many warps
// does the FIR need to keep the FP32 pipe busy?  One CTA per SM, 32*4*w threads.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(float* out, float a, float b, int iters, long long* cycles) {
  unsigned long long acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) {
    float2 v = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
    acc[i] = *reinterpret_cast<unsigned long long*>(&v);
  }
  float2 fa = make_float2(a, a), fb = make_float2(b, b);
  unsigned long long y = *reinterpret_cast<unsigned long long*>(&fa);
  unsigned long long z = *reinterpret_cast<unsigned long long*>(&fb);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(y), "l"(z));
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += reinterpret_cast<float2*>(&acc[i])->x;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sms * 1024 * sizeof(float));
  cudaMalloc(&cyc, sms * sizeof(long long));
  long long h[1024];
  for (int w = 1; w <= 8; w *= 2) {
    const int threads = 128 * w, iters = 4000;
    probe<<<sms, threads>>>(out, 1.0001f, 0.5f, 10, cyc);
    probe<<<sms, threads>>>(out, 1.0001f, 0.5f, iters, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < sms; i++) mx = h[i] > mx ? h[i] : mx;
    const double lane_ops = double(threads) * iters * 16 * 2;
    printf("warps/SMSP %d: %.1f lane-ops/clk/SM (FFMA2 issue every %.2f clk per SMSP)\n", w, lane_ops / mx,
           double(mx) / (double(iters) * 16 * w));
  }
  return 0;
}
