// FP32 FMA-pipe throughput probe for the roofline denominator (SURVEY.md §8(d):
// "re-derive the FP32 peak from a measured FFMA microbenchmark on the box").
// Measures warp-instruction throughput of FFMA (register / uniform operand)
// and FFMA2 (fma.rn.f32x2), reporting lane-ops per SM-clock and per second.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) probe(float* out, float a, float b, int iters,
                                            long long* cycles) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = threadIdx.x * 0.001f + i;
  float ra = a + threadIdx.x * 1e-9f, rb = b - threadIdx.x * 1e-9f;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    if (MODE == 0) {  // FFMA, 3 registers
#pragma unroll
      for (int i = 0; i < 16; i++) acc[i] = fmaf(acc[i], ra, rb);
    } else if (MODE == 1) {  // FFMA, uniform (kernel-param) operands
#pragma unroll
      for (int i = 0; i < 16; i++) acc[i] = fmaf(acc[i], a, b);
    } else {  // FFMA2 on pairs, uniform operands
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        unsigned long long x, r, y, z;
        float2 va = make_float2(acc[i], acc[i + 1]);
        x = *reinterpret_cast<unsigned long long*>(&va);
        float2 fa = MODE == 2 ? make_float2(a, a) : make_float2(ra, ra);
        float2 fb = MODE == 2 ? make_float2(b, b) : make_float2(rb, rb);
        y = *reinterpret_cast<unsigned long long*>(&fa);
        z = *reinterpret_cast<unsigned long long*>(&fb);
        asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(y), "l"(z));
        va = *reinterpret_cast<float2*>(&r);
        acc[i] = va.x;
        acc[i + 1] = va.y;
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int sms) {
  const int blocks = sms * 4, threads = 256, iters = 20000;
  float* out;
  long long* cyc;
  cudaMalloc(&out, blocks * threads * sizeof(float));
  cudaMalloc(&cyc, blocks * sizeof(long long));
  probe<MODE><<<blocks, threads>>>(out, 1.0001f, 0.5f, 100, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<MODE><<<blocks, threads>>>(out, 1.0001f, 0.5f, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < blocks; i++) mx = h[i] > mx ? h[i] : mx;
  double ops = double(blocks) * threads * iters * 16;
  // 4 blocks/SM co-resident: per-SM ops = ops/sms over mx cycles
  printf("%-22s %.3f ms  %.2f Tops/s  %.1f lane-ops/clk/SM  (clk %.0f MHz)\n", name, ms,
         ops / ms / 1e9, ops / sms / mx, mx / (ms * 1e3));
  cudaFree(out);
  cudaFree(cyc);
  delete[] h;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  for (int r = 0; r < 2; r++) {
    run<0>("FFMA reg", sms);
    run<1>("FFMA uniform", sms);
    run<2>("FFMA2 uniform", sms);
    run<3>("FFMA2 reg", sms);
  }
  return 0;
}
