// TMA / cp.async latency-throughput probe for the fused kernel's tile shape:
// every CTA (one per SM) repeatedly loads a G x MW tile of 8-byte elements
// from an L2-resident 2-D array into shared memory and times each load.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_1603_08081_b200/csrc/fbf_device.cuh"

using namespace fbf;

__global__ void tma_probe(const __grid_constant__ CUtensorMap tm, int iters, int rows_total, int G, int MW,
                          long long* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned ph = 0;
  long long total = 0;
  for (int it = 0; it < iters; ++it) {
    const int row = (blockIdx.x * 37 + it * 32) % (rows_total - G);
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, G * MW * 8);
      tma_load_3d(smem, &tm, bar, (blockIdx.x % 16) * 64, row, 0);
    }
    mbar_wait(bar, ph);
    ph ^= 1;
    total += clock64() - t0;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = total / iters;
}

__global__ void tma_probe_busy(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm2,
                               int iters, int rows_total, int G, int MW, long long* out, unsigned long long* wbuf,
                               int mode) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned ph = 0;
  long long total = 0;
  for (int it = 0; it < iters; ++it) {
    const int row = (blockIdx.x * 37 + it * 32) % (rows_total - G);
    // STG traffic like the (Q, P) write-back: 8 x 8 B per thread, rows 16 KB apart
    if (mode & 1)
      for (int i = 0; i < 8; ++i)
        wbuf[(size_t)((row + i + 1000) % 2048) * 2048 + (blockIdx.x % 32) * 64 + (threadIdx.x & 63) +
             (threadIdx.x >> 6) * 8 * 2048] = it;
    __syncthreads();
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, G * MW * 8);
      tma_load_3d(smem, &tm, bar, (blockIdx.x % 16) * 64, row, 0);
      if (mode & 2) {
        mbar_expect_tx(bar + 1, 32 * 64 * 8);
        tma_load_3d(smem + 100 * 1024, &tm2, bar + 1, (blockIdx.x % 32) * 64, (row + 500) % 2000, 0);
      }
    }
    mbar_wait(bar, ph);
    total += clock64() - t0;
    if (mode & 2) mbar_wait(bar + 1, ph);
    ph ^= 1;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = total / iters;
}

__global__ void ldgsts_probe(const int2* src, long long pitch, int iters, int rows_total, int G, int MW,
                             long long* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  int2* st = reinterpret_cast<int2*>(smem);
  long long total = 0;
  for (int it = 0; it < iters; ++it) {
    const int row = (blockIdx.x * 37 + it * 32) % (rows_total - G);
    const int2* base = src + row * pitch + (blockIdx.x % 16) * 64;
    const long long t0 = clock64();
    const int pairs = MW / 2;
    for (int e = threadIdx.x; e < G * pairs; e += blockDim.x) {
      const int g = e / pairs, q = e - g * pairs;
      cp_async16(st + g * MW + 2 * q, base + g * pitch + 2 * q);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    total += clock64() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = total / iters;
}

int main() {
  const int cols = 2078, rows = 2078;
  int2* buf;
  cudaMalloc(&buf, sizeof(int2) * cols * rows);
  cudaMemset(buf, 1, sizeof(int2) * cols * rows);
  long long* out;
  cudaMalloc(&out, 148 * sizeof(long long));
  std::vector<long long> h(148);
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Fn enc = reinterpret_cast<Fn>(p);
  cudaFuncSetAttribute(tma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  cudaFuncSetAttribute(ldgsts_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  const int shapes[][2] = {{32, 94}, {16, 94}, {32, 64}, {32, 112}, {8, 94}, {64, 94}};
  for (auto& s : shapes) {
    const int G = s[0], MW = s[1];
    for (int variant = 0; variant < 4; ++variant) {
      CUtensorMap tm;
      const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 1};
      const cuuint64_t strides[2] = {(cuuint64_t)cols * 8, (cuuint64_t)cols * rows * 8};
      const cuuint32_t box[3] = {(cuuint32_t)MW, (cuuint32_t)G, 1};
      const cuuint32_t es[3] = {1, 1, 1};
      const CUtensorMapL2promotion promo = variant == 1 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                                        : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, buf, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", r);
        continue;
      }
      const int grid = variant == 3 ? 1 : 148;
      if (variant <= 1 || variant == 3)
        tma_probe<<<grid, 256, 210 * 1024>>>(tm, 50, rows, G, MW, out);
      else
        ldgsts_probe<<<grid, 256, 210 * 1024>>>(buf, cols, 50, rows, G, MW, out);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h.data(), out, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0, sum = 0;
      for (int i = 0; i < grid; ++i) {
        mx = h[i] > mx ? h[i] : mx;
        sum += h[i];
      }
      const char* names[4] = {"TMA(promo256)", "TMA(nopromo)", "LDGSTS16", "TMA 1 CTA"};
      printf("G=%2d MW=%3d %-14s avg %6lld max %6lld cycles per %6d-byte tile  (%s)\n", G, MW, names[variant],
             sum / grid, mx, G * MW * 8, cudaGetErrorString(e));
    }
  }
  // kernel-like conditions: concurrent (Q, P)-shaped TMA and STG write-back
  {
    unsigned long long* wbuf;
    cudaMalloc(&wbuf, 2048ull * 2048 * 8);
    CUtensorMap tm, tm2;
    const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 1};
    const cuuint64_t strides[2] = {(cuuint64_t)cols * 8, (cuuint64_t)cols * rows * 8};
    const cuuint32_t box[3] = {94, 32, 1};
    const cuuint64_t dims2[3] = {2048, 2048, 1};
    const cuuint64_t strides2[2] = {2048 * 8, 2048ull * 2048 * 8};
    const cuuint32_t box2[3] = {64, 32, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tm2, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, wbuf, dims2, strides2, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(tma_probe_busy, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    for (int mode = 0; mode < 4; ++mode) {
      tma_probe_busy<<<148, 256, 210 * 1024>>>(tm, tm2, 50, rows, 32, 94, out, wbuf, mode);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h.data(), out, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0, sum = 0;
      for (int i = 0; i < 148; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
      printf("busy mode %d (1=STG,2=2nd TMA) avg %6lld max %6lld  (%s)\n", mode, sum / 148, mx, cudaGetErrorString(e));
    }
  }
  return 0;
}
