// TMEM read throughput on this B200: W warps per CTA (one CTA per SM) repeatedly read
// 32 lanes x 32 columns (tcgen05.ld 32x32b.x32) and wait, like the RACE compute phases.
// Reports bytes per cycle per SM for W = 1, 4, 8 warps.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include \
//        -I../../paper_2510_04008_b200/csrc tmem_read.cu -o tmem_read
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace race::tc;

__global__ void __launch_bounds__(512, 1) k_read(int iters, int batch, float* sink, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lb = uint32_t((warp & 3) * 32) << 16;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    float v[32];
    for (int b = 0; b < batch; ++b) {  // `batch` loads in flight before one wait
      tmem_ld32(tmem + lb + (((i * batch + b) * 32 + warp * 64) & 511), v);
    }
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += v[j];
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  float* sink;
  long long* cyc;
  cudaMalloc(&sink, 148 * 512 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int iters = 4096;
  for (int warps : {1, 4, 8, 16}) {
    for (int batch : {1, 2, 4}) {
      k_read<<<148, warps * 32>>>(iters, batch, sink, cyc);
      cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (long long x : h) mx = x > mx ? x : mx;
      const double bytes = double(warps) * iters * batch * 32 * 32 * 4;
      printf("warps %2d batch %d: %.1f B/cycle/SM, %.0f cycles per 4 KB load round per warp\n", warps, batch,
             bytes / mx, double(mx) / (iters * batch));
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
