// TMA streaming ceiling on this B200: persistent CTAs (one per SM) read
// [BH, N, 128] bf16 tensors in the fast-path tile pattern (128 tokens x 64
// columns per box, two boxes per tile) through an S-stage mbarrier pipeline
// and do nothing else.  Reports GB/s for 1..4 tensors and stage counts, i.e.
// the bandwidth the RACE kernels' load pattern can reach at best.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include \
//        -I../../paper_2510_04008_b200/csrc tma_stream.cu -o tma_stream -lcuda
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace race::tc;

constexpr int TILE = 32768, SUB = 16384;

template <int NT, int NW>
__global__ void __launch_bounds__(64, 1) k_stream(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                                                  const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m3,
                                                  const __grid_constant__ CUtensorMap mo,
                                                  int chunks_per_bh, int bh_count, int stages, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * NT * TILE);
  uint64_t* empty = full + 8;
  const CUtensorMap* maps[4] = {&m0, &m1, &m2, &m3};
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int total = chunks_per_bh * bh_count;
  const int c0 = int(int64_t(blockIdx.x) * total / gridDim.x), c1 = int(int64_t(blockIdx.x + 1) * total / gridDim.x);
  if (threadIdx.x == 0) {  // producer
    for (int c = c0, g = 0; c < c1; ++c, ++g) {
      const int s = g % stages;
      mbar_wait(&empty[s], ((g / stages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], NT * TILE);
      const int bh = c / chunks_per_bh, t = (c % chunks_per_bh) * 128;
      for (int k = 0; k < NT; ++k)
        for (int h = 0; h < 2; ++h)
          tma_load_3d(smem + (s * NT + k) * TILE + h * SUB, maps[k], &full[s], h * 64, t, bh, policy_evict_first());
    }
  } else if (threadIdx.x == 32) {  // consumer: touch one word, store NW tiles back (TMA), release the stage
    float acc = 0.f;
    for (int c = c0, g = 0; c < c1; ++c, ++g) {
      const int s = g % stages;
      mbar_wait(&full[s], (g / stages) & 1);
      acc += *reinterpret_cast<const float*>(smem + s * NT * TILE + (g & 255) * 16);
      if (NW) {
        const int bh = c / chunks_per_bh, t = (c % chunks_per_bh) * 128;
        for (int h = 0; h < 2; ++h) tma_store_3d(&mo, smem + s * NT * TILE + h * SUB, h * 64, t, bh);
        tma_store_commit();
        tma_store_wait_read<0>();
      }
      mbar_arrive(&empty[s]);
    }
    if (NW) tma_store_wait_all<0>();
    if (acc == 12345.f) *sink = acc;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

int main() {
  const int BH = 4, N = 131072 * 4;  // 4 x 512K tokens x 128 x bf16 = 512 MiB per tensor
  const size_t bytes = size_t(BH) * N * 128 * 2;
  void* buf[5];
  for (auto& b : buf) { cudaMalloc(&b, bytes); cudaMemset(b, 1, bytes); }
  float* sink;
  cudaMalloc(&sink, 4);
  CUtensorMap m[5];
  for (int i = 0; i < 5; ++i) {
    cuuint64_t dims[3] = {128, cuuint64_t(N), cuuint64_t(BH)};
    cuuint64_t strides[2] = {256, cuuint64_t(N) * 256};
    cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
    enc()(&m[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf[i], dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, int nt, int nw, int stages) {
    const int smem = stages * nt * TILE + 256;
    if (smem > 232448) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = sms;
    for (int w = 0; w < 2; ++w) kern<<<grid, 64, smem>>>(m[0], m[1], m[2], m[3], m[4], N / 128, BH, stages, sink);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int w = 0; w < reps; ++w) kern<<<grid, 64, smem>>>(m[0], m[1], m[2], m[3], m[4], N / 128, BH, stages, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = double(nt + nw) * bytes * reps / (ms / 1e3) / 1e9;
    printf("read %d write %d stages %d (%3d KB/CTA): %7.1f GB/s (read+write)  %s\n", nt, nw, stages, stages * nt * 32, gbs,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int stages = 1; stages <= 3; ++stages) {
    run(k_stream<2, 0>, 2, 0, stages);
    run(k_stream<2, 1>, 2, 1, stages);
    run(k_stream<3, 1>, 3, 1, stages);
    run(k_stream<4, 1>, 4, 1, stages);
    run(k_stream<2, 2>, 2, 2, stages);
  }
  return 0;
}
