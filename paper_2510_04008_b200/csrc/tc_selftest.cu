// tc_selftest.cu -- on-device check of the UMMA operand layouts / descriptors
// used by the fast path (built as a separate diagnostic library,
// libtc_selftest.so, exercised by tests/test_tc_selftest.py).
//
// One CTA: A [M x K] and B [N x K] (row-major bf16 in global memory) are
// written into shared memory in the canonical layout selected by
// (major, swizzle), one tcgen05.mma chain computes D = A B^T into TMEM, and
// D is read back with tcgen05.ld.  The host compares with torch.
#include <cstdio>

#include "tc_common.cuh"

using namespace race::tc;

namespace {

__device__ uint32_t swz_rt(uint32_t off, int sw_bytes) {
  const uint32_t mask = sw_bytes == 128 ? 7 : sw_bytes == 64 ? 3 : sw_bytes == 32 ? 1 : 0;
  return off ^ (((off >> 7) & mask) << 4);
}

// byte offset of element (mn, k) of an [MN x K] operand tile
__device__ uint32_t canon_off(int mn, int k, int MN, int K, int mn_major, int sw) {
  if (!mn_major) {
    const int per_row = sw / 2;  // elements of K per swizzle row
    const int blk = k / per_row, kin = k % per_row;
    const uint32_t off = uint32_t(blk) * MN * sw + uint32_t(mn / 8) * (8 * sw) + (mn % 8) * sw + kin * 2;
    return swz_rt(off, sw);
  }
  const int per_row = sw / 2;  // elements of MN per swizzle row
  const int blk = mn / per_row, mnin = mn % per_row;
  const uint32_t off = uint32_t(blk) * K * sw + uint32_t(k / 8) * (8 * sw) + (k % 8) * sw + mnin * 2;
  return swz_rt(off, sw);
}

__device__ uint64_t operand_desc(uint32_t base, int kk, int MN, int K, int mn_major, int sw) {
  const uint32_t layout = sw == 128 ? kSw128 : sw == 64 ? kSw64 : kSw32;
  if (!mn_major) {
    const int per_row = sw / 2;
    const int k0 = kk * 16;
    const uint32_t start = base + uint32_t(k0 / per_row) * MN * sw + (k0 % per_row) * 2;
    return smem_desc(start, 16, 8 * sw, layout);
  }
  const uint32_t start = base + uint32_t(kk) * 2 * (8 * sw);
  return smem_desc(start, uint32_t(K) * sw, 8 * sw, layout);
}

__global__ void __launch_bounds__(128) k_selftest(int M, int N, int K, int a_mn, int b_mn, int a_sw, int b_sw,
                                                  const __nv_bfloat16* __restrict__ A,
                                                  const __nv_bfloat16* __restrict__ B, float* __restrict__ D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;                    // up to 32 KB
  uint8_t* sb = smem + 32768;            // up to 32 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 65536 + 64);
  const int tid = threadIdx.x, warp = tid >> 5;

  for (int i = tid; i < 65536 / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const bool a_tmem = a_sw == 0;  // A from TMEM (columns 128.. of the allocation)
  if (!a_tmem) {
    for (int i = tid; i < M * K; i += 128) {
      const int m = i / K, k = i % K;
      *reinterpret_cast<__nv_bfloat16*>(sa + canon_off(m, k, M, K, a_mn, a_sw)) = A[i];
    }
  }
  for (int i = tid; i < N * K; i += 128) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sb + canon_off(n, k, N, K, b_mn, b_sw)) = B[i];
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(tslot);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (a_tmem) {  // thread = row: pack row tid of A into 32-bit cells (k even in the low half)
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t u[16];
      for (int j = 0; j < 16; ++j) {
        const int k = 2 * (c0 + j);
        const __nv_bfloat16 lo = k < K ? A[tid * K + k] : __float2bfloat16(0.f);
        const __nv_bfloat16 hi = k + 1 < K ? A[tid * K + k + 1] : __float2bfloat16(0.f);
        u[j] = uint32_t(*reinterpret_cast<const unsigned short*>(&lo)) |
               (uint32_t(*reinterpret_cast<const unsigned short*>(&hi)) << 16);
      }
      tmem_st16u(tmem + (uint32_t(warp * 32) << 16) + 128 + c0, u);
    }
    tmem_st_wait();
    tc_fence_before();
  }
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16(M, N, a_tmem ? 0 : a_mn, b_mn);
    for (int kk = 0; kk < K / 16; ++kk) {
      if (a_tmem)
        umma_bf16_ts(tmem, tmem + 128 + kk * 8, operand_desc(smem_u32(sb), kk, N, K, b_mn, b_sw), idesc, kk > 0);
      else
        umma_bf16(tmem, operand_desc(smem_u32(sa), kk, M, K, a_mn, a_sw),
                  operand_desc(smem_u32(sb), kk, N, K, b_mn, b_sw), idesc, kk > 0);
    }
    umma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + c0, v);
    tmem_ld_wait();
    if (row < M)
      for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}


// M = 64 MMAs on the half-subpartition TMEM layout (row 16q + i of the accumulator in DP 32q + i):
// chain 0 writes D at DP offset 0 and chain 1 at DP offset 16 of the SAME columns, each with its own
// A ([64 x K] K-major SW128 in smem, or in TMEM for ts = 1 at the chain's DP offset) and a shared B
// ([N x K] K-major SW128).  D rows 0..63 = chain 0, 64..127 = chain 1.  This is the layout two
// independent 64-token chains per CTA would use.
__global__ void __launch_bounds__(128) k_selftest_m64(int N, int K, int ts, const __nv_bfloat16* __restrict__ A,
                                                      const __nv_bfloat16* __restrict__ B, float* __restrict__ D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa0 = smem;            // 16 KB each
  uint8_t* sa1 = smem + 16384;
  uint8_t* sb = smem + 32768;     // up to 32 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 65536 + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 65536 / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  for (int i = tid; i < 128 * K; i += 128) {
    const int m = i / K, k = i % K;
    uint8_t* base = m < 64 ? sa0 : sa1;
    *reinterpret_cast<__nv_bfloat16*>(base + canon_off(m & 63, k, 64, K, 0, 128)) = A[i];
  }
  for (int i = tid; i < N * K; i += 128) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sb + canon_off(n, k, N, K, 0, 128)) = B[i];
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(tslot);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // the accumulator row of this thread's DP: chain (lane >= 16), row 16 * warp + lane % 16
  const int chain = lane >> 4, row = chain * 64 + warp * 16 + (lane & 15);
  if (ts) {  // A in TMEM columns 128.. at the same DP as its accumulator row
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t u[16];
      for (int j = 0; j < 16; ++j) {
        const int k = 2 * (c0 + j);
        const __nv_bfloat16 lo = k < K ? A[row * K + k] : __float2bfloat16(0.f);
        const __nv_bfloat16 hi = k + 1 < K ? A[row * K + k + 1] : __float2bfloat16(0.f);
        u[j] = uint32_t(*reinterpret_cast<const unsigned short*>(&lo)) |
               (uint32_t(*reinterpret_cast<const unsigned short*>(&hi)) << 16);
      }
      tmem_st16u(tmem + (uint32_t(warp * 32) << 16) + 128 + c0, u);
    }
    tmem_st_wait();
    tc_fence_before();
  }
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16(64, N, 0, 0);
    for (int ch = 0; ch < 2; ++ch) {
      const uint32_t doff = uint32_t(16 * ch) << 16;
      for (int kk = 0; kk < K / 16; ++kk) {
        if (ts)
          umma_bf16_ts(tmem + doff, tmem + doff + 128 + kk * 8, operand_desc(smem_u32(sb), kk, N, K, 0, 128), idesc,
                       kk > 0);
        else
          umma_bf16(tmem + doff, operand_desc(smem_u32(ch ? sa1 : sa0), kk, 64, K, 0, 128),
                    operand_desc(smem_u32(sb), kk, N, K, 0, 128), idesc, kk > 0);
      }
    }
    umma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + c0, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

}  // namespace

extern "C" int tc_selftest_m64(int N, int K, int ts, const void* A, const void* B, float* D, void* stream) {
  if (N % 16 || N < 16 || N > 128 || K % 64 || K > 128) return 1;
  const size_t smem = 65536 + 128;
  cudaFuncSetAttribute(k_selftest_m64, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_selftest_m64<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(N, K, ts, static_cast<const __nv_bfloat16*>(A),
                                                                     static_cast<const __nv_bfloat16*>(B), D);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "tc_selftest_m64 launch: %s\n", cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

namespace {

// Layout probe of the 16-lane TMEM load shapes: TMEM cell (dp, col) is filled with dp * 1024 + col
// by 32x32b stores, then every warp reads its quarter's first 16 DPs (lane offset 0) or second 16
// (offset 16) with tcgen05.ld.16x64b.x8 / 16x128b.x4 / 16x256b.x2 (8 registers per thread each)
// and records what each thread's register holds: out[warp][thread][reg].
template <int SHAPE>
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t* r) {
  if constexpr (SHAPE == 64)
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
  else if constexpr (SHAPE == 128)
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
  else
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}

__global__ void __launch_bounds__(128) k_ld16_probe(int shape, int lane_off, uint32_t* out) {
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<64>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t dp = warp * 32 + lane;
  for (int c0 = 0; c0 < 64; c0 += 16) {
    uint32_t u[16];
    for (int j = 0; j < 16; ++j) u[j] = dp * 1024 + c0 + j;
    tmem_st16u(tmem + (uint32_t(warp * 32) << 16) + c0, u);
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t r[8];
  const uint32_t addr = tmem + (uint32_t(warp * 32 + lane_off) << 16);
  if (shape == 64) ld16<64>(addr, r);
  else if (shape == 128) ld16<128>(addr, r);
  else ld16<256>(addr, r);
  tmem_ld_wait();
  for (int j = 0; j < 8; ++j) out[(warp * 32 + lane) * 8 + j] = r[j];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(tmem);
}

}  // namespace

extern "C" int tc_ld16_probe(int shape, int lane_off, uint32_t* out, void* stream) {
  k_ld16_probe<<<1, 128, 0, static_cast<cudaStream_t>(stream)>>>(shape, lane_off, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

namespace {
}  // namespace

extern "C" int tc_selftest_gemm(int M, int N, int K, int a_mn, int b_mn, int a_sw, int b_sw, const void* A,
                                const void* B, float* D, void* stream) {
  if (M != 128 || N % 16 || N < 16 || N > 128 || K % 16 || K > 128) return 1;
  if (M * K * 2 > 32768 || N * K * 2 > 32768) return 1;
  const size_t smem = 65536 + 128;
  cudaFuncSetAttribute(k_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_selftest<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(M, N, K, a_mn, b_mn, a_sw, b_sw,
                                                                 static_cast<const __nv_bfloat16*>(A),
                                                                 static_cast<const __nv_bfloat16*>(B), D);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "tc_selftest launch: %s\n", cudaGetErrorString(e));
    return 3;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Throughput probes (tools/tmem_probe.py): how fast one SM reads TMEM with tcgen05.ld and how many
// cycles one tcgen05.mma of the shapes the causal kernels issue takes, A from shared memory (SS) or
// from TMEM (TS).  Results (cycles) go to out[]; nothing here is on the library's hot path.
// ---------------------------------------------------------------------------
namespace {

__global__ void k_tmem_ld_rate(int iters, long long* out) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
  const uint32_t col0 = uint32_t(warp >> 2) * 32 % 512;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    float v0[32], v1[32];
    tmem_ld32(tmem + lane_base + ((col0 + 64 * (i & 3)) & 511), v0);
    tmem_ld32(tmem + lane_base + ((col0 + 64 * (i & 3) + 32) & 511), v1);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += v0[j] + v1[j];
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) out[gridDim.x] = 1;  // keep the loads live
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// n_mma tcgen05.mma of M = 128, N = n, K = 16 (bf16) per round, `rounds` rounds, each ended by a commit and
// its mbarrier wait; ts: A from TMEM (columns 256..) instead of shared memory
__global__ void k_mma_rate(int n, int ts, int n_mma, int rounds, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t idesc = idesc_bf16(128, n, 0, 0);
  long long t = 0;
  if (warp == 0) {
    const uint64_t da = smem_desc(base, 16, 1024, 2), db = smem_desc(base + 32768, 16, 1024, 2);
    for (int rd = 0; rd < rounds; ++rd) {
      const long long t0 = clock64();
      if (threadIdx.x == 0) {
        for (int i = 0; i < n_mma; ++i) {
          if (ts)
            umma_bf16_ts(tmem, tmem + 256 + (i & 7) * 8, db, idesc, 1u);
          else
            umma_bf16(tmem, da, db, idesc, 1u);
        }
        umma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, rd & 1);
      if (rd > 0) t += clock64() - t0;  // the first round warms up
    }
    if (threadIdx.x == 0) out[0] = t / (rounds - 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

}  // namespace

// cycles of `iters` x (two 32-column tcgen05.ld per warp) with `warps` warps (multiple of 4) per CTA
extern "C" int tc_tmem_ld_rate(int ctas, int warps, int iters, long long* out, void* stream) {
  k_tmem_ld_rate<<<ctas, 32 * warps, 0, static_cast<cudaStream_t>(stream)>>>(iters, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
// cycles per round of n_mma MMAs (M = 128, N = n, K = 16)
extern "C" int tc_mma_rate(int n, int ts, int n_mma, int rounds, long long* out, void* stream) {
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(k_mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_mma_rate<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(n, ts, n_mma, rounds, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
