// race_common.cuh -- shared device helpers for the RACE attention kernels.
//
// Math (see DESIGN.md and SURVEY Appendix A, verified against the reference):
//   x^ = x / ||x||   (rows with ||x|| < 1e-12 pass through; ra/core.py:114-123)
//   u_j = tanh(x^ . w_j)                     j = table*P + p  (ra/sketch.py:109)
//   phi_r (table tau) = softmax_r(beta * sum_p u_p c_rp),
//       c_rp = +1 if bit p of r is 0 else -1   (ra/sketch.py:52-74, 111-118)
//     = prod_p [match ? 1 : e_p] / prod_p (1 + e_p),  e_p = exp(-2 beta |u_p|)
//   which is exactly the max-subtracted softmax of the reference (the max
//   logit is the sign-matching corner) and the factored form of
//   ra/sketch.py:120-129, so one code path covers every P.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace race {

constexpr float kZeroRowEps = 1e-12f;       // ra/core.py:15
constexpr float kDegenerateDenEps = 1e-30f; // ra/core.py:19
constexpr int kPMax = 10;                   // corner-softmax width handled in registers

__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Corner probabilities of one table from its P tanh-projections.
// phi[r] for r < 2^P is written with stride 1.
__device__ __forceinline__ void corner_softmax(const float* u, int P, float beta, float* phi_out) {
  float e[kPMax];
  float z = 1.f;
#pragma unroll
  for (int p = 0; p < kPMax; ++p) {
    if (p < P) {
      e[p] = expf(-2.f * beta * fabsf(u[p]));
      z *= 1.f + e[p];
    }
  }
  const float rz = 1.f / z;
  const int R = 1 << P;
  for (int r = 0; r < R; ++r) {
    float prod = rz;
#pragma unroll
    for (int p = 0; p < kPMax; ++p) {
      if (p < P) {
        const bool neg_corner = (r >> p) & 1;      // c_rp = -1
        const bool u_neg = u[p] < 0.f;
        prod *= (neg_corner == u_neg) ? 1.f : e[p];
      }
    }
    phi_out[r] = prod;
  }
}

// numerically stable logistic sigma(z) (ra/sketch.py:77-84)
__device__ __forceinline__ float sigmoid_pos(float z) {
  const float e = expf(-fabsf(z));
  return z >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
}

// one bit's factor of the factored corner probability (ra/sketch.py:120-129):
// sigma(2 beta c u) with c = -1 if neg_corner else +1, written as match ? 1/(1+e) : e/(1+e),
// e = exp(-2 beta |u|) (the same form corner_softmax uses, so grouped and ungrouped agree)
__device__ __forceinline__ float corner_factor(float u, int64_t neg_corner, float beta) {
  const float e = expf(-2.f * beta * fabsf(u));
  const bool match = (neg_corner != 0) == (u < 0.f);
  return (match ? 1.f : e) / (1.f + e);
}

}  // namespace race
