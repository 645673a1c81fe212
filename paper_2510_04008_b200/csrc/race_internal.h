// race_internal.h -- geometry shared by the C-ABI layer and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace race {

// Resolved problem geometry (validated copy of race_desc_t + segmentation).
struct Geo {
  int64_t BH, H, N;
  int d, dv, P, T;
  float beta;
  int normalize, w_per_head, dtype, causal;
  int64_t nseg, seg_tokens;
  // table groups (race_abi.cu): per-token 1/D and -(dO.O)/D of the WHOLE estimator, [BH, Np];
  // when set, the generic backward kernels use them instead of their own group's D and O
  const float* ext_rden = nullptr;
  const float* ext_gden = nullptr;
};

// every kernel launch in the library bumps this (race_launch_count)
void note_launch(int n = 1);

// generic CUDA-core kernels (race_simt.cu)
size_t simt_max_smem(const Geo& g);
cudaError_t simt_aggregate(const Geo& g, const void* k, const void* v, const float* w, float* part, cudaStream_t st);
cudaError_t simt_readout(const Geo& g, const void* q, const float* w, const float* tab, void* o, float* den,
                         cudaStream_t st);
cudaError_t simt_causal_fwd(const Geo& g, const void* q, const void* k, const void* v, const float* w,
                            const float* car, void* o, float* den, float* nrm, cudaStream_t st);
cudaError_t simt_bwd_q(const Geo& g, const void* q, const void* d_o, const float* w, const float* tab, void* dq,
                       float* dpart, cudaStream_t st);
cudaError_t simt_bwd_k(const Geo& g, const void* k, const void* v, const float* w, const float* dtab, void* dk,
                       void* dv, cudaStream_t st);
cudaError_t simt_bwd_causal_q(const Geo& g, const void* q, const void* k, const void* v, const void* d_o,
                              const float* w, const float* car, void* dq, float* rden, float* gden, float* dpart,
                              cudaStream_t st);
cudaError_t simt_bwd_causal_k(const Geo& g, const void* q, const void* k, const void* v, const void* d_o,
                              const float* w, const float* rden, const float* gden, const float* dcar, void* dk,
                              void* dv, cudaStream_t st);
cudaError_t combine(const Geo& g, int mode, const float* part, const float* carry, float* out, cudaStream_t st);

}  // namespace race
