// race_internal.h -- geometry shared by the C-ABI layer and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace race {

// Element strides of one [B, H, N, width] operand (row elements contiguous): token, head, batch.
// token == 0 means the contiguous [B*H, N, width] layout.
struct Lay {
  int64_t token = 0, head = 0, batch = 0;
};
enum LayIdx { L_Q = 0, L_K, L_V, L_O, L_DO, L_DQ, L_DK, L_DV, L_COUNT };

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
  // corner groups (race_abi.cu, P > 10 or one table beyond one pass): a sub-problem of ONE table
  // whose kernels see only the 2^cb corners r = (chi << cb) | lo, lo < 2^cb.  phi_r is the factored
  // product over all P bits (ra/sketch.py:120-129): the low cb bits vary per corner, the high bits
  // are fixed to chi and contribute one per-row factor.  cb = 0: ungrouped (all P bits).
  int cb = 0;
  int64_t chi = 0;
  // grouped tcgen05 backward (race_abi.cu): the query / key backward kernels write (corner groups:
  // add) each row's dproj_j, j < T*P, into [BH*N, dproj_ld] fp32 at column dproj_col instead of
  // storing dq / dk; one pass at the end turns the summed dproj into dq, dk (dx^ = dproj . W)
  float* dproj_q = nullptr;
  float* dproj_k = nullptr;
  int dproj_ld = 0, dproj_col = 0, dproj_acc = 0;
  // strided operands (race_fwd_layout / race_bwd_layout, tcgen05 path only): e.g. [B, N, H, d] views
  Lay lay[L_COUNT];
  bool strided() const {
    for (const Lay& l : lay)
      if (l.token) return true;
    return false;
  }
};

// corners per table a kernel pass sees
__host__ __device__ inline int pass_corner_bits(const Geo& g) { return g.cb ? g.cb : g.P; }

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
// pad > 0: also zero the `pad` floats after the BH * nseg * E outputs (the causal state's alignment gap, so
// the state is bitwise deterministic; only when `out` is a race_fwd state)
cudaError_t combine(const Geo& g, int mode, const float* part, const float* carry, float* out, cudaStream_t st,
                    int pad = 0);

}  // namespace race
