// tc_fast.cuh -- shared pieces of the sm_100a fast-path kernels (race_tc.cu,
// race_tc_bwd.cu): geometry, work items, UMMA descriptors for the fixed
// operand layouts, and the per-row feature / VJP math of the compute warps.
#pragma once

#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <unordered_map>

#include "race_common.cuh"
#include "race_internal.h"
#include "tc_common.cuh"

namespace race {
namespace tcfast {

using namespace tc;

constexpr int CH = 128;              // tokens per chunk (= MMA M)
constexpr int DH = 128;              // d = dv
constexpr int SUB = CH * 64 * 2;     // one [128 x 64] bf16 SW128 sub-tile (16 KB)
constexpr int TILE = 2 * SUB;        // [128 x 128] bf16 tile (32 KB)
constexpr int WOP = 2 * 16 * 128;    // W' operand: [16 x 128] bf16, 2 SW128 sub-tiles of 2 KB
constexpr int PHI = CH * 64;         // [128 x 32] bf16 K-major SW64 (8 KB)
constexpr int NTHREADS = 192;
constexpr int NTHREADS8 = 320;      // 8-compute-warp kernels: warp 0 TMA, warp 1 MMA, 2..9 compute
constexpr int CT0 = 64;              // first compute thread of the 8-compute-warp kernels
constexpr int FP = 8;                // padded feature count
// Sketch rows (causal forward state, one per token): floats [0, 8) describe q, [8, 16) k:
// slot j < T*P holds x^.w_j = (x . w_j) / ||x|| exactly as the kernels compute it, slot 7
// holds ||x||^2.  The backward rebuilds phi and the tanh values from them instead of
// re-reading and re-projecting the other operand's tiles.
constexpr int ROWW = 16;

constexpr int LDS_T = DH + 1;        // table row stride (dv + 1)

// TMEM column map
constexpr uint32_t TM_PROJQ = 0, TM_PROJK = 16, TM_SACC = 32, TM_PM = 64, TM_NUM = 256;

struct Args {
  unsigned* dbg;  // optional host-mapped progress words (RACE_DEBUG_PROGRESS=1), [grid][256]
  int64_t BH, H, N, nseg, seg_tokens;
  int64_t Np;  // row pitch of the per-token rden / gden arrays: N rounded up to a multiple of 4
  int P, T, TP;
  int dw;   // head width d of the hyperplane rows (<= DH; tiles are zero-filled beyond it by TMA)
  int dvv;  // value width dv (<= DH): tables [F, dv + 1] have row stride ldt = dv + 1, normaliser column dv
  int ldt;
  float beta;
  int normalize, w_per_head;
  const float* w;
  const float* tin;   // tables / carries
  float* tout;        // partial tables
  float* den;
  const float* rows_in;  // [BH, N, ROWW] sketch rows saved by the causal forward (see ROWW)
  float* rows_out;
  int pf;               // chunks of L2 prefetch (cp.async.bulk.prefetch) ahead of the TMA loads
  int ttid;             // compute thread that records the per-chunk trace (RACE_TRACE_TID, default 64)
  // corner group (Geo::cb, race_abi.cu): one table of P + hb hyperplanes, of whose 2^(P+hb) corners
  // this pass sees the 2^P with high bits chi; hb = 0 otherwise
  int hb, chi;
  // table / corner groups: 1/D and -(dO.O)/D of the WHOLE estimator per token ([BH, Np]); the
  // query-side backward kernels use them instead of their own group's D and rho
  const float* ext_rd;
  const float* ext_gd;
  // grouped backward: per-row dproj out (Geo::dproj_q / dproj_k) instead of the dq / dk store
  float* dproj_out;
  int dproj_ld, dproj_col, dproj_acc;
  uint64_t hmagic;  // ceil(2^32 / H): sequence bh -> (head, batch) of the 4-D tensor maps (seq_hb)
};

// tile (c0 column, token t, sequence bh) of a make_map operand: sequence bh = b * H + h.  b = bh / H by
// a multiply-high with hmagic = ceil(2^32 / H), exact for bh, H < 2^16 (BH <= 65535 is enforced): the
// producer issues ~16 of these per chunk and sits on the chunk pipeline's critical path
__device__ __forceinline__ int2 seq_hb(const Args& a, int bh) {
  const int b = int((uint64_t(uint32_t(bh)) * a.hmagic) >> 32);
  return make_int2(bh - b * int(a.H), b);
}
// M4 (compile time): strided operands, 4-D {width, N, H, B} maps; otherwise the 3-D {width, N, B*H}
// maps of contiguous operands, with no index split on the default path
template <bool M4>
__device__ __forceinline__ void tile_load(const Args& a, void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int t,
                                          int bh, uint64_t policy) {
  if constexpr (M4) {
    const int2 hb = seq_hb(a, bh);
    tma_load_4d(dst, m, bar, c0, t, hb.x, hb.y, policy);
  } else {
    tma_load_3d(dst, m, bar, c0, t, bh, policy);
  }
}
template <bool M4>
__device__ __forceinline__ void tile_prefetch(const Args& a, const CUtensorMap* m, int c0, int t, int bh) {
  if constexpr (M4) {
    const int2 hb = seq_hb(a, bh);
    tma_prefetch_4d(m, c0, t, hb.x, hb.y);
  } else {
    tma_prefetch_3d(m, c0, t, bh);
  }
}
template <bool M4>
__device__ __forceinline__ void tile_store(const Args& a, const CUtensorMap* m, const void* src, int c0, int t, int bh) {
  if constexpr (M4) {
    const int2 hb = seq_hb(a, bh);
    tma_store_4d(m, src, c0, t, hb.x, hb.y);
  } else {
    tma_store_3d(m, src, c0, t, bh);
  }
}

// Grouped backward extras, loaded at the start of a chunk so their global-memory latency stays off the
// compute chain: the whole estimator's 1/D, -rho/D (ext) and, for corner groups, the dproj already
// summed over the table's earlier corner groups.
struct GroupPre {
  float rd, gd, prev[5];
};
__device__ __forceinline__ GroupPre group_prefetch(const Args& a, int64_t bh, int64_t t, int r, bool valid) {
  GroupPre g{0.f, 0.f, {0.f, 0.f, 0.f, 0.f, 0.f}};
  if (a.ext_rd && valid) {
    const int64_t i = bh * a.Np + t + r;
    g.rd = a.ext_rd[i];
    g.gd = a.ext_gd[i];
  }
  if (a.dproj_out && a.dproj_acc && valid) {
    const float* src = a.dproj_out + (bh * a.N + t + r) * a.dproj_ld + a.dproj_col;
#pragma unroll
    for (int j = 0; j < 5; ++j)
      if (j < a.TP) g.prev[j] = src[j];
  }
  return g;
}
// write this row's dproj_j, j < TP (plus the prefetched sum of earlier corner groups) at column
// dproj_col of the grouped-backward buffer
__device__ __forceinline__ void emit_dproj(const Args& a, int64_t row, const float* dproj, const GroupPre& pre) {
  float* dst = a.dproj_out + row * a.dproj_ld + a.dproj_col;
#pragma unroll
  for (int j = 0; j < 5; ++j)
    if (j < a.TP) dst[j] = dproj[j] + pre.prev[j];
}

#define RACE_DBG(a_, slot_, val_)                                                        \
  do {                                                                                   \
    if ((a_).dbg) *(volatile unsigned*)&(a_).dbg[blockIdx.x * 256 + (slot_)] = (val_);   \
  } while (0)

// timeline trace of CTA 0 (RACE_DEBUG_PROGRESS=1): slot ev * 32 + chunk holds clock()
#define RACE_TRACE(a_, ev_, gc_)                                                         \
  do {                                                                                   \
    if ((a_).dbg && blockIdx.x == 0 && (gc_) < 32u)                                      \
      *(volatile unsigned*)&(a_).dbg[(ev_) * 32 + (gc_)] = (unsigned)clock();            \
  } while (0)

// per-CTA start / end (globaltimer, ns) in the last 2 * 148 words of the debug buffer
__device__ __forceinline__ unsigned gtimer_lo() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return unsigned(t);
}
#define RACE_CTA_TIME(a_, which_)                                                        \
  do {                                                                                   \
    if ((a_).dbg && blockIdx.x < 148)                                                    \
      *(volatile unsigned*)&(a_).dbg[148 * 256 - 2 * 148 + 2 * blockIdx.x + (which_)] = gtimer_lo(); \
  } while (0)

// 1024-byte aligned base of the dynamic shared memory, derived by pointer arithmetic on the
// __shared__ array itself (not through an integer round trip) so that every pointer taken from it
// stays in the shared address space: the compiler then emits LDS / STS instead of generic LD / ST
__device__ __forceinline__ uint8_t* align_smem_1024(uint8_t* smem_raw) {
  return smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
}

// ---------------------------------------------------------------------------
// role helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int crow() { return ((warp_id() & 3) << 5) | lane_id(); }       // compute row
__device__ __forceinline__ uint32_t lane_base() { return uint32_t((warp_id() & 3) * 32) << 16; }
__device__ __forceinline__ void compute_bar256() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
// warp totals of 8 per-lane values by recursive halving (9 shuffles instead of 8 x 5): returns the total of
// value f = 4 b4 + 2 b3 + b2 (bits of the lane id) in every lane whose low two bits are 0 (and the
// same total in the other three lanes of its group of four); fixed order, so deterministic
__device__ __forceinline__ float warp_sum8(const float* v) {
  const int lane = threadIdx.x & 31;
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  float w[4], x[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float send = b4 ? v[k] : v[4 + k], keep = b4 ? v[4 + k] : v[k];
    w[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float send = b3 ? w[k] : w[2 + k], keep = b3 ? w[2 + k] : w[k];
    x[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  float y = (b2 ? x[1] : x[0]) + __shfl_xor_sync(0xffffffffu, b2 ? x[0] : x[1], 4);
  y += __shfl_xor_sync(0xffffffffu, y, 2);
  y += __shfl_xor_sync(0xffffffffu, y, 1);
  return y;
}
__device__ __forceinline__ void compute_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(pred));
  return pred != 0;
}

struct Item {
  int bh, seg, t0, t1;  // tokens [t0, t1) of sequence bh (32-bit: N < 2^31, B*H <= 65535)
};
__device__ __forceinline__ Item item_of(const Args& a, int64_t it) {
  Item r;
  r.bh = int(it / a.nseg);
  r.seg = int(it % a.nseg);
  r.t0 = int(r.seg * a.seg_tokens);
  r.t1 = int(r.t0 + a.seg_tokens < a.N ? r.t0 + a.seg_tokens : a.N);
  return r;
}

// contiguous item range of this CTA: [i0, i1)
__device__ __forceinline__ void cta_range(int64_t nitems, int64_t& i0, int64_t& i1) {
  i0 = int64_t(blockIdx.x) * nitems / gridDim.x;
  i1 = int64_t(blockIdx.x + 1) * nitems / gridDim.x;
}
// chunk cursor over a CTA's item range
struct Cursor {
  int it, i1, t;
  Item m;
  __device__ __forceinline__ void start(const Args& a, int64_t i0, int64_t i1_) {
    it = int(i0);
    i1 = int(i1_);
    if (it < i1) {
      m = item_of(a, it);
      t = m.t0;
    }
  }
  __device__ __forceinline__ bool ok() const { return it < i1; }
  __device__ __forceinline__ void next(const Args& a) {
    t += CH;
    if (t >= m.t1) {
      ++it;
      if (it < i1) {
        m = item_of(a, it);
        t = m.t0;
      }
    }
  }
};

// operand descriptors ------------------------------------------------------
// [128 x 128] bf16 tile from TMA (two SW128 sub-tiles), K-major, K-step kk of 16
__device__ __forceinline__ uint64_t desc_tile_k(uint32_t base, int kk) {
  return smem_desc(base + (kk >> 2) * SUB + (kk & 3) * 32, 16, 1024, kSw128);
}
// same tile used MN-major (rows = K = tokens, 128 MN = 2 sub-tiles at LBO = SUB)
__device__ __forceinline__ uint64_t desc_tile_mn(uint32_t base, int kk) {
  return smem_desc(base + kk * 2048, SUB, 1024, kSw128);
}
// W' [16 x 128] K-major SW128 (sub-tiles of 16 rows x 128 B)
__device__ __forceinline__ uint64_t desc_w(uint32_t base, int kk) {
  return smem_desc(base + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024, kSw128);
}
// [128 x 32] K-major SW64 (Phi / S operand), K-step kk in {0, 1}
__device__ __forceinline__ uint64_t desc_phi_k(uint32_t base, int kk) {
  return smem_desc(base + kk * 32, 16, 512, kSw64);
}
// same buffer used MN-major: N = 32 columns, K = 128 tokens
__device__ __forceinline__ uint64_t desc_phi_mn(uint32_t base, int kk) {
  return smem_desc(base + kk * 1024, 8192, 512, kSw64);
}

constexpr uint32_t ID_PROJ = idesc_bf16(128, 16, 0, 0);
constexpr uint32_t ID_PM = idesc_bf16(128, 128, 0, 0);
constexpr uint32_t ID_STATE = idesc_bf16(128, 32, 1, 1);
constexpr uint32_t ID_NUMA = idesc_bf16(128, 128, 0, 0);
constexpr uint32_t ID_NUMB = idesc_bf16(128, 128, 0, 1);

// ---------------------------------------------------------------------------
// compute-thread building blocks
// ---------------------------------------------------------------------------
// sum of squares of row r of a [128 x 128] SW128 tile
__device__ __forceinline__ float tile_row_sumsq(uint32_t tile, int r) {
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint4 v = ld_shared_v4(tile + h * SUB + r * 128 + ((j ^ (r & 7)) << 4));
      const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float a = bf16_lo(w4[q]), b = bf16_hi(w4[q]);
        s0 = fmaf(a, a, s0);
        s1 = fmaf(b, b, s1);
      }
    }
  }
  return s0 + s1;
}

// per-row inverse scale (1/||x|| or 1 for pass-through / unnormalised rows)
__device__ __forceinline__ float inv_scale(float sumsq, int normalize) {
  if (!normalize) return 1.f;
  const float nrm = sqrtf(sumsq);
  return nrm < kZeroRowEps ? 1.f : 1.f / nrm;
}

// W' rows 3j, 3j+1, 3j+2 = W_hi[j], W_mid[j], W_lo[j] (W to 24 bits), K-major SW128
template <int NTC = 128, int T0 = 64>
__device__ __forceinline__ void build_wop(const Args& a, int64_t bh, uint32_t wop) {
  const float* w = a.w + (a.w_per_head ? (bh % a.H) * int64_t(a.TP) * a.dw : 0);
  for (int idx = threadIdx.x - T0; idx < 16 * 16; idx += NTC) {
    const int n = idx >> 4, j = idx & 15;  // row n, 8-element chunk j
    const int hp = n / 3, piece = n % 3;
    uint32_t pk[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float v2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v = 0.f;
        if (hp < a.TP) {
          const int col = j * 8 + e * 2 + h;
          const float x = col < a.dw ? w[hp * a.dw + col] : 0.f;
          const float hi = bf16_round(x);
          const float mid = bf16_round(x - hi);
          v = piece == 0 ? hi : piece == 1 ? mid : bf16_round(x - hi - mid);
        }
        v2[h] = v;
      }
      pk[e] = pack_bf16(v2[0], v2[1]);
    }
    const uint32_t off = (j >> 3) * 2048 + n * 128 + (((j & 7) ^ (n & 7)) << 4);
    st_shared_v4(wop + off, pk[0], pk[1], pk[2], pk[3]);
  }
}

// Fast-path transcendental helpers (bf16 inputs, 1e-2 tolerance): ex2.approx has
// ~2^-22 relative error; tanh via e = 2^(-2|x| log2 e): tanh|x| = (1 - e) / (1 + e),
// accurate to ~1e-6 relative (the hardware tanh.approx, ~2^-11, would put ~1e-2 of
// error into phi at beta = 8, so it is not used).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_tanh(float x) {
  const float e = ex2_approx(-2.8853900817779268f * fabsf(x));  // exp(-2|x|)
  const float t = __fdividef(1.f - e, 1.f + e);
  return copysignf(t, x);
}
__device__ __forceinline__ float fast_exp_neg(float y) {  // exp(-y)
  return ex2_approx(-1.4426950408889634f * y);
}

// Corner group (a.hb > 0, one table): the fixed high bits chi of the pass's corners contribute
// prod_b sigma(2 beta c_b u_{P+b}) to every phi_r (factored form, ra/sketch.py:120-129), with
// u_j = tanh_of(j) for the projections j = P .. P + hb - 1.
// Compiled only into the corner-group instantiations (HB > 0, the kernels' second template
// argument): fully unrolled with compile-time indices j = P + b < 5 (hb <= HB = 2 since a pass has
// T*P <= 5 projections), so no register array is demoted to local memory and the ordinary
// instantiations carry none of this code.
template <int P, int HB, typename U>
__device__ __forceinline__ float group_weight(const Args& a, U tanh_of) {
  float m = 1.f;
#pragma unroll
  for (int b = 0; b < HB; ++b) {
    constexpr int kMax = 5;
    if (b < a.hb && P + b < kMax) {
      const float u = tanh_of(P + b < kMax ? P + b : 0);
      const float e = fast_exp_neg(2.f * a.beta * fabsf(u));
      const bool match = (((a.chi >> b) & 1) != 0) == (u < 0.f);
      m *= (match ? 1.f : e) / (1.f + e);
    }
  }
  return m;
}

// features of one row from its 16 projection columns (P compile-time, T <= 8 >> P)
template <int P, int HB = 0>
__device__ __forceinline__ void row_features(const Args& a, const float* proj, float inv, bool valid, float* phi) {
  constexpr int R = 1 << P;
  constexpr int TMAX = FP / R;
#pragma unroll
  for (int f = 0; f < FP; ++f) phi[f] = 0.f;
#pragma unroll
  for (int tau = 0; tau < TMAX; ++tau) {
    if (tau < a.T && valid) {
      float e[P], z = 1.f;
      bool neg[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int j = tau * P + p;
        const float u = fast_tanh((proj[3 * j] + proj[3 * j + 1] + proj[3 * j + 2]) * inv);
        e[p] = fast_exp_neg(2.f * a.beta * fabsf(u));
        neg[p] = u < 0.f;
        z *= 1.f + e[p];
      }
      float rz = 1.f / z;
      if constexpr (HB > 0) rz *= group_weight<P, HB>(a, [&](int j) { return fast_tanh((proj[3 * j] + proj[3 * j + 1] + proj[3 * j + 2]) * inv); });
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        float prod = rz;
#pragma unroll
        for (int p = 0; p < P; ++p) prod *= (((rr >> p) & 1) == int(neg[p])) ? 1.f : e[p];
        phi[tau * R + rr] = prod;
      }
    }
  }
}

// projections of one row as stored in the sketch rows: hat[j] = (x . w_j) / ||x||
__device__ __forceinline__ void row_hat(const Args& a, const float* proj, float inv, float* hat) {
#pragma unroll
  for (int j = 0; j < 5; ++j) hat[j] = j < a.TP ? (proj[3 * j] + proj[3 * j + 1] + proj[3 * j + 2]) * inv : 0.f;
}
// store the 8-float half of a sketch row (hat[0..5), 0, 0, ||x||^2)
__device__ __forceinline__ void store_row_half(float* dst, const float* hat, float sumsq) {
  reinterpret_cast<float4*>(dst)[0] = make_float4(hat[0], hat[1], hat[2], hat[3]);
  reinterpret_cast<float4*>(dst)[1] = make_float4(hat[4], 0.f, 0.f, sumsq);
}
// features from stored projections hat (same arithmetic as row_features[_u])
template <int P, int HB = 0>
__device__ __forceinline__ void row_features_hat(const Args& a, const float* hat, bool valid, float* phi, float* u) {
  constexpr int R = 1 << P;
  constexpr int TMAX = FP / R;
#pragma unroll
  for (int f = 0; f < FP; ++f) phi[f] = 0.f;
#pragma unroll
  for (int j = 0; j < 5; ++j) u[j] = 0.f;
#pragma unroll
  for (int tau = 0; tau < TMAX; ++tau) {
    if (tau < a.T && valid) {
      float e[P], z = 1.f;
      bool neg[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int j = tau * P + p;
        const float uu = fast_tanh(hat[j < 5 ? j : 0]);
        u[j < 5 ? j : 0] = uu;
        e[p] = fast_exp_neg(2.f * a.beta * fabsf(uu));
        neg[p] = uu < 0.f;
        z *= 1.f + e[p];
      }
      float rz = 1.f / z;
      if constexpr (HB > 0)
        rz *= group_weight<P, HB>(a, [&](int j) {
          const float uu = fast_tanh(hat[j]);
          u[j] = uu;
          return uu;
        });
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        float prod = rz;
#pragma unroll
        for (int p = 0; p < P; ++p) prod *= (((rr >> p) & 1) == int(neg[p])) ? 1.f : e[p];
        phi[tau * R + rr] = prod;
      }
    }
  }
}

// row r of a [128 x 32] SW64 operand: four 8-element bf16 blocks
__device__ __forceinline__ void write_row32(uint32_t buf, int r, const uint32_t (*blk)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t off = r * 64 + ((j ^ ((r >> 1) & 3)) << 4);
    st_shared_v4(buf + off, blk[j][0], blk[j][1], blk[j][2], blk[j][3]);
  }
}
__device__ __forceinline__ void split8(const float* x, uint32_t* hi, uint32_t* lo) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float h0 = bf16_round(x[2 * e]), h1 = bf16_round(x[2 * e + 1]);
    hi[e] = pack_bf16(h0, h1);
    lo[e] = pack_bf16(x[2 * e] - h0, x[2 * e + 1] - h1);
  }
}
// Phi_q row: [hi | lo | hi | 0];  Phi_k row: [hi | hi | lo | 0]  => Pq.Pk = qh kh + ql kh + qh kl
__device__ __forceinline__ void write_phi_q(uint32_t buf, int r, const float* phi) {
  uint32_t b[4][4];
  split8(phi, b[0], b[1]);
#pragma unroll
  for (int e = 0; e < 4; ++e) { b[2][e] = b[0][e]; b[3][e] = 0u; }
  write_row32(buf, r, b);
}
__device__ __forceinline__ void write_phi_k(uint32_t buf, int r, const float* phi) {
  uint32_t b[4][4];
  split8(phi, b[0], b[2]);
#pragma unroll
  for (int e = 0; e < 4; ++e) { b[1][e] = b[0][e]; b[3][e] = 0u; }
  write_row32(buf, r, b);
}
// S operand row c (B of num = Phi_q S): [S_hi | S_hi | S_lo | 0] over f
__device__ __forceinline__ void write_sop(uint32_t buf, int c, const float* s) {
  uint32_t b[4][4];
  split8(s, b[0], b[2]);
#pragma unroll
  for (int e = 0; e < 4; ++e) { b[1][e] = b[0][e]; b[3][e] = 0u; }
  write_row32(buf, c, b);
}


// write one [128 x 128] fp32 row (from TMEM) as bf16 into a SW128 staging tile
__device__ __forceinline__ void stage_row_bf16(uint32_t tile, int r, const float* v, int c0) {
  // v holds columns [c0, c0 + 32)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int chunk = (c0 >> 3) + j;  // 8-element chunk index 0..15
    const uint32_t off = (chunk >> 3) * SUB + r * 128 + (((chunk & 7) ^ (r & 7)) << 4);
    st_shared_v4(tile + off, pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                 pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
  }
}


// ---------------------------------------------------------------------------
// backward helpers
// ---------------------------------------------------------------------------
// W'' = [W_hi; W_hi; W_lo; 0] (blocks of 8 K-rows, hyperplane j in row 8b + j) as an
// MN-major SW128 [32 x 128] operand: B of dx^ = dProj . W with dProj = [hi | lo | hi | 0]
constexpr int W2OP = 2 * 32 * 128;  // 8 KB
__device__ __forceinline__ uint64_t desc_w2(uint32_t base, int kk) {
  return smem_desc(base + kk * 2048, 4096, 1024, kSw128);
}
template <int NTC = 128, int T0 = 64>
__device__ __forceinline__ void build_w2(const Args& a, int64_t bh, uint32_t w2) {
  const float* w = a.w + (a.w_per_head ? (bh % a.H) * int64_t(a.TP) * a.dw : 0);
  for (int idx = threadIdx.x - T0; idx < 32 * 16; idx += NTC) {
    const int k = idx >> 4, j = idx & 15;  // K-row k, 8-element column chunk j
    const int blk = k >> 3, hp = k & 7;
    uint32_t pk[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float v2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v = 0.f;
        if (blk < 3 && hp < a.TP) {
          const int col = j * 8 + e * 2 + h;
          const float x = col < a.dw ? w[hp * a.dw + col] : 0.f;
          const float hi = bf16_round(x);
          v = blk == 2 ? x - hi : hi;
        }
        v2[h] = v;
      }
      pk[e] = pack_bf16(v2[0], v2[1]);
    }
    const uint32_t off = (j >> 3) * 4096 + k * 128 + (((j & 7) ^ (k & 7)) << 4);
    st_shared_v4(w2 + off, pk[0], pk[1], pk[2], pk[3]);
  }
}

// S^T operand [16 x 128] K-major SW128 (rows f = S_hi[f], 8 + f = S_lo[f]; K = value
// column): B of y = dO . S_v^T.  Thread c owns value column c.
__device__ __forceinline__ void write_sopT(uint32_t buf, int c, const float* s) {
  const uint32_t sub = (c >> 6) * 2048;
  const uint32_t inrow = (c & 63) * 2;
#pragma unroll
  for (int f = 0; f < 8; ++f) {
    const float hi = bf16_round(s[f]);
    const __nv_bfloat16 bh = __float2bfloat16_rn(hi), bl = __float2bfloat16_rn(s[f] - hi);
    const uint32_t o1 = f * 128 + inrow, o2 = (8 + f) * 128 + inrow;
    const uint32_t p1 = sub + (o1 ^ (((o1 >> 7) & 7) << 4)), p2 = sub + (o2 ^ (((o2 >> 7) & 7) << 4));
    asm volatile("st.shared.b16 [%0], %1;" ::"r"(buf + p1), "h"(*reinterpret_cast<const unsigned short*>(&bh)) : "memory");
    asm volatile("st.shared.b16 [%0], %1;" ::"r"(buf + p2), "h"(*reinterpret_cast<const unsigned short*>(&bl)) : "memory");
  }
}

// features + the tanh values u_j (j < TP) kept for the VJP
template <int P, int HB = 0>
__device__ __forceinline__ void row_features_u(const Args& a, const float* proj, float inv, bool valid, float* phi,
                                               float* u, float* phat) {
  constexpr int R = 1 << P;
  constexpr int TMAX = FP / R;
#pragma unroll
  for (int f = 0; f < FP; ++f) phi[f] = 0.f;
#pragma unroll
  for (int j = 0; j < 5; ++j) u[j] = phat[j] = 0.f;
#pragma unroll
  for (int tau = 0; tau < TMAX; ++tau) {
    if (tau < a.T && valid) {
      float e[P], z = 1.f;
      bool neg[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int j = tau * P + p;
        const float ph = (proj[3 * j] + proj[3 * j + 1] + proj[3 * j + 2]) * inv;
        const float uu = fast_tanh(ph);
        phat[j] = ph;
        u[j] = uu;
        e[p] = fast_exp_neg(2.f * a.beta * fabsf(uu));
        neg[p] = uu < 0.f;
        z *= 1.f + e[p];
      }
      float rz = 1.f / z;
      if constexpr (HB > 0)
        rz *= group_weight<P, HB>(a, [&](int j) {
          const float ph = (proj[3 * j] + proj[3 * j + 1] + proj[3 * j + 2]) * inv;
          const float uu = fast_tanh(ph);
          phat[j] = ph;
          u[j] = uu;
          return uu;
        });
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        float prod = rz;
#pragma unroll
        for (int p = 0; p < P; ++p) prod *= (((rr >> p) & 1) == int(neg[p])) ? 1.f : e[p];
        phi[tau * R + rr] = prod;
      }
    }
  }
}

// softmax-over-corners + tanh VJP (ra/backward.py:53-90): dphi -> dproj_j, j < TP
template <int P, int HB = 0>
__device__ __forceinline__ void row_feature_vjp(const Args& a, const float* u, const float* phi, const float* dphi,
                                                float* dproj) {
  constexpr int R = 1 << P;
  constexpr int TMAX = FP / R;
#pragma unroll
  for (int j = 0; j < 8; ++j) dproj[j] = 0.f;
  if constexpr (HB > 0) {  // corner group (one table): factored VJP, exact per corner subset (ra/backward.py:65-88)
    // phi_r = prod_t sigma(2 beta c_rt u_t) => du_t = 2 beta sum_r dphi_r phi_r c_rt (1 - sigma(2 beta c_rt u_t))
    float s = 0.f, sp[P];
#pragma unroll
    for (int p = 0; p < P; ++p) sp[p] = 0.f;
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const float x = dphi[rr] * phi[rr];
      s += x;
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (!((rr >> p) & 1)) sp[p] += x;
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {  // low bits: split by c_rt = +1 (sum sp) / -1 (s - sp)
      const float sg = 1.f / (1.f + fast_exp_neg(2.f * a.beta * u[p]));  // sigma(2 beta u)
      dproj[p] = 2.f * a.beta * ((1.f - sg) * sp[p] - sg * (s - sp[p])) * (1.f - u[p] * u[p]);
    }
#pragma unroll
    for (int b = 0; b < HB; ++b) {  // high bits: c fixed by chi (compile-time indices, see group_weight)
      constexpr int kMax = 5;
      if (b < a.hb && P + b < kMax) {
        const int j = P + b < kMax ? P + b : 0;
        const float uj = u[j];
        const float sg = 1.f / (1.f + fast_exp_neg(2.f * a.beta * uj));
        const float d = ((a.chi >> b) & 1) ? -sg : (1.f - sg);
        dproj[j] = 2.f * a.beta * d * s * (1.f - uj * uj);
      }
    }
  } else {
#pragma unroll
    for (int tau = 0; tau < TMAX; ++tau) {
      if (tau < a.T) {
        float s = 0.f;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) s = fmaf(dphi[tau * R + rr], phi[tau * R + rr], s);
#pragma unroll
        for (int p = 0; p < P; ++p) {
          float du = 0.f;
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const float dl = phi[tau * R + rr] * (dphi[tau * R + rr] - s);
            du += ((rr >> p) & 1) ? -dl : dl;
          }
          const float uu = u[tau * P + p];
          dproj[tau * P + p] = a.beta * du * (1.f - uu * uu);
        }
      }
    }
  }
}

// dProj row (A of dx^ = dProj . W''): [hi | lo | hi | 0]
__device__ __forceinline__ void write_dproj(uint32_t buf, int r, const float* dproj) { write_phi_q(buf, r, dproj); }

// dx^.x^ = sum_j dproj_j phat_j
__device__ __forceinline__ float dot_from_proj(const float* dproj, const float* phat) {
  float d = 0.f;
#pragma unroll
  for (int j = 0; j < 5; ++j) d = fmaf(dproj[j], phat[j], d);
  return d;
}

struct Scale {
  float inv;     // 1/||x|| (or 1)
  bool tangent;  // apply the sphere-tangent projection (normalised, non-zero row)
};
__device__ __forceinline__ Scale row_scale(float sumsq, int normalize) {
  if (!normalize) return {1.f, false};
  const float nrm = sqrtf(sumsq);
  if (nrm < kZeroRowEps) return {1.f, false};
  return {1.f / nrm, true};
}

// dx = (dx^ - (dx^.x^) x^) / ||x|| from TMEM columns [col, col+128) (lane = row r),
// x = row r of the SW128 tile; the bf16 result overwrites row r of the same tile.
// dot_hat = dx^.x^ = sum_j dproj_j (x^.w_j): computed by the caller from the
// projections, so one pass over dx^ suffices.
__device__ __forceinline__ void tangent_row_inplace(uint32_t tmem_col, uint32_t tile, int r, Scale sc,
                                                    float dot_hat) {
  const float cx = sc.tangent ? dot_hat * sc.inv : 0.f;  // (dx^.x^) / ||x|| per unit of raw x
#pragma unroll
  for (int c0 = 0; c0 < DH; c0 += 32) {
    float v[32];
    tmem_ld32(tmem_col + c0, v);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int chunk = (c0 >> 3) + j;
      const uint32_t addr = tile + (chunk >> 3) * SUB + r * 128 + (((chunk & 7) ^ (r & 7)) << 4);
      uint32_t o[4];
      if (sc.tangent) {
        const uint4 x = ld_shared_v4(addr);
        const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          o[q] = pack_bf16((v[8 * j + 2 * q] - cx * bf16_lo(xw[q])) * sc.inv,
                           (v[8 * j + 2 * q + 1] - cx * bf16_hi(xw[q])) * sc.inv);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = pack_bf16(v[8 * j + 2 * q], v[8 * j + 2 * q + 1]);
      }
      st_shared_v4(addr, o[0], o[1], o[2], o[3]);
    }
  }
}


// ---------------------------------------------------------------------------
// 8-compute-warp helpers (warps 2..9): warp w and w+4 share TMEM lane quarter
// w % 4 (rows), and split the 128 columns into halves h = 0 / 1.
// ---------------------------------------------------------------------------
template <int N> __device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <int N> __device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
__device__ __forceinline__ int chalf() { return warp_id() >= 6 ? 1 : 0; }
__device__ __forceinline__ void cbar256() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void hbar128(int h) { asm volatile("bar.sync %0, 128;" ::"r"(2 + h) : "memory"); }

// sum of squares over columns [64h, 64h + 64) of row r (= SW128 sub-tile h)
__device__ __forceinline__ float half_row_sumsq(uint32_t tile, int r, int h) {
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint4 v = ld_shared_v4(tile + h * SUB + r * 128 + ((j ^ (r & 7)) << 4));
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float a = bf16_lo(w4[q]), b = bf16_hi(w4[q]);
      s0 = fmaf(a, a, s0);
      s1 = fmaf(b, b, s1);
    }
  }
  return s0 + s1;
}

// copy half h of row r between two SW128 tiles (same swizzle => same offsets)
__device__ __forceinline__ void copy_half_row(uint32_t dst, uint32_t src, int r, int h) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t off = h * SUB + r * 128 + (j << 4);
    const uint4 v = ld_shared_v4(src + off);
    st_shared_v4(dst + off, v.x, v.y, v.z, v.w);
  }
}


// one-pass tangent VJP for columns [64h, 64h + 64) of row r; bf16 result straight to global
__device__ __forceinline__ void tangent_half_to_global(uint32_t tmem_col, uint32_t tile, int r, int h, Scale sc,
                                                       float dot_hat, __nv_bfloat16* grow, bool store) {
  const float cx = sc.tangent ? dot_hat * sc.inv : 0.f;
#pragma unroll
  for (int c0 = 0; c0 < 64; c0 += 32) {
    float v[32];
    tmem_ld32(tmem_col + 64 * h + c0, v);
    tmem_ld_wait();
    uint32_t o[16];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int chunk = 8 * h + (c0 >> 3) + j;
      const uint4 x = ld_shared_v4(tile + h * SUB + r * 128 + (((chunk & 7) ^ (r & 7)) << 4));
      const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float a = sc.tangent ? (v[8 * j + 2 * q] - cx * bf16_lo(xw[q])) * sc.inv : v[8 * j + 2 * q];
        const float b = sc.tangent ? (v[8 * j + 2 * q + 1] - cx * bf16_hi(xw[q])) * sc.inv : v[8 * j + 2 * q + 1];
        o[4 * j + q] = pack_bf16(a, b);
      }
    }
    if (store) {
      uint4* dst = reinterpret_cast<uint4*>(grow + 64 * h + c0);
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
    }
  }
}

// TMEM columns [64h, 64h + 64) of row r -> bf16 global row
__device__ __forceinline__ void tmem_half_to_global(uint32_t tmem_col, int h, float scale, __nv_bfloat16* grow,
                                                    bool store) {
#pragma unroll
  for (int c0 = 0; c0 < 64; c0 += 32) {
    float v[32];
    tmem_ld32(tmem_col + 64 * h + c0, v);
    tmem_ld_wait();
    if (store) {
      uint4* dst = reinterpret_cast<uint4*>(grow + 64 * h + c0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        dst[j] = make_uint4(pack_bf16(v[8 * j] * scale, v[8 * j + 1] * scale),
                            pack_bf16(v[8 * j + 2] * scale, v[8 * j + 3] * scale),
                            pack_bf16(v[8 * j + 4] * scale, v[8 * j + 5] * scale),
                            pack_bf16(v[8 * j + 6] * scale, v[8 * j + 7] * scale));
    }
  }
}

// W' / W'' builds spread over the 256 compute threads
__device__ __forceinline__ void build_ops_256(const Args& a, int64_t bh, uint32_t wop, uint32_t w2) {
  const float* w = a.w + (a.w_per_head ? (bh % a.H) * int64_t(a.TP) * a.dw : 0);
  const int tid = threadIdx.x - 64;
  for (int idx = tid; idx < 16 * 16 + 32 * 16; idx += 256) {
    uint32_t pk[4];
    uint32_t off, base;
    if (idx < 256) {  // W' row n = 3j + piece
      const int n = idx >> 4, j = idx & 15, hp = n / 3, piece = n % 3;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v2[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float v = 0.f;
          if (hp < a.TP) {
            const int col = j * 8 + e * 2 + hh;
            const float x = col < a.dw ? w[hp * a.dw + col] : 0.f;
            const float hi = bf16_round(x);
            const float mid = bf16_round(x - hi);
            v = piece == 0 ? hi : piece == 1 ? mid : bf16_round(x - hi - mid);
          }
          v2[hh] = v;
        }
        pk[e] = pack_bf16(v2[0], v2[1]);
      }
      off = (j >> 3) * 2048 + n * 128 + (((j & 7) ^ (n & 7)) << 4);
      base = wop;
    } else {  // W'' K-row k = 8 blk + hp
      const int i2 = idx - 256, k = i2 >> 4, j = i2 & 15, blk = k >> 3, hp = k & 7;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v2[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float v = 0.f;
          if (blk < 3 && hp < a.TP) {
            const int col = j * 8 + e * 2 + hh;
            const float x = col < a.dw ? w[hp * a.dw + col] : 0.f;
            const float hi = bf16_round(x);
            v = blk == 2 ? x - hi : hi;
          }
          v2[hh] = v;
        }
        pk[e] = pack_bf16(v2[0], v2[1]);
      }
      off = (j >> 3) * 4096 + k * 128 + (((j & 7) ^ (k & 7)) << 4);
      base = w2;
    }
    st_shared_v4(base + off, pk[0], pk[1], pk[2], pk[3]);
  }
}

// S^T operand column c, only f in [f0, f0 + 4) (the two halves split the 8 rows)
__device__ __forceinline__ void write_sopT_half(uint32_t buf, int c, const float* s, int f0) {
  const uint32_t sub = (c >> 6) * 2048;
  const uint32_t inrow = (c & 63) * 2;
#pragma unroll
  for (int ff = 0; ff < 4; ++ff) {
    const int f = f0 + ff;
    const float hi = bf16_round(s[f]);
    const __nv_bfloat16 bh = __float2bfloat16_rn(hi), bl = __float2bfloat16_rn(s[f] - hi);
    const uint32_t o1 = f * 128 + inrow, o2 = (8 + f) * 128 + inrow;
    const uint32_t p1 = sub + (o1 ^ (((o1 >> 7) & 7) << 4)), p2 = sub + (o2 ^ (((o2 >> 7) & 7) << 4));
    asm volatile("st.shared.b16 [%0], %1;" ::"r"(buf + p1), "h"(*reinterpret_cast<const unsigned short*>(&bh)) : "memory");
    asm volatile("st.shared.b16 [%0], %1;" ::"r"(buf + p2), "h"(*reinterpret_cast<const unsigned short*>(&bl)) : "memory");
  }
}


// ---------------------------------------------------------------------------
// pointer-based variants of the row helpers: plain C++ shared-memory accesses
// (LDS/STS the compiler may batch and reorder), for the hot loops
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4* tile_chunk(uint8_t* tile, int r, int chunk) {
  return reinterpret_cast<uint4*>(tile + (chunk >> 3) * SUB + r * 128 + (((chunk & 7) ^ (r & 7)) << 4));
}
__device__ __forceinline__ float half_row_sumsq_p(uint8_t* tile, int r, int h) {
  uint4 v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = *tile_chunk(tile, r, 8 * h + j);
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t w4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float a = bf16_lo(w4[q]), b = bf16_hi(w4[q]);
      s0 = fmaf(a, a, s0);
      s1 = fmaf(b, b, s1);
    }
  }
  return s0 + s1;
}
__device__ __forceinline__ void copy_half_row_p(uint8_t* dst, uint8_t* src, int r, int h) {
  uint4 v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = *tile_chunk(src, r, 8 * h + j);
#pragma unroll
  for (int j = 0; j < 8; ++j) *tile_chunk(dst, r, 8 * h + j) = v[j];
}
// 32 fp32 values (columns [c0, c0 + 32)) -> bf16 into row r of a SW128 tile
__device__ __forceinline__ void stage32_p(uint8_t* tile, int r, const float* v, int c0) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *tile_chunk(tile, r, (c0 >> 3) + j) =
        make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                   pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
}
// tangent VJP on 32 columns [c0, c0 + 32) given the dx^ values v; x from the tile
__device__ __forceinline__ void tangent32(const float* v, uint8_t* tile, int r, int c0, Scale sc, float cx,
                                          uint32_t* o) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint4 x = *tile_chunk(tile, r, (c0 >> 3) + j);
    const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float a = sc.tangent ? (v[8 * j + 2 * q] - cx * bf16_lo(xw[q])) * sc.inv : v[8 * j + 2 * q];
      const float b = sc.tangent ? (v[8 * j + 2 * q + 1] - cx * bf16_hi(xw[q])) * sc.inv : v[8 * j + 2 * q + 1];
      o[4 * j + q] = pack_bf16(a, b);
    }
  }
}
__device__ __forceinline__ void st_global16(__nv_bfloat16* dst, const uint32_t* o) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int j = 0; j < 4; ++j) d[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
}
// columns [64h, 64h + 64): dx = tangent(dx^) straight to global (TMEM loads double-buffered)
__device__ __forceinline__ void tangent_half_p(uint32_t tmem_col, uint8_t* tile, int r, int h, Scale sc,
                                               float dot_hat, __nv_bfloat16* grow, bool store) {
  const float cx = sc.tangent ? dot_hat * sc.inv : 0.f;
  float v0[32], v1[32];
  uint32_t o[16];
  tmem_ld32(tmem_col + 64 * h, v0);
  tmem_ld_wait();
  tmem_ld32(tmem_col + 64 * h + 32, v1);
  tangent32(v0, tile, r, 64 * h, sc, cx, o);
  if (store) st_global16(grow + 64 * h, o);
  tmem_ld_wait();
  tangent32(v1, tile, r, 64 * h + 32, sc, cx, o);
  if (store) st_global16(grow + 64 * h + 32, o);
}
// columns [64h, 64h + 64): dx = tangent(dx^) written back over x in the SW128 tile
__device__ __forceinline__ void tangent_half_inplace(uint32_t tmem_col, uint8_t* tile, int r, int h, Scale sc,
                                                     float dot_hat) {
  const float cx = sc.tangent ? dot_hat * sc.inv : 0.f;
  float v0[32], v1[32];
  uint32_t o[16];
  tmem_ld32(tmem_col + 64 * h, v0);
  tmem_ld_wait();
  tmem_ld32(tmem_col + 64 * h + 32, v1);
  tangent32(v0, tile, r, 64 * h, sc, cx, o);
#pragma unroll
  for (int j = 0; j < 4; ++j) *tile_chunk(tile, r, 8 * h + j) = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
  tmem_ld_wait();
  tangent32(v1, tile, r, 64 * h + 32, sc, cx, o);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *tile_chunk(tile, r, 8 * h + 4 + j) = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
}
// fp32 hyperplane rows (TP x 128, zero-padded to 5 rows) for the CUDA-core dx^ = dproj . W
template <int NTC, int T0>
__device__ __forceinline__ void build_wf32(const Args& a, int64_t bh, float* wf) {
  const float* w = a.w + (a.w_per_head ? (bh % a.H) * int64_t(a.TP) * a.dw : 0);
  for (int idx = threadIdx.x - T0; idx < 5 * DH; idx += NTC) {
    const int j = idx / DH, c = idx % DH;
    wf[idx] = (j < a.TP && c < a.dw) ? w[j * a.dw + c] : 0.f;
  }
}
// columns [64h, 64h + 64) of row r: dx^ = dproj . W (fp32 FMA, W from smem), then the
// sphere-tangent VJP dx = (dx^ - (dx^.x^) x^) / ||x||, written as bf16 over x in the SW128 tile
__device__ __forceinline__ void dx_tangent_half(const float* dproj, const float* wf, uint8_t* tile, int r, int h,
                                                Scale sc, float dot_hat) {
  const float cx = sc.tangent ? dot_hat * sc.inv : 0.f;
#pragma unroll 2
  for (int ch = 0; ch < 8; ++ch) {  // one 16-byte chunk = 8 columns
    const int chunk = 8 * h + ch, c0 = 8 * chunk;
    float d[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) d[e] = 0.f;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const float4 w0 = *reinterpret_cast<const float4*>(wf + j * DH + c0);
      const float4 w1 = *reinterpret_cast<const float4*>(wf + j * DH + c0 + 4);
      const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) d[e] = fmaf(dproj[j], wv[e], d[e]);
    }
    uint4* px = tile_chunk(tile, r, chunk);
    const uint4 x = *px;
    const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float lo = sc.tangent ? (d[2 * q] - cx * bf16_lo(xw[q])) * sc.inv : d[2 * q];
      const float hi = sc.tangent ? (d[2 * q + 1] - cx * bf16_hi(xw[q])) * sc.inv : d[2 * q + 1];
      o[q] = pack_bf16(lo, hi);
    }
    *px = make_uint4(o[0], o[1], o[2], o[3]);
  }
}
// TMEM columns [64h, 64h + 64) -> bf16 global row (double-buffered TMEM loads)
__device__ __forceinline__ void tmem_half_to_global_p(uint32_t tmem_col, int h, __nv_bfloat16* grow, bool store) {
  float v0[32], v1[32];
  uint32_t o[16];
  tmem_ld32(tmem_col + 64 * h, v0);
  tmem_ld_wait();
  tmem_ld32(tmem_col + 64 * h + 32, v1);
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j] = pack_bf16(v0[2 * j], v0[2 * j + 1]);
  if (store) st_global16(grow + 64 * h, o);
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j] = pack_bf16(v1[2 * j], v1[2 * j + 1]);
  if (store) st_global16(grow + 64 * h + 32, o);
}
// row r of a [128 x 32] SW64 operand from four 8-element blocks
__device__ __forceinline__ void write_row32_p(uint8_t* buf, int r, const uint32_t (*blk)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<uint4*>(buf + r * 64 + ((j ^ ((r >> 1) & 3)) << 4)) =
        make_uint4(blk[j][0], blk[j][1], blk[j][2], blk[j][3]);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// [B, H, N, width] bf16 viewed as 4-D {width, N, H, B} (strides of Geo::lay[which], or the contiguous
// [B*H, N, width] layout); box {64, 128, 1, 1}; SW128.  width = the tensor's row length (d for Q, K, dQ,
// dK; dv for V, O, dO, dV), <= DH: the two 64-column boxes of a tile read zeros beyond it and stores
// beyond it are clipped, so narrower heads run on the same kernels without padded copies.  The
// per-dimension strides need not be monotonic: a [B, N, H, d] view (token stride H*d, head stride d)
// is described in place, without a transposed copy.
inline bool make_map(CUtensorMap* m, const void* ptr, const Geo& g, int width, LayIdx which) {
  auto fn = encode_fn();
  if (!fn || g.H <= 0 || g.BH % g.H) return false;
  if (!g.strided()) {  // 3-D {width, N, B*H} (kernels instantiated with M4 = false)
    cuuint64_t dims[3] = {cuuint64_t(width), cuuint64_t(g.N), cuuint64_t(g.BH)};
    cuuint64_t strides[2] = {cuuint64_t(width) * 2, cuuint64_t(g.N) * width * 2};
    cuuint32_t box[3] = {64, CH, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  const Lay& l = g.lay[which];
  const int64_t st = l.token ? l.token : width, sh = l.token ? l.head : g.N * width,
                sbt = l.token ? l.batch : g.H * g.N * width;
  cuuint64_t dims[4] = {cuuint64_t(width), cuuint64_t(g.N), cuuint64_t(g.H), cuuint64_t(g.BH / g.H)};
  cuuint64_t strides[3] = {cuuint64_t(st) * 2, cuuint64_t(sh) * 2, cuuint64_t(sbt) * 2};
  cuuint32_t box[4] = {64, CH, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// flat fp32 array of `elems` viewed 1-D, box of `box` elements (OOB reads are zero)
inline bool make_map_f32_1d(CUtensorMap* m, const void* ptr, int64_t elems, int box) {
  auto fn = encode_fn();
  if (!fn || elems <= 0 || elems >= (int64_t(1) << 32)) return false;
  cuuint64_t dims[1] = {cuuint64_t(elems)};
  cuuint64_t strides[1] = {0};
  cuuint32_t bx[1] = {cuuint32_t(box)};
  cuuint32_t es[1] = {1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, const_cast<void*>(ptr), dims, strides, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// sketch rows [rows, ROWW] fp32 (race_b200.h), box of 128 rows (OOB rows read as zero)
inline bool make_map_rows(CUtensorMap* m, const void* ptr, int64_t rows) {
  auto fn = encode_fn();
  if (!fn || rows <= 0 || rows >= (int64_t(1) << 32)) return false;
  cuuint64_t dims[2] = {cuuint64_t(ROWW), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ROWW) * 4};
  cuuint32_t bx[2] = {cuuint32_t(ROWW), cuuint32_t(CH)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

unsigned* debug_progress_device();  // race_tc.cu
// the debug buffer for kernel `name` ("fwd", "bq", "bk"), or null when RACE_TRACE_KERNEL names another
inline unsigned* trace_for(const char* name) {
  const char* k = getenv("RACE_TRACE_KERNEL");
  if (k && k[0] && strcmp(k, name) != 0) return nullptr;
  return debug_progress_device();
}
inline Args make_args(const Geo& g) {
  Args a{};
  a.dbg = debug_progress_device();
  a.BH = g.BH;
  a.H = g.H;
  a.N = g.N;
  a.Np = (g.N + 3) & ~int64_t(3);
  a.nseg = g.nseg;
  a.seg_tokens = g.seg_tokens;
  a.P = pass_corner_bits(g);  // corner bits of this pass (the kernels' template P)
  a.T = g.T;
  a.TP = g.T * g.P;           // projections (all hyperplanes of the pass's tables)
  a.hmagic = ((uint64_t(1) << 32) + uint64_t(g.H) - 1) / uint64_t(g.H);
  a.dw = g.d;
  a.dvv = g.dv;
  a.ldt = g.dv + 1;
  a.hb = g.P - a.P;
  a.chi = int(g.chi);
  a.ext_rd = g.ext_rden;
  a.ext_gd = g.ext_gden;
  a.dproj_out = nullptr;  // set per kernel (query / key side) by the launchers
  a.dproj_ld = g.dproj_ld;
  a.dproj_col = g.dproj_col;
  a.dproj_acc = g.dproj_acc;
  a.beta = g.beta;
  a.normalize = g.normalize;
  a.w_per_head = g.w_per_head;
  const char* pf = getenv("RACE_PF");  // tuning knob, off by default
  a.pf = pf && pf[0] ? atoi(pf) : 0;  // measured: L2 prefetch slows every kernel here (r01)
  const char* tt = getenv("RACE_TRACE_TID");
  a.ttid = tt && tt[0] ? atoi(tt) : 64;
  return a;
}

// per-device facts queried once (the per-call path only reads them): bit 0 = queried,
// bit 1 = sm_100, bits 8.. = SM count
inline unsigned device_facts() {
  static std::atomic<unsigned> facts[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 0;
  if (dev >= 64) dev = 63;
  unsigned f = facts[dev].load(std::memory_order_relaxed);
  if (!f) {
    int major = 0, minor = 0, n = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    f = 1u | ((major == 10 && minor == 0) ? 2u : 0u) | (unsigned(n) << 8);
    facts[dev].store(f, std::memory_order_relaxed);
  }
  return f;
}
inline bool device_is_sm100() { return (device_facts() & 2u) != 0; }
inline int num_sms() {
  const int n = int(device_facts() >> 8);
  return n > 0 ? n : 148;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): it is a driver call
// of a few microseconds, and an eager fwd+bwd makes six launches
inline cudaError_t ensure_smem_attr(const void* kernel, int smem) {
  static std::mutex mu;
  static std::unordered_map<const void*, uint64_t> done;  // kernel -> mask of devices set at >= smem
  static std::unordered_map<const void*, int> done_smem;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = uint64_t(1) << (dev & 63);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find(kernel);
    if (it != done.end() && (it->second & bit) && done_smem[kernel] >= smem) return cudaSuccess;
  }
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int& s = done_smem[kernel];
  if (s != smem) {  // a new size applies to every device again
    done[kernel] = 0;
    s = smem;
  }
  done[kernel] |= bit;
  return cudaSuccess;
}

inline unsigned grid_for(const Geo& g) {
  const int64_t items = g.BH * g.nseg;
  return unsigned(items < num_sms() ? items : num_sms());
}

// Every tcgen05 kernel is launched with programmatic stream serialisation (PDL): its CTAs may start on
// SMs the previous kernel's CTAs have left, run their prologue (barrier init, TMEM allocation, tensor-map
// prefetch) and block in grid_dep_wait() until that kernel has completed.  RACE_NO_PDL=1 disables it.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("RACE_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}
template <typename K, typename... Ts>
cudaError_t launch_nt(K kernel, int nthreads, int smem, unsigned grid, cudaStream_t st, Ts... args) {
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kernel), smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(nthreads);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, kernel, args...);
  note_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}
template <typename K, typename... Ts>
cudaError_t launch(K kernel, int smem, unsigned grid, cudaStream_t st, Ts... args) {
  return launch_nt(kernel, NTHREADS, smem, grid, st, args...);
}

}  // namespace tcfast
}  // namespace race
