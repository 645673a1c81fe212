// race_tc_bwd.cu -- sm_100a fast path, backward passes (non-causal).
//
// Query side (ra/backward.py:109-118 + the d_num/d_den prologue 201-209), per
// 128-token chunk, with D = phi_q . A and y = S_v dO (an MMA):
//   rho = (phi_q . y) / D          (= dO . O, no need to read O)
//   dphi_q = (y - rho A) / D,  G = [dO / D | -rho / D],  dS += Phi_q^T G
//   dx^ = dproj . W (MMA), dq = sphere-tangent(dx^) / ||q||
// Key side (ra/backward.py:122-128):
//   z = dS_v v (MMA), dphi_k = z + dA, dV = phi_k dS_v (MMA), dk as above.
#include <cstdlib>

#include "tc_fast.cuh"

namespace race {
namespace tcfast {

using namespace tc;

constexpr uint32_t ID_Y = idesc_bf16(128, 16, 0, 0);     // dO x S^T-op      (K, K)
constexpr uint32_t ID_DX = idesc_bf16(128, 128, 0, 1);   // dProj x W''      (K, MN)
constexpr uint32_t ID_DS = idesc_bf16(128, 32, 1, 1);    // dO^T x Phi~      (MN, MN)
constexpr uint32_t ID_DV = idesc_bf16(128, 128, 0, 0);   // Phi_k x dS-op    (K, K)

// ===========================================================================
// bwd query side (non-causal)
// ===========================================================================
namespace bq {
constexpr int STAGES = 2;
constexpr int STAGE_BYTES = 2 * TILE;  // Q (-> dQ in place), dO
constexpr int OFF_W = STAGES * STAGE_BYTES;
constexpr int OFF_W2 = OFF_W + WOP;
constexpr int OFF_SOPT = OFF_W2 + W2OP;
constexpr int OFF_PHIT = OFF_SOPT + WOP;  // Phi_q / D   (MN-major B of dS)
constexpr int OFF_DPROJ = OFF_PHIT + PHI;
constexpr int OFF_BAR = OFF_DPROJ + PHI;
}  // namespace bq


// ===========================================================================
// bwd key side (non-causal)
// ===========================================================================
namespace bk {
constexpr int STAGES = 2;
constexpr int STAGE_BYTES = 2 * TILE;  // K (-> dK in place), V (-> dV in place)
constexpr int OFF_W = STAGES * STAGE_BYTES;
constexpr int OFF_W2 = OFF_W + WOP;
constexpr int OFF_DSOPT = OFF_W2 + W2OP;   // dS^T operand [16 x 128] (B of z = V dS_v^T)
constexpr int OFF_DSOP = OFF_DSOPT + WOP;  // dS operand [128 x 32] (B of dV = Phi_k dS_v)
constexpr int OFF_PHIK = OFF_DSOP + PHI;
constexpr int OFF_DPROJ = OFF_PHIK + PHI;
constexpr int OFF_BAR = OFF_DPROJ + PHI;
constexpr uint32_t TM_P = 0, TM_Z = 16, TM_DV = 128, TM_DX = 256;
}  // namespace bk


// ===========================================================================
// Non-causal backward, 8-compute-warp contiguous-range versions (launched).
// Same math as k_bwd_q / k_bwd_k above.  W' / W'' / the table operands are
// rebuilt only when a CTA's run enters a new sequence; per-segment dS totals
// use two TMEM accumulators (segment i accumulates while segment i - 1 is
// read out); the compute warps split each 128-column pass into halves; the
// producer issues the gradient stores right before refilling a stage.
// ===========================================================================
namespace bq8n {
using bq::STAGES;
using bq::STAGE_BYTES;
using bq::OFF_W;
using bq::OFF_W2;
using bq::OFF_SOPT;
using bq::OFF_PHIT;
using bq::OFF_DPROJ;
constexpr int OFF_X = bq::OFF_BAR;  // [2 parity][2 halves][128] norm partials, da[4][8], [2 parity][128] dx^.x^
constexpr int XDOT = 2 * 256 + 32;
constexpr int OFF_BAR = OFF_X + (XDOT + 2 * 128) * 4;
constexpr int SMEM = OFF_BAR + 256 + 1024;
constexpr uint32_t TM_P = 0, TM_Y = 16, TM_DS = 32, TM_DX = 128;  // DS: two accumulators at 32 and 64
}  // namespace bq8n

template <int P, int HB = 0, bool GRP = false, bool M4 = false>
__global__ void __launch_bounds__(NTHREADS8, 1)
    k_bwd_q8(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmDO,
             const __grid_constant__ CUtensorMap tmDQ, Args a) {
  using namespace bq8n;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* full = bars;            // [2]
  uint64_t* empty = bars + 2;       // [2] MMA done with the stage
  uint64_t* dqstaged = bars + 4;    // [2] dQ staged over Q (256 arrivals)
  uint64_t* c1 = bars + 6;          // proj + y
  uint64_t* ready = bars + 7;       // Phi~, dproj staged (256)
  uint64_t* c2 = bars + 8;          // dS += ..., dx^
  uint64_t* wready = bars + 9;      // (256)
  uint64_t* acc_full = bars + 10;   // [2]
  uint64_t* acc_empty = bars + 12;  // [2] (256)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 14);

  const int warp = warp_id();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&dqstaged[i], 256);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 256);
    }
    mbar_init(c1, 1);
    mbar_init(ready, 256);
    mbar_init(c2, 1);
    mbar_init(wready, 256);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel's tail
  int64_t i0, i1;
  cta_range(a.BH * a.nseg, i0, i1);

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmDO);
      tma_prefetch_desc(&tmDQ);
      const uint64_t pol = policy_evict_first();
      int qt[2] = {0, 0}, qb[2] = {0, 0};
      auto store_dq = [&](uint32_t j) {
        const int s = j & 1;
        mbar_wait(&dqstaged[s], (j >> 1) & 1);
        if (!a.dproj_out)  // grouped backward: dq is formed from the summed dproj afterwards
          for (int h = 0; h < 2; ++h)
            tile_store<M4>(a, &tmDQ, reinterpret_cast<void*>(smem + s * STAGE_BYTES + h * SUB), h * 64, qt[s], qb[s]);
        tma_store_commit();
      };
      uint32_t gc = 0;
      Cursor cur;
      for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
        const int s = gc & 1;
        if (gc >= 2) {
          store_dq(gc - 2);
          tma_store_wait_read<0>();
        }
        mbar_wait(&empty[s], ((gc >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        uint8_t* st = smem + s * STAGE_BYTES;
        for (int h = 0; h < 2; ++h) {
          tile_load<M4>(a, st + h * SUB, &tmQ, &full[s], h * 64, cur.t, cur.m.bh, pol);
          tile_load<M4>(a, st + TILE + h * SUB, &tmDO, &full[s], h * 64, cur.t, cur.m.bh, pol);
        }
        qt[s] = cur.t;
        qb[s] = cur.m.bh;
      }
      for (uint32_t j = gc >= 2 ? gc - 2 : 0; j < gc; ++j) store_dq(j);
      tma_store_wait_all<0>();
    }
  } else if (warp == 1) {
    uint32_t gc = 0, nr = 0, ns = 0;
    int prev_bh = -1;
    for (int64_t it = i0; it < i1; ++it, ++ns) {
      const Item m = item_of(a, it);
      if (m.bh != prev_bh) {
        prev_bh = m.bh;
        mbar_wait(wready, nr & 1);
        ++nr;
      }
      if (ns >= 2) mbar_wait(&acc_empty[ns & 1], ((ns >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t dsacc = tmem + TM_DS + 32 * (ns & 1);
      for (int t = m.t0; t < m.t1; t += CH, ++gc) {
        const int s = gc & 1;
        const uint32_t stage = sb + s * STAGE_BYTES;
        mbar_wait(&full[s], (gc >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            umma_bf16(tmem + TM_P, desc_tile_k(stage, kk), desc_w(sb + OFF_W, kk), ID_PROJ, kk > 0);
            umma_bf16(tmem + TM_Y, desc_tile_k(stage + TILE, kk), desc_w(sb + OFF_SOPT, kk), ID_Y, kk > 0);
          }
          umma_commit(c1);
        }
        __syncwarp();
        mbar_wait(ready, gc & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(dsacc, desc_tile_mn(stage + TILE, kk), desc_phi_mn(sb + OFF_PHIT, kk), ID_DS,
                      (t != m.t0 || kk > 0) ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            umma_bf16(tmem + TM_DX, desc_phi_k(sb + OFF_DPROJ, kk), desc_w2(sb + OFF_W2, kk), ID_DX, kk > 0);
          umma_commit(c2);
          umma_commit(&empty[s]);
          if (t + CH >= m.t1) umma_commit(&acc_full[ns & 1]);
        }
        __syncwarp();
      }
    }
  } else {
    const int r = crow();
    const int h = chalf();
    const int qw = warp & 3;
    const uint32_t lb = lane_base();
    const float invT = 1.f / float(a.T);
    const int F = a.T << a.P;
    float* xsq = reinterpret_cast<float*>(smem + OFF_X);
    float* xda = xsq + 512;
    float A[FP];
    uint32_t gc = 0, ns = 0;
    int prev_bh = -1;
    for (int64_t it = i0; it < i1; ++it, ++ns) {
      const Item m = item_of(a, it);
      if (m.bh != prev_bh) {
        prev_bh = m.bh;
        const float* tab = a.tin + m.bh * int64_t(F) * a.ldt;
        build_wop<256>(a, m.bh, sb + OFF_W);
        build_w2<256>(a, m.bh, sb + OFF_W2);
        float scol[FP];
#pragma unroll
        for (int f = 0; f < FP; ++f) {
          scol[f] = (f < F && r < a.dvv) ? tab[f * a.ldt + r] : 0.f;
          A[f] = f < F ? tab[f * a.ldt + a.dvv] : 0.f;
        }
        if (h == 1) write_sopT(sb + OFF_SOPT, r, scol);
        fence_proxy_async();
        mbar_arrive(wready);
      }
      float dA[FP];
#pragma unroll
      for (int f = 0; f < FP; ++f) dA[f] = 0.f;
      for (int t = m.t0; t < m.t1; t += CH, ++gc) {
        const int s = gc & 1;
        uint8_t* stage = smem + s * STAGE_BYTES;
        float* xp = xsq + (gc & 1) * 256;
        const bool valid = t + r < m.t1;
        const GroupPre pre = GRP ? group_prefetch(a, m.bh, t, r, valid) : GroupPre{};
        mbar_wait(&full[s], (gc >> 1) & 1);
        xp[h * 128 + r] = half_row_sumsq_p(stage, r, h);
        compute_bar256();
        const Scale sc = row_scale(xp[r] + xp[128 + r], a.normalize);
        mbar_wait(c1, gc & 1);
        tc_fence_after();
        float proj[16], yv[16];
        tmem_ld16(tmem + lb + TM_P, proj);
        tmem_ld16(tmem + lb + TM_Y, yv);
        tmem_ld_wait();
        float phi[FP], u[5], ph[5];
        row_features_u<P, HB>(a, proj, sc.inv, valid, phi, u, ph);
        float y[FP], D = 0.f, num = 0.f;
#pragma unroll
        for (int f = 0; f < FP; ++f) {
          y[f] = yv[f] + yv[8 + f];
          D = fmaf(phi[f], A[f], D);
          num = fmaf(phi[f], y[f], num);
        }
        const bool live = valid && D * invT > kDegenerateDenEps;
        float rD = live ? 1.f / D : 0.f;
        float rho = num * rD;
        if (GRP && a.ext_rd) {  // table / corner group: normalisers of the whole estimator
          rD = pre.rd;
          rho = rD != 0.f ? -pre.gd / rD : 0.f;
        }
        float* xdot = reinterpret_cast<float*>(smem + OFF_X) + XDOT + (gc & 1) * 128;
        if (h == 0) {
          float phit[FP];
#pragma unroll
          for (int f = 0; f < FP; ++f) {
            phit[f] = phi[f] * rD;
            dA[f] = fmaf(phi[f], -rho * rD, dA[f]);
          }
          write_phi_k(sb + OFF_PHIT, r, phit);  // [hi | hi | lo | 0]: MN-major B of dS += dO^T Phi~
        } else {  // the feature VJP once, by the second half; dx^.x^ for both halves' tangent step
          float dphi[FP];
#pragma unroll
          for (int f = 0; f < FP; ++f) dphi[f] = (y[f] - rho * A[f]) * rD;
          float dproj[8];
          row_feature_vjp<P, HB>(a, u, phi, dphi, dproj);
          if (GRP && a.dproj_out && valid) emit_dproj(a, m.bh * a.N + t + r, dproj, pre);
          xdot[r] = dot_from_proj(dproj, ph);
          write_dproj(sb + OFF_DPROJ, r, dproj);
        }
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(ready);
        mbar_wait(c2, gc & 1);
        tc_fence_after();
        tangent_half_inplace(tmem + lb + TM_DX, stage, r, h, sc, xdot[r]);
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(&dqstaged[s]);
      }
      // segment done: partial dS (lane r = value column r) from its TMEM buffer, dA by a block sum
      mbar_wait(&acc_full[ns & 1], (ns >> 1) & 1);
      tc_fence_after();
      float* out = a.tout + (m.bh * a.nseg + m.seg) * int64_t(F) * a.ldt;
      if (h == 1) {
        float acc[32];
        tmem_ld32(tmem + lb + TM_DS + 32 * (ns & 1), acc);
        tmem_ld_wait();
#pragma unroll
        for (int f = 0; f < FP; ++f)
          if (f < F && r < a.dvv) out[f * a.ldt + r] = acc[f] + acc[16 + f];
      } else {
#pragma unroll
        for (int f = 0; f < FP; ++f) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) dA[f] += __shfl_xor_sync(0xffffffffu, dA[f], o);
        }
        if (lane_id() == 0) {
#pragma unroll
          for (int f = 0; f < FP; ++f) xda[qw * FP + f] = dA[f];
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[ns & 1]);
      compute_bar256();
      if (h == 0 && r < F) out[r * a.ldt + a.dvv] = ((xda[r] + xda[FP + r]) + xda[2 * FP + r]) + xda[3 * FP + r];
      compute_bar256();  // xda is reused by the next segment
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tmem);
}

namespace bk8n {
using bk::STAGES;
using bk::STAGE_BYTES;
using bk::OFF_W;
using bk::OFF_W2;
using bk::OFF_DSOPT;
using bk::OFF_DSOP;
using bk::OFF_PHIK;
using bk::OFF_DPROJ;
constexpr int OFF_X = bk::OFF_BAR;  // [2 parity][2 halves][128] norm partials, then [2 parity][128] dx^.x^
constexpr int XDOT = 2 * 256;
constexpr int OFF_BAR = OFF_X + (XDOT + 2 * 128) * 4;
constexpr int SMEM = OFF_BAR + 256 + 1024;
using bk::TM_P;
using bk::TM_Z;
using bk::TM_DV;
using bk::TM_DX;
}  // namespace bk8n

template <int P, int HB = 0, bool GRP = false, bool M4 = false>
__global__ void __launch_bounds__(NTHREADS8, 1)
    k_bwd_k8(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
             const __grid_constant__ CUtensorMap tmDK, const __grid_constant__ CUtensorMap tmDV, Args a) {
  using namespace bk8n;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* full = bars;          // [2]
  uint64_t* empty = bars + 2;     // [2] MMA done with the stage
  uint64_t* staged = bars + 4;    // [2] dK, dV staged over K, V (256)
  uint64_t* c1 = bars + 6;
  uint64_t* ready = bars + 7;     // (256)
  uint64_t* c2 = bars + 8;
  uint64_t* wready = bars + 9;    // (256)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 10);

  const int warp = warp_id();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&staged[i], 256);
    }
    mbar_init(c1, 1);
    mbar_init(ready, 256);
    mbar_init(c2, 1);
    mbar_init(wready, 256);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel's tail
  int64_t i0, i1;
  cta_range(a.BH * a.nseg, i0, i1);

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmDK);
      tma_prefetch_desc(&tmDV);
      const uint64_t pol = policy_evict_first();
      int kt[2] = {0, 0}, kb[2] = {0, 0};
      auto store_kv = [&](uint32_t j) {
        const int s = j & 1;
        mbar_wait(&staged[s], (j >> 1) & 1);
        for (int h = 0; h < 2; ++h) {
          if (!a.dproj_out)  // grouped backward: dk is formed from the summed dproj afterwards
            tile_store<M4>(a, &tmDK, reinterpret_cast<void*>(smem + s * STAGE_BYTES + h * SUB), h * 64, kt[s], kb[s]);
          tile_store<M4>(a, &tmDV, reinterpret_cast<void*>(smem + s * STAGE_BYTES + TILE + h * SUB), h * 64, kt[s], kb[s]);
        }
        tma_store_commit();
      };
      uint32_t gc = 0;
      Cursor cur;
      for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
        const int s = gc & 1;
        if (gc >= 2) {
          store_kv(gc - 2);
          tma_store_wait_read<0>();
        }
        mbar_wait(&empty[s], ((gc >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        uint8_t* st = smem + s * STAGE_BYTES;
        for (int h = 0; h < 2; ++h) {
          tile_load<M4>(a, st + h * SUB, &tmK, &full[s], h * 64, cur.t, cur.m.bh, pol);
          tile_load<M4>(a, st + TILE + h * SUB, &tmV, &full[s], h * 64, cur.t, cur.m.bh, pol);
        }
        kt[s] = cur.t;
        kb[s] = cur.m.bh;
      }
      for (uint32_t j = gc >= 2 ? gc - 2 : 0; j < gc; ++j) store_kv(j);
      tma_store_wait_all<0>();
    }
  } else if (warp == 1) {
    uint32_t gc = 0, nr = 0;
    int prev_bh = -1;
    Cursor cur;
    for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
      if (cur.m.bh != prev_bh) {
        prev_bh = cur.m.bh;
        mbar_wait(wready, nr & 1);
        ++nr;
      }
      const int s = gc & 1;
      const uint32_t stage = sb + s * STAGE_BYTES;
      mbar_wait(&full[s], (gc >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          umma_bf16(tmem + TM_P, desc_tile_k(stage, kk), desc_w(sb + OFF_W, kk), ID_PROJ, kk > 0);
          umma_bf16(tmem + TM_Z, desc_tile_k(stage + TILE, kk), desc_w(sb + OFF_DSOPT, kk), ID_Y, kk > 0);
        }
        umma_commit(c1);
      }
      __syncwarp();
      mbar_wait(ready, gc & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          umma_bf16(tmem + TM_DV, desc_phi_k(sb + OFF_PHIK, kk), desc_phi_k(sb + OFF_DSOP, kk), ID_DV, kk > 0);
          umma_bf16(tmem + TM_DX, desc_phi_k(sb + OFF_DPROJ, kk), desc_w2(sb + OFF_W2, kk), ID_DX, kk > 0);
        }
        umma_commit(c2);
        umma_commit(&empty[s]);
      }
      __syncwarp();
    }
  } else {
    const int r = crow();
    const int h = chalf();
    const uint32_t lb = lane_base();
    const int F = a.T << a.P;
    float* xsq = reinterpret_cast<float*>(smem + OFF_X);
    float dA[FP];
    uint32_t gc = 0;
    int prev_bh = -1;
    Cursor cur;
    for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
      const Item m = cur.m;
      const int t = cur.t;
      if (m.bh != prev_bh) {
        prev_bh = m.bh;
        const float* dtab = a.tin + m.bh * int64_t(F) * a.ldt;
        build_wop<256>(a, m.bh, sb + OFF_W);
        build_w2<256>(a, m.bh, sb + OFF_W2);
        float dcol[FP];
#pragma unroll
        for (int f = 0; f < FP; ++f) {
          dcol[f] = (f < F && r < a.dvv) ? dtab[f * a.ldt + r] : 0.f;
          dA[f] = f < F ? dtab[f * a.ldt + a.dvv] : 0.f;
        }
        if (h == 1) {
          write_sopT(sb + OFF_DSOPT, r, dcol);
          write_sop(sb + OFF_DSOP, r, dcol);
        }
        fence_proxy_async();
        mbar_arrive(wready);
      }
      const int s = gc & 1;
      uint8_t* stage = smem + s * STAGE_BYTES;
      float* xp = xsq + (gc & 1) * 256;
      const bool valid = t + r < m.t1;
      const GroupPre pre = GRP ? group_prefetch(a, m.bh, t, r, valid) : GroupPre{};
      mbar_wait(&full[s], (gc >> 1) & 1);
      xp[h * 128 + r] = half_row_sumsq_p(stage, r, h);
      compute_bar256();
      const Scale sc = row_scale(xp[r] + xp[128 + r], a.normalize);
      mbar_wait(c1, gc & 1);
      tc_fence_after();
      float proj[16], zv[16];
      tmem_ld16(tmem + lb + TM_P, proj);
      tmem_ld16(tmem + lb + TM_Z, zv);
      tmem_ld_wait();
      float phi[FP], u[5], ph[5];
      row_features_u<P, HB>(a, proj, sc.inv, valid, phi, u, ph);
      float* xdot = reinterpret_cast<float*>(smem + OFF_X) + XDOT + (gc & 1) * 128;
      if (h == 0) {
        write_phi_q(sb + OFF_PHIK, r, phi);  // [hi | lo | hi | 0] pairs with dS-op [hi | hi | lo | 0]
      } else {  // the feature VJP once, by the second half; dx^.x^ for both halves' tangent step
        float dphi[FP];
#pragma unroll
        for (int f = 0; f < FP; ++f) dphi[f] = zv[f] + zv[8 + f] + dA[f];
        float dproj[8];
        row_feature_vjp<P, HB>(a, u, phi, dphi, dproj);
        if (GRP && a.dproj_out && valid) emit_dproj(a, m.bh * a.N + t + r, dproj, pre);
        xdot[r] = dot_from_proj(dproj, ph);
        write_dproj(sb + OFF_DPROJ, r, dproj);
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(ready);
      mbar_wait(c2, gc & 1);
      tc_fence_after();
#pragma unroll
      for (int b = 0; b < 2; ++b) {  // dV over the dead V row (my 64 columns)
        const int c0 = 64 * h + 32 * b;
        float v[32];
        tmem_ld32(tmem + lb + TM_DV + c0, v);
        tmem_ld_wait();
        stage32_p(stage + TILE, r, v, c0);
      }
      tangent_half_inplace(tmem + lb + TM_DX, stage, r, h, sc, xdot[r]);
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&staged[s]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace tcfast

// ---- entry points ------------------------------------------------------------
cudaError_t tc_bwd_q(const Geo& g, const void* q, const void* d_o, const float* w, const float* tab, void* dq,
                     float* dpart, cudaStream_t st) {
  using namespace tcfast;
  CUtensorMap mq, mdo, mdq;
  if (!make_map(&mq, q, g, g.d, L_Q) || !make_map(&mdo, d_o, g, g.dv, L_DO) || !make_map(&mdq, dq, g, g.d, L_DQ))
    return cudaErrorInvalidValue;
  Args a = make_args(g);
  a.w = w;
  a.tin = tab;
  a.tout = dpart;
  a.dproj_out = g.dproj_q;
  const bool grp = g.ext_rden || g.dproj_q;  // a pass of a grouped backward (race_abi.cu)
#define RACE_BQ8(...) return launch_nt(k_bwd_q8<__VA_ARGS__>, NTHREADS8, bq8n::SMEM, grid_for(g), st, mq, mdo, mdq, a)
  switch (pass_corner_bits(g)) {
    case 1: if (g.strided()) RACE_BQ8(1, 0, false, true); if (grp) RACE_BQ8(1, 0, true); RACE_BQ8(1);
    case 2: if (g.strided()) RACE_BQ8(2, 0, false, true); if (grp) RACE_BQ8(2, 0, true); RACE_BQ8(2);
    default:
      if (g.strided()) RACE_BQ8(3, 0, false, true);  // strided operands: one-pass problems only
      if (g.cb) RACE_BQ8(3, 2, true);
      if (grp) RACE_BQ8(3, 0, true);
      RACE_BQ8(3);
  }
#undef RACE_BQ8
}

cudaError_t tc_bwd_k(const Geo& g, const void* k, const void* v, const float* w, const float* dtab, void* dk,
                     void* dv, cudaStream_t st) {
  using namespace tcfast;
  CUtensorMap mk, mv, mdk, mdv;
  if (!make_map(&mk, k, g, g.d, L_K) || !make_map(&mv, v, g, g.dv, L_V) || !make_map(&mdk, dk, g, g.d, L_DK) ||
      !make_map(&mdv, dv, g, g.dv, L_DV))
    return cudaErrorInvalidValue;
  Args a = make_args(g);
  a.w = w;
  a.tin = dtab;
  a.dproj_out = g.dproj_k;
  const bool grp = g.ext_rden || g.dproj_k;
#define RACE_BK8(...) \
  return launch_nt(k_bwd_k8<__VA_ARGS__>, NTHREADS8, bk8n::SMEM, grid_for(g), st, mk, mv, mdk, mdv, a)
  switch (pass_corner_bits(g)) {
    case 1: if (g.strided()) RACE_BK8(1, 0, false, true); if (grp) RACE_BK8(1, 0, true); RACE_BK8(1);
    case 2: if (g.strided()) RACE_BK8(2, 0, false, true); if (grp) RACE_BK8(2, 0, true); RACE_BK8(2);
    default:
      if (g.strided()) RACE_BK8(3, 0, false, true);  // strided operands: one-pass problems only
      if (g.cb) RACE_BK8(3, 2, true);
      if (grp) RACE_BK8(3, 0, true);
      RACE_BK8(3);
  }
#undef RACE_BK8
}

}  // namespace race
