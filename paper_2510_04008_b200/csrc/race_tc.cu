// race_tc.cu -- sm_100a fast path: persistent, warp-specialised kernels with
// TMA loads/stores, tcgen05 MMAs accumulating in TMEM, and the soft-LSH
// features computed in registers (the N x F assignment never reaches HBM).
//
// Scope: bf16 inputs, d = dv = 128, F = T * 2^P <= 8 (the reference default
// P=2, L=2 is F=8), any N and B*H.  Everything else runs on the generic
// kernels in race_simt.cu.
//
// CTA = 6 warps: warp 0 TMA producer, warp 1 MMA issuer (+ TMEM owner),
// warps 2..5 compute (thread r <-> token r of the 128-token chunk <-> TMEM
// lane r).  Work items are (b*h, segment) pairs (race_segments), taken
// round-robin by a persistent grid of one CTA per SM.
//
// Precision: the projection x.W must be fp32-exact, so W
// enters the MMA as three bf16 pieces (W_hi + W_mid + W_lo = W to 24 bits;
// bf16 x bf16 products are exact in fp32).  phi and the bucket tables enter
// as hi/lo bf16 pairs (16-bit mantissa); only the causal intra-chunk matrix
// tril(Phi_q Phi_k^T) is rounded to bf16 before multiplying V.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tc_fast.cuh"

namespace race {
namespace tcfast {

using namespace tc;

// ===========================================================================
// K1: key-side aggregation per segment (non-causal tables / causal segment totals)
// ===========================================================================
namespace agg {
constexpr int STAGES = 3;
constexpr int STAGE_BYTES = 2 * TILE;  // K, V
constexpr int OFF_STAGE = 0;
constexpr int OFF_W = STAGES * STAGE_BYTES;
constexpr int OFF_PHI = OFF_W + WOP;         // 2 buffers
constexpr int OFF_BAR = OFF_PHI + 2 * PHI;
}  // namespace agg


// ---------------------------------------------------------------------------
// K1, contiguous-range version (the one launched).  Each CTA walks a
// contiguous run of (b*h, segment) items, so W' is rebuilt only when the run
// enters a new sequence, and the per-segment accumulator is double-buffered
// in TMEM: segment i accumulates into SACC[i & 1] while the compute warps
// read out segment i - 1, so the MMA never waits for the read-out.
// ---------------------------------------------------------------------------
namespace agg2 {
using agg::STAGES;
using agg::STAGE_BYTES;
using agg::OFF_STAGE;
using agg::OFF_W;
using agg::OFF_PHI;
constexpr int OFF_BAR = agg::OFF_BAR;
constexpr int OFF_XS = OFF_BAR + 256;  // [2 segment parities][8 warps][FP] phi column sums
constexpr int SMEM = OFF_XS + 2 * 8 * FP * 4 + 1024;
static_assert(SMEM <= 232448, "k_aggregate2 shared memory");
constexpr uint32_t TM_PK = 0, TM_ACC = 32;  // accumulators at 32 and 64
}  // namespace agg2

template <int P, int HB = 0, bool M4 = false>
__global__ void __launch_bounds__(NTHREADS8, 1)
    k_aggregate2(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, Args a) {
  using namespace agg2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* full = bars;               // [STAGES]
  uint64_t* empty = bars + STAGES;     // [STAGES]
  uint64_t* proj_full = bars + 2 * STAGES;  // [2] projections of chunk g in TM_PK + 16 (g & 1)
  uint64_t* phi_full = proj_full + 2;  // [2] (128 arrivals: the warp group owning the chunk)
  uint64_t* phi_empty = phi_full + 2;  // [2]
  uint64_t* wready = phi_empty + 2;
  uint64_t* acc_full = wready + 1;     // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint64_t* pk_empty = acc_empty + 2;  // [2] projection buffer read (128 arrivals)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(pk_empty + 2);

  const int warp = warp_id();
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&phi_full[i], 128);
      mbar_init(&proj_full[i], 1);
      mbar_init(&phi_empty[i], 1);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
      mbar_init(&pk_empty[i], 128);
    }
    mbar_init(wready, 256);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<128>(tslot);
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
      const uint64_t pol = policy_evict_first();
      uint32_t gc = 0;
      Cursor cur;
      for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
        const int s = gc % STAGES;
        mbar_wait(&empty[s], ((gc / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        uint8_t* st = smem + OFF_STAGE + s * STAGE_BYTES;
        for (int h = 0; h < 2; ++h) {
          tile_load<M4>(a, st + h * SUB, &tmK, &full[s], h * 64, cur.t, cur.m.bh, pol);
          tile_load<M4>(a, st + TILE + h * SUB, &tmV, &full[s], h * 64, cur.t, cur.m.bh, pol);
        }
      }
    }
  } else if (warp == 1) {
    // The projection of chunk g + 1 is issued before the state MMA of chunk g waits for phi (two
    // TMEM projection buffers), so the compute warps find it ready; never across a sequence
    // change, where W' is rebuilt by the compute warps.
    uint32_t gc = 0, nr = 0, ns = 0, pg = 0;
    int pbh = -1;
    Cursor pc;
    pc.start(a, i0, i1);
    auto issue_proj = [&]() {  // projection of chunk pg (cursor pc)
      if (pc.m.bh != pbh) {
        pbh = pc.m.bh;
        mbar_wait(wready, nr & 1);
        ++nr;
      }
      const int s = pg % STAGES;
      mbar_wait(&full[s], (pg / STAGES) & 1);
      if (pg >= 2) mbar_wait(&pk_empty[pg & 1], ((pg >> 1) - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t stage = sb + OFF_STAGE + s * STAGE_BYTES;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(tmem + TM_PK + 16 * (pg & 1), desc_tile_k(stage, kk), desc_w(sb + OFF_W, kk), ID_PROJ, kk > 0);
        umma_commit(&proj_full[pg & 1]);
      }
      __syncwarp();
      pc.next(a);
      ++pg;
    };
    for (int64_t it = i0; it < i1; ++it, ++ns) {
      const Item m = item_of(a, it);
      if (ns >= 2) mbar_wait(&acc_empty[ns & 1], ((ns >> 1) - 1) & 1);  // segment ns - 2 read out
      tc_fence_after();
      const uint32_t acc = tmem + TM_ACC + 32 * (ns & 1);
      for (int t = m.t0; t < m.t1; t += CH, ++gc) {
        const int s = gc % STAGES;
        const uint32_t stage = sb + OFF_STAGE + s * STAGE_BYTES;
        if (pg == gc) issue_proj();                              // this chunk (first, or new sequence)
        if (pc.ok() && pc.m.bh == int64_t(m.bh)) issue_proj();  // the next one, same sequence
        mbar_wait(&phi_full[gc & 1], (gc >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t phib = sb + OFF_PHI + (gc & 1) * PHI;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(acc, desc_tile_mn(stage + TILE, kk), desc_phi_mn(phib, kk), ID_STATE,
                      (t != m.t0 || kk > 0) ? 1u : 0u);
          umma_commit(&empty[s]);
          umma_commit(&phi_empty[gc & 1]);
          if (t + CH >= m.t1) umma_commit(&acc_full[ns & 1]);
        }
        __syncwarp();
      }
    }
  } else {
    // 8 compute warps in two groups: warps 2-5 take the even chunks, warps 6-9 the odd ones, so
    // one group's features overlap the other's waits (each SMSP holds one warp of each group)
    const int r = crow();
    const int grp = chalf();
    const int F = a.T << a.P;
    float* xs = reinterpret_cast<float*>(smem + OFF_XS);
    uint32_t gc = 0, ns = 0;
    int prev_bh = -1;
    for (int64_t it = i0; it < i1; ++it, ++ns) {
      const Item m = item_of(a, it);
      if (m.bh != prev_bh) {
        prev_bh = m.bh;
        build_wop<256, CT0>(a, m.bh, sb + OFF_W);
        fence_proxy_async();
        mbar_arrive(wready);
      }
      float asum[FP];
#pragma unroll
      for (int f = 0; f < FP; ++f) asum[f] = 0.f;
      for (int t = m.t0; t < m.t1; t += CH, ++gc) {
        if (int(gc & 1) != grp) continue;
        const int s = gc % STAGES;
        const uint32_t stage = sb + OFF_STAGE + s * STAGE_BYTES;
        mbar_wait(&full[s], (gc / STAGES) & 1);
        const float sumsq = tile_row_sumsq(stage, r);
        const float inv = inv_scale(sumsq, a.normalize);
        mbar_wait(&proj_full[gc & 1], (gc >> 1) & 1);
        tc_fence_after();
        float proj[16];
        tmem_ld16(tmem + lane_base() + TM_PK + 16 * (gc & 1), proj);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&pk_empty[gc & 1]);
        float phi[FP];
        row_features<P, HB>(a, proj, inv, t + r < m.t1, phi);
#pragma unroll
        for (int f = 0; f < FP; ++f) asum[f] += phi[f];
        if (gc >= 2) mbar_wait(&phi_empty[gc & 1], ((gc >> 1) - 1) & 1);
        write_phi_k(sb + OFF_PHI + (gc & 1) * PHI, r, phi);
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(&phi_full[gc & 1]);
        if (a.rows_out && t + r < m.t1) {  // causal: the k half of this key's sketch row (off the MMA chain)
          float hat[5];
          row_hat(a, proj, inv, hat);
          store_row_half(a.rows_out + (int64_t(m.bh) * a.N + t + r) * ROWW + 8, hat, sumsq);
        }
      }
      // segment done: phi column sums of both groups (fixed order), S^T (lane r = value column r)
      // from its TMEM buffer read out by group 0
      float* xp = xs + (ns & 1) * 8 * FP;
#pragma unroll
      for (int f = 0; f < FP; ++f) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) asum[f] += __shfl_xor_sync(0xffffffffu, asum[f], o);
      }
      if (lane_id() == 0) {
#pragma unroll
        for (int f = 0; f < FP; ++f) xp[(warp - 2) * FP + f] = asum[f];
      }
      compute_bar256();
      if (grp == 0) {
        mbar_wait(&acc_full[ns & 1], (ns >> 1) & 1);
        tc_fence_after();
        float acc[32];
        tmem_ld32(tmem + lane_base() + TM_ACC + 32 * (ns & 1), acc);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&acc_empty[ns & 1]);
        float* out = a.tout + (m.bh * a.nseg + m.seg) * int64_t(F) * a.ldt;
#pragma unroll
        for (int f = 0; f < FP; ++f)
          if (f < F && r < a.dvv) out[f * a.ldt + r] = acc[f] + acc[16 + f];
        if (r < F) {
          float tot = 0.f;
#pragma unroll
          for (int w = 0; w < 8; ++w) tot += xp[w * FP + r];
          out[r * a.ldt + a.dvv] = tot;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<128>(tmem);
}

// ===========================================================================
// K2: non-causal query-side readout  O = Phi_q S_v / (Phi_q A), den = D / T
// ===========================================================================


// ---------------------------------------------------------------------------
// K2, 8-compute-warp contiguous-range version (the one launched): W' and the
// S operand are rebuilt only when the CTA's run enters a new sequence; each
// half of the compute warps handles 64 columns of every row pass (row norm
// halves exchanged through shared memory); the producer issues the O store
// right before refilling that Q buffer, so no compute warp waits on it.
// ---------------------------------------------------------------------------
namespace rdo8 {
constexpr int STAGES = 6;             // Q tiles in flight (each reused as its O staging)
constexpr int STAGE_BYTES = TILE;
constexpr int OFF_STAGE = 0;
constexpr int OFF_W = STAGES * STAGE_BYTES;
constexpr int OFF_PHI = OFF_W + WOP;  // 2 buffers
constexpr int OFF_SOP = OFF_PHI + 2 * PHI;
constexpr int OFF_X = OFF_SOP + PHI;  // [2 parity][2 halves][128] row-norm partials, then [2 parity][128] D
constexpr int OFF_BAR = OFF_X + 2 * 256 * 4 + 2 * 128 * 4;
constexpr int SMEM = OFF_BAR + 256 + 1024;
static_assert(SMEM <= 232448, "k_readout8 shared memory");
constexpr uint32_t TM_NUM_R = 128;
}  // namespace rdo8

template <int P, int HB = 0, bool M4 = false>
__global__ void __launch_bounds__(NTHREADS8, 1)
    k_readout8(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO, Args a) {
  using namespace rdo8;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* full = bars;                    // [STAGES]
  uint64_t* empty = bars + STAGES;          // [STAGES] (MMA done with the Q tile)
  uint64_t* ostaged = bars + 2 * STAGES;    // [STAGES] (O staged, 256 arrivals)
  uint64_t* proj_full = bars + 3 * STAGES;
  uint64_t* phi_full = proj_full + 1;
  uint64_t* phi_empty = phi_full + 1;       // [2]
  uint64_t* wready = phi_empty + 2;
  uint64_t* num_full = wready + 1;          // [2] (per NUM buffer: the compute warps run one chunk ahead)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(num_full + 2);

  const int warp = warp_id();
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&ostaged[i], 256);
    }
    mbar_init(proj_full, 1);
    mbar_init(phi_full, 256);
    mbar_init(&phi_empty[0], 1);
    mbar_init(&phi_empty[1], 1);
    mbar_init(wready, 256);
    mbar_init(&num_full[0], 1);
    mbar_init(&num_full[1], 1);
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
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmO);
      const uint64_t pol = policy_evict_first();
      int ot[STAGES], ob[STAGES];
      auto store_o = [&](uint32_t j) {  // O of chunk j, staged in its Q tile
        const int s = j % STAGES;
        mbar_wait(&ostaged[s], (j / STAGES) & 1);
        for (int h = 0; h < 2; ++h)
          tile_store<M4>(a, &tmO, reinterpret_cast<void*>(smem + OFF_STAGE + s * STAGE_BYTES + h * SUB), h * 64, ot[s], ob[s]);
        tma_store_commit();
      };
      uint32_t gc = 0;
      Cursor cur;
      for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
        const int s = gc % STAGES;
        if (gc >= STAGES) {
          store_o(gc - STAGES);
          tma_store_wait_read<0>();
        }
        mbar_wait(&empty[s], ((gc / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        uint8_t* st = smem + OFF_STAGE + s * STAGE_BYTES;
        for (int h = 0; h < 2; ++h) tile_load<M4>(a, st + h * SUB, &tmQ, &full[s], h * 64, cur.t, cur.m.bh, pol);
        ot[s] = cur.t;
        ob[s] = cur.m.bh;
      }
      for (uint32_t j = gc >= STAGES ? gc - STAGES : 0; j < gc; ++j) store_o(j);
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
      const int s = gc % STAGES;
      const uint32_t stage = sb + OFF_STAGE + s * STAGE_BYTES;
      mbar_wait(&full[s], (gc / STAGES) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(tmem + TM_PROJQ, desc_tile_k(stage, kk), desc_w(sb + OFF_W, kk), ID_PROJ, kk > 0);
        umma_commit(proj_full);
        umma_commit(&empty[s]);
      }
      __syncwarp();
      mbar_wait(phi_full, gc & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t phib = sb + OFF_PHI + (gc & 1) * PHI;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
          umma_bf16(tmem + TM_NUM_R + 128 * (gc & 1), desc_phi_k(phib, kk), desc_phi_k(sb + OFF_SOP, kk), ID_NUMA,
                    kk > 0);
        umma_commit(&num_full[gc & 1]);
        umma_commit(&phi_empty[gc & 1]);
      }
      __syncwarp();
    }
  } else {
    // Software-pipelined: the front half of chunk c + 1 (row norms, features, Phi_q,
    // den) runs before the back half of chunk c (numerator read-out), so the numerator
    // MMA of c + 1 overlaps the read-out of c (two NUM buffers in TMEM).
    const int r = crow();
    const int h = chalf();
    const uint32_t lb = lane_base();
    const float invT = 1.f / float(a.T);
    const int F = a.T << a.P;
    float* xsq = reinterpret_cast<float*>(smem + OFF_X);
    float A[FP];
    int prev_bh = -1;
    auto front = [&](const Cursor& c, uint32_t g) -> float {  // returns 1/D of row r
      const Item m = c.m;
      if (m.bh != prev_bh) {  // W' and S operand of this sequence (no MMA of the old one in flight)
        prev_bh = m.bh;
        const float* tab = a.tin + m.bh * int64_t(F) * a.ldt;
        build_wop<256>(a, m.bh, sb + OFF_W);
        float srow[FP];
#pragma unroll
        for (int f = 0; f < FP; ++f) {
          srow[f] = (f < F && r < a.dvv) ? tab[f * a.ldt + r] : 0.f;
          A[f] = f < F ? tab[f * a.ldt + a.dvv] : 0.f;
        }
        if (h == 1) write_sop(sb + OFF_SOP, r, srow);
        fence_proxy_async();
        mbar_arrive(wready);
      }
      const int s = g % STAGES;
      uint8_t* stage = smem + OFF_STAGE + s * STAGE_BYTES;
      float* xp = xsq + (g & 1) * 256;
      mbar_wait(&full[s], (g / STAGES) & 1);
      xp[h * 128 + r] = half_row_sumsq_p(stage, r, h);
      compute_bar256();
      const float inv = inv_scale(xp[r] + xp[128 + r], a.normalize);
      mbar_wait(proj_full, g & 1);
      tc_fence_after();
      const bool valid = c.t + r < m.t1;
      float D = 0.f;
      if (h == 0) {  // phi_q and D once, by the first half (the second half takes D in back())
        float proj[16];
        tmem_ld16(tmem + lb + TM_PROJQ, proj);
        tmem_ld_wait();
        float phi[FP];
        row_features<P, HB>(a, proj, inv, valid, phi);
#pragma unroll
        for (int f = 0; f < FP; ++f) D = fmaf(phi[f], A[f], D);
        xsq[512 + (g & 1) * 128 + r] = D;
        if (g >= 2) mbar_wait(&phi_empty[g & 1], ((g >> 1) - 1) & 1);
        write_phi_q(sb + OFF_PHI + (g & 1) * PHI, r, phi);
        fence_proxy_async();
      }
      tc_fence_before();
      mbar_arrive(phi_full);
      if (h == 0 && valid) a.den[m.bh * a.N + c.t + r] = D * invT;
      return (D * invT > kDegenerateDenEps) ? 1.f / D : 0.f;
    };
    auto back = [&](uint32_t g, float rD) {
      const int s = g % STAGES;
      uint8_t* stage = smem + OFF_STAGE + s * STAGE_BYTES;
      mbar_wait(&num_full[g & 1], (g >> 1) & 1);
      if (h == 1) {  // D of this chunk from the first half (written before its phi_full arrival)
        const float D = xsq[512 + (g & 1) * 128 + r];
        rD = (D * invT > kDegenerateDenEps) ? 1.f / D : 0.f;
      }
      tc_fence_after();
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int c0 = 64 * h + 32 * b;
        float v[32];
        tmem_ld32(tmem + lb + TM_NUM_R + 128 * (g & 1) + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= rD;
        stage32_p(stage, r, v, c0);  // the Q tile is dead (proj done, norms read): O staging
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&ostaged[s]);
    };
    uint32_t gc = 0;
    Cursor cur;
    cur.start(a, i0, i1);
    float rD = cur.ok() ? front(cur, 0) : 0.f;
    while (cur.ok()) {
      Cursor nx = cur;
      nx.next(a);
      if (nx.ok() && nx.m.bh == cur.m.bh) {
        const float rDn = front(nx, gc + 1);
        back(gc, rD);
        rD = rDn;
      } else {  // the next chunk rebuilds the S operand: finish this one first
        back(gc, rD);
        if (nx.ok()) rD = front(nx, gc + 1);
      }
      cur = nx;
      ++gc;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ===========================================================================
// K3: causal forward, chunked scan with carry-in per segment
//   num_c = Phi_q,c S_<c + tril(Phi_q,c Phi_k,c^T) V_c,   S_<c+1 = S_<c + Phi_k,c^T [V_c | 1]
// ===========================================================================
namespace cfw {
constexpr int STAGES = 2;
constexpr int STAGE_BYTES = 3 * TILE;  // Q (-> P~), K (-> O staging), V
constexpr int OFF_STAGE = 0;
constexpr int OFF_W = STAGES * STAGE_BYTES;
constexpr int OFF_PHIQ = OFF_W + WOP;
constexpr int OFF_PHIK = OFF_PHIQ + PHI;
constexpr int OFF_SOP = OFF_PHIK + PHI;
constexpr int OFF_BAR = OFF_SOP + PHI;
}  // namespace cfw

// ---------------------------------------------------------------------------
// K3, pipelined 8-compute-warp version (the one launched).
//
// Warps: 0 = TMA producer AND O-store issuer, 1 = MMA issuer, 2..9 = compute.
// Warp w and w + 4 share TMEM lane quarter w % 4 (token rows) and split each
// 128-column pass into halves h = chalf(): h = 0 owns the q-row norm and
// columns 0..63; h = 1 the k-row norm, columns 64..127, the S operand and the
// chunk total of phi_k.
//
// Each CTA walks a CONTIGUOUS range of (b*h, segment) items, so the bucket
// state S / A simply continues in TMEM / registers from one segment to the
// next; carries are loaded only when the range starts or crosses into a new
// sequence.
//
// Buffer recycling is what bounds this kernel, so each tile is released as
// early as possible: the Q and K tiles of chunk c only feed the projection MMA
// and the row norms (computed one chunk ahead, while the previous numerator
// MMA runs), so they are refilled with chunk c + 2 right after proj(c); the
// intra-chunk weights P~ = tril(Phi_q Phi_k^T) go to TMEM and enter the
// numerator MMA as its A operand (tcgen05.mma [d], [a], b); O is staged in
// the V tile once the numerator MMA has consumed it, and the producer issues
// the TMA store itself just before refilling that tile.
// ---------------------------------------------------------------------------
namespace cfw8 {
using cfw::STAGES;
using cfw::STAGE_BYTES;
using cfw::OFF_STAGE;
using cfw::OFF_W;
using cfw::OFF_PHIQ;
using cfw::OFF_PHIK;
using cfw::OFF_SOP;
constexpr int OFF_X = cfw::OFF_BAR;  // [2 parity] x { sq[2][128], rs[2][128], kp[4][8], phi_q.A[128] } floats
constexpr int XPAR = 256 + 256 + 32 + 128;
constexpr int OFF_BAR = OFF_X + 2 * XPAR * 4;
constexpr int SMEM = OFF_BAR + 256 + 1024;
constexpr uint32_t TM_PA = 192;  // P~ as bf16 pairs: 128 lanes x 64 columns
static_assert(SMEM <= 232448, "k_causal_fwd8 shared memory");
}  // namespace cfw8

// KR: the k halves of the sketch rows were written by the key-side aggregation (k_aggregate2),
// so this pass reads Q, V and those rows instead of K (no K tile, no K projection).
template <int P, bool KR, int HB = 0, bool M4 = false>
__global__ void __launch_bounds__(NTHREADS8, 1)
    k_causal_fwd8(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                  const __grid_constant__ CUtensorMap tmROWS, Args a) {
  using namespace cfw8;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* fullqk = bars;       // [2]  Q, K bytes landed
  uint64_t* fullv = bars + 2;    // [2]  V bytes landed
  uint64_t* emptyqk = bars + 4;  // [2]  proj MMA done (commit) + row norms done (1 arrive)
  uint64_t* ostaged = bars + 6;  // [2]  O staged in the V tile (256 arrivals)
  uint64_t* proj_full = bars + 8;
  uint64_t* phi_full = bars + 9;
  uint64_t* pm_full = bars + 10;
  uint64_t* pt_full = bars + 11;
  uint64_t* num_full = bars + 12;
  uint64_t* wready = bars + 13;
  uint64_t* st_full = bars + 14;  // state MMA S += V^T phi_k done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 15);

  const int warp = warp_id();
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&fullqk[i], 1);
      mbar_init(&fullv[i], 1);
      mbar_init(&emptyqk[i], 2);
      mbar_init(&ostaged[i], 256);
    }
    mbar_init(proj_full, 1);
    mbar_init(phi_full, 256);
    mbar_init(pm_full, 1);
    mbar_init(pt_full, 256);
    mbar_init(num_full, 1);
    mbar_init(st_full, 1);
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
  if (threadIdx.x == 0) RACE_CTA_TIME(a, 0);

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmO);
      const uint64_t pol = policy_evict_first();
      int ot0 = 0, ob0 = 0, ot1 = 0, ob1 = 0;  // coordinates of the O tile held by each stage
      auto store_o = [&](uint32_t j) {             // O of chunk j (V tile of stage j & 1)
        const int s = j & 1;
        mbar_wait(&ostaged[s], (j >> 1) & 1);
        const int ot = int(s ? ot1 : ot0), ob = int(s ? ob1 : ob0);
        for (int h = 0; h < 2; ++h)
          tile_store<M4>(a, &tmO, reinterpret_cast<void*>(smem + OFF_STAGE + s * STAGE_BYTES + 2 * TILE + h * SUB),
                       h * 64, ot, ob);
        tma_store_commit();
      };
      uint32_t gc = 0;
      Cursor cur;
      for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
        const int s = gc & 1;
        uint8_t* st = smem + OFF_STAGE + s * STAGE_BYTES;
        if (a.pf > 0) {  // warm L2 with the tiles a.pf chunks ahead (same sequence; a hint only)
          const int tp = int(cur.t) + a.pf * CH;
          if (tp < a.N)
            for (int h = 0; h < 2; ++h) {
              tile_prefetch<M4>(a, &tmQ, h * 64, tp, int(cur.m.bh));
              tile_prefetch<M4>(a, &tmK, h * 64, tp, int(cur.m.bh));
              tile_prefetch<M4>(a, &tmV, h * 64, tp, int(cur.m.bh));
            }
        }
        mbar_wait(&emptyqk[s], ((gc >> 1) & 1) ^ 1);
        RACE_TRACE(a, 0, gc);
        if (KR) {  // Q tile + the chunk's sketch rows (in the unused K slot)
          mbar_arrive_expect_tx(&fullqk[s], TILE + CH * ROWW * 4);
          for (int h = 0; h < 2; ++h) tile_load<M4>(a, st + h * SUB, &tmQ, &fullqk[s], h * 64, int(cur.t), int(cur.m.bh), pol);
          tma_load_2d(st + TILE, &tmROWS, &fullqk[s], 0, int(cur.m.bh) * int(a.N) + int(cur.t), pol);
        } else {
          mbar_arrive_expect_tx(&fullqk[s], 2 * TILE);
          for (int h = 0; h < 2; ++h) {
            tile_load<M4>(a, st + h * SUB, &tmQ, &fullqk[s], h * 64, int(cur.t), int(cur.m.bh), pol);
            tile_load<M4>(a, st + TILE + h * SUB, &tmK, &fullqk[s], h * 64, int(cur.t), int(cur.m.bh), pol);
          }
        }
        if (gc >= 2) {
          store_o(gc - 2);
          tma_store_wait_read<0>();
        }
        RACE_TRACE(a, 9, gc);
        mbar_arrive_expect_tx(&fullv[s], TILE);
        for (int h = 0; h < 2; ++h)
          tile_load<M4>(a, st + 2 * TILE + h * SUB, &tmV, &fullv[s], h * 64, int(cur.t), int(cur.m.bh), pol);
        if (s) { ot1 = cur.t; ob1 = cur.m.bh; } else { ot0 = cur.t; ob0 = cur.m.bh; }
      }
      for (uint32_t j = gc >= 2 ? gc - 2 : 0; j < gc; ++j) store_o(j);
      tma_store_wait_all<0>();
    }
  } else if (warp == 1) {
    uint32_t gc = 0, nr = 0;
    int64_t prev_bh = -1;
    for (int64_t it = i0; it < i1; ++it) {
      const Item m = item_of(a, it);
      if (m.bh != prev_bh) {  // compute warps (re)built W, S, A for this sequence
        prev_bh = m.bh;
        mbar_wait(wready, nr & 1);
        ++nr;
        tc_fence_after();
      }
      for (int64_t t = m.t0; t < m.t1; t += CH, ++gc) {
        const int s = gc & 1;
        const uint32_t stage = sb + OFF_STAGE + s * STAGE_BYTES;
        mbar_wait(&fullqk[s], (gc >> 1) & 1);
        RACE_TRACE(a, 1, gc);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            umma_bf16(tmem + TM_PROJQ, desc_tile_k(stage, kk), desc_w(sb + OFF_W, kk), ID_PROJ, kk > 0);
            if (!KR) umma_bf16(tmem + TM_PROJK, desc_tile_k(stage + TILE, kk), desc_w(sb + OFF_W, kk), ID_PROJ, kk > 0);
          }
          umma_commit(proj_full);
          umma_commit(&emptyqk[s]);
        }
        __syncwarp();
        mbar_wait(phi_full, gc & 1);
        RACE_TRACE(a, 2, gc);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            umma_bf16(tmem + TM_PM, desc_phi_k(sb + OFF_PHIQ, kk), desc_phi_k(sb + OFF_PHIK, kk), ID_PM, kk > 0);
          umma_commit(pm_full);  // P~ staging needs only Pm; the state update runs behind it
        }
        __syncwarp();
        mbar_wait(&fullv[s], (gc >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(tmem + TM_SACC, desc_tile_mn(stage + 2 * TILE, kk), desc_phi_mn(sb + OFF_PHIK, kk), ID_STATE, 1u);
          umma_commit(st_full);
        }
        __syncwarp();
        mbar_wait(pt_full, gc & 1);
        RACE_TRACE(a, 3, gc);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            umma_bf16(tmem + TM_NUM, desc_phi_k(sb + OFF_PHIQ, kk), desc_phi_k(sb + OFF_SOP, kk), ID_NUMA, kk > 0);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts(tmem + TM_NUM, tmem + TM_PA + kk * 8, desc_tile_mn(stage + 2 * TILE, kk), ID_NUMB, 1u);
          umma_commit(num_full);
        }
        __syncwarp();
      }
    }
  } else {
    const int r = crow();
    const int h = chalf();
    const int qw = warp & 3;  // lane quarter: rows 32qw..32qw+31
    const uint32_t lb = lane_base();
    const float invT = 1.f / float(a.T);
    const int F = a.T << a.P;
    float* xbase = reinterpret_cast<float*>(smem + OFF_X);
    {  // P~ blocks above the diagonal are never written: zero the A operand once
      uint32_t z[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) z[j] = 0u;
      tmem_st16u(tmem + lb + TM_PA + 32 * h, z);
      tmem_st16u(tmem + lb + TM_PA + 32 * h + 16, z);
      tmem_st_wait();
    }
    float A[FP], snext[FP];
    float sqq = 0.f, sqk = 0.f;  // row norms^2 of the current chunk
    float hk[5];                 // KR: stored k projections of the current chunk (h == 1)
    // row norm^2 of my row of the chunk held by stage sn; KR + h == 1: read from the sketch row
    auto stage_norm = [&](int sn) -> float {
      if (KR && h == 1) {
        const float* rw = reinterpret_cast<const float*>(smem + OFF_STAGE + sn * STAGE_BYTES + TILE) + r * ROWW + 8;
        const float4 x0 = reinterpret_cast<const float4*>(rw)[0];
        const float4 x1 = reinterpret_cast<const float4*>(rw)[1];
        hk[0] = x0.x; hk[1] = x0.y; hk[2] = x0.z; hk[3] = x0.w; hk[4] = x1.x;
        return x1.w;
      }
      return tile_row_sumsq(sb + OFF_STAGE + sn * STAGE_BYTES + h * TILE, r);
    };
    uint32_t gc = 0;
    int64_t prev_bh = -1;
    Cursor cur;
    cur.start(a, i0, i1);
    if (cur.ok()) {  // norms of the very first chunk
      mbar_wait(&fullqk[0], 0);
      const float sq = stage_norm(0);
      xbase[h * 128 + r] = sq;
      compute_bar256();
      if (threadIdx.x == CT0) mbar_arrive(&emptyqk[0]);
      sqq = xbase[r];
      sqk = xbase[128 + r];
    }
    for (; cur.ok(); ++gc) {
      const Item m = cur.m;
      const int64_t t = cur.t;
      const int s = gc & 1;
      const uint32_t stage = sb + OFF_STAGE + s * STAGE_BYTES;
      float* xpar = xbase + (gc & 1) * XPAR;
      const bool valid = t + r < m.t1;
      if (m.bh != prev_bh) {  // (re)load the sequence state: W', S_in (TMEM + S operand), A_in
        prev_bh = m.bh;
        if (threadIdx.x == a.ttid) RACE_TRACE(a, 10, gc);
        const float* car = a.tin + (m.bh * a.nseg + m.seg) * int64_t(F) * a.ldt;
        float srow[FP];
#pragma unroll
        for (int f = 0; f < FP; ++f) {
          A[f] = f < F ? car[f * a.ldt + a.dvv] : 0.f;
          srow[f] = (h == 1 && f < F && r < a.dvv) ? car[f * a.ldt + r] : 0.f;
        }
        build_wop<256, CT0>(a, m.bh, sb + OFF_W);
        if (h == 1) {  // S accumulator (lane r = value column r): cols 0..7 = S_in, the rest 0
          float z[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) z[j] = j < FP ? srow[j] : 0.f;
          tmem_st16(tmem + lb + TM_SACC, z);
#pragma unroll
          for (int j = 0; j < 16; ++j) z[j] = 0.f;
          tmem_st16(tmem + lb + TM_SACC + 16, z);
          tmem_st_wait();
          write_sop(sb + OFF_SOP, r, srow);
        }
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(wready);
        if (threadIdx.x == a.ttid) RACE_TRACE(a, 11, gc);
      }
      const float invq = inv_scale(sqq, a.normalize);
      const float invk = inv_scale(sqk, a.normalize);
      mbar_wait(proj_full, gc & 1);
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 5, gc);
      tc_fence_after();
      float phq[FP];
      if (h == 0) {
        float pq[16];
        tmem_ld16(tmem + lb + TM_PROJQ, pq);
        tmem_ld_wait();
        row_features<P, HB>(a, pq, invq, valid, phq);
        write_phi_q(sb + OFF_PHIQ, r, phq);
        if (a.rows_out && valid) {  // sketch row, q half
          float hat[5];
          row_hat(a, pq, invq, hat);
          store_row_half(a.rows_out + (m.bh * a.N + t + r) * ROWW, hat, sqq);
        }
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(phi_full);
      } else {
        float phk[FP];  // (phi_q is the first half's: this half gets phi_q . A from it below)
        if (KR) {
          float u[5];
          row_features_hat<P, HB>(a, hk, valid, phk, u);
          write_phi_k(sb + OFF_PHIK, r, phk);
        } else {
          float pk[16];
          tmem_ld16(tmem + lb + TM_PROJK, pk);
          tmem_ld_wait();
          row_features<P, HB>(a, pk, invk, valid, phk);
          write_phi_k(sb + OFF_PHIK, r, phk);
          if (a.rows_out && valid) {  // sketch row, k half
            float hat[5];
            row_hat(a, pk, invk, hat);
            store_row_half(a.rows_out + (m.bh * a.N + t + r) * ROWW + 8, hat, sqk);
          }
        }
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(phi_full);
        // chunk total of phi_k: per-quarter partials by a recursive-halving warp reduction
        static_assert(FP == 8, "warp_sum8 reduces 8 values");
        const float tot = warp_sum8(phk);
        if ((lane_id() & 3) == 0) xpar[512 + qw * FP + (lane_id() >> 2)] = tot;
      }
      float D = 0.f;
      if (h == 0) {
#pragma unroll
        for (int f = 0; f < FP; ++f) D = fmaf(phq[f], A[f], D);
        xpar[544 + r] = D;  // for the second half (read after the barrier below)
      }
      // ---- intra-chunk weights: P~ = tril(Pm) -> bf16 pairs into TMEM (my 64 columns)
      mbar_wait(pm_full, gc & 1);
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 6, gc);
      tc_fence_after();
      float rs = 0.f;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int c0 = 64 * h + 32 * b;
        if ((c0 >> 5) <= qw) {  // warp-uniform; blocks above the diagonal stay zero
          float v[32];
          uint32_t u[16];
          tmem_ld32(tmem + lb + TM_PM + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] = (c0 + j <= r) ? v[j] : 0.f;
            rs += v[j];
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) u[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
          tmem_st16u(tmem + lb + TM_PA + (c0 >> 1), u);
        }
      }
      xpar[256 + h * 128 + r] = rs;
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(pt_full);
      if (h == 1) {
        mbar_wait(st_full, gc & 1);
        tc_fence_after();
        float sacc[32];
        tmem_ld32(tmem + lb + TM_SACC, sacc);  // S_<=c (value column r)
        tmem_ld_wait();
#pragma unroll
        for (int f = 0; f < FP; ++f) snext[f] = sacc[f] + sacc[16 + f];
      }
      // ---- while the numerator MMA runs: row norms of the next chunk
      cur.next(a);
      if (cur.ok()) {
        const int sn = (gc + 1) & 1;
        mbar_wait(&fullqk[sn], ((gc + 1) >> 1) & 1);
        const float sq = stage_norm(sn);
        xpar[h * 128 + r] = sq;
      }
      compute_bar256();
      if (threadIdx.x == CT0 && cur.ok()) mbar_arrive(&emptyqk[(gc + 1) & 1]);
      sqq = xpar[r];
      sqk = xpar[128 + r];
      if (h == 1) D = xpar[544 + r];
      D += xpar[256 + r] + xpar[384 + r];
      if (h == 0 && valid) a.den[m.bh * a.N + t + r] = D * invT;
      const float rD = (D * invT > kDegenerateDenEps) ? 1.f / D : 0.f;
#pragma unroll
      for (int f = 0; f < FP; ++f)
        A[f] += ((xpar[512 + f] + xpar[512 + FP + f]) + xpar[512 + 2 * FP + f]) + xpar[512 + 3 * FP + f];
      // ---- numerator -> O (my 64 columns, staged in the consumed V tile), next S operand
      mbar_wait(num_full, gc & 1);
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 7, gc);
      tc_fence_after();
      {
        float v[2][32];
        tmem_ld32(tmem + lb + TM_NUM + 64 * h, v[0]);
        tmem_ld32(tmem + lb + TM_NUM + 64 * h + 32, v[1]);
        tmem_ld_wait();
#pragma unroll
        for (int b = 0; b < 2; ++b) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[b][j] *= rD;
          stage_row_bf16(stage + 2 * TILE, r, v[b], 64 * h + 32 * b);
        }
      }
      if (h == 1) write_sop(sb + OFF_SOP, r, snext);
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&ostaged[s]);
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 8, gc);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) RACE_CTA_TIME(a, 1);
  if (warp == 1) tmem_dealloc<512>(tmem);
}


// ---------------------------------------------------------------------------
// Sketch rows of q and k for backward calls without forward state (the
// reference itself recomputes the forward, ra/backward.py:200).  Same TMA
// tiles, same projection MMA chain and the same row-norm code as
// k_causal_fwd8, so the rows are bit-identical to the ones the forward saves.
// ---------------------------------------------------------------------------
namespace prj {
constexpr int STAGES = 2;
constexpr int STAGE_BYTES = 2 * TILE;  // Q, K
constexpr int OFF_W = STAGES * STAGE_BYTES;
constexpr int OFF_BAR = OFF_W + WOP;
constexpr int SMEM = OFF_BAR + 256 + 1024;
}  // namespace prj

template <int P, int HB = 0, bool M4 = false>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_project(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK, Args a) {
  using namespace prj;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* full = bars;          // [2]
  uint64_t* empty = bars + 2;     // [2] (MMA commit + 128 row-norm readers)
  uint64_t* proj_full = bars + 4; // [2] (TMEM projection buffer per parity)
  uint64_t* proj_empty = bars + 6;// [2] (128 readers)
  uint64_t* wready = bars + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 9);
  const int warp = warp_id();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 129);
      mbar_init(&proj_full[i], 1);
      mbar_init(&proj_empty[i], 128);
    }
    mbar_init(wready, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<64>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel's tail
  int64_t i0, i1;
  cta_range(a.BH * a.nseg, i0, i1);
  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      uint32_t gc = 0;
      Cursor cur;
      for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
        const int s = gc & 1;
        mbar_wait(&empty[s], ((gc >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        uint8_t* st = smem + s * STAGE_BYTES;
        for (int h = 0; h < 2; ++h) {
          tile_load<M4>(a, st + h * SUB, &tmQ, &full[s], h * 64, cur.t, cur.m.bh, pol);
          tile_load<M4>(a, st + TILE + h * SUB, &tmK, &full[s], h * 64, cur.t, cur.m.bh, pol);
        }
      }
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
      const uint32_t acc = tmem + 32 * s;
      mbar_wait(&full[s], (gc >> 1) & 1);
      if (gc >= 2) mbar_wait(&proj_empty[s], ((gc >> 1) - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          umma_bf16(acc, desc_tile_k(stage, kk), desc_w(sb + OFF_W, kk), ID_PROJ, kk > 0);
          umma_bf16(acc + 16, desc_tile_k(stage + TILE, kk), desc_w(sb + OFF_W, kk), ID_PROJ, kk > 0);
        }
        umma_commit(&proj_full[s]);
        umma_commit(&empty[s]);
      }
      __syncwarp();
    }
  } else {
    const int r = crow();
    uint32_t gc = 0;
    int prev_bh = -1;
    Cursor cur;
    for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
      if (cur.m.bh != prev_bh) {  // the previous projections are consumed (program order)
        prev_bh = cur.m.bh;
        build_wop(a, cur.m.bh, sb + OFF_W);
        fence_proxy_async();
        mbar_arrive(wready);
      }
      const int s = gc & 1;
      const uint32_t stage = sb + s * STAGE_BYTES;
      mbar_wait(&full[s], (gc >> 1) & 1);
      const float sqq = tile_row_sumsq(stage, r), sqk = tile_row_sumsq(stage + TILE, r);
      mbar_arrive(&empty[s]);
      mbar_wait(&proj_full[s], (gc >> 1) & 1);
      tc_fence_after();
      float pq[16], pk[16];
      tmem_ld16(tmem + lane_base() + 32 * s, pq);
      tmem_ld16(tmem + lane_base() + 32 * s + 16, pk);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&proj_empty[s]);
      if (cur.t + r < cur.m.t1) {
        float hat[5];
        float* dst = a.rows_out + (int64_t(cur.m.bh) * a.N + cur.t + r) * ROWW;
        row_hat(a, pq, inv_scale(sqq, a.normalize), hat);
        store_row_half(dst, hat, sqq);
        row_hat(a, pk, inv_scale(sqk, a.normalize), hat);
        store_row_half(dst + 8, hat, sqk);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<64>(tmem);
}

static unsigned* g_dbg_host = nullptr;
static unsigned* g_dbg_dev = nullptr;
static int g_dbg_mode = 0;  // RACE_DEBUG_PROGRESS: 1 = host-mapped (watch a hang live), 2 = device (timing traces)
constexpr size_t kDbgBytes = 148 * 256 * sizeof(unsigned);
unsigned* debug_progress_device() {
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = getenv("RACE_DEBUG_PROGRESS");
    if (e && e[0] == '1') {
      if (cudaHostAlloc(reinterpret_cast<void**>(&g_dbg_host), kDbgBytes, cudaHostAllocMapped) == cudaSuccess) {
        memset(g_dbg_host, 0, kDbgBytes);
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&g_dbg_dev), g_dbg_host, 0);
        g_dbg_mode = 1;
      }
    } else if (e && e[0] == '2') {  // device memory: trace stores do not go over PCIe
      if (cudaMalloc(reinterpret_cast<void**>(&g_dbg_dev), kDbgBytes) == cudaSuccess) {
        cudaMemset(g_dbg_dev, 0, kDbgBytes);
        g_dbg_host = static_cast<unsigned*>(calloc(1, kDbgBytes));
        g_dbg_mode = 2;
      }
    }
  });
  return g_dbg_dev;
}
}  // namespace tcfast

// ---- entry points used by race_abi.cu --------------------------------------
bool tc_supported(const Geo& g) {
  const char* off = getenv("RACE_DISABLE_FAST_PATH");  // read per call: tests flip it
  if (off && off[0] == '1') return false;
  if (!tcfast::device_is_sm100()) return false;
  // one pass: F = T * 2^cb <= 8 buckets, T * P <= 5 projections (W' holds three bf16 pieces of each in 16
  // rows), at most 3 corner bits per table; a corner group (cb < P) is one table of up to 5 hyperplanes
  const int cb = pass_corner_bits(g);
  const int F = g.T << cb;
  // head widths up to 128 (tiles are 128 wide; TMA zero-fills / clips beyond d, dv), multiples of 8
  // (16-byte row pitch of the TMA maps)
  return g.dtype == 1 && g.d >= 8 && g.d <= 128 && g.d % 8 == 0 && g.dv >= 8 && g.dv <= 128 && g.dv % 8 == 0 &&
         F <= tcfast::FP && g.T * g.P <= 5 && cb <= 3 &&
         (g.cb == 0 || g.T == 1) && g.N > 0 && g.N < (int64_t(1) << 31) && g.seg_tokens % tcfast::CH == 0 &&
         tcfast::encode_fn() != nullptr;
}

cudaError_t tc_aggregate(const Geo& g, const void* k, const void* v, const float* w, float* part, float* rows,
                         cudaStream_t st) {
  using namespace tcfast;
  CUtensorMap mk, mv;
  if (!make_map(&mk, k, g, g.d, L_K) || !make_map(&mv, v, g, g.dv, L_V)) return cudaErrorInvalidValue;
  Args a = make_args(g);
  a.w = w;
  a.tout = part;
  a.rows_out = rows;
  if (g.strided()) switch (pass_corner_bits(g)) {  // one-pass problems only (race_fwd_layout checks)
      case 1: return launch_nt(k_aggregate2<1, 0, true>, NTHREADS8, agg2::SMEM, grid_for(g), st, mk, mv, a);
      case 2: return launch_nt(k_aggregate2<2, 0, true>, NTHREADS8, agg2::SMEM, grid_for(g), st, mk, mv, a);
      default: return launch_nt(k_aggregate2<3, 0, true>, NTHREADS8, agg2::SMEM, grid_for(g), st, mk, mv, a);
    }
  switch (pass_corner_bits(g)) {
    case 1: return launch_nt(k_aggregate2<1>, NTHREADS8, agg2::SMEM, grid_for(g), st, mk, mv, a);
    case 2: return launch_nt(k_aggregate2<2>, NTHREADS8, agg2::SMEM, grid_for(g), st, mk, mv, a);
    default:
      if (g.cb) return launch_nt(k_aggregate2<3, 2>, NTHREADS8, agg2::SMEM, grid_for(g), st, mk, mv, a);
      return launch_nt(k_aggregate2<3>, NTHREADS8, agg2::SMEM, grid_for(g), st, mk, mv, a);
  }
}

cudaError_t tc_readout(const Geo& g, const void* q, const float* w, const float* tab, void* o, float* den,
                       cudaStream_t st) {
  using namespace tcfast;
  CUtensorMap mq, mo;
  if (!make_map(&mq, q, g, g.d, L_Q) || !make_map(&mo, o, g, g.dv, L_O)) return cudaErrorInvalidValue;
  Args a = make_args(g);
  a.w = w;
  a.tin = tab;
  a.den = den;
  if (g.strided()) switch (pass_corner_bits(g)) {
      case 1: return launch_nt(k_readout8<1, 0, true>, NTHREADS8, rdo8::SMEM, grid_for(g), st, mq, mo, a);
      case 2: return launch_nt(k_readout8<2, 0, true>, NTHREADS8, rdo8::SMEM, grid_for(g), st, mq, mo, a);
      default: return launch_nt(k_readout8<3, 0, true>, NTHREADS8, rdo8::SMEM, grid_for(g), st, mq, mo, a);
    }
  switch (pass_corner_bits(g)) {
    case 1: return launch_nt(k_readout8<1>, NTHREADS8, rdo8::SMEM, grid_for(g), st, mq, mo, a);
    case 2: return launch_nt(k_readout8<2>, NTHREADS8, rdo8::SMEM, grid_for(g), st, mq, mo, a);
    default:
      if (g.cb) return launch_nt(k_readout8<3, 2>, NTHREADS8, rdo8::SMEM, grid_for(g), st, mq, mo, a);
      return launch_nt(k_readout8<3>, NTHREADS8, rdo8::SMEM, grid_for(g), st, mq, mo, a);
  }
}

cudaError_t tc_project(const Geo& g, const void* q, const void* k, const float* w, float* rows, cudaStream_t st) {
  using namespace tcfast;
  if (g.BH * g.N == 0) return cudaSuccess;
  CUtensorMap mq, mk;
  if (!make_map(&mq, q, g, g.d, L_Q) || !make_map(&mk, k, g, g.d, L_K)) return cudaErrorInvalidValue;
  Args a = make_args(g);
  a.w = w;
  a.rows_out = rows;
  if (g.strided()) switch (pass_corner_bits(g)) {
      case 1: return launch(k_project<1, 0, true>, prj::SMEM, grid_for(g), st, mq, mk, a);
      case 2: return launch(k_project<2, 0, true>, prj::SMEM, grid_for(g), st, mq, mk, a);
      default: return launch(k_project<3, 0, true>, prj::SMEM, grid_for(g), st, mq, mk, a);
    }
  switch (pass_corner_bits(g)) {
    case 1: return launch(k_project<1>, prj::SMEM, grid_for(g), st, mq, mk, a);
    case 2: return launch(k_project<2>, prj::SMEM, grid_for(g), st, mq, mk, a);
    default:
      if (g.cb) return launch(k_project<3, 2>, prj::SMEM, grid_for(g), st, mq, mk, a);
      return launch(k_project<3>, prj::SMEM, grid_for(g), st, mq, mk, a);
  }
}

// krows: the k halves of nrm were written by tc_aggregate (then K is not read)
cudaError_t tc_causal_fwd(const Geo& g, const void* q, const void* k, const void* v, const float* w,
                          const float* car, void* o, float* den, float* nrm, bool krows, cudaStream_t st) {
  using namespace tcfast;
  CUtensorMap mq, mk, mv, mo, mr;
  if (!make_map(&mq, q, g, g.d, L_Q) || !make_map(&mk, k, g, g.d, L_K) || !make_map(&mv, v, g, g.dv, L_V) ||
      !make_map(&mo, o, g, g.dv, L_O))
    return cudaErrorInvalidValue;
  if (krows && (!nrm || !make_map_rows(&mr, nrm, g.BH * g.N))) return cudaErrorInvalidValue;
  if (!krows) mr = mq;  // unused
  Args a = make_args(g);
  a.w = w;
  a.tin = car;
  a.den = den;
  a.rows_out = nrm;
  a.dbg = trace_for("fwd");
  switch (pass_corner_bits(g)) {
#define RACE_FWD8(PP, HB, M4)                                                                                     \
  return krows ? launch_nt(k_causal_fwd8<PP, true, HB, M4>, NTHREADS8, cfw8::SMEM, grid_for(g), st, mq, mk, mv, mo, mr, a) \
               : launch_nt(k_causal_fwd8<PP, false, HB, M4>, NTHREADS8, cfw8::SMEM, grid_for(g), st, mq, mk, mv, mo, mr, a)
    case 1: if (g.strided()) RACE_FWD8(1, 0, true); RACE_FWD8(1, 0, false);
    case 2: if (g.strided()) RACE_FWD8(2, 0, true); RACE_FWD8(2, 0, false);
    default:
      if (g.strided()) RACE_FWD8(3, 0, true);
      if (g.cb) RACE_FWD8(3, 2, false);
      RACE_FWD8(3, 0, false);
#undef RACE_FWD8
  }
}

}  // namespace race

// diagnostic (not part of the documented ABI): host view of the progress words
extern "C" void* race_debug_progress_buffer(void) {
  race::tcfast::debug_progress_device();
  if (race::tcfast::g_dbg_mode == 2)
    cudaMemcpy(race::tcfast::g_dbg_host, race::tcfast::g_dbg_dev, race::tcfast::kDbgBytes, cudaMemcpyDeviceToHost);
  return race::tcfast::g_dbg_host;
}
extern "C" void race_debug_progress_clear(void) {
  race::tcfast::debug_progress_device();
  if (race::tcfast::g_dbg_mode == 2) cudaMemset(race::tcfast::g_dbg_dev, 0, race::tcfast::kDbgBytes);
  if (race::tcfast::g_dbg_host) memset(race::tcfast::g_dbg_host, 0, race::tcfast::kDbgBytes);
}
