// race_tc_cbwd.cu -- sm_100a fast path, causal backward (ra/backward.py:132-181).
//
// Chunk form (128 tokens, inclusive diagonal), D_t = T * den_t:
//   query side, forward scan with S_<c carried in TMEM:
//     y_t   = S_<c,v dO_t                       (MMA, N = 16)
//     E     = dO_c V_c^T,  Pm = Phi_q Phi_k^T    (MMAs, 128 x 128)
//     D_t   = phi_q,t . A_<c + sum_{j<=t} Pm_tj
//     rho_t = (phi_q,t . y_t + sum_{j<=t} Pm_tj E_tj) / D_t          (= dO_t . O_t)
//     dphi_q,t = (y_t - rho_t A_<c + sum_{j<=t} (E_tj - rho_t) phi_k,j) / D_t
//              (the sum is the MMA  tril(E - rho) . Phi_k)
//     dS_seg += Phi_q^T G,  G_t = [dO_t / D_t | -rho_t / D_t]; rden = 1/D, gden = -rho/D saved
//   key side, reverse scan with dS_>c carried in TMEM:
//     dphi_k,i = [v_i | 1] dS_>c^T + sum_{t>=i} (G_t . [v_i | 1]) phi_q,t
//     dV_i     = phi_k,i dS_>c,v + sum_{t>=i} Pm_ti dO_t / D_t
// followed by the feature / tanh / sphere-tangent VJPs (shared with race_tc_bwd.cu).
#include <cstdlib>

#include "tc_fast.cuh"

namespace race {
namespace tcfast {

using namespace tc;

constexpr uint32_t IDC_Y = idesc_bf16(128, 16, 0, 0);     // dO x S^T-op          (K, K)
constexpr uint32_t IDC_E = idesc_bf16(128, 128, 0, 0);    // dO x V^T / V x dO^T  (K, K)
constexpr uint32_t IDC_PM = idesc_bf16(128, 128, 0, 0);   // Phi x Phi^T          (K, K)
constexpr uint32_t IDC_ST = idesc_bf16(128, 32, 1, 1);    // X^T x Phi            (MN, MN)
constexpr uint32_t IDC_Z = idesc_bf16(128, 32, 0, 1);     // E~ x Phi             (K, MN)
constexpr uint32_t IDC_DX = idesc_bf16(128, 128, 0, 1);   // dProj x W''          (K, MN)
constexpr uint32_t IDC_DVA = idesc_bf16(128, 128, 0, 0);  // Phi_k x dS-op        (K, K)
constexpr uint32_t IDC_DVB = idesc_bf16(128, 128, 0, 1);  // P~^T x dO            (K, MN)

// ===========================================================================
// causal backward, query side -- pipelined 8-compute-warp version (launched)
//
// Same math as the chunk form above, restructured for latency:
//  * contiguous CTA ranges: S, A continue across segments; dS / dA totals are
//    emitted per segment;
//  * no Pm = Phi_q Phi_k^T: the two row statistics it fed factor through Phi_k,
//      sum_{j<=t} Pm_tj        = phi_q,t . C_t,   C_t = sum_{j<=t} phi_k,j  (warp scan)
//      sum_{j<=t} Pm_tj E_tj   = phi_q,t . Z_t,   Z   = tril(E) Phi_k      (MMA)
//    so dphi_q,t = (y_t + Z_t - rho_t (A_<c + C_t)) / D_t needs one MMA round
//    trip per chunk after the features, and tril(E) is packed (hi / lo bf16
//    pairs in TMEM, the A operands of Z: E to 16 bits, so rho and the key
//    side's gden = -rho / D stay fp32-exact) as soon as E lands;
//  * compute warps 2..9 split every 128-column pass into halves;
//  * Q and dO are double-buffered, so the MMA warp issues the NEXT chunk's
//    E / Y right after this chunk's dx^ / dS -- they complete while the compute
//    warps finish this chunk;
//  * dx^ = dproj . W is one MMA pair against the projection operand W'
//    itself (read MN-major: W_hi + W_mid + W_lo, i.e. W to 24 bits) with
//    dproj split hi / lo; the sphere-tangent VJP writes dq over q in its
//    tile and the producer TMA-stores it just before refilling that buffer;
//  * the row norms saved by the forward arrive by TMA with their own
//    full / empty barriers (no global loads in the compute warps).
// ===========================================================================
namespace cq8 {
constexpr int OFF_Q = 0;                       // two buffers
constexpr int OFF_V = 2 * TILE;
constexpr int OFF_DO = 3 * TILE;               // two buffers
constexpr int OFF_W = 5 * TILE;                // W' (B of the projection; B of dx^ read MN-major)
constexpr int OFF_SOPT = OFF_W + WOP;
constexpr int OFF_PHIQ = OFF_SOPT + WOP;       // phi_q / D (B of dS)
constexpr int OFF_PHIK = OFF_PHIQ + PHI;       // Phi_k (B of S and Z), then dproj (A of dx^)
constexpr int OFF_X = OFF_PHIK + PHI;          // kp[2 parity][4][8], cs[128][8] (in-warp scans of phi_k), da[4][8],
                                               // pq[128][8], dot[128]
constexpr int XKP = 0, XCS = 64, XDA = 64 + CH * FP;
constexpr int XPQ = XDA + 32, XDOT = XPQ + CH * FP;  // phi_q [128][8] and dx^.x^ [128]: first half -> second
constexpr int OFF_TOK = OFF_X + (XDOT + CH) * 4;  // [2] x sketch rows [128][ROWW] (TMA)
constexpr int TOK_BYTES = CH * ROWW * 4;
constexpr int OFF_BAR = OFF_TOK + 2 * TOK_BYTES;
constexpr int SMEM = OFF_BAR + 256 + 1024;
static_assert(SMEM <= 232448, "k_bwd_causal_q8 shared memory");
static_assert(OFF_TOK % 128 == 0, "TMA destination alignment");
constexpr uint32_t TM_Y = 0, TM_Z = 32, TM_S = 64, TM_DS = 96, TM_ETH = 128, TM_ETL = 192, TM_DX = 256,
                   TM_E = 384;
// W' [16 x 128] (rows = hyperplane pieces, d contiguous, two SW128 64-column sub-tiles) as an MN-major B
__device__ __forceinline__ uint64_t desc_wT(uint32_t base) { return smem_desc(base, 2048, 1024, kSw128); }
// dproj expanded to W's rows: K cols 3j..3j+2 = dproj_j (hi) and 16 + 3j.. (lo)
__device__ __forceinline__ void write_dproj_w(uint32_t buf, int r, const float* dproj, int tp) {
  float hi[16], lo[16];
#pragma unroll
  for (int n = 0; n < 16; ++n) {
    const int j = n / 3;
    const float x = (n < 15 && j < tp) ? dproj[j < 5 ? j : 0] : 0.f;
    hi[n] = bf16_round(x);
    lo[n] = x - hi[n];
  }
  uint32_t blk[4][4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    blk[0][e] = pack_bf16(hi[2 * e], hi[2 * e + 1]);
    blk[1][e] = pack_bf16(hi[8 + 2 * e], hi[8 + 2 * e + 1]);
    blk[2][e] = pack_bf16(lo[2 * e], lo[2 * e + 1]);
    blk[3][e] = pack_bf16(lo[8 + 2 * e], lo[8 + 2 * e + 1]);
  }
  write_row32(buf, r, blk);
}
}  // namespace cq8

template <int P, int HB = 0, bool GRP = false, bool M4 = false>
__global__ void __launch_bounds__(NTHREADS8, 1)
    k_bwd_causal_q8(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                    const __grid_constant__ CUtensorMap tmDQ, const __grid_constant__ CUtensorMap tmROWS, Args a,
                    float* __restrict__ rden, float* __restrict__ gden) {
  using namespace cq8;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* fullQ = bars + 0;      // [2]
  uint64_t* dqstaged = bars + 2;   // [2] dQ staged in the Q buffer (256 arrivals)
  uint64_t* fullO = bars + 4;      // [2]
  uint64_t* emptyO = bars + 6;     // [2] (dS MMA commit)
  uint64_t* fullT = bars + 8;      // [2] sketch rows landed
  uint64_t* emptyT = bars + 10;    // [2] sketch rows read (256 arrivals)
  uint64_t* fullV = bars + 14;
  uint64_t* emptyV = bars + 15;
  uint64_t* c1 = bars + 16;        // projection + E + Y
  uint64_t* c2 = bars + 17;        // Z + S state
  uint64_t* phi_ready = bars + 19;  // Phi_k + tril(E) staged (256 arrivals)
  uint64_t* wready = bars + 21;
  uint64_t* acc_full = bars + 22;
  uint64_t* acc_empty = bars + 23;
  uint64_t* dp_ready = bars + 24;  // dproj staged (256 arrivals)
  uint64_t* c4 = bars + 25;        // dx^ MMA
  uint64_t* dsdone = bars + 12;    // dS MMAs (after dx^) done: phi_q / D buffer free
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 26);

  const int warp = warp_id();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&fullQ[i], 1);
      mbar_init(&dqstaged[i], 256);
      mbar_init(&fullO[i], 1);
      mbar_init(&emptyO[i], 1);
      mbar_init(&fullT[i], 1);
      mbar_init(&emptyT[i], 256);
    }
    for (int i = 12; i < 19; ++i) mbar_init(&bars[i], 1);
    mbar_init(phi_ready, 256);
    mbar_init(wready, 256);
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 256);
    mbar_init(dp_ready, 256);
    mbar_init(c4, 1);
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
      tma_prefetch_desc(&tmDO);
      tma_prefetch_desc(&tmDQ);
      tma_prefetch_desc(&tmROWS);
      const uint64_t pol = policy_evict_first();
      int qt0 = 0, qb0 = 0, qt1 = 0, qb1 = 0;
      auto store_dq = [&](uint32_t j) {
        const int s = j & 1;
        mbar_wait(&dqstaged[s], (j >> 1) & 1);
        const int qt = int(s ? qt1 : qt0), qb = int(s ? qb1 : qb0);
        if (!a.dproj_out)  // grouped backward: dq is formed from the summed dproj afterwards
          for (int h = 0; h < 2; ++h)
            tile_store<M4>(a, &tmDQ, reinterpret_cast<void*>(smem + OFF_Q + s * TILE + h * SUB), h * 64, qt, qb);
        tma_store_commit();
      };
      uint32_t gc = 0;
      Cursor cur;
      for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
        if (a.pf > 0) {  // warm L2 with the tiles a.pf chunks ahead (same sequence; a hint only)
          const int tp = int(cur.t) + a.pf * CH;
          if (tp < a.N)
            for (int h = 0; h < 2; ++h) {
              tile_prefetch<M4>(a, &tmQ, h * 64, tp, int(cur.m.bh));
              tile_prefetch<M4>(a, &tmK, h * 64, tp, int(cur.m.bh));
              tile_prefetch<M4>(a, &tmV, h * 64, tp, int(cur.m.bh));
              tile_prefetch<M4>(a, &tmDO, h * 64, tp, int(cur.m.bh));
            }
        }
        const uint32_t par1 = (gc & 1) ^ 1;          // single buffers: one phase per chunk
        const uint32_t par2 = ((gc >> 1) & 1) ^ 1;   // double buffers: one phase per two chunks
        const int s = gc & 1;
        const int t = int(cur.t), bh = int(cur.m.bh);
        if (gc >= 2) {
          store_dq(gc - 2);
          tma_store_wait_read<0>();
        }
        RACE_TRACE(a, 3, gc);
        mbar_arrive_expect_tx(&fullQ[s], TILE);
        for (int h = 0; h < 2; ++h) tile_load<M4>(a, smem + OFF_Q + s * TILE + h * SUB, &tmQ, &fullQ[s], h * 64, t, bh, pol);
        if (s) { qt1 = t; qb1 = bh; } else { qt0 = t; qb0 = bh; }
        mbar_wait(&emptyT[s], par2);
        mbar_arrive_expect_tx(&fullT[s], TOK_BYTES);
        tma_load_2d(smem + OFF_TOK + s * TOK_BYTES, &tmROWS, &fullT[s], 0, bh * int(a.N) + t, pol);
        mbar_wait(emptyV, par1);
        RACE_TRACE(a, 1, gc);
        mbar_arrive_expect_tx(fullV, TILE);
        for (int h = 0; h < 2; ++h) tile_load<M4>(a, smem + OFF_V + h * SUB, &tmV, fullV, h * 64, t, bh, pol);
        mbar_wait(&emptyO[s], par2);
        RACE_TRACE(a, 2, gc);
        mbar_arrive_expect_tx(&fullO[s], TILE);
        for (int h = 0; h < 2; ++h)
          tile_load<M4>(a, smem + OFF_DO + s * TILE + h * SUB, &tmDO, &fullO[s], h * 64, t, bh, pol);
      }
      for (uint32_t j = gc >= 2 ? gc - 2 : 0; j < gc; ++j) store_dq(j);
      tma_store_wait_all<0>();
    }
  } else if (warp == 1) {
    // E / Y of chunk `gc` (issued one step ahead of its use; the q projections come from the
    // forward's sketch rows, so there is no projection MMA here)
    auto issue_front = [&](uint32_t gc) {
      const int s = gc & 1;
      mbar_wait(fullV, gc & 1);
      mbar_wait(&fullO[s], (gc >> 1) & 1);
      RACE_TRACE(a, 5, gc);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          umma_bf16(tmem + TM_E, desc_tile_k(sb + OFF_DO + s * TILE, kk), desc_tile_k(sb + OFF_V, kk), IDC_E, kk > 0);
          umma_bf16(tmem + TM_Y, desc_tile_k(sb + OFF_DO + s * TILE, kk), desc_w(sb + OFF_SOPT, kk), IDC_Y, kk > 0);
        }
        umma_commit(c1);
      }
      __syncwarp();
    };
    uint32_t gc = 0, nr = 0, ni = 0;
    int64_t prev_bh = -1;
    for (int64_t it = i0; it < i1; ++it, ++ni) {
      const Item m = item_of(a, it);
      for (int64_t t = m.t0; t < m.t1; t += CH, ++gc) {
        const uint32_t par = gc & 1;
        const int s = gc & 1;
        const bool first = t == m.t0;
        if (m.bh != prev_bh) {  // new sequence: W', S, SOPT rebuilt by the compute warps
          prev_bh = m.bh;
          mbar_wait(wready, nr & 1);
          ++nr;
          tc_fence_after();
          issue_front(gc);
        }
        mbar_wait(phi_ready, par);  // Phi_k and tril(E) (hi / lo) staged
        RACE_TRACE(a, 6, gc);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // Z = tril(E) Phi_k: dphi_q's intra-chunk term and the row statistic
            umma_bf16_ts(tmem + TM_Z, tmem + TM_ETH + kk * 8, desc_phi_mn(sb + OFF_PHIK, kk), IDC_Z, kk > 0);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // E to 16 bits: rho (and gden for the key side) stays fp32-exact
            umma_bf16_ts(tmem + TM_Z, tmem + TM_ETL + kk * 8, desc_phi_mn(sb + OFF_PHIK, kk), IDC_Z, 1u);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(tmem + TM_S, desc_tile_mn(sb + OFF_V, kk), desc_phi_mn(sb + OFF_PHIK, kk), IDC_ST, 1u);
          umma_commit(c2);
          umma_commit(emptyV);
        }
        __syncwarp();
        mbar_wait(dp_ready, par);
        RACE_TRACE(a, 8, gc);
        if (first && ni > 0) mbar_wait(acc_empty, (ni - 1) & 1);  // dS of the previous segment read out
        tc_fence_after();
        if (elect_one()) {  // dx^ = dproj . W (hi and lo halves of dproj against W' read MN-major)
          umma_bf16(tmem + TM_DX, desc_phi_k(sb + OFF_PHIK, 0), desc_wT(sb + OFF_W), IDC_DX, 0u);
          umma_bf16(tmem + TM_DX, desc_phi_k(sb + OFF_PHIK, 1), desc_wT(sb + OFF_W), IDC_DX, 1u);
          umma_commit(c4);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // the segment's dS total, off the critical path
            umma_bf16(tmem + TM_DS, desc_tile_mn(sb + OFF_DO + s * TILE, kk), desc_phi_mn(sb + OFF_PHIQ, kk), IDC_ST,
                      (!first || kk > 0) ? 1u : 0u);
          umma_commit(&emptyO[s]);
          umma_commit(dsdone);
          if (t + CH >= m.t1) umma_commit(acc_full);
        }
        __syncwarp();
        // the next chunk's front MMAs, unless it starts a new sequence (then W' changes first)
        int64_t tn = t + CH, itn = it;
        if (tn >= m.t1) {
          ++itn;
          tn = -1;
        }
        if (itn < i1) {
          const int64_t bhn = tn >= 0 ? m.bh : item_of(a, itn).bh;
          if (bhn == m.bh) issue_front(gc + 1);
        }
      }
    }
  } else {
    const int r = crow();
    const int h = chalf();
    const int qw = warp & 3;
    const uint32_t lb = lane_base();
    const float invT = 1.f / float(a.T);
    const int F = a.T << a.P;
    float* xbase = reinterpret_cast<float*>(smem + OFF_X);
    float* xcs = xbase + XCS;
    float* xda = xbase + XDA;
    {  // tril(E) blocks above the diagonal are never written: zero the A operands once
      uint32_t z[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) z[j] = 0u;
      tmem_st16u(tmem + lb + TM_ETH + 32 * h, z);
      tmem_st16u(tmem + lb + TM_ETH + 32 * h + 16, z);
      tmem_st16u(tmem + lb + TM_ETL + 32 * h, z);
      tmem_st16u(tmem + lb + TM_ETL + 32 * h + 16, z);
      tmem_st_wait();
    }
    float A[FP], dA[FP];
    uint32_t gc = 0, ni = 0;
    int64_t prev_bh = -1;
    for (int64_t it = i0; it < i1; ++it, ++ni) {
      const Item m = item_of(a, it);
      if (m.bh != prev_bh) {  // (re)load the sequence state
        prev_bh = m.bh;
        const float* car = a.tin + (m.bh * a.nseg + m.seg) * int64_t(F) * a.ldt;
        float scol[FP];
#pragma unroll
        for (int f = 0; f < FP; ++f) {
          A[f] = f < F ? car[f * a.ldt + a.dvv] : 0.f;
          scol[f] = (h == 1 && f < F && r < a.dvv) ? car[f * a.ldt + r] : 0.f;
        }
        build_wop<256>(a, m.bh, sb + OFF_W);
        if (h == 1) {
          float z[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) z[j] = j < FP ? scol[j] : 0.f;
          tmem_st16(tmem + lb + TM_S, z);
#pragma unroll
          for (int j = 0; j < 16; ++j) z[j] = 0.f;
          tmem_st16(tmem + lb + TM_S + 16, z);
          tmem_st_wait();
          write_sopT(sb + OFF_SOPT, r, scol);
        }
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(wready);
      }
#pragma unroll
      for (int f = 0; f < FP; ++f) dA[f] = 0.f;
      for (int64_t t = m.t0; t < m.t1; t += CH, ++gc) {
        const uint32_t par = gc & 1;
        const int s = gc & 1;
        uint8_t* qtile = smem + OFF_Q + s * TILE;
        float* xkp = xbase + XKP + par * 32;
        const bool valid = t + r < m.t1;
        const GroupPre pre = GRP ? group_prefetch(a, m.bh, t, r, valid) : GroupPre{};
        mbar_wait(&fullT[s], (gc >> 1) & 1);
        const float* trow = reinterpret_cast<const float*>(smem + OFF_TOK + s * TOK_BYTES) + r * ROWW;
        float hq[5], hatk[5];  // x^.w_j of this q row and of this k row (the forward's sketch row)
#pragma unroll
        for (int j = 0; j < 5; ++j) {
          hq[j] = trow[j];
          hatk[j] = trow[8 + j];
        }
        const Scale scq = row_scale(valid ? trow[7] : 0.f, a.normalize);
        mbar_arrive(&emptyT[s]);
        if (threadIdx.x == a.ttid) RACE_TRACE(a, 9, gc);
        // the first half computes phi_q (and later the feature VJP) for both; the second half computes
        // phi_k, its operand and scan, and reads phi_q back after the barrier below
        float phq[FP], uq[5];
        if (h == 1) {  // Phi_k operand, in-warp inclusive scan of phi_k (C_t) and the warp totals
          float phk[FP], uk[5];
          row_features_hat<P, HB>(a, hatk, valid, phk, uk);
          write_phi_k(sb + OFF_PHIK, r, phk);
          const int lane = lane_id();
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
            for (int f = 0; f < FP; ++f) {
              const float x = __shfl_up_sync(0xffffffffu, phk[f], o);
              if (lane >= o) phk[f] += x;
            }
          }
#pragma unroll
          for (int f = 0; f < FP; ++f) xcs[r * FP + f] = phk[f];
          if (lane == 31) {
#pragma unroll
            for (int f = 0; f < FP; ++f) xkp[qw * FP + f] = phk[f];
          }
        } else {
          row_features_hat<P, HB>(a, hq, valid, phq, uq);
#pragma unroll
          for (int f = 0; f < FP; ++f) xbase[XPQ + r * FP + f] = phq[f];
        }
        // tril(E) -> hi / lo bf16 pairs into TMEM (A operands of Z), my 64 columns
        mbar_wait(c1, par);
        tc_fence_after();
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int c0 = 64 * h + 32 * b;
          if ((c0 >> 5) <= qw) {  // warp-uniform
            float e[32];
            uint32_t uh[16], ul[16];
            tmem_ld32(tmem + lb + TM_E + c0, e);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float e0 = (c0 + 2 * j <= r) ? e[2 * j] : 0.f;
              const float e1 = (c0 + 2 * j + 1 <= r) ? e[2 * j + 1] : 0.f;
              const float h0 = bf16_round(e0), h1 = bf16_round(e1);
              uh[j] = pack_bf16(h0, h1);
              ul[j] = pack_bf16(e0 - h0, e1 - h1);
            }
            tmem_st16u(tmem + lb + TM_ETH + (c0 >> 1), uh);
            tmem_st16u(tmem + lb + TM_ETL + (c0 >> 1), ul);
          }
        }
        tmem_st_wait();
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(phi_ready);
        float yv[16];
        tmem_ld16(tmem + lb + TM_Y, yv);
        compute_bar256();  // the phi_k scans, warp totals and phi_q are visible
        if (h == 1) {
#pragma unroll
          for (int f = 0; f < FP; ++f) phq[f] = xbase[XPQ + r * FP + f];
        }
        float y[FP], C[FP], Dint = 0.f, ydot = 0.f, rs = 0.f;
        tmem_ld_wait();
#pragma unroll
        for (int f = 0; f < FP; ++f) {
          float c = xcs[r * FP + f];
          for (int w = 0; w < qw; ++w) c += xkp[w * FP + f];  // warp-uniform trip count
          C[f] = c;
          y[f] = yv[f] + yv[8 + f];
          Dint = fmaf(phq[f], A[f], Dint);
          ydot = fmaf(phq[f], y[f], ydot);
          rs = fmaf(phq[f], c, rs);
        }
        // ---- Z landed: row statistics, dphi_q -> dproj
        mbar_wait(c2, par);
        if (threadIdx.x == a.ttid) RACE_TRACE(a, 10, gc);
        tc_fence_after();
        float zhi[8], zlo[8];
        tmem_ld8(tmem + lb + TM_Z, zhi);
        tmem_ld8(tmem + lb + TM_Z + 16, zlo);
        tmem_ld_wait();
        float Z[FP], nd = 0.f;
#pragma unroll
        for (int f = 0; f < FP; ++f) {
          Z[f] = zhi[f] + zlo[f];
          nd = fmaf(phq[f], Z[f], nd);
        }
        const float D = Dint + rs;
        const bool live = valid && D * invT > kDegenerateDenEps;
        float rD = live ? 1.f / D : 0.f;
        float rho = (ydot + nd) * rD;
        if (GRP && a.ext_rd) {  // table / corner group: normalisers of the whole estimator
          rD = pre.rd;
          rho = rD != 0.f ? -pre.gd / rD : 0.f;
        }
        if (h == 0) {
          float dphi[FP];
#pragma unroll
          for (int f = 0; f < FP; ++f) dphi[f] = (y[f] + Z[f] - rho * (A[f] + C[f])) * rD;
          float dproj[8];
          row_feature_vjp<P, HB>(a, uq, phq, dphi, dproj);
          if (GRP && a.dproj_out && valid) emit_dproj(a, m.bh * a.N + t + r, dproj, pre);
          xbase[XDOT + r] = dot_from_proj(dproj, hq);  // read by the second half after c4
          write_dproj_w(sb + OFF_PHIK, r, dproj, a.TP);  // Phi_k is dead after Z and S (c2)
#pragma unroll
          for (int f = 0; f < FP; ++f) dA[f] = fmaf(phq[f], -rho * rD, dA[f]);
        } else {
          float pht[FP];
#pragma unroll
          for (int f = 0; f < FP; ++f) pht[f] = phq[f] * rD;
          write_phi_k(sb + OFF_PHIQ, r, pht);  // B of dS (the previous chunk's dS MMA is done: dsdone)
          // S_<=c for the next chunk's y (the Y MMA of this chunk completed at c1); columns 8..15
          // and 24..31 of the N = 32 product are the duplicate hi copy and padding: not read
          float shi[8], slo[8];
          tmem_ld8(tmem + lb + TM_S, shi);
          tmem_ld8(tmem + lb + TM_S + 16, slo);
          tmem_ld_wait();
          float snext[FP];
#pragma unroll
          for (int f = 0; f < FP; ++f) snext[f] = shi[f] + slo[f];
          write_sopT(sb + OFF_SOPT, r, snext);
        }
#pragma unroll
        for (int f = 0; f < FP; ++f) A[f] += ((xkp[f] + xkp[FP + f]) + xkp[2 * FP + f]) + xkp[3 * FP + f];
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(dp_ready);
        if (h == 0 && valid && !a.ext_rd) {
          rden[m.bh * a.Np + t + r] = rD;  // row pitch Np (multiple of 4: 16-byte TMA tiles)
          gden[m.bh * a.Np + t + r] = -rho * rD;
        }
        // ---- dq (my 64 columns) in place of q; the producer stores it
        mbar_wait(c4, par);
        if (threadIdx.x == a.ttid) RACE_TRACE(a, 12, gc);
        tc_fence_after();
        mbar_wait(&fullQ[s], (gc >> 1) & 1);  // q itself is only read here (x^ of the tangent step)
        tangent_half_inplace(tmem + lb + TM_DX, qtile, r, h, scq, xbase[XDOT + r]);
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(&dqstaged[s]);
        if (threadIdx.x == a.ttid) RACE_TRACE(a, 13, gc);
        mbar_wait(dsdone, par);  // the dS MMA has read phi_q / D: the next chunk may overwrite it
      }
      // ---- segment done: dS total (TMEM) and dA total (block reduction)
      mbar_wait(acc_full, ni & 1);
      tc_fence_after();
      float* out = a.tout + (m.bh * a.nseg + m.seg) * int64_t(F) * a.ldt;
      if (h == 1) {
        float acc[32];
        tmem_ld32(tmem + lb + TM_DS, acc);
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
      mbar_arrive(acc_empty);
      compute_bar256();
      if (h == 0 && r < F) out[r * a.ldt + a.dvv] = ((xda[r] + xda[FP + r]) + xda[2 * FP + r]) + xda[3 * FP + r];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) RACE_CTA_TIME(a, 1);
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ===========================================================================
// causal backward, key side -- pipelined 8-compute-warp version (launched)
//
// Same math as k_bwd_causal_k above.  Each CTA walks its contiguous item
// range BACKWARDS (the key side is a suffix scan), so dS_>c and dA continue
// across segments; compute warps split the column passes into halves; EG~ and
// P~^T live in TMEM as the A operands of Z = EG~ Phi_q and dV += P~^T dO; the
// K tile is double-buffered (dK staged in place, TMA-stored by the producer);
// dV goes straight from TMEM to global memory.  Row norms are required.
// ===========================================================================
namespace ck8 {
constexpr int OFF_K = 0;                   // one buffer (read by the tangent step only; dK staged in place)
constexpr int OFF_V = TILE;                // two buffers (dV staged in place once E / z are done)
constexpr int OFF_DO = 3 * TILE;           // two buffers
constexpr int OFF_W = 5 * TILE;            // W' (projection; read MN-major as the B of dx^)
constexpr int OFF_DSOPT = OFF_W + WOP;     // [16 x 128] B of z = V dS_v^T
constexpr int OFF_DSOP = OFF_DSOPT + WOP;  // [128 x 32] B of dV_a = Phi_k dS_v
constexpr int OFF_PHIQ = OFF_DSOP + PHI;   // [hi|hi|lo|0]  B of Pm^T (K) and of Z (MN); then dproj (A of dx^)
constexpr int OFF_PHIK = OFF_PHIQ + PHI;   // [hi|lo|hi|0]  A of Pm^T and dV_a
constexpr int OFF_PHIT = OFF_PHIK + PHI;   // phi_q / D     B of dS (MN)
constexpr int OFF_X = OFF_PHIT + PHI;      // [2 parity] x { dx^.x^ [128], unused[128], dac[4][8] }
constexpr int XPAR = 256 + 32;
constexpr int OFF_TOK = OFF_X + 2 * XPAR * 4;  // [2 parity] x { rden[128], gden[128], sketch rows[128][ROWW] } (TMA)
constexpr int TOK_BYTES = (256 + CH * ROWW) * 4;
constexpr int OFF_BAR = OFF_TOK + 2 * TOK_BYTES;
constexpr int SMEM = OFF_BAR + 512 + 1024;
static_assert(SMEM <= 232448, "k_bwd_causal_k8 shared memory");
constexpr uint32_t TM_ZV = 32, TM_Z = 48, TM_DS = 80, TM_EG = 128, TM_PT = 192, TM_E = 256,
                   TM_DX = 256, TM_PMC = 384, TM_DV = 384;
}  // namespace ck8

// reverse chunk cursor over a CTA's item range (last item, last chunk first)
struct RCursor {
  int it, i0, t;
  Item m;
  __device__ __forceinline__ void start(const Args& a, int64_t i0_, int64_t i1) {
    i0 = int(i0_);
    it = int(i1 - 1);
    if (it >= i0) {
      m = item_of(a, it);
      t = m.t0 + ((m.t1 - m.t0 - 1) / CH) * CH;
    }
  }
  __device__ __forceinline__ bool ok() const { return it >= i0; }
  __device__ __forceinline__ void next(const Args& a) {
    t -= CH;
    if (t < m.t0) {
      --it;
      if (it >= i0) {
        m = item_of(a, it);
        t = m.t0 + ((m.t1 - m.t0 - 1) / CH) * CH;
      }
    }
  }
};

template <int P, int HB = 0, bool GRP = false, bool M4 = false>
__global__ void __launch_bounds__(NTHREADS8, 1)
    k_bwd_causal_k8(const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                    const __grid_constant__ CUtensorMap tmDK, const __grid_constant__ CUtensorMap tmRD,
                    const __grid_constant__ CUtensorMap tmGD, const __grid_constant__ CUtensorMap tmROWS,
                    const __grid_constant__ CUtensorMap tmDV, Args a) {
  using namespace ck8;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* fullK = bars + 0;     // K landed (one buffer)
  uint64_t* dkstaged = bars + 2;  // dK staged in the K buffer (256 arrivals)
  uint64_t* fullV = bars + 4;     // [2]
  uint64_t* fullO = bars + 6;     // [2]
  uint64_t* emptyO = bars + 8;    // [2]
  uint64_t* c1 = bars + 11;
  uint64_t* c2 = bars + 12;
  uint64_t* c3 = bars + 13;
  uint64_t* c4 = bars + 14;
  uint64_t* phi_ready = bars + 15;
  uint64_t* pt_ready = bars + 16;
  uint64_t* dp_ready = bars + 17;
  uint64_t* dxfree = bars + 18;
  uint64_t* wready = bars + 19;
  uint64_t* eg_ready = bars + 20;  // EG~ staged in TMEM (256 arrivals)
  uint64_t* cdv = bars + 21;       // dV MMAs done
  uint64_t* fullT = bars + 22;     // [2] per-token inputs landed (parity buffers)
  uint64_t* emptyT = bars + 24;    // [2] ... consumed (256 arrivals)
  uint64_t* dvstaged = bars + 26;  // [2] dV staged in the (consumed) V buffer (256 arrivals)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 28);

  const int warp = warp_id();
  if (threadIdx.x == 0) {
    mbar_init(fullK, 1);
    mbar_init(dkstaged, 256);
    for (int i = 4; i < 15; ++i) mbar_init(&bars[i], 1);
    mbar_init(phi_ready, 256);
    mbar_init(pt_ready, 256);
    mbar_init(dp_ready, 256);
    mbar_init(dxfree, 256);
    mbar_init(wready, 256);
    mbar_init(eg_ready, 256);
    mbar_init(cdv, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&fullT[i], 1);
      mbar_init(&emptyT[i], 256);
    }
    mbar_init(&dvstaged[0], 256);
    mbar_init(&dvstaged[1], 256);
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
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmDO);
      tma_prefetch_desc(&tmDK);
      tma_prefetch_desc(&tmRD);
      tma_prefetch_desc(&tmGD);
      tma_prefetch_desc(&tmROWS);
      tma_prefetch_desc(&tmDV);
      const uint64_t pol = policy_evict_first();
      int kt = 0, kb = 0;                  // coordinates of the dK tile staged in the K buffer
      int vt[2] = {0, 0}, vb[2] = {0, 0};  // coordinates of the dV tile held by each V buffer
      auto store_dv = [&](uint32_t j) {
        const int s = j & 1;
        mbar_wait(&dvstaged[s], (j >> 1) & 1);
        for (int h = 0; h < 2; ++h)
          tile_store<M4>(a, &tmDV, reinterpret_cast<void*>(smem + OFF_V + s * TILE + h * SUB), h * 64, vt[s], vb[s]);
        tma_store_commit();
      };
      auto store_dk = [&](uint32_t j) {
        mbar_wait(dkstaged, j & 1);
        if (!a.dproj_out)  // grouped backward: dk is formed from the summed dproj afterwards
          for (int h = 0; h < 2; ++h)
            tile_store<M4>(a, &tmDK, reinterpret_cast<void*>(smem + OFF_K + h * SUB), h * 64, kt, kb);
        tma_store_commit();
      };
      uint32_t gc = 0;
      RCursor cur;
      for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
        if (a.pf > 0) {  // reverse scan: warm L2 with the tiles a.pf chunks earlier in the sequence
          const int tp = int(cur.t) - a.pf * CH;
          if (tp >= 0)
            for (int h = 0; h < 2; ++h) {
              tile_prefetch<M4>(a, &tmK, h * 64, tp, int(cur.m.bh));
              tile_prefetch<M4>(a, &tmV, h * 64, tp, int(cur.m.bh));
              tile_prefetch<M4>(a, &tmDO, h * 64, tp, int(cur.m.bh));
            }
        }
        const int s = gc & 1;
        const int t = int(cur.t), bh = int(cur.m.bh);
        {  // per-token rden, gden, row norms of this chunk (parity buffer s)
          uint8_t* tok = smem + OFF_TOK + s * TOK_BYTES;
          const int row = bh * int(a.N) + t;
          const int prow = bh * int(a.Np) + t;  // rden / gden: row pitch Np keeps every tile 16-byte aligned
          mbar_wait(&emptyT[s], ((gc >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&fullT[s], TOK_BYTES);
          tma_load_1d(tok, &tmRD, &fullT[s], prow, pol);
          tma_load_1d(tok + 512, &tmGD, &fullT[s], prow, pol);
          tma_load_2d(tok + 1024, &tmROWS, &fullT[s], 0, row, pol);
        }
        if (gc >= 2) {  // dV of chunk gc - 2 is staged in this V buffer: store it, then refill
          store_dv(gc - 2);
          tma_store_wait_read<0>();
        }
        vt[s] = t;
        vb[s] = bh;
        RACE_TRACE(a, 1, gc);
        mbar_arrive_expect_tx(&fullV[s], TILE);
        for (int h = 0; h < 2; ++h)
          tile_load<M4>(a, smem + OFF_V + s * TILE + h * SUB, &tmV, &fullV[s], h * 64, t, bh, pol);
        mbar_wait(&emptyO[s], ((gc >> 1) & 1) ^ 1);
        RACE_TRACE(a, 2, gc);
        mbar_arrive_expect_tx(&fullO[s], TILE);
        for (int h = 0; h < 2; ++h)
          tile_load<M4>(a, smem + OFF_DO + s * TILE + h * SUB, &tmDO, &fullO[s], h * 64, t, bh, pol);
        // K last: its one buffer holds the previous chunk's dK until that is stored (K is only
        // needed by the tangent step, late in the chunk)
        if (gc >= 1) {
          store_dk(gc - 1);
          tma_store_wait_read<0>();
        }
        RACE_TRACE(a, 3, gc);
        kt = t;
        kb = bh;
        mbar_arrive_expect_tx(fullK, TILE);
        for (int h = 0; h < 2; ++h) tile_load<M4>(a, smem + OFF_K + h * SUB, &tmK, fullK, h * 64, t, bh, pol);
      }
      for (uint32_t j = gc >= 2 ? gc - 2 : 0; j < gc; ++j) store_dv(j);
      if (gc >= 1) store_dk(gc - 1);
      tma_store_wait_all<0>();
    }
  } else if (warp == 1) {
    uint32_t gc = 0, nr = 0;
    int64_t prev_bh = -1;
    RCursor cur;
    for (cur.start(a, i0, i1); cur.ok(); cur.next(a), ++gc) {
      const uint32_t par = gc & 1;
      const int s = gc & 1;
      if (cur.m.bh != prev_bh) {
        prev_bh = cur.m.bh;
        mbar_wait(wready, nr & 1);
        ++nr;
        tc_fence_after();
      }
      // (no projection MMA: phi_q, phi_k and the tanh values come from the forward's sketch rows;
      // the K tile is only needed for the sphere-tangent step and as dK staging)
      if (gc > 0) mbar_wait(dxfree, (gc - 1) & 1);  // E aliases the previous chunk's dX
      mbar_wait(&fullV[s], (gc >> 1) & 1);
      mbar_wait(&fullO[s], (gc >> 1) & 1);
      RACE_TRACE(a, 5, gc);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          umma_bf16(tmem + TM_ZV, desc_tile_k(sb + OFF_V + s * TILE, kk), desc_w(sb + OFF_DSOPT, kk), IDC_Y, kk > 0);
          umma_bf16(tmem + TM_E, desc_tile_k(sb + OFF_V + s * TILE, kk), desc_tile_k(sb + OFF_DO + s * TILE, kk), IDC_E,
                    kk > 0);
        }
        umma_commit(c1);
      }
      __syncwarp();
      mbar_wait(phi_ready, par);
      RACE_TRACE(a, 6, gc);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
          umma_bf16(tmem + TM_PMC, desc_phi_k(sb + OFF_PHIK, kk), desc_phi_k(sb + OFF_PHIQ, kk), IDC_PM, kk > 0);
        umma_commit(c2);
      }
      __syncwarp();
      mbar_wait(eg_ready, par);
      tc_fence_after();
      if (elect_one()) {  // dphi_k's intra-chunk term and the dS update: the dq-critical path
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          umma_bf16_ts(tmem + TM_Z, tmem + TM_EG + kk * 8, desc_phi_mn(sb + OFF_PHIQ, kk), IDC_Z, kk > 0);
          umma_bf16(tmem + TM_DS, desc_tile_mn(sb + OFF_DO + s * TILE, kk), desc_phi_mn(sb + OFF_PHIT, kk), IDC_ST, 1u);
        }
        umma_commit(c3);
      }
      __syncwarp();
      mbar_wait(pt_ready, par);
      RACE_TRACE(a, 7, gc);
      tc_fence_after();
      if (elect_one()) {  // dV = Phi_k dS_>c,v + P~^T dO (into the consumed Pm columns)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
          umma_bf16(tmem + TM_DV, desc_phi_k(sb + OFF_PHIK, kk), desc_phi_k(sb + OFF_DSOP, kk), IDC_DVA, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ts(tmem + TM_DV, tmem + TM_PT + kk * 8, desc_tile_mn(sb + OFF_DO + s * TILE, kk), IDC_DVB, 1u);
        umma_commit(cdv);
        umma_commit(&emptyO[s]);
      }
      __syncwarp();
      RACE_TRACE(a, 22, gc);
      if (a.dbg && blockIdx.x == 0) {
        mbar_wait(cdv, par);
        RACE_TRACE(a, 23, gc);
      }
      mbar_wait(dp_ready, par);
      RACE_TRACE(a, 8, gc);
      tc_fence_after();
      if (elect_one()) {
        // dx^ = dproj . W (hi and lo halves of dproj against W' read MN-major)
        umma_bf16(tmem + TM_DX, desc_phi_k(sb + OFF_PHIQ, 0), cq8::desc_wT(sb + OFF_W), IDC_DX, 0u);
        umma_bf16(tmem + TM_DX, desc_phi_k(sb + OFF_PHIQ, 1), cq8::desc_wT(sb + OFF_W), IDC_DX, 1u);
        umma_commit(c4);
      }
      __syncwarp();
      RACE_TRACE(a, 20, gc);
      if (a.dbg && blockIdx.x == 0) {  // trace only: time the dX MMA's completion
        mbar_wait(c4, par);
        RACE_TRACE(a, 21, gc);
      }
    }
  } else {
    const int r = crow();
    const int h = chalf();
    const int qw = warp & 3;
    const uint32_t lb = lane_base();
    const int F = a.T << a.P;
    float* xbase = reinterpret_cast<float*>(smem + OFF_X);
    {  // EG~ / P~^T blocks below the diagonal are never written: zero both A operands once
      uint32_t z[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) z[j] = 0u;
#pragma unroll
      for (int c = 0; c < 64; c += 16) tmem_st16u(tmem + lb + TM_EG + 64 * h + c, z);
      tmem_st_wait();
    }
    float dA[FP];
    uint32_t gc = 0;
    int64_t prev_bh = -1;
    RCursor cur;
    cur.start(a, i0, i1);
    for (; cur.ok(); ++gc) {
      const Item m = cur.m;
      const int64_t t = cur.t;
      const uint32_t par = gc & 1;
      const int s = gc & 1;
      float* xpar = xbase + par * XPAR;
      const bool valid = t + r < m.t1;
      const GroupPre pre = GRP ? group_prefetch(a, m.bh, t, r, valid) : GroupPre{};
      if (m.bh != prev_bh) {  // (re)load the suffix state dS_>seg, dA_>seg and W', W''
        prev_bh = m.bh;
        const float* dcar = a.tin + (m.bh * a.nseg + m.seg) * int64_t(F) * a.ldt;
        float dcol[FP];
#pragma unroll
        for (int f = 0; f < FP; ++f) {
          dcol[f] = (f < F && r < a.dvv) ? dcar[f * a.ldt + r] : 0.f;
          dA[f] = f < F ? dcar[f * a.ldt + a.dvv] : 0.f;
        }
        build_wop<256, CT0>(a, m.bh, sb + OFF_W);
        if (h == 1) {
          float z[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) z[j] = j < FP ? dcol[j] : 0.f;
          tmem_st16(tmem + lb + TM_DS, z);
#pragma unroll
          for (int j = 0; j < 16; ++j) z[j] = 0.f;
          tmem_st16(tmem + lb + TM_DS + 16, z);
          tmem_st_wait();
          write_sopT(sb + OFF_DSOPT, r, dcol);
          write_sop(sb + OFF_DSOP, r, dcol);
        }
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(wready);
      }
      // per-token inputs (TMA-loaded with Q; rows past the segment end are masked by `valid`)
      const float* tok = reinterpret_cast<const float*>(smem + OFF_TOK + (gc & 1) * TOK_BYTES);
      mbar_wait(&fullT[gc & 1], (gc >> 1) & 1);
      const float rdr_c = valid ? tok[r] : 0.f, gdr_c = valid ? tok[128 + r] : 0.f;
      const float* trow = tok + 256 + r * ROWW;  // this token's sketch row
      float hatq[5], hk[5];  // x^.w_j of this q row and this k row
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        hatq[j] = trow[j];
        hk[j] = trow[8 + j];
      }
      const Scale sck = row_scale(valid ? trow[15] : 0.f, a.normalize);
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 9, gc);
      float phq[FP], uq[5], phk[FP], uk[5];
      {
        if (h == 0) {
          row_features_hat<P, HB>(a, hatq, valid, phq, uq);
          write_phi_k(sb + OFF_PHIQ, r, phq);  // [hi|hi|lo|0]
        } else {
          row_features_hat<P, HB>(a, hk, valid, phk, uk);
          write_phi_q(sb + OFF_PHIK, r, phk);  // [hi|lo|hi|0]
        }
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(phi_ready);
        if (h == 0) {
          float pht[FP], dac[FP];
#pragma unroll
          for (int f = 0; f < FP; ++f) {
            pht[f] = phq[f] * rdr_c;
            dac[f] = phq[f] * gdr_c;
          }
          write_phi_k(sb + OFF_PHIT, r, pht);
          const float tot = warp_sum8(dac);  // recursive-halving warp reduction (FP == 8)
          if ((lane_id() & 3) == 0) xpar[256 + qw * FP + (lane_id() >> 2)] = tot;
        }
      }
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 24, gc);
      compute_bar256();  // rd / gd of every query token, dA partials
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 25, gc);
      // ---- EG~ = (E^T rd + gd) masked t >= i, my 64 columns -> TMEM A operand of Z
      mbar_wait(c1, par);
      tc_fence_after();
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int c0 = 64 * h + 32 * b;
        if ((c0 >> 5) >= qw) {  // warp-uniform; blocks below the diagonal stay zero
          float e[32];
          tmem_ld32(tmem + lb + TM_E + c0, e);
          tmem_ld_wait();
          uint32_t ue[16];
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 rd4 = *reinterpret_cast<const float4*>(tok + c0 + 4 * j4);
            const float4 gd4 = *reinterpret_cast<const float4*>(tok + 128 + c0 + 4 * j4);
            const float rdv[4] = {rd4.x, rd4.y, rd4.z, rd4.w}, gdv[4] = {gd4.x, gd4.y, gd4.z, gd4.w};
            float ee[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) ee[q] = (c0 + 4 * j4 + q >= r) ? fmaf(e[4 * j4 + q], rdv[q], gdv[q]) : 0.f;
            ue[2 * j4] = pack_bf16(ee[0], ee[1]);
            ue[2 * j4 + 1] = pack_bf16(ee[2], ee[3]);
          }
          tmem_st16u(tmem + lb + TM_EG + (c0 >> 1), ue);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(eg_ready);
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 26, gc);
      // ---- P~^T = Pm^T rd masked t >= i -> TMEM A operand of dV
      mbar_wait(c2, par);
      tc_fence_after();
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int c0 = 64 * h + 32 * b;
        if ((c0 >> 5) >= qw) {
          float pm[32];
          tmem_ld32(tmem + lb + TM_PMC + c0, pm);
          tmem_ld_wait();
          uint32_t up[16];
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 rd4 = *reinterpret_cast<const float4*>(tok + c0 + 4 * j4);
            const float rdv[4] = {rd4.x, rd4.y, rd4.z, rd4.w};
            float pp[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) pp[q] = (c0 + 4 * j4 + q >= r) ? pm[4 * j4 + q] * rdv[q] : 0.f;
            up[2 * j4] = pack_bf16(pp[0], pp[1]);
            up[2 * j4 + 1] = pack_bf16(pp[2], pp[3]);
          }
          tmem_st16u(tmem + lb + TM_PT + (c0 >> 1), up);
        }
      }
      mbar_arrive(&emptyT[gc & 1]);  // last read of this chunk's per-token inputs
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(pt_ready);
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 27, gc);
      // ---- dphi_k -> dproj (Z and the dS update are done at c3)
      mbar_wait(c3, par);
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 11, gc);
      tc_fence_after();
      // (the second half, which holds phi_k, runs the feature VJP for both; the first half reads the dS
      // state out below)
      if (h == 1) {
        float zhi[8], zlo[8], zv[16];  // Z columns 8..15 / 24..31: the duplicate hi copy and padding
        tmem_ld8(tmem + lb + TM_Z, zhi);
        tmem_ld8(tmem + lb + TM_Z + 16, zlo);
        tmem_ld16(tmem + lb + TM_ZV, zv);
        tmem_ld_wait();
        float dphi[FP];
#pragma unroll
        for (int f = 0; f < FP; ++f) dphi[f] = zv[f] + zv[8 + f] + dA[f] + zhi[f] + zlo[f];
        float dproj[8];
        row_feature_vjp<P, HB>(a, uk, phk, dphi, dproj);
        if (GRP && a.dproj_out && valid) emit_dproj(a, m.bh * a.N + t + r, dproj, pre);
        xpar[r] = dot_from_proj(dproj, hk);  // dx^.x^ for both halves' tangent step (read after c4)
        cq8::write_dproj_w(sb + OFF_PHIQ, r, dproj, a.TP);  // Phi_q is dead after Pm, Z (c3)
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(dp_ready);
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 28, gc);
#pragma unroll
      for (int f = 0; f < FP; ++f)
        dA[f] += ((xpar[256 + f] + xpar[256 + FP + f]) + xpar[256 + 2 * FP + f]) + xpar[256 + 3 * FP + f];
      // ---- dV out; dS_>c-1 operands for the next (earlier) chunk once the dV MMA has read DSOP
      mbar_wait(cdv, par);
      tc_fence_after();
      if (h == 0) {
        float dhi[8], dlo[8];
        tmem_ld8(tmem + lb + TM_DS, dhi);
        tmem_ld8(tmem + lb + TM_DS + 16, dlo);
        tmem_ld_wait();
        float dsn[FP];
#pragma unroll
        for (int f = 0; f < FP; ++f) dsn[f] = dhi[f] + dlo[f];
        write_sopT(sb + OFF_DSOPT, r, dsn);
        write_sop(sb + OFF_DSOP, r, dsn);
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {  // dV (my 64 columns) into the V tile (consumed at c1); the producer stores it
        const int c0 = 64 * h + 32 * b;
        float v[32];
        tmem_ld32(tmem + lb + TM_DV + c0, v);
        tmem_ld_wait();
        stage32_p(smem + OFF_V + s * TILE, r, v, c0);
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&dvstaged[s]);
      cur.next(a);
      // ---- dk (my 64 columns) in place of k; the producer stores it
      mbar_wait(c4, par);
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 12, gc);
      tc_fence_after();
      mbar_wait(fullK, gc & 1);  // k itself is only read here (x^ of the tangent step)
      tangent_half_inplace(tmem + lb + TM_DX, smem + OFF_K, r, h, sck, xpar[r]);
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(dkstaged);
      mbar_arrive(dxfree);
      if (threadIdx.x == a.ttid) RACE_TRACE(a, 13, gc);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) RACE_CTA_TIME(a, 1);
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace tcfast

// ---- entry points ------------------------------------------------------------
cudaError_t tc_bwd_causal_q(const Geo& g, const void* q, const void* k, const void* v, const void* d_o,
                            const float* w, const float* car, const float* nrm, void* dq, float* rden, float* gden,
                            float* dpart, cudaStream_t st) {
  using namespace tcfast;
  CUtensorMap mq, mk, mv, mdo, mdq;
  if (!make_map(&mq, q, g, g.d, L_Q) || !make_map(&mk, k, g, g.d, L_K) || !make_map(&mv, v, g, g.dv, L_V) ||
      !make_map(&mdo, d_o, g, g.dv, L_DO) || !make_map(&mdq, dq, g, g.d, L_DQ))
    return cudaErrorInvalidValue;
  Args a = make_args(g);
  a.w = w;
  a.tin = car;
  a.tout = dpart;
  a.rows_in = nrm;
  a.dproj_out = g.dproj_q;
  a.dbg = trace_for("bq");
  if (!nrm) return cudaErrorInvalidValue;  // race_abi.cu always supplies the forward's rows
  CUtensorMap mrows;
  if (!make_map_rows(&mrows, nrm, g.BH * g.N)) return cudaErrorInvalidValue;
  const bool grp = g.ext_rden || g.dproj_q;  // a pass of a grouped backward (race_abi.cu)
#define RACE_CQ8(...)                                                                                           \
  return launch_nt(k_bwd_causal_q8<__VA_ARGS__>, NTHREADS8, cq8::SMEM, grid_for(g), st, mq, mk, mv, mdo, mdq, \
                   mrows, a, rden, gden)
  switch (pass_corner_bits(g)) {
    case 1: if (g.strided()) RACE_CQ8(1, 0, false, true); if (grp) RACE_CQ8(1, 0, true); RACE_CQ8(1);
    case 2: if (g.strided()) RACE_CQ8(2, 0, false, true); if (grp) RACE_CQ8(2, 0, true); RACE_CQ8(2);
    default:
      if (g.strided()) RACE_CQ8(3, 0, false, true);  // strided operands: one-pass problems only
      if (g.cb) RACE_CQ8(3, 2, true);
      if (grp) RACE_CQ8(3, 0, true);
      RACE_CQ8(3);
  }
#undef RACE_CQ8

}

cudaError_t tc_bwd_causal_k(const Geo& g, const void* q, const void* k, const void* v, const void* d_o,
                            const float* w, const float* rden, const float* gden, const float* dcar,
                            const float* nrm, void* dk, void* dv, cudaStream_t st) {
  using namespace tcfast;
  CUtensorMap mq, mk, mv, mdo, mdk, mdv;
  if (!make_map(&mq, q, g, g.d, L_Q) || !make_map(&mk, k, g, g.d, L_K) || !make_map(&mv, v, g, g.dv, L_V) ||
      !make_map(&mdo, d_o, g, g.dv, L_DO) || !make_map(&mdk, dk, g, g.d, L_DK) || !make_map(&mdv, dv, g, g.dv, L_DV))
    return cudaErrorInvalidValue;
  Args a = make_args(g);
  a.w = w;
  a.tin = dcar;
  a.rows_in = nrm;
  a.dproj_out = g.dproj_k;
  a.dbg = trace_for("bk");
  if (!nrm) return cudaErrorInvalidValue;
  CUtensorMap mrd, mgd, mrows, mdv2;
  if (!make_map(&mdv2, dv, g, g.dv, L_DV)) return cudaErrorInvalidValue;
  const int64_t np = (g.N + 3) & ~int64_t(3);
  if (!make_map_f32_1d(&mrd, rden, g.BH * np, 128) || !make_map_f32_1d(&mgd, gden, g.BH * np, 128) ||
      !make_map_rows(&mrows, nrm, g.BH * g.N))
    return cudaErrorInvalidValue;
  const bool grp = g.ext_rden || g.dproj_k;
#define RACE_CK8(...)                                                                                           \
  return launch_nt(k_bwd_causal_k8<__VA_ARGS__>, NTHREADS8, ck8::SMEM, grid_for(g), st, mk, mv, mdo, mdk, mrd, \
                   mgd, mrows, mdv2, a)
  switch (pass_corner_bits(g)) {
    case 1: if (g.strided()) RACE_CK8(1, 0, false, true); if (grp) RACE_CK8(1, 0, true); RACE_CK8(1);
    case 2: if (g.strided()) RACE_CK8(2, 0, false, true); if (grp) RACE_CK8(2, 0, true); RACE_CK8(2);
    default:
      if (g.strided()) RACE_CK8(3, 0, false, true);  // strided operands: one-pass problems only
      if (g.cb) RACE_CK8(3, 2, true);
      if (grp) RACE_CK8(3, 0, true);
      RACE_CK8(3);
  }
#undef RACE_CK8

}

}  // namespace race
