// race_simt.cu -- generic CUDA-core kernels for every RACE attention pass.
//
// These handle ANY shape the reference accepts within the shared-memory
// budget (d, dv, P, T arbitrary; N arbitrary incl. ragged tails).  They run
// entirely on the device; the sm_100a tcgen05 fast path (race_tc.cu) takes
// over for the production shapes.  Everything here follows the chunk
// formulation of DESIGN.md section 3, which restates the reference's
// per-table loops (ra/forward.py:77-144, ra/backward.py:93-235):
//
//   S      = phi(K)^T [V | 1]                                (F x (dv+1))
//   fwd    : D_t = phi_q,t . A,  O_t = phi_q,t S_v / D_t,    den_t = D_t / T
//   causal : S_<c carried across tiles/segments; intra-tile  P = tril(Phi_q Phi_k^T)
//   bwd    : y_t = S_v dO_t,  rho_t = dO_t . O_t,
//            dphi_q,t = (y_t - rho_t A) / D_t   (+ intra-tile terms, causal)
//            G_t = [dO_t / D_t | -rho_t / D_t],  dS = Phi_q^T G
//            dphi_k,i = [v_i | 1] dS^T,  dV_i = phi_k,i dS_v
//   then the softmax / tanh / row-normalisation VJPs.
//
// Determinism: no atomics; every reduction has a fixed order, so results are
// bit-identical run to run (the reference's criterion 9, ra/acceptance.py:419).
#include <cstdlib>

#include "race_common.cuh"
#include "race_internal.h"

namespace race {
namespace simt {

#ifndef RACE_SIMT_TILE
#define RACE_SIMT_TILE 32
#endif
constexpr int TILE = RACE_SIMT_TILE;  // tokens per tile
constexpr int NT = 256;    // threads per CTA

__host__ __device__ inline int odd_ld(int n) { return n | 1; }

// ---------------------------------------------------------------------------
// shared-memory plan (same arithmetic on host and device)
// ---------------------------------------------------------------------------
enum Need : unsigned {
  kW = 1u << 0, kS = 1u << 1, kAcc = 1u << 2, kXq = 1u << 3, kXk = 1u << 4,
  kDx = 1u << 5, kV = 1u << 6, kG = 1u << 7, kPhq = 1u << 8, kPhk = 1u << 9,
  kDph = 1u << 10, kY = 1u << 11, kU = 1u << 12, kDproj = 1u << 13,
  kPm = 1u << 14, kEm = 1u << 15,
};

struct Plan {
  int d, dv, P, T, R, F, TP;
  int cb;        // corner bits of this pass (< P for a corner group, Geo::cb), else P
  int64_t chi;   // fixed high corner bits of a corner group
  int ldx, ldv, ldf, ldS, ldu, ldp;
  // float offsets (all buffers are float)
  int oW, oS, oAcc, oXq, oXk, oDx, oV, oG, oPhq, oPhk, oDph, oY, oU, oDproj, oPm, oEm;
  int oPj;       // [2][TILE][ldu] projection scratch
  int oRow;      // 8 row-scalar arrays of TILE floats
  int total;     // floats

  __host__ __device__ Plan(const Geo& g, unsigned need) {
    d = g.d; dv = g.dv; P = g.P; T = g.T; cb = pass_corner_bits(g); chi = g.chi;
    R = 1 << cb; F = g.T * R; TP = g.T * g.P;
    ldx = odd_ld(d + 1); ldv = odd_ld(dv + 1); ldf = odd_ld(F); ldS = odd_ld(dv + 1);
    ldu = odd_ld(TP); ldp = TILE + 1;
    int o = 0;
    auto take = [&](unsigned bit, int n) { int r = (need & bit) ? o : -1; if (need & bit) o += (n + 3) & ~3; return r; };
    oW = take(kW, TP * d);
    oS = take(kS, F * ldS);
    oAcc = take(kAcc, F * ldS);
    oXq = take(kXq, TILE * ldx);
    oXk = take(kXk, TILE * ldx);
    oDx = take(kDx, TILE * ldx);
    oV = take(kV, TILE * ldv);
    oG = take(kG, TILE * ldv);
    oPhq = take(kPhq, TILE * ldf);
    oPhk = take(kPhk, TILE * ldf);
    oDph = take(kDph, TILE * ldf);
    oY = take(kY, TILE * ldf);
    oU = take(kU, TILE * ldu);
    oDproj = take(kDproj, TILE * ldu);
    oPm = take(kPm, TILE * ldp);
    oEm = take(kEm, TILE * ldp);
    oPj = o; o += (2 * TILE * ldu + 3) & ~3;  // projections of up to two tiles (tile_features scratch)
    oRow = o; o += 8 * TILE;
    total = o;
  }
  __host__ __device__ size_t bytes() const { return size_t(total) * sizeof(float); }
};

extern __shared__ float4 smem_f4[];

// row-scalar slots inside Plan::oRow
enum RowSlot { kScQ = 0, kScK = 1, kD = 2, kRho = 3, kRD = 4, kGD = 5, kDot = 6, kTmp = 7 };

// ---------------------------------------------------------------------------
// block-level building blocks
// ---------------------------------------------------------------------------

// Load `rows` rows (row stride `cols`) of a [*, cols] tensor into smem
// (stride ld), zero-filling rows >= rows.  If `scale` is given, also stores
// the per-row normalisation scale: ||x|| (or -1 if < 1e-12, the pass-through
// rows of ra/core.py:120-122), or 1 when normalisation is off.
template <typename Tin>
__device__ void load_rows(const Tin* __restrict__ src, int rows, int cols, float* dst, int ld,
                          float* scale, bool normalize) {
  // each warp owns RPW rows; all RPW x 4 loads of a 128-column block are issued before any is used
  constexpr int RPW = TILE / (NT / 32);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float ss[RPW];
#pragma unroll
  for (int i = 0; i < RPW; ++i) ss[i] = 0.f;
  for (int c0 = 0; c0 < cols; c0 += 128) {
    float x[RPW][4];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int r = warp + i * (NT / 32);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + lane + 32 * j;
        x[i][j] = (r < rows && c < cols) ? to_f32(src[size_t(r) * cols + c]) : 0.f;
      }
    }
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int r = warp + i * (NT / 32);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + lane + 32 * j;
        if (c < cols) {
          dst[r * ld + c] = x[i][j];
          ss[i] = fmaf(x[i][j], x[i][j], ss[i]);
        }
      }
    }
  }
  if (scale) {
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const float t = warp_sum(ss[i]);
      if (lane == 0) {
        const float nrm = sqrtf(t);
        scale[warp + i * (NT / 32)] = normalize ? (nrm < kZeroRowEps ? -1.f : nrm) : 1.f;
      }
    }
  }
}

// two load_rows at once: all loads of both tiles' 128-column blocks are in flight together
template <typename Tin>
__device__ void load_rows2(const Tin* __restrict__ srcA, int colsA, float* dstA, int ldA, float* scaleA,
                           const Tin* __restrict__ srcB, int colsB, float* dstB, int ldB, float* scaleB, int rows,
                           bool normalize) {
  constexpr int RPW = TILE / (NT / 32);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (colsA > 128 || colsB > 128) {  // wide rows: one tile after the other
    load_rows<Tin>(srcA, rows, colsA, dstA, ldA, scaleA, normalize);
    load_rows<Tin>(srcB, rows, colsB, dstB, ldB, scaleB, normalize);
    return;
  }
  float xa[RPW][4], xb[RPW][4];
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = warp + i * (NT / 32);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = lane + 32 * j;
      xa[i][j] = (r < rows && c < colsA) ? to_f32(srcA[size_t(r) * colsA + c]) : 0.f;
      xb[i][j] = (r < rows && c < colsB) ? to_f32(srcB[size_t(r) * colsB + c]) : 0.f;
    }
  }
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = warp + i * (NT / 32);
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = lane + 32 * j;
      if (c < colsA) {
        dstA[r * ldA + c] = xa[i][j];
        sa = fmaf(xa[i][j], xa[i][j], sa);
      }
      if (c < colsB) {
        dstB[r * ldB + c] = xb[i][j];
        sb = fmaf(xb[i][j], xb[i][j], sb);
      }
    }
    if (scaleA) {
      sa = warp_sum(sa);
      if (lane == 0) {
        const float nrm = sqrtf(sa);
        scaleA[r] = normalize ? (nrm < kZeroRowEps ? -1.f : nrm) : 1.f;
      }
    }
    if (scaleB) {
      sb = warp_sum(sb);
      if (lane == 0) {
        const float nrm = sqrtf(sb);
        scaleB[r] = normalize ? (nrm < kZeroRowEps ? -1.f : nrm) : 1.f;
      }
    }
  }
}

// V (or dO) tile with an appended ones column at index dv (1 for valid rows).
template <typename Tin>
__device__ void load_v_ones(const Tin* __restrict__ src, int rows, int dv, float* dst, int ld) {
  load_rows<Tin>(src, rows, dv, dst, ld, nullptr, false);
  for (int r = threadIdx.x; r < TILE; r += NT) dst[r * ld + dv] = r < rows ? 1.f : 0.f;
}

// phi (and optionally u) for the TILE rows of one or two tiles (n = 1, 2).  Two phases so that
// every thread has work: (1) items (tile, hyperplane, row): one projection x . w_j each (rows of a
// warp share w_j: broadcast; odd row stride: conflict-free), (2) items (tile, table, row): tanh and
// the corner softmax.
// one tile: items (row, table), each computing its P projections (no scratch, no barrier)
__device__ void tile_features(const Plan& pl, const float* xs, const float* scale, const float* ws,
                              float beta, float* phi, float* u_out) {
  for (int it = threadIdx.x; it < TILE * pl.T; it += NT) {
    const int tau = it / TILE, r = it % TILE;
    const float sc = scale[r];
    const float inv = sc > 0.f ? 1.f / sc : 1.f;
    float u[kPMax];
    const float* x = xs + r * pl.ldx;
    auto proj = [&](int p) {
      const float* w = ws + (tau * pl.P + p) * pl.d;
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;  // four independent chains (fixed order)
      int c = 0;
      for (; c + 4 <= pl.d; c += 4) {
        a0 = fmaf(x[c], w[c], a0);
        a1 = fmaf(x[c + 1], w[c + 1], a1);
        a2 = fmaf(x[c + 2], w[c + 2], a2);
        a3 = fmaf(x[c + 3], w[c + 3], a3);
      }
      for (; c < pl.d; ++c) a0 = fmaf(x[c], w[c], a0);
      return tanhf(((a0 + a1) + (a2 + a3)) * inv);
    };
#pragma unroll
    for (int p = 0; p < kPMax; ++p) {
      if (p < pl.cb) {
        u[p] = proj(p);
        if (u_out) u_out[r * pl.ldu + tau * pl.P + p] = u[p];
      }
    }
    float* out = phi + r * pl.ldf + tau * pl.R;
    corner_softmax(u, pl.cb, beta, out);
    if (pl.cb < pl.P) {  // corner group: the fixed high bits scale every corner of the pass
      float m = 1.f;
      for (int p = pl.cb; p < pl.P; ++p) {
        const float up = proj(p);
        if (u_out) u_out[r * pl.ldu + tau * pl.P + p] = up;
        m *= corner_factor(up, (pl.chi >> (p - pl.cb)) & 1, beta);
      }
      for (int rr = 0; rr < pl.R; ++rr) out[rr] *= m;
    }
  }
}

__device__ void tile_features_n(const Plan& pl, int n, const float* xs0, const float* sc0, float* phi0, float* u0,
                                const float* xs1, const float* sc1, float* phi1, float* u1, const float* ws,
                                float beta) {
  float* pj = reinterpret_cast<float*>(smem_f4) + pl.oPj;
  const int per = TILE * pl.TP;
  for (int it = threadIdx.x; it < n * per; it += NT) {
    const int t = it / per, rem = it % per, j = rem / TILE, r = rem % TILE;
    const float* x = (t ? xs1 : xs0) + r * pl.ldx;
    const float* w = ws + j * pl.d;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;  // four independent chains (fixed order)
    int c = 0;
    for (; c + 4 <= pl.d; c += 4) {
      a0 = fmaf(x[c], w[c], a0);
      a1 = fmaf(x[c + 1], w[c + 1], a1);
      a2 = fmaf(x[c + 2], w[c + 2], a2);
      a3 = fmaf(x[c + 3], w[c + 3], a3);
    }
    for (; c < pl.d; ++c) a0 = fmaf(x[c], w[c], a0);
    pj[(t * TILE + r) * pl.ldu + j] = (a0 + a1) + (a2 + a3);
  }
  __syncthreads();
  const int per2 = TILE * pl.T;
  for (int it = threadIdx.x; it < n * per2; it += NT) {
    const int t = it / per2, rem = it % per2, tau = rem / TILE, r = rem % TILE;
    const float sc = (t ? sc1 : sc0)[r];
    const float inv = sc > 0.f ? 1.f / sc : 1.f;
    float* u_out = t ? u1 : u0;
    float u[kPMax];
#pragma unroll
    for (int p = 0; p < kPMax; ++p) {
      if (p < pl.cb) {
        u[p] = tanhf(pj[(t * TILE + r) * pl.ldu + tau * pl.P + p] * inv);
        if (u_out) u_out[r * pl.ldu + tau * pl.P + p] = u[p];
      }
    }
    float* out = (t ? phi1 : phi0) + r * pl.ldf + tau * pl.R;
    corner_softmax(u, pl.cb, beta, out);
    if (pl.cb < pl.P) {  // corner group (see tile_features)
      float m = 1.f;
      for (int p = pl.cb; p < pl.P; ++p) {
        const float up = tanhf(pj[(t * TILE + r) * pl.ldu + tau * pl.P + p] * inv);
        if (u_out) u_out[r * pl.ldu + tau * pl.P + p] = up;
        m *= corner_factor(up, (pl.chi >> (p - pl.cb)) & 1, beta);
      }
      for (int rr = 0; rr < pl.R; ++rr) out[rr] *= m;
    }
  }
  __syncthreads();  // pj is reused by the next call
}

// Factored feature VJP of one (row, table) over the corners of a corner group (ra/backward.py:65-88):
// phi_r = prod_t sigma(2 beta c_rt u_t)  =>  du_t = 2 beta sum_r dphi_r phi_r c_rt (1 - sigma(2 beta c_rt u_t)).
// Low bits t < cb: split the sum by c_rt = +-1 (S+ and s - S+); high bits: c_t is fixed by chi, so
// du_t = 2 beta c_t (1 - sigma_t) s.  Sums over groups give the full VJP (it is linear in the corners).
// Writes dproj_t = du_t (1 - u_t^2) for the table's P projections.
__device__ __forceinline__ void group_feature_vjp(const Plan& pl, const float* ph, const float* dp, float s,
                                                  const float* u, float beta, float* dproj) {
  float splus[kPMax];
#pragma unroll
  for (int p = 0; p < kPMax; ++p) splus[p] = 0.f;
  for (int rr = 0; rr < pl.R; ++rr) {
    const float x = dp[rr] * ph[rr];
#pragma unroll
    for (int p = 0; p < kPMax; ++p)
      if (p < pl.cb && !((rr >> p) & 1)) splus[p] += x;
  }
#pragma unroll
  for (int p = 0; p < kPMax; ++p) {
    if (p < pl.cb) {
      const float sp = sigmoid_pos(2.f * beta * u[p]);  // sigma(2 beta u): c = +1 corners
      const float du = 2.f * beta * ((1.f - sp) * splus[p] - sp * (s - splus[p]));
      dproj[p] = du * (1.f - u[p] * u[p]);
    }
  }
  for (int p = pl.cb; p < pl.P; ++p) {
    const bool neg = (pl.chi >> (p - pl.cb)) & 1;  // c_t = -1
    const float sp = sigmoid_pos(2.f * beta * u[p]);
    const float du = 2.f * beta * (neg ? -sp : (1.f - sp)) * s;
    dproj[p] = du * (1.f - u[p] * u[p]);
  }
}

// Feature VJP for the TILE rows: given dphi (smem [TILE][ldf]) produce dx
// (the gradient w.r.t. the RAW input rows, i.e. including the
// row-normalisation VJP of ra/core.py:126-139) and write valid rows to dst.
// ra/backward.py:53-90 (softmax + tanh VJP), then dx^ = dproj . W.
template <typename Tout>
__device__ void tile_feature_vjp(const Plan& pl, const float* xs, const float* scale,
                                 const float* ws, float beta, const float* phi, const float* u,
                                 const float* dphi, float* dproj, float* dx, float* dots,
                                 bool normalize, int rows, Tout* __restrict__ dst) {
  // (1) softmax + tanh VJP per (row, table)
  for (int it = threadIdx.x; it < TILE * pl.T; it += NT) {
    const int tau = it / TILE, r = it % TILE;
    const float* ph = phi + r * pl.ldf + tau * pl.R;
    const float* dp = dphi + r * pl.ldf + tau * pl.R;
    float s = 0.f;
    for (int rr = 0; rr < pl.R; ++rr) s = fmaf(dp[rr], ph[rr], s);
    if (pl.cb < pl.P) {  // corner group: factored VJP, exact per corner subset (ra/backward.py:65-88)
      group_feature_vjp(pl, ph, dp, s, u + r * pl.ldu + tau * pl.P, beta, dproj + r * pl.ldu + tau * pl.P);
      continue;
    }
    float du[kPMax];
#pragma unroll
    for (int p = 0; p < kPMax; ++p) du[p] = 0.f;
    for (int rr = 0; rr < pl.R; ++rr) {
      const float dl = ph[rr] * (dp[rr] - s);
#pragma unroll
      for (int p = 0; p < kPMax; ++p)
        if (p < pl.P) du[p] += ((rr >> p) & 1) ? -dl : dl;
    }
#pragma unroll
    for (int p = 0; p < kPMax; ++p) {
      if (p < pl.P) {
        const float uu = u[r * pl.ldu + tau * pl.P + p];
        dproj[r * pl.ldu + tau * pl.P + p] = beta * du[p] * (1.f - uu * uu);
      }
    }
  }
  __syncthreads();
  // (2)-(4) a warp per row (lanes over columns, no cross-warp dependency): dx^ = dproj . W, the
  // radial component (dx^ . x^), then the sphere-tangent projection scaled by 1/||x||
  // (pass-through rows keep dx^); the projection used x^ = x / scale
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < TILE; r += NT / 32) {
    const float* dpr = dproj + r * pl.ldu;
    const float sc = scale[r];
    const bool tang = normalize && sc > 0.f;
    float dot = 0.f;
    for (int c = lane; c < pl.d; c += 32) {
      float acc = 0.f;
      for (int j = 0; j < pl.TP; ++j) acc = fmaf(dpr[j], ws[j * pl.d + c], acc);
      dx[r * pl.ldx + c] = acc;
      if (tang) dot = fmaf(acc, xs[r * pl.ldx + c], dot);
    }
    dot = tang ? warp_sum(dot) / sc : 0.f;
    if (lane == 0) dots[r] = dot;
    if (r < rows) {
      const float rs = tang ? 1.f / sc : 1.f;
      for (int c = lane; c < pl.d; c += 32) {
        float g = dx[r * pl.ldx + c];  // this lane's own value
        if (tang) g = (g - dot * xs[r * pl.ldx + c] * rs) * rs;
        dst[size_t(r) * pl.d + c] = from_f32<Tout>(g);
      }
    }
  }
}

// out[r][j] = keep(r, j) ? sum_{c < len} X[r][c] * Y[j][c] : 0 for r < nr, j < nc (both even), in
// 2 x 2 register micro-tiles (each smem value loaded feeds two FMAs); fixed summation order
template <typename Keep>
__device__ __forceinline__ void gram2(const float* X, int ldx, int nr, const float* Y, int ldy, int nc, int len,
                                      float* out, int ldo, Keep keep) {
  const int cols = nc / 2;
  for (int it = threadIdx.x; it < (nr / 2) * cols; it += NT) {
    const int r0 = 2 * (it / cols), j0 = 2 * (it % cols);
    const bool k00 = keep(r0, j0), k01 = keep(r0, j0 + 1), k10 = keep(r0 + 1, j0), k11 = keep(r0 + 1, j0 + 1);
    float a00 = 0.f, a01 = 0.f, a10 = 0.f, a11 = 0.f;
    if (k00 || k01 || k10 || k11) {
      const float* x0 = X + r0 * ldx;
      const float* x1 = x0 + ldx;
      const float* y0 = Y + j0 * ldy;
      const float* y1 = y0 + ldy;
#pragma unroll 4
      for (int c = 0; c < len; ++c) {
        const float u0 = x0[c], u1 = x1[c], w0 = y0[c], w1 = y1[c];
        a00 = fmaf(u0, w0, a00);
        a01 = fmaf(u0, w1, a01);
        a10 = fmaf(u1, w0, a10);
        a11 = fmaf(u1, w1, a11);
      }
    }
    out[r0 * ldo + j0] = k00 ? a00 : 0.f;
    out[r0 * ldo + j0 + 1] = k01 ? a01 : 0.f;
    out[(r0 + 1) * ldo + j0] = k10 ? a10 : 0.f;
    out[(r0 + 1) * ldo + j0 + 1] = k11 ? a11 : 0.f;
  }
}
template <typename Keep>
__device__ __forceinline__ void tile_gram(const float* X, int ldx, const float* Y, int ldy, int len, float* out,
                                          int ldo, Keep keep) {
  gram2(X, ldx, TILE, Y, ldy, TILE, len, out, ldo, keep);
}
struct KeepAll {
  __device__ bool operator()(int, int) const { return true; }
};

// acc[f][c] += sum_{t<TILE} A[t][f] * B[t][c] for every (f, c <= dv); each
// output is owned by one thread, so this is a fixed-order reduction.
__device__ __forceinline__ void owner_accumulate(const Plan& pl, float* acc, const float* A,
                                                 const float* B) {
  // 2 (f) x 2 (c) outputs per item: each A / B value loaded feeds two FMAs (F is even: T * 2^P)
  const int nc = pl.dv + 1, cp = (nc + 1) / 2;
  for (int o = threadIdx.x; o < (pl.F / 2) * cp; o += NT) {
    const int f0 = 2 * (o / cp), c0 = 2 * (o % cp);
    const bool c1ok = c0 + 1 < nc;
    float p00 = 0.f, p01 = 0.f, p10 = 0.f, p11 = 0.f;
#pragma unroll 8
    for (int t = 0; t < TILE; ++t) {
      const float a0 = A[t * pl.ldf + f0], a1 = A[t * pl.ldf + f0 + 1];
      const float b0 = B[t * pl.ldv + c0], b1 = c1ok ? B[t * pl.ldv + c0 + 1] : 0.f;
      p00 = fmaf(a0, b0, p00);
      p01 = fmaf(a0, b1, p01);
      p10 = fmaf(a1, b0, p10);
      p11 = fmaf(a1, b1, p11);
    }
    acc[f0 * pl.ldS + c0] += p00;
    acc[(f0 + 1) * pl.ldS + c0] += p10;
    if (c1ok) {
      acc[f0 * pl.ldS + c0 + 1] += p01;
      acc[(f0 + 1) * pl.ldS + c0 + 1] += p11;
    }
  }
}

__device__ __forceinline__ void load_w(const Plan& pl, const float* __restrict__ w, float* ws) {
  for (int i = threadIdx.x; i < pl.TP * pl.d; i += NT) ws[i] = w[i];
}

__device__ __forceinline__ void load_table(const Plan& pl, const float* __restrict__ src, float* dst) {
  const int nout = pl.F * (pl.dv + 1);
  for (int o = threadIdx.x; o < nout; o += NT) {
    const int f = o / (pl.dv + 1), c = o % (pl.dv + 1);
    dst[f * pl.ldS + c] = src ? src[o] : 0.f;
  }
}

__device__ __forceinline__ void store_table(const Plan& pl, const float* src, float* __restrict__ dst) {
  const int nout = pl.F * (pl.dv + 1);
  for (int o = threadIdx.x; o < nout; o += NT) {
    const int f = o / (pl.dv + 1), c = o % (pl.dv + 1);
    dst[o] = src[f * pl.ldS + c];
  }
}

struct Range {
  int64_t begin, end;
};
__device__ __forceinline__ Range seg_range(const Geo& g) {
  const int64_t b = int64_t(blockIdx.x) * g.seg_tokens;
  const int64_t e = b + g.seg_tokens < g.N ? b + g.seg_tokens : g.N;
  return {b, e};
}
__device__ __forceinline__ const float* w_of(const Geo& g, const float* w, int64_t bh) {
  return w + (g.w_per_head ? (bh % g.H) * int64_t(g.T * g.P * g.d) : 0);
}


// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

// part[bh][seg] = phi(K_seg)^T [V_seg | 1]
template <typename Tin>
__global__ void __launch_bounds__(NT) k_aggregate(Geo g, const Tin* __restrict__ k,
                                                  const Tin* __restrict__ v,
                                                  const float* __restrict__ w, float* __restrict__ part) {
  const Plan pl(g, kW | kAcc | kXk | kV | kPhk);
  float* sm = reinterpret_cast<float*>(smem_f4);
  float* ws = sm + pl.oW; float* acc = sm + pl.oAcc; float* xk = sm + pl.oXk;
  float* vs = sm + pl.oV; float* phk = sm + pl.oPhk; float* rowv = sm + pl.oRow;
  const int64_t bh = blockIdx.y;
  const Range rg = seg_range(g);
  load_w(pl, w_of(g, w, bh), ws);
  load_table(pl, nullptr, acc);
  for (int64_t t0 = rg.begin; t0 < rg.end; t0 += TILE) {
    const int rows = int(rg.end - t0 < TILE ? rg.end - t0 : TILE);
    __syncthreads();
    load_rows<Tin>(k + (bh * g.N + t0) * g.d, rows, g.d, xk, pl.ldx, rowv + kScK * TILE, g.normalize);
    load_v_ones<Tin>(v + (bh * g.N + t0) * g.dv, rows, g.dv, vs, pl.ldv);
    __syncthreads();
    tile_features(pl, xk, rowv + kScK * TILE, ws, g.beta, phk, nullptr);
    __syncthreads();
    owner_accumulate(pl, acc, phk, vs);
  }
  __syncthreads();
  store_table(pl, acc, part + (bh * g.nseg + blockIdx.x) * int64_t(pl.F * (g.dv + 1)));
}

// Non-causal readout: O = phi_q S_v / D, den = D / T.
template <typename Tin>
__global__ void __launch_bounds__(NT) k_readout(Geo g, const Tin* __restrict__ q,
                                                const float* __restrict__ w,
                                                const float* __restrict__ tables, Tin* __restrict__ o,
                                                float* __restrict__ den) {
  const Plan pl(g, kW | kS | kXq | kPhq);
  float* sm = reinterpret_cast<float*>(smem_f4);
  float* ws = sm + pl.oW; float* S = sm + pl.oS; float* xq = sm + pl.oXq; float* phq = sm + pl.oPhq;
  float* rowv = sm + pl.oRow;
  const int64_t bh = blockIdx.y;
  const Range rg = seg_range(g);
  load_w(pl, w_of(g, w, bh), ws);
  load_table(pl, tables + bh * int64_t(pl.F * (g.dv + 1)), S);
  const float invT = 1.f / float(g.T);
  for (int64_t t0 = rg.begin; t0 < rg.end; t0 += TILE) {
    const int rows = int(rg.end - t0 < TILE ? rg.end - t0 : TILE);
    __syncthreads();
    load_rows<Tin>(q + (bh * g.N + t0) * g.d, rows, g.d, xq, pl.ldx, rowv + kScQ * TILE, g.normalize);
    __syncthreads();
    tile_features(pl, xq, rowv + kScQ * TILE, ws, g.beta, phq, nullptr);
    __syncthreads();
    for (int r = threadIdx.x; r < TILE; r += NT) {
      float D = 0.f;
      for (int f = 0; f < pl.F; ++f) D = fmaf(phq[r * pl.ldf + f], S[f * pl.ldS + g.dv], D);
      rowv[kD * TILE + r] = D;
      if (r < rows) den[bh * g.N + t0 + r] = D * invT;
    }
    __syncthreads();
    for (int it = threadIdx.x; it < rows * g.dv; it += NT) {
      const int r = it / g.dv, c = it % g.dv;
      float num = 0.f;
      for (int f = 0; f < pl.F; ++f) num = fmaf(phq[r * pl.ldf + f], S[f * pl.ldS + c], num);
      const float D = rowv[kD * TILE + r];
      o[(bh * g.N + t0 + r) * g.dv + c] = from_f32<Tin>(D * invT <= kDegenerateDenEps ? 0.f : num / D);
    }
  }
}

// Causal forward over one segment with carry-in S_<seg.
template <typename Tin>
__global__ void __launch_bounds__(NT, 2) k_causal_fwd(Geo g, const Tin* __restrict__ q,
                                                   const Tin* __restrict__ k, const Tin* __restrict__ v,
                                                   const float* __restrict__ w,
                                                   const float* __restrict__ carries,
                                                   Tin* __restrict__ o, float* __restrict__ den,
                                                   float* __restrict__ nrm) {
  const Plan pl(g, kW | kS | kXq | kXk | kV | kPhq | kPhk | kPm);
  float* sm = reinterpret_cast<float*>(smem_f4);
  float* ws = sm + pl.oW; float* S = sm + pl.oS; float* xq = sm + pl.oXq; float* xk = sm + pl.oXk;
  float* vs = sm + pl.oV; float* phq = sm + pl.oPhq; float* phk = sm + pl.oPhk; float* Pm = sm + pl.oPm;
  float* rowv = sm + pl.oRow;
  const int64_t bh = blockIdx.y;
  const Range rg = seg_range(g);
  const int64_t tsz = int64_t(pl.F) * (g.dv + 1);
  load_w(pl, w_of(g, w, bh), ws);
  load_table(pl, carries + (bh * g.nseg + blockIdx.x) * tsz, S);
  const float invT = 1.f / float(g.T);
  for (int64_t t0 = rg.begin; t0 < rg.end; t0 += TILE) {
    const int rows = int(rg.end - t0 < TILE ? rg.end - t0 : TILE);
    __syncthreads();
    load_rows2<Tin>(q + (bh * g.N + t0) * g.d, g.d, xq, pl.ldx, rowv + kScQ * TILE, k + (bh * g.N + t0) * g.d, g.d,
                    xk, pl.ldx, rowv + kScK * TILE, rows, g.normalize);
    load_v_ones<Tin>(v + (bh * g.N + t0) * g.dv, rows, g.dv, vs, pl.ldv);
    __syncthreads();
    tile_features_n(pl, 2, xq, rowv + kScQ * TILE, phq, nullptr, xk, rowv + kScK * TILE, phk, nullptr, ws, g.beta);
    if (nrm) {  // sketch rows (race_b200.h): the generic backward only uses the row norms
      for (int r = threadIdx.x; r < rows; r += NT) {
        const float sq = rowv[kScQ * TILE + r], sk = rowv[kScK * TILE + r];
        float* row = nrm + (bh * g.N + t0 + r) * 16;
        for (int j = 0; j < 16; ++j) row[j] = 0.f;
        row[7] = sq > 0.f ? sq * sq : 0.f;
        row[15] = sk > 0.f ? sk * sk : 0.f;
      }
    }
    __syncthreads();
    tile_gram(phq, pl.ldf, phk, pl.ldf, pl.F, Pm, pl.ldp, [rows](int r, int j) { return j <= r && j < rows; });
    __syncthreads();
    for (int r = threadIdx.x; r < TILE; r += NT) {
      float D = 0.f;
      for (int f = 0; f < pl.F; ++f) D = fmaf(phq[r * pl.ldf + f], S[f * pl.ldS + g.dv], D);
      for (int j = 0; j <= r; ++j) D += Pm[r * pl.ldp + j];
      rowv[kD * TILE + r] = D;
      if (r < rows) den[bh * g.N + t0 + r] = D * invT;
    }
    __syncthreads();
    {  // num = phi_q S_<c + tril(Pm) V, 2 (rows) x 2 (columns) per item (Pm is zero above its diagonal)
      const int cp = (g.dv + 1) / 2;
      for (int it = threadIdx.x; it < (TILE / 2) * cp; it += NT) {
        const int r0 = 2 * (it / cp), c0 = 2 * (it % cp);
        if (r0 >= rows) continue;
        const bool c1 = c0 + 1 < g.dv, r1 = r0 + 1 < rows;
        float a00 = 0.f, a01 = 0.f, a10 = 0.f, a11 = 0.f;
        for (int f = 0; f < pl.F; ++f) {
          const float p0 = phq[r0 * pl.ldf + f], p1 = phq[(r0 + 1) * pl.ldf + f];
          const float s0 = S[f * pl.ldS + c0], s1 = c1 ? S[f * pl.ldS + c0 + 1] : 0.f;
          a00 = fmaf(p0, s0, a00);
          a01 = fmaf(p0, s1, a01);
          a10 = fmaf(p1, s0, a10);
          a11 = fmaf(p1, s1, a11);
        }
        for (int j = 0; j <= r0 + 1 && j < TILE; ++j) {
          const float m0 = Pm[r0 * pl.ldp + j], m1 = Pm[(r0 + 1) * pl.ldp + j];
          const float v0 = vs[j * pl.ldv + c0], v1 = c1 ? vs[j * pl.ldv + c0 + 1] : 0.f;
          a00 = fmaf(m0, v0, a00);
          a01 = fmaf(m0, v1, a01);
          a10 = fmaf(m1, v0, a10);
          a11 = fmaf(m1, v1, a11);
        }
        const float D0 = rowv[kD * TILE + r0], D1 = rowv[kD * TILE + r0 + 1];
        const bool z0 = D0 * invT <= kDegenerateDenEps, z1 = D1 * invT <= kDegenerateDenEps;
        Tin* o0 = o + (bh * g.N + t0 + r0) * g.dv + c0;
        o0[0] = from_f32<Tin>(z0 ? 0.f : a00 / D0);
        if (c1) o0[1] = from_f32<Tin>(z0 ? 0.f : a01 / D0);
        if (r1) {
          o0[g.dv] = from_f32<Tin>(z1 ? 0.f : a10 / D1);
          if (c1) o0[g.dv + 1] = from_f32<Tin>(z1 ? 0.f : a11 / D1);
        }
      }
    }
    __syncthreads();
    owner_accumulate(pl, S, phk, vs);  // S_<next tile
  }
}

// Non-causal backward, query side.
template <typename Tin>
__global__ void __launch_bounds__(NT, 2) k_bwd_q(Geo g, const Tin* __restrict__ q, const Tin* __restrict__ d_o,
                                              const float* __restrict__ w,
                                              const float* __restrict__ tables, Tin* __restrict__ dq,
                                              float* __restrict__ dpart) {
  const Plan pl(g, kW | kS | kAcc | kXq | kDx | kG | kPhq | kDph | kY | kU | kDproj);
  float* sm = reinterpret_cast<float*>(smem_f4);
  float* ws = sm + pl.oW; float* S = sm + pl.oS; float* acc = sm + pl.oAcc; float* xq = sm + pl.oXq;
  float* dx = sm + pl.oDx; float* gs = sm + pl.oG; float* phq = sm + pl.oPhq; float* dph = sm + pl.oDph;
  float* ys = sm + pl.oY; float* us = sm + pl.oU; float* dproj = sm + pl.oDproj; float* rowv = sm + pl.oRow;
  const int64_t bh = blockIdx.y;
  const Range rg = seg_range(g);
  const int64_t tsz = int64_t(pl.F) * (g.dv + 1);
  load_w(pl, w_of(g, w, bh), ws);
  load_table(pl, tables + bh * tsz, S);
  load_table(pl, nullptr, acc);
  const float invT = 1.f / float(g.T);
  for (int64_t t0 = rg.begin; t0 < rg.end; t0 += TILE) {
    const int rows = int(rg.end - t0 < TILE ? rg.end - t0 : TILE);
    __syncthreads();
    load_rows<Tin>(q + (bh * g.N + t0) * g.d, rows, g.d, xq, pl.ldx, rowv + kScQ * TILE, g.normalize);
    load_rows<Tin>(d_o + (bh * g.N + t0) * g.dv, rows, g.dv, gs, pl.ldv, nullptr, false);
    __syncthreads();
    tile_features(pl, xq, rowv + kScQ * TILE, ws, g.beta, phq, us);
    // y[t][f] = S_v[f] . dO_t
    gram2(gs, pl.ldv, TILE, S, pl.ldS, pl.F, g.dv, ys, pl.ldf, KeepAll());  // y[t][f] = S_v[f] . dO_t
    __syncthreads();
    for (int r = threadIdx.x; r < TILE; r += NT) {
      float D = 0.f, num = 0.f;
      for (int f = 0; f < pl.F; ++f) {
        D = fmaf(phq[r * pl.ldf + f], S[f * pl.ldS + g.dv], D);
        num = fmaf(phq[r * pl.ldf + f], ys[r * pl.ldf + f], num);
      }
      const bool live = r < rows && D * invT > kDegenerateDenEps;
      float rD = live ? 1.f / D : 0.f;
      float gD = live ? -num * rD * rD : 0.f;  // -(dO . O) / D
      if (g.ext_rden) {  // table group: normalisers of the whole estimator
        const int64_t i = bh * ((g.N + 3) & ~int64_t(3)) + t0 + r;
        rD = r < rows ? g.ext_rden[i] : 0.f;
        gD = r < rows ? g.ext_gden[i] : 0.f;
      }
      rowv[kRD * TILE + r] = rD;
      rowv[kGD * TILE + r] = gD;
    }
    __syncthreads();
    for (int it = threadIdx.x; it < TILE * pl.F; it += NT) {
      const int r = it / pl.F, f = it % pl.F;
      dph[r * pl.ldf + f] = ys[r * pl.ldf + f] * rowv[kRD * TILE + r] + rowv[kGD * TILE + r] * S[f * pl.ldS + g.dv];
    }
    for (int it = threadIdx.x; it < TILE * (g.dv + 1); it += NT) {
      const int r = it / (g.dv + 1), c = it % (g.dv + 1);
      gs[r * pl.ldv + c] = c < g.dv ? gs[r * pl.ldv + c] * rowv[kRD * TILE + r] : rowv[kGD * TILE + r];
    }
    __syncthreads();
    tile_feature_vjp<Tin>(pl, xq, rowv + kScQ * TILE, ws, g.beta, phq, us, dph, dproj, dx,
                          rowv + kDot * TILE, g.normalize, rows, dq + (bh * g.N + t0) * g.d);
    owner_accumulate(pl, acc, phq, gs);
  }
  __syncthreads();
  store_table(pl, acc, dpart + (bh * g.nseg + blockIdx.x) * tsz);
}

// Non-causal backward, key side given global dS.
template <typename Tin>
__global__ void __launch_bounds__(NT) k_bwd_k(Geo g, const Tin* __restrict__ k, const Tin* __restrict__ v,
                                              const float* __restrict__ w,
                                              const float* __restrict__ dtables, Tin* __restrict__ dk,
                                              Tin* __restrict__ dvo) {
  const Plan pl(g, kW | kS | kXk | kDx | kV | kPhk | kDph | kU | kDproj);
  float* sm = reinterpret_cast<float*>(smem_f4);
  float* ws = sm + pl.oW; float* dS = sm + pl.oS; float* xk = sm + pl.oXk; float* dx = sm + pl.oDx;
  float* vs = sm + pl.oV; float* phk = sm + pl.oPhk; float* dph = sm + pl.oDph; float* us = sm + pl.oU;
  float* dproj = sm + pl.oDproj; float* rowv = sm + pl.oRow;
  const int64_t bh = blockIdx.y;
  const Range rg = seg_range(g);
  load_w(pl, w_of(g, w, bh), ws);
  load_table(pl, dtables + bh * int64_t(pl.F) * (g.dv + 1), dS);
  for (int64_t t0 = rg.begin; t0 < rg.end; t0 += TILE) {
    const int rows = int(rg.end - t0 < TILE ? rg.end - t0 : TILE);
    __syncthreads();
    load_rows<Tin>(k + (bh * g.N + t0) * g.d, rows, g.d, xk, pl.ldx, rowv + kScK * TILE, g.normalize);
    load_v_ones<Tin>(v + (bh * g.N + t0) * g.dv, rows, g.dv, vs, pl.ldv);
    __syncthreads();
    tile_features(pl, xk, rowv + kScK * TILE, ws, g.beta, phk, us);
    __syncthreads();
    gram2(vs, pl.ldv, TILE, dS, pl.ldS, pl.F, g.dv + 1, dph, pl.ldf, KeepAll());  // z[t][f] = [V|1]_t . dS[f]
    {  // dV = Phi_k dS_v, 2 (rows) x 2 (columns) per item
      const int cp = (g.dv + 1) / 2;
      for (int it = threadIdx.x; it < (TILE / 2) * cp; it += NT) {
        const int r0 = 2 * (it / cp), c0 = 2 * (it % cp);
        if (r0 >= rows) continue;
        const bool c1 = c0 + 1 < g.dv, r1 = r0 + 1 < rows;
        float a00 = 0.f, a01 = 0.f, a10 = 0.f, a11 = 0.f;
        for (int f = 0; f < pl.F; ++f) {
          const float p0 = phk[r0 * pl.ldf + f], p1 = phk[(r0 + 1) * pl.ldf + f];
          const float d0 = dS[f * pl.ldS + c0], d1 = c1 ? dS[f * pl.ldS + c0 + 1] : 0.f;
          a00 = fmaf(p0, d0, a00);
          a01 = fmaf(p0, d1, a01);
          a10 = fmaf(p1, d0, a10);
          a11 = fmaf(p1, d1, a11);
        }
        Tin* o0 = dvo + (bh * g.N + t0 + r0) * g.dv + c0;
        o0[0] = from_f32<Tin>(a00);
        if (c1) o0[1] = from_f32<Tin>(a01);
        if (r1) {
          o0[g.dv] = from_f32<Tin>(a10);
          if (c1) o0[g.dv + 1] = from_f32<Tin>(a11);
        }
      }
    }
    __syncthreads();
    tile_feature_vjp<Tin>(pl, xk, rowv + kScK * TILE, ws, g.beta, phk, us, dph, dproj, dx,
                          rowv + kDot * TILE, g.normalize, rows, dk + (bh * g.N + t0) * g.d);
  }
}

// Causal backward, forward scan: dq, per-token rden / gden, per-segment dS.
template <typename Tin>
__global__ void __launch_bounds__(NT, 2) k_bwd_causal_q(Geo g, const Tin* __restrict__ q,
                                                     const Tin* __restrict__ k, const Tin* __restrict__ v,
                                                     const Tin* __restrict__ d_o, const float* __restrict__ w,
                                                     const float* __restrict__ carries, Tin* __restrict__ dq,
                                                     float* __restrict__ rden, float* __restrict__ gden,
                                                     float* __restrict__ dpart) {
  const Plan pl(g, kW | kS | kAcc | kXq | kXk | kDx | kV | kG | kPhq | kPhk | kDph | kY | kU | kDproj | kPm | kEm);
  float* sm = reinterpret_cast<float*>(smem_f4);
  float* ws = sm + pl.oW; float* S = sm + pl.oS; float* acc = sm + pl.oAcc; float* xq = sm + pl.oXq;
  float* xk = sm + pl.oXk; float* dx = sm + pl.oDx; float* vs = sm + pl.oV; float* gs = sm + pl.oG;
  float* phq = sm + pl.oPhq; float* phk = sm + pl.oPhk; float* dph = sm + pl.oDph; float* ys = sm + pl.oY;
  float* us = sm + pl.oU; float* dproj = sm + pl.oDproj; float* Pm = sm + pl.oPm; float* Em = sm + pl.oEm;
  float* rowv = sm + pl.oRow;
  const int64_t bh = blockIdx.y;
  const Range rg = seg_range(g);
  const int64_t tsz = int64_t(pl.F) * (g.dv + 1);
  load_w(pl, w_of(g, w, bh), ws);
  load_table(pl, carries + (bh * g.nseg + blockIdx.x) * tsz, S);
  load_table(pl, nullptr, acc);
  const float invT = 1.f / float(g.T);
  for (int64_t t0 = rg.begin; t0 < rg.end; t0 += TILE) {
    const int rows = int(rg.end - t0 < TILE ? rg.end - t0 : TILE);
    __syncthreads();
    load_rows<Tin>(q + (bh * g.N + t0) * g.d, rows, g.d, xq, pl.ldx, rowv + kScQ * TILE, g.normalize);
    load_rows<Tin>(k + (bh * g.N + t0) * g.d, rows, g.d, xk, pl.ldx, rowv + kScK * TILE, g.normalize);
    load_v_ones<Tin>(v + (bh * g.N + t0) * g.dv, rows, g.dv, vs, pl.ldv);
    load_rows<Tin>(d_o + (bh * g.N + t0) * g.dv, rows, g.dv, gs, pl.ldv, nullptr, false);
    __syncthreads();
    tile_features_n(pl, 2, xq, rowv + kScQ * TILE, phq, us, xk, rowv + kScK * TILE, phk, nullptr, ws, g.beta);
    __syncthreads();
    {
      auto keep = [rows](int r, int j) { return j <= r && j < rows; };
      tile_gram(phq, pl.ldf, phk, pl.ldf, pl.F, Pm, pl.ldp, keep);
      tile_gram(gs, pl.ldv, vs, pl.ldv, g.dv, Em, pl.ldp, keep);
    }
    gram2(gs, pl.ldv, TILE, S, pl.ldS, pl.F, g.dv, ys, pl.ldf, KeepAll());  // y[t][f] = S_v[f] . dO_t
    __syncthreads();
    for (int r = threadIdx.x; r < TILE; r += NT) {
      float D = 0.f, num = 0.f;
      for (int f = 0; f < pl.F; ++f) {
        D = fmaf(phq[r * pl.ldf + f], S[f * pl.ldS + g.dv], D);
        num = fmaf(phq[r * pl.ldf + f], ys[r * pl.ldf + f], num);
      }
      for (int j = 0; j <= r; ++j) {
        D += Pm[r * pl.ldp + j];
        num = fmaf(Pm[r * pl.ldp + j], Em[r * pl.ldp + j], num);
      }
      const bool live = r < rows && D * invT > kDegenerateDenEps;
      float rD = live ? 1.f / D : 0.f;
      float gD = live ? -num * rD * rD : 0.f;  // -(dO . O) / D
      const int64_t i = bh * ((g.N + 3) & ~int64_t(3)) + t0 + r;  // row pitch N rounded up to 4 (race_b200.h)
      if (g.ext_rden) {  // table group: normalisers of the whole estimator
        rD = r < rows ? g.ext_rden[i] : 0.f;
        gD = r < rows ? g.ext_gden[i] : 0.f;
      } else if (r < rows) {
        rden[i] = rD;
        gden[i] = gD;
      }
      rowv[kRD * TILE + r] = rD;
      rowv[kGD * TILE + r] = gD;
    }
    __syncthreads();
    for (int it = threadIdx.x; it < TILE * pl.F; it += NT) {
      const int r = it / pl.F, f = it % pl.F;
      const float rD = rowv[kRD * TILE + r], gD = rowv[kGD * TILE + r];
      float a = ys[r * pl.ldf + f] * rD + gD * S[f * pl.ldS + g.dv];
      const int jmax = r < rows ? r : rows - 1;
      for (int j = 0; j <= jmax; ++j) a = fmaf(fmaf(Em[r * pl.ldp + j], rD, gD), phk[j * pl.ldf + f], a);
      dph[r * pl.ldf + f] = a;
    }
    for (int it = threadIdx.x; it < TILE * (g.dv + 1); it += NT) {
      const int r = it / (g.dv + 1), c = it % (g.dv + 1);
      gs[r * pl.ldv + c] = c < g.dv ? gs[r * pl.ldv + c] * rowv[kRD * TILE + r] : rowv[kGD * TILE + r];
    }
    __syncthreads();
    tile_feature_vjp<Tin>(pl, xq, rowv + kScQ * TILE, ws, g.beta, phq, us, dph, dproj, dx,
                          rowv + kDot * TILE, g.normalize, rows, dq + (bh * g.N + t0) * g.d);
    owner_accumulate(pl, acc, phq, gs);
    owner_accumulate(pl, S, phk, vs);
  }
  __syncthreads();
  store_table(pl, acc, dpart + (bh * g.nseg + blockIdx.x) * tsz);
}

// Causal backward, reverse scan over one segment with suffix carry dS_>seg.
template <typename Tin>
__global__ void __launch_bounds__(NT, 2) k_bwd_causal_k(Geo g, const Tin* __restrict__ q,
                                                     const Tin* __restrict__ k, const Tin* __restrict__ v,
                                                     const Tin* __restrict__ d_o, const float* __restrict__ w,
                                                     const float* __restrict__ rden,
                                                     const float* __restrict__ gden,
                                                     const float* __restrict__ dcarries,
                                                     Tin* __restrict__ dk, Tin* __restrict__ dvo) {
  const Plan pl(g, kW | kS | kXq | kXk | kDx | kV | kG | kPhq | kPhk | kDph | kU | kDproj | kPm | kEm);
  float* sm = reinterpret_cast<float*>(smem_f4);
  float* ws = sm + pl.oW; float* dS = sm + pl.oS; float* xq = sm + pl.oXq; float* xk = sm + pl.oXk;
  float* dx = sm + pl.oDx; float* vs = sm + pl.oV; float* gs = sm + pl.oG; float* phq = sm + pl.oPhq;
  float* phk = sm + pl.oPhk; float* dph = sm + pl.oDph; float* us = sm + pl.oU; float* dproj = sm + pl.oDproj;
  float* PmT = sm + pl.oPm; float* EGT = sm + pl.oEm; float* rowv = sm + pl.oRow;
  const int64_t bh = blockIdx.y;
  const Range rg = seg_range(g);
  const int64_t tsz = int64_t(pl.F) * (g.dv + 1);
  load_w(pl, w_of(g, w, bh), ws);
  load_table(pl, dcarries + (bh * g.nseg + blockIdx.x) * tsz, dS);
  const int64_t ntile = (rg.end - rg.begin + TILE - 1) / TILE;
  for (int64_t ti = ntile - 1; ti >= 0; --ti) {
    const int64_t t0 = rg.begin + ti * TILE;
    const int rows = int(rg.end - t0 < TILE ? rg.end - t0 : TILE);
    __syncthreads();
    load_rows<Tin>(q + (bh * g.N + t0) * g.d, rows, g.d, xq, pl.ldx, rowv + kScQ * TILE, g.normalize);
    load_rows<Tin>(k + (bh * g.N + t0) * g.d, rows, g.d, xk, pl.ldx, rowv + kScK * TILE, g.normalize);
    load_v_ones<Tin>(v + (bh * g.N + t0) * g.dv, rows, g.dv, vs, pl.ldv);
    load_rows<Tin>(d_o + (bh * g.N + t0) * g.dv, rows, g.dv, gs, pl.ldv, nullptr, false);
    for (int r = threadIdx.x; r < TILE; r += NT) {
      rowv[kRD * TILE + r] = r < rows ? rden[bh * ((g.N + 3) & ~int64_t(3)) + t0 + r] : 0.f;
      rowv[kGD * TILE + r] = r < rows ? gden[bh * ((g.N + 3) & ~int64_t(3)) + t0 + r] : 0.f;
    }
    __syncthreads();
    tile_features_n(pl, 2, xq, rowv + kScQ * TILE, phq, nullptr, xk, rowv + kScK * TILE, phk, us, ws, g.beta);
    for (int it = threadIdx.x; it < TILE * (g.dv + 1); it += NT) {
      const int r = it / (g.dv + 1), c = it % (g.dv + 1);
      gs[r * pl.ldv + c] = c < g.dv ? gs[r * pl.ldv + c] * rowv[kRD * TILE + r] : rowv[kGD * TILE + r];
    }
    __syncthreads();
    {
      auto keep = [rows](int i, int t) { return t >= i && t < rows; };
      tile_gram(phk, pl.ldf, phq, pl.ldf, pl.F, PmT, pl.ldp, keep);
      tile_gram(vs, pl.ldv, gs, pl.ldv, g.dv + 1, EGT, pl.ldp, keep);
    }
    __syncthreads();
    gram2(vs, pl.ldv, TILE, dS, pl.ldS, pl.F, g.dv + 1, dph, pl.ldf, KeepAll());  // [V|1]_i . dS_>c[f]
    __syncthreads();
    for (int it = threadIdx.x; it < TILE * pl.F; it += NT) {
      const int i = it / pl.F, f = it % pl.F;
      float a = dph[i * pl.ldf + f];
      for (int t = i; t < rows; ++t) a = fmaf(EGT[i * pl.ldp + t], phq[t * pl.ldf + f], a);
      dph[i * pl.ldf + f] = a;
    }
    {  // dV = Phi_k dS_>c,v + P~^T dO, 2 (rows) x 2 (columns) per item (P~^T is zero below its diagonal)
      const int cp = (g.dv + 1) / 2;
      for (int it = threadIdx.x; it < (TILE / 2) * cp; it += NT) {
        const int i0 = 2 * (it / cp), c0 = 2 * (it % cp);
        if (i0 >= rows) continue;
        const bool c1 = c0 + 1 < g.dv, i1 = i0 + 1 < rows;
        float a00 = 0.f, a01 = 0.f, a10 = 0.f, a11 = 0.f;
        for (int f = 0; f < pl.F; ++f) {
          const float p0 = phk[i0 * pl.ldf + f], p1 = phk[(i0 + 1) * pl.ldf + f];
          const float d0 = dS[f * pl.ldS + c0], d1 = c1 ? dS[f * pl.ldS + c0 + 1] : 0.f;
          a00 = fmaf(p0, d0, a00);
          a01 = fmaf(p0, d1, a01);
          a10 = fmaf(p1, d0, a10);
          a11 = fmaf(p1, d1, a11);
        }
        for (int t = i0; t < rows; ++t) {
          const float m0 = PmT[i0 * pl.ldp + t], m1 = PmT[(i0 + 1) * pl.ldp + t];
          const float g0 = gs[t * pl.ldv + c0], g1 = c1 ? gs[t * pl.ldv + c0 + 1] : 0.f;
          a00 = fmaf(m0, g0, a00);
          a01 = fmaf(m0, g1, a01);
          a10 = fmaf(m1, g0, a10);
          a11 = fmaf(m1, g1, a11);
        }
        Tin* o0 = dvo + (bh * g.N + t0 + i0) * g.dv + c0;
        o0[0] = from_f32<Tin>(a00);
        if (c1) o0[1] = from_f32<Tin>(a01);
        if (i1) {
          o0[g.dv] = from_f32<Tin>(a10);
          if (c1) o0[g.dv + 1] = from_f32<Tin>(a11);
        }
      }
    }
    __syncthreads();
    tile_feature_vjp<Tin>(pl, xk, rowv + kScK * TILE, ws, g.beta, phk, us, dph, dproj, dx,
                          rowv + kDot * TILE, g.normalize, rows, dk + (bh * g.N + t0) * g.d);
    owner_accumulate(pl, dS, phq, gs);
  }
}

// Fixed-order segment reduction (see race_combine in race_b200.h).  Block =
// 32 table elements x CG segment groups: each thread sums its group's
// segments in order, the group totals are combined in group order through
// shared memory, then each thread emits its group's prefixes/suffixes.  The
// association is fixed by (nseg, CG), so results are bit-reproducible.
constexpr int CG = 16;
constexpr int CPER = 16;  // segments per group held in registers (nseg <= CG * CPER); longer groups loop
__global__ void __launch_bounds__(32 * CG) k_combine(int64_t BH, int64_t nseg, int64_t E, int mode,
                                                     const float* __restrict__ part, const float* __restrict__ carry,
                                                     float* __restrict__ out, int pad) {
  __shared__ float gs[CG][33];
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched with PDL after the partials' kernel
  if (pad > 0 && blockIdx.x == 0 && blockIdx.y == 0 && int(threadIdx.x) < pad) out[BH * nseg * E + threadIdx.x] = 0.f;
  const int lx = threadIdx.x & 31, gy = threadIdx.x >> 5;
  const int64_t e = int64_t(blockIdx.x) * 32 + lx;
  const int64_t bh = blockIdx.y;
  const int64_t per = (nseg + CG - 1) / CG;
  const int64_t s0 = gy * per, s1 = s0 + per < nseg ? s0 + per : nseg;
  const bool ok = e < E;
  const float* p = part + bh * nseg * E + e;
  const bool regs = per <= CPER;
  float x[CPER];  // this group's segment values, all loads in flight at once
  float sum = 0.f;
  if (regs) {
#pragma unroll
    for (int j = 0; j < CPER; ++j) x[j] = (ok && s0 + j < s1) ? p[(s0 + j) * E] : 0.f;
#pragma unroll
    for (int j = 0; j < CPER; ++j) sum += x[j];
  } else if (ok) {
    for (int64_t i = s0; i < s1; ++i) sum += p[i * E];
  }
  gs[gy][lx] = sum;
  __syncthreads();
  const float c = (ok && carry) ? carry[bh * E + e] : 0.f;
  if (mode == 0) {
    if (gy == 0 && ok) {
      float tot = c;
      for (int g = 0; g < CG; ++g) tot += gs[g][lx];
      out[bh * E + e] = tot;
    }
    return;
  }
  if (!ok) return;
  float base = c;
  if (mode == 1) {
    for (int g = 0; g < gy; ++g) base += gs[g][lx];
    if (regs) {
#pragma unroll
      for (int j = 0; j < CPER; ++j)
        if (s0 + j < s1) {
          out[(bh * nseg + s0 + j) * E + e] = base;
          base += x[j];
        }
    } else {
      for (int64_t i = s0; i < s1; ++i) {
        out[(bh * nseg + i) * E + e] = base;
        base += p[i * E];
      }
    }
  } else {
    for (int g = CG - 1; g > gy; --g) base += gs[g][lx];
    if (regs) {
#pragma unroll
      for (int j = CPER - 1; j >= 0; --j)
        if (s0 + j < s1) {
          out[(bh * nseg + s0 + j) * E + e] = base;
          base += x[j];
        }
    } else {
      for (int64_t i = s1 - 1; i >= s0; --i) {
        out[(bh * nseg + i) * E + e] = base;
        base += p[i * E];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
template <typename K>
static cudaError_t prep(K kernel, size_t smem) {
  // always set (also below 48 KB): resolves the kernel handle before the first launch
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
}

#define RACE_LAUNCH(KER, NEED, ...)                                                      \
  do {                                                                                   \
    const size_t smem = Plan(g, NEED).bytes();                                           \
    if (smem > kMaxSmem) return cudaErrorInvalidConfiguration;                           \
    cudaError_t e_ = prep(KER, smem);                                                    \
    if (e_ != cudaSuccess) return e_;                                                    \
    KER<<<dim3(unsigned(g.nseg), unsigned(g.BH)), NT, smem, st>>>(g, __VA_ARGS__);       \
    note_launch();                                                                       \
    return cudaGetLastError();                                                           \
  } while (0)

constexpr size_t kMaxSmem = 227 * 1024;

template <typename Tin>
struct Launch {
  static cudaError_t aggregate(const Geo& g, const void* k, const void* v, const float* w, float* part, cudaStream_t st) {
    RACE_LAUNCH(k_aggregate<Tin>, kW | kAcc | kXk | kV | kPhk, (const Tin*)k, (const Tin*)v, w, part);
  }
  static cudaError_t readout(const Geo& g, const void* q, const float* w, const float* tab, void* o, float* den,
                             cudaStream_t st) {
    RACE_LAUNCH(k_readout<Tin>, kW | kS | kXq | kPhq, (const Tin*)q, w, tab, (Tin*)o, den);
  }
  static cudaError_t causal_fwd(const Geo& g, const void* q, const void* k, const void* v, const float* w,
                                const float* car, void* o, float* den, float* nrm, cudaStream_t st) {
    RACE_LAUNCH(k_causal_fwd<Tin>, kW | kS | kXq | kXk | kV | kPhq | kPhk | kPm, (const Tin*)q, (const Tin*)k,
                (const Tin*)v, w, car, (Tin*)o, den, nrm);
  }
  static cudaError_t bwd_q(const Geo& g, const void* q, const void* d_o, const float* w, const float* tab, void* dq,
                           float* dpart, cudaStream_t st) {
    RACE_LAUNCH(k_bwd_q<Tin>, kW | kS | kAcc | kXq | kDx | kG | kPhq | kDph | kY | kU | kDproj, (const Tin*)q,
                (const Tin*)d_o, w, tab, (Tin*)dq, dpart);
  }
  static cudaError_t bwd_k(const Geo& g, const void* k, const void* v, const float* w, const float* dtab, void* dk,
                           void* dv, cudaStream_t st) {
    RACE_LAUNCH(k_bwd_k<Tin>, kW | kS | kXk | kDx | kV | kPhk | kDph | kU | kDproj, (const Tin*)k, (const Tin*)v, w,
                dtab, (Tin*)dk, (Tin*)dv);
  }
  static cudaError_t bwd_causal_q(const Geo& g, const void* q, const void* k, const void* v, const void* d_o,
                                  const float* w, const float* car, void* dq, float* rden, float* gden, float* dpart,
                                  cudaStream_t st) {
    RACE_LAUNCH(k_bwd_causal_q<Tin>,
                kW | kS | kAcc | kXq | kXk | kDx | kV | kG | kPhq | kPhk | kDph | kY | kU | kDproj | kPm | kEm,
                (const Tin*)q, (const Tin*)k, (const Tin*)v, (const Tin*)d_o, w, car, (Tin*)dq, rden, gden, dpart);
  }
  static cudaError_t bwd_causal_k(const Geo& g, const void* q, const void* k, const void* v, const void* d_o,
                                  const float* w, const float* rden, const float* gden, const float* dcar, void* dk,
                                  void* dv, cudaStream_t st) {
    RACE_LAUNCH(k_bwd_causal_k<Tin>,
                kW | kS | kXq | kXk | kDx | kV | kG | kPhq | kPhk | kDph | kU | kDproj | kPm | kEm, (const Tin*)q,
                (const Tin*)k, (const Tin*)v, (const Tin*)d_o, w, rden, gden, dcar, (Tin*)dk, (Tin*)dv);
  }
};

}  // namespace simt

// ---- dispatch used by race_abi.cu ------------------------------------------
size_t simt_max_smem(const Geo& g) {
  using namespace simt;
  return Plan(g, kW | kS | kAcc | kXq | kXk | kDx | kV | kG | kPhq | kPhk | kDph | kY | kU | kDproj | kPm | kEm).bytes();
}

#define RACE_DISPATCH(FN, ...) \
  (g.dtype == 1 ? simt::Launch<__nv_bfloat16>::FN(__VA_ARGS__) : simt::Launch<float>::FN(__VA_ARGS__))

cudaError_t simt_aggregate(const Geo& g, const void* k, const void* v, const float* w, float* part, cudaStream_t st) {
  return RACE_DISPATCH(aggregate, g, k, v, w, part, st);
}
cudaError_t simt_readout(const Geo& g, const void* q, const float* w, const float* tab, void* o, float* den,
                         cudaStream_t st) {
  return RACE_DISPATCH(readout, g, q, w, tab, o, den, st);
}
cudaError_t simt_causal_fwd(const Geo& g, const void* q, const void* k, const void* v, const float* w,
                            const float* car, void* o, float* den, float* nrm, cudaStream_t st) {
  return RACE_DISPATCH(causal_fwd, g, q, k, v, w, car, o, den, nrm, st);
}
cudaError_t simt_bwd_q(const Geo& g, const void* q, const void* d_o, const float* w, const float* tab, void* dq,
                       float* dpart, cudaStream_t st) {
  return RACE_DISPATCH(bwd_q, g, q, d_o, w, tab, dq, dpart, st);
}
cudaError_t simt_bwd_k(const Geo& g, const void* k, const void* v, const float* w, const float* dtab, void* dk,
                       void* dv, cudaStream_t st) {
  return RACE_DISPATCH(bwd_k, g, k, v, w, dtab, dk, dv, st);
}
cudaError_t simt_bwd_causal_q(const Geo& g, const void* q, const void* k, const void* v, const void* d_o,
                              const float* w, const float* car, void* dq, float* rden, float* gden, float* dpart,
                              cudaStream_t st) {
  return RACE_DISPATCH(bwd_causal_q, g, q, k, v, d_o, w, car, dq, rden, gden, dpart, st);
}
cudaError_t simt_bwd_causal_k(const Geo& g, const void* q, const void* k, const void* v, const void* d_o,
                              const float* w, const float* rden, const float* gden, const float* dcar, void* dk,
                              void* dv, cudaStream_t st) {
  return RACE_DISPATCH(bwd_causal_k, g, q, k, v, d_o, w, rden, gden, dcar, dk, dv, st);
}
cudaError_t combine(const Geo& g, int mode, const float* part, const float* carry, float* out, cudaStream_t st,
                    int pad) {
  const int64_t E = (int64_t(g.T) << pass_corner_bits(g)) * (g.dv + 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned((E + 31) / 32), unsigned(g.BH));
  cfg.blockDim = dim3(32 * simt::CG);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];  // programmatic dependent launch (see tcfast::launch_nt)
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool pdl = [] {
    const char* e = getenv("RACE_NO_PDL");
    return !(e && e[0] == '1');
  }();
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, simt::k_combine, g.BH, g.nseg, E, mode, part, carry, out, pad);
  note_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace race
