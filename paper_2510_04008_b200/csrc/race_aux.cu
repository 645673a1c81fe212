// race_aux.cu -- the validation-side entry points declared in include/race_aux.h:
// soft / hard hashing, the averaged sketch kernel, the hard-bucket estimator
// and exact angular attention (forward + VJP).
//
// These are the reference's theory / accuracy-reference functions
// (ra/sketch.py, ra/forward.py:167-212, ra/theory.py:205-241, ra/exact.py:116-218)
// moved onto the GPU.  They are quadratic or small by construction and the
// reference runs them in float64, so every kernel here computes in fp64
// (B200 keeps full-rate-class FP64 on the CUDA cores) and the results agree
// with the reference to ~1e-12 rather than to a bf16 tolerance.  None of them
// is on the RACE hot path; that is race_tc*.cu.
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>
#include <type_traits>

#include "race_aux.h"
#include "race_b200.h"
#include "race_internal.h"

namespace race {
int report(int code, const char* msg);              // race_abi.cu (thread-local error text)
int report_cuda(cudaError_t e, const char* where);  // race_abi.cu
}  // namespace race

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kDegenerate = 1e-30;  // DEGENERATE_DEN_EPS (ra/core.py:19)
constexpr double kZeroRow = 1e-12;     // ZERO_ROW_EPS (ra/core.py:15)

__device__ __forceinline__ double ld(const float* p, int64_t i) { return double(p[i]); }
__device__ __forceinline__ double ld(const double* p, int64_t i) { return p[i]; }
__device__ __forceinline__ double ld(const __nv_bfloat16* p, int64_t i) { return double(__bfloat162float(p[i])); }

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// logistic function, numerically stable on both signs (ra/sketch.py:77-84)
__device__ __forceinline__ double sigmoid(double z) {
  if (z >= 0) return 1.0 / (1.0 + exp(-z));
  const double e = exp(z);
  return e / (1.0 + e);
}

// ---------------------------------------------------------------------------
// soft_features for every table at once: one warp per row.
//   u_j = tanh(x^ . w_j), phi_{tau, r} = prod_t sigmoid(+-2 beta u_{tau P + t})
// (bit t of r: 0 -> +, 1 -> -).  This is the factored form of the reference's
// corner softmax (ra/sketch.py:111-129); both agree to ~1e-15 in fp64.
// ---------------------------------------------------------------------------
constexpr int kMaxTP = 256;

template <typename Tin>
__global__ void k_soft_features(const Tin* __restrict__ x, int64_t n, int d, const double* __restrict__ w, int P,
                                int T, double beta, int normalize, double* __restrict__ phi) {
  __shared__ double zs[8][kMaxTP];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * 8 + wid;
  if (row >= n) return;
  const Tin* xr = x + row * d;
  double ss = 0;
  for (int e = lane; e < d; e += 32) {
    const double xe = ld(xr, e);
    ss += xe * xe;
  }
  ss = warp_sum(ss);
  const double nrm = sqrt(ss);
  const double scl = (normalize && nrm >= kZeroRow) ? nrm : 1.0;  // row_normalize divides (ra/core.py:122-123)
  const int TP = T * P;
  for (int j = 0; j < TP; ++j) {
    const double* wj = w + int64_t(j) * d;
    double s = 0;
    for (int e = lane; e < d; e += 32) s += (ld(xr, e) / scl) * wj[e];
    s = warp_sum(s);
    if (lane == 0) zs[wid][j] = 2.0 * beta * tanh(s);
  }
  __syncwarp();
  const int R = 1 << P;
  double* out = phi + row * int64_t(T) * R;
  for (int tau = 0; tau < T; ++tau)
    for (int r = lane; r < R; r += 32) {
      double f = 1.0;
      for (int t = 0; t < P; ++t) {
        const double z = zs[wid][tau * P + t];
        f *= sigmoid(((r >> t) & 1) ? -z : z);
      }
      out[int64_t(tau) * R + r] = f;
    }
}

// hard_hash (ra/sketch.py:143-149): bit t of the code = (x . w_t < 0); codes [T, n]
template <typename Tin>
__global__ void k_hard_hash(const Tin* __restrict__ x, int64_t n, int d, const double* __restrict__ w, int P, int T,
                            int normalize, int32_t* __restrict__ codes) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * 8 + wid;
  if (row >= n) return;
  const Tin* xr = x + row * d;
  double scl = 1.0;
  if (normalize) {  // prepared_qk normalises first (ra/theory.py:210); a positive scale, kept for parity
    double ss = 0;
    for (int e = lane; e < d; e += 32) {
      const double xe = ld(xr, e);
      ss += xe * xe;
    }
    const double nrm = sqrt(warp_sum(ss));
    scl = nrm >= kZeroRow ? nrm : 1.0;
  }
  for (int tau = 0; tau < T; ++tau) {
    int code = 0;
    for (int t = 0; t < P; ++t) {
      const double* wj = w + int64_t(tau * P + t) * d;
      double s = 0;
      for (int e = lane; e < d; e += 32) s += (ld(xr, e) / scl) * wj[e];
      s = warp_sum(s);
      code |= (s < 0) << t;
    }
    if (lane == 0) codes[int64_t(tau) * n + row] = code;
  }
}

// race_kernel's contraction (ra/forward.py:195-202): out = scale * phi_q phi_k^T
__global__ void k_feature_gram(int64_t n, int64_t m, int f, const double* __restrict__ pq,
                               const double* __restrict__ pk, double scale, double* __restrict__ out) {
  __shared__ double a[16][17], b[16][17];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i = int64_t(blockIdx.y) * 16 + ty, j = int64_t(blockIdx.x) * 16 + tx;
  double s = 0;
  for (int c0 = 0; c0 < f; c0 += 16) {
    const int64_t ib = int64_t(blockIdx.y) * 16 + ty, jb = int64_t(blockIdx.x) * 16 + ty;
    a[ty][tx] = (ib < n && c0 + tx < f) ? pq[ib * f + c0 + tx] : 0.0;
    b[ty][tx] = (jb < m && c0 + tx < f) ? pk[jb * f + c0 + tx] : 0.0;
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 16; ++c) s += a[ty][c] * b[tx][c];
    __syncthreads();
  }
  if (i < n && j < m) out[i * m + j] = s * scale;
}

// hard-bucket statistics a[tau][r] (counts), b[tau][r][c] (value sums), fp64
// (ra/theory.py:215-219: bincount / np.add.at in float64)
template <typename Tin>
__global__ void k_hard_aggregate(int64_t n, int dv, const int32_t* __restrict__ codes_k, const Tin* __restrict__ v,
                                 int R, int T, double* __restrict__ tab) {
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  for (int tau = 0; tau < T; ++tau) {
    const int code = codes_k[int64_t(tau) * n + row];
    double* t = tab + (int64_t(tau) * R + code) * (dv + 1);
    for (int c = lane; c < dv; c += 32) atomicAdd(t + c, ld(v, row * dv + c));
    if (lane == 0) atomicAdd(t + dv, 1.0);
  }
}

// num_i = sum_tau b[tau][hq], den_i = sum_tau a[tau][hq], both / T; o = num / den (ra/theory.py:220-227)
__global__ void k_hard_readout(int64_t n, int dv, const int32_t* __restrict__ codes_q, int R, int T,
                               const double* __restrict__ tab, double* __restrict__ o, double* __restrict__ den) {
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double scale = 1.0 / T;
  double dn = 0;
  for (int tau = 0; tau < T; ++tau) dn += tab[(int64_t(tau) * R + codes_q[int64_t(tau) * n + row]) * (dv + 1) + dv];
  dn *= scale;
  const bool deg = dn <= kDegenerate;
  for (int c = lane; c < dv; c += 32) {
    double s = 0;
    for (int tau = 0; tau < T; ++tau) s += tab[(int64_t(tau) * R + codes_q[int64_t(tau) * n + row]) * (dv + 1) + c];
    s *= scale;
    o[row * dv + c] = deg ? 0.0 : s / dn;
  }
  if (lane == 0) den[row] = dn;
}

// ---------------------------------------------------------------------------
// Exact angular attention, fp64 tiles of TB rows x TB columns (256 threads):
// thread (r = tid / G, g = tid % G) owns row r of the tile and the columns
// g, g + G, ... of every row-vector accumulator (G = 256 / TB).
// ---------------------------------------------------------------------------
constexpr int kThreads = 256;
constexpr int kMaxCols = 16;  // per-thread accumulator columns: d, dv <= G * kMaxCols

__device__ __forceinline__ double sharpen(double base, int g) {  // base ** g for a positive integer g
  double r = 1.0, b = base;
  while (g) {
    if (g & 1) r *= b;
    b *= b;
    g >>= 1;
  }
  return r;
}

template <typename Tin>
__device__ __forceinline__ void load_rows(double* dst, int pitch, const Tin* src, int64_t row0, int64_t n, int cols,
                                          int rows, const double* scale) {
  for (int i = threadIdx.x; i < rows * cols; i += kThreads) {
    const int r = i / cols, c = i % cols;
    const int64_t gr = row0 + r;
    double x = gr < n ? ld(src, gr * cols + c) : 0.0;
    if (scale) x *= scale[r];
    dst[r * pitch + c] = x;
  }
}

// squared norms of TB rows -> 1/||x|| (scale) and ||x|| (norm)
template <typename Tin>
__device__ void row_norms(const Tin* src, int64_t row0, int64_t n, int cols, int rows, double* norm, double* inv) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = wid; r < rows; r += kThreads / 32) {
    double s = 0;
    const int64_t gr = row0 + r;
    if (gr < n)
      for (int c = lane; c < cols; c += 32) {
        const double x = ld(src, gr * cols + c);
        s += x * x;
      }
    s = warp_sum(s);
    if (lane == 0) {
      norm[r] = sqrt(s);
      if (inv) inv[r] = s > 0 ? 1.0 / sqrt(s) : 0.0;
    }
  }
}

// angular_kernel_matrix (ra/exact.py:116-125): S_ij = (1 - acos(clip(q.k / (|q||k|))) / pi) ** g
template <typename Tin>
__global__ void k_angular_matrix(const Tin* __restrict__ q, const Tin* __restrict__ k, int64_t n, int64_t m, int d,
                                 int g, double* __restrict__ out) {
  __shared__ double a[16][17], b[16][17];
  __shared__ double qn[16], kn[16];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i0 = int64_t(blockIdx.y) * 16, j0 = int64_t(blockIdx.x) * 16;
  double s = 0, sq = 0, sk = 0;
  for (int c0 = 0; c0 < d; c0 += 16) {
    const double qa = (i0 + ty < n && c0 + tx < d) ? ld(q, (i0 + ty) * d + c0 + tx) : 0.0;
    const double kb = (j0 + ty < m && c0 + tx < d) ? ld(k, (j0 + ty) * d + c0 + tx) : 0.0;
    a[ty][tx] = qa;
    b[ty][tx] = kb;
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 16; ++c) s += a[ty][c] * b[tx][c];
    if (tx == 0)
#pragma unroll
      for (int c = 0; c < 16; ++c) { sq += a[ty][c] * a[ty][c]; sk += b[ty][c] * b[ty][c]; }
    __syncthreads();
  }
  if (tx == 0) { qn[ty] = sqrt(sq); kn[ty] = sqrt(sk); }
  __syncthreads();
  const int64_t i = i0 + ty, j = j0 + tx;
  if (i < n && j < m) {
    const double rho = fmin(1.0, fmax(-1.0, s / (qn[ty] * kn[tx])));
    out[i * m + j] = sharpen(1.0 - acos(rho) / kPi, g);
  }
}

template <int TB>
struct Tiles {
  static constexpr int G = kThreads / TB;
};

// forward (ra/exact.py:128-166): O_i = sum_j s_ij v_j / sum_j s_ij, s_ij = sharpened angular similarity
template <typename Tin, int TB>
__global__ void __launch_bounds__(kThreads) k_angular_fwd(const Tin* __restrict__ q, const Tin* __restrict__ k,
                                                          const Tin* __restrict__ v, int64_t n, int d, int dv, int g,
                                                          int causal, double* __restrict__ o,
                                                          double* __restrict__ den_out) {
  constexpr int G = Tiles<TB>::G;
  extern __shared__ double sm[];
  const int dp = d + 1, vp = dv + 1;
  double* Qs = sm;                  // [TB][dp] raw q
  double* Ks = Qs + TB * dp;        // [TB][dp] raw k
  double* Vs = Ks + TB * dp;        // [TB][vp]
  double* S = Vs + TB * vp;         // [TB][TB + 1]
  double* qn = S + TB * (TB + 1);   // [TB]
  double* kn = qn + TB;             // [TB]
  const int tid = threadIdx.x, r = tid / G, gg = tid % G;
  const int64_t i0 = int64_t(blockIdx.x) * TB;
  load_rows(Qs, dp, q, i0, n, d, TB, nullptr);
  row_norms(q, i0, n, d, TB, qn, nullptr);
  double acc[kMaxCols];
#pragma unroll
  for (int u = 0; u < kMaxCols; ++u) acc[u] = 0;
  double den = 0;
  const int64_t jend = causal ? (i0 + TB < n ? i0 + TB : n) : n;
  for (int64_t j0 = 0; j0 < jend; j0 += TB) {
    __syncthreads();
    load_rows(Ks, dp, k, j0, n, d, TB, nullptr);
    load_rows(Vs, vp, v, j0, n, dv, TB, nullptr);
    row_norms(k, j0, n, d, TB, kn, nullptr);
    __syncthreads();
    for (int e = tid; e < TB * TB; e += kThreads) {
      const int rr = e / TB, cc = e % TB;
      const int64_t gi = i0 + rr, gj = j0 + cc;
      double s = 0;
      if (gi < n && gj < n && !(causal && gj > gi)) {
        double dot = 0;
        for (int c = 0; c < d; ++c) dot += Qs[rr * dp + c] * Ks[cc * dp + c];
        const double rho = fmin(1.0, fmax(-1.0, dot / (kn[cc] * qn[rr])));
        s = sharpen(1.0 - acos(rho) / kPi, g);
      }
      S[rr * (TB + 1) + cc] = s;
    }
    __syncthreads();
    for (int jj = 0; jj < TB; ++jj) {
      const double s = S[r * (TB + 1) + jj];
      den += s;
#pragma unroll
      for (int u = 0; u < kMaxCols; ++u) {
        const int c = gg + u * G;
        if (c < dv) acc[u] += s * Vs[jj * vp + c];
      }
    }
  }
  const int64_t gi = i0 + r;
  if (gi < n) {
    const bool deg = den <= kDegenerate;
#pragma unroll
    for (int u = 0; u < kMaxCols; ++u) {
      const int c = gg + u * G;
      if (c < dv) o[gi * dv + c] = deg ? 0.0 : acc[u] / den;
    }
    if (gg == 0) den_out[gi] = den;
  }
}

// d_rho_ij of angular_attention_vjp (ra/exact.py:194-207) for one pair
__device__ __forceinline__ void pair_grad(double rho_raw, double dov, double delta, double den, bool masked, int g,
                                          double* sims_over_den, double* d_rho) {
  const bool clipped = fabs(rho_raw) >= 1.0;
  const double rho = fmin(1.0, fmax(-1.0, rho_raw));
  const double base = 1.0 - acos(rho) / kPi;
  const bool deg = den <= kDegenerate;
  const double safe = deg ? 1.0 : den;
  const double sims = masked ? 0.0 : sharpen(base, g);
  *sims_over_den = sims / safe;
  double ds = (dov - delta) / safe;
  if (deg || masked) ds = 0.0;
  *d_rho = (clipped || ds == 0.0) ? 0.0 : ds * g * sharpen(base, g - 1) / (kPi * sqrt(1.0 - rho * rho));
}

// query side of the VJP: dq_i = unit-norm pullback of sum_j d_rho_ij kh_j (ra/exact.py:209-214)
template <typename Tin, int TB>
__global__ void __launch_bounds__(kThreads) k_angular_bwd_q(const Tin* __restrict__ q, const Tin* __restrict__ k,
                                                            const Tin* __restrict__ v, const Tin* __restrict__ d_o,
                                                            const double* __restrict__ o,
                                                            const double* __restrict__ den_in, int64_t n, int d, int dv,
                                                            int g, int causal, double* __restrict__ dq) {
  constexpr int G = Tiles<TB>::G;
  extern __shared__ double sm[];
  const int dp = d + 1, vp = dv + 1;
  double* Qh = sm;                 // [TB][dp] unit q rows
  double* Go = Qh + TB * dp;       // [TB][vp] dO rows
  double* Kh = Go + TB * vp;       // [TB][dp] unit k rows
  double* Vs = Kh + TB * dp;       // [TB][vp]
  double* Pm = Vs + TB * vp;       // [TB][TB + 1] d_rho
  double* qn = Pm + TB * (TB + 1);
  double* qi = qn + TB;
  double* kn = qi + TB;
  double* ki = kn + TB;
  double* dl = ki + TB;  // delta_i = dO_i . O_i
  double* dn = dl + TB;  // den_i
  const int tid = threadIdx.x, r = tid / G, gg = tid % G;
  const int64_t i0 = int64_t(blockIdx.x) * TB;
  row_norms(q, i0, n, d, TB, qn, qi);
  __syncthreads();
  load_rows(Qh, dp, q, i0, n, d, TB, qi);
  load_rows(Go, vp, d_o, i0, n, dv, TB, nullptr);
  {
    const int wid = tid >> 5, lane = tid & 31;
    for (int rr = wid; rr < TB; rr += kThreads / 32) {
      const int64_t gi = i0 + rr;
      double s = 0;
      if (gi < n)
        for (int c = lane; c < dv; c += 32) s += ld(d_o, gi * dv + c) * o[gi * dv + c];
      s = warp_sum(s);
      if (lane == 0) { dl[rr] = s; dn[rr] = gi < n ? den_in[gi] : 1.0; }
    }
  }
  double acc[kMaxCols];
#pragma unroll
  for (int u = 0; u < kMaxCols; ++u) acc[u] = 0;
  const int64_t jend = causal ? (i0 + TB < n ? i0 + TB : n) : n;
  for (int64_t j0 = 0; j0 < jend; j0 += TB) {
    __syncthreads();
    row_norms(k, j0, n, d, TB, kn, ki);
    __syncthreads();
    load_rows(Kh, dp, k, j0, n, d, TB, ki);
    load_rows(Vs, vp, v, j0, n, dv, TB, nullptr);
    __syncthreads();
    for (int e = tid; e < TB * TB; e += kThreads) {
      const int rr = e / TB, cc = e % TB;
      const int64_t gi = i0 + rr, gj = j0 + cc;
      double dr = 0;
      if (gi < n && gj < n) {
        double rho = 0, dov = 0;
        for (int c = 0; c < d; ++c) rho += Qh[rr * dp + c] * Kh[cc * dp + c];
        for (int c = 0; c < dv; ++c) dov += Go[rr * vp + c] * Vs[cc * vp + c];
        double w;
        pair_grad(rho, dov, dl[rr], dn[rr], causal && gj > gi, g, &w, &dr);
      }
      Pm[rr * (TB + 1) + cc] = dr;
    }
    __syncthreads();
    for (int jj = 0; jj < TB; ++jj) {
      const double p = Pm[r * (TB + 1) + jj];
#pragma unroll
      for (int u = 0; u < kMaxCols; ++u) {
        const int c = gg + u * G;
        if (c < d) acc[u] += p * Kh[jj * dp + c];
      }
    }
  }
  // pull back through x^ = x / |x|: (g - (g . x^) x^) / |x|   (G lanes of a row are adjacent)
  double dot = 0;
#pragma unroll
  for (int u = 0; u < kMaxCols; ++u) {
    const int c = gg + u * G;
    if (c < d) dot += acc[u] * Qh[r * dp + c];
  }
#pragma unroll
  for (int o2 = G / 2; o2 > 0; o2 >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o2);
  const int64_t gi = i0 + r;
  if (gi < n) {
#pragma unroll
    for (int u = 0; u < kMaxCols; ++u) {
      const int c = gg + u * G;
      if (c < d) dq[gi * d + c] = (acc[u] - dot * Qh[r * dp + c]) / qn[r];
    }
  }
}

// key side: dk_j = pullback of sum_i d_rho_ij qh_i, dv_j = sum_i (s_ij / den_i) dO_i
template <typename Tin, int TB>
__global__ void __launch_bounds__(kThreads) k_angular_bwd_k(const Tin* __restrict__ q, const Tin* __restrict__ k,
                                                            const Tin* __restrict__ v, const Tin* __restrict__ d_o,
                                                            const double* __restrict__ o,
                                                            const double* __restrict__ den_in, int64_t n, int d, int dv,
                                                            int g, int causal, double* __restrict__ dk,
                                                            double* __restrict__ dvout) {
  constexpr int G = Tiles<TB>::G;
  extern __shared__ double sm[];
  const int dp = d + 1, vp = dv + 1;
  double* Kh = sm;                  // [TB][dp] unit k rows (this CTA's keys)
  double* Vs = Kh + TB * dp;        // [TB][vp]
  double* Qh = Vs + TB * vp;        // [TB][dp] unit q rows (streamed)
  double* Go = Qh + TB * dp;        // [TB][vp] dO rows (streamed)
  double* Pm = Go + TB * vp;        // [TB keys][TB + 1] d_rho^T
  double* Wm = Pm + TB * (TB + 1);  // [TB keys][TB + 1] (s / den)^T
  double* kn = Wm + TB * (TB + 1);
  double* ki = kn + TB;
  double* qn = ki + TB;
  double* qi = qn + TB;
  double* dl = qi + TB;
  double* dn = dl + TB;
  const int tid = threadIdx.x, r = tid / G, gg = tid % G;
  const int64_t j0 = int64_t(blockIdx.x) * TB;
  row_norms(k, j0, n, d, TB, kn, ki);
  __syncthreads();
  load_rows(Kh, dp, k, j0, n, d, TB, ki);
  load_rows(Vs, vp, v, j0, n, dv, TB, nullptr);
  double ak[kMaxCols], av[kMaxCols];
#pragma unroll
  for (int u = 0; u < kMaxCols; ++u) ak[u] = av[u] = 0;
  const int64_t istart = causal ? j0 : 0;  // causal: only queries i >= j see key j
  for (int64_t i0 = istart - (istart % TB); i0 < n; i0 += TB) {
    __syncthreads();
    row_norms(q, i0, n, d, TB, qn, qi);
    {
      const int wid = tid >> 5, lane = tid & 31;
      for (int rr = wid; rr < TB; rr += kThreads / 32) {
        const int64_t gi = i0 + rr;
        double s = 0;
        if (gi < n)
          for (int c = lane; c < dv; c += 32) s += ld(d_o, gi * dv + c) * o[gi * dv + c];
        s = warp_sum(s);
        if (lane == 0) { dl[rr] = s; dn[rr] = gi < n ? den_in[gi] : 1.0; }
      }
    }
    __syncthreads();
    load_rows(Qh, dp, q, i0, n, d, TB, qi);
    load_rows(Go, vp, d_o, i0, n, dv, TB, nullptr);
    __syncthreads();
    for (int e = tid; e < TB * TB; e += kThreads) {
      const int cc = e / TB, rr = e % TB;  // cc: key of this CTA, rr: query of the streamed tile
      const int64_t gi = i0 + rr, gj = j0 + cc;
      double dr = 0, w = 0;
      if (gi < n && gj < n) {
        double rho = 0, dov = 0;
        for (int c = 0; c < d; ++c) rho += Qh[rr * dp + c] * Kh[cc * dp + c];
        for (int c = 0; c < dv; ++c) dov += Go[rr * vp + c] * Vs[cc * vp + c];
        pair_grad(rho, dov, dl[rr], dn[rr], causal && gj > gi, g, &w, &dr);
      }
      Pm[cc * (TB + 1) + rr] = dr;
      Wm[cc * (TB + 1) + rr] = w;
    }
    __syncthreads();
    for (int ii = 0; ii < TB; ++ii) {
      const double p = Pm[r * (TB + 1) + ii], w = Wm[r * (TB + 1) + ii];
#pragma unroll
      for (int u = 0; u < kMaxCols; ++u) {
        const int c = gg + u * G;
        if (c < d) ak[u] += p * Qh[ii * dp + c];
        if (c < dv) av[u] += w * Go[ii * vp + c];
      }
    }
  }
  double dot = 0;
#pragma unroll
  for (int u = 0; u < kMaxCols; ++u) {
    const int c = gg + u * G;
    if (c < d) dot += ak[u] * Kh[r * dp + c];
  }
#pragma unroll
  for (int o2 = G / 2; o2 > 0; o2 >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o2);
  const int64_t gj = j0 + r;
  if (gj < n) {
#pragma unroll
    for (int u = 0; u < kMaxCols; ++u) {
      const int c = gg + u * G;
      if (c < d) dk[gj * d + c] = (ak[u] - dot * Kh[r * dp + c]) / kn[r];
      if (c < dv) dvout[gj * dv + c] = av[u];
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int bad(const char* msg) { return race::report(RACE_EBADSHAPE, msg); }

int launched(const char* where) {
  race::note_launch();
  return race::report_cuda(cudaGetLastError(), where);
}

template <typename F>
int dispatch(int32_t dtype, F&& f) {
  switch (dtype) {
    case RACE_F32: return f(static_cast<const float*>(nullptr));
    case RACE_BF16: return f(static_cast<const __nv_bfloat16*>(nullptr));
    case RACE_F64: return f(static_cast<const double*>(nullptr));
    default: return race::report(RACE_EUNSUPPORTED, "aux: dtype must be RACE_F32, RACE_BF16 or RACE_F64");
  }
}

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

template <int TB>
size_t fwd_smem(int d, int dv) { return sizeof(double) * (size_t(TB) * (2 * (d + 1) + (dv + 1) + TB + 1) + 2 * TB); }
template <int TB>
size_t bwd_smem(int d, int dv) {
  return sizeof(double) * (size_t(TB) * (2 * (d + 1) + 2 * (dv + 1) + 2 * (TB + 1)) + 6 * TB);
}

// row_normalize (ra/core.py:114-123) and row_normalize_vjp (ra/core.py:126-139): one warp per
// row, fp64.  Rows with norm < ZERO_ROW_EPS pass through (forward) / pass the cotangent through (VJP).
template <typename Tin>
__global__ void k_row_normalize(const Tin* __restrict__ x, const Tin* __restrict__ g, int64_t n, int d,
                                double* __restrict__ out) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * 8 + wid;
  if (row >= n) return;
  const Tin* xr = x + row * d;
  double ss = 0;
  for (int e = lane; e < d; e += 32) {
    const double xe = ld(xr, e);
    ss += xe * xe;
  }
  const double nrm = sqrt(warp_sum(ss));
  const bool small = nrm < kZeroRow;
  const double scl = small ? 1.0 : nrm;
  double* orow = out + row * d;
  if (!g) {
    for (int e = lane; e < d; e += 32) orow[e] = ld(xr, e) / scl;
    return;
  }
  const Tin* gr = g + row * d;
  double radial = 0;
  for (int e = lane; e < d; e += 32) radial += ld(gr, e) * (ld(xr, e) / scl);
  radial = warp_sum(radial);
  for (int e = lane; e < d; e += 32)
    orow[e] = small ? ld(gr, e) : (ld(gr, e) - radial * (ld(xr, e) / scl)) / scl;
}

// tile height for (d, dv): 32 rows while every accumulator fits kMaxCols columns per thread, else 16
int pick_tb(int d, int dv) {
  const int mx = d > dv ? d : dv;
  if (mx <= Tiles<32>::G * kMaxCols) return 32;
  if (mx <= Tiles<16>::G * kMaxCols) return 16;
  return 0;
}

}  // namespace

extern "C" {

int race_aux_row_normalize(int32_t dtype, int64_t n, int32_t d, const void* x, const void* g, double* out,
                           void* stream) {
  if (n < 0 || d < 1) return bad("row_normalize: bad shape");
  if (n == 0) return RACE_OK;
  return dispatch(dtype, [&](auto tag) {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
    k_row_normalize<T><<<unsigned((n + 7) / 8), 256, 0, S(stream)>>>(static_cast<const T*>(x),
                                                                      static_cast<const T*>(g), n, d, out);
    return launched("row_normalize");
  });
}

int race_aux_soft_features(int32_t dtype, int64_t n, int32_t d, const void* x, const double* w, int32_t hyperplanes,
                           int32_t tables, double beta, int32_t normalize, double* phi, void* stream) {
  if (n < 0 || d < 1 || hyperplanes < 1 || hyperplanes > 20 || tables < 1) return bad("soft_features: bad shape");
  if (int64_t(hyperplanes) * tables > kMaxTP) return bad("soft_features: tables * hyperplanes > 256");
  if (!(beta > 0) || !std::isfinite(beta)) return bad("beta must be positive and finite");
  if (n == 0) return RACE_OK;
  return dispatch(dtype, [&](auto tag) {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
    k_soft_features<T><<<unsigned((n + 7) / 8), 256, 0, S(stream)>>>(static_cast<const T*>(x), n, d, w, hyperplanes,
                                                                      tables, beta, normalize, phi);
    return launched("soft_features");
  });
}

int race_aux_hard_hash(int32_t dtype, int64_t n, int32_t d, const void* x, const double* w, int32_t hyperplanes,
                       int32_t tables, int32_t normalize, int32_t* codes, void* stream) {
  if (n < 0 || d < 1 || hyperplanes < 1 || hyperplanes > 30 || tables < 1) return bad("hard_hash: bad shape");
  if (n == 0) return RACE_OK;
  return dispatch(dtype, [&](auto tag) {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
    k_hard_hash<T><<<unsigned((n + 7) / 8), 256, 0, S(stream)>>>(static_cast<const T*>(x), n, d, w, hyperplanes,
                                                                  tables, normalize, codes);
    return launched("hard_hash");
  });
}

int race_aux_feature_gram(int64_t n, int64_t m, int32_t f, const double* phi_q, const double* phi_k, double scale,
                          double* out, void* stream) {
  if (n < 0 || m < 0 || f < 1) return bad("feature_gram: bad shape");
  if (n == 0 || m == 0) return RACE_OK;
  if ((n + 15) / 16 > 65535) return bad("feature_gram: n too large");
  dim3 grid(unsigned((m + 15) / 16), unsigned((n + 15) / 16));
  k_feature_gram<<<grid, 256, 0, S(stream)>>>(n, m, f, phi_q, phi_k, scale, out);
  return launched("feature_gram");
}

size_t race_aux_hard_workspace_bytes(int32_t dv, int32_t hyperplanes, int32_t tables) {
  return sizeof(double) * (size_t(tables) << hyperplanes) * size_t(dv + 1);
}

int race_aux_hard_attention(int32_t dtype, int64_t n, int32_t dv, const int32_t* codes_q, const int32_t* codes_k,
                            const void* v, int32_t hyperplanes, int32_t tables, double* o, double* den,
                            void* workspace, void* stream) {
  if (n < 0 || dv < 1 || hyperplanes < 1 || hyperplanes > 20 || tables < 1) return bad("hard_attention: bad shape");
  if (n == 0) return RACE_OK;
  if (!workspace) return bad("hard_attention: workspace is required");
  const int R = 1 << hyperplanes;
  double* tab = static_cast<double*>(workspace);
  if (int rc = race::report_cuda(
          cudaMemsetAsync(tab, 0, race_aux_hard_workspace_bytes(dv, hyperplanes, tables), S(stream)), "memset"))
    return rc;
  return dispatch(dtype, [&](auto tag) {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
    const unsigned blocks = unsigned((n + 7) / 8);
    k_hard_aggregate<T><<<blocks, 256, 0, S(stream)>>>(n, dv, codes_k, static_cast<const T*>(v), R, tables, tab);
    if (int rc = launched("hard_aggregate")) return rc;
    k_hard_readout<<<blocks, 256, 0, S(stream)>>>(n, dv, codes_q, R, tables, tab, o, den);
    return launched("hard_readout");
  });
}

int race_aux_angular_kernel(int32_t dtype, int64_t n, int64_t m, int32_t d, const void* q, const void* k,
                            int32_t gamma, double* out, void* stream) {
  if (n < 0 || m < 0 || d < 1 || gamma < 1) return bad("angular_kernel: bad shape");
  if (n == 0 || m == 0) return RACE_OK;
  if ((n + 15) / 16 > 65535) return bad("angular_kernel: n too large");
  dim3 grid(unsigned((m + 15) / 16), unsigned((n + 15) / 16));
  return dispatch(dtype, [&](auto tag) {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
    k_angular_matrix<T><<<grid, 256, 0, S(stream)>>>(static_cast<const T*>(q), static_cast<const T*>(k), n, m, d,
                                                      gamma, out);
    return launched("angular_kernel");
  });
}

int race_aux_angular_fwd(int32_t dtype, int64_t n, int32_t d, int32_t dv, const void* q, const void* k,
                         const void* v, int32_t gamma, int32_t causal, double* o, double* den, void* stream) {
  if (n < 0 || d < 1 || dv < 1 || gamma < 1) return bad("angular_fwd: bad shape");
  const int tb = pick_tb(d, dv);
  if (!tb) return race::report(RACE_EUNSUPPORTED, "angular attention: d and dv must be <= 256");
  if (n == 0) return RACE_OK;
  return dispatch(dtype, [&](auto tag) {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
    auto run = [&](auto kern, size_t smem, int rows) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      kern<<<unsigned((n + rows - 1) / rows), kThreads, smem, S(stream)>>>(
          static_cast<const T*>(q), static_cast<const T*>(k), static_cast<const T*>(v), n, d, dv, gamma, causal, o,
          den);
      return launched("angular_fwd");
    };
    return tb == 32 ? run(k_angular_fwd<T, 32>, fwd_smem<32>(d, dv), 32)
                    : run(k_angular_fwd<T, 16>, fwd_smem<16>(d, dv), 16);
  });
}

int race_aux_angular_bwd(int32_t dtype, int64_t n, int32_t d, int32_t dv, const void* q, const void* k,
                         const void* v, const void* d_o, const double* o, const double* den, int32_t gamma,
                         int32_t causal, double* dq, double* dk, double* dv_out, void* stream) {
  if (n < 0 || d < 1 || dv < 1 || gamma < 1) return bad("angular_bwd: bad shape");
  const int tb = pick_tb(d, dv);
  if (!tb) return race::report(RACE_EUNSUPPORTED, "angular attention: d and dv must be <= 256");
  if (n == 0) return RACE_OK;
  return dispatch(dtype, [&](auto tag) {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
    const T* Q = static_cast<const T*>(q);
    const T* K = static_cast<const T*>(k);
    const T* V = static_cast<const T*>(v);
    const T* GO = static_cast<const T*>(d_o);
    auto run = [&](auto kq, auto kk, size_t smem, int rows) {
      const unsigned blocks = unsigned((n + rows - 1) / rows);
      cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      kq<<<blocks, kThreads, smem, S(stream)>>>(Q, K, V, GO, o, den, n, d, dv, gamma, causal, dq);
      if (int rc = launched("angular_bwd_q")) return rc;
      kk<<<blocks, kThreads, smem, S(stream)>>>(Q, K, V, GO, o, den, n, d, dv, gamma, causal, dk, dv_out);
      return launched("angular_bwd_k");
    };
    return tb == 32 ? run(k_angular_bwd_q<T, 32>, k_angular_bwd_k<T, 32>, bwd_smem<32>(d, dv), 32)
                    : run(k_angular_bwd_q<T, 16>, k_angular_bwd_k<T, 16>, bwd_smem<16>(d, dv), 16);
  });
}

}  // extern "C"
