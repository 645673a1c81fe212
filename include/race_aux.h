/*
 * race_aux.h -- C ABI of the validation-side GPU functions: soft / hard
 * hashing, the averaged sketch kernel, the hard-bucket estimator and exact
 * angular attention.  These replace the reference's theory and
 * accuracy-reference functions; they are
 * not on the RACE hot path (include/race_b200.h).
 *
 * Every kernel computes in float64, as the reference does for these
 * functions, so results match it to ~1e-12.  Inputs x, q, k, v, d_o are
 * DEVICE pointers to contiguous row-major matrices of element type `dtype`
 * (RACE_F32, RACE_BF16 or RACE_F64); hyperplanes w are float64 [T*P, d] in
 * the reference's (m, l) task order (ra/forward.py:128); every output is
 * float64.  Return codes and race_last_error() as in race_b200.h.
 */
#ifndef RACE_AUX_H
#define RACE_AUX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RACE_F64 2 /* extra element type accepted by the race_aux_* entries */

/* row_normalize (ra/core.py:114-123) when g is NULL: out = x / ||x|| per
 * row, rows with ||x|| < 1e-12 unchanged.  With g (same dtype and shape
 * as x): row_normalize_vjp (ra/core.py:126-139), out = (g - (g.x^)x^) /
 * ||x||, zero-guarded rows pass g through.  out is float64 [n, d].       */
int race_aux_row_normalize(int32_t dtype, int64_t n, int32_t d, const void* x,
                           const void* g, double* out, void* stream);

/* soft_features of every table (ra/sketch.py:87-129): phi [n, T * 2^P],
 * column tau * 2^P + r = softmax mass of row x on corner r of table tau.
 * normalize = 1 applies row_normalize first (ra/core.py:114-123), as
 * race_kernel does (ra/forward.py:184-185).  P <= 20, T * P <= 256.      */
int race_aux_soft_features(int32_t dtype, int64_t n, int32_t d, const void* x,
                           const double* w, int32_t hyperplanes,
                           int32_t tables, double beta, int32_t normalize,
                           double* phi, void* stream);

/* hard_hash per table (ra/sketch.py:143-149): codes [T, n] int32, bit t =
 * (x . w_t < 0).                                                          */
int race_aux_hard_hash(int32_t dtype, int64_t n, int32_t d, const void* x,
                       const double* w, int32_t hyperplanes, int32_t tables,
                       int32_t normalize, int32_t* codes, void* stream);

/* out [n, m] = scale * phi_q [n, f] phi_k [m, f]^T: the contraction of
 * race_kernel (ra/forward.py:195-202; scale = 1 / total_tables).          */
int race_aux_feature_gram(int64_t n, int64_t m, int32_t f,
                          const double* phi_q, const double* phi_k,
                          double scale, double* out, void* stream);

/* hard_race_attention given hard_hash codes of q and k
 * (ra/theory.py:205-227): o [n, dv], den [n] (averaged; rows with
 * den <= 1e-30 are zero).  workspace: race_aux_hard_workspace_bytes().   */
size_t race_aux_hard_workspace_bytes(int32_t dv, int32_t hyperplanes,
                                     int32_t tables);
int race_aux_hard_attention(int32_t dtype, int64_t n, int32_t dv,
                            const int32_t* codes_q, const int32_t* codes_k,
                            const void* v, int32_t hyperplanes,
                            int32_t tables, double* o, double* den,
                            void* workspace, void* stream);

/* angular_kernel_matrix (ra/exact.py:116-125): out [n, m].               */
int race_aux_angular_kernel(int32_t dtype, int64_t n, int64_t m, int32_t d,
                            const void* q, const void* k, int32_t gamma,
                            double* out, void* stream);

/* angular_attention (ra/exact.py:128-166): o [n, dv] (degenerate rows
 * zero), den [n] = row similarity sums.  d, dv <= 256.                    */
int race_aux_angular_fwd(int32_t dtype, int64_t n, int32_t d, int32_t dv,
                         const void* q, const void* k, const void* v,
                         int32_t gamma, int32_t causal, double* o,
                         double* den, void* stream);

/* angular_attention_vjp (ra/exact.py:169-218) given the forward's o, den. */
int race_aux_angular_bwd(int32_t dtype, int64_t n, int32_t d, int32_t dv,
                         const void* q, const void* k, const void* v,
                         const void* d_o, const double* o, const double* den,
                         int32_t gamma, int32_t causal, double* dq,
                         double* dk, double* dv_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RACE_AUX_H */
