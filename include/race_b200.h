/*
 * race_b200.h -- C ABI of the B200-native RACE attention hot path.
 *
 * The reference (arXiv 2510.04008, /root/reference/pkg/src/race_attention)
 * is pure Python + numpy and has no FFI layer: its hot-path entry points are
 *
 *   race_attention(inp, cfg, workers)            ra/forward.py:147
 *   race_attention_vjp(inp, cfg, d_out, workers) ra/backward.py:184
 *   accumulate_num_den(q, k, v, cfg, workers)    ra/forward.py:124
 *
 * Each function below replaces one step of those (cited per entry).  The
 * Python drop-in (paper_2510_04008_b200/attention.py over functional.py and
 * the ctypes table in _lib.py) binds them; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - All tensor pointers are DEVICE pointers, contiguous, row-major:
 *       q, k, dq, dk : [BH, N, d]        v, o, d_o, dv : [BH, N, dv]
 *       den          : [BH, N] float32   (the reference's averaged den)
 *       w            : [H, T*P, d] float32 (w_per_head=1) or [T*P, d] (0);
 *                      tables in the reference's (m, l) task order
 *                      (ra/forward.py:128); head of row bh is bh % H.
 *       tables       : [BH, F, dv+1] float32, F = T * 2^P, column dv is
 *                      the normaliser ("ones") column:  S = phi(K)^T [V | 1].
 *       seg tables   : [BH, nseg, F, dv+1] float32 (see race_segments).
 *   - Input/output element type is desc->dtype (f32 or bf16); every
 *     accumulation is fp32.
 *   - No hidden allocation, no global mutable state; all launches go on the
 *     caller's stream.  Scratch comes from a caller-provided workspace of
 *     race_workspace_bytes() bytes.
 *   - Return value: RACE_OK, or a RACE_E* code; race_last_error() gives text.
 */
#ifndef RACE_B200_H
#define RACE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RACE_ABI_VERSION 1

enum race_status {
  RACE_OK = 0,
  RACE_EBADSHAPE = 1,    /* inconsistent / non-positive sizes            */
  RACE_EUNSUPPORTED = 2, /* valid config the CUDA path does not support  */
  RACE_ECUDA = 3,        /* a CUDA launch / runtime error                */
};

enum race_dtype { RACE_F32 = 0, RACE_BF16 = 1 };

enum race_combine_mode {
  RACE_COMBINE_TOTAL = 0,  /* out[bh]      = carry + sum_s part[bh][s]     */
  RACE_COMBINE_PREFIX = 1, /* out[bh][s]   = carry + sum_{s'<s} part[bh][s'] */
  RACE_COMBINE_SUFFIX = 2, /* out[bh][s]   = carry + sum_{s'>s} part[bh][s'] */
};

/* Problem descriptor; mirrors SketchConfig (ra/core.py:45-90) plus shapes. */
typedef struct race_desc {
  int32_t abi_version;  /* RACE_ABI_VERSION                                  */
  int32_t dtype;        /* race_dtype of q, k, v, o, d_o, dq, dk, dv         */
  int64_t batch_heads;  /* B*H                                               */
  int64_t heads;        /* H                                                 */
  int64_t n;            /* tokens of this (shard of the) sequence            */
  int32_t dim;          /* d                                                 */
  int32_t dim_v;        /* dv                                                */
  int32_t hyperplanes;  /* P          (SketchConfig.hyperplanes)             */
  int32_t tables;       /* T = M * L  (SketchConfig.total_tables)            */
  float beta;           /* softmax temperature (SketchConfig.beta)           */
  int32_t causal;       /* SketchConfig.causal                               */
  int32_t normalize;    /* SketchConfig.normalize_inputs                     */
  int32_t w_per_head;   /* 1: w is [H, T*P, d]; 0: [T*P, d]                  */
  int32_t reserved[4];  /* must be zero                                      */
} race_desc_t;

int race_abi_version(void);
const char* race_last_error(void);

/* Number of kernels this library has launched in this process (diagnostic;
 * bench.py reports launches per step from it).                            */
int64_t race_launch_count(void);

/* 0 = generic SIMT kernels, 1 = sm_100a tcgen05/TMA fast path for this desc. */
int race_fast_path(const race_desc_t* desc);

/* How race_fwd / race_bwd run this desc: `passes` kernel passes (1 = the
 * whole sketch at once; more = table or corner groups, see
 * race_workspace_bytes), each over `tables_per_pass` tables and 2^corner_bits
 * corners per table; fast = 1 when every pass runs on the sm_100a tcgen05
 * kernels (bf16, d = dv = 128: any P <= 3 via table groups and P = 4, 5 via
 * corner groups of 8 corners), 0 for the CUDA-core kernels.              */
int race_group_plan(const race_desc_t* desc, int64_t* passes,
                    int32_t* tables_per_pass, int32_t* corner_bits,
                    int32_t* fast);

/* Sequence segmentation shared by every kernel: tokens are cut into nseg
 * contiguous segments of seg_tokens (a multiple of 128) per (b, h).  The
 * causal carries and all per-segment partial tables use this split.       */
int race_segments(const race_desc_t* desc, int64_t* nseg, int64_t* seg_tokens);

/* Scratch bytes needed by any entry point below for this desc.
 *
 * Sketches whose F = T * 2^P buckets do not fit one kernel pass (and every
 * P in [11, 20], which SketchConfig accepts, ra/core.py:71) run race_fwd /
 * race_bwd as groups: whole tables per pass, or, when one table does not
 * fit, 2^cb of its corners per pass with the factored per-bit features
 * (ra/sketch.py:120-129, ra/backward.py:65-88); the groups' numerators,
 * denominators and gradients are summed.  Their state is the summed
 * numerators and denominators (race_state_elems); the split-phase entries
 * below return RACE_EUNSUPPORTED for them.                                */
int race_workspace_bytes(const race_desc_t* desc, size_t* bytes);

/* Elements (float32) of the state race_fwd saves for race_bwd:
 * non-causal: tables [BH, F, dv+1];
 * causal: carries [BH, nseg, F, dv+1], padded to a multiple of 64 floats
 *         (so what follows starts 256-byte aligned), then the sketch rows
 *         [BH, N, 16]: per token, floats 0..7 describe q and 8..15 k; slot j
 *         (j < T*P) holds x^.w_j = (x.w_j)/||x|| and slot 7 holds ||x||^2.
 *         The backward rebuilds phi from them instead of re-reading the
 *         other operand (the generic path fills only the norms).
 * grouped descs (race_group_plan passes > 1): the summed (unaveraged)
 *         numerators [BH, N, dv] then denominators [BH, N] of the whole
 *         estimator, from which race_bwd takes 1/D and -(dO.O)/D without
 *         re-running the grouped forward; for groups on the tcgen05 path
 *         (race_group_plan fast) these are padded to
 *         64 floats and followed by every pass's own state (the layout
 *         above for that pass's tables), so race_bwd does not re-aggregate
 *         the passes either.                                              */
int race_state_elems(const race_desc_t* desc, int64_t* elems);

/* ---- monolithic single-device entry points ---------------------------- */

/* Forward: o = num / den, den = averaged denominator (ra/forward.py:147-164,
 * accumulate_num_den ra/forward.py:124-144).  Rows whose averaged den is
 * <= 1e-30 are written as zeros (ra/forward.py:157-163); the host derives
 * degenerate_rows from den.  `state` (may be NULL) receives what race_bwd
 * needs (race_state_elems floats).                                        */
int race_fwd(const race_desc_t* desc, const void* q, const void* k,
             const void* v, const float* w, void* o, float* den,
             float* state, void* workspace, void* stream);

/* Backward (ra/backward.py:184-235).  If state is NULL it is recomputed
 * from k, v exactly as race_fwd would (the reference recomputes too,
 * ra/backward.py:200).  dq, dk, dv may alias q, k, v respectively
 * (in-place backward: the inputs are dead after it, so a training step can
 * hold 4 instead of 7 N x d tensors during the backward).                 */
int race_bwd(const race_desc_t* desc, const void* q, const void* k,
             const void* v, const float* w, const void* d_o,
             const float* state, void* dq, void* dk, void* dv,
             void* workspace, void* stream);

/* ---- strided operands ------------------------------------------------ */

/* Element strides of one [B, H, N, width] operand whose rows (width
 * elements) are contiguous: token, head and batch strides.  token == 0
 * means the default contiguous [B*H, N, width] layout.  Example: the q of
 * a fused projection qkv[B, N, 3, H, d] has token = 3*H*d, head = d,
 * batch = N*3*H*d; an O written as [B, N, H, dv] has token = H*dv.       */
typedef struct {
  int64_t token, head, batch;
} race_stride_t;

typedef struct {
  race_stride_t q, k, v, o, d_o, dq, dk, dv;
} race_layout_t;

/* race_fwd / race_bwd on strided operands (layout may be NULL: contiguous).
 * Strides are multiples of 8 elements.  Strided operands run on the
 * one-pass tcgen05 path only (bf16, d and dv <= 128 and multiples of 8,
 * F <= 8), which reads and writes them in place through 4-D TMA maps --
 * no transposed copies; otherwise RACE_EUNSUPPORTED.  No in-place
 * backward with a layout.  Sizes, workspace and state are those of the
 * same desc.  (No reference counterpart: the reference takes one 2-D
 * matrix per head, ra/bench.py:172-178.)                                  */
int race_fwd_layout(const race_desc_t* desc, const race_layout_t* layout,
                    const void* q, const void* k, const void* v,
                    const float* w, void* o, float* den, float* state,
                    void* workspace, void* stream);
int race_bwd_layout(const race_desc_t* desc, const race_layout_t* layout,
                    const void* q, const void* k, const void* v,
                    const float* w, const void* d_o, const float* state,
                    void* dq, void* dk, void* dv, void* workspace,
                    void* stream);

/* ---- split-phase entry points (sequence sharding across GPUs) --------- */

/* Key-side aggregation per segment: part[bh][s] = phi(K_s)^T [V_s | 1]
 * (ra/forward.py:84-87 per table; concatenated over tables).             */
int race_kside_partials(const race_desc_t* desc, const void* k, const void* v,
                        const float* w, float* part, void* workspace,
                        void* stream);

/* race_kside_partials that also writes the k halves (floats 8..15) of the
 * causal sketch rows [BH, N, 16] into rownorms, for race_fwd_causal_krows.
 * Non-causal descs and the generic path leave rownorms untouched.         */
int race_kside_partials_rows(const race_desc_t* desc, const void* k,
                             const void* v, const float* w, float* part,
                             float* rownorms, void* workspace, void* stream);

/* Fixed-order (deterministic) reduction of per-segment tables; carry may
 * be NULL (= 0) and is [BH, F, dv+1].  out is [BH, F, dv+1] for TOTAL and
 * [BH, nseg, F, dv+1] for PREFIX / SUFFIX.                                */
int race_combine(const race_desc_t* desc, int32_t mode, const float* part,
                 const float* carry, float* out, void* stream);

/* Non-causal query-side readout with global tables (ra/forward.py:93-96,
 * 157-163).                                                               */
int race_fwd_readout(const race_desc_t* desc, const void* q, const float* w,
                     const float* tables, void* o, float* den,
                     void* workspace, void* stream);

/* Causal chunked scan given per-segment carry-in tables
 * (ra/forward.py:100-121).  rownorms (may be NULL) receives the sketch
 * rows [BH, N, 16] (see race_state_elems).                                */
int race_fwd_causal(const race_desc_t* desc, const void* q, const void* k,
                    const void* v, const float* w, const float* carries,
                    void* o, float* den, float* rownorms, void* workspace,
                    void* stream);

/* race_fwd_causal given rownorms whose k halves race_kside_partials_rows
 * wrote: the fast path then reads Q, V and those rows instead of K (the k
 * projections are not recomputed) and fills in the q halves.  Same
 * outputs as race_fwd_causal.                                             */
int race_fwd_causal_krows(const race_desc_t* desc, const void* q,
                          const void* k, const void* v, const float* w,
                          const float* carries, void* o, float* den,
                          float* rownorms, void* workspace, void* stream);

/* Non-causal backward, query side: dq and per-segment partial dS
 * (ra/backward.py:109-118 + the d_num/d_den prologue 201-209).           */
int race_bwd_qside(const race_desc_t* desc, const void* q, const void* d_o,
                   const float* w, const float* tables, void* dq,
                   float* dpart, void* workspace, void* stream);

/* Non-causal backward, key side given global dS (ra/backward.py:122-128). */
int race_bwd_kside(const race_desc_t* desc, const void* k, const void* v,
                   const float* w, const float* dtables, void* dk, void* dv,
                   void* workspace, void* stream);

/* Causal backward, forward-direction scan: dq, per-token normaliser terms
 * rden = 1/(T*den), gden = -(dO.O)/(T*den) ([BH, Np] float32, row pitch
 * Np = N rounded up to a multiple of 4), and per-segment dS totals
 * (ra/backward.py:142-168).  rownorms (may be NULL = recompute into the
 * workspace) is what race_fwd_causal wrote (sketch rows).                 */
int race_bwd_causal_q(const race_desc_t* desc, const void* q, const void* k,
                      const void* v, const void* d_o, const float* w,
                      const float* carries, const float* rownorms, void* dq,
                      float* rden, float* gden, float* dpart, void* workspace,
                      void* stream);

/* Causal backward, reverse-direction scan given per-segment suffix dS
 * (ra/backward.py:169-180).                                               */
int race_bwd_causal_k(const race_desc_t* desc, const void* q, const void* k,
                      const void* v, const void* d_o, const float* w,
                      const float* rden, const float* gden,
                      const float* dcarries, const float* rownorms, void* dk,
                      void* dv, void* workspace, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RACE_B200_H */
