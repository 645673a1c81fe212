#include <cstdlib>
// race_abi.cu -- the extern "C" boundary declared in include/race_b200.h.
//
// Validation mirrors the reference's ValueError rules (SketchConfig
// ra/core.py:70-82, AttnInputs ra/exact.py:34-39); the Python layer maps the
// returned status back to ValueError.  Every entry point is stream-ordered,
// allocation-free and thread-safe (the only global is the thread-local error
// string).
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "race_b200.h"
#include "race_internal.h"

namespace race {
// fast path (race_tc.cu)
bool tc_supported(const Geo& g);
cudaError_t tc_aggregate(const Geo& g, const void* k, const void* v, const float* w, float* part, float* rows,
                         cudaStream_t st);
cudaError_t tc_readout(const Geo& g, const void* q, const float* w, const float* tab, void* o, float* den,
                       cudaStream_t st);
cudaError_t tc_bwd_q(const Geo& g, const void* q, const void* d_o, const float* w, const float* tab, void* dq,
                     float* dpart, cudaStream_t st);
cudaError_t tc_bwd_k(const Geo& g, const void* k, const void* v, const float* w, const float* dtab, void* dk,
                     void* dv, cudaStream_t st);
cudaError_t tc_bwd_causal_q(const Geo& g, const void* q, const void* k, const void* v, const void* d_o,
                            const float* w, const float* car, const float* nrm, void* dq, float* rden, float* gden,
                            float* dpart, cudaStream_t st);
cudaError_t tc_bwd_causal_k(const Geo& g, const void* q, const void* k, const void* v, const void* d_o,
                            const float* w, const float* rden, const float* gden, const float* dcar,
                            const float* nrm, void* dk, void* dv, cudaStream_t st);
cudaError_t tc_project(const Geo& g, const void* q, const void* k, const float* w, float* rows, cudaStream_t st);
cudaError_t tc_causal_fwd(const Geo& g, const void* q, const void* k, const void* v, const float* w,
                          const float* car, void* o, float* den, float* nrm, bool krows, cudaStream_t st);
}  // namespace race

namespace race {
static std::atomic<int64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace race

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return RACE_OK;
  if (e == cudaErrorInvalidConfiguration)
    return fail(RACE_EUNSUPPORTED, "%s: shape needs more shared memory than an sm_100a CTA has", where);
  return fail(RACE_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

constexpr int64_t kSegTarget = 148 * 8;  // CTAs to aim for across all (b, h)

int resolve(const race_desc_t* d, race::Geo* g) {
  if (!d) return fail(RACE_EBADSHAPE, "null descriptor");
  if (d->abi_version != RACE_ABI_VERSION)
    return fail(RACE_EBADSHAPE, "abi_version %d != %d", d->abi_version, RACE_ABI_VERSION);
  if (d->dtype != RACE_F32 && d->dtype != RACE_BF16) return fail(RACE_EUNSUPPORTED, "dtype %d", d->dtype);
  if (d->batch_heads < 1 || d->heads < 1 || d->n < 0 || d->dim < 1 || d->dim_v < 1)
    return fail(RACE_EBADSHAPE, "bad sizes BH=%lld H=%lld N=%lld d=%d dv=%d", (long long)d->batch_heads,
                (long long)d->heads, (long long)d->n, d->dim, d->dim_v);
  if (d->batch_heads % d->heads) return fail(RACE_EBADSHAPE, "batch_heads not a multiple of heads");
  if (d->hyperplanes < 1 || d->hyperplanes > 20)
    return fail(RACE_EBADSHAPE, "hyperplanes must be in [1, 20], got %d", d->hyperplanes);
  if (d->tables < 1) return fail(RACE_EBADSHAPE, "tables must be >= 1");
  if (!(std::isfinite(d->beta) && d->beta > 0.f)) return fail(RACE_EBADSHAPE, "beta must be positive and finite");
  if (d->batch_heads > 65535) return fail(RACE_EUNSUPPORTED, "batch*heads > 65535");
  if (d->hyperplanes > 10) return fail(RACE_EUNSUPPORTED, "P=%d > 10 corner bits is not supported on the GPU path", d->hyperplanes);
  g->BH = d->batch_heads;
  g->H = d->heads;
  g->N = d->n;
  g->d = d->dim;
  g->dv = d->dim_v;
  g->P = d->hyperplanes;
  g->T = d->tables;
  g->beta = d->beta;
  g->normalize = d->normalize ? 1 : 0;
  g->w_per_head = d->w_per_head ? 1 : 0;
  g->dtype = d->dtype;
  g->causal = d->causal ? 1 : 0;
  const int64_t F = int64_t(d->tables) << d->hyperplanes;
  if (F > 4096 || F * (d->dim_v + 1) > (1 << 22))
    return fail(RACE_EUNSUPPORTED, "F=%lld buckets x dv=%d too large for the GPU path", (long long)F, d->dim_v);
  int64_t target = (kSegTarget + g->BH - 1) / g->BH;
  if (target < 1) target = 1;
  int64_t per = (g->N + target - 1) / target;
  per = ((per + 127) / 128) * 128;
  if (per < 128) per = 128;
  g->seg_tokens = per;
  g->nseg = g->N > 0 ? (g->N + per - 1) / per : 1;
  if (g->nseg > 0x7fffffff) return fail(RACE_EUNSUPPORTED, "too many segments");
  if (race::simt_max_smem(*g) > 227 * 1024 && !race::tc_supported(*g))
    return fail(RACE_EUNSUPPORTED, "d=%d dv=%d F=%lld exceed the shared-memory budget of the generic path", g->d,
                g->dv, (long long)F);
  return RACE_OK;
}

int64_t table_elems(const race::Geo& g) { return (int64_t(g.T) << g.P) * (g.dv + 1); }

struct WsLayout {
  float* part;
  float* tables;   // [BH, nseg, E] (enough for carries too)
  float* dpart;
  float* dtables;  // [BH, nseg, E]
  float* rden;
  float* gden;
  float* rows;     // [BH, N, 16] sketch rows when the caller has no forward state
  size_t bytes;
};

WsLayout ws_layout(const race::Geo& g, void* base) {
  const int64_t E = table_elems(g);
  const int64_t segE = g.BH * g.nseg * E;
  const int64_t tok = g.BH * (g.N > 0 ? g.N : 1);
  const int64_t ptok = g.BH * (g.N > 0 ? (g.N + 3) & ~int64_t(3) : 4);  // rden / gden rows padded to 16 bytes
  auto al = [](int64_t n) { return (n + 63) & ~int64_t(63); };
  WsLayout w{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](int64_t n) { float* r = p ? reinterpret_cast<float*>(p + off) : nullptr; off += al(n) * sizeof(float); return r; };
  w.part = take(segE);
  w.tables = take(segE);
  w.dpart = take(segE);
  w.dtables = take(segE);
  w.rden = take(ptok);
  w.gden = take(ptok);
  w.rows = take(16 * tok);
  w.bytes = off;
  return w;
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int race_abi_version(void) { return RACE_ABI_VERSION; }
const char* race_last_error(void) { return g_err.c_str(); }
int64_t race_launch_count(void) { return race::g_launches.load(std::memory_order_relaxed); }

int race_fast_path(const race_desc_t* desc) {
  race::Geo g;
  if (resolve(desc, &g) != RACE_OK) return 0;
  return race::tc_supported(g) ? 1 : 0;
}

int race_segments(const race_desc_t* desc, int64_t* nseg, int64_t* seg_tokens) {
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (nseg) *nseg = g.nseg;
  if (seg_tokens) *seg_tokens = g.seg_tokens;
  return RACE_OK;
}

int race_workspace_bytes(const race_desc_t* desc, size_t* bytes) {
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  *bytes = ws_layout(g, nullptr).bytes;
  return RACE_OK;
}

int race_state_elems(const race_desc_t* desc, int64_t* elems) {
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  *elems = g.BH * (g.causal ? g.nseg : 1) * table_elems(g) + (g.causal ? 16 * g.BH * g.N : 0);
  return RACE_OK;
}

int race_kside_partials(const race_desc_t* desc, const void* k, const void* v, const float* w, float* part,
                        void* workspace, void* stream) {
  (void)workspace;
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (g.N == 0) return RACE_OK;
  if (race::tc_supported(g)) return cuda_status(race::tc_aggregate(g, k, v, w, part, nullptr, S(stream)), "tc_aggregate");
  return cuda_status(race::simt_aggregate(g, k, v, w, part, S(stream)), "aggregate");
}

int race_kside_partials_rows(const race_desc_t* desc, const void* k, const void* v, const float* w, float* part,
                             float* rownorms, void* workspace, void* stream) {
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (g.N == 0) return RACE_OK;
  if (!g.causal || !race::tc_supported(g) || !rownorms)
    return race_kside_partials(desc, k, v, w, part, workspace, stream);
  return cuda_status(race::tc_aggregate(g, k, v, w, part, rownorms, S(stream)), "tc_aggregate");
}

int race_combine(const race_desc_t* desc, int32_t mode, const float* part, const float* carry, float* out,
                 void* stream) {
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (mode < 0 || mode > 2) return fail(RACE_EBADSHAPE, "combine mode %d", mode);
  if (g.N == 0 && mode != RACE_COMBINE_TOTAL) return RACE_OK;
  if (g.N == 0) {
    // empty shard: total is just the carry (or zero)
    const size_t n = size_t(g.BH * table_elems(g)) * sizeof(float);
    cudaError_t e = carry ? cudaMemcpyAsync(out, carry, n, cudaMemcpyDeviceToDevice, S(stream))
                          : cudaMemsetAsync(out, 0, n, S(stream));
    return cuda_status(e, "combine(empty)");
  }
  return cuda_status(race::combine(g, mode, part, carry, out, S(stream)), "combine");
}

int race_fwd_readout(const race_desc_t* desc, const void* q, const float* w, const float* tables, void* o,
                     float* den, void* workspace, void* stream) {
  (void)workspace;
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (g.N == 0) return RACE_OK;
  if (race::tc_supported(g)) return cuda_status(race::tc_readout(g, q, w, tables, o, den, S(stream)), "tc_readout");
  return cuda_status(race::simt_readout(g, q, w, tables, o, den, S(stream)), "readout");
}

int race_fwd_causal(const race_desc_t* desc, const void* q, const void* k, const void* v, const float* w,
                    const float* carries, void* o, float* den, float* rownorms, void* workspace, void* stream) {
  (void)workspace;
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (g.N == 0) return RACE_OK;
  if (race::tc_supported(g))
    return cuda_status(race::tc_causal_fwd(g, q, k, v, w, carries, o, den, rownorms, false, S(stream)), "tc_causal_fwd");
  return cuda_status(race::simt_causal_fwd(g, q, k, v, w, carries, o, den, rownorms, S(stream)), "causal_fwd");
}

int race_fwd_causal_krows(const race_desc_t* desc, const void* q, const void* k, const void* v, const float* w,
                          const float* carries, void* o, float* den, float* rownorms, void* workspace,
                          void* stream) {
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (g.N == 0) return RACE_OK;
  if (!g.causal) return fail(RACE_EBADSHAPE, "race_fwd_causal_krows needs a causal desc");
  if (!rownorms) return fail(RACE_EBADSHAPE, "race_fwd_causal_krows needs the sketch rows");
  if (race::tc_supported(g))
    return cuda_status(race::tc_causal_fwd(g, q, k, v, w, carries, o, den, rownorms, true, S(stream)),
                       "tc_causal_fwd");
  return race_fwd_causal(desc, q, k, v, w, carries, o, den, rownorms, workspace, stream);
}

int race_bwd_qside(const race_desc_t* desc, const void* q, const void* d_o, const float* w, const float* tables,
                   void* dq, float* dpart, void* workspace, void* stream) {
  (void)workspace;
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (g.N == 0) return RACE_OK;
  if (race::tc_supported(g))
    return cuda_status(race::tc_bwd_q(g, q, d_o, w, tables, dq, dpart, S(stream)), "tc_bwd_qside");
  return cuda_status(race::simt_bwd_q(g, q, d_o, w, tables, dq, dpart, S(stream)), "bwd_qside");
}

int race_bwd_kside(const race_desc_t* desc, const void* k, const void* v, const float* w, const float* dtables,
                   void* dk, void* dv, void* workspace, void* stream) {
  (void)workspace;
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (g.N == 0) return RACE_OK;
  if (race::tc_supported(g))
    return cuda_status(race::tc_bwd_k(g, k, v, w, dtables, dk, dv, S(stream)), "tc_bwd_kside");
  return cuda_status(race::simt_bwd_k(g, k, v, w, dtables, dk, dv, S(stream)), "bwd_kside");
}

int race_bwd_causal_q(const race_desc_t* desc, const void* q, const void* k, const void* v, const void* d_o,
                      const float* w, const float* carries, const float* rownorms, void* dq, float* rden,
                      float* gden, float* dpart, void* workspace, void* stream) {
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (g.N == 0) return RACE_OK;
  if (race::tc_supported(g)) {
    if (!rownorms) {  // recompute the forward's sketch rows (bit-identical)
      if (!workspace) return fail(RACE_EBADSHAPE, "workspace is required");
      float* rows = ws_layout(g, workspace).rows;
      if (int rc = cuda_status(race::tc_project(g, q, k, w, rows, S(stream)), "tc_project")) return rc;
      rownorms = rows;
    }
    return cuda_status(race::tc_bwd_causal_q(g, q, k, v, d_o, w, carries, rownorms, dq, rden, gden, dpart, S(stream)),
                       "tc_bwd_causal_q");
  }
  return cuda_status(race::simt_bwd_causal_q(g, q, k, v, d_o, w, carries, dq, rden, gden, dpart, S(stream)),
                     "bwd_causal_q");
}

int race_bwd_causal_k(const race_desc_t* desc, const void* q, const void* k, const void* v, const void* d_o,
                      const float* w, const float* rden, const float* gden, const float* dcarries,
                      const float* rownorms, void* dk, void* dv, void* workspace, void* stream) {
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (g.N == 0) return RACE_OK;
  if (race::tc_supported(g)) {
    if (!rownorms) {
      if (!workspace) return fail(RACE_EBADSHAPE, "workspace is required");
      float* rows = ws_layout(g, workspace).rows;
      if (int rc = cuda_status(race::tc_project(g, q, k, w, rows, S(stream)), "tc_project")) return rc;
      rownorms = rows;
    }
    return cuda_status(race::tc_bwd_causal_k(g, q, k, v, d_o, w, rden, gden, dcarries, rownorms, dk, dv, S(stream)),
                       "tc_bwd_causal_k");
  }
  return cuda_status(race::simt_bwd_causal_k(g, q, k, v, d_o, w, rden, gden, dcarries, dk, dv, S(stream)),
                     "bwd_causal_k");
}

int race_fwd(const race_desc_t* desc, const void* q, const void* k, const void* v, const float* w, void* o,
             float* den, float* state, void* workspace, void* stream) {
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (g.N == 0) return RACE_OK;
  if (!workspace) return fail(RACE_EBADSHAPE, "workspace is required");
  WsLayout ws = ws_layout(g, workspace);
  float* tabs = state ? state : ws.tables;
  static const bool no_krows = getenv("RACE_NO_KROWS") != nullptr;  // A/B diagnostic
  if (g.causal && !no_krows) {
    // the aggregation also writes the k halves of the sketch rows, so the scan reads Q, V and those rows
    float* nrm = state ? state + g.BH * g.nseg * table_elems(g) : ws.rows;
    if (int rc = race_kside_partials_rows(desc, k, v, w, ws.part, nrm, workspace, stream)) return rc;
    if (int rc = race_combine(desc, RACE_COMBINE_PREFIX, ws.part, nullptr, tabs, stream)) return rc;
    return race_fwd_causal_krows(desc, q, k, v, w, tabs, o, den, nrm, workspace, stream);
  }
  if (int rc = race_kside_partials(desc, k, v, w, ws.part, workspace, stream)) return rc;
  if (g.causal) {
    if (int rc = race_combine(desc, RACE_COMBINE_PREFIX, ws.part, nullptr, tabs, stream)) return rc;
    float* nrm = state ? state + g.BH * g.nseg * table_elems(g) : nullptr;
    return race_fwd_causal(desc, q, k, v, w, tabs, o, den, nrm, workspace, stream);
  }
  if (int rc = race_combine(desc, RACE_COMBINE_TOTAL, ws.part, nullptr, tabs, stream)) return rc;
  return race_fwd_readout(desc, q, w, tabs, o, den, workspace, stream);
}

int race_bwd(const race_desc_t* desc, const void* q, const void* k, const void* v, const float* w, const void* d_o,
             const float* state, void* dq, void* dk, void* dv, void* workspace, void* stream) {
  race::Geo g;
  if (int rc = resolve(desc, &g)) return rc;
  if (g.N == 0) return RACE_OK;
  if (!workspace) return fail(RACE_EBADSHAPE, "workspace is required");
  WsLayout ws = ws_layout(g, workspace);
  const float* tabs = state;
  if (!tabs) {
    if (int rc = race_kside_partials(desc, k, v, w, ws.part, workspace, stream)) return rc;
    if (int rc = race_combine(desc, g.causal ? RACE_COMBINE_PREFIX : RACE_COMBINE_TOTAL, ws.part, nullptr,
                              ws.tables, stream))
      return rc;
    tabs = ws.tables;
  }
  if (!g.causal) {
    if (int rc = race_bwd_qside(desc, q, d_o, w, tabs, dq, ws.dpart, workspace, stream)) return rc;
    if (int rc = race_combine(desc, RACE_COMBINE_TOTAL, ws.dpart, nullptr, ws.dtables, stream)) return rc;
    return race_bwd_kside(desc, k, v, w, ws.dtables, dk, dv, workspace, stream);
  }
  const float* nrm = state ? state + g.BH * g.nseg * table_elems(g) : nullptr;
  if (!nrm && race::tc_supported(g)) {  // once for both passes
    if (int rc = cuda_status(race::tc_project(g, q, k, w, ws.rows, S(stream)), "tc_project")) return rc;
    nrm = ws.rows;
  }
  if (int rc = race_bwd_causal_q(desc, q, k, v, d_o, w, tabs, nrm, dq, ws.rden, ws.gden, ws.dpart, workspace,
                                 stream))
    return rc;
  if (int rc = race_combine(desc, RACE_COMBINE_SUFFIX, ws.dpart, nullptr, ws.dtables, stream)) return rc;
  return race_bwd_causal_k(desc, q, k, v, d_o, w, ws.rden, ws.gden, ws.dtables, nrm, dk, dv, workspace, stream);
}

}  // extern "C"
