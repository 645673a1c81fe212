// race_abi.cu -- the extern "C" boundary declared in include/race_b200.h.
//
// Validation mirrors the reference's ValueError rules (SketchConfig
// ra/core.py:70-82, AttnInputs ra/exact.py:34-39); the Python layer maps the
// returned status back to ValueError.  Every entry point is stream-ordered,
// allocation-free and thread-safe (globals: the thread-local error string and
// call layout, and a mutex-guarded per-shape segmentation cache).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>

#include "race_common.cuh"

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

}  // namespace

namespace race {  // error reporting for race_aux.cu
int report(int code, const char* msg) { return fail(code, "%s", msg); }
int report_cuda(cudaError_t e, const char* where) { return cuda_status(e, where); }
}  // namespace race

namespace {

// work items to aim for across all (b, h): tcgen05 kernels; RACE_SEG_TARGET overrides (tuning)
const int64_t kSegTarget = [] {
  const char* e = getenv("RACE_SEG_TARGET");
  return e && e[0] ? int64_t(atoll(e)) : int64_t(148) * 8;
}();
// CUDA-core kernels (one CTA per item, 2 per SM); RACE_SIMT_SEG_TARGET overrides (tuning)
const int64_t kSegTargetSimt = [] {
  const char* e = getenv("RACE_SIMT_SEG_TARGET");
  return e && e[0] ? int64_t(atoll(e)) : int64_t(148) * 2 * 7;
}();

// operand strides of the race_fwd_layout / race_bwd_layout call in progress on this thread (every entry
// point it calls resolves its Geo through resolve_shape, which copies them in)
thread_local const race_layout_t* t_layout = nullptr;

// segment length (a multiple of 128 tokens) for about `items` work items across all (b, h)
int64_t segment_for(int64_t BH, int64_t N, int64_t items) {
  int64_t target = (items + BH - 1) / BH;
  if (target < 1) target = 1;
  int64_t per = (N + target - 1) / target;
  per = ((per + 127) / 128) * 128;
  return per < 128 ? 128 : per;
}

// tcgen05 path: the persistent kernels give each of the 148 CTAs a contiguous range of items (cta_range:
// an even split by count) and carry the bucket state across the items of a range, but every item end
// drains the pipeline (partial totals out).  Among 1, 2, 4 and 8 items per CTA, take the segment length
// whose busiest CTA has the fewest 128-token chunks, and among those the fewest items (measured at the
// headline shape: 8 items per CTA 457 us, 2 items per CTA 451 us per causal step).  Cached per shape.
int64_t fast_segment(int64_t BH, int64_t N) {
  static std::mutex mu;
  static std::map<std::pair<int64_t, int64_t>, int64_t> cache;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({BH, N});
    if (it != cache.end()) return it->second;
  }
  const int64_t G = 148, cps = (N + 127) / 128;
  int64_t best = 0, best_load = INT64_MAX;
  for (int64_t per_cta = 1; per_cta <= 8; per_cta *= 2) {
    const int64_t seg = segment_for(BH, N, G * per_cta), sc = seg / 128;
    const int64_t nseg = N > 0 ? (N + seg - 1) / seg : 1, items = BH * nseg;
    const int64_t grid = items < G ? items : G;
    int64_t load = 0;
    for (int64_t b = 0; b < grid; ++b) {  // chunks of CTA b's item range
      int64_t sum = 0;
      for (int64_t i = b * items / grid; i < (b + 1) * items / grid; ++i) {
        const int64_t s = i % nseg;
        sum += s + 1 < nseg ? sc : cps - s * sc;
      }
      load = sum > load ? sum : load;
    }
    if (load < best_load) {  // ties keep the earlier (longer-segment) candidate
      best_load = load;
      best = seg;
    }
  }
  std::lock_guard<std::mutex> lock(mu);
  cache[{BH, N}] = best;
  return best;
}

int resolve_shape(const race_desc_t* d, race::Geo* g) {
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
  // Segments are the work items.  The tcgen05 kernels walk contiguous item ranges of a persistent
  // grid (148 CTAs): ~8 items per SM.  The CUDA-core kernels launch one CTA per item, two resident
  // per SM: aim for ~7 full waves of 2 x 148 so the last wave's tail is small (3.5 waves of 512-token
  // segments left the last wave half empty at N = 131072, H = 4).
  const bool fast_capable = g->dtype == RACE_BF16 && g->d <= 128 && g->dv <= 128 && g->d % 8 == 0 && g->dv % 8 == 0;
  g->seg_tokens = fast_capable && !getenv("RACE_SEG_TARGET") ? fast_segment(g->BH, g->N)
                                                              : segment_for(g->BH, g->N, fast_capable ? kSegTarget
                                                                                                    : kSegTargetSimt);
  g->nseg = g->N > 0 ? (g->N + g->seg_tokens - 1) / g->seg_tokens : 1;
  if (g->nseg > 0x7fffffff) return fail(RACE_EUNSUPPORTED, "too many segments");
  if (t_layout) {
    const race_stride_t* src[race::L_COUNT] = {&t_layout->q,  &t_layout->k,  &t_layout->v,  &t_layout->o,
                                               &t_layout->d_o, &t_layout->dq, &t_layout->dk, &t_layout->dv};
    for (int i = 0; i < race::L_COUNT; ++i) g->lay[i] = race::Lay{src[i]->token, src[i]->head, src[i]->batch};
  }
  return RACE_OK;
}

// one pass of the kernels holds all F = T * 2^cb buckets of a row in shared memory (cb = P unless
// the pass is a corner group); the corner softmax of a pass covers at most kPMax bits
bool fits(const race::Geo& g) {
  const int cb = race::pass_corner_bits(g);
  if (cb > race::kPMax) return false;
  const int64_t F = int64_t(g.T) << cb;
  if (F > 4096 || F * (g.dv + 1) > (1 << 22)) return false;
  return race::tc_supported(g) || race::simt_max_smem(g) <= 227 * 1024;
}

int resolve(const race_desc_t* d, race::Geo* g) {
  if (int rc = resolve_shape(d, g)) return rc;
  if (!fits(*g))
    return fail(RACE_EUNSUPPORTED, "d=%d dv=%d with F=%lld buckets exceeds one pass of the GPU kernels", g->d,
                g->dv, (long long)(int64_t(g->T) << g->P));
  return RACE_OK;
}

// Groups: the estimator is a sum over tables (ra/forward.py:124-144) and, within a table, over its
// corners, so a config whose F does not fit one pass runs as
//   table groups:  tg tables per pass (cb = 0), or, when even one table does not fit (or P > 10),
//   corner groups: one table per pass and 2^cb of its corners (cb < P), T * 2^(P - cb) passes.
// tg == T, cb == 0 means no grouping.
struct GroupPlan {
  int tg = 0;  // tables per group
  int cb = 0;  // corner bits per group (0: whole tables)
  int64_t count(const race::Geo& g) const {
    return cb ? int64_t(g.T) << (g.P - cb) : (g.T + tg - 1) / tg;
  }
  bool grouped(const race::Geo& g) const { return cb || tg < g.T; }
};

// bf16 heads of width 128 whose sketch is beyond one tcgen05 pass still run on the tcgen05 kernels
// when it splits into passes that each are one (table groups for P <= 3, corner groups of 8 corners
// for P = 4, 5): several fast passes beat one pass of the CUDA-core kernels by far at these widths
bool fast_grouping(const race::Geo& g, GroupPlan* gp) {
  if (g.dtype != RACE_BF16 || g.d > 128 || g.dv > 128 || race::tc_supported(g)) return false;
  race::Geo s = g;
  if (g.P <= 3) {
    int tg = 1;
    while ((tg + 1) * g.P <= 5 && ((tg + 1) << g.P) <= 8) ++tg;
    if (tg >= g.T) return false;
    s.T = tg;
    if (!race::tc_supported(s)) return false;
    gp->tg = tg;
    gp->cb = 0;
    return true;
  }
  if (g.P > 5) return false;
  s.T = 1;
  s.cb = 3;
  if (!race::tc_supported(s)) return false;
  gp->tg = 1;
  gp->cb = 3;
  return true;
}

int group_plan(const race_desc_t* d, race::Geo* g, GroupPlan* gp) {
  if (int rc = resolve_shape(d, g)) return rc;
  *gp = GroupPlan{};
  if (fast_grouping(*g, gp)) return RACE_OK;
  if (fits(*g)) {
    gp->tg = g->T;
    return RACE_OK;
  }
  race::Geo s = *g;
  if (g->P <= race::kPMax) {
    for (s.T = g->T - 1; s.T >= 1 && !fits(s); --s.T) {
    }
    if (s.T >= 1) {
      gp->tg = s.T;
      return RACE_OK;
    }
  }
  s.T = 1;
  for (s.cb = (g->P - 1 < race::kPMax ? g->P - 1 : race::kPMax); s.cb >= 1 && !fits(s); --s.cb) {
  }
  if (s.cb < 1)
    return fail(RACE_EUNSUPPORTED, "d=%d dv=%d P=%d: even two corners of one table exceed one pass of the GPU kernels",
                g->d, g->dv, g->P);
  if ((int64_t(g->T) << (g->P - s.cb)) > (int64_t(1) << 24))
    return fail(RACE_EUNSUPPORTED, "P=%d T=%d: more than 2^24 corner groups", g->P, g->T);
  gp->tg = 1;
  gp->cb = s.cb;
  return RACE_OK;
}

// Geo of group i of the plan (table group: tables [t0, t0+cnt); corner group: table t0, high bits chi)
race::Geo group_geo(const race::Geo& g, const GroupPlan& gp, int64_t i, int* t0, int* cnt) {
  race::Geo s = g;
  s.ext_rden = s.ext_gden = nullptr;
  if (gp.cb) {
    const int hb = g.P - gp.cb;
    *t0 = int(i >> hb);
    *cnt = 1;
    s.T = 1;
    s.cb = gp.cb;
    s.chi = i & ((int64_t(1) << hb) - 1);
  } else {
    *t0 = int(i * gp.tg);
    *cnt = g.T - *t0 < gp.tg ? g.T - *t0 : gp.tg;
    s.T = *cnt;
  }
  return s;
}

int64_t table_elems(const race::Geo& g) { return (int64_t(g.T) << race::pass_corner_bits(g)) * (g.dv + 1); }

// causal state = carries [BH, nseg, F, dv+1] then the sketch rows [BH, N, 16]; the rows start on a
// 256-byte boundary (the kernels write them with 16-byte vector stores / TMA) whatever F, dv, BH, nseg
int64_t carry_elems(const race::Geo& g) { return (g.BH * g.nseg * table_elems(g) + 63) & ~int64_t(63); }

struct WsLayout {
  float* part;
  float* tables;   // [BH, nseg, E] (enough for carries too)
  float* dpart;
  float* dtables;  // [BH, nseg, E]
  float* rden;
  float* gden;
  float* rows;     // [BH, N, 16] sketch rows when the caller has no forward state
  void* dqtmp;     // [BH, N, d] generic causal path only: dq when it aliases q (in-place backward)
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
  // the generic causal key-side pass re-reads q after the query-side pass wrote dq
  w.dqtmp = (g.causal && !race::tc_supported(g)) ? take((tok * g.d * (g.dtype == RACE_BF16 ? 2 : 4) + 3) / 4)
                                                  : nullptr;
  w.bytes = off;
  return w;
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// Table groups (group_plan): scratch layout and the elementwise kernels that
// sum the groups' numerators / denominators and gradients.
// ---------------------------------------------------------------------------
struct GroupWs {
  void* sub;        // workspace of one group's sub-problem
  float* w;         // [H, tg * P, d] hyperplanes of the group (w_per_head)
  void* o;          // [BH, N, dv] one group's output (dtype)
  float* den;       // [BH, N]
  float* num_acc;   // [BH, N, dv] sum of numerators
  float* d_acc;     // [BH, N] sum of (unaveraged) denominators
  float* rden;      // [BH, Np] 1 / D of the whole estimator
  float* gden;      // [BH, Np] -(dO . O) / D
  void* dq;         // [BH, N, d] one group's gradients (dtype)
  void* dk;
  void* dv;
  float* dq_acc;    // fp32 sums
  float* dk_acc;
  float* dv_acc;
  float* dproj_q;   // [BH*N, T*P] summed dproj of the query / key side (tcgen05 groups)
  float* dproj_k;
  void* dv_pass;    // [passes, BH, N, dv] each tcgen05 pass's dV (backward) or O (forward), summed once
  float* den_pass;  // [passes, BH, N] each tcgen05 pass's den (forward)
  size_t bytes;
};

constexpr int64_t kMaxPassBuffers = 16;

GroupWs group_ws(const race::Geo& g, const GroupPlan& gp, void* base) {
  int t0, tg;
  const race::Geo s = group_geo(g, gp, 0, &t0, &tg);
  const int64_t tok = g.BH * (g.N > 0 ? g.N : 1);
  const int64_t ptok = g.BH * (g.N > 0 ? (g.N + 3) & ~int64_t(3) : 4);
  const size_t e = g.dtype == RACE_BF16 ? 2 : 4;
  GroupWs w{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t n) -> void* { void* r = p ? p + off : nullptr; off += (n + 255) & ~size_t(255); return r; };
  w.sub = take(ws_layout(s, nullptr).bytes);
  w.w = static_cast<float*>(take(sizeof(float) * size_t(g.H) * tg * g.P * g.d));
  w.o = take(e * tok * g.dv);
  w.den = static_cast<float*>(take(sizeof(float) * tok));
  w.num_acc = static_cast<float*>(take(sizeof(float) * tok * g.dv));
  w.d_acc = static_cast<float*>(take(sizeof(float) * tok));
  w.rden = static_cast<float*>(take(sizeof(float) * ptok));
  w.gden = static_cast<float*>(take(sizeof(float) * ptok));
  w.dq = take(e * tok * g.d);
  w.dk = take(e * tok * g.d);
  w.dv = take(e * tok * g.dv);
  w.dq_acc = static_cast<float*>(take(sizeof(float) * tok * g.d));
  w.dk_acc = static_cast<float*>(take(sizeof(float) * tok * g.d));
  w.dv_acc = static_cast<float*>(take(sizeof(float) * tok * g.dv));
  w.dproj_q = static_cast<float*>(take(sizeof(float) * tok * g.T * g.P));
  w.dproj_k = static_cast<float*>(take(sizeof(float) * tok * g.T * g.P));
  // per-pass dV buffers only for a few tcgen05 passes (P = 20 corner groups would be 2^17 passes)
  const bool passbuf = gp.count(g) <= kMaxPassBuffers && race::tc_supported(s);
  w.dv_pass = passbuf ? take(e * tok * g.dv * size_t(gp.count(g))) : nullptr;
  w.den_pass = passbuf ? static_cast<float*>(take(sizeof(float) * tok * size_t(gp.count(g)))) : nullptr;
  w.bytes = off;
  return w;
}

using race::from_f32;
using race::to_f32;

// 4-wide element access (16-byte fp32 / 8-byte bf16 vectors); callers check the alignment
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u), __uint_as_float(u.y << 16),
                     __uint_as_float(u.y & 0xffff0000u));
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ void st4(__nv_bfloat16* p, float4 v) {
  const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  *reinterpret_cast<uint2*>(p) = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
}

// num_acc (+)= o_g * D_g, d_acc (+)= D_g with D_g = den_g * tg (den_g is the group's averaged den);
// one warp per kAccRows rows (no index division per element; every load of the rows issued before the
// first store), 4 columns per lane step when VEC
constexpr int kAccRows = 4;
template <typename T, bool VEC>
__global__ void k_group_fwd_acc(int64_t rows, int dv, const T* __restrict__ o, const float* __restrict__ den, float tg,
                                int first, float* __restrict__ num_acc, float* __restrict__ d_acc) {
  const int64_t r0 = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * kAccRows;
  const int lane = threadIdx.x & 31;
  if (r0 >= rows) return;
  if (VEC && dv <= 128) {  // every load of the warp's rows first
    const int c = 4 * lane;
    float4 x[kAccRows], acc[kAccRows];
    float D[kAccRows];
#pragma unroll
    for (int q = 0; q < kAccRows; ++q) {
      const int64_t r = r0 + q;
      const bool ok = r < rows && c < dv;
      D[q] = r < rows ? den[r] * tg : 0.f;
      x[q] = ok ? ld4(o + r * dv + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      acc[q] = (ok && !first) ? ld4(num_acc + r * dv + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < kAccRows; ++q) {
      const int64_t r = r0 + q;
      if (r < rows && c < dv)
        st4(num_acc + r * dv + c, make_float4(fmaf(x[q].x, D[q], acc[q].x), fmaf(x[q].y, D[q], acc[q].y),
                                              fmaf(x[q].z, D[q], acc[q].z), fmaf(x[q].w, D[q], acc[q].w)));
    }
  } else {
    for (int q = 0; q < kAccRows && r0 + q < rows; ++q) {
      const int64_t r = r0 + q;
      const float D = den[r] * tg;
      const T* orow = o + r * dv;
      float* nrow = num_acc + r * dv;
      if (VEC) {
        for (int c = 4 * lane; c < dv; c += 128) {
          const float4 x = ld4(orow + c);
          float4 a = first ? make_float4(0.f, 0.f, 0.f, 0.f) : ld4(nrow + c);
          st4(nrow + c, make_float4(fmaf(x.x, D, a.x), fmaf(x.y, D, a.y), fmaf(x.z, D, a.z), fmaf(x.w, D, a.w)));
        }
      } else {
        for (int c = lane; c < dv; c += 32) nrow[c] = fmaf(to_f32(orow[c]), D, first ? 0.f : nrow[c]);
      }
    }
  }
  if (lane < kAccRows && r0 + lane < rows) {
    const int64_t r = r0 + lane;
    const float D = den[r] * tg;
    d_acc[r] = first ? D : d_acc[r] + D;
  }
}

// o = num / D (zero when the averaged den is degenerate, ra/forward.py:157-163), den = D / T
template <typename T, bool VEC>
__global__ void k_group_fwd_out(int64_t rows, int dv, const float* __restrict__ num_acc,
                                const float* __restrict__ d_acc, float T_, T* __restrict__ o, float* __restrict__ den) {
  const int64_t r0 = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * kAccRows;
  const int lane = threadIdx.x & 31;
  if (r0 >= rows) return;
  if (VEC && dv <= 128) {
    const int c = 4 * lane;
    float4 a[kAccRows];
    float rD[kAccRows];
#pragma unroll
    for (int q = 0; q < kAccRows; ++q) {
      const int64_t r = r0 + q;
      const float D = r < rows ? d_acc[r] : 0.f;
      rD[q] = D / T_ > race::kDegenerateDenEps ? 1.f / D : 0.f;
      a[q] = (r < rows && c < dv) ? ld4(num_acc + r * dv + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < kAccRows; ++q) {
      const int64_t r = r0 + q;
      if (r < rows && c < dv)
        st4(o + r * dv + c, make_float4(a[q].x * rD[q], a[q].y * rD[q], a[q].z * rD[q], a[q].w * rD[q]));
    }
  } else {
    for (int q = 0; q < kAccRows && r0 + q < rows; ++q) {
      const int64_t r = r0 + q;
      const float D = d_acc[r];
      const bool live = D / T_ > race::kDegenerateDenEps;
      const float rD = live ? 1.f / D : 0.f;
      const float* nrow = num_acc + r * dv;
      T* orow = o + r * dv;
      if (VEC) {
        for (int c = 4 * lane; c < dv; c += 128) {
          const float4 a = ld4(nrow + c);
          st4(orow + c, make_float4(a.x * rD, a.y * rD, a.z * rD, a.w * rD));
        }
      } else {
        for (int c = lane; c < dv; c += 32) orow[c] = from_f32<T>(live ? nrow[c] / D : 0.f);
      }
    }
  }
  if (lane < kAccRows && r0 + lane < rows) den[r0 + lane] = d_acc[r0 + lane] / T_;
}

// rden = 1 / D, gden = -(dO . O) / D of the whole estimator; one warp per row
template <typename T>
__global__ void k_group_rg(int64_t BH, int64_t N, int dv, const float* __restrict__ num_acc,
                           const float* __restrict__ d_acc, const T* __restrict__ d_o, float T_,
                           float* __restrict__ rden, float* __restrict__ gden, int vec) {
  const int64_t rows = BH * N;
  const int64_t r0 = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * kAccRows;
  const int lane = threadIdx.x & 31;
  if (r0 >= rows) return;
  float rD[kAccRows], dot[kAccRows];
#pragma unroll
  for (int q = 0; q < kAccRows; ++q) {
    const int64_t r = r0 + q;
    const float D = r < rows ? d_acc[r] : 0.f;
    rD[q] = D / T_ > race::kDegenerateDenEps ? 1.f / D : 0.f;
    dot[q] = 0.f;
  }
  if (vec && dv <= 128) {  // 4 columns per lane (16-byte fp32 / 8-byte bf16 loads; the host checked the alignment)
    const int c = 4 * lane;
    float4 g[kAccRows], n[kAccRows];
#pragma unroll
    for (int q = 0; q < kAccRows; ++q) {
      const int64_t r = r0 + q;
      const bool ok = r < rows && c < dv;
      g[q] = ok ? ld4(d_o + r * dv + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      n[q] = ok ? ld4(num_acc + r * dv + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < kAccRows; ++q)
      dot[q] = fmaf(g[q].x, n[q].x * rD[q],
                    fmaf(g[q].y, n[q].y * rD[q], fmaf(g[q].z, n[q].z * rD[q], g[q].w * (n[q].w * rD[q]))));
  } else {
#pragma unroll
    for (int q = 0; q < kAccRows; ++q) {
      const int64_t r = r0 + q;
      if (r < rows)
        for (int c = lane; c < dv; c += 32) dot[q] = fmaf(to_f32(d_o[r * dv + c]), num_acc[r * dv + c] * rD[q], dot[q]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int q = 0; q < kAccRows; ++q) dot[q] += __shfl_xor_sync(0xffffffffu, dot[q], o);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < kAccRows; ++q) {
      const int64_t r = r0 + q;
      if (r < rows) {
        const int64_t i = (r / N) * ((N + 3) & ~int64_t(3)) + r % N;
        rden[i] = rD[q];
        gden[i] = -dot[q] * rD[q];
      }
    }
  }
}

// gradient sum over groups: mode 0 acc = x, 1 acc += x, 2 out = (acc + x) in the output dtype
// (the last group's add fused with the cast); 4 elements per thread when VEC
template <typename T, bool VEC>
__global__ void k_group_grad_acc(int64_t n, const T* __restrict__ x, int mode, float* __restrict__ acc,
                                 T* __restrict__ out) {
  const int64_t i0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * (VEC ? 4 : 1);
  if (i0 >= n) return;
  if (VEC && i0 + 4 <= n) {
    float4 v = ld4(x + i0);
    if (mode) {
      const float4 a = ld4(acc + i0);
      v = make_float4(v.x + a.x, v.y + a.y, v.z + a.z, v.w + a.w);
    }
    if (mode == 2) st4(out + i0, v);
    else st4(acc + i0, v);
    return;
  }
  for (int64_t i = i0; i < n && i < i0 + (VEC ? 4 : 1); ++i) {
    const float v = to_f32(x[i]) + (mode ? acc[i] : 0.f);
    if (mode == 2) out[i] = from_f32<T>(v);
    else acc[i] = v;
  }
}

// Grouped tcgen05 forward: every pass keeps its O (dtype) and den; this one pass forms the whole estimator's
// numerator num = sum_i O_i D_i (fma chain in pass order, D_i = den_i * tables_i) and denominator
// d = sum_i D_i -- the same fp32 operations, in the same order, as k_group_fwd_acc pass by pass -- writes
// them (the grouped state) and, for the final output, O = num / d and den = d / T as k_group_fwd_out.
// One warp per kAccRows rows, dv <= 128, 4 columns per lane.
template <typename T>
__global__ void k_group_fwd_final(int64_t rows, int dv, int passes, const T* __restrict__ o_pass,
                                  const float* __restrict__ den_pass, float tg_first, float tg_last, float T_,
                                  float* __restrict__ num_acc, float* __restrict__ d_acc, T* __restrict__ o,
                                  float* __restrict__ den) {
  const int64_t r0 = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * kAccRows;
  const int lane = threadIdx.x & 31;
  if (r0 >= rows) return;
  const int c = 4 * lane;
#pragma unroll
  for (int q = 0; q < kAccRows; ++q) {
    const int64_t r = r0 + q;
    if (r >= rows) break;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float dsum = 0.f;
    for (int i = 0; i < passes; ++i) {
      const float D = den_pass[int64_t(i) * rows + r] * (i + 1 == passes ? tg_last : tg_first);
      dsum = i == 0 ? D : dsum + D;
      if (c < dv) {
        const float4 x = ld4(o_pass + (int64_t(i) * rows + r) * dv + c);
        acc = make_float4(fmaf(x.x, D, acc.x), fmaf(x.y, D, acc.y), fmaf(x.z, D, acc.z), fmaf(x.w, D, acc.w));
      }
    }
    if (c < dv) st4(num_acc + r * dv + c, acc);
    if (lane == 0) d_acc[r] = dsum;
    if (o) {
      const float rD = dsum / T_ > race::kDegenerateDenEps ? 1.f / dsum : 0.f;
      if (c < dv) st4(o + r * dv + c, make_float4(acc.x * rD, acc.y * rD, acc.z * rD, acc.w * rD));
      if (lane == 0) den[r] = dsum / T_;
    }
  }
}

// dV of the grouped tcgen05 backward: the passes' dV (dtype) summed in pass order in fp32 and cast once --
// the same additions, in the same order, as accumulating pass by pass (k_group_grad_acc modes 0, 1, 2),
// with one read of each pass's dV instead of a read-modify-write of an fp32 sum per pass
template <typename T>
__global__ void k_group_sum_passes(int64_t n, int passes, const T* __restrict__ x, T* __restrict__ out) {
  const int64_t i0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (i0 >= n) return;
  if (i0 + 4 <= n) {
    float4 acc = ld4(x + i0);
    for (int p = 1; p < passes; ++p) {
      const float4 v = ld4(x + int64_t(p) * n + i0);
      acc = make_float4(v.x + acc.x, v.y + acc.y, v.z + acc.z, v.w + acc.w);
    }
    st4(out + i0, acc);
    return;
  }
  for (int64_t i = i0; i < n; ++i) {
    float acc = to_f32(x[i]);
    for (int p = 1; p < passes; ++p) acc = to_f32(x[int64_t(p) * n + i]) + acc;
    out[i] = from_f32<T>(acc);
  }
}

// dx from the summed per-row dproj of all groups (grouped tcgen05 backward): dx^ = sum_j dproj_j w_j over
// every hyperplane, then the sphere-tangent VJP dx = (dx^ - (dx^.x^) x^) / ||x|| of ra/core.py:126-139
// (zero-norm rows and unnormalised inputs pass dx^ through).  One warp per row; the hyperplanes of every
// head sit in shared memory (each chunk read once per kDxRows rows of one sequence), the rows' dproj in
// lane registers (broadcast by shuffles), and a lane's columns c = lane + 32 i in registers.  FULL: d is
// exactly 128 NCH (no per-lane column guards in the inner loop).
constexpr int kDxRows = 4;  // rows per warp iteration (independent chains: latency hiding)
// NCH = 4-column chunks per lane (d <= 128 * NCH); 32-bit shared-memory indexing throughout
template <typename T, int NCH, bool FULL>
__global__ void __launch_bounds__(256, 3) k_dx_from_dproj(int64_t rows, int64_t N, int d, int tp,
                                                       const T* __restrict__ x, const float* __restrict__ dproj,
                                                       const float* __restrict__ w, int nheads_w, int H,
                                                       int normalize, T* __restrict__ dx) {
  extern __shared__ float4 wsm4[];  // [nheads_w, tp, d / 4] float4
  const int d4 = FULL ? 32 * NCH : d / 4;
  const int hstride = tp * d4;
  {
    const float4* w4 = reinterpret_cast<const float4*>(w);
    const int nw4 = nheads_w * hstride;
    for (int i = threadIdx.x; i < nw4; i += blockDim.x) wsm4[i] = w4[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t nquads = (rows + kDxRows - 1) / kDxRows;
  for (int64_t qd = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; qd < nquads; qd += nwarps) {
    const int64_t r0 = qd * kDxRows;
    const int nr = int(rows - r0 < kDxRows ? rows - r0 : kDxRows);  // rows of this quad (warp-uniform)
    // sequence of the quad's first row (32-bit division when the sizes allow it: the common case)
    const int64_t bh0 = (rows < (int64_t(1) << 31)) ? int64_t(uint32_t(r0) / uint32_t(N)) : r0 / N;
    const bool one_seq = (r0 - bh0 * N) + nr <= N;  // all rows in one sequence: one W block
    float4 xv[kDxRows][NCH], acc[kDxRows][NCH];
    float mine[kDxRows];
#pragma unroll
    for (int q = 0; q < kDxRows; ++q) {  // every load of the quad first
      const int64_t rr = r0 + (q < nr ? q : 0);
      mine[q] = (q < nr && lane < tp) ? dproj[rr * tp + lane] : 0.f;
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        const int c4 = lane + 32 * i;
        xv[q][i] = (q < nr && (FULL || c4 < d4)) ? ld4(x + rr * d + 4 * c4) : make_float4(0.f, 0.f, 0.f, 0.f);
        acc[q][i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    // dx^ = sum_j dproj_j w_j: dproj_j broadcast by shuffles, each W chunk read once for the quad's rows
    if (one_seq || nheads_w == 1) {
      const int wbase = (nheads_w > 1 ? int(uint32_t(bh0) % uint32_t(H)) * hstride : 0) + lane;
      for (int j = 0; j < tp; ++j) {  // tp <= 32 (checked by the caller)
        float pj[kDxRows];
#pragma unroll
        for (int q = 0; q < kDxRows; ++q) pj[q] = __shfl_sync(0xffffffffu, mine[q], j);
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          if (FULL || lane + 32 * i < d4) {
            const float4 wv = wsm4[wbase + j * d4 + 32 * i];
#pragma unroll
            for (int q = 0; q < kDxRows; ++q) {
              acc[q][i].x = fmaf(pj[q], wv.x, acc[q][i].x);
              acc[q][i].y = fmaf(pj[q], wv.y, acc[q][i].y);
              acc[q][i].z = fmaf(pj[q], wv.z, acc[q][i].z);
              acc[q][i].w = fmaf(pj[q], wv.w, acc[q][i].w);
            }
          }
        }
      }
    } else {  // the quad straddles two sequences (rare): W block per row
      int wb[kDxRows];
#pragma unroll
      for (int q = 0; q < kDxRows; ++q) wb[q] = int(((r0 + (q < nr ? q : 0)) / N) % H) * hstride + lane;
      for (int j = 0; j < tp; ++j) {
#pragma unroll
        for (int q = 0; q < kDxRows; ++q) {
          const float pj = __shfl_sync(0xffffffffu, mine[q], j);
#pragma unroll
          for (int i = 0; i < NCH; ++i) {
            if (FULL || lane + 32 * i < d4) {
              const float4 wv = wsm4[wb[q] + j * d4 + 32 * i];
              acc[q][i].x = fmaf(pj, wv.x, acc[q][i].x);
              acc[q][i].y = fmaf(pj, wv.y, acc[q][i].y);
              acc[q][i].z = fmaf(pj, wv.z, acc[q][i].z);
              acc[q][i].w = fmaf(pj, wv.w, acc[q][i].w);
            }
          }
        }
      }
    }
    float ss[kDxRows], dot[kDxRows];
#pragma unroll
    for (int q = 0; q < kDxRows; ++q) {
      ss[q] = 0.f;
      dot[q] = 0.f;
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        const float4 a = xv[q][i];
        ss[q] = fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, fmaf(a.w, a.w, ss[q]))));
        dot[q] += acc[q][i].x * a.x + acc[q][i].y * a.y + acc[q][i].z * a.z + acc[q][i].w * a.w;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < kDxRows; ++q) {
        ss[q] += __shfl_xor_sync(0xffffffffu, ss[q], o);
        dot[q] += __shfl_xor_sync(0xffffffffu, dot[q], o);
      }
#pragma unroll
    for (int q = 0; q < kDxRows; ++q) {
      if (q < nr) {
        const int64_t r = r0 + q;
        const bool tang = normalize && ss[q] >= race::kZeroRowEps * race::kZeroRowEps;  // ||x|| >= eps
        const float inv = tang ? rsqrtf(ss[q]) : 1.f;
        const float dt = tang ? dot[q] * inv : 0.f;  // dx^ . x^
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const int c4 = lane + 32 * i;
          if (FULL || c4 < d4) {
            float4 o = acc[q][i];
            if (tang)
              o = make_float4((o.x - dt * xv[q][i].x * inv) * inv, (o.y - dt * xv[q][i].y * inv) * inv,
                              (o.z - dt * xv[q][i].z * inv) * inv, (o.w - dt * xv[q][i].w * inv) * inv);
            st4(dx + r * d + 4 * c4, o);
          }
        }
      }
    }
  }
}

unsigned blocks_for(int64_t n, int t = 256) { return unsigned((n + t - 1) / t); }
inline unsigned acc_blocks(int64_t rows) { return blocks_for((rows + kAccRows - 1) / kAccRows * 32); }

template <typename F>
cudaError_t by_dtype(int dtype, F&& f) {
  return dtype == RACE_BF16 ? f(static_cast<__nv_bfloat16*>(nullptr)) : f(static_cast<float*>(nullptr));
}

// (sub-descriptor, hyperplanes) of the group of `cnt` tables starting at table t0
const float* group_w(const race::Geo& g, const float* w, int t0, int cnt, const GroupWs& ws, cudaStream_t st,
                     cudaError_t* err) {
  const size_t row = size_t(g.P) * g.d * sizeof(float);
  if (!g.w_per_head) return w + size_t(t0) * g.P * g.d;
  *err = cudaMemcpy2DAsync(ws.w, cnt * row, w + size_t(t0) * g.P * g.d, size_t(g.T) * row, cnt * row, size_t(g.H),
                           cudaMemcpyDeviceToDevice, st);
  return ws.w;
}

// Table and corner groups on the tcgen05 path keep each pass's own forward state (its carries and sketch
// rows, or its tables) after the summed numerators / denominators, so the grouped backward skips each
// pass's aggregation, projection and combine.  Layout: [num BH*N*dv | den BH*N | pad to 64 | pass 0 | pass 1 ...].
bool saves_pass_states(const race::Geo& g, const GroupPlan& gp) {
  if (!gp.grouped(g)) return false;
  int t0, cnt;
  const int64_t n = gp.count(g);
  return race::tc_supported(group_geo(g, gp, 0, &t0, &cnt)) && race::tc_supported(group_geo(g, gp, n - 1, &t0, &cnt));
}
int64_t pass_state_elems(const race::Geo& gs) {
  const int64_t e = gs.causal ? carry_elems(gs) + 16 * gs.BH * gs.N : gs.BH * table_elems(gs);
  return (e + 63) & ~int64_t(63);
}
// offset (floats) of pass i's state in a grouped state buffer
int64_t pass_state_offset(const race::Geo& g, const GroupPlan& gp, int64_t i) {
  int64_t off = (g.BH * g.N * (g.dv + 1) + 63) & ~int64_t(63);
  for (int64_t j = 0; j < i; ++j) {
    int t0, cnt;
    off += pass_state_elems(group_geo(g, gp, j, &t0, &cnt));
  }
  return off;
}

int fwd_grouped(const race_desc_t* desc, const race::Geo& g, const GroupPlan& gp, const void* q, const void* k,
                const void* v, const float* w, void* o, float* den, float* state, void* workspace, void* stream,
                bool final_out);
int bwd_grouped(const race_desc_t* desc, const race::Geo& g, const GroupPlan& gp, const void* q, const void* k,
                const void* v, const float* w, const void* d_o, const float* state, void* dq, void* dk, void* dv,
                void* workspace, void* stream);

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

int race_group_plan(const race_desc_t* desc, int64_t* passes, int32_t* tables_per_pass, int32_t* corner_bits,
                    int32_t* fast) {
  race::Geo g;
  GroupPlan gp;
  if (int rc = group_plan(desc, &g, &gp)) return rc;
  int t0, cnt;
  const race::Geo s = gp.grouped(g) ? group_geo(g, gp, 0, &t0, &cnt) : g;
  if (passes) *passes = gp.grouped(g) ? gp.count(g) : 1;
  if (tables_per_pass) *tables_per_pass = gp.grouped(g) ? gp.tg : g.T;
  if (corner_bits) *corner_bits = race::pass_corner_bits(s);
  if (fast) *fast = race::tc_supported(s) ? 1 : 0;
  return RACE_OK;
}

int race_segments(const race_desc_t* desc, int64_t* nseg, int64_t* seg_tokens) {
  race::Geo g;
  GroupPlan gp;
  if (int rc = group_plan(desc, &g, &gp)) return rc;
  if (nseg) *nseg = g.nseg;
  if (seg_tokens) *seg_tokens = g.seg_tokens;
  return RACE_OK;
}

int race_workspace_bytes(const race_desc_t* desc, size_t* bytes) {
  race::Geo g;
  GroupPlan gp;
  if (int rc = group_plan(desc, &g, &gp)) return rc;
  *bytes = gp.grouped(g) ? group_ws(g, gp, nullptr).bytes : ws_layout(g, nullptr).bytes;
  return RACE_OK;
}

int race_state_elems(const race_desc_t* desc, int64_t* elems) {
  race::Geo g;
  GroupPlan gp;
  if (int rc = group_plan(desc, &g, &gp)) return rc;
  if (gp.grouped(g)) {  // table / corner groups: the summed numerators [BH, N, dv] and denominators [BH, N]
    *elems = saves_pass_states(g, gp) ? pass_state_offset(g, gp, gp.count(g)) : g.BH * g.N * (g.dv + 1);
    return RACE_OK;
  }
  *elems = g.causal ? carry_elems(g) + 16 * g.BH * g.N : g.BH * table_elems(g);
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
  GroupPlan gp;
  if (int rc = group_plan(desc, &g, &gp)) return rc;
  if (g.N == 0) return RACE_OK;
  if (!workspace) return fail(RACE_EBADSHAPE, "workspace is required");
  if (gp.grouped(g)) {
    return fwd_grouped(desc, g, gp, q, k, v, w, o, den, state, workspace, stream, true);
  }
  WsLayout ws = ws_layout(g, workspace);
  float* tabs = state ? state : ws.tables;
  if (g.causal) {
    // the aggregation also writes the k halves of the sketch rows, so the scan reads Q, V and those rows
    float* nrm = state ? state + carry_elems(g) : ws.rows;
    if (int rc = race_kside_partials_rows(desc, k, v, w, ws.part, nrm, workspace, stream)) return rc;
    // into a state: the carries' alignment gap is zeroed too, so the whole state is deterministic
    const int pad = state ? int(carry_elems(g) - g.BH * g.nseg * table_elems(g)) : 0;
    if (int rc = cuda_status(race::combine(g, RACE_COMBINE_PREFIX, ws.part, nullptr, tabs, S(stream), pad),
                             "combine"))
      return rc;
    return race_fwd_causal_krows(desc, q, k, v, w, tabs, o, den, nrm, workspace, stream);
  }
  if (int rc = race_kside_partials(desc, k, v, w, ws.part, workspace, stream)) return rc;
  if (int rc = race_combine(desc, RACE_COMBINE_TOTAL, ws.part, nullptr, tabs, stream)) return rc;
  return race_fwd_readout(desc, q, w, tabs, o, den, workspace, stream);
}

int race_bwd(const race_desc_t* desc, const void* q, const void* k, const void* v, const float* w, const void* d_o,
             const float* state, void* dq, void* dk, void* dv, void* workspace, void* stream) {
  race::Geo g;
  GroupPlan gp;
  if (int rc = group_plan(desc, &g, &gp)) return rc;
  if (g.N == 0) return RACE_OK;
  if (!workspace) return fail(RACE_EBADSHAPE, "workspace is required");
  if (gp.grouped(g)) {
    return bwd_grouped(desc, g, gp, q, k, v, w, d_o, state, dq, dk, dv, workspace, stream);
  }
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
  const float* nrm = state ? state + carry_elems(g) : nullptr;
  if (!nrm && race::tc_supported(g)) {  // once for both passes
    if (int rc = cuda_status(race::tc_project(g, q, k, w, ws.rows, S(stream)), "tc_project")) return rc;
    nrm = ws.rows;
  }
  // in-place backward (dq == q): the generic key-side pass still reads q, so dq goes through scratch
  const bool dq_later = dq == q && ws.dqtmp;
  void* dq1 = dq_later ? ws.dqtmp : dq;
  if (int rc = race_bwd_causal_q(desc, q, k, v, d_o, w, tabs, nrm, dq1, ws.rden, ws.gden, ws.dpart, workspace,
                                 stream))
    return rc;
  if (int rc = race_combine(desc, RACE_COMBINE_SUFFIX, ws.dpart, nullptr, ws.dtables, stream)) return rc;
  if (int rc = race_bwd_causal_k(desc, q, k, v, d_o, w, ws.rden, ws.gden, ws.dtables, nrm, dk, dv, workspace, stream))
    return rc;
  if (!dq_later) return RACE_OK;
  const size_t n = size_t(g.BH * g.N) * g.d * (g.dtype == RACE_BF16 ? 2 : 4);
  return cuda_status(cudaMemcpyAsync(dq, ws.dqtmp, n, cudaMemcpyDeviceToDevice, S(stream)), "dq copy");
}

// strided operands: the tcgen05 path reads and writes them through 4-D TMA maps; everything else
// (CUDA-core kernels, grouped sketches, split-phase calls) takes the contiguous layout
static int check_layout(const race_desc_t* desc, const race_layout_t* lay, race::Geo* g) {
  const race_layout_t* saved = t_layout;
  t_layout = nullptr;
  GroupPlan gp;
  int rc = group_plan(desc, g, &gp);
  t_layout = saved;
  if (rc) return rc;
  const race_stride_t* all[race::L_COUNT] = {&lay->q, &lay->k, &lay->v, &lay->o, &lay->d_o, &lay->dq, &lay->dk, &lay->dv};
  bool any = false;
  for (const race_stride_t* s : all) {
    if (!s->token) continue;
    any = true;
    if (s->token < 0 || s->head < 0 || s->batch < 0 || s->token % 8 || s->head % 8 || s->batch % 8)
      return fail(RACE_EBADSHAPE, "operand strides must be non-negative multiples of 8 elements (16 bytes)");
  }
  if (any && (gp.grouped(*g) || !race::tc_supported(*g)))
    return fail(RACE_EUNSUPPORTED, "strided operands need the one-pass tcgen05 path (bf16, d and dv <= 128 "
                                   "multiples of 8, F <= 8); pass contiguous [B*H, N, d] tensors otherwise");
  return RACE_OK;
}

struct LayoutScope {  // the layout is visible to every entry point the call runs, and only to them
  explicit LayoutScope(const race_layout_t* l) { t_layout = l; }
  ~LayoutScope() { t_layout = nullptr; }
};

int race_fwd_layout(const race_desc_t* desc, const race_layout_t* layout, const void* q, const void* k, const void* v,
                    const float* w, void* o, float* den, float* state, void* workspace, void* stream) {
  if (layout) {
    race::Geo g;
    if (int rc = check_layout(desc, layout, &g)) return rc;
  }
  LayoutScope scope(layout);
  return race_fwd(desc, q, k, v, w, o, den, state, workspace, stream);
}

int race_bwd_layout(const race_desc_t* desc, const race_layout_t* layout, const void* q, const void* k, const void* v,
                    const float* w, const void* d_o, const float* state, void* dq, void* dk, void* dv,
                    void* workspace, void* stream) {
  if (layout) {
    race::Geo g;
    if (int rc = check_layout(desc, layout, &g)) return rc;
    if (dq == q || dk == k || dv == v) return fail(RACE_EUNSUPPORTED, "in-place backward needs contiguous operands");
  }
  LayoutScope scope(layout);
  return race_bwd(desc, q, k, v, w, d_o, state, dq, dk, dv, workspace, stream);
}

}  // extern "C"

namespace {

// Forward over the groups: num_acc / d_acc (the workspace's, or the caller's state: [BH, N, dv] then
// [BH, N]) sum the groups' numerators and denominators; final_out writes o and den from them.
int fwd_grouped(const race_desc_t* desc, const race::Geo& g, const GroupPlan& gp, const void* q, const void* k,
                const void* v, const float* w, void* o, float* den, float* state, void* workspace, void* stream,
                bool final_out) {
  GroupWs ws = group_ws(g, gp, workspace);
  if (state) {
    ws.num_acc = state;
    ws.d_acc = state + g.BH * g.N * g.dv;
  }
  const int64_t rows = g.BH * g.N;
  const int64_t ngroups = gp.count(g);
  const cudaStream_t st = S(stream);
  // tcgen05 passes keep their own O and den; k_group_fwd_final sums them once (else: per-pass accumulation)
  const size_t esz = g.dtype == RACE_BF16 ? 2 : 4;
  const bool pass_o = ws.dv_pass && ws.den_pass && g.dv % 4 == 0 && g.dv <= 128 &&
                      (reinterpret_cast<uintptr_t>(ws.num_acc) % 16) == 0 &&
                      (!final_out || (reinterpret_cast<uintptr_t>(o) % (4 * esz)) == 0);
  int tg_first = 1, tg_last = 1;
  for (int64_t i = 0; i < ngroups; ++i) {
    int t0, cnt;
    const race::Geo gs = group_geo(g, gp, i, &t0, &cnt);
    if (i == 0) tg_first = cnt;
    if (i + 1 == ngroups) tg_last = cnt;
    void* oi = pass_o ? static_cast<char*>(ws.dv_pass) + size_t(i) * rows * g.dv * esz : ws.o;
    float* deni = pass_o ? ws.den_pass + size_t(i) * rows : ws.den;
    cudaError_t e = cudaSuccess;
    const float* wg = group_w(g, w, t0, cnt, ws, st, &e);
    if (int rc = cuda_status(e, "table group hyperplanes")) return rc;
    if (!gp.cb) {  // table group: a plain sub-problem (may run on the tcgen05 path)
      race_desc_t sd = *desc;
      sd.tables = cnt;
      float* pst = state && saves_pass_states(g, gp) ? state + pass_state_offset(g, gp, i) : nullptr;
      if (int rc = race_fwd(&sd, q, k, v, wg, oi, deni, pst, ws.sub, stream)) return rc;
    } else {  // corner group: the kernels restricted to the group's corners
      const WsLayout sub = ws_layout(gs, ws.sub);
      const bool fast = race::tc_supported(gs);
      // tcgen05 passes with a grouped state: this pass's carries / tables and sketch rows go into it
      float* pst = state && fast && saves_pass_states(g, gp) ? state + pass_state_offset(g, gp, i) : nullptr;
      float* tabs = pst ? pst : sub.tables;
      float* prow = pst && g.causal ? pst + carry_elems(gs) : sub.rows;
      const int pad = pst && g.causal ? int(carry_elems(gs) - gs.BH * gs.nseg * table_elems(gs)) : 0;
      e = fast ? race::tc_aggregate(gs, k, v, wg, sub.part, nullptr, st) : race::simt_aggregate(gs, k, v, wg, sub.part, st);
      if (e == cudaSuccess)
        e = race::combine(gs, g.causal ? RACE_COMBINE_PREFIX : RACE_COMBINE_TOTAL, sub.part, nullptr, tabs, st, pad);
      if (e == cudaSuccess) {
        if (fast)
          e = g.causal ? race::tc_causal_fwd(gs, q, k, v, wg, tabs, oi, deni, prow, false, st)
                       : race::tc_readout(gs, q, wg, tabs, oi, deni, st);
        else
          e = g.causal ? race::simt_causal_fwd(gs, q, k, v, wg, sub.tables, ws.o, ws.den, nullptr, st)
                       : race::simt_readout(gs, q, wg, sub.tables, ws.o, ws.den, st);
      }
      if (int rc = cuda_status(e, "corner group forward")) return rc;
    }
    if (pass_o) continue;
    e = by_dtype(g.dtype, [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      if (g.dv % 4 == 0 && (reinterpret_cast<uintptr_t>(ws.num_acc) % 16) == 0)
        k_group_fwd_acc<T, true><<<acc_blocks(rows), 256, 0, st>>>(
            rows, g.dv, static_cast<const T*>(ws.o), ws.den, float(cnt), i == 0, ws.num_acc, ws.d_acc);
      else
        k_group_fwd_acc<T, false><<<acc_blocks(rows), 256, 0, st>>>(
            rows, g.dv, static_cast<const T*>(ws.o), ws.den, float(cnt), i == 0, ws.num_acc, ws.d_acc);
      race::note_launch();
      return cudaGetLastError();
    });
    if (int rc = cuda_status(e, "table group sum")) return rc;
  }
  if (pass_o) {
    cudaError_t e = by_dtype(g.dtype, [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      k_group_fwd_final<T><<<acc_blocks(rows), 256, 0, st>>>(
          rows, g.dv, int(ngroups), static_cast<const T*>(ws.dv_pass), ws.den_pass, float(tg_first), float(tg_last),
          float(g.T), ws.num_acc, ws.d_acc, final_out ? static_cast<T*>(o) : nullptr, final_out ? den : nullptr);
      race::note_launch();
      return cudaGetLastError();
    });
    return cuda_status(e, "table group sum and output");
  }
  if (!final_out) return RACE_OK;
  cudaError_t e = by_dtype(g.dtype, [&](auto* tag) {
    using T = std::remove_pointer_t<decltype(tag)>;
    const bool vec = g.dv % 4 == 0 && (reinterpret_cast<uintptr_t>(o) % (4 * sizeof(T))) == 0 &&
                     (reinterpret_cast<uintptr_t>(ws.num_acc) % 16) == 0;
    if (vec)
      k_group_fwd_out<T, true><<<acc_blocks(rows), 256, 0, S(stream)>>>(rows, g.dv, ws.num_acc, ws.d_acc,
                                                                            float(g.T), static_cast<T*>(o), den);
    else
      k_group_fwd_out<T, false><<<acc_blocks(rows), 256, 0, S(stream)>>>(rows, g.dv, ws.num_acc, ws.d_acc,
                                                                             float(g.T), static_cast<T*>(o), den);
    race::note_launch();
    return cudaGetLastError();
  });
  return cuda_status(e, "table group output");
}

// Backward with table groups: the per-token normalisers 1/D and -(dO.O)/D of the whole
// estimator come from a grouped forward; each group then runs the generic backward kernels
// with those normalisers (Geo::ext_rden/ext_gden) and the groups' gradients are summed.
// Backward over the groups: the whole estimator's 1/D and -(dO.O)/D from the saved sums (state) or a
// recomputed grouped forward, then each group's backward with those normalisers; gradients summed.
int bwd_grouped(const race_desc_t* desc, const race::Geo& g, const GroupPlan& gp, const void* q, const void* k,
                const void* v, const float* w, const void* d_o, const float* state, void* dq, void* dk, void* dv,
                void* workspace, void* stream) {
  GroupWs ws = group_ws(g, gp, workspace);
  const int64_t rows = g.BH * g.N;
  if (state) {
    ws.num_acc = const_cast<float*>(state);
    ws.d_acc = const_cast<float*>(state) + rows * g.dv;
  } else if (int rc = fwd_grouped(desc, g, gp, q, k, v, w, nullptr, nullptr, nullptr, workspace, stream, false)) {
    return rc;
  }
  cudaError_t e = by_dtype(g.dtype, [&](auto* tag) {
    using T = std::remove_pointer_t<decltype(tag)>;
    const int vec = g.dv % 4 == 0 && (reinterpret_cast<uintptr_t>(d_o) % 16) == 0 &&
                    (reinterpret_cast<uintptr_t>(ws.num_acc) % 16) == 0;
    k_group_rg<T><<<acc_blocks(rows), 256, 0, S(stream)>>>(g.BH, g.N, g.dv, ws.num_acc, ws.d_acc,
                                                                static_cast<const T*>(d_o), float(g.T), ws.rden,
                                                                ws.gden,
                                                                vec);
    race::note_launch();
    return cudaGetLastError();
  });
  if (int rc = cuda_status(e, "table group normalisers")) return rc;
  const int64_t ngroups = gp.count(g);
  // tcgen05 groups: the query / key kernels emit each row's dproj (summed over corner groups) instead
  // of dq / dk, and one pass at the end forms dq, dk from them (no per-group dq / dk accumulation)
  int t0_, cnt_;
  const int tp_all = g.T * g.P;
  const bool dproj_mode = race::tc_supported(group_geo(g, gp, 0, &t0_, &cnt_)) &&
                          size_t(g.w_per_head ? g.H : 1) * tp_all * g.d * sizeof(float) <= 160 * 1024 &&
                          tp_all <= 32 && g.d % 4 == 0 && g.d <= 256 && (reinterpret_cast<uintptr_t>(q) & 15) == 0 &&
                          (reinterpret_cast<uintptr_t>(k) & 15) == 0 && (reinterpret_cast<uintptr_t>(dq) & 15) == 0 &&
                          (reinterpret_cast<uintptr_t>(dk) & 15) == 0 && (reinterpret_cast<uintptr_t>(dv) & 15) == 0 &&
                          (reinterpret_cast<uintptr_t>(w) & 15) == 0;
  // each tcgen05 pass keeps its own dV and k_group_sum_passes adds them once at the end
  const bool pass_dv = dproj_mode && ws.dv_pass != nullptr;
  if (dproj_mode && gp.cb) {  // corner groups add into their table's columns
    e = cudaMemsetAsync(ws.dproj_q, 0, sizeof(float) * rows * tp_all, S(stream));
    if (e == cudaSuccess) e = cudaMemsetAsync(ws.dproj_k, 0, sizeof(float) * rows * tp_all, S(stream));
    if (int rc = cuda_status(e, "dproj init")) return rc;
  }
  for (int64_t i = 0; i < ngroups; ++i) {
    int t0, cnt;
    race::Geo gs = group_geo(g, gp, i, &t0, &cnt);
    gs.ext_rden = ws.rden;
    gs.ext_gden = ws.gden;
    if (dproj_mode) {
      gs.dproj_q = ws.dproj_q;
      gs.dproj_k = ws.dproj_k;
      gs.dproj_ld = tp_all;
      gs.dproj_col = t0 * g.P;
      gs.dproj_acc = gp.cb ? 1 : 0;
    }
    const float* wg = group_w(g, w, t0, cnt, ws, S(stream), &e);
    if (int rc = cuda_status(e, "table group hyperplanes")) return rc;
    const WsLayout sub = ws_layout(gs, ws.sub);
    const cudaStream_t st = S(stream);
    // tcgen05 passes keep their own dV; one kernel sums them at the end
    void* dvp = pass_dv ? static_cast<char*>(ws.dv_pass) + size_t(i) * rows * g.dv * (g.dtype == RACE_BF16 ? 2 : 4)
                        : ws.dv;
    const float* pst = state && saves_pass_states(g, gp) ? state + pass_state_offset(g, gp, i) : nullptr;
    if (pst) {  // this pass's forward state (tables / carries and sketch rows) saved by the grouped forward
      if (!g.causal) {
        e = race::tc_bwd_q(gs, q, d_o, wg, pst, ws.dq, sub.dpart, st);
        if (e == cudaSuccess) e = race::combine(gs, RACE_COMBINE_TOTAL, sub.dpart, nullptr, sub.dtables, st);
        if (e == cudaSuccess) e = race::tc_bwd_k(gs, k, v, wg, sub.dtables, ws.dk, dvp, st);
      } else {
        float* prow = const_cast<float*>(pst) + carry_elems(gs);
        e = race::tc_bwd_causal_q(gs, q, k, v, d_o, wg, pst, prow, ws.dq, sub.rden, sub.gden, sub.dpart, st);
        if (e == cudaSuccess) e = race::combine(gs, RACE_COMBINE_SUFFIX, sub.dpart, nullptr, sub.dtables, st);
        if (e == cudaSuccess)
          e = race::tc_bwd_causal_k(gs, q, k, v, d_o, wg, ws.rden, ws.gden, sub.dtables, prow, ws.dk, dvp, st);
      }
    } else if (race::tc_supported(gs)) {  // tcgen05 kernels, query side on the whole estimator's 1/D, -rho/D
      e = race::tc_aggregate(gs, k, v, wg, sub.part, nullptr, st);
      if (!g.causal) {
        if (e == cudaSuccess) e = race::combine(gs, RACE_COMBINE_TOTAL, sub.part, nullptr, sub.tables, st);
        if (e == cudaSuccess) e = race::tc_bwd_q(gs, q, d_o, wg, sub.tables, ws.dq, sub.dpart, st);
        if (e == cudaSuccess) e = race::combine(gs, RACE_COMBINE_TOTAL, sub.dpart, nullptr, sub.dtables, st);
        if (e == cudaSuccess) e = race::tc_bwd_k(gs, k, v, wg, sub.dtables, ws.dk, dvp, st);
      } else {
        if (e == cudaSuccess) e = race::tc_project(gs, q, k, wg, sub.rows, st);
        if (e == cudaSuccess) e = race::combine(gs, RACE_COMBINE_PREFIX, sub.part, nullptr, sub.tables, st);
        if (e == cudaSuccess)
          e = race::tc_bwd_causal_q(gs, q, k, v, d_o, wg, sub.tables, sub.rows, ws.dq, sub.rden, sub.gden, sub.dpart,
                                    st);
        if (e == cudaSuccess) e = race::combine(gs, RACE_COMBINE_SUFFIX, sub.dpart, nullptr, sub.dtables, st);
        if (e == cudaSuccess)
          e = race::tc_bwd_causal_k(gs, q, k, v, d_o, wg, ws.rden, ws.gden, sub.dtables, sub.rows, ws.dk, dvp, st);
      }
    } else {
    e = race::simt_aggregate(gs, k, v, wg, sub.part, st);
    if (!g.causal) {
      if (e == cudaSuccess) e = race::combine(gs, RACE_COMBINE_TOTAL, sub.part, nullptr, sub.tables, st);
      if (e == cudaSuccess) e = race::simt_bwd_q(gs, q, d_o, wg, sub.tables, ws.dq, sub.dpart, st);
      if (e == cudaSuccess) e = race::combine(gs, RACE_COMBINE_TOTAL, sub.dpart, nullptr, sub.dtables, st);
      if (e == cudaSuccess) e = race::simt_bwd_k(gs, k, v, wg, sub.dtables, ws.dk, ws.dv, st);
    } else {
      if (e == cudaSuccess) e = race::combine(gs, RACE_COMBINE_PREFIX, sub.part, nullptr, sub.tables, st);
      if (e == cudaSuccess)
        e = race::simt_bwd_causal_q(gs, q, k, v, d_o, wg, sub.tables, ws.dq, nullptr, nullptr, sub.dpart, st);
      if (e == cudaSuccess) e = race::combine(gs, RACE_COMBINE_SUFFIX, sub.dpart, nullptr, sub.dtables, st);
      if (e == cudaSuccess)
        e = race::simt_bwd_causal_k(gs, q, k, v, d_o, wg, ws.rden, ws.gden, sub.dtables, ws.dk, ws.dv, st);
    }
    }
    if (int rc = cuda_status(e, "table group backward")) return rc;
    e = by_dtype(g.dtype, [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      const int mode = i == 0 ? 0 : (i + 1 == ngroups ? 2 : 1);
      auto acc = [&](int64_t n, const void* x, float* a, void* out) {
        const bool vec = (reinterpret_cast<uintptr_t>(out) % (4 * sizeof(T))) == 0 &&
                         (reinterpret_cast<uintptr_t>(a) % 16) == 0;
        if (vec)
          k_group_grad_acc<T, true><<<blocks_for((n + 3) / 4), 256, 0, st>>>(n, static_cast<const T*>(x), mode, a,
                                                                             static_cast<T*>(out));
        else
          k_group_grad_acc<T, false><<<blocks_for(n), 256, 0, st>>>(n, static_cast<const T*>(x), mode, a,
                                                                    static_cast<T*>(out));
      };
      if (!dproj_mode) {  // (dproj mode: dq, dk from the summed dproj at the end)
        acc(rows * g.d, ws.dq, ws.dq_acc, dq);
        acc(rows * g.d, ws.dk, ws.dk_acc, dk);
      }
      if (!pass_dv) acc(rows * g.dv, ws.dv, ws.dv_acc, dv);  // (else: the pass buffers, summed below)
      race::note_launch((dproj_mode ? 0 : 2) + (pass_dv ? 0 : 1));
      return cudaGetLastError();
    });
    if (int rc = cuda_status(e, "table group gradient sum")) return rc;
  }
  if (pass_dv) {
    e = by_dtype(g.dtype, [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      const int64_t n = rows * g.dv;
      k_group_sum_passes<T><<<blocks_for((n + 3) / 4), 256, 0, S(stream)>>>(n, int(ngroups),
                                                                           static_cast<const T*>(ws.dv_pass),
                                                                           static_cast<T*>(dv));
      race::note_launch();
      return cudaGetLastError();
    });
    if (int rc = cuda_status(e, "dv from the passes")) return rc;
  }
  if (!dproj_mode) return RACE_OK;  // the last group's accumulation wrote dq, dk, dv
  e = by_dtype(g.dtype, [&](auto* tag) {
    using T = std::remove_pointer_t<decltype(tag)>;
    const int nheads_w = g.w_per_head ? int(g.H) : 1;
    const size_t smem = sizeof(float) * size_t(nheads_w) * tp_all * g.d;
    auto kern = g.d == 128 ? k_dx_from_dproj<T, 1, true>
                : g.d <= 128 ? k_dx_from_dproj<T, 1, false>
                : g.d == 256 ? k_dx_from_dproj<T, 2, true> : k_dx_from_dproj<T, 2, false>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (err != cudaSuccess) return err;
    const unsigned grid = unsigned(std::min<int64_t>(blocks_for((rows + kDxRows - 1) / kDxRows * 32), 148 * 8));
    kern<<<grid, 256, smem, S(stream)>>>(rows, g.N, g.d, tp_all, static_cast<const T*>(q), ws.dproj_q, w, nheads_w,
                                         int(g.H), g.normalize, static_cast<T*>(dq));
    kern<<<grid, 256, smem, S(stream)>>>(rows, g.N, g.d, tp_all, static_cast<const T*>(k), ws.dproj_k, w, nheads_w,
                                         int(g.H), g.normalize, static_cast<T*>(dk));
    race::note_launch(2);
    return cudaGetLastError();
  });
  return cuda_status(e, "dq, dk from dproj");
}

}  // namespace
