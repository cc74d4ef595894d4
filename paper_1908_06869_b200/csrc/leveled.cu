// Stage (f): the leveled-measurement merge (XSP "leveled experimentation").
//
// Reference semantics: LeveledRunGroup (leveled.cpp:56-84), event_latencies
// (:98-122), chain_of (:124-141), compute_overhead (:145-231). Each level set
// of the chain holds repeated runs; every event (model, layer i, kernel (i,k))
// gets a trimmed-mean latency per set, the overhead of each chain step is the
// wider set's latency minus the narrower one's (small negatives clamped), and
// the accurate latency of an event comes from the set whose deepest level is
// the event's own. The event universe and all per-(set, event) reductions run
// on the device; only the chain order (a handful of sets) is decided on the host.
// Compiled with -fmad=false (fp64 op order as the reference).

#include <algorithm>
#include <numeric>
#include <vector>

#include "ctx.h"
#include "prims.cuh"

namespace xsp {

constexpr int kMaxRunsL = 64;

__device__ double trimmed_mean_l(double* v, uint32_t n, double f) {
  for (uint32_t i = 1; i < n; ++i) {
    double x = v[i];
    uint32_t j = i;
    while (j > 0 && v[j - 1] > x) {
      v[j] = v[j - 1];
      --j;
    }
    v[j] = x;
  }
  uint32_t drop = (uint32_t)floor(f * (double)n);
  double s = 0.0;
  for (uint32_t i = drop; i < n - drop; ++i) s = __dadd_rn(s, v[i]);
  return s / (double)(n - 2 * drop);
}

// rank of a level (span.hpp:51-59)
__host__ __device__ __forceinline__ int level_rank(uint32_t l) { return l == 0 ? 1 : (l == 1 ? 2 : 3); }

struct LevArgs {
  uint32_t S;             // sets in chain order
  const uint32_t* soff;   // [S + 1] offsets into tr
  const uint32_t* tr;     // traces of the sets, chain order
  const uint32_t* lv;     // [S] level masks
  const uint32_t* t_layer_off;
  const uint32_t* t_kernel_off;
  const uint32_t* l_koff;
  const uint64_t* layer_dur;
  const uint64_t* kernel_dur;
  const uint32_t* model_row;
  const uint64_t* begin;
  const uint64_t* end;
  uint32_t* lmax;    // [1] max layer count over sets with L
  uint32_t* kmax;    // [lmax_cap] max kernel count of layer i over sets with L and G
  uint32_t* kbase;   // [lmax+1] exclusive scan of kmax
  uint32_t n_events;
  double trim, noise;
  uint8_t* ev_level;
  uint32_t* ev_layer;
  uint32_t* ev_kernel;
  double* lat;
  double* overhead;
  uint8_t* step_flags;
  double* accurate;
};

__device__ __forceinline__ bool has_level(uint32_t mask, uint32_t l) { return (mask >> l) & 1u; }

// universe of layer events: max layer count over the traces of sets with L
__global__ void k_lev_layers(LevArgs a, uint32_t total_runs) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= total_runs) return;
  uint32_t s = 0;
  while (s + 1 < a.S && a.soff[s + 1] <= q) ++s;
  if (!has_level(a.lv[s], XSP_LEVEL_LAYER)) return;
  const uint32_t t = a.tr[q];
  atomicMax(a.lmax, a.t_layer_off[t + 1] - a.t_layer_off[t]);
}

// universe of kernel events: per layer index, max kernel count over sets with L and G
__global__ void k_lev_kernels(LevArgs a, uint32_t total_runs) {
  const uint32_t q = blockIdx.x;  // one block per run
  if (q >= total_runs) return;
  uint32_t s = 0;
  while (s + 1 < a.S && a.soff[s + 1] <= q) ++s;
  if (!has_level(a.lv[s], XSP_LEVEL_LAYER) || !has_level(a.lv[s], XSP_LEVEL_KERNEL)) return;
  const uint32_t t = a.tr[q];
  const uint32_t l0 = a.t_layer_off[t], l1 = a.t_layer_off[t + 1];
  for (uint32_t g = l0 + threadIdx.x; g < l1; g += blockDim.x)
    atomicMax(a.kmax + (g - l0), a.l_koff[g + 1] - a.l_koff[g]);
}

// event keys in (rank, layer_index, kernel_index) order
__global__ void k_lev_keys(LevArgs a) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.n_events) return;
  const uint32_t L = *a.lmax;
  if (e == 0) {
    a.ev_level[e] = XSP_LEVEL_MODEL;
    a.ev_layer[e] = 0;
    a.ev_kernel[e] = 0;
  } else if (e <= L) {
    a.ev_level[e] = XSP_LEVEL_LAYER;
    a.ev_layer[e] = e - 1;
    a.ev_kernel[e] = 0;
  } else {
    const uint32_t k = e - 1 - L;
    uint32_t lo = 0, hi = L;  // kbase[lo] <= k < kbase[lo + 1]
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (a.kbase[mid] <= k) lo = mid; else hi = mid;
    }
    while (lo + 1 < L && a.kbase[lo + 1] <= k) ++lo;
    a.ev_level[e] = XSP_LEVEL_KERNEL;
    a.ev_layer[e] = lo;
    a.ev_kernel[e] = k - a.kbase[lo];
  }
}

// event_latencies (leveled.cpp:98-122): trimmed mean over the runs of the set
// that contain the event; NaN when no run does (or the set lacks the level).
__global__ void k_lev_latency(LevArgs a) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= a.S * a.n_events) return;
  const uint32_t s = q / a.n_events, e = q % a.n_events;
  const uint8_t lv = a.ev_level[e];
  const uint32_t mask = a.lv[s];
  double v[kMaxRunsL];
  uint32_t n = 0;
  const bool set_has = lv == XSP_LEVEL_MODEL ||
                       (has_level(mask, XSP_LEVEL_LAYER) &&
                        (lv == XSP_LEVEL_LAYER || has_level(mask, XSP_LEVEL_KERNEL)));
  // every run of the set that holds the event, in run order
  auto each = [&](auto fn) {
    const uint32_t li = a.ev_layer[e], ki = a.ev_kernel[e];
    for (uint32_t q = a.soff[s]; q < a.soff[s + 1]; ++q) {
      const uint32_t t = a.tr[q];
      if (lv == XSP_LEVEL_MODEL) {
        const uint32_t m = a.model_row[t];
        fn((double)clamp_dur(a.begin[m], a.end[m]));
        continue;
      }
      const uint32_t l0 = a.t_layer_off[t];
      if (li >= a.t_layer_off[t + 1] - l0) continue;
      if (lv == XSP_LEVEL_LAYER) {
        fn((double)a.layer_dur[l0 + li]);
      } else {
        const uint32_t g = l0 + li;
        if (ki >= a.l_koff[g + 1] - a.l_koff[g]) continue;
        fn((double)a.kernel_dur[a.l_koff[g] + ki]);
      }
    }
  };
  if (set_has) {
    each([&](double x) {
      if (n < kMaxRunsL) v[n] = x;
      ++n;
    });
  }
  // more than kMaxRunsL samples: selection over the runs instead of a sort
  a.lat[q] = !n ? nan("") : n <= kMaxRunsL ? trimmed_mean_l(v, n, a.trim) : trimmed_mean_select(each, n, a.trim);
}

// per chain step: overhead = wide - narrow with the clamp rule (:182-203); the
// accurate latency from the set whose deepest rank is the event's (:164-171).
__global__ void k_lev_steps(LevArgs a) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.n_events) return;
  const int er = level_rank(a.ev_level[e]);
  double acc = nan("");
  for (uint32_t s = 0; s < a.S; ++s) {
    int deepest = 0;
    for (uint32_t l = 0; l < 4; ++l)
      if (has_level(a.lv[s], l)) deepest = max(deepest, level_rank(l));
    const double x = a.lat[(uint64_t)s * a.n_events + e];
    if (deepest == er && !isnan(x)) acc = x;
  }
  a.accurate[e] = acc;
  for (uint32_t s = 0; s + 1 < a.S; ++s) {
    const double before = a.lat[(uint64_t)s * a.n_events + e];
    const double after = a.lat[(uint64_t)(s + 1) * a.n_events + e];
    uint8_t fl = 0;
    double ov = nan("");
    if (!isnan(before)) fl |= XSP_EV_IN_NARROW;
    if (!isnan(after)) fl |= XSP_EV_IN_WIDE;
    if ((fl & XSP_EV_IN_NARROW) && (fl & XSP_EV_IN_WIDE)) {
      ov = __dsub_rn(after, before);
      if (ov < 0.0) {
        if (-ov <= __dmul_rn(a.noise, before)) {
          ov = 0.0;
          fl |= XSP_EV_CLAMPED;
        } else {
          fl |= XSP_EV_NEGATIVE;
        }
      }
    }
    a.overhead[(uint64_t)s * a.n_events + e] = ov;
    a.step_flags[(uint64_t)s * a.n_events + e] = fl;
  }
}

namespace {
template <typename K, typename... Args>
void launch(xsp_ctx* ctx, K kernel, uint64_t n, cudaStream_t st, Args... args) {
  if (n == 0) return;
  kernel<<<ceil_div(n, 256), 256, 0, st>>>(args...);
  ++ctx->launches;
}

// std::set<Level> ordering (lexicographic over ascending elements)
bool levelset_less(uint32_t a, uint32_t b) {
  for (uint32_t l = 0; l < 4; ++l) {
    const bool ia = (a >> l) & 1u, ib = (b >> l) & 1u;
    if (ia == ib) continue;
    // first difference: the set holding l is smaller unless the other one ends here
    return ia ? (b >> (l + 1)) != 0 : (a >> (l + 1)) == 0;
  }
  return false;
}
}  // namespace

void run_leveled(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_corr_out* corr, const xsp_level_sets* sets,
                 const xsp_analysis_opts* opts, xsp_overhead_out* out, cudaStream_t st) {
  const uint32_t NS = sets->n_sets;
  out->status = XSP_L_OK;
  out->err_a = out->err_b = 0;
  // traces must have correlated without ambiguity (LeveledRunGroup::add, :69-75)
  {
    const uint32_t T = corr->n_traces;
    std::vector<int32_t> status(T);
    std::vector<uint32_t> amb(T + 1);
    XSP_CUDA(cudaMemcpyAsync(status.data(), corr->trace_status, T * 4ull, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaMemcpyAsync(amb.data(), corr->trace_amb_off, (T + 1) * 4ull, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaStreamSynchronize(st));
    std::vector<uint32_t> traces(sets->trace_idx, sets->trace_idx + sets->set_off[NS]);
    std::sort(traces.begin(), traces.end());
    for (uint32_t t : traces) {
      if (t >= T) throw std::invalid_argument("level set references a trace beyond the correlation");
      if (status[t] != XSP_T_OK) {
        out->status = XSP_L_TRACE_FAILED;
        out->err_a = t;
        return;
      }
      if (amb[t + 1] != amb[t]) {
        out->status = XSP_L_AMBIGUOUS;
        out->err_a = t;
        return;
      }
    }
  }
  // chain_of (:124-141): map order (std::set<Level> lexicographic), then by size
  std::vector<uint32_t> order(NS);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
    return levelset_less(sets->levels[x], sets->levels[y]);
  });
  std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
    return __builtin_popcount(sets->levels[x]) < __builtin_popcount(sets->levels[y]);
  });
  static thread_local std::vector<uint32_t> chain;
  chain = order;
  out->chain = chain.data();
  out->n_sets = NS;
  for (uint32_t i = 1; i < NS; ++i) {
    const uint32_t narrow = sets->levels[order[i - 1]], wide = sets->levels[order[i]];
    if (narrow & ~wide) {
      // reported, but per-set latencies are still computed (accurate_latency)
      if (out->status == XSP_L_OK) {
        out->status = XSP_L_NOT_CHAIN;
        out->err_a = order[i - 1];
        out->err_b = order[i];
      }
    }
  }
  if (NS < 2 && out->status == XSP_L_OK) {
    out->status = XSP_L_TOO_FEW;
    out->err_a = NS;
  }
  if (NS == 0) return;
  const uint32_t total_runs = sets->set_off[NS];
  uint32_t* hs = ctx->h<uint32_t>("l.sets_h", 2ull * NS + 2 + total_runs);
  uint32_t* htr = hs + 2 * NS + 1;
  uint32_t q = 0;
  for (uint32_t i = 0; i < NS; ++i) {
    const uint32_t s = order[i];
    hs[i] = q;                      // soff
    hs[NS + 1 + i] = sets->levels[s];
    for (uint32_t k = sets->set_off[s]; k < sets->set_off[s + 1]; ++k) htr[q++] = sets->trace_idx[k];
  }
  hs[NS] = q;
  uint32_t* ds = ctx->d<uint32_t>("l.sets", 2ull * NS + 2 + total_runs);
  XSP_CUDA(cudaMemcpyAsync(ds, hs, (2ull * NS + 1 + total_runs) * 4, cudaMemcpyHostToDevice, st));
  LevArgs a;
  a.S = NS;
  a.soff = ds;
  a.lv = ds + NS + 1;
  a.tr = ds + 2 * NS + 1;
  a.t_layer_off = corr->trace_layer_off;
  a.t_kernel_off = corr->trace_kernel_off;
  a.l_koff = corr->layer_kernel_off;
  a.layer_dur = corr->layer_dur;
  a.kernel_dur = corr->kernel_dur;
  a.model_row = corr->trace_model_row;
  a.begin = c->begin_ns;
  a.end = c->end_ns;
  a.trim = opts->trim_fraction;
  a.noise = opts->noise_tolerance;
  a.lmax = ctx->d<uint32_t>("l.lmax", 1);
  XSP_CUDA(cudaMemsetAsync(a.lmax, 0, 4, st));
  launch(ctx, k_lev_layers, total_runs, st, a, total_runs);
  uint32_t* hl = ctx->h<uint32_t>("l.lmax_h", 4);
  XSP_CUDA(cudaMemcpyAsync(hl, a.lmax, 4, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  const uint32_t L = hl[0];
  a.kmax = ctx->d<uint32_t>("l.kmax", L + 1);
  a.kbase = ctx->d<uint32_t>("l.kbase", L + 1);
  XSP_CUDA(cudaMemsetAsync(a.kmax, 0, (L + 1) * 4ull, st));
  if (total_runs) {
    k_lev_kernels<<<total_runs, 256, 0, st>>>(a, total_runs);
    ++ctx->launches;
  }
  uint32_t* scan_tmp = ctx->d<uint32_t>("l.scan", scan_scratch_elems(L + 16));
  exclusive_scan<uint32_t, uint32_t>(a.kmax, a.kbase, L, scan_tmp, a.kbase + L, st, &ctx->launches);
  XSP_CUDA(cudaMemcpyAsync(hl + 1, a.kbase + L, 4, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  const uint32_t NK = L ? hl[1] : 0;
  const uint32_t NE = 1 + L + NK;
  a.n_events = NE;
  out->n_events = NE;
  out->ev_level = a.ev_level = ctx->d<uint8_t>("l.ev_level", NE);
  out->ev_layer = a.ev_layer = ctx->d<uint32_t>("l.ev_layer", NE);
  out->ev_kernel = a.ev_kernel = ctx->d<uint32_t>("l.ev_kernel", NE);
  out->lat = a.lat = ctx->d<double>("l.lat", (uint64_t)NS * NE);
  out->overhead = a.overhead = ctx->d<double>("l.ov", (uint64_t)(NS - 1) * NE);
  out->step_flags = a.step_flags = ctx->d<uint8_t>("l.flags", (uint64_t)(NS - 1) * NE);
  out->accurate = a.accurate = ctx->d<double>("l.acc", NE);
  ctx->stage_begin("leveled", st);
  launch(ctx, k_lev_keys, NE, st, a);
  launch(ctx, k_lev_latency, (uint64_t)NS * NE, st, a);
  launch(ctx, k_lev_steps, NE, st, a);
  ctx->stage_end("leveled", st);
}

}  // namespace xsp
