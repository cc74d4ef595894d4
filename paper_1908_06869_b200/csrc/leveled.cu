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
// Many groups (one LeveledRunGroup per model) go through one batch: every kernel
// covers all groups' runs / events (group found by binary search over offsets),
// so a batch costs three host round trips, not three per group.
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

// Per-group views over the batch: sets in chain order, concatenated over groups.
struct LevBatch {
  uint32_t G;                  // groups with outputs
  const uint32_t* g_set0;      // [G + 1] first set of each group
  const uint32_t* set_soff;    // [NS + 1] run offsets of the sets
  const uint32_t* set_lv;      // [NS] level masks
  const uint32_t* set_group;   // [NS]
  const uint32_t* run_tr;      // [R] trace of each run
  const uint32_t* run_set;     // [R] set of each run
  const uint32_t* t_layer_off;
  const uint32_t* t_kernel_off;
  const uint32_t* l_koff;
  const uint64_t* layer_dur;
  const uint64_t* kernel_dur;
  const uint32_t* model_row;
  const uint64_t* begin;
  const uint64_t* end;
  uint32_t* lmax;              // [G] max layer count over the group's sets with L
  const uint32_t* koff;        // [G + 1] offsets of the groups' kmax rows (L_g + 1 each)
  uint32_t* kmax;              // per group, per layer index: max kernel count over sets with L and G
  uint32_t* kbase;             // exclusive scan of kmax over the whole batch
  uint32_t* nk;                // [G] kernel events of each group
  const uint64_t* ev_base;     // [G + 1] event offsets
  const uint64_t* lat_base;    // [G + 1] offsets of the (set, event) latencies
  const uint64_t* ov_base;     // [G + 1] offsets of the (step, event) overheads
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

// largest g with off[g] <= q (off ascending, off[0] = 0)
template <typename T>
__device__ __forceinline__ uint32_t seg_of(const T* __restrict__ off, uint32_t G, uint64_t q) {
  uint32_t lo = 0, hi = G;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((uint64_t)off[mid] <= q) lo = mid; else hi = mid;
  }
  return lo;
}

// universe of layer events: max layer count over the traces of sets with L
__global__ void k_lev_layers(LevBatch a, uint32_t total_runs) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= total_runs) return;
  const uint32_t s = a.run_set[q];
  if (!has_level(a.set_lv[s], XSP_LEVEL_LAYER)) return;
  const uint32_t t = a.run_tr[q];
  atomicMax(a.lmax + a.set_group[s], a.t_layer_off[t + 1] - a.t_layer_off[t]);
}

// universe of kernel events: per layer index, max kernel count over sets with L and G
__global__ void k_lev_kernels(LevBatch a, uint32_t total_runs) {
  const uint32_t q = blockIdx.x;  // one block per run
  if (q >= total_runs) return;
  const uint32_t s = a.run_set[q];
  if (!has_level(a.set_lv[s], XSP_LEVEL_LAYER) || !has_level(a.set_lv[s], XSP_LEVEL_KERNEL)) return;
  uint32_t* km = a.kmax + a.koff[a.set_group[s]];
  const uint32_t t = a.run_tr[q];
  const uint32_t l0 = a.t_layer_off[t], l1 = a.t_layer_off[t + 1];
  for (uint32_t g = l0 + threadIdx.x; g < l1; g += blockDim.x)
    atomicMax(km + (g - l0), a.l_koff[g + 1] - a.l_koff[g]);
}

// kernel events of each group (its kmax rows' total)
__global__ void k_lev_nk(LevBatch a) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.G) return;
  const uint32_t L = a.lmax[g], k0 = a.koff[g];
  a.nk[g] = L ? a.kbase[k0 + L] - a.kbase[k0] : 0;
}

// event keys in (rank, layer_index, kernel_index) order
__global__ void k_lev_keys(LevBatch a, uint64_t total_events) {
  const uint64_t eg = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (eg >= total_events) return;
  const uint32_t grp = seg_of(a.ev_base, a.G, eg);
  const uint32_t e = (uint32_t)(eg - a.ev_base[grp]);
  const uint32_t L = a.lmax[grp];
  const uint32_t* kb = a.kbase + a.koff[grp];
  if (e == 0) {
    a.ev_level[eg] = XSP_LEVEL_MODEL;
    a.ev_layer[eg] = 0;
    a.ev_kernel[eg] = 0;
  } else if (e <= L) {
    a.ev_level[eg] = XSP_LEVEL_LAYER;
    a.ev_layer[eg] = e - 1;
    a.ev_kernel[eg] = 0;
  } else {
    const uint32_t k = e - 1 - L + kb[0];  // in the batch-wide scan
    uint32_t lo = 0, hi = L;  // kb[lo] <= k < kb[lo + 1]
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (kb[mid] <= k) lo = mid; else hi = mid;
    }
    while (lo + 1 < L && kb[lo + 1] <= k) ++lo;
    a.ev_level[eg] = XSP_LEVEL_KERNEL;
    a.ev_layer[eg] = lo;
    a.ev_kernel[eg] = k - kb[lo];
  }
}

// event_latencies (leveled.cpp:98-122): trimmed mean over the runs of the set
// that contain the event; NaN when no run does (or the set lacks the level).
__global__ void k_lev_latency(LevBatch a, uint64_t total) {
  const uint64_t qg = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (qg >= total) return;
  const uint32_t grp = seg_of(a.lat_base, a.G, qg);
  const uint64_t ne = a.ev_base[grp + 1] - a.ev_base[grp];
  const uint64_t ql = qg - a.lat_base[grp];
  const uint32_t s = a.g_set0[grp] + (uint32_t)(ql / ne);
  const uint64_t eg = a.ev_base[grp] + ql % ne;
  const uint8_t lv = a.ev_level[eg];
  const uint32_t mask = a.set_lv[s];
  double v[kMaxRunsL];
  uint32_t n = 0;
  const bool set_has = lv == XSP_LEVEL_MODEL ||
                       (has_level(mask, XSP_LEVEL_LAYER) &&
                        (lv == XSP_LEVEL_LAYER || has_level(mask, XSP_LEVEL_KERNEL)));
  // every run of the set that holds the event, in run order
  auto each = [&](auto fn) {
    const uint32_t li = a.ev_layer[eg], ki = a.ev_kernel[eg];
    for (uint32_t q = a.set_soff[s]; q < a.set_soff[s + 1]; ++q) {
      const uint32_t t = a.run_tr[q];
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
  a.lat[qg] = !n ? nan("") : n <= kMaxRunsL ? trimmed_mean_l(v, n, a.trim) : trimmed_mean_select(each, n, a.trim);
}

// per chain step: overhead = wide - narrow with the clamp rule (:182-203); the
// accurate latency from the set whose deepest rank is the event's (:164-171).
__global__ void k_lev_steps(LevBatch a, uint64_t total_events) {
  const uint64_t eg = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (eg >= total_events) return;
  const uint32_t grp = seg_of(a.ev_base, a.G, eg);
  const uint64_t ne = a.ev_base[grp + 1] - a.ev_base[grp], e = eg - a.ev_base[grp];
  const uint32_t s0 = a.g_set0[grp], S = a.g_set0[grp + 1] - s0;
  const double* lat = a.lat + a.lat_base[grp];
  const int er = level_rank(a.ev_level[eg]);
  double acc = nan("");
  for (uint32_t s = 0; s < S; ++s) {
    int deepest = 0;
    for (uint32_t l = 0; l < 4; ++l)
      if (has_level(a.set_lv[s0 + s], l)) deepest = max(deepest, level_rank(l));
    const double x = lat[(uint64_t)s * ne + e];
    if (deepest == er && !isnan(x)) acc = x;
  }
  a.accurate[eg] = acc;
  for (uint32_t s = 0; s + 1 < S; ++s) {
    const double before = lat[(uint64_t)s * ne + e];
    const double after = lat[(uint64_t)(s + 1) * ne + e];
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
    a.overhead[a.ov_base[grp] + (uint64_t)s * ne + e] = ov;
    a.step_flags[a.ov_base[grp] + (uint64_t)s * ne + e] = fl;
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

void run_leveled_batch(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_corr_out* corr, uint32_t n_groups,
                       const xsp_level_sets* sets, const xsp_analysis_opts* opts, xsp_overhead_out* outs,
                       cudaStream_t st) {
  if (!n_groups) return;
  // traces must have correlated without ambiguity (LeveledRunGroup::add, :69-75)
  const uint32_t T = corr->n_traces;
  int32_t* status = ctx->h<int32_t>("l.status_h", T + 1ull);
  uint32_t* amb = ctx->h<uint32_t>("l.amb_h", T + 1ull);
  XSP_CUDA(cudaMemcpyAsync(status, corr->trace_status, T * 4ull, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaMemcpyAsync(amb, corr->trace_amb_off, (T + 1) * 4ull, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  // chain storage (host pointers handed out in outs[g].chain, valid until the next call)
  static thread_local std::vector<std::vector<uint32_t>> chains;
  chains.assign(n_groups, {});
  std::vector<uint32_t> act;  // groups with device outputs
  std::vector<uint32_t> g_set0{0}, set_soff{0}, set_lv, set_group, run_tr, run_set;
  for (uint32_t gi = 0; gi < n_groups; ++gi) {
    const xsp_level_sets* ls = sets + gi;
    xsp_overhead_out* out = outs + gi;
    const uint32_t NS = ls->n_sets;
    out->status = XSP_L_OK;
    out->err_a = out->err_b = 0;
    {
      std::vector<uint32_t> traces(ls->trace_idx, ls->trace_idx + ls->set_off[NS]);
      std::sort(traces.begin(), traces.end());
      bool bad = false;
      for (uint32_t t : traces) {
        if (t >= T) throw std::invalid_argument("level set references a trace beyond the correlation");
        if (status[t] != XSP_T_OK) {
          out->status = XSP_L_TRACE_FAILED;
          out->err_a = t;
          bad = true;
          break;
        }
        if (amb[t + 1] != amb[t]) {
          out->status = XSP_L_AMBIGUOUS;
          out->err_a = t;
          bad = true;
          break;
        }
      }
      if (bad) continue;
    }
    // chain_of (:124-141): map order (std::set<Level> lexicographic), then by size
    std::vector<uint32_t>& order = chains[gi];
    order.resize(NS);
    std::iota(order.begin(), order.end(), 0u);
    std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
      return levelset_less(ls->levels[x], ls->levels[y]);
    });
    std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
      return __builtin_popcount(ls->levels[x]) < __builtin_popcount(ls->levels[y]);
    });
    out->chain = order.data();
    out->n_sets = NS;
    for (uint32_t i = 1; i < NS; ++i) {
      const uint32_t narrow = ls->levels[order[i - 1]], wide = ls->levels[order[i]];
      if ((narrow & ~wide) && out->status == XSP_L_OK) {
        // reported, but per-set latencies are still computed (accurate_latency)
        out->status = XSP_L_NOT_CHAIN;
        out->err_a = order[i - 1];
        out->err_b = order[i];
      }
    }
    if (NS < 2 && out->status == XSP_L_OK) {
      out->status = XSP_L_TOO_FEW;
      out->err_a = NS;
    }
    if (NS == 0) continue;
    const uint32_t g = (uint32_t)act.size();
    act.push_back(gi);
    for (uint32_t i = 0; i < NS; ++i) {
      const uint32_t s = order[i];
      set_lv.push_back(ls->levels[s]);
      set_group.push_back(g);
      for (uint32_t k = ls->set_off[s]; k < ls->set_off[s + 1]; ++k) {
        run_tr.push_back(ls->trace_idx[k]);
        run_set.push_back((uint32_t)set_lv.size() - 1);
      }
      set_soff.push_back((uint32_t)run_tr.size());
    }
    g_set0.push_back((uint32_t)set_lv.size());
  }
  const uint32_t G = (uint32_t)act.size();
  if (!G) return;
  const uint32_t NSall = (uint32_t)set_lv.size(), R = (uint32_t)run_tr.size();
  // one upload: [g_set0 G+1][set_soff NS+1][set_lv NS][set_group NS][run_tr R][run_set R]
  const uint64_t nw = (G + 1ull) + (NSall + 1ull) + 2ull * NSall + 2ull * R;
  uint32_t* hw = ctx->h<uint32_t>("l.batch_h", nw);
  uint32_t* p = hw;
  for (auto* v : {&g_set0, &set_soff, &set_lv, &set_group, &run_tr, &run_set}) {
    std::copy(v->begin(), v->end(), p);
    p += v->size();
  }
  uint32_t* dw = ctx->d<uint32_t>("l.batch", nw);
  XSP_CUDA(cudaMemcpyAsync(dw, hw, nw * 4, cudaMemcpyHostToDevice, st));
  LevBatch a;
  a.G = G;
  a.g_set0 = dw;
  a.set_soff = a.g_set0 + (G + 1);
  a.set_lv = a.set_soff + (NSall + 1);
  a.set_group = a.set_lv + NSall;
  a.run_tr = a.set_group + NSall;
  a.run_set = a.run_tr + R;
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
  a.lmax = ctx->d<uint32_t>("l.lmax", G);
  XSP_CUDA(cudaMemsetAsync(a.lmax, 0, G * 4ull, st));
  launch(ctx, k_lev_layers, R, st, a, R);
  uint32_t* hl = ctx->h<uint32_t>("l.lmax_h", 2ull * G + 2);
  XSP_CUDA(cudaMemcpyAsync(hl, a.lmax, G * 4ull, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  // kmax rows: L_g + 1 per group
  uint32_t* hko = ctx->h<uint32_t>("l.koff_h", G + 1ull);
  hko[0] = 0;
  for (uint32_t g = 0; g < G; ++g) hko[g + 1] = hko[g] + hl[g] + 1;
  const uint32_t KR = hko[G];
  uint32_t* dko = ctx->d<uint32_t>("l.koff", G + 1ull);
  XSP_CUDA(cudaMemcpyAsync(dko, hko, (G + 1ull) * 4, cudaMemcpyHostToDevice, st));
  a.koff = dko;
  a.kmax = ctx->d<uint32_t>("l.kmax", KR + 1ull);
  a.kbase = ctx->d<uint32_t>("l.kbase", KR + 1ull);
  a.nk = ctx->d<uint32_t>("l.nk", G);
  XSP_CUDA(cudaMemsetAsync(a.kmax, 0, (KR + 1ull) * 4, st));
  if (R) {
    k_lev_kernels<<<R, 256, 0, st>>>(a, R);
    ++ctx->launches;
  }
  uint32_t* scan_tmp = ctx->d<uint32_t>("l.scan", scan_scratch_elems(KR + 16));
  exclusive_scan<uint32_t, uint32_t>(a.kmax, a.kbase, KR, scan_tmp, a.kbase + KR, st, &ctx->launches);
  launch(ctx, k_lev_nk, G, st, a);
  XSP_CUDA(cudaMemcpyAsync(hl + G, a.nk, G * 4ull, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  // event / latency / overhead offsets
  uint64_t* hb = ctx->h<uint64_t>("l.bases_h", 3ull * (G + 1));
  uint64_t *hev = hb, *hlat = hb + (G + 1), *hov = hb + 2 * (G + 1);
  hev[0] = hlat[0] = hov[0] = 0;
  for (uint32_t g = 0; g < G; ++g) {
    const uint32_t S = g_set0[g + 1] - g_set0[g];
    const uint64_t NE = 1ull + hl[g] + (hl[g] ? hl[G + g] : 0);
    hev[g + 1] = hev[g] + NE;
    hlat[g + 1] = hlat[g] + S * NE;
    hov[g + 1] = hov[g] + (S - 1) * NE;
  }
  uint64_t* db = ctx->d<uint64_t>("l.bases", 3ull * (G + 1));
  XSP_CUDA(cudaMemcpyAsync(db, hb, 3ull * (G + 1) * 8, cudaMemcpyHostToDevice, st));
  a.ev_base = db;
  a.lat_base = db + (G + 1);
  a.ov_base = db + 2 * (G + 1);
  const uint64_t NEall = hev[G];
  a.ev_level = ctx->d<uint8_t>("l.ev_level", NEall);
  a.ev_layer = ctx->d<uint32_t>("l.ev_layer", NEall);
  a.ev_kernel = ctx->d<uint32_t>("l.ev_kernel", NEall);
  a.lat = ctx->d<double>("l.lat", hlat[G] + 1);
  a.overhead = ctx->d<double>("l.ov", hov[G] + 1);
  a.step_flags = ctx->d<uint8_t>("l.flags", hov[G] + 1);
  a.accurate = ctx->d<double>("l.acc", NEall);
  for (uint32_t g = 0; g < G; ++g) {
    xsp_overhead_out* out = outs + act[g];
    out->n_events = (uint32_t)(hev[g + 1] - hev[g]);
    out->ev_level = a.ev_level + hev[g];
    out->ev_layer = a.ev_layer + hev[g];
    out->ev_kernel = a.ev_kernel + hev[g];
    out->lat = a.lat + hlat[g];
    out->overhead = a.overhead + hov[g];
    out->step_flags = a.step_flags + hov[g];
    out->accurate = a.accurate + hev[g];
  }
  ctx->stage_begin("leveled", st);
  launch(ctx, k_lev_keys, NEall, st, a, NEall);
  launch(ctx, k_lev_latency, hlat[G], st, a, hlat[G]);
  launch(ctx, k_lev_steps, NEall, st, a, NEall);
  ctx->stage_end("leveled", st);
}

void run_leveled(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_corr_out* corr, const xsp_level_sets* sets,
                 const xsp_analysis_opts* opts, xsp_overhead_out* out, cudaStream_t st) {
  run_leveled_batch(ctx, c, corr, 1, sets, opts, out, st);
}

}  // namespace xsp
