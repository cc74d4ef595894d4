// libstrata_b200: leveled experimentation (reference: leveled.hpp / leveled.cpp).
// Event latencies per level set, step differences and the clamp rule run on the
// GPU (xsp_leveled_host); this file files runs, rebuilds the report's maps and
// warnings, and raises the reference's errors.
#include <algorithm>
#include <cmath>
#include <iterator>
#include <tuple>

#include "pack.hpp"
#include "strata/leveled.hpp"

namespace strata {

char level_letter(Level level) {
  switch (level) {
    case Level::Model: return 'M';
    case Level::Layer: return 'L';
    case Level::Kernel: return 'G';
    case Level::Api: return 'A';
  }
  return '?';
}

std::string level_set_label(const LevelSet& levels) {
  std::string s;
  for (Level l : levels) {
    if (!s.empty()) s += '+';
    s += level_letter(l);
  }
  return s;
}

std::string event_label(const LeveledEventKey& key) {
  if (key.level == Level::Model) return "model";
  if (key.level == Level::Layer) return "layer " + std::to_string(key.layer_index);
  return "layer " + std::to_string(key.layer_index) + " kernel " + std::to_string(key.kernel_index);
}

void LeveledRunGroup::add(const TraceBundle& bundle) {
  if (runs.empty()) {
    batch_size = bundle.meta.batch_size;
    system = bundle.meta.system;
  } else {
    if (bundle.meta.batch_size != batch_size)
      throw LeveledError("runs mix batch sizes " + std::to_string(batch_size) + " and " +
                         std::to_string(bundle.meta.batch_size));
    if (!(bundle.meta.system == system)) throw LeveledError("runs mix system specifications");
  }
  CorrelationResult r = correlate(bundle);
  if (!r.ambiguities.empty())
    throw LeveledError("trace " + std::to_string(bundle.meta.trace_id) + " has " +
                       std::to_string(r.ambiguities.size()) +
                       " ambiguous span(s); resolve with a serialized rerun before leveling");
  runs[bundle.meta.profiling_levels].push_back(std::move(r.tree));
}

LeveledRunGroup LeveledRunGroup::from_bundles(const std::vector<TraceBundle>& bundles) {
  LeveledRunGroup g;
  for (const TraceBundle& b : bundles) g.add(b);
  return g;
}

namespace {

int deepest_rank(const LevelSet& levels) {
  int d = 0;
  for (Level l : levels) d = std::max(d, rank(l));
  return d;
}

template <typename T>
std::vector<T> take(const T* src, std::size_t n) {
  return src ? std::vector<T>(src, src + n) : std::vector<T>(n);
}

// Device pass over every level set of the group (sets in map order).
struct LevelLatencies {
  std::vector<LevelSet> sets;     // map order
  std::int32_t status = 0;
  std::uint32_t err_a = 0, err_b = 0;
  std::vector<std::uint32_t> chain;  // chain position -> set index
  std::vector<LeveledEventKey> events;
  std::vector<double> lat, overhead, accurate;  // [S][E], [S-1][E], [E]
  std::vector<std::uint8_t> flags;              // [S-1][E]
  std::size_t E = 0;
};

LevelLatencies run_leveled(const LeveledRunGroup& group, const AnalysisOptions& options) {
  LevelLatencies r;
  std::vector<const EntityTree*> trees;
  std::vector<std::uint32_t> set_off{0}, idx, masks;
  for (const auto& [levels, ts] : group.runs) {
    r.sets.push_back(levels);
    masks.push_back(b200::level_mask(levels));
    for (const EntityTree& t : ts) {
      idx.push_back(static_cast<std::uint32_t>(trees.size()));
      trees.push_back(&t);
    }
    set_off.push_back(static_cast<std::uint32_t>(idx.size()));
  }
  const b200::PackedTrees p = b200::pack_trees(trees);
  const xsp_span_cols cols = p.cols();
  const xsp_corr_out corr = p.corr();
  xsp_level_sets ls;
  ls.n_sets = static_cast<std::uint32_t>(r.sets.size());
  ls.set_off = set_off.data();
  ls.trace_idx = idx.data();
  ls.levels = masks.data();
  xsp_analysis_opts o{options.trim_fraction, options.epsilon, options.noise_tolerance, 0};
  xsp_overhead_out out;
  b200::check(xsp_leveled_host(b200::ctx(), &cols, &corr, &ls, &o, &out));
  r.status = out.status;
  r.err_a = out.err_a;
  r.err_b = out.err_b;
  const std::size_t S = out.n_sets, E = out.n_events;
  r.E = E;
  if (S == 0) return r;
  r.chain = take(out.chain, S);
  const auto lev = take(out.ev_level, E);
  const auto lay = take(out.ev_layer, E);
  const auto ker = take(out.ev_kernel, E);
  for (std::size_t e = 0; e < E; ++e) r.events.push_back({static_cast<Level>(lev[e]), lay[e], ker[e]});
  r.lat = take(out.lat, S * E);
  r.overhead = take(out.overhead, (S - 1) * E);
  r.flags = take(out.step_flags, (S - 1) * E);
  r.accurate = take(out.accurate, E);
  return r;
}

LevelSet difference(const LevelSet& wide, const LevelSet& narrow) {
  LevelSet d;
  std::set_difference(wide.begin(), wide.end(), narrow.begin(), narrow.end(), std::inserter(d, d.begin()));
  return d;
}

}  // namespace

OverheadReport compute_overhead(const LeveledRunGroup& group, const AnalysisOptions& options) {
  const LevelLatencies L = run_leveled(group, options);
  if (L.status == XSP_L_NOT_CHAIN)
    throw LeveledError("profiling-level sets " + level_set_label(L.sets[L.err_a]) + " and " +
                       level_set_label(L.sets[L.err_b]) + " do not form an inclusion chain");
  if (L.status == XSP_L_TOO_FEW)
    throw LeveledError("overhead needs at least two chained level sets; got " + std::to_string(L.sets.size()));
  if (L.status != XSP_L_OK) throw LeveledError("leveled run group could not be evaluated");
  const std::size_t S = L.chain.size(), E = L.E;
  OverheadReport rep;
  rep.noise_tolerance = options.noise_tolerance;
  rep.rows.resize(E);
  for (std::size_t e = 0; e < E; ++e) {
    rep.rows[e].event = L.events[e];
    if (!std::isnan(L.accurate[e])) rep.rows[e].accurate_latency_ns = L.accurate[e];
  }
  for (std::size_t s = 0; s + 1 < S; ++s) {
    const LevelSet& narrow = L.sets[L.chain[s]];
    const LevelSet& wide = L.sets[L.chain[s + 1]];
    const LevelSet added = difference(wide, narrow);
    for (std::size_t e = 0; e < E; ++e) {
      const std::uint8_t f = L.flags[s * E + e];
      if (!(f & XSP_EV_IN_NARROW)) continue;
      if (!(f & XSP_EV_IN_WIDE)) {
        rep.warnings.push_back(event_label(L.events[e]) + " visible under " + level_set_label(narrow) +
                               " but not under " + level_set_label(wide));
        continue;
      }
      if (f & XSP_EV_CLAMPED) rep.rows[e].clamped = true;
      if (f & XSP_EV_NEGATIVE)
        rep.warnings.push_back(event_label(L.events[e]) + ": overhead of added level(s) " + level_set_label(added) +
                               " is negative beyond noise tolerance");
      rep.rows[e].overhead_by_added_levels[added] = L.overhead[s * E + e];
    }
    const int dn = deepest_rank(narrow);
    for (std::size_t e = 0; e < E; ++e) {
      const std::uint8_t f = L.flags[s * E + e];
      if ((f & XSP_EV_IN_WIDE) && !(f & XSP_EV_IN_NARROW) && rank(L.events[e].level) <= dn)
        rep.warnings.push_back(event_label(L.events[e]) + " visible under " + level_set_label(wide) +
                               " but not under " + level_set_label(narrow));
    }
  }
  for (const OverheadRow& row : rep.rows)
    if (row.event.level == Level::Model) {
      rep.model_overhead_by_added_levels = row.overhead_by_added_levels;
      break;
    }
  return rep;
}

double accurate_latency(const LeveledRunGroup& group, const LeveledEventKey& event, const AnalysisOptions& options) {
  const LevelLatencies L = run_leveled(group, options);
  for (std::size_t set = 0; set < L.sets.size(); ++set) {
    if (deepest_rank(L.sets[set]) != rank(event.level)) continue;
    const std::size_t pos = static_cast<std::size_t>(std::find(L.chain.begin(), L.chain.end(), set) - L.chain.begin());
    auto it = std::lower_bound(L.events.begin(), L.events.end(), event,
                               [](const LeveledEventKey& a, const LeveledEventKey& b) {
                                 return std::tuple(rank(a.level), a.layer_index, a.kernel_index) <
                                        std::tuple(rank(b.level), b.layer_index, b.kernel_index);
                               });
    const bool found = it != L.events.end() && *it == event;
    const double v = found ? L.lat[pos * L.E + static_cast<std::size_t>(it - L.events.begin())] : std::nan("");
    if (std::isnan(v))
      throw LeveledError(event_label(event) + " not present in the " + level_set_label(L.sets[set]) + " run");
    return v;
  }
  throw LeveledError("no run has " + std::string(1, level_letter(event.level)) + " as its deepest profiling level");
}

}  // namespace strata
