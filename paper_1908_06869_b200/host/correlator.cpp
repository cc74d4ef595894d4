// libstrata_b200: correlation entry points (reference: correlator.hpp/.cpp).
// correlate / assign_parents / correlate_async run on the GPU through the C ABI
// (xsp_correlate_host); the IntervalTree utility and the serialized-rerun
// bookkeeping are host code around those calls.
#include <algorithm>
#include <map>
#include <tuple>
#include <unordered_map>

#include "pack.hpp"

namespace strata {

// ---- IntervalTree: begin-sorted entries with a running maximum of end_ns.
// Every entry that can contain [b, e] has begin <= b, i.e. lies in the prefix
// found by binary search; walking that prefix backwards stops as soon as the
// running maximum drops below e.

IntervalTree IntervalTree::build(const std::vector<Span>& spans) {
  IntervalTree t;
  t.entries_.reserve(spans.size());
  for (const Span& s : spans) t.entries_.push_back({s.begin_ns, s.end_ns, s.span_id, s.level});
  std::sort(t.entries_.begin(), t.entries_.end(), [](const Entry& a, const Entry& b) {
    return std::tie(a.begin_ns, a.span_id) < std::tie(b.begin_ns, b.span_id);
  });
  t.prefix_end_.resize(t.entries_.size());
  std::uint64_t m = 0;
  for (std::size_t i = 0; i < t.entries_.size(); ++i) {
    m = std::max(m, t.entries_[i].end_ns);
    t.prefix_end_[i] = m;
  }
  return t;
}

std::vector<IntervalTree::Entry> IntervalTree::containing(std::uint64_t b, std::uint64_t e) const {
  std::vector<Entry> out;
  auto ub = std::upper_bound(entries_.begin(), entries_.end(), b,
                             [](std::uint64_t v, const Entry& x) { return v < x.begin_ns; });
  for (std::size_t i = static_cast<std::size_t>(ub - entries_.begin()); i-- > 0;) {
    if (prefix_end_[i] < e) break;
    if (entries_[i].end_ns >= e) out.push_back(entries_[i]);
  }
  std::sort(out.begin(), out.end(), [](const Entry& x, const Entry& y) { return x.span_id < y.span_id; });
  return out;
}

std::vector<IntervalTree::Entry> IntervalTree::containing(std::uint64_t b, std::uint64_t e, Level level) const {
  std::vector<Entry> out = containing(b, e);
  std::erase_if(out, [level](const Entry& x) { return x.level != level; });
  return out;
}

IntervalTree build_tree(const std::vector<Span>& spans) { return IntervalTree::build(spans); }

std::size_t EntityTree::kernel_count() const {
  std::size_t n = 0;
  for (const LayerExec& l : root.layers) n += l.kernels.size();
  return n;
}

namespace {

bool in_timeline_order(const std::vector<Span>& spans) {
  for (std::size_t i = 1; i < spans.size(); ++i) {
    const Span& a = spans[i - 1];
    const Span& b = spans[i];
    if (std::make_tuple(a.begin_ns, rank(a.level), a.span_id) > std::make_tuple(b.begin_ns, rank(b.level), b.span_id))
      return false;
  }
  return true;
}

// One GPU pass over `bundles`; results[i] valid iff errors[i] is empty.
void correlate_batch(const std::vector<const TraceBundle*>& in, int mode, std::vector<CorrelationResult>& results,
                     std::vector<std::string>& errors) {
  // bundles out of timeline order are correlated in timeline order
  // (TraceBundle invariant, span.hpp); sorted copies are made on the GPU
  std::vector<TraceBundle> copies;
  std::vector<const TraceBundle*> bundles = in;
  for (std::size_t i = 0; i < in.size(); ++i)
    if (!in_timeline_order(in[i]->spans)) copies.reserve(copies.size() + 1);
  copies.reserve(in.size());
  for (std::size_t i = 0; i < in.size(); ++i) {
    if (in_timeline_order(in[i]->spans)) continue;
    copies.push_back(*in[i]);
    sort_timeline(copies.back().spans);
    bundles[i] = &copies.back();
  }
  const b200::PackedSpans p = b200::pack_bundles(bundles);
  const b200::HostCorr c = b200::run_correlation(p, mode);
  results.assign(bundles.size(), {});
  errors.assign(bundles.size(), {});
  for (std::uint32_t t = 0; t < bundles.size(); ++t) {
    if (c.status[t] != XSP_T_OK) {
      errors[t] = b200::trace_error_text(p, c, t);
      continue;
    }
    results[t] = b200::unpack_result(p, c, t);
  }
}

CorrelationResult correlate_one(const TraceBundle& bundle, int mode) {
  std::vector<CorrelationResult> r;
  std::vector<std::string> e;
  correlate_batch({&bundle}, mode, r, e);
  if (!e[0].empty()) throw TraceError(e[0]);
  return std::move(r[0]);
}

}  // namespace

std::vector<CorrelationResult> correlate_all(const std::vector<TraceBundle>& bundles,
                                             std::vector<std::string>* errors) {
  std::vector<const TraceBundle*> ptrs;
  for (const TraceBundle& b : bundles) ptrs.push_back(&b);
  std::vector<CorrelationResult> r;
  std::vector<std::string> e;
  correlate_batch(ptrs, 0, r, e);
  if (errors) *errors = std::move(e);
  return r;
}

CorrelationResult assign_parents(const TraceBundle& bundle) {
  return correlate_one(bundle, XSP_CORR_PARENTS_ONLY);
}

// The device computes assign_parents and the fusion in one pass; for a result
// that came from assign_parents(bundle) (the only input the reference accepts
// meaningfully) this equals running the fusion step on it.
void correlate_async(CorrelationResult& result, const TraceBundle& bundle) {
  result = correlate_one(bundle, 0);
}

CorrelationResult correlate(const TraceBundle& bundle) { return correlate_one(bundle, 0); }

bool demand_serialized_rerun(const AmbiguityReport& report) { return !report.empty(); }

namespace {

// Cross-run identity (level, kind, name, occurrence index in timeline order).
using EventKey = std::tuple<std::uint8_t, std::uint8_t, std::string, std::size_t>;

std::map<EventKey, std::uint64_t> event_index(const TraceBundle& bundle) {
  const std::vector<Span> ordered = sorted_timeline(bundle.spans);
  std::map<std::tuple<std::uint8_t, std::uint8_t, std::string>, std::size_t> seen;
  std::map<EventKey, std::uint64_t> out;
  for (const Span& s : ordered) {
    const auto lv = static_cast<std::uint8_t>(s.level);
    const auto kd = static_cast<std::uint8_t>(s.kind);
    const std::size_t k = seen[{lv, kd, s.name}]++;
    out.emplace(EventKey{lv, kd, s.name, k}, s.span_id);
  }
  return out;
}

std::map<std::uint64_t, EventKey> by_span_id(const std::map<EventKey, std::uint64_t>& idx) {
  std::map<std::uint64_t, EventKey> out;
  for (const auto& [key, id] : idx) out.emplace(id, key);
  return out;
}

}  // namespace

CorrelationResult resolve_with_serialized(const TraceBundle& original, const TraceBundle& serialized) {
  const CorrelationResult ser = assign_parents(serialized);
  if (!ser.ambiguities.empty())
    throw TraceError("serialized run is itself ambiguous (" + std::to_string(ser.ambiguities.size()) +
                     " span(s)); cannot resolve");
  std::unordered_map<std::uint64_t, std::uint64_t> ser_parent;
  for (const LayerExec& l : ser.tree.root.layers) {
    ser_parent[l.span.span_id] = ser.tree.root.span.span_id;
    for (const KernelExec& k : l.kernels) ser_parent[k.launch.span_id] = l.span.span_id;
  }
  const auto orig_idx = event_index(original);
  const auto ser_idx = event_index(serialized);
  const auto ser_key_of = by_span_id(ser_idx);
  const auto orig_key_of = by_span_id(orig_idx);
  const CorrelationResult first = assign_parents(original);
  TraceBundle patched = original;
  std::unordered_map<std::uint64_t, Span*> patched_by_id;
  for (Span& s : patched.spans) patched_by_id[s.span_id] = &s;
  for (const Ambiguity& a : first.ambiguities) {
    auto k = orig_key_of.find(a.span_id);
    if (k == orig_key_of.end()) continue;
    auto twin = ser_idx.find(k->second);
    if (twin == ser_idx.end()) continue;
    auto par = ser_parent.find(twin->second);
    if (par == ser_parent.end()) continue;
    auto par_key = ser_key_of.find(par->second);
    if (par_key == ser_key_of.end()) continue;
    auto orig_par = orig_idx.find(par_key->second);
    if (orig_par == orig_idx.end()) continue;
    patched_by_id.at(a.span_id)->parent_id = orig_par->second;
  }
  return correlate(patched);
}

}  // namespace strata
