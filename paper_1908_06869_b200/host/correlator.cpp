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

// ---- IntervalTree (correlator.cpp:66-126): entries sorted by (begin_ns, span_id),
// an implicit balanced BST over that array (node of [lo, hi) = its midpoint)
// augmented with the subtree maximum of end_ns. A query prunes a subtree whose
// maximum end is below e and the right part of any node that begins after b:
// O(log n + k) per query, as the reference's augmented tree.

IntervalTree IntervalTree::build(const std::vector<Span>& spans) {
  IntervalTree t;
  t.entries_.reserve(spans.size());
  for (const Span& s : spans) t.entries_.push_back({s.begin_ns, s.end_ns, s.span_id, s.level});
  std::sort(t.entries_.begin(), t.entries_.end(), [](const Entry& a, const Entry& b) {
    return std::tie(a.begin_ns, a.span_id) < std::tie(b.begin_ns, b.span_id);
  });
  t.subtree_max_end_.assign(t.entries_.size(), 0);
  t.fill_max(0, t.entries_.size());
  return t;
}

std::uint64_t IntervalTree::fill_max(std::size_t lo, std::size_t hi) {
  if (lo >= hi) return 0;
  const std::size_t mid = lo + (hi - lo) / 2;
  std::uint64_t m = entries_[mid].end_ns;
  m = std::max(m, fill_max(lo, mid));
  m = std::max(m, fill_max(mid + 1, hi));
  subtree_max_end_[mid] = m;
  return m;
}

void IntervalTree::query(std::size_t lo, std::size_t hi, std::uint64_t b, std::uint64_t e,
                         std::vector<Entry>& out) const {
  while (lo < hi) {
    const std::size_t mid = lo + (hi - lo) / 2;
    if (subtree_max_end_[mid] < e) return;  // nothing in [lo, hi) reaches e
    query(lo, mid, b, e, out);
    if (entries_[mid].begin_ns > b) return;  // mid and everything right of it begin after b
    if (entries_[mid].end_ns >= e) out.push_back(entries_[mid]);
    lo = mid + 1;  // right subtree (tail iteration)
  }
}

std::vector<IntervalTree::Entry> IntervalTree::containing(std::uint64_t b, std::uint64_t e) const {
  std::vector<Entry> out;
  query(0, entries_.size(), b, e, out);
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

// Emission phase of an orphan (correlator.cpp:168-363): 0 layer pass, 1 kernel
// pass, 2 execution without cid — these three walk bundle.spans in order —
// then 3 launch fusion (tree order) and 4 leftover executions (by span_id).
int orphan_phase(const std::string& reason) {
  if (reason == "layer-level span with non-sync kind" || reason == "outside the model interval" ||
      reason.ends_with("is not the model span"))
    return 0;
  if (reason == "contained in no layer interval" || reason.ends_with("is not a layer in the tree")) return 1;
  if (reason == "execution record without correlation id") return 2;
  return 3;
}

// A bundle out of timeline order (outside the TraceBundle contract, span.hpp)
// is correlated in timeline order; the reference walks such a bundle in file
// order, which only changes the order of the orphans its span walks emit
// (phases 0-2): those are put back into file order here.
void file_order_orphans(const TraceBundle& original, CorrelationResult& r) {
  std::unordered_map<std::uint64_t, std::size_t> pos;
  for (std::size_t i = original.spans.size(); i-- > 0;) pos[original.spans[i].span_id] = i;
  auto& o = r.tree.orphans;
  std::size_t a = 0;
  while (a < o.size()) {
    const int ph = orphan_phase(o[a].reason);
    std::size_t b = a + 1;
    while (b < o.size() && orphan_phase(o[b].reason) == ph) ++b;
    if (ph < 3)
      std::stable_sort(o.begin() + a, o.begin() + b,
                       [&](const OrphanSpan& x, const OrphanSpan& y) { return pos[x.span_id] < pos[y.span_id]; });
    a = b;
  }
}

// One GPU pass over `bundles`; results[i] valid iff errors[i] is empty.
void correlate_batch(const std::vector<const TraceBundle*>& in, int mode, std::vector<CorrelationResult>& results,
                     std::vector<std::string>& errors) {
  // bundles out of timeline order are correlated in timeline order
  // (TraceBundle invariant, span.hpp); sorted copies are made on the GPU
  std::vector<TraceBundle> copies;
  std::vector<const TraceBundle*> bundles = in;
  std::vector<bool> resorted(in.size(), false);
  copies.reserve(in.size());
  for (std::size_t i = 0; i < in.size(); ++i) {
    if (in_timeline_order(in[i]->spans)) continue;
    copies.push_back(*in[i]);
    sort_timeline(copies.back().spans);
    bundles[i] = &copies.back();
    resorted[i] = true;
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
    if (resorted[t]) file_order_orphans(*in[t], results[t]);
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

namespace {

// Same tree shape and exception lists, compared by span ids (the tree holds
// copies of the bundle's spans).
bool same_parent_assignment(const CorrelationResult& a, const CorrelationResult& b) {
  if (a.tree.root.span.span_id != b.tree.root.span.span_id) return false;
  if (a.tree.root.layers.size() != b.tree.root.layers.size()) return false;
  for (std::size_t i = 0; i < a.tree.root.layers.size(); ++i) {
    const LayerExec& x = a.tree.root.layers[i];
    const LayerExec& y = b.tree.root.layers[i];
    if (x.span.span_id != y.span.span_id || x.layer_index != y.layer_index ||
        x.kernels.size() != y.kernels.size())
      return false;
    for (std::size_t k = 0; k < x.kernels.size(); ++k) {
      if (x.kernels[k].launch.span_id != y.kernels[k].launch.span_id) return false;
      if (x.kernels[k].exec.has_value() != y.kernels[k].exec.has_value()) return false;
    }
  }
  return a.tree.orphans == b.tree.orphans && a.ambiguities == b.ambiguities;
}

}  // namespace

// correlate_async (correlator.cpp:287-364) fuses the launches of `result`'s
// tree with the bundle's execution records. The device computes the parent
// assignment and that fusion in one pass, so the given result must be the
// parent assignment of `bundle` (what assign_parents returns, and the only
// input the reference documents, correlator.hpp:144-146); it is checked, on
// the GPU, against assign_parents(bundle), and a result that was edited after
// assign_parents is rejected with a UsageError instead of being replaced.
void correlate_async(CorrelationResult& result, const TraceBundle& bundle) {
  if (!same_parent_assignment(result, correlate_one(bundle, XSP_CORR_PARENTS_ONLY)))
    throw UsageError("correlate_async: result is not assign_parents(bundle); the B200 drop-in fuses "
                     "unmodified parent assignments only");
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
