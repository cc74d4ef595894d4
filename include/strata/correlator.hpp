// strata correlator — drop-in header of the B200 implementation.
//
// Same API as the reference's correlator.hpp: the IntervalTree index, the
// entity tree (model -> layers -> kernels), orphan/ambiguity diagnostics and
// assign_parents / correlate_async / correlate / resolve_with_serialized.
// correlate() and its two halves run on the GPU (xsp_correlate, include/xsp.h).
#ifndef STRATA_CORRELATOR_HPP
#define STRATA_CORRELATOR_HPP

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "strata/span.hpp"

namespace strata {

// Static containment index over closed intervals.
class IntervalTree {
 public:
  struct Entry {
    std::uint64_t begin_ns = 0;
    std::uint64_t end_ns = 0;
    std::uint64_t span_id = 0;
    Level level = Level::Model;
  };

  IntervalTree() = default;
  static IntervalTree build(const std::vector<Span>& spans);

  // Entries whose interval contains [begin_ns, end_ns] (self included), by span_id.
  std::vector<Entry> containing(std::uint64_t begin_ns, std::uint64_t end_ns) const;
  std::vector<Entry> containing(std::uint64_t begin_ns, std::uint64_t end_ns, Level level) const;

  std::size_t size() const { return entries_.size(); }

 private:
  std::vector<Entry> entries_;  // by (begin_ns, span_id)
  // implicit balanced BST over entries_ (the node of [lo, hi) is mid = (lo + hi) / 2):
  // subtree_max_end_[mid] = max end_ns over [lo, hi)
  std::vector<std::uint64_t> subtree_max_end_;
  std::uint64_t fill_max(std::size_t lo, std::size_t hi);
  void query(std::size_t lo, std::size_t hi, std::uint64_t b, std::uint64_t e, std::vector<Entry>& out) const;
};

struct KernelExec {
  Span launch;
  std::optional<Span> exec;  // == launch for synchronous kernel spans
  std::optional<KernelMetrics> metrics;

  std::uint64_t duration_ns() const { return exec ? exec->duration_ns() : 0; }
  const std::string& kernel_name() const { return exec ? exec->name : launch.name; }
};

struct LayerExec {
  Span span;
  std::uint32_t layer_index = 0;
  std::string layer_type;
  std::int64_t alloc_bytes = 0;
  std::vector<KernelExec> kernels;

  std::uint64_t duration_ns() const { return span.duration_ns(); }
};

struct ModelRun {
  Span span;
  std::vector<LayerExec> layers;

  std::uint64_t duration_ns() const { return span.duration_ns(); }
};

struct OrphanSpan {
  std::uint64_t span_id = 0;
  std::string reason;
  bool operator==(const OrphanSpan&) const = default;
};

struct EntityTree {
  ModelRun root;
  std::vector<OrphanSpan> orphans;

  std::size_t kernel_count() const;
};

struct Ambiguity {
  std::uint64_t span_id = 0;
  std::vector<std::uint64_t> candidate_parents;  // by span_id
  bool operator==(const Ambiguity&) const = default;
};
using AmbiguityReport = std::vector<Ambiguity>;

struct CorrelationResult {
  EntityTree tree;
  AmbiguityReport ambiguities;
};

IntervalTree build_tree(const std::vector<Span>& spans);

// Parent assignment by closed-interval containment (explicit parent ids win).
CorrelationResult assign_parents(const TraceBundle& bundle);

// Launch/exec fusion by correlation id over a result of assign_parents(bundle).
void correlate_async(CorrelationResult& result, const TraceBundle& bundle);

CorrelationResult correlate(const TraceBundle& bundle);

// Batched form: one GPU pass over many bundles. Entry i holds the result of
// correlate(bundles[i]) or, when that throws, the TraceError text in errors[i].
std::vector<CorrelationResult> correlate_all(const std::vector<TraceBundle>& bundles,
                                             std::vector<std::string>* errors);

bool demand_serialized_rerun(const AmbiguityReport& report);

CorrelationResult resolve_with_serialized(const TraceBundle& original, const TraceBundle& serialized);

}  // namespace strata

#endif  // STRATA_CORRELATOR_HPP
