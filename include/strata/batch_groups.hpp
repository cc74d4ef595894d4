// B200 drop-in for the reference's batch grouping of an experiment
// (proj/src/cli.cpp:358-399, build_batch_groups; used by `strata analyze`):
// for every batch size the runs of the deepest profiling-level group sampled
// at that size, correlated into one AnalysisInput. All of a RunSet's selected
// bundles are correlated in ONE batched GPU pass (correlate_all).
#ifndef STRATA_BATCH_GROUPS_HPP
#define STRATA_BATCH_GROUPS_HPP

#include <cstdint>
#include <vector>

#include "strata/analysis.hpp"
#include "strata/collector.hpp"

namespace strata {

struct BatchGroup {
  std::uint32_t batch_size = 1;
  LevelSet levels;
  AnalysisInput input;
};

// Deepest level set per batch size (most levels; ties broken toward the
// lexicographically greater set), batch sizes ascending. Throws the first
// TraceError correlate() would throw, or, for a run with ambiguous kernels,
// "trace <id> has <n> ambiguous spans; resolve them first (correlate
// --serialized-rerun) or profile serialized".
std::vector<BatchGroup> build_batch_groups(const RunSet& runs);

}  // namespace strata

#endif  // STRATA_BATCH_GROUPS_HPP
