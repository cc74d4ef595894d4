// strata leveled experimentation — drop-in header of the B200 implementation.
//
// Same API as the reference's leveled.hpp: LeveledRunGroup (runs filed by
// profiling-level set), the overhead report and accurate_latency. The
// per-event trimmed means and step differences run on the GPU (xsp_leveled).
#ifndef STRATA_LEVELED_HPP
#define STRATA_LEVELED_HPP

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "strata/analysis.hpp"
#include "strata/correlator.hpp"
#include "strata/span.hpp"

namespace strata {

struct LeveledError : TraceError {
  using TraceError::TraceError;
};

char level_letter(Level level);              // M, L, G, A
std::string level_set_label(const LevelSet& levels);  // e.g. "M+L+G"

// Cross-run identity of an event: level, layer position, kernel position.
struct LeveledEventKey {
  Level level = Level::Model;
  std::uint32_t layer_index = 0;
  std::uint32_t kernel_index = 0;
  auto operator<=>(const LeveledEventKey&) const = default;
};

std::string event_label(const LeveledEventKey& key);

struct LeveledRunGroup {
  std::uint32_t batch_size = 1;
  SystemSpec system;
  std::map<LevelSet, std::vector<EntityTree>> runs;

  void add(const TraceBundle& bundle);
  static LeveledRunGroup from_bundles(const std::vector<TraceBundle>& bundles);
};

struct OverheadRow {
  LeveledEventKey event;
  std::optional<double> accurate_latency_ns;
  std::map<LevelSet, double> overhead_by_added_levels;
  bool clamped = false;
  bool operator==(const OverheadRow&) const = default;
};

struct OverheadReport {
  std::vector<OverheadRow> rows;
  std::map<LevelSet, double> model_overhead_by_added_levels;
  double noise_tolerance = 0.0;
  std::vector<std::string> warnings;
  bool operator==(const OverheadReport&) const = default;
};

OverheadReport compute_overhead(const LeveledRunGroup& group, const AnalysisOptions& options = {});

double accurate_latency(const LeveledRunGroup& group, const LeveledEventKey& event,
                        const AnalysisOptions& options = {});

}  // namespace strata

#endif  // STRATA_LEVELED_HPP
