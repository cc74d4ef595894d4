// B200 drop-in for the reference's strata/collector.hpp (proj/include/strata/
// collector.hpp): the JSONL wire format of trace bundles, merge of per-tracer
// bundles and the RunSet grouping of an experiment's runs. Same names,
// signatures, exceptions and error texts as the reference (collector.cpp).
//
// ingest() parses the records on the host (a self-contained JSON reader, no
// third-party JSON library) and then orders and validates the bundle on the
// GPU (sort_timeline / validate_bundle, stages (b) and (a) of the hot path);
// merge() unions span sets and re-sorts on the GPU.
#ifndef STRATA_COLLECTOR_HPP
#define STRATA_COLLECTOR_HPP

#include <cstdint>
#include <iosfwd>
#include <map>
#include <string>
#include <vector>

#include "strata/span.hpp"

namespace strata {

struct IngestError : TraceError {
  using TraceError::TraceError;
};

struct MergeError : TraceError {
  using TraceError::TraceError;
};

struct IoError : TraceError {
  using TraceError::TraceError;
};

// One JSON object per line: {"rec":"meta",...} once, then {"rec":"span",...}.
std::string encode_meta_record(const RunMeta& meta);    // collector.cpp:188-190
std::string encode_span_record(const Span& span);       // collector.cpp:192-194

SystemSpec parse_system_spec(const std::string& json_text);  // collector.cpp:196-200
std::string encode_system_spec(const SystemSpec& spec);      // collector.cpp:202-207
SystemSpec load_system_spec(const std::string& path);        // collector.cpp:209-215

// Parses a JSONL stream into a timeline-ordered, validated bundle
// (collector.cpp:219-266). Throws IngestError naming the offending line.
TraceBundle ingest(std::istream& stream);
TraceBundle ingest_string(const std::string& text);

// Union of per-tracer bundles of ONE run (collector.cpp:273-297): same trace
// and metadata, span ids unique across the inputs; MergeError otherwise.
TraceBundle merge(const std::vector<TraceBundle>& bundles);

void persist(const TraceBundle& bundle, const std::string& path);
TraceBundle load(const std::string& path);

std::string to_jsonl(const TraceBundle& bundle);

// The runs of an experiment grouped by (batch size, profiling level set)
// (collector.cpp:320-345).
struct RunSet {
  struct GroupKey {
    std::uint32_t batch_size = 0;
    LevelSet levels;

    auto operator<=>(const GroupKey&) const = default;
  };

  SystemSpec system;
  std::map<GroupKey, std::vector<TraceBundle>> groups;

  /// Adds a bundle; the system spec must agree across the set and a
  /// (trace_id, run_index) may appear once per group (MergeError).
  void add(TraceBundle bundle);

  static RunSet from_bundles(std::vector<TraceBundle> bundles);
};

}  // namespace strata

#endif  // STRATA_COLLECTOR_HPP
