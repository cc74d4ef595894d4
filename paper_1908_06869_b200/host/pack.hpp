// Internal to libstrata_b200: the GPU context and the AoS <-> SoA adapters
// between strata's value types (TraceBundle, EntityTree) and the C ABI columns.
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "strata/analysis.hpp"
#include "strata/correlator.hpp"
#include "strata/span.hpp"
#include "xsp.h"

namespace strata::b200 {

// The calling thread's xsp context on the current device. Throws if there is
// no CUDA device: this library has no CPU fallback.
xsp_ctx* ctx();
// Throws std::runtime_error with xsp_last_error() unless st == XSP_OK.
void check(xsp_status st);

constexpr std::uint32_t kNone = 0xFFFFFFFFu;

// Interned string table in byte-lexicographic order (id order == string order).
struct Strings {
  std::vector<std::string> sorted;
  std::unordered_map<std::string, std::uint32_t> id;
  void add(const std::string& s) { id.emplace(s, 0); }
  void finish();
};

// Span columns of a batch of bundles (include/xsp.h layout).
struct PackedSpans {
  std::vector<std::uint64_t> span_id, parent_id, begin, end, cid;
  std::vector<std::uint8_t> flags;
  std::vector<std::uint32_t> name_id;
  std::vector<std::uint64_t> flops, dram_read, dram_write;
  std::vector<double> occupancy;
  std::vector<std::int64_t> alloc_bytes;
  std::vector<std::uint32_t> type_id;
  std::vector<std::uint64_t> span_off;
  std::vector<std::uint32_t> levels;
  Strings names, types;
  std::vector<const Span*> row;  // span of each row

  xsp_span_cols cols() const;
  xsp_traces traces() const;
};

std::uint32_t level_mask(const LevelSet& levels);
LevelSet mask_levels(std::uint32_t mask);

// Columns of `bundles` (each must be in timeline order, see sorted_copy).
PackedSpans pack_bundles(const std::vector<const TraceBundle*>& bundles);

// metrics_from_tags / the layer tag readers of the reference (span.cpp:67-101,
// correlator.cpp:44-59).
std::int64_t tag_int_or0(const TagMap& tags, const char* key);
std::string tag_string_or_empty(const TagMap& tags, const char* key);

// Host copy of a correlation (pinned ctx memory is reused by the next call).
struct HostCorr {
  std::uint32_t n_traces = 0;
  std::vector<std::int32_t> status;
  std::vector<std::uint32_t> err_row, model_row, t_layer_off, t_kernel_off, t_orphan_off, t_amb_off;
  std::vector<std::uint32_t> layer_row, layer_kernel_off, layer_attr_row;
  std::vector<std::uint32_t> k_launch, k_exec, k_mrow;
  std::vector<std::uint32_t> orphan_row;
  std::vector<std::uint8_t> orphan_reason;
  std::vector<std::uint32_t> amb_row, amb_cand_off, amb_cand_row;
};

HostCorr run_correlation(const PackedSpans& p, int mode);

// Reference message texts (correlator.cpp) rebuilt from a fault code + rows.
std::string trace_error_text(const PackedSpans& p, const HostCorr& c, std::uint32_t t);
std::string orphan_text(const PackedSpans& p, std::uint8_t reason, std::uint32_t row);

// Build the CorrelationResult of trace t (Span copies from the input bundle).
CorrelationResult unpack_result(const PackedSpans& p, const HostCorr& c, std::uint32_t t);

// ---- analysis / leveling inputs packed from entity trees

struct PackedTrees {
  // span columns: one row per model span and per layer span
  std::vector<std::uint64_t> zeros64, begin, end;
  std::vector<std::uint8_t> flags;
  std::vector<std::uint32_t> name_id;
  std::vector<std::uint64_t> flops, dram_read, dram_write;
  std::vector<double> occupancy;
  // correlation columns
  std::vector<std::int32_t> status;
  std::vector<std::uint32_t> model_row, t_layer_off, t_kernel_off, t_amb_off;
  std::vector<std::uint32_t> layer_row, layer_kernel_off;
  std::vector<std::uint64_t> layer_dur, kernel_dur;
  std::vector<std::uint32_t> kernel_mrow, kernel_name;
  std::vector<double> kernel_occ;
  // layer table (a5-a7): one row per layer, in layer order
  std::vector<std::uint32_t> layer_attr_row, type_id;
  std::vector<std::int64_t> alloc_bytes;
  Strings names, types;

  xsp_span_cols cols() const;
  xsp_corr_out corr() const;
};

// One trace per tree, in order.
PackedTrees pack_trees(const std::vector<const EntityTree*>& trees);

}  // namespace strata::b200
