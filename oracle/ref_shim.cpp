// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" shim over the UNMODIFIED reference library (strata, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libxsp_ref.so).
// It lets the Python parity suite
//   * generate traces with the reference's own generators
//     (simprof emit_run, tests/test_support.hpp random_nested_bundle /
//      random_async_bundle) and export them as SoA columns, and
//   * run the reference correlate / a8-a15 / compute_overhead on SoA columns and
//     export the results as flat arrays,
// so the CUDA path can be diffed against the reference itself.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load this.
// Built with -fvisibility=hidden: only the xspref_* entry points are exported,
// so the reference's strata:: symbols never collide with anything else.

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <random>
#include <set>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>
#include <atomic>

#include "strata/analysis.hpp"
#include "strata/collector.hpp"
#include "strata/correlator.hpp"
#include "strata/leveled.hpp"
#include "strata/report.hpp"
#include "strata/simprof.hpp"
#include "strata/span.hpp"
#include "test_support.hpp"  // reference tests/test_support.hpp (generators)

#define XSPREF_API extern "C" __attribute__((visibility("default")))

using namespace strata;

namespace {

// ---------------------------------------------------------------------------
// A bag of named flat arrays; Python reads them with xspref_bag_get.
struct Bag {
  struct Arr {
    char dtype;  // 'Q' u64, 'q' i64, 'I' u32, 'i' i32, 'B' u8, 'd' f64, 's' bytes
    std::vector<std::uint8_t> bytes;
  };
  std::map<std::string, Arr> arrays;
  std::vector<std::string> keys;  // insertion order for listing

  template <typename T>
  std::vector<std::uint8_t>& slot(const std::string& name, char dtype) {
    auto it = arrays.find(name);
    if (it == arrays.end()) {
      keys.push_back(name);
      it = arrays.emplace(name, Arr{dtype, {}}).first;
    }
    return it->second.bytes;
  }
  template <typename T>
  void push(const std::string& name, char dtype, T v) {
    auto& b = slot<T>(name, dtype);
    const auto* p = reinterpret_cast<const std::uint8_t*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
  void u64(const std::string& n, std::uint64_t v) { push(n, 'Q', v); }
  void i64(const std::string& n, std::int64_t v) { push(n, 'q', v); }
  void u32(const std::string& n, std::uint32_t v) { push(n, 'I', v); }
  void i32(const std::string& n, std::int32_t v) { push(n, 'i', v); }
  void u8(const std::string& n, std::uint8_t v) { push(n, 'B', v); }
  void f64(const std::string& n, double v) { push(n, 'd', v); }
  void ensure(const std::string& n, char dtype) { slot<char>(n, dtype); }
  // strings: concatenated bytes + u64 offsets (n+1)
  void str(const std::string& n, const std::string& s) {
    auto& off = slot<std::uint64_t>(n + ".off", 'Q');
    auto& data = slot<char>(n + ".data", 's');
    if (off.empty()) {
      std::uint64_t z = 0;
      const auto* p = reinterpret_cast<const std::uint8_t*>(&z);
      off.insert(off.end(), p, p + 8);
    }
    data.insert(data.end(), s.begin(), s.end());
    std::uint64_t end = data.size();
    const auto* p = reinterpret_cast<const std::uint8_t*>(&end);
    off.insert(off.end(), p, p + 8);
  }
  void str_init(const std::string& n) {
    auto& off = slot<std::uint64_t>(n + ".off", 'Q');
    slot<char>(n + ".data", 's');
    if (off.empty()) {
      std::uint64_t z = 0;
      const auto* p = reinterpret_cast<const std::uint8_t*>(&z);
      off.insert(off.end(), p, p + 8);
    }
  }
};

constexpr std::uint8_t kHasParent = 1u << 4;
constexpr std::uint8_t kHasCid = 1u << 5;
constexpr std::uint8_t kHasMetrics = 1u << 6;

std::uint32_t levels_to_mask(const LevelSet& s) {
  std::uint32_t m = 0;
  for (Level l : s) m |= 1u << static_cast<unsigned>(l);
  return m;
}
LevelSet mask_to_levels(std::uint32_t m) {
  LevelSet s;
  for (unsigned l = 0; l < 4; ++l)
    if (m & (1u << l)) s.insert(static_cast<Level>(l));
  return s;
}

// Mirrors the reference's private tag readers (correlator.cpp:44-59).
std::string tag_str(const TagMap& tags, const char* key) {
  auto it = tags.find(key);
  if (it == tags.end()) return {};
  if (const auto* s = std::get_if<std::string>(&it->second)) return *s;
  return {};
}
std::int64_t tag_i64(const TagMap& tags, const char* key) {
  auto it = tags.find(key);
  if (it == tags.end()) return 0;
  if (const auto* i = std::get_if<std::int64_t>(&it->second)) return *i;
  if (const auto* d = std::get_if<double>(&it->second))
    return static_cast<std::int64_t>(*d);
  return 0;
}

struct BundleList {
  std::vector<TraceBundle> bundles;
};

// ---------------------------------------------------------------------------
// SoA import (the same column contract as include/xsp.h)
struct SoaIn {
  std::uint64_t n_spans;
  const std::uint64_t* span_id;
  const std::uint64_t* parent_id;
  const std::uint64_t* begin_ns;
  const std::uint64_t* end_ns;
  const std::uint64_t* cid;
  const std::uint8_t* flags;
  const std::uint32_t* name_id;
  const std::uint64_t* flops;
  const std::uint64_t* dram_read;
  const std::uint64_t* dram_write;
  const double* occupancy;
  const std::int64_t* alloc_bytes;
  const std::uint32_t* type_id;
  std::uint32_t n_traces;
  const std::uint64_t* trace_span_off;  // n_traces+1
  const std::uint64_t* trace_id;
  const std::uint32_t* trace_levels;
  const std::uint32_t* trace_batch;
  const std::uint32_t* trace_run;
  const std::uint8_t* trace_serialized;
  const char* names_data;
  const std::uint64_t* names_off;
  std::uint32_t n_names;
  const char* types_data;
  const std::uint64_t* types_off;
  std::uint32_t n_types;
  const char* system_name;
  double peak_flops;
  double mem_bw;
};

std::vector<TraceBundle> import_soa(const SoaIn& in) {
  auto name_of = [&](std::uint32_t id) {
    return std::string(in.names_data + in.names_off[id],
                       in.names_data + in.names_off[id + 1]);
  };
  auto type_of = [&](std::uint32_t id) {
    return std::string(in.types_data + in.types_off[id],
                       in.types_data + in.types_off[id + 1]);
  };
  std::vector<TraceBundle> out(in.n_traces);
  std::uint64_t metric_row = 0, attr_row = 0;
  for (std::uint32_t t = 0; t < in.n_traces; ++t) {
    TraceBundle& b = out[t];
    b.meta.trace_id = in.trace_id[t];
    b.meta.profiling_levels = mask_to_levels(in.trace_levels[t]);
    b.meta.batch_size = in.trace_batch[t];
    b.meta.run_index = in.trace_run[t];
    b.meta.serialized = in.trace_serialized[t] != 0;
    b.meta.system = SystemSpec{in.system_name, in.peak_flops, in.mem_bw};
    for (std::uint64_t i = in.trace_span_off[t]; i < in.trace_span_off[t + 1]; ++i) {
      Span s;
      s.span_id = in.span_id[i];
      s.trace_id = b.meta.trace_id;
      const std::uint8_t f = in.flags[i];
      s.level = static_cast<Level>(f & 3u);
      s.kind = static_cast<SpanKind>((f >> 2) & 3u);
      if (f & kHasParent) s.parent_id = in.parent_id[i];
      if (f & kHasCid) s.correlation_id = in.cid[i];
      s.begin_ns = in.begin_ns[i];
      s.end_ns = in.end_ns[i];
      s.name = name_of(in.name_id[i]);
      if (f & kHasMetrics) {
        KernelMetrics m{in.flops[metric_row], in.dram_read[metric_row],
                        in.dram_write[metric_row], in.occupancy[metric_row]};
        metrics_to_tags(m, s.tags);
        ++metric_row;
      }
      if (s.level == Level::Layer) {
        std::string ty = type_of(in.type_id[attr_row]);
        if (!ty.empty()) s.tags[kTagLayerType] = ty;
        if (in.alloc_bytes[attr_row] != 0) s.tags[kTagAllocBytes] = in.alloc_bytes[attr_row];
        ++attr_row;
      }
      b.spans.push_back(std::move(s));
    }
  }
  return out;
}

// ---------------------------------------------------------------------------
// SoA export of generated bundles.
void export_soa(const std::vector<TraceBundle>& bundles, Bag& bag) {
  std::set<std::string> names, types;
  for (const auto& b : bundles)
    for (const auto& s : b.spans) {
      names.insert(s.name);
      if (s.level == Level::Layer) types.insert(tag_str(s.tags, kTagLayerType));
    }
  std::unordered_map<std::string, std::uint32_t> name_id, type_id;
  bag.str_init("names");
  bag.str_init("types");
  for (const auto& n : names) {
    name_id.emplace(n, static_cast<std::uint32_t>(name_id.size()));
    bag.str("names", n);
  }
  for (const auto& n : types) {
    type_id.emplace(n, static_cast<std::uint32_t>(type_id.size()));
    bag.str("types", n);
  }
  for (const char* k : {"span_id", "parent_id", "begin_ns", "end_ns", "cid", "flops",
                        "dram_read", "dram_write", "trace_span_off", "trace_id"})
    bag.ensure(k, 'Q');
  for (const char* k : {"name_id", "type_id", "trace_levels", "trace_batch", "trace_run"})
    bag.ensure(k, 'I');
  bag.ensure("flags", 'B');
  bag.ensure("trace_serialized", 'B');
  bag.ensure("occupancy", 'd');
  bag.ensure("alloc_bytes", 'q');
  std::uint64_t off = 0;
  bag.u64("trace_span_off", 0);
  for (const auto& b : bundles) {
    bag.u64("trace_id", b.meta.trace_id);
    bag.u32("trace_levels", levels_to_mask(b.meta.profiling_levels));
    bag.u32("trace_batch", b.meta.batch_size);
    bag.u32("trace_run", b.meta.run_index);
    bag.u8("trace_serialized", b.meta.serialized ? 1 : 0);
    for (const auto& s : b.spans) {
      std::uint8_t f = static_cast<std::uint8_t>(static_cast<unsigned>(s.level) |
                                                 (static_cast<unsigned>(s.kind) << 2));
      if (s.parent_id) f |= kHasParent;
      if (s.correlation_id) f |= kHasCid;
      auto m = metrics_from_tags(s.tags);
      if (m) f |= kHasMetrics;
      bag.u64("span_id", s.span_id);
      bag.u64("parent_id", s.parent_id.value_or(0));
      bag.u64("begin_ns", s.begin_ns);
      bag.u64("end_ns", s.end_ns);
      bag.u64("cid", s.correlation_id.value_or(0));
      bag.u8("flags", f);
      bag.u32("name_id", name_id.at(s.name));
      if (m) {
        bag.u64("flops", m->flop_count_sp);
        bag.u64("dram_read", m->dram_read_bytes);
        bag.u64("dram_write", m->dram_write_bytes);
        bag.f64("occupancy", m->achieved_occupancy);
      }
      if (s.level == Level::Layer) {
        bag.i64("alloc_bytes", tag_i64(s.tags, kTagAllocBytes));
        bag.u32("type_id", type_id.at(tag_str(s.tags, kTagLayerType)));
      }
    }
    off += b.spans.size();
    bag.u64("trace_span_off", off);
  }
  if (!bundles.empty()) {
    const auto& sys = bundles.front().meta.system;
    bag.str_init("system_name");
    bag.str("system_name", sys.name);
    bag.f64("system_peak", sys.peak_flops);
    bag.f64("system_bw", sys.memory_bandwidth_bytes_per_s);
  }
}

// ---------------------------------------------------------------------------
// Canonical result export.

// Orphan reason codes (the C ABI's xsp_orphan_reason values).
std::uint8_t reason_code(const std::string& r) {
  if (r == "layer-level span with non-sync kind") return 1;
  if (r.rfind("explicit parent ", 0) == 0 && r.find("is not the model span") != std::string::npos) return 2;
  if (r == "outside the model interval") return 3;
  if (r.rfind("explicit parent ", 0) == 0 && r.find("is not a layer in the tree") != std::string::npos) return 4;
  if (r == "contained in no layer interval") return 5;
  if (r == "execution record without correlation id") return 6;
  if (r == "launch without correlation id") return 7;
  if (r == "launch has no matching execution record") return 8;
  if (r == "execution record without matching launch") return 9;
  return 255;
}

using RowMap = std::unordered_map<std::uint64_t, std::uint64_t>;
RowMap row_map(const TraceBundle& b, std::uint64_t base) {
  RowMap m;
  for (std::uint64_t i = 0; i < b.spans.size(); ++i) m.emplace(b.spans[i].span_id, base + i);
  return m;
}

void export_correlation(const std::vector<TraceBundle>& bundles,
                        const std::vector<CorrelationResult*>& results,
                        const std::vector<std::string>& errors, Bag& bag) {
  for (const char* k : {"t_layer_off", "layer_kernel_off", "t_orphan_off", "t_amb_off",
                        "amb_cand_off", "t_model_row", "layer_row", "kernel_launch_row",
                        "kernel_exec_row", "orphan_row", "amb_row", "amb_cand_row",
                        "kernel_flops", "kernel_read", "kernel_write"})
    bag.ensure(k, 'Q');
  bag.ensure("t_status", 'i');
  bag.ensure("layer_index", 'I');
  bag.ensure("orphan_reason", 'B');
  bag.ensure("kernel_has_metrics", 'B');
  bag.ensure("kernel_occ", 'd');
  bag.ensure("layer_alloc", 'q');
  bag.str_init("t_error");
  bag.str_init("orphan_text");
  bag.str_init("layer_type");
  std::uint64_t base = 0, nl = 0, nk = 0, no = 0, na = 0, nc = 0;
  bag.u64("t_layer_off", 0);
  bag.u64("layer_kernel_off", 0);
  bag.u64("t_orphan_off", 0);
  bag.u64("t_amb_off", 0);
  bag.u64("amb_cand_off", 0);
  for (std::size_t t = 0; t < bundles.size(); ++t) {
    const TraceBundle& b = bundles[t];
    RowMap rows = row_map(b, base);
    const CorrelationResult* r = results[t];
    bag.i32("t_status", r ? 0 : 1);
    bag.str("t_error", errors[t]);
    if (r) {
      const auto& root = r->tree.root;
      bag.u64("t_model_row", rows.at(root.span.span_id));
      for (const LayerExec& l : root.layers) {
        bag.u64("layer_row", rows.at(l.span.span_id));
        bag.u32("layer_index", l.layer_index);
        bag.str("layer_type", l.layer_type);
        bag.i64("layer_alloc", l.alloc_bytes);
        for (const KernelExec& k : l.kernels) {
          bag.u64("kernel_launch_row", rows.at(k.launch.span_id));
          bag.u64("kernel_exec_row", k.exec ? rows.at(k.exec->span_id) : ~0ull);
          bag.u8("kernel_has_metrics", k.metrics ? 1 : 0);
          KernelMetrics m = k.metrics.value_or(KernelMetrics{});
          bag.u64("kernel_flops", m.flop_count_sp);
          bag.u64("kernel_read", m.dram_read_bytes);
          bag.u64("kernel_write", m.dram_write_bytes);
          bag.f64("kernel_occ", m.achieved_occupancy);
          ++nk;
        }
        bag.u64("layer_kernel_off", nk);
        ++nl;
      }
      for (const OrphanSpan& o : r->tree.orphans) {
        bag.u64("orphan_row", rows.at(o.span_id));
        bag.u8("orphan_reason", reason_code(o.reason));
        bag.str("orphan_text", o.reason);
        ++no;
      }
      for (const Ambiguity& a : r->ambiguities) {
        bag.u64("amb_row", rows.at(a.span_id));
        for (auto c : a.candidate_parents) {
          bag.u64("amb_cand_row", rows.at(c));
          ++nc;
        }
        bag.u64("amb_cand_off", nc);
        ++na;
      }
    } else {
      bag.u64("t_model_row", ~0ull);
    }
    bag.u64("t_layer_off", nl);
    bag.u64("t_orphan_off", no);
    bag.u64("t_amb_off", na);
    base += b.spans.size();
  }
}

std::int8_t opt_bool(const std::optional<bool>& b) { return b ? (*b ? 1 : 0) : -1; }
double opt_d(const std::optional<double>& d) { return d ? *d : std::nan(""); }

}  // namespace

// ===========================================================================
// Bags
XSPREF_API void xspref_bag_free(void* h) { delete static_cast<Bag*>(h); }
XSPREF_API int xspref_bag_count(void* h) {
  return static_cast<int>(static_cast<Bag*>(h)->keys.size());
}
XSPREF_API const char* xspref_bag_key(void* h, int i) {
  return static_cast<Bag*>(h)->keys[static_cast<std::size_t>(i)].c_str();
}
XSPREF_API int xspref_bag_get(void* h, const char* name, const void** data,
                              std::uint64_t* nbytes, char* dtype) {
  auto* bag = static_cast<Bag*>(h);
  auto it = bag->arrays.find(name);
  if (it == bag->arrays.end()) return -1;
  *data = it->second.bytes.data();
  *nbytes = it->second.bytes.size();
  *dtype = it->second.dtype;
  return 0;
}

// ===========================================================================
// Generators
XSPREF_API void* xspref_list_new() { return new BundleList; }
XSPREF_API void xspref_list_free(void* h) { delete static_cast<BundleList*>(h); }
XSPREF_API std::uint64_t xspref_list_size(void* h) {
  return static_cast<BundleList*>(h)->bundles.size();
}
XSPREF_API void* xspref_rng_new(std::uint64_t seed) { return new std::mt19937_64(seed); }
XSPREF_API void xspref_rng_free(void* h) { delete static_cast<std::mt19937_64*>(h); }

static thread_local std::string g_err;
XSPREF_API const char* xspref_last_error() { return g_err.c_str(); }

/// simprof::emit_run (simprof.cpp:278-343) for a named fixture or a model JSON.
XSPREF_API int xspref_emit(void* list, const char* model_name_or_json, std::uint32_t batch,
                           std::uint32_t levels_mask, std::uint64_t layer_oh,
                           std::uint64_t kernel_oh, double metric_mult, int serialized,
                           std::uint32_t run_index, std::uint64_t jitter_max,
                           std::uint64_t jitter_seed) {
  try {
    std::string arg(model_name_or_json);
    SyntheticModel model =
        (!arg.empty() && arg[0] == '{') ? parse_model(arg) : fixture_by_name(arg);
    OverheadProfile oh{layer_oh, kernel_oh, metric_mult};
    JitterProfile jit{jitter_max, jitter_seed};
    static_cast<BundleList*>(list)->bundles.push_back(emit_run(
        model, batch, mask_to_levels(levels_mask), oh, serialized != 0, run_index, jit));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

/// simprof::emit_leveled_chain (simprof.cpp:345-361).
XSPREF_API int xspref_emit_chain(void* list, const char* model_name, std::uint32_t batch,
                                 std::uint64_t layer_oh, std::uint64_t kernel_oh,
                                 double metric_mult) {
  try {
    std::string arg(model_name);
    SyntheticModel model =
        (!arg.empty() && arg[0] == '{') ? parse_model(arg) : fixture_by_name(arg);
    OverheadProfile oh{layer_oh, kernel_oh, metric_mult};
    for (auto& b : emit_leveled_chain(model, batch, oh))
      static_cast<BundleList*>(list)->bundles.push_back(std::move(b));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

/// tests/test_support.hpp:204-258.
XSPREF_API void xspref_random_nested(void* list, void* rng, std::uint64_t max_spans,
                                     double explicit_fraction) {
  static_cast<BundleList*>(list)->bundles.push_back(testing::random_nested_bundle(
      *static_cast<std::mt19937_64*>(rng), max_spans, explicit_fraction));
}

/// tests/test_support.hpp:262-319.
XSPREF_API void xspref_random_async(void* list, void* rng, std::uint64_t pairs) {
  static_cast<BundleList*>(list)->bundles.push_back(
      testing::random_async_bundle(*static_cast<std::mt19937_64*>(rng), pairs));
}

/// Shuffle the spans of the last bundle and (optionally) re-sort them, as the
/// reference's file-order test does (test_correlator.cpp:315-327).
XSPREF_API void xspref_shuffle_last(void* list, void* rng, int resort) {
  auto& b = static_cast<BundleList*>(list)->bundles.back();
  std::shuffle(b.spans.begin(), b.spans.end(), *static_cast<std::mt19937_64*>(rng));
  if (resort) sort_timeline(b.spans);
}

XSPREF_API void* xspref_list_export(void* list) {
  auto* bag = new Bag;
  export_soa(static_cast<BundleList*>(list)->bundles, *bag);
  return bag;
}

// ===========================================================================
// Reference operations over SoA input

/// correlate() (correlator.cpp:366-370) per trace; TraceError -> status 1 + text.
XSPREF_API void* xspref_correlate(const SoaIn* in) {
  std::vector<TraceBundle> bundles = import_soa(*in);
  std::vector<CorrelationResult> res(bundles.size());
  std::vector<CorrelationResult*> ptrs(bundles.size(), nullptr);
  std::vector<std::string> errs(bundles.size());
  for (std::size_t t = 0; t < bundles.size(); ++t) {
    try {
      res[t] = correlate(bundles[t]);
      ptrs[t] = &res[t];
    } catch (const TraceError& e) {
      errs[t] = e.what();
    }
  }
  auto* bag = new Bag;
  export_correlation(bundles, ptrs, errs, *bag);
  return bag;
}

/// validate_bundle() (span.cpp:129-192) per trace. span_trace_id (optional)
/// overrides Span::trace_id; tag_bits (optional, XSP_TAG_* of include/xsp.h)
/// turns metric tags into raw forms the decoded columns cannot carry: bits 0-2
/// store an int64 < 0 under flop_count_sp / dram_read_bytes / dram_write_bytes,
/// and a metric span WITHOUT bit 3 stores achieved_occupancy as an int64 tag.
XSPREF_API void* xspref_validate(const SoaIn* in, const std::uint64_t* span_trace_id,
                                 const std::uint8_t* tag_bits) {
  std::vector<TraceBundle> bundles = import_soa(*in);
  std::uint64_t row = 0;
  for (auto& b : bundles) {
    for (auto& sp : b.spans) {
      if (span_trace_id) sp.trace_id = span_trace_id[row];
      if (tag_bits) {
        const std::uint8_t tb = tag_bits[row];
        const char* keys[3] = {kTagFlopCountSp, kTagDramReadBytes, kTagDramWriteBytes};
        for (int k = 0; k < 3; ++k)
          if (tb & (1u << k)) sp.tags[keys[k]] = static_cast<std::int64_t>(-1 - (std::int64_t)(row % 7));
        auto it = sp.tags.find(kTagAchievedOccupancy);
        if (it != sp.tags.end() && !(tb & 8u))
          it->second = static_cast<std::int64_t>(std::get<double>(it->second));
      }
      ++row;
    }
  }
  auto* bag = new Bag;
  bag->ensure("trace", 'I');
  bag->ensure("span_id", 'Q');
  bag->str_init("rule");
  bag->str_init("detail");
  for (std::size_t t = 0; t < bundles.size(); ++t) {
    for (const auto& issue : validate_bundle(bundles[t])) {
      bag->u32("trace", static_cast<std::uint32_t>(t));
      bag->u64("span_id", issue.span_id);
      bag->str("rule", issue.rule);
      bag->str("detail", issue.detail);
    }
  }
  return bag;
}

/// resolve_with_serialized() (correlator.cpp:379-456) per trace pair: trace t of
/// `in` against trace t of `ser`; TraceError -> status 1 + text.
XSPREF_API void* xspref_resolve(const SoaIn* in, const SoaIn* ser) {
  std::vector<TraceBundle> orig = import_soa(*in);
  std::vector<TraceBundle> sers = import_soa(*ser);
  std::vector<CorrelationResult> res(orig.size());
  std::vector<CorrelationResult*> ptrs(orig.size(), nullptr);
  std::vector<std::string> errs(orig.size());
  for (std::size_t t = 0; t < orig.size(); ++t) {
    try {
      res[t] = resolve_with_serialized(orig[t], sers.at(t));
      ptrs[t] = &res[t];
    } catch (const TraceError& e) {
      errs[t] = e.what();
    }
  }
  auto* bag = new Bag;
  export_correlation(orig, ptrs, errs, *bag);
  return bag;
}

/// Wall-clock timing of the reference hot path (correlate + a8..a15) over a
/// set of groups, `threads` workers with one group per task. Returns seconds.
/// groups: [first_trace, n_runs] pairs.
XSPREF_API double xspref_time_pipeline(const SoaIn* in, const std::uint32_t* group_first,
                                       const std::uint32_t* group_runs, std::uint32_t n_groups,
                                       int threads, int reps) {
  std::vector<TraceBundle> bundles = import_soa(*in);
  SystemSpec spec{in->system_name, in->peak_flops, in->mem_bw};
  std::atomic<std::uint64_t> sink{0};
  auto t0 = std::chrono::steady_clock::now();
  for (int rep = 0; rep < reps; ++rep) {
    std::atomic<std::uint32_t> next{0};
    auto worker = [&]() {
      for (;;) {
        std::uint32_t g = next.fetch_add(1);
        if (g >= n_groups) break;
        AnalysisInput input;
        input.batch_size = bundles[group_first[g]].meta.batch_size;
        for (std::uint32_t r = 0; r < group_runs[g]; ++r)
          input.runs.push_back(correlate(bundles[group_first[g] + r]).tree);
        std::uint64_t acc = 0;
        acc += a8_kernel_table(input, spec).rows.size();
        acc += a9_kernel_roofline(input, spec).points.size();
        acc += a10_by_name(input, spec).rows.size();
        acc += a11_by_layer(input, spec).rows.size();
        acc += a12_metrics_per_layer(input).total_flops.size();
        acc += a13_gpu_vs_nongpu(input).rows.size();
        acc += a14_layer_roofline(input, spec).points.size();
        acc += a15_model_aggregate({input}, spec).rows.size();
        sink += acc;
      }
    };
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
  }
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count() / reps + (sink == ~0ull ? 1 : 0);
}

/// a8..a15 (analysis.cpp:342-586) per group; groups are consecutive trace
/// ranges [first, first+runs). Trees come from correlate() of each trace.
XSPREF_API void* xspref_analyze(const SoaIn* in, const std::uint32_t* group_first,
                                const std::uint32_t* group_runs, std::uint32_t n_groups,
                                double trim, double noise) {
  std::vector<TraceBundle> bundles = import_soa(*in);
  SystemSpec spec{in->system_name, in->peak_flops, in->mem_bw};
  AnalysisOptions opts;
  opts.trim_fraction = trim;
  opts.noise_tolerance = noise;
  std::unordered_map<std::string, std::uint32_t> name_id;
  for (std::uint32_t i = 0; i < in->n_names; ++i)
    name_id.emplace(std::string(in->names_data + in->names_off[i],
                                in->names_data + in->names_off[i + 1]),
                    i);
  auto* bag = new Bag;
  for (const char* k : {"g_kernel_off", "g_layer_off", "g_name_off", "k_flops", "k_read",
                        "k_write", "l_flops", "l_read", "l_write", "l_count", "n_count",
                        "n_flops", "n_read", "n_write", "m_flops", "m_read", "m_write",
                        "m_count"})
    bag->ensure(k, 'Q');
  for (const char* k : {"k_name", "k_layer", "l_index", "l_name", "n_name", "m_batch"})
    bag->ensure(k, 'I');
  for (const char* k : {"k_lat", "k_occ", "k_ai", "k_tput", "l_layer_lat", "l_kern_lat",
                        "l_occ", "l_ai", "l_tput", "l_gpu", "l_nongpu", "l_gpu_share",
                        "l_nongpu_share", "n_lat", "n_pct", "n_occ", "n_ai", "n_tput",
                        "m_lat", "m_kern_lat", "m_occ", "m_ai", "m_tput", "m_gpu",
                        "m_gpu_pct", "a10_model_lat", "k9_ai", "k9_tput", "l14_ai",
                        "l14_tput", "m_throughput"})
    bag->ensure(k, 'd');
  for (const char* k : {"k_bound", "l_bound", "l_flagged", "n_bound", "m_bound", "k9_in",
                        "k9_bound", "l14_in", "l14_bound", "mr_in", "mr_bound"})
    bag->ensure(k, 'B');
  bag->ensure("g_status", 'i');
  bag->str_init("g_error");
  bag->ensure("g_type_off", 'Q');
  bag->ensure("y_count", 'Q');
  bag->ensure("y_alloc", 'q');
  bag->ensure("y_lat", 'd');
  bag->str_init("y_type");
  std::uint64_t nk = 0, nl = 0, nn = 0, ny = 0;
  bag->u64("g_kernel_off", 0);
  bag->u64("g_layer_off", 0);
  bag->u64("g_name_off", 0);
  bag->u64("g_type_off", 0);
  for (std::uint32_t g = 0; g < n_groups; ++g) {
    try {
      AnalysisInput input;
      input.batch_size = bundles[group_first[g]].meta.batch_size;
      for (std::uint32_t r = 0; r < group_runs[g]; ++r)
        input.runs.push_back(correlate(bundles[group_first[g] + r]).tree);
      KernelInfoTable a8 = a8_kernel_table(input, spec, opts);
      RooflineReport a9 = a9_kernel_roofline(input, spec, opts);
      KernelNameTable a10 = a10_by_name(input, spec, opts);
      LayerAggregateTable a11 = a11_by_layer(input, spec, opts);
      GpuNonGpuTable a13 = a13_gpu_vs_nongpu(input, opts);
      RooflineReport a14 = a14_layer_roofline(input, spec, opts);
      ModelAggregateTable a15 = a15_model_aggregate({input}, spec, opts);
      RooflineReport mr = model_roofline({input}, spec, opts);
      ModelInfoTable a1 = a1_model_info({input}, opts);
      LayerTypeTable a5 = a5_a6_a7_by_type(input, opts);
      for (const auto& row : a5.rows) {
        bag->str("y_type", row.type);
        bag->u64("y_count", row.count);
        bag->f64("y_lat", row.total_latency_ns);
        bag->i64("y_alloc", row.total_alloc_bytes);
      }
      ny += a5.rows.size();
      bag->i32("g_status", 0);
      bag->str("g_error", "");
      for (const auto& row : a8.rows) {
        bag->u32("k_name", name_id.at(row.name));
        bag->u32("k_layer", row.layer_index);
        bag->f64("k_lat", row.latency_ns);
        bag->u64("k_flops", row.flops);
        bag->u64("k_read", row.dram_read_bytes);
        bag->u64("k_write", row.dram_write_bytes);
        bag->f64("k_occ", row.achieved_occupancy);
        bag->f64("k_ai", opt_d(row.arithmetic_intensity));
        bag->f64("k_tput", opt_d(row.arithmetic_throughput));
        bag->u8("k_bound", static_cast<std::uint8_t>(opt_bool(row.memory_bound)));
      }
      // a9: points and exclusions share one ordinal space ("kernel <i>: name").
      {
        std::vector<std::uint8_t> in_(a8.rows.size(), 0);
        std::vector<double> ai(a8.rows.size(), std::nan("")), tp(a8.rows.size(), std::nan(""));
        std::vector<std::uint8_t> bd(a8.rows.size(), 255);
        for (const auto& p : a9.points) {
          std::size_t ord = std::stoull(p.subject.substr(7));
          in_[ord] = 1;
          ai[ord] = p.arithmetic_intensity;
          tp[ord] = p.arithmetic_throughput;
          bd[ord] = p.memory_bound ? 1 : 0;
        }
        for (std::size_t i = 0; i < a8.rows.size(); ++i) {
          bag->u8("k9_in", in_[i]);
          bag->f64("k9_ai", ai[i]);
          bag->f64("k9_tput", tp[i]);
          bag->u8("k9_bound", bd[i]);
        }
      }
      nk += a8.rows.size();
      bag->f64("a10_model_lat", a10.model_latency_ns);
      for (const auto& row : a10.rows) {
        bag->u32("n_name", name_id.at(row.name));
        bag->u64("n_count", row.count);
        bag->f64("n_lat", row.total_latency_ns);
        bag->f64("n_pct", row.latency_percent);
        bag->u64("n_flops", row.total_flops);
        bag->u64("n_read", row.total_dram_read_bytes);
        bag->u64("n_write", row.total_dram_write_bytes);
        bag->f64("n_occ", row.weighted_achieved_occupancy);
        bag->f64("n_ai", opt_d(row.arithmetic_intensity));
        bag->f64("n_tput", opt_d(row.arithmetic_throughput));
        bag->u8("n_bound", static_cast<std::uint8_t>(opt_bool(row.memory_bound)));
      }
      nn += a10.rows.size();
      for (std::size_t i = 0; i < a11.rows.size(); ++i) {
        const auto& row = a11.rows[i];
        bag->u32("l_index", row.layer_index);
        bag->u32("l_name", name_id.at(row.name));
        bag->f64("l_layer_lat", row.layer_latency_ns);
        bag->f64("l_kern_lat", row.kernel_latency_ns);
        bag->u64("l_flops", row.total_flops);
        bag->u64("l_read", row.total_dram_read_bytes);
        bag->u64("l_write", row.total_dram_write_bytes);
        bag->f64("l_occ", row.weighted_achieved_occupancy);
        bag->u64("l_count", row.kernel_count);
        bag->f64("l_ai", opt_d(row.arithmetic_intensity));
        bag->f64("l_tput", opt_d(row.arithmetic_throughput));
        bag->u8("l_bound", static_cast<std::uint8_t>(opt_bool(row.memory_bound)));
        const auto& r13 = a13.rows[i];
        bag->f64("l_gpu", r13.gpu_latency_ns);
        bag->f64("l_nongpu", r13.non_gpu_latency_ns);
        bag->f64("l_gpu_share", r13.gpu_share);
        bag->f64("l_nongpu_share", r13.non_gpu_share);
        bag->u8("l_flagged", r13.flagged ? 1 : 0);
      }
      {
        std::vector<std::uint8_t> in_(a11.rows.size(), 0);
        std::vector<double> ai(a11.rows.size(), std::nan("")), tp(a11.rows.size(), std::nan(""));
        std::vector<std::uint8_t> bd(a11.rows.size(), 255);
        for (const auto& p : a14.points) {
          std::size_t ord = std::stoull(p.subject.substr(6));
          in_[ord] = 1;
          ai[ord] = p.arithmetic_intensity;
          tp[ord] = p.arithmetic_throughput;
          bd[ord] = p.memory_bound ? 1 : 0;
        }
        for (std::size_t i = 0; i < a11.rows.size(); ++i) {
          bag->u8("l14_in", in_[i]);
          bag->f64("l14_ai", ai[i]);
          bag->f64("l14_tput", tp[i]);
          bag->u8("l14_bound", bd[i]);
        }
      }
      nl += a11.rows.size();
      const auto& m = a15.rows.at(0);
      bag->u32("m_batch", m.batch_size);
      bag->f64("m_lat", m.model_latency_ns);
      bag->f64("m_kern_lat", m.kernel_latency_ns);
      bag->u64("m_flops", m.total_flops);
      bag->u64("m_read", m.total_dram_read_bytes);
      bag->u64("m_write", m.total_dram_write_bytes);
      bag->f64("m_occ", m.weighted_achieved_occupancy);
      bag->u64("m_count", m.kernel_count);
      bag->f64("m_ai", opt_d(m.arithmetic_intensity));
      bag->f64("m_tput", opt_d(m.arithmetic_throughput));
      bag->u8("m_bound", static_cast<std::uint8_t>(opt_bool(m.memory_bound)));
      bag->f64("m_gpu", a13.model_gpu_latency_ns);
      bag->f64("m_gpu_pct", a13.model_gpu_percent);
      bag->f64("m_throughput", a1.rows.at(0).throughput);
      bag->u8("mr_in", mr.points.empty() ? 0 : 1);
      bag->u8("mr_bound", mr.points.empty() ? 255 : (mr.points[0].memory_bound ? 1 : 0));
    } catch (const TraceError& e) {
      bag->i32("g_status", 1);
      bag->str("g_error", e.what());
      // keep per-group arrays aligned
      for (const char* k : {"m_batch"}) bag->u32(k, 0);
      for (const char* k : {"m_flops", "m_read", "m_write", "m_count"}) bag->u64(k, 0);
      for (const char* k : {"m_lat", "m_kern_lat", "m_occ", "m_ai", "m_tput", "m_gpu",
                            "m_gpu_pct", "a10_model_lat", "m_throughput"})
        bag->f64(k, std::nan(""));
      for (const char* k : {"m_bound", "mr_in", "mr_bound"}) bag->u8(k, 255);
    }
    bag->u64("g_kernel_off", nk);
    bag->u64("g_layer_off", nl);
    bag->u64("g_name_off", nn);
    bag->u64("g_type_off", ny);
  }
  return bag;
}

/// LeveledRunGroup::from_bundles + compute_overhead (leveled.cpp:56-231) over
/// ALL traces of the input (one leveled group).
XSPREF_API void* xspref_leveled(const SoaIn* in, double trim, double noise) {
  std::vector<TraceBundle> bundles = import_soa(*in);
  AnalysisOptions opts;
  opts.trim_fraction = trim;
  opts.noise_tolerance = noise;
  auto* bag = new Bag;
  bag->ensure("o_level", 'B');
  bag->ensure("o_layer", 'I');
  bag->ensure("o_kernel", 'I');
  bag->ensure("o_accurate", 'd');
  bag->ensure("o_clamped", 'B');
  bag->ensure("o_ov_mask", 'I');  // added-levels mask per overhead entry
  bag->ensure("o_ov_val", 'd');
  bag->ensure("o_ov_off", 'Q');
  bag->ensure("model_ov_mask", 'I');
  bag->ensure("model_ov_val", 'd');
  bag->str_init("warnings");
  bag->str_init("error");
  try {
    LeveledRunGroup group = LeveledRunGroup::from_bundles(bundles);
    OverheadReport rep = compute_overhead(group, opts);
    bag->i32("status", 0);
    bag->str("error", "");
    std::uint64_t nov = 0;
    bag->u64("o_ov_off", 0);
    for (const auto& row : rep.rows) {
      bag->u8("o_level", static_cast<std::uint8_t>(row.event.level));
      bag->u32("o_layer", row.event.layer_index);
      bag->u32("o_kernel", row.event.kernel_index);
      bag->f64("o_accurate", opt_d(row.accurate_latency_ns));
      bag->u8("o_clamped", row.clamped ? 1 : 0);
      for (const auto& [levels, v] : row.overhead_by_added_levels) {
        bag->u32("o_ov_mask", levels_to_mask(levels));
        bag->f64("o_ov_val", v);
        ++nov;
      }
      bag->u64("o_ov_off", nov);
    }
    for (const auto& [levels, v] : rep.model_overhead_by_added_levels) {
      bag->u32("model_ov_mask", levels_to_mask(levels));
      bag->f64("model_ov_val", v);
    }
    for (const auto& w : rep.warnings) bag->str("warnings", w);
  } catch (const TraceError& e) {
    bag->i32("status", 1);
    bag->str("error", e.what());
  }
  return bag;
}

/// Reference trimmed_mean (analysis.cpp:28-39) for scalar pinning.
XSPREF_API double xspref_trimmed_mean(const double* v, std::uint64_t n, double f) {
  return trimmed_mean(std::vector<double>(v, v + n), f);
}

// The reference report's CSV of one analysis table (a8..a14) of analysis group g
// (report.cpp to_csv(to_table(...))). Returns malloc'd NUL-terminated text (free
// with xspref_free_text), or nullptr with xspref_last_error set.
XSPREF_API char* xspref_report_csv(const SoaIn* in, std::uint32_t first, std::uint32_t runs, int table,
                                   double trim, double noise) {
  try {
    std::vector<TraceBundle> bundles = import_soa(*in);
    SystemSpec spec{in->system_name, in->peak_flops, in->mem_bw};
    AnalysisOptions opts;
    opts.trim_fraction = trim;
    opts.noise_tolerance = noise;
    AnalysisInput input;
    input.batch_size = bundles[first].meta.batch_size;
    for (std::uint32_t r = 0; r < runs; ++r) input.runs.push_back(correlate(bundles[first + r]).tree);
    Table t;
    switch (table) {
      case 8: t = to_table(a8_kernel_table(input, spec, opts)); break;
      case 9: t = to_table(a9_kernel_roofline(input, spec, opts), "a9"); break;
      case 10: t = to_table(a10_by_name(input, spec, opts)); break;
      case 11: t = to_table(a11_by_layer(input, spec, opts)); break;
      case 12: t = to_table(a12_metrics_per_layer(input, opts)); break;
      case 13: t = to_table(a13_gpu_vs_nongpu(input, opts)); break;
      case 14: t = to_table(a14_layer_roofline(input, spec, opts), "a14"); break;
      default: throw std::invalid_argument("table");
    }
    const std::string csv = to_csv(t);
    char* out = static_cast<char*>(std::malloc(csv.size() + 1));
    std::memcpy(out, csv.data(), csv.size() + 1);
    return out;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

XSPREF_API void xspref_free_text(char* p) { std::free(p); }

// The reference's JSONL wire form (collector.cpp to_jsonl) of bundle i of a list.
XSPREF_API char* xspref_list_jsonl(void* list, std::uint64_t i) {
  const auto& b = static_cast<BundleList*>(list)->bundles;
  const std::string t = to_jsonl(b.at(i));
  char* out = static_cast<char*>(std::malloc(t.size() + 1));
  std::memcpy(out, t.data(), t.size() + 1);
  return out;
}

// The reference's ingest() (collector.cpp:219-266) of each NUL-separated JSONL
// stream, exported as SoA columns like xspref_list_export; nullptr with
// xspref_last_error = the IngestError text on failure.
XSPREF_API void* xspref_ingest(const char* text, const std::uint64_t* off, std::uint32_t n) {
  try {
    std::vector<TraceBundle> bundles;
    for (std::uint32_t i = 0; i < n; ++i) bundles.push_back(ingest_string(std::string(text + off[i], text + off[i + 1])));
    auto* bag = new Bag;
    export_soa(bundles, *bag);
    return bag;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
