// libstrata_b200: analyses (reference: analysis.hpp / analysis.cpp).
// The repetition combining and every per-kernel / per-layer / per-name /
// per-model reduction behind A1..A15 run on the GPU (xsp_analyze_host) over
// the packed entity trees; this file turns the result columns back into the
// reference's value types and raises the reference's errors.
#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>

#include "pack.hpp"

namespace strata {

// ---- scalar primitives (analysis.cpp:28-71)

double trimmed_mean(std::vector<double> values, double trim_fraction) {
  if (values.empty()) throw AnalysisError("trimmed mean of an empty sample");
  if (!(trim_fraction >= 0.0 && trim_fraction < 0.5)) throw AnalysisError("trim fraction must lie in [0, 0.5)");
  std::sort(values.begin(), values.end());
  const auto cut = static_cast<std::size_t>(std::floor(trim_fraction * static_cast<double>(values.size())));
  double sum = 0.0;
  for (std::size_t i = cut; i + cut < values.size(); ++i) sum += values[i];
  return sum / static_cast<double>(values.size() - 2 * cut);
}

std::optional<double> arithmetic_intensity(double flops, double read_bytes, double write_bytes) {
  const double bytes = read_bytes + write_bytes;
  if (bytes <= 0.0) return std::nullopt;
  return flops / bytes;
}

double arithmetic_throughput(double flops, double latency_ns) {
  if (latency_ns <= 0.0) throw AnalysisError("throughput of a zero-latency subject");
  return flops / (latency_ns / 1e9);
}

double ideal_arithmetic_intensity(const SystemSpec& spec) { return spec.peak_flops / spec.memory_bandwidth_bytes_per_s; }

std::optional<RooflinePoint> classify(std::string subject, double flops, double read_bytes, double write_bytes,
                                      double latency_ns, const SystemSpec& spec) {
  const auto ai = arithmetic_intensity(flops, read_bytes, write_bytes);
  if (!ai || latency_ns <= 0.0) return std::nullopt;
  RooflinePoint p;
  p.subject = std::move(subject);
  p.arithmetic_intensity = *ai;
  p.arithmetic_throughput = arithmetic_throughput(flops, latency_ns);
  p.memory_bound = *ai < ideal_arithmetic_intensity(spec);
  return p;
}

namespace {

template <typename T>
std::vector<T> take(const T* src, std::size_t n) {
  return src ? std::vector<T>(src, src + n) : std::vector<T>(n);
}

// Host copy of xsp_tables_out for a list of AnalysisInputs.
struct Tables {
  std::vector<const AnalysisInput*> groups;
  std::vector<std::string> names;
  std::vector<std::int32_t> status;
  std::vector<std::uint32_t> err_arg, loff, koff, noff;
  std::vector<std::uint32_t> k_name, k_layer;
  std::vector<double> k_lat, k_occ, k_ai, k_tput;
  std::vector<std::uint64_t> k_flops, k_read, k_write;
  std::vector<std::int8_t> k_bound;
  std::vector<std::uint8_t> k_in;
  std::vector<double> l_layer_lat, l_kern_lat, l_occ, l_ai, l_tput, l_nongpu, l_gshare, l_ngshare;
  std::vector<std::uint64_t> l_flops, l_read, l_write, l_count;
  std::vector<std::int8_t> l_bound;
  std::vector<std::uint8_t> l_flag, l_in;
  std::vector<std::uint32_t> n_name;
  std::vector<std::uint64_t> n_count, n_flops, n_read, n_write;
  std::vector<double> n_lat, n_pct, n_occ, n_ai, n_tput;
  std::vector<std::int8_t> n_bound;
  std::vector<double> m_lat, m_klat, m_occ, m_ai, m_tput, m_gpu, m_gpct, m_tp;
  std::vector<std::uint64_t> m_flops, m_read, m_write, m_count;
  std::vector<std::int8_t> m_bound;
  std::vector<std::uint8_t> m_in;
  std::vector<std::string> types;
  std::vector<std::uint32_t> yoff, y_type;
  std::vector<std::uint64_t> y_count;
  std::vector<double> y_lat;
  std::vector<std::int64_t> y_alloc;

  // AnalysisError of group g, as combine() / trimmed_mean raise it
  void check(std::size_t g) const {
    switch (status[g]) {
      case XSP_G_OK: return;
      case XSP_G_NO_RUNS: throw AnalysisError("analysis input holds no runs");
      case XSP_G_LAYER_COUNT: throw AnalysisError("repetitions disagree on layer count");
      case XSP_G_KERNEL_COUNT:
        throw AnalysisError("repetitions disagree on kernel count of layer " + std::to_string(err_arg[g]));
      case XSP_G_BAD_TRIM:
        throw AnalysisError("trim fraction must lie in [0, 0.5)");
      default: throw AnalysisError("analysis failed");
    }
  }
};

std::optional<double> opt(double v) { return std::isnan(v) ? std::nullopt : std::optional<double>(v); }
std::optional<bool> optb(std::int8_t v) { return v < 0 ? std::nullopt : std::optional<bool>(v != 0); }

Tables run_tables(const std::vector<const AnalysisInput*>& groups, const SystemSpec& spec,
                  const AnalysisOptions& options) {
  std::vector<const EntityTree*> trees;
  std::vector<std::uint32_t> first, runs, batch;
  for (const AnalysisInput* in : groups) {
    first.push_back(static_cast<std::uint32_t>(trees.size()));
    runs.push_back(static_cast<std::uint32_t>(in->runs.size()));
    batch.push_back(in->batch_size);
    for (const EntityTree& t : in->runs) trees.push_back(&t);
  }
  const b200::PackedTrees p = b200::pack_trees(trees);
  const xsp_span_cols cols = p.cols();
  const xsp_corr_out corr = p.corr();
  xsp_groups g;
  g.n_groups = static_cast<std::uint32_t>(groups.size());
  g.first_trace = first.data();
  g.n_runs = runs.data();
  g.batch_size = batch.data();
  xsp_system_spec sys{spec.peak_flops, spec.memory_bandwidth_bytes_per_s};
  xsp_analysis_opts o{options.trim_fraction, options.epsilon, options.noise_tolerance, 0};
  xsp_tables_out t;
  b200::check(xsp_analyze_host(b200::ctx(), &cols, &corr, &g, &sys, &o, &t));
  Tables r;
  r.groups = groups;
  r.names = p.names.sorted;
  const std::size_t G = t.n_groups, L = t.n_layers, K = t.n_kernels, N = t.n_names;
  r.status = take(t.group_status, G);
  r.err_arg = take(t.group_err_arg, G);
  r.loff = take(t.group_layer_off, G + 1);
  r.koff = take(t.group_kernel_off, G + 1);
  r.noff = take(t.group_name_off, G + 1);
  r.k_name = take(t.k_name, K);
  r.k_layer = take(t.k_layer, K);
  r.k_lat = take(t.k_lat, K);
  r.k_occ = take(t.k_occ, K);
  r.k_ai = take(t.k_ai, K);
  r.k_tput = take(t.k_tput, K);
  r.k_flops = take(t.k_flops, K);
  r.k_read = take(t.k_read, K);
  r.k_write = take(t.k_write, K);
  r.k_bound = take(t.k_bound, K);
  r.k_in = take(t.k_roofline_in, K);
  r.l_layer_lat = take(t.l_layer_lat, L);
  r.l_kern_lat = take(t.l_kern_lat, L);
  r.l_occ = take(t.l_occ, L);
  r.l_ai = take(t.l_ai, L);
  r.l_tput = take(t.l_tput, L);
  r.l_nongpu = take(t.l_nongpu, L);
  r.l_gshare = take(t.l_gpu_share, L);
  r.l_ngshare = take(t.l_nongpu_share, L);
  r.l_flops = take(t.l_flops, L);
  r.l_read = take(t.l_read, L);
  r.l_write = take(t.l_write, L);
  r.l_count = take(t.l_count, L);
  r.l_bound = take(t.l_bound, L);
  r.l_flag = take(t.l_flagged, L);
  r.l_in = take(t.l_roofline_in, L);
  r.n_name = take(t.n_name, N);
  r.n_count = take(t.n_count, N);
  r.n_flops = take(t.n_flops, N);
  r.n_read = take(t.n_read, N);
  r.n_write = take(t.n_write, N);
  r.n_lat = take(t.n_lat, N);
  r.n_pct = take(t.n_pct, N);
  r.n_occ = take(t.n_occ, N);
  r.n_ai = take(t.n_ai, N);
  r.n_tput = take(t.n_tput, N);
  r.n_bound = take(t.n_bound, N);
  r.m_lat = take(t.m_lat, G);
  r.m_klat = take(t.m_kern_lat, G);
  r.m_occ = take(t.m_occ, G);
  r.m_ai = take(t.m_ai, G);
  r.m_tput = take(t.m_tput, G);
  r.m_gpu = take(t.m_gpu, G);
  r.m_gpct = take(t.m_gpu_pct, G);
  r.m_tp = take(t.m_throughput, G);
  r.m_flops = take(t.m_flops, G);
  r.m_read = take(t.m_read, G);
  r.m_write = take(t.m_write, G);
  r.m_count = take(t.m_count, G);
  r.m_bound = take(t.m_bound, G);
  r.m_in = take(t.m_roofline_in, G);
  const std::size_t Y = t.n_type_rows;
  r.types = p.types.sorted;
  r.yoff = take(t.group_type_off, G + 1);
  r.y_type = take(t.y_type, Y);
  r.y_count = take(t.y_count, Y);
  r.y_lat = take(t.y_lat, Y);
  r.y_alloc = take(t.y_alloc, Y);
  return r;
}

Tables one(const AnalysisInput& input, const SystemSpec& spec, const AnalysisOptions& options) {
  Tables t = run_tables({&input}, spec, options);
  t.check(0);
  return t;
}

// Groups ordered by batch size; a batch size may appear once (analysis.cpp:213-229).
Tables by_batch(const std::vector<AnalysisInput>& groups, const SystemSpec& spec, const AnalysisOptions& options) {
  if (groups.empty()) throw AnalysisError("no runs to analyze");
  std::vector<const AnalysisInput*> order;
  for (const AnalysisInput& g : groups) order.push_back(&g);
  std::stable_sort(order.begin(), order.end(),
                   [](const AnalysisInput* a, const AnalysisInput* b) { return a->batch_size < b->batch_size; });
  for (std::size_t i = 1; i < order.size(); ++i)
    if (order[i]->batch_size == order[i - 1]->batch_size)
      throw AnalysisError("batch size " + std::to_string(order[i]->batch_size) + " appears in more than one group");
  Tables t = run_tables(order, spec, options);
  for (std::size_t g = 0; g < order.size(); ++g) t.check(g);
  return t;
}

const SystemSpec kNoSpec{"", 1.0, 1.0};

}  // namespace

// ---- A1

ThroughputCurve throughput_curve(const std::vector<AnalysisInput>& groups, const AnalysisOptions& options) {
  const Tables t = by_batch(groups, kNoSpec, options);
  ThroughputCurve c;
  for (std::size_t g = 0; g < t.groups.size(); ++g)
    c.points.push_back({t.groups[g]->batch_size, t.m_tp[g], t.m_lat[g]});
  return c;
}

ModelInfoTable a1_model_info(const std::vector<AnalysisInput>& groups, const AnalysisOptions& options) {
  const ThroughputCurve curve = throughput_curve(groups, options);
  ModelInfoTable table;
  for (const ThroughputPoint& p : curve.points) {
    table.rows.push_back({p.batch_size, p.batch_latency_ns, p.throughput});
    if (p.batch_size == 1) table.online_latency_ns = p.batch_latency_ns;
    table.max_throughput = std::max(table.max_throughput, p.throughput);
  }
  return table;
}

OptimalBatch optimal_batch_size(const ThroughputCurve& curve, double epsilon) {
  if (curve.points.empty()) throw AnalysisError("empty throughput curve");
  if (curve.points.size() == 1)
    return {curve.points.front().batch_size, "single-point curve; no doubling step to evaluate"};
  for (std::size_t i = 0; i + 1 < curve.points.size(); ++i)
    if (curve.points[i + 1].throughput <= (1.0 + epsilon) * curve.points[i].throughput)
      return {curve.points[i].batch_size, ""};
  return {curve.points.back().batch_size, ""};
}

// ---- A2..A7

LayerInfoTable a2_layer_table(const AnalysisInput& input, const AnalysisOptions& options) {
  const Tables t = one(input, kNoSpec, options);
  LayerInfoTable table;
  const auto& layers = input.runs.front().root.layers;
  for (std::size_t i = 0; i < layers.size(); ++i) {
    const LayerExec& l = layers[i];
    LayerInfoRow row;
    row.layer_index = l.layer_index;
    row.name = l.span.name;
    row.type = l.layer_type;
    row.shape = b200::tag_string_or_empty(l.span.tags, kTagShape);
    row.latency_ns = t.l_layer_lat[i];
    row.alloc_bytes = l.alloc_bytes;
    table.rows.push_back(std::move(row));
  }
  return table;
}

LayerSeries a3_a4_layer_series(const AnalysisInput& input, const AnalysisOptions& options) {
  const Tables t = one(input, kNoSpec, options);
  LayerSeries s;
  const auto& layers = input.runs.front().root.layers;
  for (std::size_t i = 0; i < layers.size(); ++i) {
    s.latency_ns.push_back(t.l_layer_lat[i]);
    s.alloc_bytes.push_back(layers[i].alloc_bytes);
  }
  return s;
}

// a5 / a6 / a7 rows come from the GPU (k_names_fast keyed by layer type, in
// layer order; rows by total latency desc, type asc — analysis.cpp:315-337).
LayerTypeTable a5_a6_a7_by_type(const AnalysisInput& input, const AnalysisOptions& options) {
  const Tables t = one(input, kNoSpec, options);
  LayerTypeTable table;
  for (std::uint32_t j = t.yoff[0]; j < t.yoff[1]; ++j) {
    LayerTypeRow r;
    r.type = t.types[t.y_type[j]];
    r.count = t.y_count[j];
    r.total_latency_ns = t.y_lat[j];
    r.total_alloc_bytes = t.y_alloc[j];
    table.rows.push_back(std::move(r));
  }
  return table;
}

// ---- A8..A10

namespace {
std::uint32_t layer_index_of(const AnalysisInput& in, std::uint32_t position) {
  return in.runs.front().root.layers[position].layer_index;
}
}  // namespace

KernelInfoTable a8_kernel_table(const AnalysisInput& input, const SystemSpec& spec, const AnalysisOptions& options) {
  const Tables t = one(input, spec, options);
  KernelInfoTable table;
  for (std::size_t k = t.koff[0]; k < t.koff[1]; ++k) {
    KernelInfoRow row;
    row.name = t.names[t.k_name[k]];
    row.layer_index = layer_index_of(input, t.k_layer[k]);
    row.latency_ns = t.k_lat[k];
    row.flops = t.k_flops[k];
    row.dram_read_bytes = t.k_read[k];
    row.dram_write_bytes = t.k_write[k];
    row.achieved_occupancy = t.k_occ[k];
    row.arithmetic_intensity = opt(t.k_ai[k]);
    row.arithmetic_throughput = opt(t.k_tput[k]);
    row.memory_bound = optb(t.k_bound[k]);
    table.rows.push_back(std::move(row));
  }
  return table;
}

RooflineReport a9_kernel_roofline(const AnalysisInput& input, const SystemSpec& spec,
                                  const AnalysisOptions& options) {
  const Tables t = one(input, spec, options);
  RooflineReport rep;
  for (std::size_t k = t.koff[0]; k < t.koff[1]; ++k) {
    std::string subject = "kernel " + std::to_string(k - t.koff[0]) + ": " + t.names[t.k_name[k]];
    if (t.k_in[k])
      rep.points.push_back({std::move(subject), t.k_ai[k], t.k_tput[k], t.k_bound[k] == 1});
    else
      rep.excluded.push_back(std::move(subject));
  }
  return rep;
}

KernelNameTable a10_by_name(const AnalysisInput& input, const SystemSpec& spec, const AnalysisOptions& options) {
  const Tables t = one(input, spec, options);
  KernelNameTable table;
  table.model_latency_ns = t.m_lat[0];
  for (std::size_t n = t.noff[0]; n < t.noff[1]; ++n) {
    KernelNameRow row;
    row.name = t.names[t.n_name[n]];
    row.count = t.n_count[n];
    row.total_latency_ns = t.n_lat[n];
    row.latency_percent = t.n_pct[n];
    row.total_flops = t.n_flops[n];
    row.total_dram_read_bytes = t.n_read[n];
    row.total_dram_write_bytes = t.n_write[n];
    row.weighted_achieved_occupancy = t.n_occ[n];
    row.arithmetic_intensity = opt(t.n_ai[n]);
    row.arithmetic_throughput = opt(t.n_tput[n]);
    row.memory_bound = optb(t.n_bound[n]);
    table.rows.push_back(std::move(row));
  }
  return table;
}

// ---- A11..A14

LayerAggregateTable a11_by_layer(const AnalysisInput& input, const SystemSpec& spec,
                                 const AnalysisOptions& options) {
  const Tables t = one(input, spec, options);
  LayerAggregateTable table;
  const auto& layers = input.runs.front().root.layers;
  for (std::size_t i = 0; i < layers.size(); ++i) {
    LayerAggregateRow row;
    row.layer_index = layers[i].layer_index;
    row.name = layers[i].span.name;
    row.type = layers[i].layer_type;
    row.layer_latency_ns = t.l_layer_lat[i];
    row.kernel_latency_ns = t.l_kern_lat[i];
    row.total_flops = t.l_flops[i];
    row.total_dram_read_bytes = t.l_read[i];
    row.total_dram_write_bytes = t.l_write[i];
    row.weighted_achieved_occupancy = t.l_occ[i];
    row.kernel_count = t.l_count[i];
    row.arithmetic_intensity = opt(t.l_ai[i]);
    row.arithmetic_throughput = opt(t.l_tput[i]);
    row.memory_bound = optb(t.l_bound[i]);
    table.rows.push_back(std::move(row));
  }
  return table;
}

LayerMetricsSeries a12_metrics_per_layer(const AnalysisInput& input, const AnalysisOptions& options) {
  const Tables t = one(input, kNoSpec, options);
  LayerMetricsSeries s;
  s.total_flops = t.l_flops;
  s.total_dram_read_bytes = t.l_read;
  s.total_dram_write_bytes = t.l_write;
  return s;
}

GpuNonGpuTable a13_gpu_vs_nongpu(const AnalysisInput& input, const AnalysisOptions& options) {
  const Tables t = one(input, kNoSpec, options);
  GpuNonGpuTable table;
  table.model_latency_ns = t.m_lat[0];
  const auto& layers = input.runs.front().root.layers;
  for (std::size_t i = 0; i < layers.size(); ++i)
    table.rows.push_back({layers[i].layer_index, t.l_kern_lat[i], t.l_nongpu[i], t.l_gshare[i], t.l_ngshare[i],
                          t.l_flag[i] != 0});
  table.model_gpu_latency_ns = t.m_gpu[0];
  table.model_gpu_percent = t.m_gpct[0];
  return table;
}

RooflineReport a14_layer_roofline(const AnalysisInput& input, const SystemSpec& spec,
                                  const AnalysisOptions& options) {
  const Tables t = one(input, spec, options);
  RooflineReport rep;
  const auto& layers = input.runs.front().root.layers;
  for (std::size_t i = 0; i < layers.size(); ++i) {
    std::string subject = "layer " + std::to_string(layers[i].layer_index) + ": " + layers[i].span.name;
    if (t.l_in[i])
      rep.points.push_back({std::move(subject), t.l_ai[i], t.l_tput[i], t.l_bound[i] == 1});
    else
      rep.excluded.push_back(std::move(subject));
  }
  return rep;
}

// ---- A15 + model roofline

ModelAggregateTable a15_model_aggregate(const std::vector<AnalysisInput>& groups, const SystemSpec& spec,
                                        const AnalysisOptions& options) {
  const Tables t = by_batch(groups, spec, options);
  ModelAggregateTable table;
  for (std::size_t g = 0; g < t.groups.size(); ++g) {
    ModelAggregateRow row;
    row.batch_size = t.groups[g]->batch_size;
    row.model_latency_ns = t.m_lat[g];
    row.kernel_latency_ns = t.m_klat[g];
    row.total_flops = t.m_flops[g];
    row.total_dram_read_bytes = t.m_read[g];
    row.total_dram_write_bytes = t.m_write[g];
    row.weighted_achieved_occupancy = t.m_occ[g];
    row.kernel_count = t.m_count[g];
    row.arithmetic_intensity = opt(t.m_ai[g]);
    row.arithmetic_throughput = opt(t.m_tput[g]);
    row.memory_bound = optb(t.m_bound[g]);
    table.rows.push_back(std::move(row));
  }
  return table;
}

RooflineReport model_roofline(const std::vector<AnalysisInput>& groups, const SystemSpec& spec,
                              const AnalysisOptions& options) {
  const ModelAggregateTable table = a15_model_aggregate(groups, spec, options);
  RooflineReport rep;
  for (const ModelAggregateRow& row : table.rows) {
    std::string subject = "batch " + std::to_string(row.batch_size);
    if (row.arithmetic_intensity && row.kernel_latency_ns > 0.0)
      rep.points.push_back({std::move(subject), *row.arithmetic_intensity, row.arithmetic_throughput.value_or(0.0),
                            row.memory_bound.value_or(false)});
    else
      rep.excluded.push_back(std::move(subject));
  }
  return rep;
}

// ---- stage attribution (analysis.cpp:600-645)

const char* stage_name(Stage stage) {
  switch (stage) {
    case Stage::Beginning: return "B";
    case Stage::Middle: return "M";
    case Stage::End: return "E";
  }
  return "?";
}

StageAttribution stage_attribution(const AnalysisInput& input, const AnalysisOptions& options) {
  const Tables t = one(input, kNoSpec, options);
  const auto& layers = input.runs.front().root.layers;
  const std::size_t n = layers.size();
  StageAttribution out;
  out.layer_count = n;
  out.degenerate = n < 3;
  out.beginning_size = (n + 2) / 3;
  const std::size_t rest = n - out.beginning_size;
  out.middle_size = (rest + 1) / 2;
  out.end_size = rest - out.middle_size;
  auto dominant = [&](auto&& value_of) {
    double sums[3] = {0.0, 0.0, 0.0};
    for (std::size_t i = 0; i < n; ++i) {
      const int s = i < out.beginning_size ? 0 : (i < out.beginning_size + out.middle_size ? 1 : 2);
      sums[s] += value_of(i);
    }
    int best = 0;
    for (int s = 1; s < 3; ++s)
      if (sums[s] > sums[best]) best = s;
    return static_cast<Stage>(best);
  };
  out.latency_stage = dominant([&](std::size_t i) { return t.l_layer_lat[i]; });
  out.alloc_memory_stage = dominant([&](std::size_t i) { return static_cast<double>(layers[i].alloc_bytes); });
  out.flops_stage = dominant([&](std::size_t i) { return static_cast<double>(t.l_flops[i]); });
  out.memory_access_stage =
      dominant([&](std::size_t i) { return static_cast<double>(t.l_read[i] + t.l_write[i]); });
  return out;
}

}  // namespace strata
