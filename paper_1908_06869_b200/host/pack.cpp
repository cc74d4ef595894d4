// libstrata_b200: GPU context and the AoS <-> SoA adapters.
#include "pack.hpp"

#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>

namespace strata::b200 {

namespace {
struct CtxHolder {
  xsp_ctx* c = nullptr;
  ~CtxHolder() {
    if (c) xsp_ctx_destroy(c);
  }
};
thread_local CtxHolder g_ctx;
}  // namespace

xsp_ctx* ctx() {
  if (!g_ctx.c) {
    int dev = 0;
    if (const char* e = std::getenv("XSP_DEVICE")) dev = std::atoi(e);
    const xsp_status st = xsp_ctx_create(dev, &g_ctx.c);
    if (st == XSP_E_NO_DEVICE)
      throw std::runtime_error("strata (B200): no CUDA device available; this build has no CPU fallback");
    if (st != XSP_OK) throw std::runtime_error("strata (B200): xsp_ctx_create failed");
  }
  return g_ctx.c;
}

void check(xsp_status st) {
  if (st != XSP_OK) throw std::runtime_error(std::string("strata (B200): ") + xsp_last_error(ctx()));
}

void Strings::finish() {
  sorted.clear();
  sorted.reserve(id.size());
  for (auto& kv : id) sorted.push_back(kv.first);
  std::sort(sorted.begin(), sorted.end());
  for (std::uint32_t i = 0; i < sorted.size(); ++i) id[sorted[i]] = i;
}

std::uint32_t level_mask(const LevelSet& levels) {
  std::uint32_t m = 0;
  for (Level l : levels) m |= 1u << static_cast<unsigned>(l);
  return m;
}
LevelSet mask_levels(std::uint32_t mask) {
  LevelSet s;
  for (unsigned l = 0; l < 4; ++l)
    if (mask >> l & 1u) s.insert(static_cast<Level>(l));
  return s;
}

std::int64_t tag_int_or0(const TagMap& tags, const char* key) {
  auto it = tags.find(key);
  if (it == tags.end()) return 0;
  if (auto* v = std::get_if<std::int64_t>(&it->second)) return *v;
  if (auto* d = std::get_if<double>(&it->second)) return static_cast<std::int64_t>(*d);
  return 0;
}
std::string tag_string_or_empty(const TagMap& tags, const char* key) {
  auto it = tags.find(key);
  if (it == tags.end()) return {};
  if (auto* s = std::get_if<std::string>(&it->second)) return *s;
  return {};
}

template <typename T>
static T* ptr(const std::vector<T>& v) {
  return v.empty() ? nullptr : const_cast<T*>(v.data());
}

xsp_span_cols PackedSpans::cols() const {
  xsp_span_cols c;
  c.n_spans = span_id.size();
  c.span_id = ptr(span_id);
  c.parent_id = ptr(parent_id);
  c.begin_ns = ptr(begin);
  c.end_ns = ptr(end);
  c.cid = ptr(cid);
  c.flags = ptr(flags);
  c.name_id = ptr(name_id);
  c.n_metric_rows = flops.size();
  c.flops = ptr(flops);
  c.dram_read = ptr(dram_read);
  c.dram_write = ptr(dram_write);
  c.occupancy = ptr(occupancy);
  c.n_layer_rows = alloc_bytes.size();
  c.alloc_bytes = ptr(alloc_bytes);
  c.type_id = ptr(type_id);
  return c;
}

xsp_traces PackedSpans::traces() const {
  xsp_traces t;
  t.n_traces = static_cast<std::uint32_t>(levels.size());
  t.span_off = ptr(span_off);
  t.levels = ptr(levels);
  return t;
}

PackedSpans pack_bundles(const std::vector<const TraceBundle*>& bundles) {
  PackedSpans p;
  std::size_t n = 0;
  for (auto* b : bundles) n += b->spans.size();
  for (auto* b : bundles)
    for (const Span& s : b->spans) {
      p.names.add(s.name);
      if (s.level == Level::Layer) p.types.add(tag_string_or_empty(s.tags, kTagLayerType));
    }
  p.names.finish();
  p.types.finish();
  p.span_id.reserve(n);
  p.parent_id.reserve(n);
  p.begin.reserve(n);
  p.end.reserve(n);
  p.cid.reserve(n);
  p.flags.reserve(n);
  p.name_id.reserve(n);
  p.row.reserve(n);
  p.span_off.push_back(0);
  for (auto* b : bundles) {
    for (const Span& s : b->spans) {
      std::uint8_t f = static_cast<std::uint8_t>(static_cast<unsigned>(s.level) |
                                                 (static_cast<unsigned>(s.kind) << 2));
      if (s.parent_id) f |= XSP_F_PARENT;
      if (s.correlation_id) f |= XSP_F_CID;
      if (auto m = metrics_from_tags(s.tags)) {
        f |= XSP_F_METRICS;
        p.flops.push_back(m->flop_count_sp);
        p.dram_read.push_back(m->dram_read_bytes);
        p.dram_write.push_back(m->dram_write_bytes);
        p.occupancy.push_back(m->achieved_occupancy);
      }
      if (s.level == Level::Layer) {
        p.alloc_bytes.push_back(tag_int_or0(s.tags, kTagAllocBytes));
        p.type_id.push_back(p.types.id.at(tag_string_or_empty(s.tags, kTagLayerType)));
      }
      p.span_id.push_back(s.span_id);
      p.parent_id.push_back(s.parent_id.value_or(0));
      p.begin.push_back(s.begin_ns);
      p.end.push_back(s.end_ns);
      p.cid.push_back(s.correlation_id.value_or(0));
      p.flags.push_back(f);
      p.name_id.push_back(p.names.id.at(s.name));
      p.row.push_back(&s);
    }
    p.span_off.push_back(p.span_id.size());
    p.levels.push_back(level_mask(b->meta.profiling_levels));
  }
  return p;
}

template <typename T>
static std::vector<T> take(const T* src, std::size_t n) {
  return src ? std::vector<T>(src, src + n) : std::vector<T>(n);
}

HostCorr run_correlation(const PackedSpans& p, int mode) {
  const xsp_span_cols cols = p.cols();
  const xsp_traces tr = p.traces();
  xsp_corr_out o;
  check(xsp_correlate_host(ctx(), &cols, &tr, mode, &o));
  HostCorr c;
  const std::uint32_t T = o.n_traces;
  c.n_traces = T;
  c.status = take(o.trace_status, T);
  c.err_row = take(o.trace_err_row, 2ull * T);
  c.model_row = take(o.trace_model_row, T);
  c.t_layer_off = take(o.trace_layer_off, T + 1ull);
  c.t_kernel_off = take(o.trace_kernel_off, T + 1ull);
  c.t_orphan_off = take(o.trace_orphan_off, T + 1ull);
  c.t_amb_off = take(o.trace_amb_off, T + 1ull);
  c.layer_row = take(o.layer_row, o.n_layers);
  c.layer_kernel_off = take(o.layer_kernel_off, o.n_layers + 1);
  c.layer_attr_row = take(o.layer_attr_row, o.n_layers);
  c.k_launch = take(o.kernel_launch_row, o.n_kernels);
  c.k_exec = take(o.kernel_exec_row, o.n_kernels);
  c.k_mrow = take(o.kernel_metric_row, o.n_kernels);
  c.orphan_row = take(o.orphan_row, o.n_orphans);
  c.orphan_reason = take(o.orphan_reason, o.n_orphans);
  c.amb_row = take(o.amb_row, o.n_ambiguities);
  c.amb_cand_off = take(o.amb_cand_off, o.n_ambiguities + 1);
  c.amb_cand_row = take(o.amb_cand_row, o.n_candidates);
  return c;
}

std::string trace_error_text(const PackedSpans& p, const HostCorr& c, std::uint32_t t) {
  const std::uint32_t a = c.err_row[2 * t], b = c.err_row[2 * t + 1];
  switch (c.status[t]) {
    case XSP_T_NO_MODEL:
      return "bundle has no model span; nothing to correlate";
    case XSP_T_MULTI_MODEL:
      return "bundle has more than one model span";
    case XSP_T_SKIP_LEVEL:
      return "span " + std::to_string(p.row[a]->span_id) + " ('" + p.row[a]->name +
             "') is kernel-level but the run did not profile the layer level; parents cannot skip a level";
    case XSP_T_DUP_EXEC_CID:
    case XSP_T_DUP_LAUNCH_CID:
      return "correlation id " + std::to_string(*p.row[b]->correlation_id) + " is shared by " +
             (c.status[t] == XSP_T_DUP_EXEC_CID ? "execution" : "launch") + " spans " +
             std::to_string(p.row[a]->span_id) + " and " + std::to_string(p.row[b]->span_id);
    default:
      return {};
  }
}

std::string orphan_text(const PackedSpans& p, std::uint8_t reason, std::uint32_t row) {
  const Span& s = *p.row[row];
  switch (reason) {
    case XSP_O_LAYER_NON_SYNC: return "layer-level span with non-sync kind";
    case XSP_O_LAYER_BAD_PARENT:
      return "explicit parent " + std::to_string(*s.parent_id) + " is not the model span";
    case XSP_O_LAYER_OUTSIDE_MODEL: return "outside the model interval";
    case XSP_O_KERNEL_BAD_PARENT:
      return "explicit parent " + std::to_string(*s.parent_id) + " is not a layer in the tree";
    case XSP_O_KERNEL_NO_LAYER: return "contained in no layer interval";
    case XSP_O_EXEC_NO_CID: return "execution record without correlation id";
    case XSP_O_LAUNCH_NO_CID: return "launch without correlation id";
    case XSP_O_LAUNCH_NO_EXEC: return "launch has no matching execution record";
    case XSP_O_EXEC_NO_LAUNCH: return "execution record without matching launch";
    default: return "unknown";
  }
}

CorrelationResult unpack_result(const PackedSpans& p, const HostCorr& c, std::uint32_t t) {
  CorrelationResult r;
  r.tree.root.span = *p.row[c.model_row[t]];
  const std::uint32_t l0 = c.t_layer_off[t], l1 = c.t_layer_off[t + 1];
  r.tree.root.layers.resize(l1 - l0);
  for (std::uint32_t g = l0; g < l1; ++g) {
    LayerExec& L = r.tree.root.layers[g - l0];
    const Span& ls = *p.row[c.layer_row[g]];
    L.span = ls;
    L.layer_index = g - l0;
    L.layer_type = tag_string_or_empty(ls.tags, kTagLayerType);
    L.alloc_bytes = tag_int_or0(ls.tags, kTagAllocBytes);
    const std::uint32_t k0 = c.layer_kernel_off[g], k1 = c.layer_kernel_off[g + 1];
    L.kernels.resize(k1 - k0);
    for (std::uint32_t j = k0; j < k1; ++j) {
      KernelExec& K = L.kernels[j - k0];
      K.launch = *p.row[c.k_launch[j]];
      if (c.k_exec[j] != kNone) {
        K.exec = *p.row[c.k_exec[j]];
        K.metrics = metrics_from_tags(K.exec->tags);
      }
    }
  }
  for (std::uint32_t o = c.t_orphan_off[t]; o < c.t_orphan_off[t + 1]; ++o)
    r.tree.orphans.push_back({p.row[c.orphan_row[o]]->span_id, orphan_text(p, c.orphan_reason[o], c.orphan_row[o])});
  for (std::uint32_t a = c.t_amb_off[t]; a < c.t_amb_off[t + 1]; ++a) {
    Ambiguity amb;
    amb.span_id = p.row[c.amb_row[a]]->span_id;
    for (std::uint32_t q = c.amb_cand_off[a]; q < c.amb_cand_off[a + 1]; ++q)
      amb.candidate_parents.push_back(p.row[c.amb_cand_row[q]]->span_id);
    r.ambiguities.push_back(std::move(amb));
  }
  return r;
}

// ---- entity trees -> analysis columns

xsp_span_cols PackedTrees::cols() const {
  xsp_span_cols c;
  c.n_spans = begin.size();
  c.span_id = ptr(zeros64);
  c.parent_id = ptr(zeros64);
  c.begin_ns = ptr(begin);
  c.end_ns = ptr(end);
  c.cid = ptr(zeros64);
  c.flags = ptr(flags);
  c.name_id = ptr(name_id);
  c.n_metric_rows = flops.size();
  c.flops = ptr(flops);
  c.dram_read = ptr(dram_read);
  c.dram_write = ptr(dram_write);
  c.occupancy = ptr(occupancy);
  c.n_layer_rows = alloc_bytes.size();
  c.alloc_bytes = ptr(alloc_bytes);
  c.type_id = ptr(type_id);
  return c;
}

xsp_corr_out PackedTrees::corr() const {
  xsp_corr_out o;
  std::memset(&o, 0, sizeof(o));
  o.n_traces = static_cast<std::uint32_t>(status.size());
  o.n_layers = layer_row.size();
  o.n_kernels = kernel_dur.size();
  o.trace_status = ptr(status);
  o.trace_model_row = ptr(model_row);
  o.trace_layer_off = ptr(t_layer_off);
  o.trace_kernel_off = ptr(t_kernel_off);
  o.trace_amb_off = ptr(t_amb_off);
  o.layer_row = ptr(layer_row);
  o.layer_kernel_off = ptr(layer_kernel_off);
  o.layer_dur = ptr(layer_dur);
  o.layer_attr_row = ptr(layer_attr_row);
  o.kernel_metric_row = ptr(kernel_mrow);
  o.kernel_dur = ptr(kernel_dur);
  o.kernel_name = ptr(kernel_name);
  o.kernel_occ = ptr(kernel_occ);
  return o;
}

PackedTrees pack_trees(const std::vector<const EntityTree*>& trees) {
  PackedTrees p;
  for (auto* t : trees) {
    p.names.add(t->root.span.name);
    for (const LayerExec& L : t->root.layers) {
      p.names.add(L.span.name);
      p.types.add(L.layer_type);
      for (const KernelExec& K : L.kernels) p.names.add(K.kernel_name());
    }
  }
  p.names.finish();
  p.types.finish();
  p.t_layer_off.push_back(0);
  p.t_kernel_off.push_back(0);
  p.t_amb_off.push_back(0);
  p.layer_kernel_off.push_back(0);
  auto add_span = [&](const Span& s, Level lv) {
    p.begin.push_back(s.begin_ns);
    p.end.push_back(s.end_ns);
    p.flags.push_back(static_cast<std::uint8_t>(lv));
    p.name_id.push_back(p.names.id.at(s.name));
    p.zeros64.push_back(0);
    return static_cast<std::uint32_t>(p.begin.size() - 1);
  };
  for (auto* t : trees) {
    p.status.push_back(XSP_T_OK);
    p.model_row.push_back(add_span(t->root.span, Level::Model));
    for (const LayerExec& L : t->root.layers) {
      p.layer_row.push_back(add_span(L.span, Level::Layer));
      p.layer_dur.push_back(L.duration_ns());
      p.layer_attr_row.push_back(static_cast<std::uint32_t>(p.alloc_bytes.size()));
      p.alloc_bytes.push_back(L.alloc_bytes);
      p.type_id.push_back(p.types.id.at(L.layer_type));
      for (const KernelExec& K : L.kernels) {
        p.kernel_dur.push_back(K.duration_ns());
        p.kernel_name.push_back(p.names.id.at(K.kernel_name()));
        if (K.metrics) {
          p.kernel_mrow.push_back(static_cast<std::uint32_t>(p.flops.size()));
          p.flops.push_back(K.metrics->flop_count_sp);
          p.dram_read.push_back(K.metrics->dram_read_bytes);
          p.dram_write.push_back(K.metrics->dram_write_bytes);
          p.occupancy.push_back(K.metrics->achieved_occupancy);
          p.kernel_occ.push_back(K.metrics->achieved_occupancy);
        } else {
          p.kernel_mrow.push_back(kNone);
          p.kernel_occ.push_back(0.0);
        }
      }
      p.layer_kernel_off.push_back(static_cast<std::uint32_t>(p.kernel_dur.size()));
    }
    p.t_layer_off.push_back(static_cast<std::uint32_t>(p.layer_row.size()));
    p.t_kernel_off.push_back(static_cast<std::uint32_t>(p.kernel_dur.size()));
    p.t_amb_off.push_back(0);
  }
  return p;
}

}  // namespace strata::b200
