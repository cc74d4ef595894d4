// The extern "C" boundary (include/xsp.h): context management, argument
// checking, error capture, and the host-buffer entry points.

#include <cstring>
#include <new>
#include <stdexcept>

#include "ctx.h"
#include "prims.cuh"

#define XSP_API extern "C" __attribute__((visibility("default")))

namespace xsp {
void pack_host(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_traces* tr, xsp_packed_cols* out);
uint64_t stage_tables_packed(xsp_ctx* ctx, const xsp_packed_cols* pk, const xsp_span_cols* hc, uint64_t s0,
                             uint64_t s1, uint64_t m0, uint64_t m1, uint64_t l0, uint64_t l1, uint32_t* name_id,
                             uint64_t* flops, uint64_t* rd, uint64_t* wr, double* occ, int64_t* alloc,
                             uint32_t* type_id, const std::string& tag, cudaStream_t st, void* deferred);
uint64_t stage_packed(xsp_ctx* ctx, const xsp_packed_cols* pk, uint64_t s0, uint64_t s1, uint8_t* flags,
                      uint32_t* name_id, uint64_t* begin, uint64_t* end, uint64_t* cid, uint64_t* parent,
                      const std::string& tag, cudaStream_t st, void* deferred = nullptr);
bool run_host_chunked(xsp_ctx* ctx, const xsp_span_cols* hc, const xsp_traces* ht, const xsp_groups* groups,
                      const xsp_system_spec* spec, const xsp_analysis_opts* opts, xsp_corr_out* corr_host,
                      xsp_tables_out* tab_host,
                      const xsp_packed_cols* pk = nullptr);
void run_sort_timeline(xsp_ctx* ctx, uint64_t n, const uint64_t* begin, const uint8_t* flags, const uint64_t* sid,
                       uint32_t T, const uint64_t* off, uint32_t* perm, uint32_t* was_sorted, cudaStream_t st);
void run_validate(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_traces* tr, const xsp_validate_in* vin,
                  xsp_validation_out* out, cudaStream_t st);
void run_report_csv(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr, const xsp_groups* groups,
                    const xsp_tables_out* t, const xsp_string_table* names, const xsp_string_table* types,
                    uint32_t group, int table, char** text, uint64_t* len, int to_host, cudaStream_t st);
void run_ingest_jsonl(xsp_ctx* ctx, const char* htext, const uint64_t* soff, uint32_t S, xsp_ingest_out* out,
                      cudaStream_t st);
void comm_unique_id(void* id);
void comm_init(xsp_ctx* ctx, int world, int rank, const void* id);
void run_combine_tables(xsp_ctx* ctx, xsp_tables_out* local, const uint32_t* group_ids, uint32_t G_local,
                        uint32_t G_total, const uint32_t* l_row_map, int top_k, xsp_tables_out* out,
                        uint64_t* bytes_sent, cudaStream_t st);
void run_resolve(xsp_ctx* ctx, const xsp_span_cols* oc, const xsp_traces* ot, const xsp_span_cols* sc,
                 const xsp_traces* stt, xsp_corr_out* out, cudaStream_t st);
}

namespace {

xsp_status guard(xsp_ctx* ctx, const char* what, auto&& body) {
  if (!ctx) return XSP_E_INVALID;
  ctx->launches = 0;
  const uint64_t xfer0 = xsp::g_xfer_launches;
  try {
    XSP_CUDA(cudaSetDevice(ctx->device));
    body();
    ctx->launches += xsp::g_xfer_launches - xfer0;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw CudaError(std::string("kernel launch: ") + cudaGetErrorString(e));
    ctx->last_error.clear();
    return XSP_OK;
  } catch (const CudaError& e) {
    ctx->last_error = std::string(what) + ": " + e.what();
    return XSP_E_CUDA;
  } catch (const std::invalid_argument& e) {
    ctx->last_error = std::string(what) + ": " + e.what();
    return XSP_E_INVALID;
  } catch (const std::bad_alloc&) {
    ctx->last_error = std::string(what) + ": host allocation failed";
    return XSP_E_NOMEM;
  } catch (const std::runtime_error& e) {
    ctx->last_error = std::string(what) + ": " + e.what();
    if (std::string(e.what()) == "UNSORTED") {
      ctx->last_error = std::string(what) + ": a trace is not in timeline order (begin_ns, rank, span_id)";
      return XSP_E_UNSORTED;
    }
    return XSP_E_INVALID;
  } catch (const std::exception& e) {  // no C++ exception crosses the C ABI
    ctx->last_error = std::string(what) + ": internal error: " + e.what();
    return XSP_E_INVALID;
  }
}

void check_cols(const xsp_span_cols* c, const xsp_traces* t) {
  if (!c) throw std::invalid_argument("null columns");
  if (c->n_spans && (!c->span_id || !c->parent_id || !c->begin_ns || !c->end_ns || !c->cid || !c->flags ||
                     !c->name_id))
    throw std::invalid_argument("null span column");
  if (c->n_metric_rows && (!c->flops || !c->dram_read || !c->dram_write || !c->occupancy))
    throw std::invalid_argument("null metric column");
  if (c->n_layer_rows && (!c->alloc_bytes || !c->type_id)) throw std::invalid_argument("null layer column");
  if (t && (!t->span_off || (t->n_traces && !t->levels))) throw std::invalid_argument("null trace column");
}

template <typename T>
T* to_dev(xsp_ctx* ctx, const std::string& name, const T* src, uint64_t count, cudaStream_t st) {
  T* d = ctx->d<T>("h2d." + name, count ? count : 1);
  if (count) {
    XSP_CUDA(cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, st));
    ctx->h2d_bytes += count * sizeof(T);
  }
  return d;
}

template <typename T>
T* to_host(xsp_ctx* ctx, const std::string& name, const T* src, uint64_t count, cudaStream_t st) {
  T* h = ctx->h<T>("d2h." + name, count ? count : 1);
  if (count) {
    XSP_CUDA(cudaMemcpyAsync(h, src, count * sizeof(T), cudaMemcpyDeviceToHost, st));
    ctx->d2h_bytes += count * sizeof(T);
  }
  return h;
}

xsp_span_cols upload_cols(xsp_ctx* ctx, const xsp_span_cols* hc, cudaStream_t st) {
  const uint64_t n = hc->n_spans;
  xsp_span_cols dc;
  dc.n_spans = n;
  dc.span_id = to_dev(ctx, "span_id", hc->span_id, n, st);
  dc.parent_id = to_dev(ctx, "parent_id", hc->parent_id, n, st);
  dc.begin_ns = to_dev(ctx, "begin", hc->begin_ns, n, st);
  dc.end_ns = to_dev(ctx, "end", hc->end_ns, n, st);
  dc.cid = to_dev(ctx, "cid", hc->cid, n, st);
  dc.flags = to_dev(ctx, "flags", hc->flags, n, st);
  dc.name_id = to_dev(ctx, "name", hc->name_id, n, st);
  dc.n_metric_rows = hc->n_metric_rows;
  dc.flops = to_dev(ctx, "flops", hc->flops, hc->n_metric_rows, st);
  dc.dram_read = to_dev(ctx, "read", hc->dram_read, hc->n_metric_rows, st);
  dc.dram_write = to_dev(ctx, "write", hc->dram_write, hc->n_metric_rows, st);
  dc.occupancy = to_dev(ctx, "occ", hc->occupancy, hc->n_metric_rows, st);
  dc.n_layer_rows = hc->n_layer_rows;
  dc.alloc_bytes = to_dev(ctx, "alloc", hc->alloc_bytes, hc->n_layer_rows, st);
  dc.type_id = to_dev(ctx, "type", hc->type_id, hc->n_layer_rows, st);
  return dc;
}

xsp_traces upload_traces(xsp_ctx* ctx, const xsp_traces* ht, cudaStream_t st) {
  xsp_traces dt;
  dt.n_traces = ht->n_traces;
  dt.span_off = to_dev(ctx, "span_off", ht->span_off, (uint64_t)ht->n_traces + 1, st);
  dt.levels = to_dev(ctx, "levels", ht->levels, ht->n_traces, st);
  return dt;
}

// the columns analysis / leveling read from a (host) correlation
xsp_corr_out upload_corr(xsp_ctx* ctx, const xsp_corr_out* h, cudaStream_t st) {
  xsp_corr_out d = *h;
  const uint64_t T = h->n_traces, L = h->n_layers, K = h->n_kernels;
  d.trace_status = to_dev(ctx, "c.t_status", h->trace_status, T, st);
  d.trace_model_row = to_dev(ctx, "c.t_model", h->trace_model_row, T, st);
  d.trace_layer_off = to_dev(ctx, "c.t_loff", h->trace_layer_off, T + 1, st);
  d.trace_kernel_off = to_dev(ctx, "c.t_koff", h->trace_kernel_off, T + 1, st);
  d.trace_amb_off = to_dev(ctx, "c.t_aoff", h->trace_amb_off, T + 1, st);
  d.layer_row = to_dev(ctx, "c.l_row", h->layer_row, L, st);
  d.layer_kernel_off = to_dev(ctx, "c.l_koff", h->layer_kernel_off, L + 1, st);
  d.layer_dur = to_dev(ctx, "c.l_dur", h->layer_dur, L, st);
  d.layer_attr_row = h->layer_attr_row ? to_dev(ctx, "c.l_attr", h->layer_attr_row, L, st) : nullptr;
  d.kernel_metric_row = to_dev(ctx, "c.k_mrow", h->kernel_metric_row, K, st);
  d.kernel_dur = to_dev(ctx, "c.k_dur", h->kernel_dur, K, st);
  d.kernel_name = to_dev(ctx, "c.k_name", h->kernel_name, K, st);
  d.kernel_occ = to_dev(ctx, "c.k_occ", h->kernel_occ, K, st);
  return d;
}

void download_corr(xsp_ctx* ctx, const xsp_corr_out& dcorr, xsp_corr_out* c, cudaStream_t st) {
  const uint32_t T = dcorr.n_traces;
  *c = dcorr;
  c->trace_status = to_host(ctx, "t_status", dcorr.trace_status, T, st);
  c->trace_err_row = to_host(ctx, "t_err", dcorr.trace_err_row, 2ull * T, st);
  c->trace_model_row = to_host(ctx, "t_model", dcorr.trace_model_row, T, st);
  c->trace_layer_off = to_host(ctx, "t_loff", dcorr.trace_layer_off, T + 1ull, st);
  c->trace_kernel_off = to_host(ctx, "t_koff", dcorr.trace_kernel_off, T + 1ull, st);
  c->trace_orphan_off = to_host(ctx, "t_ooff", dcorr.trace_orphan_off, T + 1ull, st);
  c->trace_amb_off = to_host(ctx, "t_aoff", dcorr.trace_amb_off, T + 1ull, st);
  c->layer_row = to_host(ctx, "l_row", dcorr.layer_row, dcorr.n_layers, st);
  c->layer_kernel_off = to_host(ctx, "l_koff", dcorr.layer_kernel_off, dcorr.n_layers + 1, st);
  c->layer_dur = ctx->host_out == XSP_HOST_OUT_ROWS ? nullptr : to_host(ctx, "l_dur", dcorr.layer_dur, dcorr.n_layers, st);
  c->layer_attr_row = to_host(ctx, "l_attr", dcorr.layer_attr_row, dcorr.n_layers, st);
  c->kernel_launch_row = to_host(ctx, "k_launch", dcorr.kernel_launch_row, dcorr.n_kernels, st);
  c->kernel_exec_row = to_host(ctx, "k_exec", dcorr.kernel_exec_row, dcorr.n_kernels, st);
  c->kernel_metric_row = to_host(ctx, "k_mrow", dcorr.kernel_metric_row, dcorr.n_kernels, st);
  c->kernel_dur = ctx->host_out == XSP_HOST_OUT_ROWS ? nullptr : to_host(ctx, "k_dur", dcorr.kernel_dur, dcorr.n_kernels, st);
  c->kernel_name = ctx->host_out == XSP_HOST_OUT_ROWS ? nullptr : to_host(ctx, "k_name", dcorr.kernel_name, dcorr.n_kernels, st);
  c->kernel_occ = ctx->host_out == XSP_HOST_OUT_ROWS ? nullptr : to_host(ctx, "k_occ", dcorr.kernel_occ, dcorr.n_kernels, st);
  c->orphan_row = to_host(ctx, "o_row", dcorr.orphan_row, dcorr.n_orphans, st);
  c->orphan_reason = to_host(ctx, "o_reason", dcorr.orphan_reason, dcorr.n_orphans, st);
  c->amb_row = to_host(ctx, "a_row", dcorr.amb_row, dcorr.n_ambiguities, st);
  c->amb_cand_off = to_host(ctx, "a_coff", dcorr.amb_cand_off, dcorr.n_ambiguities + 1, st);
  c->amb_cand_row = to_host(ctx, "a_crow", dcorr.amb_cand_row, dcorr.n_candidates, st);
}

void download_tables(xsp_ctx* ctx, const xsp_tables_out& dtab, const xsp_analysis_opts* opts, xsp_tables_out* t,
                     cudaStream_t st) {
  const uint32_t G = dtab.n_groups;
  const uint64_t L = dtab.n_layers, K = dtab.n_kernels, N = dtab.n_names;
  const uint64_t tk = opts->top_k ? opts->top_k : 1;
  *t = dtab;
#define BACK(field, count) t->field = to_host(ctx, "t." #field, dtab.field, (count), st)
  BACK(group_status, G);
  BACK(group_err_arg, G);
  BACK(group_layer_off, G + 1ull);
  BACK(group_kernel_off, G + 1ull);
  BACK(group_name_off, G + 1ull);
  BACK(k_name, K); BACK(k_layer, K); BACK(k_lat, K); BACK(k_flops, K); BACK(k_read, K);
  BACK(k_write, K); BACK(k_occ, K); BACK(k_ai, K); BACK(k_tput, K); BACK(k_bound, K);
  BACK(k_roofline_in, K);
  BACK(l_index, L); BACK(l_row, L); BACK(l_layer_lat, L); BACK(l_kern_lat, L); BACK(l_flops, L);
  BACK(l_read, L); BACK(l_write, L); BACK(l_occ, L); BACK(l_count, L); BACK(l_ai, L);
  BACK(l_tput, L); BACK(l_bound, L); BACK(l_nongpu, L); BACK(l_gpu_share, L);
  BACK(l_nongpu_share, L); BACK(l_flagged, L); BACK(l_roofline_in, L); BACK(l_topk, L * tk);
  BACK(n_name, N); BACK(n_count, N); BACK(n_lat, N); BACK(n_pct, N); BACK(n_flops, N);
  BACK(n_read, N); BACK(n_write, N); BACK(n_occ, N); BACK(n_ai, N); BACK(n_tput, N);
  BACK(n_bound, N);
  BACK(m_lat, G); BACK(m_kern_lat, G); BACK(m_flops, G); BACK(m_read, G); BACK(m_write, G);
  BACK(m_occ, G); BACK(m_count, G); BACK(m_ai, G); BACK(m_tput, G); BACK(m_bound, G);
  BACK(m_gpu, G); BACK(m_gpu_pct, G); BACK(m_throughput, G); BACK(m_roofline_in, G);
  const uint64_t Y = dtab.n_type_rows;
  BACK(group_type_off, G + 1ull);
  BACK(y_type, Y); BACK(y_count, Y); BACK(y_lat, Y); BACK(y_alloc, Y);
#undef BACK
}

void download_overhead(xsp_ctx* ctx, const xsp_overhead_out& d, xsp_overhead_out* o, cudaStream_t st) {
  *o = d;
  if (d.status == XSP_L_AMBIGUOUS || d.status == XSP_L_TRACE_FAILED || d.n_sets == 0) return;
  const uint64_t E = d.n_events, S = d.n_sets;
  o->ev_level = to_host(ctx, "l.ev_level", d.ev_level, E, st);
  o->ev_layer = to_host(ctx, "l.ev_layer", d.ev_layer, E, st);
  o->ev_kernel = to_host(ctx, "l.ev_kernel", d.ev_kernel, E, st);
  o->lat = to_host(ctx, "l.lat", d.lat, S * E, st);
  o->overhead = to_host(ctx, "l.ov", d.overhead, (S - 1) * E, st);
  o->step_flags = to_host(ctx, "l.flags", d.step_flags, (S - 1) * E, st);
  o->accurate = to_host(ctx, "l.acc", d.accurate, E, st);
}

}  // namespace

XSP_API int xsp_abi_version(void) { return XSP_ABI_VERSION; }

XSP_API xsp_status xsp_ctx_create(int device, xsp_ctx** out) {
  if (!out) return XSP_E_INVALID;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return XSP_E_NO_DEVICE;
  if (device < 0 || device >= n) return XSP_E_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return XSP_E_CUDA;
  auto* ctx = new (std::nothrow) xsp_ctx;
  if (!ctx) return XSP_E_NOMEM;
  ctx->device = device;
  *out = ctx;
  return XSP_OK;
}

XSP_API void xsp_ctx_destroy(xsp_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  delete ctx;
}

XSP_API const char* xsp_last_error(const xsp_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

XSP_API uint64_t xsp_last_launch_count(const xsp_ctx* ctx) { return ctx ? ctx->launches : 0; }

XSP_API void xsp_last_transfer_bytes(const xsp_ctx* ctx, uint64_t* h2d, uint64_t* d2h) {
  if (h2d) *h2d = ctx ? ctx->h2d_bytes : 0;
  if (d2h) *d2h = ctx ? ctx->d2h_bytes : 0;
}

XSP_API void* xsp_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) return nullptr;
  return p;
}

XSP_API void xsp_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

XSP_API xsp_status xsp_set_host_outputs(xsp_ctx* ctx, uint32_t mode) {
  if (!ctx) return XSP_E_INVALID;
  if (mode != XSP_HOST_OUT_ALL && mode != XSP_HOST_OUT_ROWS) {
    ctx->last_error = "xsp_set_host_outputs: unknown mode";
    return XSP_E_INVALID;
  }
  ctx->host_out = mode;
  return XSP_OK;
}

XSP_API void xsp_set_profiling(xsp_ctx* ctx, int enabled) {
  if (ctx) ctx->profiling = enabled != 0;
}

XSP_API void xsp_stage_reset(xsp_ctx* ctx) {
  if (!ctx) return;
  ctx->stage_collect();
  for (auto& s : ctx->stages) {
    s.ms = 0.0;
    s.calls = 0;
  }
}

XSP_API int xsp_stage_times(xsp_ctx* ctx, int max, const char** names, double* total_ms, uint64_t* count) {
  if (!ctx) return 0;
  ctx->stage_collect();
  int n = static_cast<int>(ctx->stages.size());
  for (int i = 0; i < n && i < max; ++i) {
    if (names) names[i] = ctx->stages[i].name.c_str();
    if (total_ms) total_ms[i] = ctx->stages[i].ms;
    if (count) count[i] = ctx->stages[i].calls;
  }
  return n;
}

XSP_API xsp_status xsp_copy_to_host(xsp_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guard(ctx, "xsp_copy_to_host", [&] {
    if (bytes) XSP_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
  });
}

XSP_API xsp_status xsp_correlate(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_traces* traces, int mode,
                                 xsp_corr_out* out, void* stream) {
  return guard(ctx, "xsp_correlate", [&] {
    check_cols(cols, traces);
    if (!traces || !out) throw std::invalid_argument("null argument");
    std::memset(out, 0, sizeof(*out));
    xsp::run_correlate(ctx, cols, traces, mode, out, static_cast<cudaStream_t>(stream));
  });
}

XSP_API xsp_status xsp_analyze(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                               const xsp_groups* groups, const xsp_system_spec* spec,
                               const xsp_analysis_opts* opts, xsp_tables_out* out, void* stream) {
  return guard(ctx, "xsp_analyze", [&] {
    if (!cols || !corr || !groups || !spec || !opts || !out) throw std::invalid_argument("null argument");
    if (groups->n_groups && (!groups->first_trace || !groups->n_runs || !groups->batch_size))
      throw std::invalid_argument("null group column");
    std::memset(out, 0, sizeof(*out));
    xsp::run_analyze(ctx, cols, corr, groups, spec, opts, out, static_cast<cudaStream_t>(stream));
  });
}

XSP_API xsp_status xsp_run(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_traces* traces,
                           const xsp_groups* groups, const xsp_system_spec* spec, const xsp_analysis_opts* opts,
                           xsp_corr_out* corr, xsp_tables_out* tables, void* stream) {
  return guard(ctx, "xsp_run", [&] {
    check_cols(cols, traces);
    if (!traces || !corr || !groups || !spec || !opts || !tables) throw std::invalid_argument("null argument");
    if (groups->n_groups && (!groups->first_trace || !groups->n_runs || !groups->batch_size))
      throw std::invalid_argument("null group column");
    std::memset(corr, 0, sizeof(*corr));
    std::memset(tables, 0, sizeof(*tables));
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    xsp::run_correlate(ctx, cols, traces, 1, corr, st);
    xsp::run_analyze(ctx, cols, corr, groups, spec, opts, tables, st);
  });
}

XSP_API xsp_status xsp_leveled(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                               const xsp_level_sets* sets, const xsp_analysis_opts* opts,
                               xsp_overhead_out* out, void* stream) {
  return guard(ctx, "xsp_leveled", [&] {
    if (!cols || !corr || !sets || !opts || !out) throw std::invalid_argument("null argument");
    if (!sets->set_off || (sets->n_sets && (!sets->trace_idx || !sets->levels)))
      throw std::invalid_argument("null level-set column");
    std::memset(out, 0, sizeof(*out));
    xsp::run_leveled(ctx, cols, corr, sets, opts, out, static_cast<cudaStream_t>(stream));
  });
}

XSP_API xsp_status xsp_leveled_batch(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                                     uint32_t n_groups, const xsp_level_sets* sets, const xsp_analysis_opts* opts,
                                     xsp_overhead_out* outs, void* stream) {
  return guard(ctx, "xsp_leveled_batch", [&] {
    if (!cols || !corr || !opts || (n_groups && (!sets || !outs))) throw std::invalid_argument("null argument");
    for (uint32_t g = 0; g < n_groups; ++g)
      if (!sets[g].set_off || (sets[g].n_sets && (!sets[g].trace_idx || !sets[g].levels)))
        throw std::invalid_argument("null level-set column");
    if (n_groups) std::memset(outs, 0, n_groups * sizeof(*outs));
    xsp::run_leveled_batch(ctx, cols, corr, n_groups, sets, opts, outs, static_cast<cudaStream_t>(stream));
  });
}

XSP_API xsp_status xsp_resolve_serialized(xsp_ctx* ctx, const xsp_span_cols* oc, const xsp_traces* ot,
                                          const xsp_span_cols* sc, const xsp_traces* stt, xsp_corr_out* out,
                                          void* stream) {
  return guard(ctx, "xsp_resolve_serialized", [&] {
    check_cols(oc, ot);
    check_cols(sc, stt);
    if (!ot || !stt || !out) throw std::invalid_argument("null argument");
    std::memset(out, 0, sizeof(*out));
    xsp::run_resolve(ctx, oc, ot, sc, stt, out, static_cast<cudaStream_t>(stream));
  });
}

XSP_API xsp_status xsp_resolve_serialized_host(xsp_ctx* ctx, const xsp_span_cols* hoc, const xsp_traces* hot,
                                               const xsp_span_cols* hsc, const xsp_traces* hst,
                                               xsp_corr_out* out) {
  return guard(ctx, "xsp_resolve_serialized_host", [&] {
    check_cols(hoc, hot);
    check_cols(hsc, hst);
    if (!hot || !hst || !out) throw std::invalid_argument("null argument");
    cudaStream_t st = nullptr;
    ctx->h2d_bytes = ctx->d2h_bytes = 0;
    xsp_span_cols doc = upload_cols(ctx, hoc, st);
    xsp_traces dot = upload_traces(ctx, hot, st);
    // the serialized batch under its own buffer names
    ctx->tag = ".ser";
    xsp_span_cols dsc = upload_cols(ctx, hsc, st);
    xsp_traces dst = upload_traces(ctx, hst, st);
    ctx->tag.clear();
    xsp_corr_out dcorr;
    std::memset(&dcorr, 0, sizeof(dcorr));
    xsp::run_resolve(ctx, &doc, &dot, &dsc, &dst, &dcorr, st);
    download_corr(ctx, dcorr, out, st);
    XSP_CUDA(cudaStreamSynchronize(st));
  });
}

XSP_API xsp_status xsp_validate(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_traces* traces,
                                const xsp_validate_in* in, xsp_validation_out* out, void* stream) {
  return guard(ctx, "xsp_validate", [&] {
    check_cols(cols, traces);
    if (!traces || !out) throw std::invalid_argument("null argument");
    std::memset(out, 0, sizeof(*out));
    xsp::run_validate(ctx, cols, traces, in, out, static_cast<cudaStream_t>(stream));
  });
}

XSP_API xsp_status xsp_validate_host(xsp_ctx* ctx, const xsp_span_cols* hc, const xsp_traces* ht,
                                     const xsp_validate_in* hin, xsp_validation_out* out) {
  return guard(ctx, "xsp_validate_host", [&] {
    check_cols(hc, ht);
    if (!ht || !out) throw std::invalid_argument("null argument");
    cudaStream_t st = nullptr;
    ctx->h2d_bytes = ctx->d2h_bytes = 0;
    xsp_span_cols dc = upload_cols(ctx, hc, st);
    xsp_traces dt = upload_traces(ctx, ht, st);
    xsp_validate_in din{nullptr, nullptr, nullptr};
    if (hin) {
      const uint64_t n = hc->n_spans;
      if (hin->trace_id) din.trace_id = to_dev(ctx, "v.trace_id", hin->trace_id, n, st);
      if (hin->meta_trace_id) din.meta_trace_id = to_dev(ctx, "v.meta_tid", hin->meta_trace_id, ht->n_traces, st);
      if (hin->tag_bits) din.tag_bits = to_dev(ctx, "v.tag_bits", hin->tag_bits, n, st);
    }
    xsp_validation_out d;
    std::memset(&d, 0, sizeof(d));
    xsp::run_validate(ctx, &dc, &dt, &din, &d, st);
    out->n_issues = d.n_issues;
    out->trace_issue_off = to_host(ctx, "v.trace_off", d.trace_issue_off, (uint64_t)ht->n_traces + 1, st);
    out->issue_row = to_host(ctx, "v.row", d.issue_row, d.n_issues, st);
    out->issue_rule = to_host(ctx, "v.rule", d.issue_rule, d.n_issues, st);
    XSP_CUDA(cudaStreamSynchronize(st));
  });
}

XSP_API xsp_status xsp_sort_timeline(xsp_ctx* ctx, uint64_t n, const uint64_t* begin, const uint8_t* flags,
                                     const uint64_t* span_id, uint32_t n_traces, const uint64_t* span_off,
                                     uint32_t* perm, int* was_sorted, void* stream) {
  return guard(ctx, "xsp_sort_timeline", [&] {
    if (!span_off || !perm || (n && (!begin || !flags || !span_id))) throw std::invalid_argument("null argument");
    if (n >= 0xFFFFFFF0ull) throw std::invalid_argument("more than 2^32-16 spans in one call");
    uint32_t sorted = 0;
    xsp::run_sort_timeline(ctx, n, begin, flags, span_id, n_traces, span_off, perm, &sorted,
                           static_cast<cudaStream_t>(stream));
    if (was_sorted) *was_sorted = (int)sorted;
  });
}

XSP_API xsp_status xsp_sort_timeline_host(xsp_ctx* ctx, uint64_t n, const uint64_t* begin, const uint8_t* flags,
                                          const uint64_t* span_id, uint32_t n_traces, const uint64_t* span_off,
                                          uint32_t* perm, int* was_sorted) {
  return guard(ctx, "xsp_sort_timeline_host", [&] {
    if (!span_off || !perm || (n && (!begin || !flags || !span_id))) throw std::invalid_argument("null argument");
    if (n >= 0xFFFFFFF0ull) throw std::invalid_argument("more than 2^32-16 spans in one call");
    cudaStream_t st = nullptr;
    const uint64_t* db = to_dev(ctx, "s.begin", begin, n, st);
    const uint8_t* df = to_dev(ctx, "s.flags", flags, n, st);
    const uint64_t* ds = to_dev(ctx, "s.sid", span_id, n, st);
    const uint64_t* doff = to_dev(ctx, "s.off", span_off, (uint64_t)n_traces + 1, st);
    uint32_t* dperm = ctx->d<uint32_t>("s.perm", n ? n : 1);
    uint32_t sorted = 0;
    xsp::run_sort_timeline(ctx, n, db, df, ds, n_traces, doff, dperm, &sorted, st);
    if (n) XSP_CUDA(cudaMemcpy(perm, dperm, n * 4, cudaMemcpyDeviceToHost));
    if (was_sorted) *was_sorted = (int)sorted;
  });
}

XSP_API xsp_status xsp_correlate_host(xsp_ctx* ctx, const xsp_span_cols* hc, const xsp_traces* ht, int mode,
                                      xsp_corr_out* out) {
  return guard(ctx, "xsp_correlate_host", [&] {
    check_cols(hc, ht);
    if (!ht || !out) throw std::invalid_argument("null argument");
    cudaStream_t st = nullptr;
    ctx->h2d_bytes = ctx->d2h_bytes = 0;
    xsp_span_cols dc = upload_cols(ctx, hc, st);
    xsp_traces dt = upload_traces(ctx, ht, st);
    xsp_corr_out dcorr;
    std::memset(&dcorr, 0, sizeof(dcorr));
    xsp::run_correlate(ctx, &dc, &dt, mode, &dcorr, st);
    download_corr(ctx, dcorr, out, st);
    XSP_CUDA(cudaStreamSynchronize(st));
  });
}

XSP_API xsp_status xsp_analyze_host(xsp_ctx* ctx, const xsp_span_cols* hc, const xsp_corr_out* hcorr,
                                    const xsp_groups* groups, const xsp_system_spec* spec,
                                    const xsp_analysis_opts* opts, xsp_tables_out* out) {
  return guard(ctx, "xsp_analyze_host", [&] {
    check_cols(hc, nullptr);
    if (!hcorr || !groups || !spec || !opts || !out) throw std::invalid_argument("null argument");
    cudaStream_t st = nullptr;
    ctx->h2d_bytes = ctx->d2h_bytes = 0;
    xsp_span_cols dc = upload_cols(ctx, hc, st);
    xsp_corr_out dcorr = upload_corr(ctx, hcorr, st);
    xsp_tables_out dtab;
    std::memset(&dtab, 0, sizeof(dtab));
    xsp::run_analyze(ctx, &dc, &dcorr, groups, spec, opts, &dtab, st);
    download_tables(ctx, dtab, opts, out, st);
    XSP_CUDA(cudaStreamSynchronize(st));
  });
}

XSP_API xsp_status xsp_report_csv(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                                  const xsp_groups* groups, const xsp_tables_out* tables,
                                  const xsp_string_table* names, const xsp_string_table* types, uint32_t group,
                                  int table, char** text, uint64_t* len, void* stream) {
  return guard(ctx, "xsp_report_csv", [&] {
    if (!cols || !corr || !groups || !tables || !names || !text || !len) throw std::invalid_argument("null argument");
    xsp::run_report_csv(ctx, cols, corr, groups, tables, names, types, group, table, text, len, 0,
                        static_cast<cudaStream_t>(stream));
  });
}

XSP_API xsp_status xsp_report_csv_host(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                                       const xsp_groups* groups, const xsp_tables_out* tables,
                                       const xsp_string_table* names, const xsp_string_table* types,
                                       uint32_t group, int table, char** text, uint64_t* len, void* stream) {
  return guard(ctx, "xsp_report_csv_host", [&] {
    if (!cols || !corr || !groups || !tables || !names || !text || !len) throw std::invalid_argument("null argument");
    xsp::run_report_csv(ctx, cols, corr, groups, tables, names, types, group, table, text, len, 1,
                        static_cast<cudaStream_t>(stream));
  });
}

XSP_API xsp_status xsp_ingest_jsonl(xsp_ctx* ctx, const char* text, const uint64_t* stream_off,
                                    uint32_t n_streams, xsp_ingest_out* out, void* stream) {
  return guard(ctx, "xsp_ingest_jsonl", [&] {
    if (!out || !stream_off || (n_streams && !text)) throw std::invalid_argument("null argument");
    xsp::run_ingest_jsonl(ctx, text, stream_off, n_streams, out, static_cast<cudaStream_t>(stream));
  });
}

XSP_API xsp_status xsp_pack_host(xsp_ctx* ctx, const xsp_span_cols* hc, const xsp_traces* ht,
                                 xsp_packed_cols* out) {
  return guard(ctx, "xsp_pack_host", [&] {
    check_cols(hc, ht);
    if (!ht || !out) throw std::invalid_argument("null argument");
    xsp::pack_host(ctx, hc, ht, out);
  });
}

XSP_API xsp_status xsp_run_host_packed(xsp_ctx* ctx, const xsp_packed_cols* pk, const xsp_span_cols* hc,
                                       const xsp_traces* ht, const xsp_groups* groups, const xsp_system_spec* spec,
                                       const xsp_analysis_opts* opts, xsp_corr_out* corr_host,
                                       xsp_tables_out* tab_host, void* stream) {
  return guard(ctx, "xsp_run_host_packed", [&] {
    if (!pk || !hc || !ht || !groups || !spec || !opts || !corr_host || !tab_host)
      throw std::invalid_argument("null argument");
    if (pk->n_spans != hc->n_spans) throw std::invalid_argument("packed and host columns disagree on n_spans");
    if (groups->n_groups && (!groups->first_trace || !groups->n_runs || !groups->batch_size))
      throw std::invalid_argument("null group column");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ctx->h2d_bytes = ctx->d2h_bytes = 0;
    if (xsp::run_host_chunked(ctx, hc, ht, groups, spec, opts, corr_host, tab_host, pk)) return;
    // single shot: span_id and the tables as xsp_run_host uploads them, the
    // span columns unpacked on the device
    const uint64_t n = pk->n_spans;
    const uint64_t nm_rows = hc->n_metric_rows, nl_rows = hc->n_layer_rows;
    xsp_span_cols dc;
    dc.n_spans = n;
    dc.span_id = to_dev(ctx, "span_id", hc->span_id, n, st);
    dc.n_metric_rows = nm_rows;
    dc.n_layer_rows = nl_rows;
    uint64_t* d_fl = ctx->d<uint64_t>("pk1.fl", nm_rows + 1);
    uint64_t* d_rd = ctx->d<uint64_t>("pk1.rd", nm_rows + 1);
    uint64_t* d_wr = ctx->d<uint64_t>("pk1.wr", nm_rows + 1);
    double* d_oc = ctx->d<double>("pk1.oc", nm_rows + 1);
    int64_t* d_al = ctx->d<int64_t>("pk1.al", nl_rows + 1);
    uint32_t* d_ty = ctx->d<uint32_t>("pk1.ty", nl_rows + 1);
    uint8_t* f = ctx->d<uint8_t>("pk1.f", n + 1);
    uint32_t* nm = ctx->d<uint32_t>("pk1.n", n + 1);
    uint64_t* b = ctx->d<uint64_t>("pk1.b", n + 1);
    uint64_t* e = ctx->d<uint64_t>("pk1.e", n + 1);
    uint64_t* c = ctx->d<uint64_t>("pk1.c", n + 1);
    uint64_t* p = ctx->d<uint64_t>("pk1.p", n + 1);
    ctx->h2d_bytes += xsp::stage_packed(ctx, pk, 0, n, f, nm, b, e, c, p, "pk1.", st);
    ctx->h2d_bytes += xsp::stage_tables_packed(ctx, pk, hc, 0, n, 0, nm_rows, 0, nl_rows, nm, d_fl, d_rd, d_wr, d_oc,
                                               d_al, d_ty, "pk1t.", st, nullptr);
    dc.flops = d_fl;
    dc.dram_read = d_rd;
    dc.dram_write = d_wr;
    dc.occupancy = d_oc;
    dc.alloc_bytes = d_al;
    dc.type_id = d_ty;
    dc.flags = f;
    dc.name_id = nm;
    dc.begin_ns = b;
    dc.end_ns = e;
    dc.cid = c;
    dc.parent_id = p;
    xsp_traces dt = upload_traces(ctx, ht, st);
    xsp_corr_out dcorr;
    std::memset(&dcorr, 0, sizeof(dcorr));
    xsp::run_correlate(ctx, &dc, &dt, 0, &dcorr, st);
    xsp_tables_out dtab;
    std::memset(&dtab, 0, sizeof(dtab));
    xsp::run_analyze(ctx, &dc, &dcorr, groups, spec, opts, &dtab, st);
    download_corr(ctx, dcorr, corr_host, st);
    download_tables(ctx, dtab, opts, tab_host, st);
    XSP_CUDA(cudaStreamSynchronize(st));
  });
}

XSP_API xsp_status xsp_comm_unique_id(void* id128) {
  if (!id128) return XSP_E_INVALID;
  try {
    xsp::comm_unique_id(id128);
    return XSP_OK;
  } catch (...) {
    return XSP_E_CUDA;
  }
}

XSP_API xsp_status xsp_comm_init(xsp_ctx* ctx, int world, int rank, const void* id128) {
  return guard(ctx, "xsp_comm_init", [&] {
    if (!id128) throw std::invalid_argument("null argument");
    xsp::comm_init(ctx, world, rank, id128);
  });
}

XSP_API xsp_status xsp_combine_tables(xsp_ctx* ctx, xsp_tables_out* local, const uint32_t* group_ids,
                                      uint32_t n_local, uint32_t n_groups_total, const uint32_t* l_row_map,
                                      uint32_t top_k, xsp_tables_out* out, uint64_t* bytes_sent, void* stream) {
  return guard(ctx, "xsp_combine_tables", [&] {
    if (!local || !out || (n_local && !group_ids)) throw std::invalid_argument("null argument");
    if (top_k > 8) throw std::invalid_argument("top_k must be <= 8");
    xsp::run_combine_tables(ctx, local, group_ids, n_local, n_groups_total, l_row_map, (int)top_k, out,
                            bytes_sent, static_cast<cudaStream_t>(stream));
  });
}

XSP_API xsp_status xsp_leveled_host(xsp_ctx* ctx, const xsp_span_cols* hc, const xsp_corr_out* hcorr,
                                    const xsp_level_sets* sets, const xsp_analysis_opts* opts,
                                    xsp_overhead_out* out) {
  return guard(ctx, "xsp_leveled_host", [&] {
    check_cols(hc, nullptr);
    if (!hcorr || !sets || !opts || !out) throw std::invalid_argument("null argument");
    cudaStream_t st = nullptr;
    xsp_span_cols dc = upload_cols(ctx, hc, st);
    xsp_corr_out dcorr = upload_corr(ctx, hcorr, st);
    xsp_overhead_out dov;
    std::memset(&dov, 0, sizeof(dov));
    xsp::run_leveled(ctx, &dc, &dcorr, sets, opts, &dov, st);
    download_overhead(ctx, dov, out, st);
    XSP_CUDA(cudaStreamSynchronize(st));
  });
}

XSP_API xsp_status xsp_run_host(xsp_ctx* ctx, const xsp_span_cols* hc, const xsp_traces* ht,
                                const xsp_groups* groups, const xsp_system_spec* spec,
                                const xsp_analysis_opts* opts, xsp_corr_out* corr_host,
                                xsp_tables_out* tab_host, void* stream) {
  return guard(ctx, "xsp_run_host", [&] {
    check_cols(hc, ht);
    if (!ht || !groups || !spec || !opts || !corr_host || !tab_host) throw std::invalid_argument("null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ctx->h2d_bytes = ctx->d2h_bytes = 0;
    if (groups->n_groups && (!groups->first_trace || !groups->n_runs || !groups->batch_size))
      throw std::invalid_argument("null group column");
    // large batches: chunked pipeline overlapping H2D, compute and D2H (pipeline.cu)
    if (xsp::run_host_chunked(ctx, hc, ht, groups, spec, opts, corr_host, tab_host)) return;
    xsp_span_cols dc = upload_cols(ctx, hc, st);
    xsp_traces dt = upload_traces(ctx, ht, st);
    xsp_corr_out dcorr;
    std::memset(&dcorr, 0, sizeof(dcorr));
    xsp::run_correlate(ctx, &dc, &dt, 0, &dcorr, st);
    xsp_tables_out dtab;
    std::memset(&dtab, 0, sizeof(dtab));
    xsp::run_analyze(ctx, &dc, &dcorr, groups, spec, opts, &dtab, st);
    download_corr(ctx, dcorr, corr_host, st);
    download_tables(ctx, dtab, opts, tab_host, st);
    XSP_CUDA(cudaStreamSynchronize(st));
  });
}
