/*
 * xsp.h — the C ABI of the B200 span-correlation / analysis hot path.
 *
 * This is the drop-in boundary under the reference's C++ ingest/correlate/analyze
 * API (namespace strata in /root/reference/proj/include/strata/ *.hpp). Every entry
 * point below names the reference interface it replaces. The ABI carries plain
 * pointers and sizes only: span columns (structure of arrays), trace and group
 * descriptors, and ctx-owned result columns. No C++ or torch types cross it.
 *
 *   reference                                   this ABI
 *   ------------------------------------------  -------------------------------
 *   TraceBundle / Span (span.hpp:81-171)        xsp_span_cols + trace offsets
 *   correlate()   (correlator.hpp:164)          xsp_correlate
 *   assign_parents + correlate_async (:154,161) (both inside xsp_correlate)
 *   resolve_with_serialized (correlator.hpp:176) xsp_resolve_serialized
 *   a5..a15, model_roofline (analysis.hpp:128-366) xsp_analyze
 *   LeveledRunGroup + compute_overhead (leveled.hpp:60-109) xsp_leveled
 *   validate_bundle (span.hpp:187)              xsp_validate / xsp_validate_host
 *   sort_timeline (span.hpp:190)                xsp_sort_timeline / xsp_sort_timeline_host
 *
 * Ownership: the caller owns all inputs. Result columns live in ctx-owned device
 * memory and stay valid until the next call on the same ctx or xsp_ctx_destroy.
 * Threading: a ctx is bound to one device and is not re-entrant; use one ctx per
 * stream/thread (distinct ctxs may run concurrently).
 * Errors: every call returns an xsp_status; xsp_last_error(ctx) gives a one-line
 * description. Per-trace faults of the reference (TraceError thrown by
 * assign_parents / correlate_async) are reported per trace in
 * xsp_corr_out.trace_status with the span rows needed to rebuild the reference's
 * exact message text (see xsp_trace_status).
 */
#ifndef XSP_H
#define XSP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XSP_ABI_VERSION 1

typedef struct xsp_ctx xsp_ctx;
typedef int32_t xsp_status;

enum {
  XSP_OK = 0,
  XSP_E_INVALID = 1,   /* bad argument */
  XSP_E_CUDA = 2,      /* CUDA runtime failure (message in xsp_last_error) */
  XSP_E_NOMEM = 3,     /* device allocation failed */
  XSP_E_UNSORTED = 4,  /* a trace is not in timeline order and sorting was disabled */
  XSP_E_NO_DEVICE = 5  /* no CUDA device: there is no CPU fallback */
};

/* ---- span columns ------------------------------------------------------- */

/* flags byte per span: bits 0-1 level (strata::Level: Model 0, Layer 1, Kernel 2,
 * Api 3), bits 2-3 kind (strata::SpanKind: Sync 0, Launch 1, Exec 2), then the
 * presence bits of Span's optional members and of KernelMetrics tags. */
#define XSP_LEVEL_MODEL 0u
#define XSP_LEVEL_LAYER 1u
#define XSP_LEVEL_KERNEL 2u
#define XSP_LEVEL_API 3u
#define XSP_KIND_SYNC 0u
#define XSP_KIND_LAUNCH 1u
#define XSP_KIND_EXEC 2u
#define XSP_F_PARENT 0x10u  /* parent_id present   (Span::parent_id, span.hpp:84)      */
#define XSP_F_CID 0x20u     /* correlation_id present (span.hpp:90)                    */
#define XSP_F_METRICS 0x40u /* metrics_from_tags() != nullopt (span.hpp:131)           */

/* All spans of all traces of one call, trace after trace; rows [off[t], off[t+1])
 * belong to trace t. Columns are indexed by span row except the two compact
 * side tables:
 *   metric table: one row per span with XSP_F_METRICS, in span-row order
 *                 (the decoded KernelMetrics of span.cpp:284-296);
 *   layer table:  one row per span with level == Layer, in span-row order
 *                 ("alloc_bytes" tag via tag_int, "layer_type" interned,
 *                  correlator.cpp:197-202).
 * name_id / type_id index string tables interned in byte-lexicographic order,
 * so id order equals std::string order (a10 / a5 sort by name). */
typedef struct xsp_span_cols {
  uint64_t n_spans;
  const uint64_t* span_id;
  const uint64_t* parent_id; /* read iff XSP_F_PARENT */
  const uint64_t* begin_ns;
  const uint64_t* end_ns;
  const uint64_t* cid; /* read iff XSP_F_CID */
  const uint8_t* flags;
  const uint32_t* name_id;
  uint64_t n_metric_rows;
  const uint64_t* flops;      /* flop_count_sp */
  const uint64_t* dram_read;  /* dram_read_bytes */
  const uint64_t* dram_write; /* dram_write_bytes */
  const double* occupancy;    /* achieved_occupancy */
  uint64_t n_layer_rows;
  const int64_t* alloc_bytes;
  const uint32_t* type_id;
} xsp_span_cols;

/* One trace (= one TraceBundle): its span rows and RunMeta::profiling_levels
 * as a bit mask (1 << level). */
typedef struct xsp_traces {
  uint32_t n_traces;
  const uint64_t* span_off; /* [n_traces + 1] */
  const uint32_t* levels;   /* [n_traces] */
} xsp_traces;

/* ---- correlation -------------------------------------------------------- */

/* Per-trace fault codes: the TraceErrors assign_parents / correlate_async throw.
 * err_row[2t], err_row[2t+1] name the span rows the message quotes. */
typedef enum xsp_trace_status {
  XSP_T_OK = 0,
  XSP_T_NO_MODEL = 1,        /* "bundle has no model span; nothing to correlate"        (correlator.cpp:143-145) */
  XSP_T_MULTI_MODEL = 2,     /* "bundle has more than one model span"                   (:147-150) */
  XSP_T_SKIP_LEVEL = 3,      /* "span <id> ('<name>') is kernel-level but ..."  row a   (:151-157) */
  XSP_T_DUP_EXEC_CID = 4,    /* "correlation id C is shared by execution spans A and B" (:296-302) */
  XSP_T_DUP_LAUNCH_CID = 5,  /* "... is shared by launch spans A and B"                 (:308-316) */
  /* xsp_resolve_serialized only (correlator.cpp:381-386): */
  XSP_T_SER_AMBIGUOUS = 6,   /* "serialized run is itself ambiguous (N span(s)); cannot resolve"; err_row[2t] = N */
  XSP_T_SER_FAILED = 7       /* assign_parents(serialized) failed; err_row = the serialized trace's err rows
                                (rows of the SERIALIZED batch) and that trace's status says which fault */
} xsp_trace_status_code;

/* Orphan reasons (OrphanSpan::reason text, correlator.cpp:168-363). */
typedef enum xsp_orphan_reason {
  XSP_O_LAYER_NON_SYNC = 1,        /* "layer-level span with non-sync kind" */
  XSP_O_LAYER_BAD_PARENT = 2,      /* "explicit parent <P> is not the model span" */
  XSP_O_LAYER_OUTSIDE_MODEL = 3,   /* "outside the model interval" */
  XSP_O_KERNEL_BAD_PARENT = 4,     /* "explicit parent <P> is not a layer in the tree" */
  XSP_O_KERNEL_NO_LAYER = 5,       /* "contained in no layer interval" */
  XSP_O_EXEC_NO_CID = 6,           /* "execution record without correlation id" */
  XSP_O_LAUNCH_NO_CID = 7,         /* "launch without correlation id" */
  XSP_O_LAUNCH_NO_EXEC = 8,        /* "launch has no matching execution record" */
  XSP_O_EXEC_NO_LAUNCH = 9         /* "execution record without matching launch" */
} xsp_orphan_reason;

/* Correlation result (CorrelationResult, correlator.hpp:134-137) as columns.
 * Rows are global span rows of the input. Layers are in layer_index order
 * (begin_ns, span_id) per trace; kernels are in tree order (layer, then launch
 * (begin_ns, span_id)). All pointers are DEVICE pointers owned by the ctx. */
typedef struct xsp_corr_out {
  uint32_t n_traces;
  uint32_t n_failed; /* traces with trace_status != XSP_T_OK */
  uint64_t n_layers, n_kernels, n_orphans, n_ambiguities, n_candidates;
  int32_t* trace_status;     /* [n_traces] xsp_trace_status_code */
  uint32_t* trace_err_row;   /* [2 n_traces] */
  uint32_t* trace_model_row; /* [n_traces] row of the model span (UINT32_MAX if none) */
  uint32_t* trace_layer_off; /* [n_traces + 1] into layer columns */
  uint32_t* trace_kernel_off;/* [n_traces + 1] into kernel columns */
  uint32_t* trace_orphan_off;/* [n_traces + 1] */
  uint32_t* trace_amb_off;   /* [n_traces + 1] */
  /* layers (LayerExec) */
  uint32_t* layer_row;        /* span row */
  uint32_t* layer_kernel_off; /* [n_layers + 1] CSR into kernel columns */
  uint64_t* layer_dur;        /* Span::duration_ns of the layer span */
  uint32_t* layer_attr_row;   /* row of the layer table (alloc_bytes, type_id) */
  /* kernels (KernelExec) */
  uint32_t* kernel_launch_row;
  uint32_t* kernel_exec_row;   /* == launch row for a synchronous kernel span */
  uint32_t* kernel_metric_row; /* metric-table row of the exec, UINT32_MAX if none */
  uint64_t* kernel_dur;        /* KernelExec::duration_ns (exec span) */
  uint32_t* kernel_name;       /* KernelExec::kernel_name() name_id */
  double* kernel_occ;          /* metrics->achieved_occupancy, 0 without metrics */
  /* diagnostics, in the reference's output order */
  uint32_t* orphan_row;
  uint8_t* orphan_reason; /* xsp_orphan_reason */
  uint32_t* amb_row;      /* ambiguities sorted by span_id */
  uint32_t* amb_cand_off; /* [n_ambiguities + 1] */
  uint32_t* amb_cand_row; /* candidate layer rows sorted by span_id */
} xsp_corr_out;

/* ---- analysis ------------------------------------------------------------ */

typedef struct xsp_system_spec { /* SystemSpec (span.hpp:139-145) */
  double peak_flops;
  double memory_bandwidth_bytes_per_s;
} xsp_system_spec;

typedef struct xsp_analysis_opts { /* AnalysisOptions (analysis.hpp:47-51) */
  double trim_fraction;   /* 0.2 */
  double epsilon;         /* 0.05 */
  double noise_tolerance; /* 0.01 */
  uint32_t top_k;         /* kernels kept per layer in the top-k table (north star (e)) */
} xsp_analysis_opts;

/* One AnalysisInput (analysis.hpp:42-45): runs are the correlated traces
 * [first_trace, first_trace + n_runs) of the xsp_corr_out. */
typedef struct xsp_groups {
  uint32_t n_groups;
  const uint32_t* first_trace; /* [n_groups] */
  const uint32_t* n_runs;      /* [n_groups] */
  const uint32_t* batch_size;  /* [n_groups] */
} xsp_groups;

/* Optional-value encoding in the tables: std::optional<double> absent = NaN;
 * std::optional<bool> memory_bound: -1 absent, 0 false, 1 true. */
enum {
  XSP_G_OK = 0,
  XSP_G_NO_RUNS = 1,          /* "analysis input holds no runs" (analysis.cpp:103-105) */
  XSP_G_LAYER_COUNT = 2,      /* "repetitions disagree on layer count" (:108-110) */
  XSP_G_KERNEL_COUNT = 3,     /* "repetitions disagree on kernel count of layer <i>" (:112-115) */
  XSP_G_TRACE_FAILED = 4,     /* a run's correlation failed (see trace_status) */
  XSP_G_BAD_TRIM = 5          /* "trim fraction must lie in [0, 0.5)" (:30-32) */
};

/* All DEVICE pointers owned by the ctx. Kernel and layer rows follow the first
 * run's tree order ("canonical" run of combine(), analysis.cpp:102-170). */
typedef struct xsp_tables_out {
  uint32_t n_groups;
  uint64_t n_layers, n_kernels, n_names;
  int32_t* group_status;   /* [n_groups] XSP_G_* */
  uint32_t* group_err_arg; /* layer index for XSP_G_KERNEL_COUNT */
  uint32_t* group_layer_off;  /* [n_groups + 1] */
  uint32_t* group_kernel_off; /* [n_groups + 1] */
  uint32_t* group_name_off;   /* [n_groups + 1] */
  /* a8 / a9: KernelInfoRow per kernel (analysis.cpp:342-397) */
  uint32_t* k_name; uint32_t* k_layer;
  double* k_lat; uint64_t* k_flops; uint64_t* k_read; uint64_t* k_write; double* k_occ;
  double* k_ai; double* k_tput; int8_t* k_bound;
  uint8_t* k_roofline_in; /* a9: classify() != nullopt */
  /* a11 / a12 / a13 / a14: per layer (analysis.cpp:437-525) */
  uint32_t* l_index; uint32_t* l_row;
  double* l_layer_lat; double* l_kern_lat;
  uint64_t* l_flops; uint64_t* l_read; uint64_t* l_write; double* l_occ; uint64_t* l_count;
  double* l_ai; double* l_tput; int8_t* l_bound;
  double* l_nongpu; double* l_gpu_share; double* l_nongpu_share; uint8_t* l_flagged;
  uint8_t* l_roofline_in; /* a14 */
  uint32_t* l_topk;       /* [n_layers * top_k] kernel ordinals within the group, UINT32_MAX pad */
  /* a10: per (group, kernel name), sorted by total latency desc, name asc */
  uint32_t* n_name; uint64_t* n_count; double* n_lat; double* n_pct;
  uint64_t* n_flops; uint64_t* n_read; uint64_t* n_write; double* n_occ;
  double* n_ai; double* n_tput; int8_t* n_bound;
  /* a15 / model_roofline / a13 totals / a1: per group */
  double* m_lat; double* m_kern_lat; uint64_t* m_flops; uint64_t* m_read; uint64_t* m_write;
  double* m_occ; uint64_t* m_count; double* m_ai; double* m_tput; int8_t* m_bound;
  double* m_gpu; double* m_gpu_pct; double* m_throughput;
  uint8_t* m_roofline_in;
  /* a5 / a6 / a7 (analysis.cpp:315-337): per (group, layer type) over the
   * combined layers in execution order — layer count, total trimmed-mean
   * latency (fp64, summed in layer order) and total alloc_bytes of the first
   * run; rows sorted by total latency desc, type asc. type_id indexes the
   * layer-type string table (byte-lexicographic, so id order = string order). */
  uint64_t n_type_rows;
  uint32_t* group_type_off; /* [n_groups + 1] */
  uint32_t* y_type; uint64_t* y_count; double* y_lat; int64_t* y_alloc;
} xsp_tables_out;

/* ---- leveled measurement (stage f) ----------------------------------------- */

/* Level sets of one LeveledRunGroup (leveled.hpp:60-71): set s holds the
 * correlated traces trace_idx[set_off[s] .. set_off[s+1]) of an xsp_corr_out
 * (its repetitions, in order), captured at profiling levels `levels[s]` (bit
 * mask). HOST arrays. */
typedef struct xsp_level_sets {
  uint32_t n_sets;
  const uint32_t* set_off;   /* [n_sets + 1] */
  const uint32_t* trace_idx; /* [set_off[n_sets]] */
  const uint32_t* levels;    /* [n_sets] */
} xsp_level_sets;

enum {
  XSP_L_OK = 0,
  XSP_L_TOO_FEW = 1,      /* "overhead needs at least two chained level sets; got N" (leveled.cpp:148-151) */
  XSP_L_NOT_CHAIN = 2,    /* "profiling-level sets A and B do not form an inclusion chain" (:131-138); err_a/err_b = set indices */
  XSP_L_AMBIGUOUS = 3,    /* a trace has ambiguities (LeveledRunGroup::add, :69-75); err_a = trace */
  XSP_L_TRACE_FAILED = 4  /* a trace's correlation failed; err_a = trace */
};

/* Event flags per chain step (leveled.cpp:182-213). */
#define XSP_EV_IN_NARROW 0x01u   /* event visible in the narrower set of the step */
#define XSP_EV_IN_WIDE 0x02u     /* event visible in the wider set of the step */
#define XSP_EV_CLAMPED 0x04u     /* small negative overhead clamped to 0 */
#define XSP_EV_NEGATIVE 0x08u    /* negative beyond noise tolerance (kept, warning) */

/* compute_overhead (leveled.cpp:145-231) as columns. Events are the union of
 * the sets' LeveledEventKeys sorted by (rank(level), layer_index, kernel_index);
 * sets are in chain order (ascending size). DEVICE pointers owned by the ctx. */
typedef struct xsp_overhead_out {
  int32_t status;
  uint32_t err_a, err_b;
  uint32_t n_sets;        /* chain length */
  uint32_t n_events;
  const uint32_t* chain;  /* HOST: chain position -> input set index */
  uint8_t* ev_level;      /* Level (Model 0, Layer 1, Kernel 2) */
  uint32_t* ev_layer;
  uint32_t* ev_kernel;
  double* lat;            /* [n_sets * n_events] trimmed-mean latency per set, NaN if absent */
  double* overhead;       /* [(n_sets-1) * n_events] wide - narrow (after clamping), NaN if absent */
  uint8_t* step_flags;    /* [(n_sets-1) * n_events] XSP_EV_* */
  double* accurate;       /* [n_events] accurate_latency_ns, NaN if no set qualifies */
} xsp_overhead_out;

/* ---- bundle validation (stage a) ------------------------------------------- */

/* validate_bundle (span.cpp:129-192) rules, in the reference's per-span report
 * order, then the bundle-level rules. */
enum {
  XSP_V_NEG_DURATION = 0,  /* "negative duration"            */
  XSP_V_CID_MISSING = 1,   /* "correlation_id missing"       */
  XSP_V_CID_ON_SYNC = 2,   /* "correlation_id on sync span"  */
  XSP_V_DUP_SPAN_ID = 3,   /* "duplicate span_id"            */
  XSP_V_TRACE_ID = 4,      /* "trace_id mismatch"            */
  XSP_V_OUT_OF_ORDER = 5,  /* "out of order"                 */
  XSP_V_NEG_FLOPS = 6,     /* "negative metric" flop_count_sp    */
  XSP_V_NEG_READ = 7,      /* "negative metric" dram_read_bytes  */
  XSP_V_NEG_WRITE = 8,     /* "negative metric" dram_write_bytes */
  XSP_V_OCC_RANGE = 9,     /* "occupancy out of range"       */
  XSP_V_NO_MODEL = 10,     /* "model span missing"      (bundle level) */
  XSP_V_MULTI_MODEL = 11,  /* "multiple model spans"    (bundle level) */
  XSP_V_MODEL_LEVEL = 12   /* "model level disabled"    (bundle level) */
};

/* Raw-tag facts the decoded metric columns cannot carry (metrics_from_tags
 * clamps negatives, span.cpp:88-101), recorded by the ingest side per span. */
#define XSP_TAG_NEG_FLOPS 0x01u  /* flop_count_sp tag is an int64 < 0     */
#define XSP_TAG_NEG_READ 0x02u   /* dram_read_bytes tag is an int64 < 0   */
#define XSP_TAG_NEG_WRITE 0x04u  /* dram_write_bytes tag is an int64 < 0  */
#define XSP_TAG_OCC_DOUBLE 0x08u /* achieved_occupancy tag holds a double */

/* Optional validation inputs (any pointer may be NULL: the rule it feeds is
 * then skipped). Same memory space as the columns. */
typedef struct xsp_validate_in {
  const uint64_t* trace_id;      /* [n_spans] Span::trace_id                      */
  const uint64_t* meta_trace_id; /* [n_traces] RunMeta::trace_id (with trace_id)  */
  const uint8_t* tag_bits;       /* [n_spans] XSP_TAG_* bits                       */
} xsp_validate_in;

/* ValidationReport of every trace: issues of trace t are
 * [trace_issue_off[t], trace_issue_off[t+1]) in report order. issue_row is the
 * global span row (UINT32_MAX for bundle-level issues, whose span_id is 0). */
typedef struct xsp_validation_out {
  uint64_t n_issues;
  uint32_t* trace_issue_off; /* [n_traces + 1] */
  uint32_t* issue_row;
  uint8_t* issue_rule;       /* XSP_V_* */
} xsp_validation_out;

/* ---- API ------------------------------------------------------------------ */

xsp_status xsp_ctx_create(int device, xsp_ctx** out);
void xsp_ctx_destroy(xsp_ctx* ctx);
const char* xsp_last_error(const xsp_ctx* ctx);
int xsp_abi_version(void);

/* correlate() for every trace (correlator.cpp:366-370 = assign_parents 141-282 +
 * correlate_async 287-364). Inputs are DEVICE pointers. Traces must be in
 * timeline order (sort_timeline, span.hpp:161-163), else XSP_E_UNSORTED.
 * mode: 0, or XSP_CORR_PARENTS_ONLY for assign_parents alone (kernel launches
 * keep no exec: kernel_exec_row = UINT32_MAX; no fusion orphans or cid faults).
 * stream: a cudaStream_t (NULL = legacy default stream). Asynchronous except
 * for the small count read-backs needed to size the outputs. */
#define XSP_CORR_PARENTS_ONLY 2
xsp_status xsp_correlate(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_traces* traces, int mode,
                         xsp_corr_out* out, void* stream);

/* resolve_with_serialized (correlator.cpp:379-456) for every trace pair: trace t
 * of `original` (a concurrent run) is re-correlated with the parents its
 * serialized twin (trace t of `serialized`) assigns to its ambiguous kernels,
 * matched by (level, kind, name, occurrence in timeline order). Both batches
 * must share one name table (equal name_id = equal name). The result is the
 * correlate() of the patched original batch. DEVICE pointers; synchronous.
 * A pair whose serialized trace is ambiguous or fails gets XSP_T_SER_*. */
xsp_status xsp_resolve_serialized(xsp_ctx* ctx, const xsp_span_cols* original, const xsp_traces* original_traces,
                                  const xsp_span_cols* serialized, const xsp_traces* serialized_traces,
                                  xsp_corr_out* out, void* stream);
/* Host-buffer form (results in ctx-owned pinned host memory, like xsp_correlate_host). */
xsp_status xsp_resolve_serialized_host(xsp_ctx* ctx, const xsp_span_cols* original,
                                       const xsp_traces* original_traces, const xsp_span_cols* serialized,
                                       const xsp_traces* serialized_traces, xsp_corr_out* out);

/* sort_timeline (span.cpp:112-127) for every trace, DEVICE pointers (perm is a
 * caller-owned device array of n_spans): as xsp_sort_timeline_host below.
 * Synchronous (the presorted check and the fallback decision read back a flag). */
xsp_status xsp_sort_timeline(xsp_ctx* ctx, uint64_t n_spans, const uint64_t* begin_ns, const uint8_t* flags,
                             const uint64_t* span_id, uint32_t n_traces, const uint64_t* span_off,
                             uint32_t* perm, int* was_sorted, void* stream);

/* sort_timeline (span.cpp:112-127) for every trace: perm[j] = input row of the
 * span at position j once each trace [span_off[t], span_off[t+1]) is stably
 * sorted by (begin_ns, rank(level), span_id). *was_sorted = 1 when the input
 * already was (perm is then the identity). HOST pointers; synchronous. */
xsp_status xsp_sort_timeline_host(xsp_ctx* ctx, uint64_t n_spans, const uint64_t* begin_ns,
                                  const uint8_t* flags, const uint64_t* span_id, uint32_t n_traces,
                                  const uint64_t* span_off, uint32_t* perm, int* was_sorted);

/* Host-buffer forms used by the C++ drop-in (libstrata_b200): inputs are HOST
 * pointers, copied to the device; results are copied back into ctx-owned pinned
 * host memory (pointers valid until the next call on the ctx). Synchronous.
 * xsp_analyze_host / xsp_leveled_host take a HOST xsp_corr_out (e.g. packed from
 * existing entity trees); only the columns the analysis reads must be set:
 * trace_status, trace_model_row, trace_layer_off, trace_kernel_off,
 * trace_amb_off, layer_row, layer_kernel_off, layer_dur, kernel_metric_row,
 * kernel_dur, kernel_name, kernel_occ; a5-a7 also read layer_attr_row and the
 * layer table (type_id, alloc_bytes) when they are set. */
xsp_status xsp_correlate_host(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_traces* traces, int mode,
                              xsp_corr_out* out);
xsp_status xsp_analyze_host(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                            const xsp_groups* groups, const xsp_system_spec* spec,
                            const xsp_analysis_opts* opts, xsp_tables_out* out);
xsp_status xsp_leveled_host(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                            const xsp_level_sets* sets, const xsp_analysis_opts* opts,
                            xsp_overhead_out* out);

/* a8..a15 + model_roofline + a1 throughput + top-k for every group over a
 * correlation computed by xsp_correlate on the same ctx. cols must be the same
 * columns given to xsp_correlate. */
xsp_status xsp_analyze(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                       const xsp_groups* groups, const xsp_system_spec* spec,
                       const xsp_analysis_opts* opts, xsp_tables_out* out, void* stream);

/* LeveledRunGroup + compute_overhead (leveled.cpp:56-231) over a correlation
 * computed by xsp_correlate on the same ctx. Uses opts->trim_fraction and
 * opts->noise_tolerance. Synchronous (the chain order is decided on the host). */
xsp_status xsp_leveled(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                       const xsp_level_sets* sets, const xsp_analysis_opts* opts, xsp_overhead_out* out,
                       void* stream);
/* xsp_leveled for n_groups LeveledRunGroups at once (e.g. one per model): group
 * g's level sets are sets[g] and its result outs[g], exactly as xsp_leveled
 * would fill them (device columns in ctx-owned buffers shared by the batch,
 * chain pointers in ctx-owned host memory; both valid until the next call).
 * The whole batch costs three host round trips instead of three per group. */
xsp_status xsp_leveled_batch(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                             uint32_t n_groups, const xsp_level_sets* sets, const xsp_analysis_opts* opts,
                             xsp_overhead_out* outs, void* stream);

/* End-to-end convenience for host-resident inputs: copies the HOST columns to the
 * device, runs xsp_correlate + xsp_analyze, and copies every result column back
 * into ctx-owned pinned host memory (pointers in *corr_host / *tables_host are
 * HOST pointers valid until the next call). Synchronous. Large batches are cut
 * at group boundaries into chunks whose copies and kernels overlap; with
 * page-locked inputs the span_id column is read in place (zero-copy) by chunks
 * without explicit-parent kernels (XSP_NO_ZERO_COPY=1 disables that). */
xsp_status xsp_run_host(xsp_ctx* ctx, const xsp_span_cols* host_cols,
                        const xsp_traces* host_traces, const xsp_groups* groups,
                        const xsp_system_spec* spec, const xsp_analysis_opts* opts,
                        xsp_corr_out* corr_host, xsp_tables_out* tables_host, void* stream);

/* Columns the host-buffer calls (xsp_run_host, xsp_run_host_packed) copy back.
 * XSP_HOST_OUT_ALL (the default) copies every xsp_corr_out column.
 * XSP_HOST_OUT_ROWS skips the four columns that are lookups into the caller's
 * own span and metric columns and leaves them NULL:
 *   layer_dur[l]   = end_ns - begin_ns of span layer_row[l] (0 if end < begin),
 *   kernel_dur[k]  = the same of span kernel_exec_row[k],
 *   kernel_name[k] = name_id[kernel_exec_row[k]],
 *   kernel_occ[k]  = occupancy[kernel_metric_row[k]] (0 if UINT32_MAX).
 * What remains is what the reference's CorrelationResult carries (EntityTree
 * nodes refer to spans; correlator.hpp:40-75) plus every analysis table. */
#define XSP_HOST_OUT_ALL 0u
#define XSP_HOST_OUT_ROWS 1u
xsp_status xsp_set_host_outputs(xsp_ctx* ctx, uint32_t mode);

/* ---- packed host input (fewer PCIe bytes for xsp_run_host) -----------------
 * The same spans as an xsp_span_cols, with the 8-byte span columns packed:
 * begin as a u32 delta from the previous span (XSP_PACK_ESC: the value is in the
 * escape list; forced at every trace start and every 256-span block start),
 * end as a u32 duration, cid as a u32 offset from its 256-span block's base and
 * stored only for spans with XSP_F_CID, parent_id stored only for spans with
 * XSP_F_PARENT. Escapes: esc_key = row << 2 | kind (0 begin, 1 end, 2 cid),
 * ascending, with esc_val the raw value. flags / name_id are as in
 * xsp_span_cols; the metric and layer tables and span_id stay in the
 * xsp_span_cols given next to it. xsp_pack_host builds one (host arrays in
 * ctx-owned pinned memory, valid until the next xsp_pack_host). name_id and
 * the metric / layer tables are byte-width coded, occupancy dictionary coded
 * (XSP_PACK_TABLES=0 leaves them raw). C3: 52 -> 24 B per span on the wire. */
#define XSP_PACK_ESC 0xFFFFFFFFu
#define XSP_PACK_BLOCK 256u
/* Byte-width coded column, in blocks of XSP_PACK_BLOCK values: every value of
 * block b is width[b] (0..8) little-endian bytes, the block's values starting
 * at data + boff[b] (width 0: the block is all zero). */
typedef struct xsp_bw_col {
  const uint8_t* width;  /* [ceil(n / XSP_PACK_BLOCK)]; NULL: column not coded */
  const uint64_t* boff;  /* [ceil(n / XSP_PACK_BLOCK) + 1] */
  const uint8_t* data;
  const uint64_t* base;  /* [ceil(n / XSP_PACK_BLOCK)] frame of reference added to
                            every value of the block (NULL: none) */
} xsp_bw_col;
typedef struct xsp_packed_cols {
  uint64_t n_spans;
  const uint8_t* flags;
  const uint32_t* name_id;
  const uint32_t* dbegin;
  const uint32_t* dur;
  uint64_t n_cid;
  const uint32_t* dcid;          /* [n_cid] */
  uint64_t n_parent;
  const uint64_t* parent;        /* [n_parent] */
  uint64_t n_blocks;             /* ceil(n_spans / 256) */
  const uint64_t* blk_cid_base;  /* [n_blocks] */
  const uint32_t* blk_cid0;      /* [n_blocks] cid entries before the block */
  const uint32_t* blk_par0;      /* [n_blocks] parent entries before the block */
  uint64_t n_esc;
  const uint64_t* esc_key;
  const uint64_t* esc_val;
  /* name_id and the metric / layer tables, byte-width coded (alloc_bytes as
   * its u64 two's complement); a NULL width sends that column raw (name_id
   * above, the tables from the xsp_span_cols given next to the packed input) */
  xsp_bw_col name_bw;                      /* n_spans values */
  xsp_bw_col flops_bw, read_bw, write_bw;  /* n_metric_rows values */
  xsp_bw_col alloc_bw, type_bw;            /* n_layer_rows values */
  /* occupancy as indexes into a dictionary of its distinct values (first
   * appearance order); occ_dict_n == 0: occupancy raw */
  uint32_t occ_dict_n;
  uint32_t occ_idx_bytes;  /* 1 (<= 256 values) or 2 (<= 65536) */
  const double* occ_dict;
  const uint8_t* occ_idx;  /* [n_metric_rows * occ_idx_bytes], little-endian */
  /* dbegin / dur / dcid + 1 (mod 2^32, so XSP_PACK_ESC codes as 0), byte-width
   * coded; a NULL width sends the raw u32 arrays above */
  xsp_bw_col dbegin_bw, dur_bw; /* n_spans values */
  xsp_bw_col dcid_bw;           /* n_cid values */
  xsp_bw_col parent_bw;         /* n_parent values, with a per-block base; NULL width: `parent` raw */
  /* [n_blocks + 1] metric rows / layer rows / non-layer explicit-parent spans
   * before each block (a chunk's table rows without a pass over its flags);
   * NULL: counted from the flags */
  const uint32_t* blk_met0;
  const uint32_t* blk_lay0;
  const uint32_t* blk_cpar0;
} xsp_packed_cols;
xsp_status xsp_pack_host(xsp_ctx* ctx, const xsp_span_cols* host_cols, const xsp_traces* host_traces,
                         xsp_packed_cols* out);
/* xsp_run_host with the span columns taken from `packed` (unpacked on the
 * device chunk by chunk); host_cols supplies span_id, the metric and the layer
 * tables. Same outputs as xsp_run_host. */
xsp_status xsp_run_host_packed(xsp_ctx* ctx, const xsp_packed_cols* packed, const xsp_span_cols* host_cols,
                               const xsp_traces* host_traces, const xsp_groups* groups,
                               const xsp_system_spec* spec, const xsp_analysis_opts* opts,
                               xsp_corr_out* corr_host, xsp_tables_out* tables_host, void* stream);

/* correlate + analyze in one call on device-resident columns: xsp_correlate
 * (mode 1) then xsp_analyze over its result, the reference's pipeline of
 * correlate (correlator.cpp:366-370) followed by a8..a15 per analysis group
 * (analysis.cpp:342-586). Outputs as for the two calls; one host round trip
 * fewer between them. */
xsp_status xsp_run(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_traces* traces,
                   const xsp_groups* groups, const xsp_system_spec* spec, const xsp_analysis_opts* opts,
                   xsp_corr_out* corr, xsp_tables_out* tables, void* stream);

/* validate_bundle (span.cpp:129-192) for every trace. Device pointers; the
 * result columns are ctx-owned device memory. Synchronous (one count read-back). */
xsp_status xsp_validate(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_traces* traces,
                        const xsp_validate_in* in, xsp_validation_out* out, void* stream);
/* Host-buffer form (results in ctx-owned pinned host memory). */
xsp_status xsp_validate_host(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_traces* traces,
                             const xsp_validate_in* in, xsp_validation_out* out);

/* ---- report emission --------------------------------------
 * A string table: n strings, string i = bytes[off[i], off[i+1]) (HOST arrays,
 * off has n + 1 entries). names = the batch's name table (name_id order),
 * types = its layer-type table (type_id order). */
typedef struct xsp_string_table {
  uint32_t n;
  const char* bytes;
  const uint64_t* off;
} xsp_string_table;

/* The reference report's CSV file of one analysis table of one group
 * (report.cpp:42-147 to_csv over the :166-330 to_table converters), written on
 * the GPU from the device tables of the preceding xsp_analyze / xsp_run on this
 * ctx (which stay valid): table = 8 (a8 kernel info), 9 (a9 kernel roofline),
 * 10 (a10 by name), 11 (a11 by layer), 12 (a12 metrics per layer), 13 (a13 GPU
 * vs non-GPU), 14 (a14 layer roofline). cols / corr / groups are the arguments
 * of that analysis (device columns; corr is read for a11's layer types).
 * *text is ctx-owned device memory (xsp_report_csv) or ctx-owned pinned host
 * memory, NUL-terminated (xsp_report_csv_host), valid until the next report
 * call; *len excludes the NUL. Doubles are printed like std::to_chars (shortest
 * round trip), integers like std::to_string, cells CSV-quoted as csv_quote. */
xsp_status xsp_report_csv(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                          const xsp_groups* groups, const xsp_tables_out* tables,
                          const xsp_string_table* names, const xsp_string_table* types, uint32_t group,
                          int table, char** text, uint64_t* len, void* stream);
xsp_status xsp_report_csv_host(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                               const xsp_groups* groups, const xsp_tables_out* tables,
                               const xsp_string_table* names, const xsp_string_table* types, uint32_t group,
                               int table, char** text, uint64_t* len, void* stream);

/* ---- JSONL ingest -------------------------------------------
 * ingest() (collector.cpp:219-266) of n_streams JSONL streams on the GPU: stream
 * i = text[stream_off[i], stream_off[i+1]) (HOST text) is one TraceBundle,
 * trace i of the result. Span columns (device, ctx-owned, each trace in
 * timeline order: sort_timeline applied) carry the same values the C++
 * drop-in's packing of the ingested bundles gives, names / layer types interned
 * in lexicographic order over all streams. XSP_INGEST_HOST: stream bad_stream
 * holds something the device path does not cover exactly (string escapes or
 * non-ASCII bytes, a non-canonical record layout, a number outside the exact
 * cases, a missing / repeated meta record, a trace_id mismatch or a validation
 * issue): the caller parses with the host ingest, which returns the result or
 * the reference's IngestError text. Host pointers in *out stay valid until the
 * next xsp_ingest_jsonl call on the same thread. */
#define XSP_INGEST_OK 0
#define XSP_INGEST_HOST 1
typedef struct xsp_ingest_out {
  int32_t status;
  uint32_t bad_stream;
  xsp_span_cols cols;        /* device */
  xsp_traces traces;         /* device span_off / levels */
  const uint64_t* span_off_host;
  const uint32_t* levels_host;
  const uint64_t* trace_id;  /* host, per stream (RunMeta) */
  const uint32_t* trace_batch;
  const uint32_t* trace_run;
  const uint8_t* trace_serialized;
  xsp_string_table names;    /* host */
  xsp_string_table types;    /* host */
  const char* system_name;   /* stream 0's system spec */
  double peak_flops, mem_bw;
} xsp_ingest_out;
xsp_status xsp_ingest_jsonl(xsp_ctx* ctx, const char* text, const uint64_t* stream_off, uint32_t n_streams,
                            xsp_ingest_out* out, void* stream);

/* ---- multi-GPU table combine over NCCL -----------------
 * xsp_comm_unique_id: rank 0 creates the 128-byte NCCL unique id, which the
 * caller shares with the other ranks out of band (e.g. a torch.distributed
 * broadcast). xsp_comm_init: every rank joins the communicator (world ranks,
 * one ctx / GPU per rank). NCCL is loaded at run time (libnccl.so.2). */
xsp_status xsp_comm_unique_id(void* id128);
xsp_status xsp_comm_init(xsp_ctx* ctx, int world, int rank, const void* id128);

/* Trace-sharded analysis: rank r analysed the groups group_ids[0..n_local)
 * (HOST array of global group indices, in its local group order) with
 * xsp_analyze on this ctx (`local` = those device tables). Every rank calls;
 * the tables travel to rank 0 with NCCL send/recv (one contiguous block per
 * column and rank) and rank 0 lays them out in global group order (0 ..
 * n_groups_total - 1) — the tables of an unsharded run — in ctx-owned device
 * memory (*out; zeroed on other ranks). l_row_map (device, optional): global
 * span row of every local span row; the sender rewrites its l_row with it.
 * top_k as given to xsp_analyze. *bytes_sent (optional): table bytes this rank
 * sent. Synchronous. */
xsp_status xsp_combine_tables(xsp_ctx* ctx, xsp_tables_out* local, const uint32_t* group_ids, uint32_t n_local,
                              uint32_t n_groups_total, const uint32_t* l_row_map, uint32_t top_k,
                              xsp_tables_out* out, uint64_t* bytes_sent, void* stream);

/* Bytes moved host->device and device->host by the last xsp_run_host call. */
void xsp_last_transfer_bytes(const xsp_ctx* ctx, uint64_t* h2d, uint64_t* d2h);

/* Number of CUDA kernel launches issued by the last API call on this ctx. */
uint64_t xsp_last_launch_count(const xsp_ctx* ctx);

/* Per-stage device timing: when enabled, every call records CUDA events around
 * each stage (on the stream the stage's kernels are launched on) and accumulates
 * the elapsed times until xsp_stage_reset. xsp_stage_times fills up to `max`
 * entries (stage name, total ms, number of timed executions) and returns the
 * number of stages. */
void xsp_set_profiling(xsp_ctx* ctx, int enabled);
void xsp_stage_reset(xsp_ctx* ctx);
int xsp_stage_times(xsp_ctx* ctx, int max, const char** names, double* total_ms, uint64_t* count);

/* Synchronous device->host copy of `bytes` from a result column (helper for
 * callers that do not link the CUDA runtime themselves). */
xsp_status xsp_copy_to_host(xsp_ctx* ctx, void* dst, const void* src, size_t bytes);

/* Pinned host allocation helpers (cudaHostAlloc) for callers staging inputs. */
void* xsp_host_alloc(size_t bytes);
void xsp_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* XSP_H */
