"""ctypes mirror of include/xsp.h (the C ABI of the CUDA hot path).

The library is loaded from this package's lib/ directory (built in-tree by
``make -C paper_1908_06869_b200``). There is no CPU fallback: if the library
is missing, or no CUDA device is present when a context is created, the call
raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XSP_LIB") or os.path.join(_HERE, "lib", "libxsp.so")  # XSP_LIB: tuning variants

u8p = C.POINTER(C.c_uint8)
i8p = C.POINTER(C.c_int8)
u32p = C.POINTER(C.c_uint32)
i32p = C.POINTER(C.c_int32)
u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)

# status codes
XSP_OK = 0
XSP_E_INVALID = 1
XSP_E_CUDA = 2
XSP_E_NOMEM = 3
XSP_E_UNSORTED = 4
XSP_E_NO_DEVICE = 5

# flags byte
F_PARENT = 0x10
F_CID = 0x20
F_METRICS = 0x40
LEVEL_MODEL, LEVEL_LAYER, LEVEL_KERNEL, LEVEL_API = 0, 1, 2, 3
KIND_SYNC, KIND_LAUNCH, KIND_EXEC = 0, 1, 2

# per-trace status (xsp_trace_status)
T_OK, T_NO_MODEL, T_MULTI_MODEL, T_SKIP_LEVEL, T_DUP_EXEC_CID, T_DUP_LAUNCH_CID, T_SER_AMBIGUOUS, T_SER_FAILED = range(8)
# per-group status
G_OK, G_NO_RUNS, G_LAYER_COUNT, G_KERNEL_COUNT, G_TRACE_FAILED, G_BAD_TRIM = range(6)


class SpanCols(C.Structure):
    _fields_ = [
        ("n_spans", C.c_uint64),
        ("span_id", u64p), ("parent_id", u64p), ("begin_ns", u64p), ("end_ns", u64p),
        ("cid", u64p), ("flags", u8p), ("name_id", u32p),
        ("n_metric_rows", C.c_uint64),
        ("flops", u64p), ("dram_read", u64p), ("dram_write", u64p), ("occupancy", f64p),
        ("n_layer_rows", C.c_uint64),
        ("alloc_bytes", i64p), ("type_id", u32p),
    ]


class Traces(C.Structure):
    _fields_ = [("n_traces", C.c_uint32), ("span_off", u64p), ("levels", u32p)]


CORR_FIELDS = [
    ("trace_status", i32p, "T"), ("trace_err_row", u32p, "2T"), ("trace_model_row", u32p, "T"),
    ("trace_layer_off", u32p, "T1"), ("trace_kernel_off", u32p, "T1"),
    ("trace_orphan_off", u32p, "T1"), ("trace_amb_off", u32p, "T1"),
    ("layer_row", u32p, "L"), ("layer_kernel_off", u32p, "L1"), ("layer_dur", u64p, "L"),
    ("layer_attr_row", u32p, "L"),
    ("kernel_launch_row", u32p, "K"), ("kernel_exec_row", u32p, "K"),
    ("kernel_metric_row", u32p, "K"), ("kernel_dur", u64p, "K"), ("kernel_name", u32p, "K"),
    ("kernel_occ", f64p, "K"),
    ("orphan_row", u32p, "O"), ("orphan_reason", u8p, "O"),
    ("amb_row", u32p, "A"), ("amb_cand_off", u32p, "A1"), ("amb_cand_row", u32p, "AC"),
]


class CorrOut(C.Structure):
    _fields_ = [
        ("n_traces", C.c_uint32), ("n_failed", C.c_uint32),
        ("n_layers", C.c_uint64), ("n_kernels", C.c_uint64), ("n_orphans", C.c_uint64),
        ("n_ambiguities", C.c_uint64), ("n_candidates", C.c_uint64),
    ] + [(n, t) for n, t, _ in CORR_FIELDS]


class SystemSpec(C.Structure):
    _fields_ = [("peak_flops", C.c_double), ("memory_bandwidth_bytes_per_s", C.c_double)]


class AnalysisOpts(C.Structure):
    _fields_ = [("trim_fraction", C.c_double), ("epsilon", C.c_double),
                ("noise_tolerance", C.c_double), ("top_k", C.c_uint32)]


class Groups(C.Structure):
    _fields_ = [("n_groups", C.c_uint32), ("first_trace", u32p), ("n_runs", u32p),
                ("batch_size", u32p)]


TABLE_FIELDS = [
    ("group_status", i32p, "G"), ("group_err_arg", u32p, "G"),
    ("group_layer_off", u32p, "G1"), ("group_kernel_off", u32p, "G1"),
    ("group_name_off", u32p, "G1"),
    ("k_name", u32p, "K"), ("k_layer", u32p, "K"), ("k_lat", f64p, "K"), ("k_flops", u64p, "K"),
    ("k_read", u64p, "K"), ("k_write", u64p, "K"), ("k_occ", f64p, "K"), ("k_ai", f64p, "K"),
    ("k_tput", f64p, "K"), ("k_bound", i8p, "K"), ("k_roofline_in", u8p, "K"),
    ("l_index", u32p, "L"), ("l_row", u32p, "L"), ("l_layer_lat", f64p, "L"),
    ("l_kern_lat", f64p, "L"), ("l_flops", u64p, "L"), ("l_read", u64p, "L"),
    ("l_write", u64p, "L"), ("l_occ", f64p, "L"), ("l_count", u64p, "L"), ("l_ai", f64p, "L"),
    ("l_tput", f64p, "L"), ("l_bound", i8p, "L"), ("l_nongpu", f64p, "L"),
    ("l_gpu_share", f64p, "L"), ("l_nongpu_share", f64p, "L"), ("l_flagged", u8p, "L"),
    ("l_roofline_in", u8p, "L"), ("l_topk", u32p, "LK"),
    ("n_name", u32p, "N"), ("n_count", u64p, "N"), ("n_lat", f64p, "N"), ("n_pct", f64p, "N"),
    ("n_flops", u64p, "N"), ("n_read", u64p, "N"), ("n_write", u64p, "N"), ("n_occ", f64p, "N"),
    ("n_ai", f64p, "N"), ("n_tput", f64p, "N"), ("n_bound", i8p, "N"),
    ("m_lat", f64p, "G"), ("m_kern_lat", f64p, "G"), ("m_flops", u64p, "G"),
    ("m_read", u64p, "G"), ("m_write", u64p, "G"), ("m_occ", f64p, "G"), ("m_count", u64p, "G"),
    ("m_ai", f64p, "G"), ("m_tput", f64p, "G"), ("m_bound", i8p, "G"), ("m_gpu", f64p, "G"),
    ("m_gpu_pct", f64p, "G"), ("m_throughput", f64p, "G"), ("m_roofline_in", u8p, "G"),
    # a5 / a6 / a7 by layer type (after the n_type_rows count in the C struct)
    ("group_type_off", u32p, "G1"), ("y_type", u32p, "Y"), ("y_count", u64p, "Y"), ("y_lat", f64p, "Y"),
    ("y_alloc", i64p, "Y"),
]


_TYPE_FIELDS = ("group_type_off", "y_type", "y_count", "y_lat", "y_alloc")


class TablesOut(C.Structure):
    _fields_ = [
        ("n_groups", C.c_uint32),
        ("n_layers", C.c_uint64), ("n_kernels", C.c_uint64), ("n_names", C.c_uint64),
    ] + [(n, t) for n, t, _ in TABLE_FIELDS if n not in _TYPE_FIELDS] + [("n_type_rows", C.c_uint64)] + [
        (n, t) for n, t, _ in TABLE_FIELDS if n in _TYPE_FIELDS]


class LevelSets(C.Structure):
    _fields_ = [("n_sets", C.c_uint32), ("set_off", u32p), ("trace_idx", u32p), ("levels", u32p)]


class OverheadOut(C.Structure):
    _fields_ = [("status", C.c_int32), ("err_a", C.c_uint32), ("err_b", C.c_uint32),
                ("n_sets", C.c_uint32), ("n_events", C.c_uint32), ("chain", u32p),
                ("ev_level", u8p), ("ev_layer", u32p), ("ev_kernel", u32p), ("lat", f64p),
                ("overhead", f64p), ("step_flags", u8p), ("accurate", f64p)]


class ValidateIn(C.Structure):
    _fields_ = [("trace_id", u64p), ("meta_trace_id", u64p), ("tag_bits", u8p)]


class ValidationOut(C.Structure):
    _fields_ = [("n_issues", C.c_uint64), ("trace_issue_off", u32p), ("issue_row", u32p),
                ("issue_rule", u8p)]


# validate_bundle rules (xsp.h XSP_V_*) with the reference's (rule, detail) texts (span.cpp:129-192)
VALIDATION_RULES = [
    ("negative duration", "end_ns precedes begin_ns"),
    ("correlation_id missing", "launch/exec spans require a correlation_id"),
    ("correlation_id on sync span", "sync spans must not carry a correlation_id"),
    ("duplicate span_id", ""),
    ("trace_id mismatch", "span belongs to a different trace"),
    ("out of order", "timeline must be sorted by (begin_ns, rank, span_id)"),
    ("negative metric", "flop_count_sp"),
    ("negative metric", "dram_read_bytes"),
    ("negative metric", "dram_write_bytes"),
    ("occupancy out of range", "achieved_occupancy must lie in [0,1]"),
    ("model span missing", "a bundle requires exactly one model/sync span"),
    ("multiple model spans", "a bundle requires exactly one model/sync span"),
    ("model level disabled", "profiling_levels must always contain model"),
]
TAG_NEG_FLOPS, TAG_NEG_READ, TAG_NEG_WRITE, TAG_OCC_DOUBLE = 1, 2, 4, 8


class StringTable(C.Structure):
    _fields_ = [("n", C.c_uint32), ("bytes", C.c_char_p), ("off", u64p)]


class BwCol(C.Structure):
    _fields_ = [("width", u8p), ("boff", u64p), ("data", u8p), ("base", u64p)]


class PackedCols(C.Structure):
    _fields_ = [("n_spans", C.c_uint64), ("flags", u8p), ("name_id", u32p), ("dbegin", u32p), ("dur", u32p),
                ("n_cid", C.c_uint64), ("dcid", u32p), ("n_parent", C.c_uint64), ("parent", u64p),
                ("n_blocks", C.c_uint64), ("blk_cid_base", u64p), ("blk_cid0", u32p), ("blk_par0", u32p),
                ("n_esc", C.c_uint64), ("esc_key", u64p), ("esc_val", u64p),
                ("name_bw", BwCol), ("flops_bw", BwCol), ("read_bw", BwCol), ("write_bw", BwCol),
                ("alloc_bw", BwCol), ("type_bw", BwCol), ("occ_dict_n", C.c_uint32), ("occ_idx_bytes", C.c_uint32),
                ("occ_dict", C.POINTER(C.c_double)), ("occ_idx", u8p),
                ("dbegin_bw", BwCol), ("dur_bw", BwCol), ("dcid_bw", BwCol), ("parent_bw", BwCol),
                ("blk_met0", u32p), ("blk_lay0", u32p), ("blk_cpar0", u32p)]


class StringTableOut(C.Structure):  # xsp_string_table as returned by the library
    _fields_ = [("n", C.c_uint32), ("bytes", C.c_void_p), ("off", u64p)]


class IngestOut(C.Structure):
    _fields_ = [("status", C.c_int32), ("bad_stream", C.c_uint32), ("cols", SpanCols), ("traces", Traces),
                ("span_off_host", u64p), ("levels_host", u32p), ("trace_id", u64p), ("trace_batch", u32p),
                ("trace_run", u32p), ("trace_serialized", u8p), ("names", StringTableOut),
                ("types", StringTableOut), ("system_name", C.c_char_p), ("peak_flops", C.c_double),
                ("mem_bw", C.c_double)]


INGEST_OK, INGEST_HOST = 0, 1

# report tables (xsp_report_csv): a8..a14
REPORT_TABLES = {"a8": 8, "a9": 9, "a10": 10, "a11": 11, "a12": 12, "a13": 13, "a14": 14}

HOST_OUT_ALL, HOST_OUT_ROWS = 0, 1  # xsp_set_host_outputs
L_OK, L_TOO_FEW, L_NOT_CHAIN, L_AMBIGUOUS, L_TRACE_FAILED = range(5)
EV_IN_NARROW, EV_IN_WIDE, EV_CLAMPED, EV_NEGATIVE = 1, 2, 4, 8

# exported symbols of libxsp.so, i.e. the functions include/xsp.h declares
EXPORTS = [
    "xsp_abi_version", "xsp_ctx_create", "xsp_ctx_destroy", "xsp_last_error", "xsp_correlate",
    "xsp_analyze", "xsp_run", "xsp_run_host", "xsp_last_transfer_bytes", "xsp_last_launch_count",
    "xsp_host_alloc", "xsp_host_free", "xsp_copy_to_host", "xsp_set_profiling", "xsp_stage_reset",
    "xsp_stage_times", "xsp_leveled", "xsp_sort_timeline_host", "xsp_correlate_host",
    "xsp_analyze_host", "xsp_leveled_host", "xsp_validate", "xsp_validate_host", "xsp_sort_timeline", "xsp_resolve_serialized",
    "xsp_resolve_serialized_host", "xsp_report_csv", "xsp_report_csv_host", "xsp_comm_unique_id",
    "xsp_comm_init", "xsp_combine_tables", "xsp_ingest_jsonl", "xsp_pack_host", "xsp_run_host_packed",
    "xsp_set_host_outputs", "xsp_leveled_batch",
]

_lib = None


class XspError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"xsp status {status}: {message}")
        self.status = status


def load() -> C.CDLL:
    """Load libxsp.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_LOCAL)
    P = C.c_void_p
    lib.xsp_abi_version.restype = C.c_int
    lib.xsp_ctx_create.argtypes = [C.c_int, C.POINTER(P)]
    lib.xsp_ctx_create.restype = C.c_int32
    lib.xsp_ctx_destroy.argtypes = [P]
    lib.xsp_last_error.argtypes = [P]
    lib.xsp_last_error.restype = C.c_char_p
    lib.xsp_correlate.argtypes = [P, C.POINTER(SpanCols), C.POINTER(Traces), C.c_int,
                                  C.POINTER(CorrOut), P]
    lib.xsp_correlate.restype = C.c_int32
    lib.xsp_analyze.argtypes = [P, C.POINTER(SpanCols), C.POINTER(CorrOut), C.POINTER(Groups),
                                C.POINTER(SystemSpec), C.POINTER(AnalysisOpts),
                                C.POINTER(TablesOut), P]
    lib.xsp_analyze.restype = C.c_int32
    lib.xsp_run.argtypes = [P, C.POINTER(SpanCols), C.POINTER(Traces), C.POINTER(Groups),
                            C.POINTER(SystemSpec), C.POINTER(AnalysisOpts),
                            C.POINTER(CorrOut), C.POINTER(TablesOut), P]
    lib.xsp_run.restype = C.c_int32
    lib.xsp_run_host.argtypes = [P, C.POINTER(SpanCols), C.POINTER(Traces), C.POINTER(Groups),
                                 C.POINTER(SystemSpec), C.POINTER(AnalysisOpts),
                                 C.POINTER(CorrOut), C.POINTER(TablesOut), P]
    lib.xsp_run_host.restype = C.c_int32
    lib.xsp_last_transfer_bytes.argtypes = [P, u64p, u64p]
    lib.xsp_last_launch_count.argtypes = [P]
    lib.xsp_last_launch_count.restype = C.c_uint64
    lib.xsp_host_alloc.argtypes = [C.c_size_t]
    lib.xsp_host_alloc.restype = P
    lib.xsp_host_free.argtypes = [P]
    lib.xsp_copy_to_host.argtypes = [P, P, P, C.c_size_t]
    lib.xsp_copy_to_host.restype = C.c_int32
    lib.xsp_set_profiling.argtypes = [P, C.c_int]
    lib.xsp_stage_reset.argtypes = [P]
    lib.xsp_stage_times.argtypes = [P, C.c_int, C.POINTER(C.c_char_p), f64p, u64p]
    lib.xsp_stage_times.restype = C.c_int
    lib.xsp_leveled.argtypes = [P, C.POINTER(SpanCols), C.POINTER(CorrOut), C.POINTER(LevelSets),
                                C.POINTER(AnalysisOpts), C.POINTER(OverheadOut), P]
    lib.xsp_leveled.restype = C.c_int32
    lib.xsp_leveled_batch.argtypes = [P, C.POINTER(SpanCols), C.POINTER(CorrOut), C.c_uint32, C.POINTER(LevelSets),
                                      C.POINTER(AnalysisOpts), C.POINTER(OverheadOut), P]
    lib.xsp_leveled_batch.restype = C.c_int32
    lib.xsp_sort_timeline_host.argtypes = [P, C.c_uint64, u64p, u8p, u64p, C.c_uint32, u64p, u32p,
                                           C.POINTER(C.c_int)]
    lib.xsp_sort_timeline_host.restype = C.c_int32
    lib.xsp_sort_timeline.argtypes = [P, C.c_uint64, P, P, P, C.c_uint32, P, P, C.POINTER(C.c_int), P]
    lib.xsp_sort_timeline.restype = C.c_int32
    lib.xsp_correlate_host.argtypes = [P, C.POINTER(SpanCols), C.POINTER(Traces), C.c_int, C.POINTER(CorrOut)]
    lib.xsp_correlate_host.restype = C.c_int32
    lib.xsp_validate.argtypes = [P, C.POINTER(SpanCols), C.POINTER(Traces), C.POINTER(ValidateIn),
                                 C.POINTER(ValidationOut), P]
    lib.xsp_validate.restype = C.c_int32
    lib.xsp_resolve_serialized_host.argtypes = [P, C.POINTER(SpanCols), C.POINTER(Traces), C.POINTER(SpanCols),
                                                C.POINTER(Traces), C.POINTER(CorrOut)]
    lib.xsp_resolve_serialized_host.restype = C.c_int32
    lib.xsp_validate_host.argtypes = [P, C.POINTER(SpanCols), C.POINTER(Traces), C.POINTER(ValidateIn),
                                      C.POINTER(ValidationOut)]
    lib.xsp_validate_host.restype = C.c_int32
    for fn in (lib.xsp_report_csv, lib.xsp_report_csv_host):
        fn.argtypes = [P, C.POINTER(SpanCols), C.POINTER(CorrOut), C.POINTER(Groups), C.POINTER(TablesOut),
                       C.POINTER(StringTable), C.POINTER(StringTable), C.c_uint32, C.c_int,
                       C.POINTER(C.c_char_p), u64p, P]
        fn.restype = C.c_int32
    lib.xsp_pack_host.argtypes = [P, C.POINTER(SpanCols), C.POINTER(Traces), C.POINTER(PackedCols)]
    lib.xsp_set_host_outputs.argtypes = [P, C.c_uint32]
    lib.xsp_set_host_outputs.restype = C.c_int
    lib.xsp_pack_host.restype = C.c_int32
    lib.xsp_run_host_packed.argtypes = [P, C.POINTER(PackedCols), C.POINTER(SpanCols), C.POINTER(Traces),
                                        C.POINTER(Groups), C.POINTER(SystemSpec), C.POINTER(AnalysisOpts),
                                        C.POINTER(CorrOut), C.POINTER(TablesOut), P]
    lib.xsp_run_host_packed.restype = C.c_int32
    lib.xsp_ingest_jsonl.argtypes = [P, C.c_char_p, u64p, C.c_uint32, C.POINTER(IngestOut), P]
    lib.xsp_ingest_jsonl.restype = C.c_int32
    lib.xsp_comm_unique_id.argtypes = [P]
    lib.xsp_comm_unique_id.restype = C.c_int32
    lib.xsp_comm_init.argtypes = [P, C.c_int, C.c_int, P]
    lib.xsp_comm_init.restype = C.c_int32
    lib.xsp_combine_tables.argtypes = [P, C.POINTER(TablesOut), u32p, C.c_uint32, C.c_uint32, P, C.c_uint32,
                                       C.POINTER(TablesOut), u64p, P]
    lib.xsp_combine_tables.restype = C.c_int32
    _lib = lib
    return lib
