"""TEST INFRASTRUCTURE — Python handle on the reference oracle (oracle/_ref/libxsp_ref.so).

The library is the UNMODIFIED reference (strata, /root/reference/proj/src)
plus oracle/ref_shim.cpp, built by `make -C oracle ref`. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
use this module, and only as the checker or as the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libxsp_ref.so")

_DT = {"Q": np.uint64, "q": np.int64, "I": np.uint32, "i": np.int32, "B": np.uint8,
       "d": np.float64, "s": np.uint8}


class SoaIn(C.Structure):
    _fields_ = [
        ("n_spans", C.c_uint64),
        ("span_id", C.c_void_p), ("parent_id", C.c_void_p), ("begin_ns", C.c_void_p),
        ("end_ns", C.c_void_p), ("cid", C.c_void_p), ("flags", C.c_void_p), ("name_id", C.c_void_p),
        ("flops", C.c_void_p), ("dram_read", C.c_void_p), ("dram_write", C.c_void_p),
        ("occupancy", C.c_void_p), ("alloc_bytes", C.c_void_p), ("type_id", C.c_void_p),
        ("n_traces", C.c_uint32),
        ("trace_span_off", C.c_void_p), ("trace_id", C.c_void_p), ("trace_levels", C.c_void_p),
        ("trace_batch", C.c_void_p), ("trace_run", C.c_void_p), ("trace_serialized", C.c_void_p),
        ("names_data", C.c_void_p), ("names_off", C.c_void_p), ("n_names", C.c_uint32),
        ("types_data", C.c_void_p), ("types_off", C.c_void_p), ("n_types", C.c_uint32),
        ("system_name", C.c_char_p), ("peak_flops", C.c_double), ("mem_bw", C.c_double),
    ]


_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"{REF_LIB} missing: run `make -C {HERE} ref`")
        L = C.CDLL(REF_LIB, mode=C.RTLD_LOCAL)
        P = C.c_void_p
        L.xspref_bag_count.argtypes = [P]
        L.xspref_bag_key.argtypes = [P, C.c_int]
        L.xspref_bag_key.restype = C.c_char_p
        L.xspref_bag_get.argtypes = [P, C.c_char_p, C.POINTER(P), C.POINTER(C.c_uint64),
                                     C.c_char_p]
        L.xspref_bag_free.argtypes = [P]
        L.xspref_list_new.restype = P
        L.xspref_list_free.argtypes = [P]
        L.xspref_list_size.argtypes = [P]
        L.xspref_list_size.restype = C.c_uint64
        L.xspref_rng_new.argtypes = [C.c_uint64]
        L.xspref_rng_new.restype = P
        L.xspref_rng_free.argtypes = [P]
        L.xspref_last_error.restype = C.c_char_p
        L.xspref_emit.argtypes = [P, C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                  C.c_double, C.c_int, C.c_uint32, C.c_uint64, C.c_uint64]
        L.xspref_emit_chain.argtypes = [P, C.c_char_p, C.c_uint32, C.c_uint64, C.c_uint64,
                                        C.c_double]
        L.xspref_random_nested.argtypes = [P, P, C.c_uint64, C.c_double]
        L.xspref_random_async.argtypes = [P, P, C.c_uint64]
        L.xspref_shuffle_last.argtypes = [P, P, C.c_int]
        L.xspref_list_export.argtypes = [P]
        L.xspref_list_export.restype = P
        L.xspref_correlate.argtypes = [C.POINTER(SoaIn)]
        L.xspref_correlate.restype = P
        L.xspref_analyze.argtypes = [C.POINTER(SoaIn), P, P, C.c_uint32, C.c_double, C.c_double]
        L.xspref_analyze.restype = P
        L.xspref_leveled.argtypes = [C.POINTER(SoaIn), C.c_double, C.c_double]
        L.xspref_validate.argtypes = [C.POINTER(SoaIn), C.c_void_p, C.c_void_p]
        L.xspref_resolve.argtypes = [C.POINTER(SoaIn), C.POINTER(SoaIn)]
        L.xspref_resolve.restype = P
        L.xspref_validate.restype = P
        L.xspref_leveled.restype = P
        L.xspref_time_pipeline.argtypes = [C.POINTER(SoaIn), P, P, C.c_uint32, C.c_int, C.c_int]
        L.xspref_time_pipeline.restype = C.c_double
        L.xspref_trimmed_mean.argtypes = [P, C.c_uint64, C.c_double]
        L.xspref_trimmed_mean.restype = C.c_double
        _lib = L
    return _lib


def read_bag(h) -> Tuple[Dict[str, np.ndarray], Dict[str, List[bytes]]]:
    """All arrays of a bag; string arrays (x.off / x.data) are returned split."""
    L = lib()
    arrays: Dict[str, np.ndarray] = {}
    for i in range(L.xspref_bag_count(h)):
        key = L.xspref_bag_key(h, i)
        ptr, nb, dt = C.c_void_p(), C.c_uint64(), C.create_string_buffer(1)
        L.xspref_bag_get(h, key, C.byref(ptr), C.byref(nb), dt)
        dtype = _DT[dt.raw.decode()]
        if nb.value:
            buf = (C.c_char * nb.value).from_address(ptr.value)
            arrays[key.decode()] = np.frombuffer(buf, dtype=dtype).copy()
        else:
            arrays[key.decode()] = np.zeros(0, dtype=dtype)
    L.xspref_bag_free(h)
    strings: Dict[str, List[bytes]] = {}
    for k in [k for k in arrays if k.endswith(".off")]:
        base = k[:-4]
        off, data = arrays.pop(k), arrays.pop(base + ".data").tobytes()
        strings[base] = [data[off[i]:off[i + 1]] for i in range(len(off) - 1)]
    return arrays, strings


class Generator:
    """Reference trace generators: simprof emit_run / emit_leveled_chain and the
    test_support.hpp random bundles (with the reference's own mt19937_64)."""

    def __init__(self):
        self.L = lib()
        self.h = self.L.xspref_list_new()
        self._rngs = {}

    def __del__(self):
        try:
            self.L.xspref_list_free(self.h)
            for r in self._rngs.values():
                self.L.xspref_rng_free(r)
        except Exception:
            pass

    def rng(self, seed: int):
        if seed not in self._rngs:
            self._rngs[seed] = self.L.xspref_rng_new(seed)
        return self._rngs[seed]

    def emit(self, model: str, batch: int = 1, levels: int = 0b111, layer_oh: int = 0,
             kernel_oh: int = 0, metric_mult: float = 1.0, serialized: bool = False,
             run_index: int = 0, jitter_max: int = 0, jitter_seed: int = 0) -> "Generator":
        rc = self.L.xspref_emit(self.h, model.encode(), batch, levels, layer_oh, kernel_oh,
                                metric_mult, int(serialized), run_index, jitter_max, jitter_seed)
        if rc:
            raise RuntimeError(self.L.xspref_last_error().decode())
        return self

    def chain(self, model: str, batch: int = 1, layer_oh: int = 0, kernel_oh: int = 0,
              metric_mult: float = 1.0) -> "Generator":
        rc = self.L.xspref_emit_chain(self.h, model.encode(), batch, layer_oh, kernel_oh, metric_mult)
        if rc:
            raise RuntimeError(self.L.xspref_last_error().decode())
        return self

    def random_nested(self, rng_seed: int, max_spans: int, explicit_fraction: float = 0.2):
        self.L.xspref_random_nested(self.h, self.rng(rng_seed), max_spans, explicit_fraction)
        return self

    def random_async(self, rng_seed: int, pairs: int):
        self.L.xspref_random_async(self.h, self.rng(rng_seed), pairs)
        return self

    def shuffle_last(self, rng_seed: int, resort: bool = True):
        self.L.xspref_shuffle_last(self.h, self.rng(rng_seed), int(resort))
        return self

    def batch(self):
        from paper_1908_06869_b200.columns import SpanBatch
        arrays, strings = read_bag(self.L.xspref_list_export(self.h))
        return SpanBatch.from_bag(arrays, strings)


def soa_in(b) -> Tuple[SoaIn, list]:
    """SoaIn view of a SpanBatch (returns the struct and the buffers to keep alive)."""
    keep = []

    def p(a):
        a = np.ascontiguousarray(a)
        keep.append(a)
        return a.ctypes.data if a.size else None

    def strtab(lst):
        data = b"".join(lst)
        off = np.zeros(len(lst) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(x) for x in lst]) if lst else []
        buf = C.create_string_buffer(data or b"\0", max(len(data), 1))
        keep.append(buf)
        return C.cast(buf, C.c_void_p), p(off), len(lst)

    s = SoaIn()
    s.n_spans = b.n_spans
    for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags", "name_id", "flops",
              "dram_read", "dram_write", "occupancy", "alloc_bytes", "type_id", "trace_span_off",
              "trace_id", "trace_levels", "trace_batch", "trace_run", "trace_serialized"):
        setattr(s, k, p(getattr(b, k)))
    s.n_traces = b.n_traces
    s.names_data, s.names_off, s.n_names = strtab(b.names)
    s.types_data, s.types_off, s.n_types = strtab(b.types)
    s.system_name = b.system_name
    s.peak_flops = b.peak_flops
    s.mem_bw = b.mem_bw
    return s, keep


def correlate(b):
    s, keep = soa_in(b)
    return read_bag(lib().xspref_correlate(C.byref(s)))


def analyze(b, first: Sequence[int], runs: Sequence[int], trim=0.2, noise=0.01):
    s, keep = soa_in(b)
    f = np.ascontiguousarray(first, dtype=np.uint32)
    r = np.ascontiguousarray(runs, dtype=np.uint32)
    return read_bag(lib().xspref_analyze(C.byref(s), f.ctypes.data, r.ctypes.data, f.size, trim, noise))


def list_jsonl(gen: "Generator", i: int) -> bytes:
    """to_jsonl of bundle i of a generator's list (the reference's wire form)."""
    L = lib()
    L.xspref_list_jsonl.restype = C.c_void_p
    L.xspref_list_jsonl.argtypes = [C.c_void_p, C.c_uint64]
    L.xspref_free_text.argtypes = [C.c_void_p]
    p = L.xspref_list_jsonl(gen.h, i)
    try:
        return C.string_at(p)
    finally:
        L.xspref_free_text(p)


def ingest(streams):
    """The reference's ingest() of each JSONL stream -> SpanBatch (one trace per
    stream); raises RuntimeError(IngestError text) on failure."""
    from paper_1908_06869_b200.columns import SpanBatch
    L = lib()
    L.xspref_ingest.restype = C.c_void_p
    L.xspref_ingest.argtypes = [C.c_char_p, C.c_void_p, C.c_uint32]
    blob = b"".join(streams)
    off = np.concatenate([[0], np.cumsum([len(x) for x in streams])]).astype(np.uint64)
    h = L.xspref_ingest(blob, off.ctypes.data, len(streams))
    if not h:
        raise RuntimeError(L.xspref_last_error().decode())
    arrays, strings = read_bag(h)
    return SpanBatch.from_bag(arrays, strings)


def report_csv(b, first: int, runs: int, table: int, trim=0.2, noise=0.01) -> bytes:
    """The reference report's CSV (to_csv(to_table(aN(...)))) of analysis table N of
    the group of traces [first, first + runs)."""
    L = lib()
    L.xspref_report_csv.restype = C.c_void_p
    L.xspref_report_csv.argtypes = [C.POINTER(SoaIn), C.c_uint32, C.c_uint32, C.c_int, C.c_double, C.c_double]
    L.xspref_free_text.argtypes = [C.c_void_p]
    s, keep = soa_in(b)
    p = L.xspref_report_csv(C.byref(s), first, runs, table, trim, noise)
    if not p:
        raise RuntimeError(L.xspref_last_error().decode())
    try:
        return C.string_at(p)
    finally:
        L.xspref_free_text(p)


def resolve(original, serialized):
    """resolve_with_serialized per trace pair, as correlate() returns it."""
    s1, k1 = soa_in(original)
    s2, k2 = soa_in(serialized)
    return read_bag(lib().xspref_resolve(C.byref(s1), C.byref(s2)))


def validate(b, span_trace_id=None, tag_bits=None):
    """validate_bundle per trace: list (per trace) of (span_id, rule, detail)."""
    s, keep = soa_in(b)
    tid = None if span_trace_id is None else np.ascontiguousarray(span_trace_id, dtype=np.uint64)
    tb = None if tag_bits is None else np.ascontiguousarray(tag_bits, dtype=np.uint8)
    arrays, strings = read_bag(lib().xspref_validate(C.byref(s), None if tid is None else tid.ctypes.data,
                                                     None if tb is None else tb.ctypes.data))
    out = [[] for _ in range(b.n_traces)]
    for t, sid, rule, det in zip(arrays["trace"], arrays["span_id"], strings["rule"], strings["detail"]):
        out[int(t)].append((int(sid), rule.decode(), det.decode()))
    return out


def leveled(b, trim=0.2, noise=0.01):
    s, keep = soa_in(b)
    return read_bag(lib().xspref_leveled(C.byref(s), trim, noise))


def time_pipeline(b, first, runs, threads: int, reps: int = 1) -> float:
    s, keep = soa_in(b)
    f = np.ascontiguousarray(first, dtype=np.uint32)
    r = np.ascontiguousarray(runs, dtype=np.uint32)
    return lib().xspref_time_pipeline(C.byref(s), f.ctypes.data, r.ctypes.data, f.size, threads, reps)


def trimmed_mean(values, f):
    v = np.ascontiguousarray(values, dtype=np.float64)
    return lib().xspref_trimmed_mean(v.ctypes.data, v.size, f)
