"""Columnar (structure-of-arrays) span batches: the input format of the C ABI.

A SpanBatch holds the spans of one or more traces (TraceBundles, reference
span.hpp:161-171) as flat numpy columns, trace after trace, in timeline order
within each trace. The metric table has one row per span carrying
XSP_F_METRICS and the layer table one row per level==Layer span, both in span
order (include/xsp.h).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _capi as capi

SPAN_COLS = {
    "span_id": np.uint64, "parent_id": np.uint64, "begin_ns": np.uint64, "end_ns": np.uint64,
    "cid": np.uint64, "flags": np.uint8, "name_id": np.uint32,
}
METRIC_COLS = {"flops": np.uint64, "dram_read": np.uint64, "dram_write": np.uint64,
               "occupancy": np.float64}
LAYER_COLS = {"alloc_bytes": np.int64, "type_id": np.uint32}
TRACE_COLS = {"trace_span_off": np.uint64, "trace_id": np.uint64, "trace_levels": np.uint32,
              "trace_batch": np.uint32, "trace_run": np.uint32, "trace_serialized": np.uint8}


def _ptr(a: np.ndarray, typ):
    return a.ctypes.data_as(typ) if a.size else C.cast(C.c_void_p(0), typ)


@dataclass
class SpanBatch:
    span_id: np.ndarray
    parent_id: np.ndarray
    begin_ns: np.ndarray
    end_ns: np.ndarray
    cid: np.ndarray
    flags: np.ndarray
    name_id: np.ndarray
    flops: np.ndarray
    dram_read: np.ndarray
    dram_write: np.ndarray
    occupancy: np.ndarray
    alloc_bytes: np.ndarray
    type_id: np.ndarray
    trace_span_off: np.ndarray
    trace_id: np.ndarray
    trace_levels: np.ndarray
    trace_batch: np.ndarray
    trace_run: np.ndarray
    trace_serialized: np.ndarray
    names: List[bytes] = field(default_factory=list)
    types: List[bytes] = field(default_factory=list)
    system_name: bytes = b"tesla-v100-sxm2"
    peak_flops: float = 15.7e12
    mem_bw: float = 900e9

    def __post_init__(self):
        for k, dt in {**SPAN_COLS, **METRIC_COLS, **LAYER_COLS, **TRACE_COLS}.items():
            setattr(self, k, np.ascontiguousarray(getattr(self, k), dtype=dt))

    # ---- sizes
    @property
    def n_spans(self) -> int:
        return int(self.span_id.size)

    @property
    def n_traces(self) -> int:
        return int(self.trace_levels.size)

    def level(self) -> np.ndarray:
        return self.flags & 3

    def kind(self) -> np.ndarray:
        return (self.flags >> 2) & 3

    # ---- C ABI views (host pointers; keep self alive while used)
    def cols(self) -> capi.SpanCols:
        c = capi.SpanCols()
        c.n_spans = self.n_spans
        c.span_id = _ptr(self.span_id, capi.u64p)
        c.parent_id = _ptr(self.parent_id, capi.u64p)
        c.begin_ns = _ptr(self.begin_ns, capi.u64p)
        c.end_ns = _ptr(self.end_ns, capi.u64p)
        c.cid = _ptr(self.cid, capi.u64p)
        c.flags = _ptr(self.flags, capi.u8p)
        c.name_id = _ptr(self.name_id, capi.u32p)
        c.n_metric_rows = int(self.flops.size)
        c.flops = _ptr(self.flops, capi.u64p)
        c.dram_read = _ptr(self.dram_read, capi.u64p)
        c.dram_write = _ptr(self.dram_write, capi.u64p)
        c.occupancy = _ptr(self.occupancy, capi.f64p)
        c.n_layer_rows = int(self.alloc_bytes.size)
        c.alloc_bytes = _ptr(self.alloc_bytes, capi.i64p)
        c.type_id = _ptr(self.type_id, capi.u32p)
        return c

    def traces(self) -> capi.Traces:
        t = capi.Traces()
        t.n_traces = self.n_traces
        t.span_off = _ptr(self.trace_span_off, capi.u64p)
        t.levels = _ptr(self.trace_levels, capi.u32p)
        return t

    def nbytes_inputs(self) -> int:
        """Bytes of every input column the C ABI reads (span + side tables + traces)."""
        cols = list(SPAN_COLS) + list(METRIC_COLS) + list(LAYER_COLS)
        return int(sum(getattr(self, k).nbytes for k in cols) + self.trace_span_off.nbytes
                   + self.trace_levels.nbytes)

    def pinned(self) -> "SpanBatch":
        """A copy whose columns live in page-locked host memory (fast H2D/D2H)."""
        import torch
        keep = []

        def pin(a):
            view = {np.uint64: np.int64, np.uint32: np.int32}.get(a.dtype.type, a.dtype.type)
            t = torch.from_numpy(np.ascontiguousarray(a).view(view)).pin_memory()
            keep.append(t)
            return t.numpy().view(a.dtype)

        kw = {k: pin(getattr(self, k)) for k in {**SPAN_COLS, **METRIC_COLS, **LAYER_COLS, **TRACE_COLS}}
        out = SpanBatch(**kw, names=self.names, types=self.types, system_name=self.system_name,
                        peak_flops=self.peak_flops, mem_bw=self.mem_bw)
        out._pinned = keep
        return out

    def name(self, name_id: int) -> str:
        return self.names[int(name_id)].decode()

    # ---- construction
    @classmethod
    def from_bag(cls, bag: Dict[str, np.ndarray], strings: Dict[str, List[bytes]]) -> "SpanBatch":
        kw = {k: bag[k] for k in {**SPAN_COLS, **METRIC_COLS, **LAYER_COLS, **TRACE_COLS}}
        sysname = strings.get("system_name", [b"tesla-v100-sxm2"])
        return cls(**kw, names=list(strings["names"]), types=list(strings["types"]),
                   system_name=sysname[0] if sysname else b"",
                   peak_flops=float(bag["system_peak"][0]) if "system_peak" in bag else 15.7e12,
                   mem_bw=float(bag["system_bw"][0]) if "system_bw" in bag else 900e9)

    @classmethod
    def concat(cls, batches: Sequence["SpanBatch"]) -> "SpanBatch":
        """Concatenate batches, re-interning names/types in lexicographic order."""
        names = sorted({n for b in batches for n in b.names})
        types = sorted({n for b in batches for n in b.types})
        nid = {n: i for i, n in enumerate(names)}
        tid = {n: i for i, n in enumerate(types)}
        parts: Dict[str, list] = {k: [] for k in {**SPAN_COLS, **METRIC_COLS, **LAYER_COLS, **TRACE_COLS}}
        base = 0
        for b in batches:
            nmap = np.array([nid[n] for n in b.names], dtype=np.uint32)
            tmap = np.array([tid[n] for n in b.types], dtype=np.uint32)
            for k in SPAN_COLS:
                v = getattr(b, k)
                parts[k].append(nmap[v] if (k == "name_id" and v.size) else v)
            for k in METRIC_COLS:
                parts[k].append(getattr(b, k))
            parts["alloc_bytes"].append(b.alloc_bytes)
            parts["type_id"].append(tmap[b.type_id] if b.type_id.size else b.type_id)
            parts["trace_span_off"].append(b.trace_span_off[:-1] + base)
            for k in ("trace_id", "trace_levels", "trace_batch", "trace_run", "trace_serialized"):
                parts[k].append(getattr(b, k))
            base += b.n_spans
        parts["trace_span_off"].append(np.array([base], dtype=np.uint64))
        kw = {k: (np.concatenate(v) if v else np.zeros(0)) for k, v in parts.items()}
        first = batches[0]
        return cls(**kw, names=names, types=types, system_name=first.system_name,
                   peak_flops=first.peak_flops, mem_bw=first.mem_bw)

    def trace_slice(self, t0: int, t1: int) -> "SpanBatch":
        """Traces [t0, t1) as a new batch (same string tables)."""
        s0, s1 = int(self.trace_span_off[t0]), int(self.trace_span_off[t1])
        lay = self.level() == capi.LEVEL_LAYER
        met = (self.flags & capi.F_METRICS) != 0
        m0, m1 = int(met[:s0].sum()), int(met[:s1].sum())
        l0, l1 = int(lay[:s0].sum()), int(lay[:s1].sum())
        kw = {k: getattr(self, k)[s0:s1] for k in SPAN_COLS}
        kw.update({k: getattr(self, k)[m0:m1] for k in METRIC_COLS})
        kw.update({k: getattr(self, k)[l0:l1] for k in LAYER_COLS})
        kw["trace_span_off"] = self.trace_span_off[t0:t1 + 1] - s0
        for k in ("trace_id", "trace_levels", "trace_batch", "trace_run", "trace_serialized"):
            kw[k] = getattr(self, k)[t0:t1]
        return SpanBatch(**kw, names=self.names, types=self.types, system_name=self.system_name,
                         peak_flops=self.peak_flops, mem_bw=self.mem_bw)

    def select_traces(self, idx: Sequence[int]) -> "SpanBatch":
        """Traces idx (any order, repeats allowed) as a new batch (same string tables)."""
        idx = np.asarray(idx, dtype=np.int64)
        off = self.trace_span_off.astype(np.int64)
        lay = (self.level() == capi.LEVEL_LAYER).astype(np.int64)
        met = ((self.flags & capi.F_METRICS) != 0).astype(np.int64)
        moff = np.concatenate([[0], np.cumsum(met)])[off]
        loff = np.concatenate([[0], np.cumsum(lay)])[off]

        def rows(o):
            return np.concatenate([np.arange(o[t], o[t + 1]) for t in idx.tolist()]) if idx.size else \
                np.zeros(0, np.int64)

        sr, mr, lr = rows(off), rows(moff), rows(loff)
        kw = {k: getattr(self, k)[sr] for k in SPAN_COLS}
        kw.update({k: getattr(self, k)[mr] for k in METRIC_COLS})
        kw.update({k: getattr(self, k)[lr] for k in LAYER_COLS})
        kw["trace_span_off"] = np.concatenate([[0], np.cumsum(off[idx + 1] - off[idx])]).astype(np.uint64)
        for k in ("trace_id", "trace_levels", "trace_batch", "trace_run", "trace_serialized"):
            kw[k] = getattr(self, k)[idx]
        return SpanBatch(**kw, names=self.names, types=self.types, system_name=self.system_name,
                         peak_flops=self.peak_flops, mem_bw=self.mem_bw)


_LEVEL_NAMES = ["model", "layer", "kernel", "api"]
_KIND_NAMES = ["sync", "launch", "exec"]


def to_jsonl(b: SpanBatch, t: int) -> bytes:
    """Trace t of b in the reference's JSONL wire form (encode_meta_record /
    encode_span_record: keys in order, no whitespace; collector.cpp:188-194):
    the metric table row of a span becomes its four metric tags, the layer table
    row its alloc_bytes / layer_type tags. Doubles are written as Python's
    shortest round-trip repr (the reference's writer may pick other digits of
    the same double). Used to build ingest workloads and tests."""
    import json
    lv = int(b.trace_levels[t])
    s0, s1 = int(b.trace_span_off[t]), int(b.trace_span_off[t + 1])
    f_all = b.flags
    met = (f_all & capi.F_METRICS) != 0
    lay = (f_all & 3) == capi.LEVEL_LAYER
    m0, a0 = int(met[:s0].sum()), int(lay[:s0].sum())
    sysname = b.system_name.decode() if isinstance(b.system_name, bytes) else b.system_name
    out = [("{\"batch_size\":%d,\"levels\":[%s],\"rec\":\"meta\",\"run_index\":%d,\"serialized\":%s,"
            "\"system\":{\"mem_bw\":%r,\"name\":%s,\"peak_flops\":%r},\"trace_id\":%d}")
           % (int(b.trace_batch[t]), ",".join(json.dumps(_LEVEL_NAMES[i]) for i in range(4) if lv >> i & 1),
              int(b.trace_run[t]), "true" if int(b.trace_serialized[t]) else "false", float(b.mem_bw),
              json.dumps(sysname), float(b.peak_flops), int(b.trace_id[t]))]
    tid = int(b.trace_id[t])
    qn = [json.dumps(n.decode()) for n in b.names]
    qt = [json.dumps(n.decode()) for n in b.types]
    fl = f_all[s0:s1].tolist()
    beg, end = b.begin_ns[s0:s1].tolist(), b.end_ns[s0:s1].tolist()
    cid, par, sid = b.cid[s0:s1].tolist(), b.parent_id[s0:s1].tolist(), b.span_id[s0:s1].tolist()
    nid = b.name_id[s0:s1].tolist()
    nm = int(met[s0:s1].sum())
    na = int(lay[s0:s1].sum())
    occ = b.occupancy[m0:m0 + nm].tolist()
    rd, wr, fo = b.dram_read[m0:m0 + nm].tolist(), b.dram_write[m0:m0 + nm].tolist(), b.flops[m0:m0 + nm].tolist()
    al, ty = b.alloc_bytes[a0:a0 + na].tolist(), b.type_id[a0:a0 + na].tolist()
    kinds = ["sync", "launch", "exec", "?"]
    levels = _LEVEL_NAMES
    mi = ai = 0
    tail = ',"trace_id":%d}' % tid
    for k in range(s1 - s0):
        f = fl[k]
        if f & 0x40:
            tags = '"achieved_occupancy":%r,"dram_read_bytes":%d,"dram_write_bytes":%d,"flop_count_sp":%d' % (
                occ[mi], rd[mi], wr[mi], fo[mi])
            mi += 1
        else:
            tags = ""
        if (f & 3) == 1:
            tags = '"alloc_bytes":%d,"layer_type":%s' % (al[ai], qt[ty[ai]])
            ai += 1
        out.append('{"begin_ns":%d,"correlation_id":%s,"end_ns":%d,"kind":"%s","level":"%s","name":%s,'
                   '"parent_id":%s,"rec":"span","span_id":%d,"tags":{%s}' % (
                       beg[k], cid[k] if f & 0x20 else "null", end[k], kinds[(f >> 2) & 3], levels[f & 3],
                       qn[nid[k]], par[k] if f & 0x10 else "null", sid[k], tags) + tail)
    return ("\n".join(out) + "\n").encode()
