"""Host-side mirror of the reference correlate / analyze interface over the C ABI.

Reference interface (namespace strata):
  correlate(const TraceBundle&)                 correlator.hpp:164
  a8_kernel_table ... a15_model_aggregate       analysis.hpp:256-366
Here a whole batch of traces (SpanBatch) goes through ONE C-ABI call and the
results come back as numpy columns; per-trace faults (the reference's
TraceError) are reported per trace with the reference's exact message text.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as capi
from .columns import SpanBatch

_NP = {capi.u8p: np.uint8, capi.i8p: np.int8, capi.u32p: np.uint32, capi.i32p: np.int32,
       capi.u64p: np.uint64, capi.i64p: np.int64, capi.f64p: np.float64}

ORPHAN_TEXT = {
    1: "layer-level span with non-sync kind",
    2: "explicit parent {p} is not the model span",
    3: "outside the model interval",
    4: "explicit parent {p} is not a layer in the tree",
    5: "contained in no layer interval",
    6: "execution record without correlation id",
    7: "launch without correlation id",
    8: "launch has no matching execution record",
    9: "execution record without matching launch",
}


def _copy(ptr, typ, count: int) -> np.ndarray:
    dt = _NP[typ]
    if count == 0 or not ptr:
        return np.zeros(0, dtype=dt)
    addr = C.cast(ptr, C.c_void_p).value
    buf = (C.c_char * (count * np.dtype(dt).itemsize)).from_address(addr)
    return np.frombuffer(buf, dtype=dt).copy()


@dataclass
class CorrResult:
    """CorrelationResult columns for every trace of a batch (include/xsp.h xsp_corr_out)."""
    n_traces: int
    n_failed: int
    cols: Dict[str, np.ndarray]
    n_layers: int = 0
    n_kernels: int = 0
    n_orphans: int = 0
    n_ambiguities: int = 0
    n_candidates: int = 0

    def __getattr__(self, k):
        try:
            return self.__dict__["cols"][k]
        except KeyError as e:
            raise AttributeError(k) from e

    def error_message(self, batch: SpanBatch, t: int) -> str:
        """The what() text of the TraceError the reference throws for trace t ('' if none)."""
        s = int(self.trace_status[t])
        a, b = (int(x) for x in self.trace_err_row[2 * t:2 * t + 2])
        if s == capi.T_OK:
            return ""
        if s == capi.T_NO_MODEL:
            return "bundle has no model span; nothing to correlate"
        if s == capi.T_MULTI_MODEL:
            return "bundle has more than one model span"
        if s == capi.T_SER_AMBIGUOUS:
            return f"serialized run is itself ambiguous ({a} span(s)); cannot resolve"
        if s == capi.T_SER_FAILED:
            return "serialized run failed to correlate (see the serialized batch)"
        if s == capi.T_SKIP_LEVEL:
            return (f"span {int(batch.span_id[a])} ('{batch.name(batch.name_id[a])}') is kernel-level "
                    "but the run did not profile the layer level; parents cannot skip a level")
        kind = "execution" if s == capi.T_DUP_EXEC_CID else "launch"
        return (f"correlation id {int(batch.cid[b])} is shared by {kind} spans "
                f"{int(batch.span_id[a])} and {int(batch.span_id[b])}")

    def orphan_text(self, batch: SpanBatch, j: int) -> str:
        r = int(self.orphan_reason[j])
        row = int(self.orphan_row[j])
        return ORPHAN_TEXT[r].format(p=int(batch.parent_id[row]))


@dataclass
class Tables:
    """a8..a15 columns for every group (include/xsp.h xsp_tables_out)."""
    n_groups: int
    cols: Dict[str, np.ndarray]
    n_layers: int = 0
    n_kernels: int = 0
    n_names: int = 0

    def __getattr__(self, k):
        try:
            return self.__dict__["cols"][k]
        except KeyError as e:
            raise AttributeError(k) from e


def fill_lookups(corr: "CorrResult", batch: SpanBatch) -> None:
    """The four xsp_corr_out columns XSP_HOST_OUT_ROWS does not copy back, as the
    lookups include/xsp.h defines them (filled only where absent)."""
    def dur(rows):
        b, e = batch.begin_ns[rows], batch.end_ns[rows]
        return np.where(e >= b, e - b, 0).astype(np.uint64)
    c = corr.cols
    lr = c["layer_row"].astype(np.int64)
    xr = c["kernel_exec_row"].astype(np.int64)
    mr = c["kernel_metric_row"]
    if not c.get("layer_dur", np.zeros(0)).size and lr.size:
        c["layer_dur"] = dur(lr)
    if not c.get("kernel_dur", np.zeros(0)).size and xr.size:
        c["kernel_dur"] = dur(xr)
        c["kernel_name"] = batch.name_id[xr].astype(np.uint32)
        has = mr != 0xFFFFFFFF
        occ = np.zeros(xr.size, dtype=np.float64)
        occ[has] = batch.occupancy[mr[has].astype(np.int64)]
        c["kernel_occ"] = occ


def _corr_counts(o: capi.CorrOut) -> Dict[str, int]:
    T = o.n_traces
    return {"T": T, "2T": 2 * T, "T1": T + 1, "L": o.n_layers, "L1": o.n_layers + 1,
            "K": o.n_kernels, "O": o.n_orphans, "A": o.n_ambiguities, "A1": o.n_ambiguities + 1,
            "AC": o.n_candidates}


def _tab_counts(o: capi.TablesOut, top_k: int) -> Dict[str, int]:
    G = o.n_groups
    return {"G": G, "G1": G + 1, "K": o.n_kernels, "L": o.n_layers, "N": o.n_names,
            "LK": o.n_layers * max(top_k, 1), "Y": o.n_type_rows}


class DeviceBatch:
    """A SpanBatch resident in HBM (torch tensors are only the allocator here)."""

    def __init__(self, batch: SpanBatch, device: int = 0):
        import torch
        self.batch = batch
        self.t = {}
        for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags", "name_id", "flops",
                  "dram_read", "dram_write", "occupancy", "alloc_bytes", "type_id", "trace_span_off",
                  "trace_levels"):
            a = getattr(batch, k)
            view = {np.uint64: np.int64, np.uint32: np.int32}.get(a.dtype.type, a.dtype.type)
            self.t[k] = torch.from_numpy(np.ascontiguousarray(a).view(view)).to(f"cuda:{device}")
        self.nbytes = sum(int(x.numel() * x.element_size()) for x in self.t.values())

    def ptr(self, k) -> int:
        x = self.t[k]
        return x.data_ptr() if x.numel() else 0

    def _p(self, k, typ):
        x = self.t[k]
        return C.cast(C.c_void_p(x.data_ptr() if x.numel() else 0), typ)

    def cols(self) -> capi.SpanCols:
        b = self.batch
        c = capi.SpanCols()
        c.n_spans = b.n_spans
        for k, typ in (("span_id", capi.u64p), ("parent_id", capi.u64p), ("begin_ns", capi.u64p),
                       ("end_ns", capi.u64p), ("cid", capi.u64p), ("flags", capi.u8p),
                       ("name_id", capi.u32p), ("flops", capi.u64p), ("dram_read", capi.u64p),
                       ("dram_write", capi.u64p), ("occupancy", capi.f64p),
                       ("alloc_bytes", capi.i64p), ("type_id", capi.u32p)):
            setattr(c, k, self._p(k, typ))
        c.n_metric_rows = int(b.flops.size)
        c.n_layer_rows = int(b.alloc_bytes.size)
        return c

    def traces(self) -> capi.Traces:
        t = capi.Traces()
        t.n_traces = self.batch.n_traces
        t.span_off = self._p("trace_span_off", capi.u64p)
        t.levels = self._p("trace_levels", capi.u32p)
        return t


class Engine:
    """One xsp context on one CUDA device (no CPU fallback)."""

    def __init__(self, device: int = 0):
        self.lib = capi.load()
        self.ctx = C.c_void_p()
        st = self.lib.xsp_ctx_create(device, C.byref(self.ctx))
        if st != capi.XSP_OK:
            raise capi.XspError(st, "xsp_ctx_create failed (no CUDA device?)")

    def close(self):
        if self.ctx:
            self.lib.xsp_ctx_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st != capi.XSP_OK:
            raise capi.XspError(st, self.lib.xsp_last_error(self.ctx).decode())

    @property
    def launches(self) -> int:
        return int(self.lib.xsp_last_launch_count(self.ctx))

    def transfer_bytes(self) -> Tuple[int, int]:
        h, d = C.c_uint64(), C.c_uint64()
        self.lib.xsp_last_transfer_bytes(self.ctx, C.byref(h), C.byref(d))
        return int(h.value), int(d.value)

    @staticmethod
    def make_groups(first: Sequence[int], runs: Sequence[int], batch: Sequence[int]):
        f = np.ascontiguousarray(first, dtype=np.uint32)
        r = np.ascontiguousarray(runs, dtype=np.uint32)
        b = np.ascontiguousarray(batch, dtype=np.uint32)
        g = capi.Groups()
        g.n_groups = f.size
        g.first_trace = f.ctypes.data_as(capi.u32p)
        g.n_runs = r.ctypes.data_as(capi.u32p)
        g.batch_size = b.ctypes.data_as(capi.u32p)
        return g, (f, r, b)

    @staticmethod
    def make_opts(trim=0.2, epsilon=0.05, noise=0.01, top_k=3):
        o = capi.AnalysisOpts()
        o.trim_fraction, o.epsilon, o.noise_tolerance, o.top_k = trim, epsilon, noise, top_k
        return o

    # ---- device-resident path (inputs already in HBM; results stay in HBM)
    def correlate_device(self, dbatch: DeviceBatch, stream=None) -> capi.CorrOut:
        cols, trs = dbatch.cols(), dbatch.traces()
        co = capi.CorrOut()
        self._check(self.lib.xsp_correlate(self.ctx, C.byref(cols), C.byref(trs), 1, C.byref(co),
                                           C.c_void_p(stream)))
        return co

    def analyze_device(self, dbatch: DeviceBatch, corr: capi.CorrOut, groups, trim=0.2, noise=0.01,
                       top_k=3, stream=None) -> capi.TablesOut:
        g, keep = self.make_groups(*groups)
        spec = capi.SystemSpec(dbatch.batch.peak_flops, dbatch.batch.mem_bw)
        opts = self.make_opts(trim=trim, noise=noise, top_k=top_k)
        cols = dbatch.cols()
        to = capi.TablesOut()
        self._check(self.lib.xsp_analyze(self.ctx, C.byref(cols), C.byref(corr), C.byref(g),
                                         C.byref(spec), C.byref(opts), C.byref(to), C.c_void_p(stream)))
        return to

    def run_device(self, dbatch: DeviceBatch, groups, trim=0.2, noise=0.01, top_k=3, stream=None):
        """correlate + analyze of device-resident columns in one C-ABI call (xsp_run);
        the argument structs are built once per (batch, groups) and reused."""
        key = (id(dbatch), id(groups), trim, noise, top_k)
        if getattr(self, "_run_key", None) != key:
            g, keep = self.make_groups(*groups)
            spec = capi.SystemSpec(dbatch.batch.peak_flops, dbatch.batch.mem_bw)
            self._run_args = (dbatch.cols(), dbatch.traces(), g, spec, self.make_opts(trim=trim, noise=noise,
                                                                                      top_k=top_k), keep, dbatch)
            self._run_key = key
        cols, trs, g, spec, opts, _, _ = self._run_args
        co, to = capi.CorrOut(), capi.TablesOut()
        self._check(self.lib.xsp_run(self.ctx, C.byref(cols), C.byref(trs), C.byref(g), C.byref(spec),
                                     C.byref(opts), C.byref(co), C.byref(to), C.c_void_p(stream)))
        return co, to

    # ---- JSONL ingest (xsp_ingest_jsonl)
    def ingest_jsonl(self, streams, stream=None) -> Tuple[Optional[SpanBatch], int]:
        """ingest() of each JSONL stream (bytes) on the GPU -> (SpanBatch with one
        trace per stream, -1), or (None, stream) when that stream needs the
        reference-exact host parser (xsp.h XSP_INGEST_HOST)."""
        from .leveled import _d2h
        blob = b"".join(streams)
        off = np.zeros(len(streams) + 1, dtype=np.uint64)
        if streams:
            off[1:] = np.cumsum([len(x) for x in streams])
        out = capi.IngestOut()
        self._check(self.lib.xsp_ingest_jsonl(self.ctx, blob, off.ctypes.data_as(capi.u64p), len(streams),
                                              C.byref(out), C.c_void_p(stream)))
        if out.status != capi.INGEST_OK:
            return None, int(out.bad_stream)
        c = out.cols
        n, M, Lr, T = int(c.n_spans), int(c.n_metric_rows), int(c.n_layer_rows), len(streams)
        d = lambda ptr, dt, k: _d2h(self.lib, self.ctx, ptr, dt, k)
        h = lambda ptr, dt, k: _copy(ptr, {np.uint64: capi.u64p, np.uint32: capi.u32p, np.uint8: capi.u8p}[dt], k)

        def strings(t):
            o = _copy(t.off, capi.u64p, t.n + 1)
            raw = C.string_at(t.bytes, int(o[-1])) if t.n and o[-1] else b""
            return [raw[int(o[i]):int(o[i + 1])] for i in range(t.n)]

        b = SpanBatch(span_id=d(c.span_id, np.uint64, n), parent_id=d(c.parent_id, np.uint64, n),
                      begin_ns=d(c.begin_ns, np.uint64, n), end_ns=d(c.end_ns, np.uint64, n),
                      cid=d(c.cid, np.uint64, n), flags=d(c.flags, np.uint8, n), name_id=d(c.name_id, np.uint32, n),
                      flops=d(c.flops, np.uint64, M), dram_read=d(c.dram_read, np.uint64, M),
                      dram_write=d(c.dram_write, np.uint64, M), occupancy=d(c.occupancy, np.float64, M),
                      alloc_bytes=d(c.alloc_bytes, np.int64, Lr), type_id=d(c.type_id, np.uint32, Lr),
                      trace_span_off=h(out.span_off_host, np.uint64, T + 1), trace_id=h(out.trace_id, np.uint64, T),
                      trace_levels=h(out.levels_host, np.uint32, T), trace_batch=h(out.trace_batch, np.uint32, T),
                      trace_run=h(out.trace_run, np.uint32, T), trace_serialized=h(out.trace_serialized, np.uint8, T),
                      names=strings(out.names), types=strings(out.types),
                      system_name=out.system_name or b"", peak_flops=out.peak_flops, mem_bw=out.mem_bw)
        return b, -1

    # ---- multi-GPU table combine (xsp_comm_init / xsp_combine_tables)
    def comm_init(self, world: int, rank: int, dist=None):
        """Join an NCCL communicator of `world` ranks; rank 0's unique id travels
        over torch.distributed (`dist`, any backend) when world > 1."""
        uid = (C.c_char * 128)()
        if rank == 0:
            st = self.lib.xsp_comm_unique_id(uid)
            if st != capi.XSP_OK:
                raise capi.XspError(st, "ncclGetUniqueId failed")
        if world > 1:
            obj = [bytes(uid) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            C.memmove(uid, obj[0], 128)
        self._check(self.lib.xsp_comm_init(self.ctx, world, rank, uid))

    def combine_tables(self, local: capi.TablesOut, group_ids, n_groups_total: int, l_row_map_ptr: int = 0,
                       top_k: int = 3, stream=None) -> Tuple[capi.TablesOut, int]:
        """xsp_combine_tables: every rank's device tables to rank 0 in global group
        order over NCCL; returns (rank 0's device tables, bytes this rank sent)."""
        gid = np.ascontiguousarray(group_ids, dtype=np.uint32)
        out = capi.TablesOut()
        sent = C.c_uint64(0)
        self._check(self.lib.xsp_combine_tables(self.ctx, C.byref(local), gid.ctypes.data_as(capi.u32p), gid.size,
                                                n_groups_total, C.c_void_p(l_row_map_ptr or None), top_k,
                                                C.byref(out), C.byref(sent), C.c_void_p(stream)))
        return out, sent.value

    def tables_to_host(self, to: capi.TablesOut, top_k: int = 3) -> "Tables":
        """Host copy of device tables (xsp_copy_to_host per column)."""
        from .leveled import _d2h
        tc = _tab_counts(to, top_k)
        cols = {}
        for name, typ, kind in capi.TABLE_FIELDS:
            cols[name] = _d2h(self.lib, self.ctx, getattr(to, name), _NP[typ], tc[kind])
        return Tables(to.n_groups, cols, to.n_layers, to.n_kernels, to.n_names)

    @staticmethod
    def string_table(strings):
        """xsp_string_table of a list of byte strings; returns (struct, arrays to keep alive)."""
        blob = b"".join(strings)
        off = np.zeros(len(strings) + 1, dtype=np.uint64)
        if strings:
            off[1:] = np.cumsum([len(x) for x in strings])
        st = capi.StringTable(len(strings), blob, off.ctypes.data_as(capi.u64p))
        return st, (blob, off)

    def report_csv(self, dbatch: DeviceBatch, corr: capi.CorrOut, groups, tables: capi.TablesOut, group: int,
                   table: str, stream=None) -> bytes:
        """The reference report's CSV file (report.cpp to_csv(to_table(...))) of one
        analysis table of one group, formatted on the GPU (xsp_report_csv_host) from
        the tables of the preceding analyze_device / run_device on this engine."""
        g, keep = self.make_groups(*groups)
        names, k1 = self.string_table(dbatch.batch.names)
        types, k2 = self.string_table(dbatch.batch.types)
        cols = dbatch.cols()
        text = C.c_char_p()
        n = C.c_uint64()
        self._check(self.lib.xsp_report_csv_host(self.ctx, C.byref(cols), C.byref(corr), C.byref(g),
                                                 C.byref(tables), C.byref(names), C.byref(types), group,
                                                 capi.REPORT_TABLES[table], C.byref(text), C.byref(n),
                                                 C.c_void_p(stream)))
        return C.string_at(C.cast(text, C.c_void_p).value, n.value)

    @staticmethod
    def make_level_sets(sets):
        """xsp_level_sets of [(level mask, trace indices)] (one LeveledRunGroup);
        returns (struct, arrays to keep alive)."""
        off = np.zeros(len(sets) + 1, dtype=np.uint32)
        tr = []
        for i, (_, idx) in enumerate(sets):
            tr.extend(idx)
            off[i + 1] = len(tr)
        tr = np.array(tr, dtype=np.uint32)
        lv = np.array([m for m, _ in sets], dtype=np.uint32)
        ls = capi.LevelSets(len(sets), off.ctypes.data_as(capi.u32p), tr.ctypes.data_as(capi.u32p),
                            lv.ctypes.data_as(capi.u32p))
        return ls, (off, tr, lv)

    def leveled_device(self, dbatch: DeviceBatch, corr: capi.CorrOut, level_sets, trim=0.2, noise=0.01,
                       stream=None) -> capi.OverheadOut:
        """compute_overhead (leveled.cpp:145-231) of one LeveledRunGroup over a
        device correlation (xsp_leveled); level_sets from make_level_sets."""
        cols = dbatch.cols()
        out = capi.OverheadOut()
        opts = self.make_opts(trim=trim, noise=noise)
        self._check(self.lib.xsp_leveled(self.ctx, C.byref(cols), C.byref(corr), C.byref(level_sets),
                                         C.byref(opts), C.byref(out), C.c_void_p(stream)))
        return out

    def leveled_batch_device(self, dbatch: DeviceBatch, corr: capi.CorrOut, level_sets_list, trim=0.2,
                             noise=0.01, stream=None):
        """xsp_leveled_batch: compute_overhead of many LeveledRunGroups in one
        call; level_sets_list = [make_level_sets(...)[0], ...]. Returns the
        OverheadOut of every group (valid until the next leveled call)."""
        cols = dbatch.cols()
        n = len(level_sets_list)
        arr = (capi.LevelSets * max(n, 1))(*level_sets_list)
        outs = (capi.OverheadOut * max(n, 1))()
        opts = self.make_opts(trim=trim, noise=noise)
        self._check(self.lib.xsp_leveled_batch(self.ctx, C.byref(cols), C.byref(corr), n, arr, C.byref(opts),
                                               outs, C.c_void_p(stream)))
        self._lev_keep = (arr, level_sets_list)
        return list(outs)[:n]

    def pack_host(self, batch: SpanBatch) -> capi.PackedCols:
        """xsp_pack_host: the batch's span columns in the packed wire form (ctx-owned
        pinned arrays, valid until the next pack_host on this engine)."""
        self._pack_src = batch  # flags / name_id are referenced, not copied
        cols, trs = batch.cols(), batch.traces()
        pk = capi.PackedCols()
        self._check(self.lib.xsp_pack_host(self.ctx, C.byref(cols), C.byref(trs), C.byref(pk)))
        return pk

    def run_host_packed(self, packed: capi.PackedCols, batch: SpanBatch, groups=None, trim=0.2, noise=0.01,
                        top_k=3, raw: bool = False):
        """xsp_run_host_packed: run_host with the span columns taken from `packed`
        (batch supplies span_id and the metric / layer tables)."""
        if groups is None:
            T = batch.n_traces
            groups = (np.arange(T), np.ones(T), batch.trace_batch)
        g, keep = self.make_groups(*groups)
        spec = capi.SystemSpec(batch.peak_flops, batch.mem_bw)
        opts = self.make_opts(trim=trim, noise=noise, top_k=top_k)
        cols, trs = batch.cols(), batch.traces()
        co, to = capi.CorrOut(), capi.TablesOut()
        self._check(self.lib.xsp_run_host_packed(self.ctx, C.byref(packed), C.byref(cols), C.byref(trs), C.byref(g),
                                                 C.byref(spec), C.byref(opts), C.byref(co), C.byref(to), None))
        if raw:
            return co, to
        cc = _corr_counts(co)
        corr = CorrResult(co.n_traces, co.n_failed,
                          {n: _copy(getattr(co, n), t, cc[k]) for n, t, k in capi.CORR_FIELDS},
                          co.n_layers, co.n_kernels, co.n_orphans, co.n_ambiguities, co.n_candidates)
        tc = _tab_counts(to, top_k)
        tabs = Tables(to.n_groups, {n: _copy(getattr(to, n), t, tc[k]) for n, t, k in capi.TABLE_FIELDS},
                      to.n_layers, to.n_kernels, to.n_names)
        return corr, tabs

    def set_host_outputs(self, mode: int):
        """xsp_set_host_outputs: capi.HOST_OUT_ROWS leaves layer_dur / kernel_dur /
        kernel_name / kernel_occ on the device (fill_lookups rebuilds them)."""
        self._check(self.lib.xsp_set_host_outputs(self.ctx, mode))

    def set_profiling(self, on: bool):
        self.lib.xsp_set_profiling(self.ctx, int(on))

    def stage_reset(self):
        self.lib.xsp_stage_reset(self.ctx)

    def stage_times(self) -> Dict[str, Tuple[float, int]]:
        n = self.lib.xsp_stage_times(self.ctx, 0, None, None, None)
        names = (C.c_char_p * max(n, 1))()
        ms = (C.c_double * max(n, 1))()
        cnt = (C.c_uint64 * max(n, 1))()
        self.lib.xsp_stage_times(self.ctx, n, names, ms, cnt)
        return {names[i].decode(): (ms[i], int(cnt[i])) for i in range(n)}

    def sort_timeline(self, batch: SpanBatch) -> Tuple[np.ndarray, bool]:
        """sort_timeline (span.cpp:112-127) of every trace: (perm, was_sorted), perm[j] =
        input row of the span at position j (xsp_sort_timeline_host)."""
        perm = np.zeros(max(batch.n_spans, 1), dtype=np.uint32)
        ws = C.c_int()
        self._check(self.lib.xsp_sort_timeline_host(
            self.ctx, batch.n_spans, batch.begin_ns.ctypes.data_as(capi.u64p),
            batch.flags.ctypes.data_as(capi.u8p), batch.span_id.ctypes.data_as(capi.u64p), batch.n_traces,
            batch.trace_span_off.ctypes.data_as(capi.u64p), perm.ctypes.data_as(capi.u32p), C.byref(ws)))
        return perm[:batch.n_spans], bool(ws.value)

    def sort_timeline_device(self, dbatch: "DeviceBatch", perm_ptr: int, stream=None) -> bool:
        """Device-resident sort_timeline into a caller-owned device u32 array."""
        b = dbatch
        ws = C.c_int()
        self._check(self.lib.xsp_sort_timeline(
            self.ctx, b.batch.n_spans, C.c_void_p(b.ptr("begin_ns")), C.c_void_p(b.ptr("flags")),
            C.c_void_p(b.ptr("span_id")), b.batch.n_traces, C.c_void_p(b.ptr("trace_span_off")),
            C.c_void_p(perm_ptr), C.byref(ws), C.c_void_p(stream)))
        return bool(ws.value)

    def resolve_serialized(self, original: SpanBatch, serialized: SpanBatch) -> CorrResult:
        """resolve_with_serialized (correlator.cpp:379-456) for every trace pair
        (xsp_resolve_serialized_host); both batches share one name table."""
        if original.names != serialized.names:
            raise ValueError("resolve_serialized: the batches must share one name table")
        oc, ot = original.cols(), original.traces()
        sc, stt = serialized.cols(), serialized.traces()
        co = capi.CorrOut()
        self._check(self.lib.xsp_resolve_serialized_host(self.ctx, C.byref(oc), C.byref(ot), C.byref(sc),
                                                         C.byref(stt), C.byref(co)))
        cc = _corr_counts(co)
        return CorrResult(co.n_traces, co.n_failed,
                          {n: _copy(getattr(co, n), t, cc[k]) for n, t, k in capi.CORR_FIELDS},
                          co.n_layers, co.n_kernels, co.n_orphans, co.n_ambiguities, co.n_candidates)

    def validate(self, batch: SpanBatch, span_trace_id: Optional[np.ndarray] = None,
                 tag_bits: Optional[np.ndarray] = None) -> List[List[Tuple[int, int]]]:
        """validate_bundle (span.cpp:129-192) of every trace (xsp_validate_host).

        span_trace_id: per-span Span::trace_id (checked against batch.trace_id);
        tag_bits: per-span XSP_TAG_* raw-tag facts. Returns, per trace, the
        (span row or -1, rule) issues in the reference's report order."""
        cols, trs = batch.cols(), batch.traces()
        vin = capi.ValidateIn()
        keep = []
        if span_trace_id is not None:
            a = np.ascontiguousarray(span_trace_id, dtype=np.uint64)
            m = np.ascontiguousarray(batch.trace_id, dtype=np.uint64)
            keep += [a, m]
            vin.trace_id, vin.meta_trace_id = a.ctypes.data_as(capi.u64p), m.ctypes.data_as(capi.u64p)
        if tag_bits is not None:
            tb = np.ascontiguousarray(tag_bits, dtype=np.uint8)
            keep.append(tb)
            vin.tag_bits = tb.ctypes.data_as(capi.u8p)
        out = capi.ValidationOut()
        self._check(self.lib.xsp_validate_host(self.ctx, C.byref(cols), C.byref(trs), C.byref(vin),
                                               C.byref(out)))
        n = int(out.n_issues)
        off = _copy(out.trace_issue_off, capi.u32p, batch.n_traces + 1)
        row = _copy(out.issue_row, capi.u32p, n).astype(np.int64)
        rule = _copy(out.issue_rule, capi.u8p, n)
        row[row == 0xFFFFFFFF] = -1
        return [list(zip(row[off[t]:off[t + 1]].tolist(), rule[off[t]:off[t + 1]].tolist()))
                for t in range(batch.n_traces)]

    def run_host(self, batch: SpanBatch, groups: Optional[Tuple[Sequence[int], Sequence[int], Sequence[int]]] = None,
                 trim=0.2, noise=0.01, top_k=3, peak_flops=None, mem_bw=None,
                 raw: bool = False) -> Tuple[CorrResult, Tables]:
        """correlate + analyze a host-resident batch end to end (xsp_run_host).

        groups: (first_trace, n_runs, batch_size) arrays; default one group per trace.
        raw=True returns the C structs whose columns stay in ctx-owned pinned memory."""
        if groups is None:
            T = batch.n_traces
            groups = (np.arange(T), np.ones(T), batch.trace_batch)
        g, keep = self.make_groups(*groups)
        spec = capi.SystemSpec(batch.peak_flops if peak_flops is None else peak_flops,
                               batch.mem_bw if mem_bw is None else mem_bw)
        opts = self.make_opts(trim=trim, noise=noise, top_k=top_k)
        cols, trs = batch.cols(), batch.traces()
        co, to = capi.CorrOut(), capi.TablesOut()
        self._check(self.lib.xsp_run_host(self.ctx, C.byref(cols), C.byref(trs), C.byref(g),
                                          C.byref(spec), C.byref(opts), C.byref(co), C.byref(to),
                                          None))
        if raw:
            return co, to
        cc = _corr_counts(co)
        corr = CorrResult(co.n_traces, co.n_failed,
                          {n: _copy(getattr(co, n), t, cc[k]) for n, t, k in capi.CORR_FIELDS},
                          co.n_layers, co.n_kernels, co.n_orphans, co.n_ambiguities, co.n_candidates)
        tc = _tab_counts(to, top_k)
        tabs = Tables(to.n_groups, {n: _copy(getattr(to, n), t, tc[k]) for n, t, k in capi.TABLE_FIELDS},
                      to.n_layers, to.n_kernels, to.n_names)
        return corr, tabs
