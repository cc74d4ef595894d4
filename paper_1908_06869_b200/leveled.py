"""Leveled-measurement merge (stage f) over the C ABI, with the reference's report.

Reference: LeveledRunGroup::add / from_bundles (leveled.cpp:56-84) and
compute_overhead (:145-231). The per-(level set, event) trimmed means, the
per-step overhead subtraction and the clamp rule run on the device
(xsp_leveled); this module reproduces the host-side bookkeeping of the report:
run grouping and its faults, row order, overhead maps keyed by the added level
set, and the warning strings, verbatim.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import _capi as capi
from .columns import SpanBatch

LETTER = {0: "M", 1: "L", 2: "G", 3: "A"}  # level_letter (leveled.cpp:24-32)
RANK = {0: 1, 1: 2, 2: 3, 3: 3}


def level_set_label(mask: int) -> str:
    """level_set_label (leveled.cpp:34-41): letters in Level order joined by '+'."""
    return "+".join(LETTER[l] for l in range(4) if mask >> l & 1)


def event_label(level: int, layer: int, kernel: int) -> str:
    """event_label (leveled.cpp:43-51)."""
    if level == 0:
        return "model"
    if level == 1:
        return f"layer {layer}"
    return f"layer {layer} kernel {kernel}"


def deepest_rank(mask: int) -> int:
    return max((RANK[l] for l in range(4) if mask >> l & 1), default=0)


@dataclass
class OverheadRow:
    level: int
    layer_index: int
    kernel_index: int
    accurate_latency_ns: Optional[float]
    overhead_by_added_levels: Dict[int, float]  # added-level mask -> ns
    clamped: bool


@dataclass
class OverheadReport:
    rows: List[OverheadRow] = field(default_factory=list)
    model_overhead_by_added_levels: Dict[int, float] = field(default_factory=dict)
    noise_tolerance: float = 0.0
    warnings: List[str] = field(default_factory=list)


class LeveledError(RuntimeError):
    pass


def _d2h(lib, ctx, ptr, dtype, count):
    out = np.zeros(count, dtype=dtype)
    if count:
        st = lib.xsp_copy_to_host(ctx, out.ctypes.data, C.cast(ptr, C.c_void_p), out.nbytes)
        if st != capi.XSP_OK:
            raise capi.XspError(st, lib.xsp_last_error(ctx).decode())
    return out


def compute_overhead(engine, batch: SpanBatch, trim: float = 0.2, noise: float = 0.01,
                     system=None) -> OverheadReport:
    """LeveledRunGroup::from_bundles(all traces of `batch`) + compute_overhead.

    Raises LeveledError / a TraceError-equivalent RuntimeError with the
    reference's message on the reference's faults."""
    from .engine import DeviceBatch
    lib, ctx = engine.lib, engine.ctx
    dev = DeviceBatch(batch)
    co = engine.correlate_device(dev)
    T = batch.n_traces
    status = _d2h(lib, ctx, co.trace_status, np.int32, T)
    amb_off = _d2h(lib, ctx, co.trace_amb_off, np.uint32, T + 1)
    err_rows = _d2h(lib, ctx, co.trace_err_row, np.uint32, 2 * T)
    # LeveledRunGroup::add per bundle, in order (leveled.cpp:56-77)
    sets: Dict[int, List[int]] = {}
    batch0 = None
    for t in range(T):
        if t > 0 and int(batch.trace_batch[t]) != batch0:
            raise LeveledError(f"runs mix batch sizes {batch0} and {int(batch.trace_batch[t])}")
        if t == 0:
            batch0 = int(batch.trace_batch[0])
        if status[t] != capi.T_OK:
            from .engine import CorrResult
            cr = CorrResult(T, 0, {"trace_status": status, "trace_err_row": err_rows})
            raise RuntimeError(cr.error_message(batch, t))
        namb = int(amb_off[t + 1] - amb_off[t])
        if namb:
            raise LeveledError(f"trace {int(batch.trace_id[t])} has {namb} ambiguous span(s); "
                               "resolve with a serialized rerun before leveling")
        sets.setdefault(int(batch.trace_levels[t]), []).append(t)
    masks = list(sets.keys())
    off = np.zeros(len(masks) + 1, dtype=np.uint32)
    tr = []
    for i, m in enumerate(masks):
        tr.extend(sets[m])
        off[i + 1] = len(tr)
    tr = np.array(tr, dtype=np.uint32)
    lv = np.array(masks, dtype=np.uint32)
    ls = capi.LevelSets(len(masks), off.ctypes.data_as(capi.u32p), tr.ctypes.data_as(capi.u32p),
                        lv.ctypes.data_as(capi.u32p))
    opts = engine.make_opts(trim=trim, noise=noise)
    out = capi.OverheadOut()
    cols = dev.cols()
    engine._check(lib.xsp_leveled(ctx, C.byref(cols), C.byref(co), C.byref(ls), C.byref(opts),
                                  C.byref(out), None))
    if out.status == capi.L_NOT_CHAIN:
        raise LeveledError(f"profiling-level sets {level_set_label(masks[out.err_a])} and "
                           f"{level_set_label(masks[out.err_b])} do not form an inclusion chain")
    if out.status == capi.L_TOO_FEW:
        raise LeveledError(f"overhead needs at least two chained level sets; got {out.err_a}")
    if out.status != capi.L_OK:
        raise LeveledError(f"leveled status {out.status}")
    S, E = out.n_sets, out.n_events
    chain = [masks[out.chain[i]] for i in range(S)]
    lev = _d2h(lib, ctx, out.ev_level, np.uint8, E)
    lay = _d2h(lib, ctx, out.ev_layer, np.uint32, E)
    ker = _d2h(lib, ctx, out.ev_kernel, np.uint32, E)
    ov = _d2h(lib, ctx, out.overhead, np.float64, (S - 1) * E).reshape(S - 1, E)
    fl = _d2h(lib, ctx, out.step_flags, np.uint8, (S - 1) * E).reshape(S - 1, E)
    acc = _d2h(lib, ctx, out.accurate, np.float64, E)
    rep = OverheadReport(noise_tolerance=noise)
    labels = [event_label(int(lev[e]), int(lay[e]), int(ker[e])) for e in range(E)]
    maps = [dict() for _ in range(E)]
    clamped = np.zeros(E, dtype=bool)
    for s in range(S - 1):
        narrow, wide = chain[s], chain[s + 1]
        added = wide & ~narrow
        for e in range(E):
            f = int(fl[s, e])
            if f & capi.EV_IN_NARROW:
                if not f & capi.EV_IN_WIDE:
                    rep.warnings.append(f"{labels[e]} visible under {level_set_label(narrow)} but not under "
                                        f"{level_set_label(wide)}")
                    continue
                if f & capi.EV_NEGATIVE:
                    rep.warnings.append(f"{labels[e]}: overhead of added level(s) {level_set_label(added)} "
                                        "is negative beyond noise tolerance")
                clamped[e] |= bool(f & capi.EV_CLAMPED)
                maps[e][added] = float(ov[s, e])
        dn = deepest_rank(narrow)
        for e in range(E):
            f = int(fl[s, e])
            if f & capi.EV_IN_WIDE and not f & capi.EV_IN_NARROW and RANK[int(lev[e])] <= dn:
                rep.warnings.append(f"{labels[e]} visible under {level_set_label(wide)} but not under "
                                    f"{level_set_label(narrow)}")
    for e in range(E):
        rep.rows.append(OverheadRow(int(lev[e]), int(lay[e]), int(ker[e]),
                                    None if np.isnan(acc[e]) else float(acc[e]), maps[e], bool(clamped[e])))
    if rep.rows and rep.rows[0].level == 0:
        rep.model_overhead_by_added_levels = dict(rep.rows[0].overhead_by_added_levels)
    return rep
