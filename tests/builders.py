"""Hand-built traces for edge cases (mirrors make_span / bundle_of in the
reference's tests/test_correlator.cpp:39-58)."""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import numpy as np

from paper_1908_06869_b200 import SpanBatch
from paper_1908_06869_b200 import _capi as capi

MODEL, LAYER, KERNEL, API = 0, 1, 2, 3
SYNC, LAUNCH, EXEC = 0, 1, 2
RANK = {MODEL: 1, LAYER: 2, KERNEL: 3, API: 3}
MLG = (1 << MODEL) | (1 << LAYER) | (1 << KERNEL)


def span(id, level, begin, end, kind=SYNC, parent=None, cid=None, name=None, metrics=None,
         layer_type=None, alloc=0):
    return dict(id=id, level=level, begin=begin, end=end, kind=kind, parent=parent, cid=cid,
                name=name if name is not None else f"s{id}", metrics=metrics,
                layer_type=layer_type or "", alloc=alloc)


def sort_timeline(spans: List[dict]) -> List[dict]:
    """span.cpp:112-122: stable sort by (begin_ns, rank(level), span_id)."""
    return sorted(spans, key=lambda s: (s["begin"], RANK[s["level"]], s["id"]))


def batch_of(traces: Sequence[Sequence[dict]], levels: Optional[Sequence[int]] = None,
             sort: bool = True, batch_sizes=None) -> SpanBatch:
    """One SpanBatch holding each span list as one trace."""
    names = sorted({s["name"].encode() for tr in traces for s in tr})
    types = sorted({s["layer_type"].encode() for tr in traces for s in tr if s["level"] == LAYER})
    nid = {n: i for i, n in enumerate(names)}
    tid = {n: i for i, n in enumerate(types)}
    cols: Dict[str, list] = {k: [] for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid",
                                             "flags", "name_id", "flops", "dram_read",
                                             "dram_write", "occupancy", "alloc_bytes", "type_id")}
    off = [0]
    for tr in traces:
        tr = sort_timeline(list(tr)) if sort else list(tr)
        for s in tr:
            f = s["level"] | (s["kind"] << 2)
            if s["parent"] is not None:
                f |= capi.F_PARENT
            if s["cid"] is not None:
                f |= capi.F_CID
            if s["metrics"] is not None:
                f |= capi.F_METRICS
                fl, rd, wr, oc = s["metrics"]
                cols["flops"].append(fl)
                cols["dram_read"].append(rd)
                cols["dram_write"].append(wr)
                cols["occupancy"].append(oc)
            if s["level"] == LAYER:
                cols["alloc_bytes"].append(s["alloc"])
                cols["type_id"].append(tid[s["layer_type"].encode()])
            cols["span_id"].append(s["id"])
            cols["parent_id"].append(s["parent"] or 0)
            cols["begin_ns"].append(s["begin"])
            cols["end_ns"].append(s["end"])
            cols["cid"].append(s["cid"] or 0)
            cols["flags"].append(f)
            cols["name_id"].append(nid[s["name"].encode()])
        off.append(off[-1] + len(tr))
    T = len(traces)
    lv = list(levels) if levels is not None else [MLG] * T
    bs = list(batch_sizes) if batch_sizes is not None else [1] * T
    u64 = ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flops", "dram_read", "dram_write")
    return SpanBatch(**{k: np.array(v, dtype=np.uint64) if k in u64 else np.array(v) for k, v in cols.items()},
                     trace_span_off=np.array(off), trace_id=np.arange(T) + 9,
                     trace_levels=np.array(lv), trace_batch=np.array(bs),
                     trace_run=np.zeros(T), trace_serialized=np.zeros(T),
                     names=names, types=types, system_name=b"testbed", peak_flops=1.0e12,
                     mem_bw=1.0e11)
