"""Time-range sharding of ONE long trace across ranks (BASELINE config 4).

A single 200M-span trace cannot be split by trace, so it is split by time: rank
r owns the rows [cut_r, cut_{r+1}) of the trace's timeline. Cuts are placed at
quiescent rows, where nothing the correlation relates crosses the boundary:

  * c is a layer/sync span, and every layer span before c ends before c begins
    (no containment candidate of a child at or after c lies before c: the
    carried open-parent set is empty by construction; correlator.cpp:141-282);
  * every correlation id before c is smaller than every id at or after c, so
    each launch->exec pair and each duplicate-cid check stays inside one shard
    (correlator.cpp:287-364);
  * no kernel-level span names an explicit parent (those could point across a
    cut; layers may, their parent is the model span).

Long-running traces have such instants at every host synchronisation (the C4
generator, synth.c4, drains its streams every `block_layers` layers); the cut
nearest after each rank's nominal start row is taken, and a trace without any
yields fewer shards.

Each shard is correlated and analysed on its own GPU as a standalone trace:
the model span row plus the shard's rows (the model is the only cross-shard
parent). What a shard needs from the others is the carry of counts — layer,
kernel, metric and layer-table rows before it — which the combine applies when
it rebases the shard tables. The per-shard results travel once to rank 0 as
byte tensors over torch.distributed (all_gather: NCCL over NVLink on GPUs,
gloo in the CPU tests), and `combine` rebuilds the unsharded result:

  * layers, kernels, a8/a9 and a11-a14 rows: concatenated and rebased (bit-exact);
  * orphans: merged per reference emission phase (layer pass, kernel pass,
    exec without cid, launch fusion in tree order, then leftover executions by
    span_id); ambiguities by span_id (bit-exact);
  * a10 / a15 / a13 totals: u64 counters and latency sums added across shards.
    A single trace is one run, so latencies are integer ns and every partial
    sum below 2^53 is exact in any order: bit-exact. The occupancy-weighted
    sums sum(occ * lat) are re-associated across shards: within 1e-12 relative
    (the north star allows 1e-9 for derived fp64 ratios).

compute(sub_batch) -> (CorrResult, Tables) is pluggable: Engine.run_host on a
GPU, the C oracle port in the CPU tests (tests/test_timeshard.py).
"""
from __future__ import annotations

import pickle
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as capi
from .columns import SpanBatch
from .engine import CorrResult, Tables

_NONE32 = np.uint32(0xFFFFFFFF)


def quiescent_cuts(b: SpanBatch) -> np.ndarray:
    """Rows of the (single) trace of `b` at which a shard may start (ascending)."""
    if b.n_traces != 1:
        raise ValueError("time-range sharding takes a batch holding one trace")
    n = b.n_spans
    f = b.flags
    lvl, kind = f & 3, (f >> 2) & 3
    if n < 2:
        return np.zeros(0, np.int64)
    if np.any(((f & capi.F_PARENT) != 0) & (lvl >= capi.LEVEL_KERNEL)):
        return np.zeros(0, np.int64)
    is_layer = (lvl == capi.LEVEL_LAYER)
    model_rows = np.nonzero((lvl == capi.LEVEL_MODEL) & (kind == capi.KIND_SYNC))[0]
    m0 = int(model_rows[0]) if model_rows.size else 0
    # (1) every layer span before c ends before c begins
    lend = np.where(is_layer, b.end_ns, np.uint64(0)).astype(np.uint64)
    pre_max_end = np.concatenate([[np.uint64(0)], np.maximum.accumulate(lend)[:-1]])
    ok = is_layer & (kind == capi.KIND_SYNC) & (pre_max_end < b.begin_ns)
    # (2) correlation ids before c all smaller than those at or after c
    has = (f & capi.F_CID) != 0
    c_hi = np.where(has, b.cid, np.uint64(0))
    c_lo = np.where(has, b.cid, np.uint64(np.iinfo(np.uint64).max))
    pre_max = np.concatenate([[np.uint64(0)], np.maximum.accumulate(c_hi)[:-1]])
    suf_min = np.minimum.accumulate(c_lo[::-1])[::-1]
    ok &= pre_max < suf_min
    ok[:m0 + 1] = False
    return np.nonzero(ok)[0].astype(np.int64)


def choose_cuts(cands: np.ndarray, n: int, world: int) -> List[int]:
    """Shard start rows [0, c_1, ..., c_k] (k < world when cuts are scarce)."""
    starts = [0]
    for r in range(1, world):
        nominal = r * n // world
        i = int(np.searchsorted(cands, nominal, side="left"))
        if i < cands.size and int(cands[i]) > starts[-1]:
            starts.append(int(cands[i]))
    return starts


def shard_rows(b: SpanBatch, lo: int, hi: int) -> np.ndarray:
    """Global rows of the shard [lo, hi): the model span first when it lies before lo."""
    lvl, kind = b.flags & 3, (b.flags >> 2) & 3
    models = np.nonzero((lvl == capi.LEVEL_MODEL) & (kind == capi.KIND_SYNC))[0]
    rows = np.arange(lo, hi, dtype=np.int64)
    if models.size and int(models[0]) < lo:
        rows = np.concatenate([[int(models[0])], rows])
    return rows


def sub_batch(b: SpanBatch, rows: np.ndarray) -> Tuple[SpanBatch, np.ndarray, np.ndarray]:
    """The shard as a standalone one-trace batch, with the global metric-table and
    layer-table rows of its side-table entries."""
    met = (b.flags & capi.F_METRICS) != 0
    lay = (b.flags & 3) == capi.LEVEL_LAYER
    mrow = np.cumsum(met) - met  # metric row of every span (valid where met)
    arow = np.cumsum(lay) - lay
    sel_m = mrow[rows[met[rows]]]
    sel_a = arow[rows[lay[rows]]]
    cols = {k: getattr(b, k)[rows] for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags",
                                              "name_id")}
    sub = SpanBatch(**cols, flops=b.flops[sel_m], dram_read=b.dram_read[sel_m], dram_write=b.dram_write[sel_m],
                    occupancy=b.occupancy[sel_m], alloc_bytes=b.alloc_bytes[sel_a], type_id=b.type_id[sel_a],
                    trace_span_off=np.array([0, rows.size], np.uint64), trace_id=b.trace_id[:1],
                    trace_levels=b.trace_levels[:1], trace_batch=b.trace_batch[:1], trace_run=b.trace_run[:1],
                    trace_serialized=b.trace_serialized[:1], names=b.names, types=b.types,
                    system_name=b.system_name, peak_flops=b.peak_flops, mem_bw=b.mem_bw)
    return sub, sel_m.astype(np.int64), sel_a.astype(np.int64)


# ---------------------------------------------------------------------------
# combine

_CAT = np.array([9, 0, 0, 0, 1, 1, 2, 3, 3, 4], np.int64)  # orphan reason -> emission phase
_T_PRIORITY = {capi.T_NO_MODEL: 0, capi.T_MULTI_MODEL: 1, capi.T_SKIP_LEVEL: 2, capi.T_DUP_EXEC_CID: 3,
               capi.T_DUP_LAUNCH_CID: 4}


def _roof(flops, rd, wr, lat, peak, bw):
    """roofline() of csrc/analyze.cu / analysis.cpp:41-71 in numpy float64."""
    flops, rd, wr, lat = (np.asarray(x) for x in (flops, rd, wr, lat))
    bytes_ = rd.astype(np.float64) + wr.astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        ai = np.where(bytes_ <= 0.0, np.nan, flops.astype(np.float64) / bytes_)
        tput = np.where(lat > 0.0, flops.astype(np.float64) / (lat / 1e9), np.nan)
    bound = np.where(bytes_ <= 0.0, -1, (ai < peak / bw).astype(np.int64)).astype(np.int8)
    return ai, tput, bound


def combine(b: SpanBatch, parts: Sequence[dict], top_k: int = 3) -> Tuple[CorrResult, Tables]:
    """The unsharded (CorrResult, Tables) of b's single trace from per-shard parts
    in timeline order; a part = {"rows", "mrows", "arows", "corr", "tabs"}."""
    cc, tc = {}, {}
    # ---- correlation
    L = K = 0
    lay, ker = {k: [] for k in ("layer_row", "layer_dur", "layer_attr_row", "layer_koff")}, \
        {k: [] for k in ("kernel_launch_row", "kernel_exec_row", "kernel_metric_row", "kernel_dur",
                         "kernel_name", "kernel_occ")}
    orph, amb, cand_rows, cand_cnt = [], [], [], []
    status = None
    for p in parts:
        c, rows, mrows, arows = p["corr"], p["rows"], p["mrows"], p["arows"]
        st = int(c.trace_status[0])
        if st != capi.T_OK:
            er = c.trace_err_row[:2].astype(np.int64)
            glob = [int(rows[x]) if x != 0xFFFFFFFF else 0xFFFFFFFF for x in er]
            if status is None or _T_PRIORITY[st] < _T_PRIORITY[status[0]]:
                status = (st, glob)
            continue
        nl, nk = int(c.n_layers), int(c.n_kernels)
        lay["layer_row"].append(rows[c.layer_row.astype(np.int64)])
        lay["layer_dur"].append(c.layer_dur)
        lay["layer_attr_row"].append(arows[c.layer_attr_row.astype(np.int64)])
        lay["layer_koff"].append(c.layer_kernel_off[:-1].astype(np.int64) + K)
        ker["kernel_launch_row"].append(rows[c.kernel_launch_row.astype(np.int64)])
        ker["kernel_exec_row"].append(rows[c.kernel_exec_row.astype(np.int64)])
        mr = c.kernel_metric_row.astype(np.int64)
        ker["kernel_metric_row"].append(np.where(mr == 0xFFFFFFFF, 0xFFFFFFFF, mrows[np.minimum(mr, max(mrows.size - 1, 0))]))
        for k in ("kernel_dur", "kernel_name", "kernel_occ"):
            ker[k].append(getattr(c, k))
        orow = rows[c.orphan_row.astype(np.int64)]
        orph.append((orow, c.orphan_reason))
        arow = rows[c.amb_row.astype(np.int64)]
        amb.append(arow)
        coff = c.amb_cand_off.astype(np.int64)
        for j in range(arow.size):
            cand_rows.append(rows[c.amb_cand_row[coff[j]:coff[j + 1]].astype(np.int64)])
        L += nl
        K += nk
    u32 = lambda x: np.asarray(x, dtype=np.int64).astype(np.uint32)
    cat = lambda parts_: np.concatenate(parts_) if parts_ else np.zeros(0)
    if status is not None:
        cc = {"trace_status": np.array([status[0]], np.int32), "trace_err_row": u32(status[1]),
              "trace_model_row": np.array([parts[0]["rows"][0]], np.uint32)}
        empty = CorrResult(1, 1, cc)
        return empty, None
    cc["trace_status"] = np.zeros(1, np.int32)
    cc["trace_err_row"] = np.full(2, _NONE32, np.uint32)
    cc["trace_model_row"] = u32([parts[0]["rows"][int(parts[0]["corr"].trace_model_row[0])]])
    cc["trace_layer_off"] = u32([0, L])
    cc["trace_kernel_off"] = u32([0, K])
    cc["layer_row"] = u32(cat(lay["layer_row"]))
    cc["layer_kernel_off"] = u32(np.concatenate(lay["layer_koff"] + [[K]]))
    cc["layer_dur"] = np.concatenate(lay["layer_dur"]).astype(np.uint64) if L else np.zeros(0, np.uint64)
    cc["layer_attr_row"] = u32(cat(lay["layer_attr_row"]))
    for k in ("kernel_launch_row", "kernel_exec_row", "kernel_metric_row", "kernel_name"):
        cc[k] = u32(cat(ker[k]))
    cc["kernel_dur"] = np.concatenate(ker["kernel_dur"]).astype(np.uint64) if K else np.zeros(0, np.uint64)
    cc["kernel_occ"] = np.concatenate(ker["kernel_occ"]).astype(np.float64) if K else np.zeros(0)
    # orphans: phase order, shard (= timeline / tree) order inside a phase, and
    # the leftover executions of phase 4 by span_id (correlator.cpp:355-363)
    o_rows = np.concatenate([o[0] for o in orph]) if orph else np.zeros(0, np.int64)
    o_reason = np.concatenate([o[1] for o in orph]).astype(np.uint8) if orph else np.zeros(0, np.uint8)
    o_cat = _CAT[o_reason.astype(np.int64)]
    key2 = np.where(o_cat == 4, b.span_id[o_rows.astype(np.int64)] if o_rows.size else 0, 0)
    order = np.lexsort((np.arange(o_rows.size), key2, o_cat))
    cc["orphan_row"] = u32(o_rows[order])
    cc["orphan_reason"] = o_reason[order]
    cc["trace_orphan_off"] = u32([0, o_rows.size])
    a_rows = np.concatenate(amb) if amb else np.zeros(0, np.int64)
    aorder = np.argsort(b.span_id[a_rows.astype(np.int64)], kind="stable") if a_rows.size else np.zeros(0, np.int64)
    cc["amb_row"] = u32(a_rows[aorder])
    cands = [cand_rows[i] for i in aorder]
    cc["amb_cand_off"] = u32(np.concatenate([[0], np.cumsum([x.size for x in cands])]) if cands else [0])
    cc["amb_cand_row"] = u32(np.concatenate(cands)) if cands else np.zeros(0, np.uint32)
    cc["trace_amb_off"] = u32([0, a_rows.size])
    corr = CorrResult(1, 0, cc, L, K, int(o_rows.size), int(a_rows.size), int(cc["amb_cand_row"].size))

    # ---- tables of the single group (one run)
    tabs_parts = [p["tabs"] for p in parts]
    if any(int(t.group_status[0]) != capi.G_OK for t in tabs_parts):
        first_bad = next(t for t in tabs_parts if int(t.group_status[0]) != capi.G_OK)
        return corr, first_bad
    kcols = ["k_name", "k_layer", "k_lat", "k_flops", "k_read", "k_write", "k_occ", "k_ai", "k_tput", "k_bound",
             "k_roofline_in"]
    lcols = ["l_index", "l_row", "l_layer_lat", "l_kern_lat", "l_flops", "l_read", "l_write", "l_occ", "l_count",
             "l_ai", "l_tput", "l_bound", "l_nongpu", "l_gpu_share", "l_nongpu_share", "l_flagged", "l_roofline_in"]
    lbase = kbase = 0
    acc = {k: [] for k in kcols + lcols + ["l_topk"]}
    for p, t in zip(parts, tabs_parts):
        nl, nk = int(t.n_layers), int(t.n_kernels)
        for k in kcols:
            v = t.cols[k]
            acc[k].append(v + np.uint32(lbase) if k == "k_layer" else v)
        for k in lcols:
            v = t.cols[k]
            if k == "l_index":
                v = v + np.uint32(lbase)
            elif k == "l_row":
                v = p["rows"][v.astype(np.int64)].astype(np.uint32)
            acc[k].append(v)
        tk = t.cols["l_topk"]
        acc["l_topk"].append(np.where(tk == _NONE32, _NONE32, tk + np.uint32(kbase)).astype(np.uint32))
        lbase += nl
        kbase += nk
    for k in acc:
        tc[k] = np.concatenate(acc[k]) if acc[k] else tabs_parts[0].cols[k][:0]
    t0 = tabs_parts[0]
    tc["group_status"] = np.zeros(1, np.int32)
    tc["group_err_arg"] = np.zeros(1, np.uint32)
    tc["group_layer_off"] = u32([0, lbase])
    tc["group_kernel_off"] = u32([0, kbase])
    peak, bw = b.peak_flops, b.mem_bw
    # a15 / model_roofline / a13 totals / a1: counters and latency sums across shards
    mlat = float(t0.m_lat[0])
    lat = 0.0
    occw = 0.0
    gpu = 0.0
    f = r = w = cnt = 0
    for t in tabs_parts:
        kl = float(t.m_kern_lat[0])
        lat += kl
        occw += float(t.m_occ[0]) * kl
        gpu += float(t.m_gpu[0])
        f += int(t.m_flops[0]); r += int(t.m_read[0]); w += int(t.m_write[0]); cnt += int(t.m_count[0])
    ai, tput, bound = _roof([f], [r], [w], [lat], peak, bw)
    tc.update({"m_lat": np.array([mlat]), "m_kern_lat": np.array([lat]),
               "m_flops": np.array([f], np.uint64), "m_read": np.array([r], np.uint64),
               "m_write": np.array([w], np.uint64), "m_occ": np.array([occw / lat if lat > 0.0 else 0.0]),
               "m_count": np.array([cnt], np.uint64), "m_ai": ai, "m_tput": tput, "m_bound": bound,
               "m_gpu": np.array([gpu]), "m_gpu_pct": np.array([gpu / mlat * 100.0]),
               "m_throughput": t0.m_throughput.copy(),
               "m_roofline_in": np.array([1 if (bound[0] >= 0 and lat > 0.0) else 0], np.uint8)})
    # a10 by name: per-name sums across shards, then total latency desc, name asc
    names: dict = {}
    for t in tabs_parts:
        for j in range(int(t.n_names)):
            nm = int(t.n_name[j])
            e = names.setdefault(nm, [0, 0.0, 0.0, 0, 0, 0])
            e[0] += int(t.n_count[j])
            e[1] += float(t.n_lat[j])
            e[2] += float(t.n_occ[j]) * float(t.n_lat[j])
            e[3] += int(t.n_flops[j]); e[4] += int(t.n_read[j]); e[5] += int(t.n_write[j])
    ids = np.array(sorted(names), np.uint32)
    nlat = np.array([names[i][1] for i in ids.tolist()])
    order = np.lexsort((ids, -nlat))
    ids, nlat = ids[order], nlat[order]
    get = lambda k, dt: np.array([names[i][k] for i in ids.tolist()], dt)
    nf, nr, nw = get(3, np.uint64), get(4, np.uint64), get(5, np.uint64)
    occs = get(2, np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        nocc = np.where(nlat > 0.0, occs / nlat, 0.0)
    ai, tput, bound = _roof(nf, nr, nw, nlat, peak, bw)
    tc.update({"n_name": ids, "n_count": get(0, np.uint64), "n_lat": nlat, "n_pct": nlat / mlat * 100.0,
               "n_flops": nf, "n_read": nr, "n_write": nw, "n_occ": nocc, "n_ai": ai, "n_tput": tput,
               "n_bound": bound})
    tc["group_name_off"] = u32([0, ids.size])
    # a5 / a6 / a7: per-type sums across shards (integer latencies of one run:
    # exact), then total latency desc, type asc
    if "y_type" in t0.cols:
        ytab: dict = {}
        for t in tabs_parts:
            for j in range(t.cols["y_type"].size):
                e = ytab.setdefault(int(t.cols["y_type"][j]), [0, 0.0, 0])
                e[0] += int(t.cols["y_count"][j])
                e[1] += float(t.cols["y_lat"][j])
                e[2] += int(t.cols["y_alloc"][j])
        yid = np.array(sorted(ytab), np.uint32)
        ylat = np.array([ytab[i][1] for i in yid.tolist()])
        yo = np.lexsort((yid, -ylat))
        yid, ylat = yid[yo], ylat[yo]
        tc["y_type"] = yid
        tc["y_count"] = np.array([ytab[i][0] for i in yid.tolist()], np.uint64)
        tc["y_lat"] = ylat
        tc["y_alloc"] = np.array([ytab[i][2] for i in yid.tolist()], np.int64)
        tc["group_type_off"] = u32([0, yid.size])
    for name, _, _ in capi.TABLE_FIELDS:  # dtype parity with the engine's columns
        if name in tc and name in t0.cols:
            tc[name] = tc[name].astype(t0.cols[name].dtype)
    return corr, Tables(1, tc, lbase, kbase, int(ids.size))


# ---------------------------------------------------------------------------
# ranks

def _allgather_bytes(payload: bytes, dist, device) -> List[bytes]:
    """all_gather of variable-size byte strings as uint8 tensors (NCCL on CUDA
    tensors, gloo on CPU tensors)."""
    import torch
    world = dist.get_world_size()
    n = torch.tensor([len(payload)], dtype=torch.int64, device=device)
    sizes = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(sizes, n)
    cap = int(max(int(s.item()) for s in sizes))
    buf = torch.zeros(cap, dtype=torch.uint8, device=device)
    if payload:
        buf[:len(payload)] = torch.frombuffer(bytearray(payload), dtype=torch.uint8).to(device)
    outs = [torch.empty(cap, dtype=torch.uint8, device=device) for _ in range(world)]
    dist.all_gather(outs, buf)
    return [bytes(o[:int(s.item())].cpu().numpy().tobytes()) for o, s in zip(outs, sizes)]


def run_time_sharded(b: SpanBatch, compute: Callable[[SpanBatch], Tuple[CorrResult, Tables]], rank: int,
                     world: int, dist=None, device="cpu", top_k: int = 3
                     ) -> Optional[Tuple[CorrResult, Optional[Tables], List[int]]]:
    """Correlate + analyse this rank's time range of b's single trace; rank 0 returns
    the combined unsharded result and the shard start rows (None on other ranks)."""
    starts = choose_cuts(quiescent_cuts(b), b.n_spans, world)
    bounds = starts + [b.n_spans]
    part = None
    if rank < len(starts):
        rows = shard_rows(b, bounds[rank], bounds[rank + 1])
        sub, mrows, arows = sub_batch(b, rows)
        corr, tabs = compute(sub)
        part = {"rows": rows, "mrows": mrows, "arows": arows, "corr": corr, "tabs": tabs}
    if world == 1:
        gathered = [part]
    else:
        blobs = _allgather_bytes(pickle.dumps(part, protocol=pickle.HIGHEST_PROTOCOL), dist, device)
        gathered = [pickle.loads(x) for x in blobs]
    if rank != 0:
        return None
    parts = [p for p in gathered if p is not None]
    corr, tabs = combine(b, parts, top_k)
    return corr, tabs, starts
