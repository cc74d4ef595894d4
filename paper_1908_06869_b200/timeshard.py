"""Time-range sharding of ONE long trace with a carried open-parent boundary
(BASELINE config 4).

A single 200M-span trace cannot be split by trace, so it is split by time:
rank r owns the timeline rows [lo_r, lo_{r+1}), lo_r = r*n/world moved forward
past a run of equal begin_ns (so no tie of the reference's kernel order
(begin, span_id) straddles a cut). Nothing has to be quiescent at a cut; what
crosses it is carried or routed:

  * the model span (TraceBundle::model_span, span.cpp:103-108: the first
    model/sync span) travels to every rank: layer placement (correlator.cpp:
    169-204) only needs it;
  * the open-parent boundary: the containment candidates of a child are the
    placed layers that begin at or before it and end at or after it
    (IntervalTree::containing, correlator.cpp:99-118, 228-231). Every child of
    rank r begins at or after begin(lo_r), so its candidates in earlier ranges
    are exactly the placed layers there that end at or after begin(lo_r): the
    carry. Each rank publishes its layer spans that end past the next cut
    (allgather), every later rank keeps the placed ones that reach its own cut;
    they enter its sub-batch as ordinary layer rows ahead of its range;
  * explicit parents (correlator.cpp:222-229): the parent_ids kernel-level rows
    name are requested from all ranks (allgather); answered placed layers
    outside the range join the sub-batch at their timeline position (a layer
    after the range can never be a containment candidate of the range);
  * the cid join (correlator.cpp:287-364): every correlation id c has ONE owner
    rank p(c). When the ranks' launch cid windows [min, max] are ordered and
    disjoint (cids grow with launch time, the normal case) p(c) is the rank
    whose window range holds c: own launches stay
    put and executions are routed to their launch's rank in one all-to-all.
    Otherwise p(c) = c mod world: launches send (cid, row, rank) to p(c), which
    detects cross-rank duplicate launch ids and forwards each execution to its
    launch's rank (or keeps it: no launch). Either way all executions of a cid
    meet on one rank, so duplicate-execution faults and leftovers are exact;
  * the global layer_index is an exclusive scan of the ranks' own placed-layer
    counts (layers are ordered by (begin, span_id) = timeline order).

Each rank correlates + analyses its sub-batch (own rows minus the executions
routed away, plus the carried / referenced layers, the model span and the
executions routed in) as one standalone trace on its GPU. `combine` rebuilds
the unsharded result on rank 0 from the per-rank tables:

  * layers: every rank's OWN placed layers in rank order; carried layers are
    dropped and their kernels re-attached to the owner's layer (the kernel
    table is stably regrouped by global layer index; within a layer the ranks'
    kernels follow in timeline order);
  * layers whose kernels sit on several ranks are recomputed from their final
    a8 rows in tree order (the reference's Accumulator chain, bit-exact), the
    others keep their owner's row; a5-a7 drop carried layers' contributions;
  * orphans per reference emission phase (layer pass, kernel pass, exec without
    cid by timeline row; launch fusion in tree order; leftover executions by
    span_id); ambiguities by span_id; faults by the reference's check order;
  * a10 / a15 totals: u64 counters and integer-ns latency sums add exactly;
    the occupancy-weighted ratios sum(occ*lat)/sum(lat) are re-associated
    across ranks (within 1e-12 relative; the north star allows 1e-9).

The per-rank tables travel to rank 0 as one byte tensor per rank (fixed column
order, no pickling) over torch.distributed: NCCL over NVLink on GPUs, gloo in
the CPU tests. compute(sub_batch) -> (CorrResult, Tables) is
pluggable: the CUDA engine on a GPU, the C oracle port in the CPU tests.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as capi
from .columns import SpanBatch
from .engine import CorrResult, Tables

_NONE32 = np.uint32(0xFFFFFFFF)
_U64MAX = np.uint64(0xFFFFFFFFFFFFFFFF)

# one span travelling between ranks: its columns plus global row / table rows
REC = np.dtype([("row", "<i8"), ("span_id", "<u8"), ("parent_id", "<u8"), ("begin_ns", "<u8"),
                ("end_ns", "<u8"), ("cid", "<u8"), ("flops", "<u8"), ("dram_read", "<u8"),
                ("dram_write", "<u8"), ("occupancy", "<f8"), ("mrow", "<i8"), ("alloc_bytes", "<i8"),
                ("arow", "<i8"), ("name_id", "<u4"), ("type_id", "<u4"), ("flags", "u1")])


# ---------------------------------------------------------------------------
# communicators: numpy arrays in, numpy arrays out

class ThreadWorld:
    """In-process world of `world` ranks run as threads (tests: worlds 2/3/7)."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots: list = [None] * world

    def comm(self, rank: int) -> "ThreadComm":
        return ThreadComm(self, rank)

    def run(self, fn: Callable[["ThreadComm"], object]) -> list:
        out, errs = [None] * self.world, []

        def main(r):
            try:
                out[r] = fn(self.comm(r))
            except BaseException as e:  # noqa: BLE001 - re-raised below
                errs.append(e)
                self.barrier.abort()

        th = [threading.Thread(target=main, args=(r,)) for r in range(self.world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        return out


class ThreadComm:
    def __init__(self, w: ThreadWorld, rank: int):
        self.w, self.rank, self.world = w, rank, w.world

    def allgather(self, a: np.ndarray) -> List[np.ndarray]:
        w = self.w
        w.slots[self.rank] = np.ascontiguousarray(a)
        w.barrier.wait()
        out = [x.copy() for x in w.slots]
        w.barrier.wait()
        return out

    def alltoallv(self, parts: Sequence[np.ndarray]) -> List[np.ndarray]:
        w = self.w
        w.slots[self.rank] = [np.ascontiguousarray(p) for p in parts]
        w.barrier.wait()
        out = [w.slots[s][self.rank].copy() for s in range(self.world)]
        w.barrier.wait()
        return out

    def gather_bytes(self, payload: np.ndarray) -> Optional[List[np.ndarray]]:
        got = self.allgather(payload)
        return got if self.rank == 0 else None


class TorchComm:
    """The same collectives over torch.distributed (NCCL on CUDA tensors, gloo on CPU)."""

    def __init__(self, dist, device="cpu"):
        self.dist, self.device = dist, device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def _t(self, a: np.ndarray):
        import torch
        u8 = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
        return torch.from_numpy(u8.copy()).to(self.device)

    def _sizes(self, n: int) -> List[int]:
        import torch
        t = torch.tensor([n], dtype=torch.int64, device=self.device)
        out = [torch.zeros(1, dtype=torch.int64, device=self.device) for _ in range(self.world)]
        self.dist.all_gather(out, t)
        return [int(x.item()) for x in out]

    def allgather(self, a: np.ndarray) -> List[np.ndarray]:
        import torch
        a = np.ascontiguousarray(a)
        sizes = self._sizes(a.nbytes)
        cap = max(max(sizes), 1)
        buf = torch.zeros(cap, dtype=torch.uint8, device=self.device)
        if a.nbytes:
            buf[:a.nbytes] = self._t(a)
        outs = [torch.empty(cap, dtype=torch.uint8, device=self.device) for _ in range(self.world)]
        self.dist.all_gather(outs, buf)
        return [o[:s].cpu().numpy().view(a.dtype) for o, s in zip(outs, sizes)]

    def alltoallv(self, parts: Sequence[np.ndarray]) -> List[np.ndarray]:
        """all_to_all of variable byte counts: one all_gather of the send sizes and
        one all_gather of every rank's packed send buffer (gloo has no all-to-all;
        the exchanged volume here is the routed executions, a small share of a
        trace)."""
        import torch
        dt = parts[0].dtype
        send = [np.ascontiguousarray(p) for p in parts]
        counts = np.array([p.nbytes for p in send], np.int64)
        allc = self.allgather(counts)
        packed = np.concatenate([p.view(np.uint8).reshape(-1) for p in send]) if counts.sum() else \
            np.zeros(0, np.uint8)
        blobs = self.allgather(packed)
        out = []
        for s in range(self.world):
            c = allc[s]
            off = int(c[:self.rank].sum())
            out.append(blobs[s][off:off + int(c[self.rank])].view(dt))
        del torch
        return out

    def gather_bytes(self, payload: np.ndarray) -> Optional[List[np.ndarray]]:
        got = self.allgather(payload)
        return got if self.rank == 0 else None


# ---------------------------------------------------------------------------
# planning

def shard_bounds(b: SpanBatch, world: int) -> List[int]:
    """Range starts lo_0 = 0 <= lo_1 <= ... (nominal r*n/world moved past equal begin_ns)."""
    n = b.n_spans
    los = [0]
    for r in range(1, world):
        c = max(r * n // world, los[-1])
        while 0 < c < n and b.begin_ns[c] == b.begin_ns[c - 1]:
            c += 1
        los.append(min(c, n))
    return los + [n]


def _roles(f: np.ndarray):
    lvl, kind = f & 3, (f >> 2) & 3
    layer = lvl == capi.LEVEL_LAYER
    launch = (kind == capi.KIND_LAUNCH) & (lvl >= capi.LEVEL_KERNEL)
    synck = (kind == capi.KIND_SYNC) & (lvl == capi.LEVEL_KERNEL)
    exe = kind == capi.KIND_EXEC
    model = (lvl == capi.LEVEL_MODEL) & (kind == capi.KIND_SYNC)
    return layer, launch, synck, exe, model


class _Local:
    """Rank r's rows [lo, hi) of b; nothing outside the range is read."""

    def __init__(self, b: SpanBatch, lo: int, hi: int):
        self.b, self.lo, self.hi = b, lo, hi
        self.f = b.flags[lo:hi]
        self.met = (self.f & capi.F_METRICS) != 0
        self.lay = (self.f & 3) == capi.LEVEL_LAYER
        self.mloc = np.cumsum(self.met) - self.met  # local metric row of each span
        self.aloc = np.cumsum(self.lay) - self.lay
        self.moff = self.aoff = 0

    def col(self, k):
        return getattr(self.b, k)[self.lo:self.hi]

    def records(self, idx: np.ndarray) -> np.ndarray:
        """REC records of local rows idx."""
        b, lo = self.b, self.lo
        idx = np.asarray(idx, np.int64)
        r = np.zeros(idx.size, REC)
        g = idx + lo
        r["row"] = g
        for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags", "name_id"):
            r[k] = getattr(b, k)[g]
        met, lay = self.met[idx], self.lay[idx]
        mr = np.where(met, self.moff + self.mloc[idx], -1)
        ar = np.where(lay, self.aoff + self.aloc[idx], -1)
        r["mrow"], r["arow"] = mr, ar
        if met.any():
            m = mr[met]
            for k in ("flops", "dram_read", "dram_write", "occupancy"):
                r[k][met] = getattr(b, k)[m]
        if lay.any():
            a = ar[lay]
            r["alloc_bytes"][lay] = b.alloc_bytes[a]
            r["type_id"][lay] = b.type_id[a]
        return r


@dataclass
class Shard:
    """One rank's sub-batch and the maps back to the global trace."""
    sub: SpanBatch
    rows: np.ndarray      # sub row -> global row
    mrows: np.ndarray     # sub metric row -> global metric row
    arows: np.ndarray     # sub layer-table row -> global layer-table row
    lo: int
    hi: int
    dup_launch: Tuple[int, int]  # cross-rank duplicate launch cid found by this rank's directory (rows) or (-1,-1)
    stats: Dict[str, int]


def _placed(rec_or_cols, model) -> np.ndarray:
    """Layer placement (correlator.cpp:169-204) of layer-level rows given the model span."""
    f = rec_or_cols["flags"]
    sync = ((f >> 2) & 3) == capi.KIND_SYNC
    if model is None:
        return np.zeros(f.size, bool)
    haspar = (f & capi.F_PARENT) != 0
    inside = (rec_or_cols["begin_ns"] >= model["begin_ns"]) & (rec_or_cols["end_ns"] <= model["end_ns"])
    return sync & np.where(haspar, rec_or_cols["parent_id"] == model["span_id"], inside)


def prepare(b: SpanBatch, lo: int, hi: int, comm) -> Shard:
    """Build rank comm.rank's sub-batch for its range [lo, hi) of b's single trace
    (the carry, the explicit-parent layers, the routed executions)."""
    if b.n_traces != 1:
        raise ValueError("time-range sharding takes a batch holding one trace")
    rank, world = comm.rank, comm.world
    L = _Local(b, lo, hi)
    f = L.f
    layer, launch, synck, exe, model_m = _roles(f)
    has_c = (f & capi.F_CID) != 0
    begin, end, cid = L.col("begin_ns"), L.col("end_ns"), L.col("cid")
    lc = cid[launch & has_c]
    mono = bool(lc.size < 2 or np.all(lc[1:] > lc[:-1]))
    mrow_local = int(np.argmax(model_m)) if model_m.any() else -1
    # ---- exchange 1: counts, first model row, launch cid window, range begin
    summ = np.array([int(L.met.sum()), int(L.lay.sum()), mrow_local if mrow_local >= 0 else 2 ** 64 - 1,
                     int(lc.min()) if lc.size else 0, int(lc.max()) if lc.size else 0, int(mono), int(lc.size),
                     hi - lo, int(begin[0]) if hi > lo else 0], np.uint64)
    S = np.stack(comm.allgather(summ))
    nmet, nlay = S[:, 0].astype(np.int64), S[:, 1].astype(np.int64)
    L.moff, L.aoff = int(nmet[:rank].sum()), int(nlay[:rank].sum())
    has_model = S[:, 2] != _U64MAX
    mrank = int(np.argmax(has_model)) if has_model.any() else -1
    nonempty = S[:, 7] > 0
    # begin of the first row of every later range (the cut instants)
    next_begin = None
    for q in range(rank + 1, world):
        if nonempty[q]:
            next_begin = S[q, 8]
            break
    # ---- exchange 2: the model span + this range's layers that end past the next cut
    esc = np.zeros(0, np.int64)
    if next_begin is not None:
        esc = np.nonzero(layer & (end >= next_begin))[0]
    mine = L.records(esc)
    if mrank == rank:
        mine = np.concatenate([L.records([mrow_local]), mine])
    got = comm.allgather(mine)
    model = None
    if mrank >= 0:
        model = got[mrank][0]
    carried = []
    if hi > lo:
        for q in range(rank):
            g = got[q]
            if model is not None and q == mrank:
                g = g[1:]
            g = g[(g["end_ns"] >= begin[0]) & ((g["flags"] & 3) == capi.LEVEL_LAYER)]
            g = g[_placed(g, model)]
            carried.append(g)
    carried = np.concatenate(carried) if carried else np.zeros(0, REC)
    # ---- exchange 3/4: explicit parents of kernel-level rows that name a layer outside the range
    kpar = (launch | synck) & ((f & capi.F_PARENT) != 0)
    req = np.unique(L.col("parent_id")[kpar]).astype(np.uint64)
    reqs = comm.allgather(req)
    others = [reqs[q] for q in range(world) if q != rank and reqs[q].size]
    ans = np.zeros(0, REC)
    if others and model is not None:
        want = np.unique(np.concatenate(others))
        lay_idx = np.nonzero(layer)[0]
        hit = lay_idx[np.isin(L.col("span_id")[lay_idx], want)]
        if hit.size:
            ans = L.records(hit)
            ans = ans[_placed(ans, model)]
    answers = comm.allgather(ans)
    referenced = []
    if req.size:
        for q in range(world):
            if q != rank and answers[q].size:
                a = answers[q]
                referenced.append(a[np.isin(a["span_id"], req)])
    referenced = np.concatenate(referenced) if referenced else np.zeros(0, REC)
    # ---- cid ownership and execution routing
    win = [(int(S[q, 3]), int(S[q, 4])) for q in range(world) if S[q, 6] > 0]
    wranks = [q for q in range(world) if S[q, 6] > 0]
    window_mode = bool(wranks) and all(win[i][1] < win[i + 1][0] for i in range(len(win) - 1))
    ex_idx = np.nonzero(exe & has_c)[0]
    ex_cid = cid[ex_idx]
    dup_launch = (-1, -1)
    stats = {"routed_out": 0, "routed_in": 0, "carried": int(carried.size), "referenced": int(referenced.size),
             "window_mode": int(window_mode)}
    if window_mode:
        lows = np.array([w[0] for w in win], np.uint64)
        pos = np.searchsorted(lows, ex_cid, side="right") - 1
        dest = np.array(wranks, np.int64)[np.maximum(pos, 0)]
        send_idx = [ex_idx[dest == q] if q != rank else np.zeros(0, np.int64) for q in range(world)]
        got_ex = comm.alltoallv([L.records(s) for s in send_idx])
        moved = np.concatenate(send_idx) if send_idx else np.zeros(0, np.int64)
        routed_in = np.concatenate([g for q, g in enumerate(got_ex) if q != rank])
    else:
        # directory: launch (cid, row, rank) -> p(c) = cid mod world
        li = np.nonzero(launch & has_c)[0]
        DIR = np.dtype([("cid", "<u8"), ("row", "<i8"), ("rank", "<i8")])
        d = np.zeros(li.size, DIR)
        d["cid"], d["row"], d["rank"] = cid[li], li + lo, rank
        pl = (cid[li] % np.uint64(world)).astype(np.int64)
        dirs = comm.alltoallv([d[pl == q] for q in range(world)])
        D = np.concatenate(dirs)
        D = D[np.lexsort((D["row"], D["cid"]))]
        if D.size > 1:
            same = D["cid"][1:] == D["cid"][:-1]
            if same.any():
                j = np.nonzero(same)[0]  # D[j+1] repeats D[j]'s cid: second occurrence and later
                first_of = np.searchsorted(D["cid"], D["cid"][j + 1], side="left")
                k = int(np.argmin(D["row"][j + 1]))
                dup_launch = (int(D["row"][first_of[k]]), int(D["row"][j + 1][k]))
        # hop 1: executions to p(c)
        pe = (ex_cid % np.uint64(world)).astype(np.int64)
        send1 = [ex_idx[pe == q] for q in range(world)]
        hop1 = np.concatenate(comm.alltoallv([L.records(s) for s in send1]))
        # hop 2: from p(c) to the launch's rank (no launch: stay at p(c))
        if D.size:
            first = np.ones(D.size, bool)
            first[1:] = D["cid"][1:] != D["cid"][:-1]
            Du = D[first]
            k = np.searchsorted(Du["cid"], hop1["cid"])
            k = np.minimum(k, Du.size - 1)
            found = Du["cid"][k] == hop1["cid"]
            dest = np.where(found, Du["rank"][k], rank)
        else:
            dest = np.full(hop1.size, rank, np.int64)
        hop2 = comm.alltoallv([hop1[dest == q] for q in range(world)])
        got_all = np.concatenate(hop2)
        moved = ex_idx  # every own execution with a cid went through p(c)
        own_back = got_all[(got_all["row"] >= lo) & (got_all["row"] < hi)]
        routed_in = got_all[(got_all["row"] < lo) | (got_all["row"] >= hi)]
        moved = np.setdiff1d(moved, own_back["row"].astype(np.int64) - lo, assume_unique=True)
    stats["routed_out"], stats["routed_in"] = int(moved.size), int(routed_in.size)
    # ---- assemble: records before the range, own rows kept, records after the range
    keep = np.ones(hi - lo, bool)
    keep[moved] = False
    ext = [carried, referenced, routed_in]
    if model is not None and not (lo <= int(model["row"]) < hi):
        ext.append(model[None])
    ext = np.concatenate(ext) if any(x.size for x in ext) else np.zeros(0, REC)
    if ext.size:
        ext = ext[np.argsort(ext["row"], kind="stable")]
        ext = ext[np.concatenate([[True], ext["row"][1:] != ext["row"][:-1]])]
    before, after = ext[ext["row"] < lo], ext[ext["row"] >= hi]
    own = np.nonzero(keep)[0]
    rows = np.concatenate([before["row"], own + lo, after["row"]]).astype(np.int64)
    cols = {}
    for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags", "name_id"):
        cols[k] = np.concatenate([before[k], L.col(k)[own], after[k]]).astype(getattr(b, k).dtype)
    om = own[L.met[own]]
    oa = own[L.lay[own]]
    bm, am = before[before["mrow"] >= 0], after[after["mrow"] >= 0]
    ba, aa = before[before["arow"] >= 0], after[after["arow"] >= 0]
    mrows = np.concatenate([bm["mrow"], L.moff + L.mloc[om], am["mrow"]]).astype(np.int64)
    arows = np.concatenate([ba["arow"], L.aoff + L.aloc[oa], aa["arow"]]).astype(np.int64)
    m_lo = L.moff
    for k in ("flops", "dram_read", "dram_write", "occupancy"):
        own_v = getattr(b, k)[m_lo + L.mloc[om]] if om.size else getattr(b, k)[:0]
        cols[k] = np.concatenate([bm[k], own_v, am[k]]).astype(getattr(b, k).dtype)
    for k in ("alloc_bytes", "type_id"):
        own_v = getattr(b, k)[L.aoff + L.aloc[oa]] if oa.size else getattr(b, k)[:0]
        cols[k] = np.concatenate([ba[k], own_v, aa[k]]).astype(getattr(b, k).dtype)
    sub = SpanBatch(**cols, trace_span_off=np.array([0, rows.size], np.uint64), trace_id=b.trace_id[:1],
                    trace_levels=b.trace_levels[:1], trace_batch=b.trace_batch[:1], trace_run=b.trace_run[:1],
                    trace_serialized=b.trace_serialized[:1], names=b.names, types=b.types,
                    system_name=b.system_name, peak_flops=b.peak_flops, mem_bw=b.mem_bw)
    return Shard(sub, rows, mrows, arows, lo, hi, dup_launch, stats)


# ---------------------------------------------------------------------------
# combine

_CAT = np.array([9, 0, 0, 0, 1, 1, 2, 3, 3, 4], np.int64)  # orphan reason -> emission phase


def _roof(flops, rd, wr, lat, peak, bw):
    """roofline() of csrc/analyze.cu / analysis.cpp:41-71 in numpy float64."""
    flops, rd, wr, lat = (np.asarray(x) for x in (flops, rd, wr, lat))
    bytes_ = rd.astype(np.float64) + wr.astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        ai = np.where(bytes_ <= 0.0, np.nan, flops.astype(np.float64) / bytes_)
        tput = np.where(lat > 0.0, flops.astype(np.float64) / (lat / 1e9), np.nan)
    bound = np.where(bytes_ <= 0.0, -1, (ai < peak / bw).astype(np.int64)).astype(np.int8)
    return ai, tput, bound


def _fault(b: SpanBatch, parts: Sequence[dict]) -> Optional[Tuple[int, Tuple[int, int]]]:
    """The fault the reference throws first (correlator.cpp:141-160, 287-316):
    no model; the earliest multi-model / skip-level span; the earliest second
    execution of a cid; the earliest second launch of a cid."""
    NONE = 0xFFFFFFFF
    pre, dex, dla = [], [], []
    for p in parts:
        c, rows = p["corr"], p["rows"]
        st = int(c.trace_status[0])
        er = [int(rows[x]) if x != NONE else NONE for x in c.trace_err_row[:2].astype(np.int64)]
        if st == capi.T_NO_MODEL:
            return st, (NONE, NONE)
        if st in (capi.T_MULTI_MODEL, capi.T_SKIP_LEVEL):
            pre.append((er[0], st, tuple(er)))
        elif st == capi.T_DUP_EXEC_CID:
            dex.append((er[1], st, tuple(er)))
        elif st == capi.T_DUP_LAUNCH_CID:
            dla.append((er[1], st, tuple(er)))
        dl = p.get("dup_launch", (-1, -1))
        if dl[0] >= 0:
            dla.append((dl[1], capi.T_DUP_LAUNCH_CID, dl))
    for lst in (pre, dex, dla):
        if lst:
            _, st, er = min(lst)
            return st, er
    return None


def combine(b: SpanBatch, parts: Sequence[dict], top_k: int = 3, noise: float = 0.01
            ) -> Tuple[CorrResult, Optional[Tables]]:
    """The unsharded (CorrResult, Tables) of b's single trace from per-rank parts in
    rank order; a part = {"rows", "mrows", "arows", "lo", "hi", "corr", "tabs",
    "dup_launch", "fusion_parents" (global layer rows of its launch-fusion
    orphans, fusion_orphan_parents)}."""
    u32 = lambda x: np.asarray(x, dtype=np.int64).astype(np.uint32)
    flt = _fault(b, parts)
    if flt is not None:
        st, er = flt
        cc = {"trace_status": np.array([st], np.int32), "trace_err_row": u32(er),
              "trace_model_row": np.array([0], np.uint32)}
        return CorrResult(1, 1, cc), None
    # ---- global layer list: every part's own placed layers, in part order
    own_rows, part_layer_g = [], []
    for p in parts:
        c = p["corr"]
        lr = p["rows"][c.layer_row.astype(np.int64)]
        p["_lrows"] = lr
        p["_own"] = (lr >= p["lo"]) & (lr < p["hi"])
        own_rows.append(lr[p["_own"]])
    g_rows = np.concatenate(own_rows) if own_rows else np.zeros(0, np.int64)
    NL = int(g_rows.size)
    for p in parts:
        g = np.searchsorted(g_rows, p["_lrows"])
        assert np.all(g_rows[np.minimum(g, max(NL - 1, 0))] == p["_lrows"]) if p["_lrows"].size else True
        p["_lg"] = g
    # ---- kernels: regroup by global layer (stable: parts in order, tree order inside)
    kg, kp, kl = [], [], []
    for pi, p in enumerate(parts):
        c = p["corr"]
        koff = c.layer_kernel_off.astype(np.int64)
        cnt = np.diff(koff)
        kg.append(np.repeat(p["_lg"], cnt))
        kp.append(np.full(int(koff[-1]) if koff.size else 0, pi, np.int64))
        kl.append(np.arange(int(koff[-1]) if koff.size else 0, dtype=np.int64))
    KG = np.concatenate(kg) if kg else np.zeros(0, np.int64)
    KP, KLOC = np.concatenate(kp), np.concatenate(kl)
    perm = np.argsort(KG, kind="stable")
    NK = int(KG.size)
    final_pos = np.empty(NK, np.int64)
    final_pos[perm] = np.arange(NK)
    part_base = np.concatenate([[0], np.cumsum([int(p["corr"].n_kernels) for p in parts])])

    def gather_k(get, dtype):
        v = np.concatenate([get(p) for p in parts]) if parts else np.zeros(0, dtype)
        return v[perm].astype(dtype)

    cc = {}
    cc["trace_status"] = np.zeros(1, np.int32)
    cc["trace_err_row"] = np.full(2, _NONE32, np.uint32)
    mp = next(p for p in parts if p["lo"] <= int(p["rows"][int(p["corr"].trace_model_row[0])]) < p["hi"]) \
        if any(int(p["corr"].trace_model_row[0]) != 0xFFFFFFFF for p in parts) else parts[0]
    cc["trace_model_row"] = u32([mp["rows"][int(mp["corr"].trace_model_row[0])]])
    cc["trace_layer_off"] = u32([0, NL])
    cc["trace_kernel_off"] = u32([0, NK])
    cc["layer_row"] = u32(g_rows)
    cc["layer_kernel_off"] = u32(np.concatenate([[0], np.cumsum(np.bincount(KG, minlength=NL))]) if NL else [0])
    cc["layer_dur"] = np.concatenate([p["corr"].layer_dur[p["_own"]] for p in parts]).astype(np.uint64)
    cc["layer_attr_row"] = u32(np.concatenate([p["arows"][p["corr"].layer_attr_row.astype(np.int64)][p["_own"]]
                                               for p in parts]))
    rowmap = lambda p, x: np.where(x == _NONE32, 0xFFFFFFFF, p["rows"][np.minimum(x.astype(np.int64),
                                                                                    max(p["rows"].size - 1, 0))])
    mmap = lambda p, x: np.where(x == _NONE32, 0xFFFFFFFF, p["mrows"][np.minimum(x.astype(np.int64),
                                                                                   max(p["mrows"].size - 1, 0))])
    cc["kernel_launch_row"] = u32(gather_k(lambda p: rowmap(p, p["corr"].kernel_launch_row), np.int64))
    cc["kernel_exec_row"] = u32(gather_k(lambda p: rowmap(p, p["corr"].kernel_exec_row), np.int64))
    cc["kernel_metric_row"] = u32(gather_k(lambda p: mmap(p, p["corr"].kernel_metric_row), np.int64))
    cc["kernel_dur"] = gather_k(lambda p: p["corr"].kernel_dur, np.uint64)
    cc["kernel_name"] = gather_k(lambda p: p["corr"].kernel_name, np.uint32)
    cc["kernel_occ"] = gather_k(lambda p: p["corr"].kernel_occ, np.float64)
    # ---- orphans: phase, then (timeline row | tree position | span_id)
    o_rows, o_reason, o_key = [], [], []
    for pi, p in enumerate(parts):
        c = p["corr"]
        r = p["rows"][c.orphan_row.astype(np.int64)]
        rs = c.orphan_reason.astype(np.int64)
        cat = _CAT[rs]
        key = np.zeros((r.size, 3), np.int64)
        key[:, 0] = cat
        key[:, 1] = r
        f3 = np.nonzero(cat == 3)[0]
        if f3.size:  # launch fusion: tree order = (global layer, part, position)
            par = p["fusion_parents"]
            key[f3, 1] = np.searchsorted(g_rows, par)
            key[f3, 2] = pi * (1 << 40) + f3
        o_rows.append(r), o_reason.append(rs), o_key.append(key)
    R = np.concatenate(o_rows) if o_rows else np.zeros(0, np.int64)
    RS = np.concatenate(o_reason) if o_reason else np.zeros(0, np.int64)
    KY = np.concatenate(o_key) if o_key else np.zeros((0, 3), np.int64)
    if RS.size:
        KY[KY[:, 0] == 4, 1:] = 0
        order = np.lexsort((KY[:, 2], KY[:, 1], KY[:, 0]))
        # leftover executions (phase 4) sort by the unsigned span_id
        o4 = np.nonzero(KY[order, 0] == 4)[0]
        if o4.size:
            idx4 = order[o4]
            order[o4] = idx4[np.argsort(b.span_id[R[idx4]], kind="stable")]
    else:
        order = np.zeros(0, np.int64)
    cc["orphan_row"] = u32(R[order])
    cc["orphan_reason"] = RS[order].astype(np.uint8)
    cc["trace_orphan_off"] = u32([0, R.size])
    # ---- ambiguities by span_id
    a_rows, a_cands = [], []
    for p in parts:
        c = p["corr"]
        a_rows.append(p["rows"][c.amb_row.astype(np.int64)])
        off = c.amb_cand_off.astype(np.int64)
        cr = p["rows"][c.amb_cand_row.astype(np.int64)]
        a_cands.extend(cr[off[j]:off[j + 1]] for j in range(c.amb_row.size))
    A = np.concatenate(a_rows) if a_rows else np.zeros(0, np.int64)
    ao = np.argsort(b.span_id[A], kind="stable") if A.size else np.zeros(0, np.int64)
    cands = [a_cands[i] for i in ao]
    cc["amb_row"] = u32(A[ao])
    cc["amb_cand_off"] = u32(np.concatenate([[0], np.cumsum([x.size for x in cands])]) if cands else [0])
    cc["amb_cand_row"] = u32(np.concatenate(cands)) if cands else np.zeros(0, np.uint32)
    cc["trace_amb_off"] = u32([0, A.size])
    corr = CorrResult(1, 0, cc, NL, NK, int(R.size), int(A.size), int(cc["amb_cand_row"].size))

    # ---- tables of the single group (one run)
    tabs_parts = [p["tabs"] for p in parts]
    if any(t is None for t in tabs_parts):
        return corr, None
    bad = [t for t in tabs_parts if int(t.group_status[0]) != capi.G_OK]
    if bad:
        return corr, bad[0]
    t0 = tabs_parts[0]
    K = top_k
    tc = {}
    kcols = ["k_name", "k_lat", "k_flops", "k_read", "k_write", "k_occ", "k_ai", "k_tput", "k_bound",
             "k_roofline_in"]
    for k in kcols:
        tc[k] = gather_k(lambda p, k=k: p["tabs"].cols[k], t0.cols[k].dtype)
    tc["k_layer"] = KG[perm].astype(np.uint32)
    # layers with kernels on more than one part are recomputed from their final a8 rows
    owner_part = np.zeros(NL, np.int64)
    lcols = ["l_layer_lat", "l_kern_lat", "l_flops", "l_read", "l_write", "l_occ", "l_count", "l_ai", "l_tput",
             "l_bound", "l_nongpu", "l_gpu_share", "l_nongpu_share", "l_flagged", "l_roofline_in"]
    acc = {k: [] for k in lcols}
    topk_parts = []
    for pi, p in enumerate(parts):
        t, own = p["tabs"], p["_own"]
        owner_part[p["_lg"][own]] = pi
        for k in lcols:
            acc[k].append(t.cols[k][own])
        tk = t.cols["l_topk"].reshape(-1, K)[own].astype(np.int64)
        glob = np.where(tk == 0xFFFFFFFF, -1, final_pos[np.minimum(part_base[pi] + tk, max(NK - 1, 0))])
        topk_parts.append(glob)
    for k in lcols:
        tc[k] = np.concatenate(acc[k]).astype(t0.cols[k].dtype)
    topk = np.concatenate(topk_parts) if topk_parts else np.zeros((0, K), np.int64)
    split = np.zeros(NL, bool)
    if NK:
        split[KG[KP != owner_part[KG]]] = True
    koff = cc["layer_kernel_off"].astype(np.int64)
    peak, bw = b.peak_flops, b.mem_bw
    for li in np.nonzero(split)[0].tolist():
        k0, k1 = int(koff[li]), int(koff[li + 1])
        lat = 0.0
        occw = 0.0
        fl = rd = wr = 0
        for j in range(k0, k1):  # the Accumulator in tree order (analysis.cpp:172-192)
            kl = float(tc["k_lat"][j])
            lat += kl
            fl += int(tc["k_flops"][j]); rd += int(tc["k_read"][j]); wr += int(tc["k_write"][j])
            occw += float(tc["k_occ"][j]) * kl
        ll = float(tc["l_layer_lat"][li])
        ai, tput, bound = _roof([fl], [rd], [wr], [lat], peak, bw)
        non = ll - lat
        upd = {"l_kern_lat": lat, "l_flops": fl, "l_read": rd, "l_write": wr,
               "l_occ": occw / lat if lat > 0.0 else 0.0, "l_count": k1 - k0, "l_ai": ai[0], "l_tput": tput[0],
               "l_bound": bound[0], "l_nongpu": non, "l_gpu_share": lat / ll if ll > 0.0 else 0.0,
               "l_nongpu_share": non / ll if ll > 0.0 else 0.0, "l_flagged": 1 if non < -(noise * ll) else 0,
               "l_roofline_in": 1 if (bound[0] >= 0 and lat > 0.0) else 0}
        for k, v in upd.items():
            tc[k][li] = v
        kk = np.arange(k0, k1)
        best = sorted(kk.tolist(), key=lambda j: (-float(tc["k_lat"][j]), j))[:K]
        topk[li] = -1
        topk[li, :len(best)] = best
    tc["l_topk"] = np.where(topk < 0, 0xFFFFFFFF, topk).astype(np.uint32).reshape(-1)
    tc["l_index"] = np.arange(NL, dtype=np.uint32)
    tc["l_row"] = u32(g_rows)
    tc["group_status"] = np.zeros(1, np.int32)
    tc["group_err_arg"] = np.zeros(1, np.uint32)
    tc["group_layer_off"] = u32([0, NL])
    tc["group_kernel_off"] = u32([0, NK])
    # ---- a15 / model_roofline / a13 totals: counters and latency sums across parts
    mlat = float(t0.m_lat[0])
    lat = occw = gpu = 0.0
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
    # ---- a10 by name: per-name sums across parts, then total latency desc, name asc
    nm = np.concatenate([t.n_name for t in tabs_parts]).astype(np.int64)
    if nm.size:
        uid, inv = np.unique(nm, return_inverse=True)
        cat = lambda k: np.concatenate([t.cols[k] for t in tabs_parts])
        nlat_all = cat("n_lat").astype(np.float64)
        s_cnt = np.zeros(uid.size, np.uint64)
        np.add.at(s_cnt, inv, cat("n_count").astype(np.uint64))
        s_lat = np.zeros(uid.size)
        np.add.at(s_lat, inv, nlat_all)
        s_occ = np.zeros(uid.size)
        np.add.at(s_occ, inv, cat("n_occ").astype(np.float64) * nlat_all)
        sums = {}
        for k in ("n_flops", "n_read", "n_write"):
            v = np.zeros(uid.size, np.uint64)
            np.add.at(v, inv, cat(k).astype(np.uint64))
            sums[k] = v
        order = np.lexsort((uid, -s_lat))
        ids, nlat = uid[order].astype(np.uint32), s_lat[order]
        with np.errstate(divide="ignore", invalid="ignore"):
            nocc = np.where(nlat > 0.0, s_occ[order] / nlat, 0.0)
        nf, nr, nw = (sums[k][order] for k in ("n_flops", "n_read", "n_write"))
        ai, tput, bound = _roof(nf, nr, nw, nlat, peak, bw)
        tc.update({"n_name": ids, "n_count": s_cnt[order], "n_lat": nlat, "n_pct": nlat / mlat * 100.0,
                   "n_flops": nf, "n_read": nr, "n_write": nw, "n_occ": nocc, "n_ai": ai, "n_tput": tput,
                   "n_bound": bound})
    else:
        for k in ("n_name", "n_count", "n_lat", "n_pct", "n_flops", "n_read", "n_write", "n_occ", "n_ai",
                  "n_tput", "n_bound"):
            tc[k] = t0.cols[k][:0]
    tc["group_name_off"] = u32([0, tc["n_name"].size])
    # ---- a5 / a6 / a7: per-type sums over OWN layers (carried layers subtracted)
    if "y_type" in t0.cols:
        ytab: dict = {}
        for p, t in zip(parts, tabs_parts):
            for j in range(t.cols["y_type"].size):
                e = ytab.setdefault(int(t.cols["y_type"][j]), [0, 0.0, 0])
                e[0] += int(t.cols["y_count"][j])
                e[1] += float(t.cols["y_lat"][j])
                e[2] += int(t.cols["y_alloc"][j])
            # carried / referenced layers count on their owner only
            for j in np.nonzero(~p["_own"])[0].tolist():
                ar = int(p["arows"][int(p["corr"].layer_attr_row[j])])
                e = ytab[int(b.type_id[ar])]
                e[0] -= 1
                e[1] -= float(t.cols["l_layer_lat"][j])
                e[2] -= int(b.alloc_bytes[ar])
        ytab = {k: v for k, v in ytab.items() if v[0] > 0}
        yid = np.array(sorted(ytab), np.uint32)
        ylat = np.array([ytab[i][1] for i in yid.tolist()])
        yo = np.lexsort((yid, -ylat)) if yid.size else np.zeros(0, np.int64)
        yid, ylat = yid[yo], ylat[yo]
        tc["y_type"] = yid
        tc["y_count"] = np.array([ytab[i][0] for i in yid.tolist()], np.uint64)
        tc["y_lat"] = ylat
        tc["y_alloc"] = np.array([ytab[i][2] for i in yid.tolist()], np.int64)
        tc["group_type_off"] = u32([0, yid.size])
    for name, _, _ in capi.TABLE_FIELDS:  # dtype parity with the engine's columns
        if name in tc and name in t0.cols:
            tc[name] = tc[name].astype(t0.cols[name].dtype)
    return corr, Tables(1, tc, NL, NK, int(tc["n_name"].size))


def fusion_orphan_parents(shard: Shard, corr: CorrResult) -> np.ndarray:
    """Global row of the parent layer of each launch-fusion orphan (reasons 7/8) of a
    shard: the launch sat in the tree before fusion dropped it (correlator.cpp:
    320-345), under its explicit parent or under its single containing placed
    layer — the first placed layer of the sub-batch (timeline order) whose
    running max end reaches the launch's end among those beginning at or before it."""
    cat = _CAT[corr.orphan_reason.astype(np.int64)]
    f3 = np.nonzero(cat == 3)[0]
    if not f3.size:
        return np.zeros(0, np.int64)
    sub = shard.sub
    lr = corr.layer_row.astype(np.int64)  # placed layers of the sub-batch (sub rows, timeline order)
    lb, le = sub.begin_ns[lr], sub.end_ns[lr]
    pmax = np.maximum.accumulate(le) if le.size else le
    by_sid = {int(s): i for i, s in enumerate(sub.span_id[lr].tolist())}
    out = np.empty(f3.size, np.int64)
    for j, o in enumerate(f3.tolist()):
        row = int(corr.orphan_row[o])
        if int(sub.flags[row]) & capi.F_PARENT:
            li = by_sid[int(sub.parent_id[row])]
        else:
            last = int(np.searchsorted(lb, sub.begin_ns[row], side="right"))  # layers beginning at/before
            li = int(np.searchsorted(pmax[:last], sub.end_ns[row], side="left"))
        out[j] = shard.rows[lr[li]]
    return out


# ---------------------------------------------------------------------------
# table transport (one byte tensor per rank, fixed column order)

_SCALARS = ("n_layers", "n_kernels", "n_orphans", "n_ambiguities", "n_candidates")


def pack_part(shard: Shard, corr: CorrResult, tabs: Optional[Tables], fusion_parents: np.ndarray) -> np.ndarray:
    """One rank's result as a flat uint8 buffer: a header of column byte sizes,
    then the columns (correlation, maps, tables) in a fixed order."""
    cols: List[np.ndarray] = [np.array([shard.lo, shard.hi, shard.dup_launch[0], shard.dup_launch[1],
                                        1 if tabs is not None else 0], np.int64)]
    cols += [np.array([getattr(corr, k) for k in _SCALARS], np.int64)]
    for name, _, _ in capi.CORR_FIELDS:
        cols.append(np.asarray(corr.cols.get(name, np.zeros(0, np.uint8))))
    cols += [shard.rows, shard.mrows, shard.arows, np.asarray(fusion_parents, np.int64)]
    if tabs is not None:
        cols.append(np.array([tabs.n_layers, tabs.n_kernels, tabs.n_names], np.int64))
        for name, _, _ in capi.TABLE_FIELDS:
            cols.append(np.asarray(tabs.cols.get(name, np.zeros(0, np.uint8))))
    sizes = np.array([c.nbytes for c in cols], np.int64)
    head = np.concatenate([[sizes.size], sizes]).astype(np.int64)
    return np.concatenate([head.view(np.uint8)] + [np.ascontiguousarray(c).view(np.uint8).reshape(-1)
                                                   for c in cols])


def unpack_part(buf: np.ndarray, proto_corr_dtypes: Dict[str, np.dtype], proto_tab_dtypes: Dict[str, np.dtype]
                ) -> dict:
    """Inverse of pack_part (dtypes from capi field declarations)."""
    n = int(buf[:8].view(np.int64)[0])
    sizes = buf[8:8 + 8 * n].view(np.int64)
    off = 8 + 8 * n
    chunks = []
    for s in sizes.tolist():
        chunks.append(buf[off:off + s])
        off += s
    it = iter(chunks)
    meta = next(it).view(np.int64)
    sc = next(it).view(np.int64)
    cc = {name: next(it).view(proto_corr_dtypes[name]) for name, _, _ in capi.CORR_FIELDS}
    corr = CorrResult(1, int(cc["trace_status"][0] != capi.T_OK), cc, *[int(x) for x in sc])
    rows, mrows, arows, fp = (next(it).view(np.int64) for _ in range(4))
    tabs = None
    if meta[4]:
        tn = next(it).view(np.int64)
        tcols = {name: next(it).view(proto_tab_dtypes[name]) for name, _, _ in capi.TABLE_FIELDS}
        tabs = Tables(1, tcols, int(tn[0]), int(tn[1]), int(tn[2]))
    return {"rows": rows, "mrows": mrows, "arows": arows, "lo": int(meta[0]), "hi": int(meta[1]),
            "dup_launch": (int(meta[2]), int(meta[3])), "corr": corr, "tabs": tabs, "fusion_parents": fp}


_NPT = {capi.u8p: np.uint8, capi.i8p: np.int8, capi.u32p: np.uint32, capi.i32p: np.int32,
        capi.u64p: np.uint64, capi.i64p: np.int64, capi.f64p: np.float64}
CORR_DTYPES = {name: np.dtype(_NPT[t]) for name, t, _ in capi.CORR_FIELDS}
TAB_DTYPES = {name: np.dtype(_NPT[t]) for name, t, _ in capi.TABLE_FIELDS}


# ---------------------------------------------------------------------------
# ranks

def run_time_sharded(b: SpanBatch, compute: Callable[..., Tuple[CorrResult, Tables]], comm,
                     top_k: int = 3, noise: float = 0.01
                     ) -> Optional[Tuple[CorrResult, Optional[Tables], List[int]]]:
    """Correlate + analyse this rank's time range of b's single trace; rank 0 returns
    the combined unsharded result and the range starts (None on other ranks).

    compute(sub_batch) -> (CorrResult, Tables)."""
    bounds = shard_bounds(b, comm.world)
    lo, hi = bounds[comm.rank], bounds[comm.rank + 1]
    sh = prepare(b, lo, hi, comm)
    corr, tabs = compute(sh.sub)
    fp = np.zeros(0, np.int64)
    if int(corr.trace_status[0]) == capi.T_OK:
        fp = fusion_orphan_parents(sh, corr)
    blobs = comm.gather_bytes(pack_part(sh, corr, tabs, fp))
    if comm.rank != 0:
        return None
    parts = [unpack_part(x, CORR_DTYPES, TAB_DTYPES) for x in blobs]
    corr, tabs = combine(b, parts, top_k=top_k, noise=noise)
    return corr, tabs, bounds[:-1]
