"""Multi-GPU sharding of the correlate + analyze path (one process per GPU).

The unit of work is an analysis group: the R repetition traces of one
(model, batch size) pair (analysis.cpp:102-140 combines exactly those). Traces
and groups are independent, so the path shards with NO data-path collective:
every rank correlates and analyses the groups assigned to it, and only the
finished tables travel, once, to rank 0 (a control-path gather). Per-GPU work
is fixed as ranks are added ("weak" scaling in bench.py); for a fixed corpus
`assign_groups` balances spans across ranks (LPT: longest group to the least
loaded rank).

compute(batch, groups) -> Tables is pluggable: Engine.run_host on a GPU, the C
oracle in the CPU tests (tests/test_shard.py, gloo, world_size 2).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as capi
from .columns import SpanBatch
from .engine import Tables

Groups = Tuple[np.ndarray, np.ndarray, np.ndarray]  # (first_trace, n_runs, batch_size)


def group_spans(batch: SpanBatch, groups: Groups) -> np.ndarray:
    """Spans per group (the work weight)."""
    first, runs = np.asarray(groups[0], np.int64), np.asarray(groups[1], np.int64)
    off = batch.trace_span_off.astype(np.int64)
    return off[first + runs] - off[first]


def assign_groups(weights: Sequence[int], world: int) -> np.ndarray:
    """Rank of every group: longest-processing-time-first greedy (deterministic:
    ties broken by group index, then by rank)."""
    w = np.asarray(weights, dtype=np.int64)
    order = np.lexsort((np.arange(w.size), -w))
    load = np.zeros(world, dtype=np.int64)
    rank = np.empty(w.size, dtype=np.int64)
    for g in order:
        r = int(np.argmin(load))
        rank[g] = r
        load[r] += w[g]
    return rank


def shard(batch: SpanBatch, groups: Groups, ranks: np.ndarray, rank: int
          ) -> Tuple[Optional[SpanBatch], Groups, np.ndarray, np.ndarray]:
    """This rank's sub-batch (its groups' traces, in global group order), its
    group arrays (first trace re-based), the global ids of those groups, and
    the global first span row of every local trace (to map span rows back)."""
    first, runs, bsz = (np.asarray(x, np.int64) for x in groups)
    gids = np.nonzero(ranks == rank)[0]
    if gids.size == 0:
        z = np.zeros(0, np.int64)
        return None, (z, z, z), gids, z
    parts, lfirst, t = [], [], 0
    span_base = []
    for g in gids:
        t0, t1 = int(first[g]), int(first[g] + runs[g])
        parts.append(batch.trace_slice(t0, t1))
        span_base.append(batch.trace_span_off[t0:t1].astype(np.int64))
        lfirst.append(t)
        t += t1 - t0
    sub = SpanBatch.concat(parts) if len(parts) > 1 else parts[0]
    if sub.names != batch.names or sub.types != batch.types:
        raise ValueError("shard: string tables changed (batch names must be interned in sorted order)")
    return sub, (np.array(lfirst), runs[gids], bsz[gids]), gids, np.concatenate(span_base)


def _local_to_global_rows(rows: np.ndarray, sub: SpanBatch, span_base: np.ndarray) -> np.ndarray:
    off = sub.trace_span_off.astype(np.int64)
    t = np.searchsorted(off, rows.astype(np.int64), side="right") - 1
    return (rows.astype(np.int64) - off[t] + span_base[t]).astype(np.uint32)


def combine(parts: List[Tuple[Tables, np.ndarray]], n_groups: int, top_k: int) -> Tables:
    """Merge per-rank tables (each with its global group ids) into one Tables in
    global group order. Row blocks of each group are copied whole; the CSR
    offsets are rebuilt. Column meaning is unchanged (include/xsp.h)."""
    owner = np.full(n_groups, -1, np.int64)
    local = np.zeros(n_groups, np.int64)
    for p, (_, gids) in enumerate(parts):
        owner[gids] = p
        local[gids] = np.arange(gids.size)
    if (owner < 0).any():
        raise ValueError(f"combine: groups {np.nonzero(owner < 0)[0][:8].tolist()} missing")
    kinds = {n: k for n, _, k in capi.TABLE_FIELDS}
    csr = {"K": "group_kernel_off", "L": "group_layer_off", "N": "group_name_off", "LK": "group_layer_off",
           "Y": "group_type_off"}
    offsets = ("group_kernel_off", "group_layer_off", "group_name_off", "group_type_off")
    cols = {}
    for name, kind in kinds.items():
        if name in offsets:
            continue
        if kind == "G":
            proto = parts[0][0].cols[name]
            out = np.empty(n_groups, dtype=proto.dtype)
            for tabs, gids in parts:
                out[gids] = tabs.cols[name]
            cols[name] = out
            continue
        mult = max(top_k, 1) if kind == "LK" else 1
        offn = csr[kind]
        blocks = []
        for g in range(n_groups):
            tabs = parts[owner[g]][0]
            o = tabs.cols[offn]
            i = local[g]
            blocks.append(tabs.cols[name][int(o[i]) * mult:int(o[i + 1]) * mult])
        cols[name] = np.concatenate(blocks) if blocks else parts[0][0].cols[name][:0]
    for offn in offsets:
        sizes = np.zeros(n_groups, np.int64)
        for tabs, gids in parts:
            o = tabs.cols[offn].astype(np.int64)
            sizes[gids] = o[1:] - o[:-1]
        cols[offn] = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint32)
    return Tables(n_groups, cols, int(cols["group_layer_off"][-1]), int(cols["group_kernel_off"][-1]),
                  int(cols["group_name_off"][-1]))


_NPT = {capi.u8p: np.uint8, capi.i8p: np.int8, capi.u32p: np.uint32, capi.i32p: np.int32,
        capi.u64p: np.uint64, capi.i64p: np.int64, capi.f64p: np.float64}


def pack_tables(tabs: Optional[Tables], gids: np.ndarray) -> np.ndarray:
    """One rank's tables + global group ids as a flat byte array (column sizes
    first, then the columns in include/xsp.h order; no pickling)."""
    cols = [np.asarray(gids, np.int64)]
    if tabs is not None:
        cols += [np.asarray(tabs.cols[name]) for name, _, _ in capi.TABLE_FIELDS]
    sizes = np.array([c.nbytes for c in cols], np.int64)
    head = np.concatenate([[sizes.size], sizes]).astype(np.int64)
    return np.concatenate([head.view(np.uint8)] + [np.ascontiguousarray(c).view(np.uint8).reshape(-1) for c in cols])


def unpack_tables(buf: np.ndarray) -> Optional[Tuple[Tables, np.ndarray]]:
    n = int(buf[:8].view(np.int64)[0])
    sizes = buf[8:8 + 8 * n].view(np.int64)
    off = 8 + 8 * n
    chunks = []
    for sz in sizes.tolist():
        chunks.append(buf[off:off + sz])
        off += sz
    gids = chunks[0].view(np.int64)
    if n == 1:
        return None
    cols = {name: chunks[1 + i].view(_NPT[t]) for i, (name, t, _) in enumerate(capi.TABLE_FIELDS)}
    G = int(cols["group_status"].size)
    return Tables(G, cols), gids


def run_sharded(batch: SpanBatch, groups: Groups, compute: Callable[[SpanBatch, Groups], Tables],
                rank: int, world: int, top_k: int = 3, dist=None, comm=None) -> Optional[Tables]:
    """Correlate + analyse this rank's share and gather the tables on rank 0
    (returns them there, None elsewhere). The tables travel as one byte tensor
    per rank over `comm` (timeshard.TorchComm over torch.distributed — gloo in
    the CPU tests; run_sharded_device uses the NCCL C-ABI combine on GPUs) or,
    given only `dist`, a TorchComm on CPU tensors. world == 1 needs neither."""
    n_groups = len(groups[0])
    ranks = assign_groups(group_spans(batch, groups), world)
    sub, lgroups, gids, span_base = shard(batch, groups, ranks, rank)
    tabs = None
    if sub is not None:
        tabs = compute(sub, lgroups)
        tabs.cols["l_row"] = _local_to_global_rows(tabs.cols["l_row"], sub, span_base)
    if world == 1:
        gathered = [pack_tables(tabs, gids)]
    else:
        if comm is None:
            from .timeshard import TorchComm
            comm = TorchComm(dist, "cpu")
        gathered = comm.gather_bytes(pack_tables(tabs, gids))
    if rank != 0:
        return None
    parts = [p for p in (unpack_tables(b) for b in gathered) if p is not None]
    return combine(parts, n_groups, top_k)


def l_row_map(sub: SpanBatch, span_base: np.ndarray) -> np.ndarray:
    """Global span row of every span row of a rank's sub-batch."""
    off = sub.trace_span_off.astype(np.int64)
    out = np.empty(sub.n_spans, np.uint32)
    for t in range(sub.n_traces):
        out[off[t]:off[t + 1]] = span_base[t] + np.arange(off[t + 1] - off[t])
    return out


def run_sharded_device(engine, batch: SpanBatch, groups: Groups, rank: int, world: int, dist=None,
                       top_k: int = 3, stream=None):
    """The GPU form: rank r correlates + analyses its groups device-resident
    (xsp_run) and the device tables are combined on rank 0 with NCCL
    (xsp_combine_tables; the engine must have joined the communicator with
    Engine.comm_init). Returns (rank 0's host Tables or None, bytes sent)."""
    import torch
    from .engine import DeviceBatch
    n_groups = len(groups[0])
    ranks = assign_groups(group_spans(batch, groups), world)
    sub, lgroups, gids, span_base = shard(batch, groups, ranks, rank)
    if sub is None:  # no groups on this rank: an empty batch still takes part in the combine
        raise ValueError("run_sharded_device: every rank needs at least one group")
    dev = DeviceBatch(sub, torch.cuda.current_device())
    _, to = engine.run_device(dev, lgroups, top_k=top_k, stream=stream)
    rmap = torch.from_numpy(l_row_map(sub, span_base).view(np.int32)).to(f"cuda:{torch.cuda.current_device()}")
    out, sent = engine.combine_tables(to, gids, n_groups, rmap.data_ptr(), top_k=top_k, stream=stream)
    if rank != 0:
        return None, sent
    return engine.tables_to_host(out, top_k), sent
