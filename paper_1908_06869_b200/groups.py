"""Experiment grouping over trace descriptors: the reference's RunSet
(collector.cpp:320-345) and build_batch_groups (cli.cpp:358-399) for a
SpanBatch's traces (trace_batch, trace_levels, trace_id, trace_run).

  * run_set(batch): (batch_size, level set) -> trace indices in batch order,
    with the reference's MergeError for a (trace_id, run_index) seen twice in
    one group. (The system-spec check is per batch: a SpanBatch has one spec.)
  * batch_groups(batch): per batch size (ascending) the deepest level set
    sampled at that size (most levels; ties -> the lexicographically greater
    set, std::set<Level> order), as the trace order + xsp_groups arguments the
    analysis takes: one analysis group of R runs per batch size.
  * check_unambiguous(corr, batch, order): the TraceError build_batch_groups
    throws for a run with ambiguous kernels (cli.cpp:387-393).
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np

from .columns import SpanBatch


class MergeError(ValueError):
    pass


class TraceError(ValueError):
    pass


def _levels(mask: int) -> Tuple[int, ...]:
    return tuple(l for l in range(4) if mask >> l & 1)


def run_set(batch: SpanBatch) -> Dict[Tuple[int, Tuple[int, ...]], List[int]]:
    groups: Dict[Tuple[int, Tuple[int, ...]], List[int]] = {}
    seen: Dict[Tuple[int, Tuple[int, ...]], set] = {}
    for t in range(batch.n_traces):
        key = (int(batch.trace_batch[t]), _levels(int(batch.trace_levels[t])))
        run = (int(batch.trace_id[t]), int(batch.trace_run[t]))
        if run in seen.setdefault(key, set()):
            raise MergeError(f"duplicate run (trace {run[0]}, run_index {run[1]})")
        seen[key].add(run)
        groups.setdefault(key, []).append(t)
    return dict(sorted(groups.items()))


def batch_groups(batch: SpanBatch):
    """(trace order, (first, runs, batch_size), level sets): take
    batch.select_traces(order) and analyse it with the groups."""
    deepest: Dict[int, Tuple[int, Tuple[int, ...]]] = {}
    for key in run_set(batch):
        b, lv = key
        cur = deepest.get(b)
        if cur is None or len(lv) > len(cur[1]) or (len(lv) == len(cur[1]) and cur[1] < lv):
            deepest[b] = key
    rs = run_set(batch)
    order, first, runs, sizes, levels = [], [], [], [], []
    for b in sorted(deepest):
        tr = rs[deepest[b]]
        first.append(len(order))
        runs.append(len(tr))
        sizes.append(b)
        levels.append(deepest[b][1])
        order.extend(tr)
    return np.array(order, np.int64), (np.array(first), np.array(runs), np.array(sizes)), levels


def check_unambiguous(corr, batch: SpanBatch) -> None:
    """Raise the reference's TraceError for the first trace (batch order) with ambiguities."""
    off = corr.trace_amb_off.astype(np.int64)
    for t in range(batch.n_traces):
        n = int(off[t + 1] - off[t])
        if n:
            raise TraceError(f"trace {int(batch.trace_id[t])} has {n} ambiguous spans; resolve them first"
                             " (correlate --serialized-rerun) or profile serialized")
