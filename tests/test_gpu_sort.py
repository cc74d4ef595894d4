"""GPU parity for stage (b): xsp_sort_timeline (csrc/sort.cu) against a stable
lexsort by (trace, begin_ns, rank(level), span_id) — the order std::stable_sort
gives with the reference's timeline_key (span.cpp:112-127) — and against the
reference's own sorted_timeline through the C++ drop-in tests. Covers the
per-trace shared-memory path and the global radix-sort fallback."""
import numpy as np
import pytest

from paper_1908_06869_b200 import synth
from paper_1908_06869_b200.columns import SpanBatch

pytestmark = pytest.mark.gpu


def expected_perm(b):
    t = np.searchsorted(b.trace_span_off, np.arange(b.n_spans, dtype=np.uint64), "right") - 1
    lv = (b.flags & 3).astype(np.int64)
    rank = np.where(lv >= 2, 3, lv + 1)
    return np.lexsort((b.span_id, rank, b.begin_ns, t)).astype(np.uint32)


def shuffled(b, seed, frac=1.0):
    """Rows of every trace permuted at random (frac of the traces)."""
    rng = np.random.default_rng(seed)
    perm = np.arange(b.n_spans)
    off = b.trace_span_off
    for t in range(b.n_traces):
        if rng.random() < frac:
            lo, hi = int(off[t]), int(off[t + 1])
            perm[lo:hi] = lo + rng.permutation(hi - lo)
    cols = {k: getattr(b, k)[perm] for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags",
                                              "name_id")}
    return SpanBatch(**cols, flops=b.flops, dram_read=b.dram_read, dram_write=b.dram_write,
                     occupancy=b.occupancy, alloc_bytes=b.alloc_bytes, type_id=b.type_id,
                     trace_span_off=b.trace_span_off, trace_id=b.trace_id, trace_levels=b.trace_levels,
                     trace_batch=b.trace_batch, trace_run=b.trace_run, trace_serialized=b.trace_serialized,
                     names=b.names, types=b.types)


def test_presorted_identity(engine):
    b, *_ = synth.c3(runs=2, n_models=4)
    perm, was = engine.sort_timeline(b)
    assert was and np.array_equal(perm, np.arange(b.n_spans, dtype=np.uint32))


@pytest.mark.parametrize("seed", [1, 2])
def test_shuffled_c3(engine, seed):
    b, *_ = synth.c3(runs=2, n_models=6)
    s = shuffled(b, seed, frac=0.7)
    perm, was = engine.sort_timeline(s)
    assert not was
    assert np.array_equal(perm, expected_perm(s))


def test_ties_and_levels(engine):
    """Equal begins across levels and equal (begin, rank) broken by span_id."""
    rng = np.random.default_rng(5)
    n_tr, per = 50, 300
    n = n_tr * per
    b = SpanBatch(span_id=rng.integers(0, 50, n).astype(np.uint64), parent_id=np.zeros(n, np.uint64),
                  begin_ns=rng.integers(1000, 1010, n).astype(np.uint64),
                  end_ns=np.full(n, 5000, np.uint64), cid=np.zeros(n, np.uint64),
                  flags=rng.integers(0, 4, n).astype(np.uint8), name_id=np.zeros(n, np.uint32),
                  flops=np.zeros(0, np.uint64), dram_read=np.zeros(0, np.uint64),
                  dram_write=np.zeros(0, np.uint64), occupancy=np.zeros(0), alloc_bytes=np.zeros(0, np.int64),
                  type_id=np.zeros(0, np.uint32), trace_span_off=np.arange(n_tr + 1, dtype=np.uint64) * per,
                  trace_id=np.arange(n_tr), trace_levels=np.full(n_tr, 7), trace_batch=np.ones(n_tr),
                  trace_run=np.zeros(n_tr), trace_serialized=np.zeros(n_tr), names=[b"x"], types=[])
    perm, was = engine.sort_timeline(b)
    assert np.array_equal(perm, expected_perm(b))


def test_fallback_wide_keys_and_long_trace(engine):
    """Keys wider than 63 bits (huge begin and span_id ranges) and a trace longer
    than one CTA's capacity take the global radix sort."""
    rng = np.random.default_rng(6)
    lens = [3, 20000, 1, 0, 700]
    n = sum(lens)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    beg = rng.integers(0, 2 ** 62, n).astype(np.uint64)
    beg[:3] = [5, 5, 5]
    b = SpanBatch(span_id=rng.integers(0, 2 ** 63, n).astype(np.uint64), parent_id=np.zeros(n, np.uint64),
                  begin_ns=beg, end_ns=beg, cid=np.zeros(n, np.uint64),
                  flags=rng.integers(0, 4, n).astype(np.uint8), name_id=np.zeros(n, np.uint32),
                  flops=np.zeros(0, np.uint64), dram_read=np.zeros(0, np.uint64),
                  dram_write=np.zeros(0, np.uint64), occupancy=np.zeros(0), alloc_bytes=np.zeros(0, np.int64),
                  type_id=np.zeros(0, np.uint32), trace_span_off=off, trace_id=np.arange(len(lens)),
                  trace_levels=np.full(len(lens), 7), trace_batch=np.ones(len(lens)),
                  trace_run=np.zeros(len(lens)), trace_serialized=np.zeros(len(lens)), names=[b"x"], types=[])
    perm, was = engine.sort_timeline(b)
    assert np.array_equal(perm, expected_perm(b))


def test_size_classes_boundaries(engine):
    """Traces at the edges of every shared-memory size class (4096 / 8192 /
    16384 spans per CTA), with begin ties broken by rank and span_id."""
    rng = np.random.default_rng(7)
    lens = [4096, 4097, 8192, 8193, 16384, 2, 31, 33, 5000]
    n = sum(lens)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    beg = rng.integers(10 ** 9, 10 ** 9 + 20000, n).astype(np.uint64)
    b = SpanBatch(span_id=rng.integers(0, 4000, n).astype(np.uint64), parent_id=np.zeros(n, np.uint64),
                  begin_ns=beg, end_ns=beg + 5, cid=np.zeros(n, np.uint64),
                  flags=rng.integers(0, 4, n).astype(np.uint8), name_id=np.zeros(n, np.uint32),
                  flops=np.zeros(0, np.uint64), dram_read=np.zeros(0, np.uint64),
                  dram_write=np.zeros(0, np.uint64), occupancy=np.zeros(0), alloc_bytes=np.zeros(0, np.int64),
                  type_id=np.zeros(0, np.uint32), trace_span_off=off, trace_id=np.arange(len(lens)),
                  trace_levels=np.full(len(lens), 7), trace_batch=np.ones(len(lens)),
                  trace_run=np.zeros(len(lens)), trace_serialized=np.zeros(len(lens)), names=[b"x"], types=[])
    perm, was = engine.sort_timeline(b)
    assert not was
    assert np.array_equal(perm, expected_perm(b))


def _batch(lens, beg, sid, flags):
    n = sum(lens)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    return SpanBatch(span_id=sid, parent_id=np.zeros(n, np.uint64), begin_ns=beg, end_ns=beg + 5,
                     cid=np.zeros(n, np.uint64), flags=flags, name_id=np.zeros(n, np.uint32),
                     flops=np.zeros(0, np.uint64), dram_read=np.zeros(0, np.uint64),
                     dram_write=np.zeros(0, np.uint64), occupancy=np.zeros(0), alloc_bytes=np.zeros(0, np.int64),
                     type_id=np.zeros(0, np.uint32), trace_span_off=off, trace_id=np.arange(len(lens)),
                     trace_levels=np.full(len(lens), 7), trace_batch=np.ones(len(lens)),
                     trace_run=np.zeros(len(lens)), trace_serialized=np.zeros(len(lens)), names=[b"x"], types=[])


def test_wide_span_ids_tie_runs(engine):
    """span_id ranges too wide to pack beside begin (random 64-bit ids): keys
    carry (begin, rank, index) and runs of equal (begin, rank) are ordered by
    span_id afterwards; duplicate span_ids stay in input order."""
    rng = np.random.default_rng(8)
    lens = [300, 5000, 9000, 40, 1]
    n = sum(lens)
    beg = rng.integers(10 ** 12, 10 ** 12 + 400, n).astype(np.uint64)
    sid = rng.integers(0, 2 ** 63, n).astype(np.uint64)
    sid[::7] = sid[1::7][: len(sid[::7])]  # duplicates
    b = _batch(lens, beg, sid, rng.integers(0, 4, n).astype(np.uint8))
    perm, was = engine.sort_timeline(b)
    assert not was
    assert np.array_equal(perm, expected_perm(b))


def test_long_tie_run_falls_back(engine):
    """A run of > 1024 spans with equal (begin, rank) and wide span_ids takes the
    global radix sort."""
    rng = np.random.default_rng(9)
    lens = [3000, 200]
    n = sum(lens)
    beg = np.full(n, 7, np.uint64)
    beg[3000:] = rng.integers(0, 50, 200).astype(np.uint64)
    sid = rng.integers(0, 2 ** 63, n).astype(np.uint64)
    b = _batch(lens, beg, sid, np.full(n, 2, np.uint8))
    perm, was = engine.sort_timeline(b)
    assert not was
    assert np.array_equal(perm, expected_perm(b))
