"""GPU parity for stage (a) invariants: xsp_validate (csrc/validate.cu) against the
UNMODIFIED reference validate_bundle (span.cpp:129-192, via oracle/_ref) on the
same bundles: every issue, in the reference's report order, with its span_id,
rule and detail text."""
import numpy as np
import pytest

from oracle import ref
from paper_1908_06869_b200 import _capi as capi
from paper_1908_06869_b200 import synth
from paper_1908_06869_b200.columns import SpanBatch

pytestmark = pytest.mark.gpu


def span_trace_ids(b):
    t = np.searchsorted(b.trace_span_off, np.arange(b.n_spans, dtype=np.uint64), "right") - 1
    return b.trace_id[t].astype(np.uint64)


def gpu_report(engine, b, tid=None, tb=None):
    out = []
    for issues in engine.validate(b, tid, tb):
        rep = []
        for row, rule in issues:
            text, det = capi.VALIDATION_RULES[rule]
            rep.append((0 if row < 0 else int(b.span_id[row]), text, det))
        out.append(rep)
    return out


def check(engine, b, tid=None, tb=None):
    got = gpu_report(engine, b, tid, tb)
    want = ref.validate(b, tid, tb)
    assert len(got) == len(want)
    for t, (g, w) in enumerate(zip(got, want)):
        assert g == w, f"trace {t}: {g[:6]} != {w[:6]}"
    return got


def fixture_batch():
    g = ref.Generator()
    for f in ("resnet-like", "overlap", "async-straggler", "minimal"):
        g.emit(f, batch=2)
    g.random_nested(5, 3000)
    g.random_async(6, 500)
    return g.batch()


def test_clean_batches(engine, has_ref):
    b = fixture_batch()
    got = check(engine, b)
    assert all(len(x) == 0 for x in got)
    c3, *_ = synth.c3(runs=2, n_models=3)
    got = check(engine, c3, span_trace_ids(c3))
    assert all(len(x) == 0 for x in got)


def mutate(b, seed):
    """Corrupt a copy of `b` with every rule's violation at random rows."""
    rng = np.random.default_rng(seed)
    cols = {k: getattr(b, k).copy() for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags",
                                              "name_id", "flops", "dram_read", "dram_write", "occupancy",
                                              "alloc_bytes", "type_id", "trace_span_off", "trace_id",
                                              "trace_levels", "trace_batch", "trace_run", "trace_serialized")}
    n = b.n_spans
    pick = lambda k: rng.choice(n, size=k, replace=False)
    # negative duration
    r = pick(20)
    cols["end_ns"][r] = cols["begin_ns"][r] - np.uint64(1) - rng.integers(0, 50, r.size).astype(np.uint64)
    # cid presence flips (launch/exec without cid, sync with cid)
    r = pick(30)
    cols["flags"][r] ^= np.uint8(capi.F_CID)
    # duplicate span ids within a trace (copy the id of the previous span)
    r = pick(25)
    r = r[r > 0]
    cols["span_id"][r] = cols["span_id"][r - 1]
    # out of order: swap begins of neighbours
    r = pick(25)
    r = r[r + 1 < n]
    a, c = cols["begin_ns"][r].copy(), cols["begin_ns"][r + 1].copy()
    cols["begin_ns"][r], cols["begin_ns"][r + 1] = c + np.uint64(7), a
    # model spans: drop one (turn into a layer) and duplicate one
    # (level changes keep the layer table aligned: only non-layer spans change level)
    off = cols["trace_span_off"]
    cols["flags"][int(off[1])] = (cols["flags"][int(off[1])] & ~np.uint8(3)) | np.uint8(capi.LEVEL_KERNEL)
    if b.n_traces > 3:
        lv = cols["flags"][int(off[3]):int(off[4])] & 3
        k = int(off[3]) + int(np.nonzero(lv == capi.LEVEL_KERNEL)[0][0])
        cols["flags"][k] = cols["flags"][k] & ~np.uint8(0x0F)  # model / sync
    cols["trace_levels"][-1] &= ~np.uint32(1)
    out = SpanBatch(**cols, names=b.names, types=b.types, system_name=b.system_name,
                    peak_flops=b.peak_flops, mem_bw=b.mem_bw)
    tid = span_trace_ids(out)
    r = pick(15)
    tid[r] += np.uint64(1000)
    tb = np.zeros(n, dtype=np.uint8)
    met = np.nonzero(cols["flags"] & capi.F_METRICS)[0]
    tb[met] = capi.TAG_OCC_DOUBLE
    tb[rng.choice(met, size=min(20, met.size), replace=False)] |= capi.TAG_NEG_FLOPS
    tb[rng.choice(met, size=min(20, met.size), replace=False)] |= capi.TAG_NEG_READ | capi.TAG_NEG_WRITE
    tb[rng.choice(met, size=min(10, met.size), replace=False)] &= ~np.uint8(capi.TAG_OCC_DOUBLE)
    mrow = rng.choice(met.size, size=min(25, met.size), replace=False)
    out.occupancy[mrow] = rng.choice([-0.25, 1.5, 2.0, -1e-9, 1.0 + 1e-12, 0.0, 1.0], size=mrow.size)
    return out, tid, tb


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_every_rule(engine, has_ref, seed):
    b, tid, tb = mutate(fixture_batch(), seed)
    got = check(engine, b, tid, tb)
    rules = {x[1] for rep in got for x in rep}
    for must in ("negative duration", "correlation_id missing", "duplicate span_id", "trace_id mismatch",
                 "out of order", "negative metric", "occupancy out of range", "model span missing",
                 "multiple model spans", "model level disabled"):
        assert must in rules, must


def test_without_optional_columns(engine, has_ref):
    b, _, _ = mutate(fixture_batch(), 9)
    # no trace ids, no tag bits: the reference sees consistent ids and decoded tags
    got = gpu_report(engine, b)
    want = ref.validate(b, None, np.full(b.n_spans, capi.TAG_OCC_DOUBLE, dtype=np.uint8))
    # occupancy range needs the tag bit; compare the rest
    strip = lambda reps: [[x for x in r if x[1] != "occupancy out of range"] for r in reps]
    assert strip(got) == strip(want)


def test_empty_and_tiny_traces(engine, has_ref):
    g = ref.Generator()
    g.emit("minimal")
    b = g.batch()
    # append an empty trace
    off = np.concatenate([b.trace_span_off, b.trace_span_off[-1:]])
    b2 = SpanBatch(**{k: getattr(b, k) for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags",
                                                  "name_id", "flops", "dram_read", "dram_write", "occupancy",
                                                  "alloc_bytes", "type_id")},
                   trace_span_off=off, trace_id=np.append(b.trace_id, 77),
                   trace_levels=np.append(b.trace_levels, 7), trace_batch=np.append(b.trace_batch, 1),
                   trace_run=np.append(b.trace_run, 0), trace_serialized=np.append(b.trace_serialized, 0),
                   names=b.names, types=b.types)
    got = check(engine, b2)
    assert got[-1] == [(0, "model span missing", "a bundle requires exactly one model/sync span")]


def test_c3_scale_duplicates(engine):
    """Size-independent property at a few million spans: duplicating k ids yields
    exactly k duplicate issues, on the later rows."""
    b, *_ = synth.c3(runs=3, n_models=12)
    rng = np.random.default_rng(4)
    off = b.trace_span_off
    t = rng.choice(b.n_traces, size=40, replace=False)
    rows = [int(off[x]) + 5 for x in t]
    sid = b.span_id.copy()
    for r in rows:
        sid[r + 3] = sid[r]  # later row repeats an earlier id of the same trace
    b.span_id = sid
    got = engine.validate(b)
    dups = sorted(row for rep in got for row, rule in rep if rule == 3)
    others = [(row, rule) for rep in got for row, rule in rep if rule not in (3, 5)]
    assert dups == sorted(r + 3 for r in rows)
    assert others == []
