"""GPU parity for stage (f), the leveled-measurement merge, against the reference's
LeveledRunGroup::from_bundles + compute_overhead (oracle/_ref)."""
import numpy as np
import pytest

from oracle import ref
from paper_1908_06869_b200.leveled import LeveledError, compute_overhead

pytestmark = pytest.mark.gpu

M, ML, MLG = 0b001, 0b011, 0b111


def compare(report, bag):
    arrays, strings = bag
    assert int(arrays["status"][0]) == 0, strings["error"]
    n = len(arrays["o_level"])
    assert len(report.rows) == n
    off = arrays["o_ov_off"]
    for i, row in enumerate(report.rows):
        assert row.level == int(arrays["o_level"][i])
        assert row.layer_index == int(arrays["o_layer"][i])
        assert row.kernel_index == int(arrays["o_kernel"][i])
        acc = arrays["o_accurate"][i]
        if np.isnan(acc):
            assert row.accurate_latency_ns is None
        else:
            assert row.accurate_latency_ns == acc
        assert row.clamped == bool(arrays["o_clamped"][i])
        want = {int(arrays["o_ov_mask"][j]): float(arrays["o_ov_val"][j]) for j in range(off[i], off[i + 1])}
        assert row.overhead_by_added_levels == want, (i, row.overhead_by_added_levels, want)
    want_model = {int(m): float(v) for m, v in zip(arrays["model_ov_mask"], arrays["model_ov_val"])}
    assert report.model_overhead_by_added_levels == want_model
    assert report.warnings == [w.decode() for w in strings["warnings"]]


def run(engine, gen, **kw):
    b = gen.batch()
    return compute_overhead(engine, b, **kw), ref.leveled(b, **{k: v for k, v in kw.items()})


def test_overhead_chain_recovers_injected_overhead(engine, has_ref):
    """Criterion 7 (acceptance_main.cpp:154-179): 157 ms / 58.2 ms / 0.24 ms exactly."""
    g = ref.Generator().chain("overhead-chain", 1, 15_700_000, 0, 2.0)
    rep, bag = run(engine, g)
    compare(rep, bag)
    assert rep.warnings == []
    assert rep.model_overhead_by_added_levels[0b010] == 157_000_000.0
    assert rep.model_overhead_by_added_levels[0b100] == 58_200_000.0
    layer0 = next(r for r in rep.rows if r.level == 1 and r.layer_index == 0)
    assert layer0.overhead_by_added_levels[0b100] == 240_000.0


@pytest.mark.parametrize("model", ["resnet-like", "mobilenet-like", "minimal", "async-straggler"])
def test_chain_fixtures(engine, has_ref, model):
    g = ref.Generator().chain(model, 2, 15_700_000, 1000, 1.5)
    compare(*run(engine, g))


def test_repetitions_with_jitter_and_clamping(engine, has_ref):
    """Trimmed means over repeated runs per level set; jitter larger than the injected
    overhead produces clamped and negative-beyond-noise steps (leveled.cpp:190-201)."""
    g = ref.Generator()
    for levels in (M, ML, MLG):
        for r in range(5):
            g.emit("overhead-chain", 1, levels, 0, 0, 1.0, False, r, 400_000, 31 * r + levels)
    for noise in (0.01, 0.0, 0.5):
        rep, bag = run(engine, g, noise=noise)
        compare(rep, bag)


def test_more_than_64_repetitions_per_set(engine, has_ref):
    """Level sets of 70 repetitions (the selection path of the trimmed mean)."""
    g = ref.Generator()
    for levels in (M, ML, MLG):
        for r in range(70):
            g.emit("minimal", 1, levels, 0, 0, 1.0, False, r, 300_000, 7 * r + levels)
    compare(*run(engine, g))


def test_structure_changes_across_the_chain(engine, has_ref):
    """Events present in one set only produce the 'visible under' warnings."""
    g = ref.Generator()
    g.emit("minimal", 1, M).emit("resnet-like", 1, ML).emit("resnet-like", 1, MLG)
    compare(*run(engine, g))


def test_two_sets_and_order_independence(engine, has_ref):
    g = ref.Generator()
    g.emit("resnet-like", 1, MLG, 1_000_000).emit("resnet-like", 1, M)
    compare(*run(engine, g))


def test_faults(engine, has_ref):
    b = ref.Generator().emit("resnet-like", 1, MLG).batch()
    with pytest.raises(LeveledError, match="at least two chained level sets; got 1"):
        compute_overhead(engine, b)
    b = ref.Generator().emit("resnet-like", 1, ML).emit("resnet-like", 1, 0b1001).batch()
    with pytest.raises(LeveledError) as e:
        compute_overhead(engine, b)
    _, strings = ref.leveled(b)
    assert str(e.value) == strings["error"][0].decode()
    assert "M+L and M+A do not form an inclusion chain" in str(e.value)
    # a bundle the correlator rejects: the TraceError propagates unchanged
    b = ref.Generator().emit("resnet-like", 1, ML).emit("resnet-like", 1, 0b101).batch()
    with pytest.raises(RuntimeError) as e:
        compute_overhead(engine, b)
    assert str(e.value) == ref.leveled(b)[1]["error"][0].decode()
    b = ref.Generator().emit("overlap", 1, M).emit("overlap", 1, MLG).batch()
    with pytest.raises(LeveledError, match="ambiguous span"):
        compute_overhead(engine, b)
    b = ref.Generator().emit("minimal", 1, M).emit("minimal", 2, ML).batch()
    with pytest.raises(LeveledError, match="runs mix batch sizes 1 and 2"):
        compute_overhead(engine, b)


def test_synthetic_leveled_corpus_per_model(engine, has_ref):
    """The bench's leveled workload (synth.leveled_corpus: C2 at scale): each
    model's {M}, {M,L}, {M,L,G} x R runs, one LeveledRunGroup per model, against
    the reference; and the device path the bench times (one correlation of the
    whole corpus, one xsp_leveled per model) agrees with the per-model report."""
    from paper_1908_06869_b200 import synth
    from paper_1908_06869_b200.engine import DeviceBatch
    models = synth.make_models(4, seed=3, max_layers=400)
    b, sets = synth.leveled_corpus(models, runs=5)
    dev = DeviceBatch(b)
    co = engine.correlate_device(dev)
    for s in sets:
        idx = [t for _, tr in s for t in tr]
        sub = b.select_traces(idx)
        rep = compute_overhead(engine, sub)
        compare(rep, ref.leveled(sub))
        assert rep.model_overhead_by_added_levels  # the injected per-level overhead is visible
        ls, keep = engine.make_level_sets(s)
        out = engine.leveled_device(dev, co, ls)
        assert out.status == 0 and out.n_sets == 3 and out.n_events == len(rep.rows)


def test_leveled_batch_equals_per_group(engine):
    """xsp_leveled_batch over many LeveledRunGroups (the bench's one-call-per-
    batch path) returns, group by group, exactly what xsp_leveled returns:
    statuses, chains, event keys, per-set latencies, overheads, flags and
    accurate latencies (bit for bit) — including groups that report
    TOO_FEW / NOT_CHAIN and an empty group."""
    from paper_1908_06869_b200 import synth
    from paper_1908_06869_b200.engine import DeviceBatch
    from paper_1908_06869_b200.leveled import _d2h
    models = synth.make_models(5, seed=7, max_layers=300)
    b, sets = synth.leveled_corpus(models, runs=4)
    # extra groups: one set only, a non-chain pair, no sets, sets in reverse order
    extra = [sets[0][:1], [(0b011, sets[1][1][1]), (0b101, sets[1][2][1])], [], list(reversed(sets[2]))]
    groups = sets + extra
    dev = DeviceBatch(b)
    co = engine.correlate_device(dev)
    keep = [engine.make_level_sets(s) for s in groups]

    def arrays(o):
        ne, ns = o.n_events, o.n_sets
        cols = {"ev_level": (o.ev_level, np.uint8, ne), "ev_layer": (o.ev_layer, np.uint32, ne),
                "ev_kernel": (o.ev_kernel, np.uint32, ne), "lat": (o.lat, np.float64, ns * ne),
                "overhead": (o.overhead, np.float64, max(ns - 1, 0) * ne),
                "step_flags": (o.step_flags, np.uint8, max(ns - 1, 0) * ne),
                "accurate": (o.accurate, np.float64, ne)}
        out = {k: _d2h(engine.lib, engine.ctx, p, t, n) for k, (p, t, n) in cols.items()}
        out["chain"] = [o.chain[i] for i in range(ns)] if ns and o.chain else []
        return (o.status, o.err_a, o.err_b, ns, ne), out

    single = [arrays(engine.leveled_device(dev, co, ls)) for ls, _ in keep]
    batch = engine.leveled_batch_device(dev, co, [ls for ls, _ in keep])
    assert len(batch) == len(groups)
    got = [arrays(o) for o in batch]
    statuses = [g[0][0] for g in got]
    assert statuses[:len(sets)] == [0] * len(sets) and statuses[len(sets):] == [1, 2, 1, 0], statuses
    for (h1, a1), (h2, a2) in zip(single, got):
        assert h1 == h2
        for k in a1:
            x, y = np.asarray(a1[k]), np.asarray(a2[k])
            assert x.shape == y.shape and np.array_equal(x.view(np.uint8), y.view(np.uint8)), k
