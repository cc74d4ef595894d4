"""Experiment grouping over trace descriptors (paper_1908_06869_b200/groups.py):
RunSet (collector.cpp:320-345) and build_batch_groups (cli.cpp:358-399).
CPU tests check the grouping itself and, through the C oracle port, that the
selected traces analyse like the reference's per-batch AnalysisInput; the GPU
test runs the grouped batch through the CUDA engine against the reference."""
import numpy as np
import pytest

from paper_1908_06869_b200 import groups


def experiment():
    from oracle import ref
    g = ref.Generator()
    # batch 1: {M,L,G} x 3 runs and {M,L} x 2 runs; batch 2: {M,L,G} x 2; batch 4: {M} x 2 and {M,L} x 2
    for r in range(3):
        g.emit("resnet-like", batch=1, run_index=r, jitter_max=500, jitter_seed=r + 1)
    for r in range(2):
        g.emit("resnet-like", batch=1, levels=0b011, run_index=r, jitter_max=500, jitter_seed=r + 10)
    for r in range(2):
        g.emit("resnet-like", batch=4, levels=0b001, run_index=r)
    for r in range(2):
        g.emit("resnet-like", batch=2, run_index=r, jitter_max=500, jitter_seed=r + 20)
    for r in range(2):
        g.emit("resnet-like", batch=4, levels=0b011, run_index=r, jitter_max=300, jitter_seed=r + 30)
    return g.batch()


def test_run_set_keys_and_duplicates():
    b = experiment()
    rs = groups.run_set(b)
    assert list(rs) == sorted(rs)
    assert {k: len(v) for k, v in rs.items()} == {(1, (0, 1)): 2, (1, (0, 1, 2)): 3, (2, (0, 1, 2)): 2,
                                                   (4, (0,)): 2, (4, (0, 1)): 2}
    dup = b.select_traces([0, 1, 0])
    with pytest.raises(groups.MergeError, match=r"duplicate run \(trace \d+, run_index 0\)"):
        groups.run_set(dup)


def test_batch_groups_pick_the_deepest_level_set():
    b = experiment()
    order, (first, runs, sizes), levels = groups.batch_groups(b)
    assert sizes.tolist() == [1, 2, 4] and runs.tolist() == [3, 2, 2]
    assert levels == [(0, 1, 2), (0, 1, 2), (0, 1)]
    sel = b.select_traces(order)
    assert sel.trace_batch.tolist() == [1, 1, 1, 2, 2, 4, 4]
    assert sel.n_spans == sum(int(b.trace_span_off[t + 1] - b.trace_span_off[t]) for t in order)


def test_selected_traces_analyse_like_the_reference():
    from oracle import port, ref
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from parity import compare_tables
    b = experiment()
    order, g, _ = groups.batch_groups(b)
    sel = b.select_traces(order)
    c, t = port.run(sel, groups=g)
    aa, ast = ref.analyze(sel, g[0], g[1])
    compare_tables(sel, t, aa, ast)


def test_ambiguous_run_is_rejected():
    from oracle import port, ref
    gen = ref.Generator()
    gen.emit("overlap")
    b = gen.batch()
    c, _ = port.run(b, analyze=False)
    assert c.n_ambiguities > 0
    with pytest.raises(groups.TraceError, match="ambiguous spans; resolve them first"):
        groups.check_unambiguous(c, b)


@pytest.mark.gpu
def test_grouped_batch_on_gpu(engine, has_ref):
    from oracle import ref
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from parity import compare_tables
    b = experiment()
    order, g, _ = groups.batch_groups(b)
    sel = b.select_traces(order)
    corr, tabs = engine.run_host(sel, groups=g)
    groups.check_unambiguous(corr, sel)
    aa, ast = ref.analyze(sel, g[0], g[1])
    compare_tables(sel, tabs, aa, ast)


def test_leveled_corpus_is_a_valid_chain():
    """synth.leveled_corpus: per model three level sets whose runs the reference
    accepts as one LeveledRunGroup, with the injected overhead recovered."""
    from oracle import ref
    from paper_1908_06869_b200 import synth
    models = synth.make_models(2, seed=3, max_layers=200)
    b, sets = synth.leveled_corpus(models, runs=3)
    for s in sets:
        assert [m for m, _ in s] == [0b001, 0b011, 0b111]
        sub = b.select_traces([t for _, tr in s for t in tr])
        arrays, strings = ref.leveled(sub)
        assert int(arrays["status"][0]) == 0, strings["error"]
        ov = dict(zip(arrays["model_ov_mask"].tolist(), arrays["model_ov_val"].tolist()))
        assert ov[0b010] > 0 and ov[0b100] > 0
