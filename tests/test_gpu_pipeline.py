"""The chunked host pipeline behind xsp_run_host (csrc/pipeline.cu): batches cut
at group boundaries, H2D / compute / D2H overlapped on two streams, chunk
results re-based into the global columns. Results must be byte-identical to a
single-shot run and to the reference."""
import numpy as np
import pytest

import cases
from builders import KERNEL, MLG, MODEL, batch_of
from oracle import ref
from paper_1908_06869_b200 import synth
from parity import compare_correlation, compare_tables

pytestmark = pytest.mark.gpu


def _same(a, b, what):
    assert set(a) == set(b), what
    for k in a:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        assert x.dtype == y.dtype and x.shape == y.shape, (what, k, x.shape, y.shape)
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), (what, k)


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("chunks", [2, 7])
def test_chunked_equals_single_shot(engine, monkeypatch, chunks, pinned):
    """pinned: page-locked inputs, span_id read in place (zero-copy) by the chunks."""
    b, gf, gr, gb = synth.c3(runs=3, n_models=6, batches=(1, 4, 16), seed=11)
    monkeypatch.setenv("XSP_CHUNK_SPANS", "0")
    c1, t1 = engine.run_host(b, groups=(gf, gr, gb))
    monkeypatch.setenv("XSP_CHUNK_SPANS", str(b.n_spans // chunks))
    c2, t2 = engine.run_host(b.pinned() if pinned else b, groups=(gf, gr, gb))
    for k in ("n_traces", "n_failed", "n_layers", "n_kernels", "n_orphans", "n_ambiguities", "n_candidates"):
        assert getattr(c1, k) == getattr(c2, k), k
    _same(c1.cols, c2.cols, "corr")
    assert (t1.n_groups, t1.n_layers, t1.n_kernels, t1.n_names) == (t2.n_groups, t2.n_layers, t2.n_kernels,
                                                                    t2.n_names)
    _same(t1.cols, t2.cols, "tables")
    h2d, d2h = engine.transfer_bytes()
    assert h2d >= b.nbytes_inputs() - (b.span_id.nbytes if pinned else 0)


@pytest.mark.parametrize("pinned", [False, True])
def test_chunked_edge_cases_match_reference(engine, has_ref, monkeypatch, pinned):
    """Orphans, ambiguities, fused launches and per-trace faults spread over
    many tiny chunks: every re-based row / offset must still match the reference.
    pinned: span_id read zero-copy except in chunks with explicit-parent kernels."""
    traces = [cases.nesting(), cases.dup_launch_cid(), cases.fusion(), cases.dup_exec_cid(),
              cases.no_model(), cases.two_models(), cases.skip_level(), cases.orphans(),
              cases.overlapping_layers(), cases.unmatched_async(), cases.mixed_orphan_order(),
              cases.explicit_beats_containment(), cases.layer_attrs()] * 3
    levels = [MLG] * len(traces)
    for i in range(6, len(traces), 13):
        levels[i] = (1 << MODEL) | (1 << KERNEL)
    b = batch_of(traces, levels=levels)
    monkeypatch.setenv("XSP_CHUNK_SPANS", "12")
    corr, tabs = engine.run_host(b.pinned() if pinned else b)
    ra, rs = ref.correlate(b)
    compare_correlation(b, corr, ra, rs)
    aa, ast = ref.analyze(b, np.arange(b.n_traces), np.ones(b.n_traces))
    compare_tables(b, tabs, aa, ast)
