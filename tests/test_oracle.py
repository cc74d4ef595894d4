"""CPU-only: pin the oracles before trusting them.

1. The reference itself, built from its sources (oracle/_ref), passes its own
   acceptance gate (11 criteria, acceptance_main.cpp).
2. The plain-C restatement (oracle/xsp_oracle.c) equals the reference on the
   reference's fixtures, generators, known-answer edge cases and fault cases.
3. The committed golden fixtures (tests/golden) still equal the reference.
"""
import os
import subprocess

import numpy as np
import pytest

import cases
from builders import KERNEL, MLG, MODEL, batch_of
from oracle import port, ref
from parity import compare_correlation, compare_tables

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIXTURES = ["minimal", "resnet-like", "mobilenet-like", "overlap", "async-straggler", "overhead-chain"]


def both(b, groups=None, trim=0.2, noise=0.01):
    corr, tabs = port.run(b, groups=groups, trim=trim, noise=noise)
    ra, rs = ref.correlate(b)
    compare_correlation(b, corr, ra, rs)
    first, runs = (np.arange(b.n_traces), np.ones(b.n_traces)) if groups is None else groups[:2]
    aa, ast = ref.analyze(b, first, runs, trim=trim, noise=noise)
    compare_tables(b, tabs, aa, ast)
    return corr, tabs


def test_reference_acceptance_gate(has_ref):
    exe = os.path.join(ROOT, "oracle", "_ref", "strata_acceptance")
    if not os.path.exists(exe):
        pytest.skip("acceptance binary not built")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all 11 criteria passed" in out.stdout


def test_fixture_sizes(has_ref):
    """test_simprof.cpp:306-314: resnet-like = 234 layers / 293 kernels, 821 spans/run."""
    b = ref.Generator().emit("resnet-like").batch()
    assert b.n_spans == 821
    corr, _ = both(b)
    assert corr.n_layers == 234 and corr.n_kernels == 293


@pytest.mark.parametrize("fixture", FIXTURES)
def test_port_fixtures(has_ref, fixture):
    g = ref.Generator()
    for batch in (1, 2, 4, 8):
        g.emit(fixture, batch=batch)
    both(g.batch())


def test_port_repetitions(has_ref):
    g = ref.Generator()
    for r in range(10):
        g.emit("resnet-like", batch=4, run_index=r, jitter_max=1000, jitter_seed=100 + r)
    both(g.batch(), groups=([0], [10], [4]))


@pytest.mark.parametrize("runs", [40, 80])
def test_port_many_repetitions(has_ref, runs):
    """The branches the GPU tests compare the port on (test_gpu_analysis_paths.py):
    more than 32 and more than 64 repetitions per group, pinned to the reference."""
    from paper_1908_06869_b200 import synth
    b, gf, gr, gb = synth.c3(runs=runs, n_models=2, batches=(1, 8), seed=runs, min_layers=20, max_layers=40)
    both(b, groups=(gf, gr, gb))


def test_port_durations_beyond_32_bits(has_ref):
    """Execution durations above 2^32 ns and occupancies unsorted across runs."""
    from paper_1908_06869_b200 import _capi as capi
    from paper_1908_06869_b200 import synth
    b, gf, gr, gb = synth.c3(runs=20, n_models=2, batches=(1, 4), seed=5, min_layers=20, max_layers=60)
    rng = np.random.default_rng(9)
    execs = np.nonzero(((b.flags >> 2) & 3) == capi.KIND_EXEC)[0]
    big = rng.choice(execs, size=execs.size // 4, replace=False)
    b.end_ns[big] += np.uint64(1) << np.uint64(33)
    b.occupancy[:] = rng.random(b.occupancy.size)
    both(b, groups=(gf, gr, gb))


def test_port_trim_fractions(has_ref):
    g = ref.Generator()
    for r in range(7):
        g.emit("mobilenet-like", batch=2, run_index=r, jitter_max=5000, jitter_seed=r)
    b = g.batch()
    for trim in (0.0, 0.1, 0.3, 0.49):
        both(b, groups=([0], [7], [2]), trim=trim)
    both(b, groups=([0], [7], [2]), trim=0.5)  # invalid -> AnalysisError


def test_port_random_nested(has_ref):
    g = ref.Generator()
    for i in range(40):
        g.random_nested(99, 20 + 37 * i)
    for frac in (0.0, 1.0):
        g.random_nested(5, 3000, frac)
    b = g.batch()
    corr, _ = port.run(b, analyze=False)
    ra, rs = ref.correlate(b)
    compare_correlation(b, corr, ra, rs)


def test_port_async(has_ref):
    g = ref.Generator().random_async(7, 5000).random_async(15, 500)
    both(g.batch())


@pytest.mark.parametrize("case", ["nesting", "layer_attrs", "explicit_beats_containment",
                                  "overlapping_layers", "orphans", "fusion", "unmatched_async",
                                  "mixed_orphan_order", "max_end", "max_end_orphan",
                                  "model_span_id_shared"])
def test_port_edge_cases(has_ref, case):
    both(batch_of([getattr(cases, case)()]))


def test_port_faults(has_ref):
    traces = [cases.nesting(), cases.dup_launch_cid(), cases.fusion(), cases.dup_exec_cid(),
              cases.no_model(), cases.two_models(), cases.skip_level(), []]
    levels = [MLG] * len(traces)
    levels[6] = (1 << MODEL) | (1 << KERNEL)
    b = batch_of(traces, levels=levels)
    corr, _ = port.run(b, analyze=False)
    ra, rs = ref.correlate(b)
    compare_correlation(b, corr, ra, rs)
    assert list(corr.trace_status) == [0, 5, 0, 4, 1, 2, 3, 1]


def test_trimmed_mean_known_answers(has_ref):
    """trimmed_mean vs the sort-slice restatement (test_support.hpp:44-51)."""
    rng = np.random.default_rng(2026)
    for _ in range(200):
        v = rng.uniform(-1e6, 1e6, size=int(rng.integers(1, 40)))
        f = float(rng.uniform(0, 0.4999))
        s = np.sort(v)
        drop = int(np.floor(f * len(v)))
        acc = 0.0
        for x in s[drop:len(v) - drop]:
            acc += float(x)
        assert ref.trimmed_mean(v, f) == acc / (len(v) - 2 * drop)


def _golden_files():
    gdir = os.path.join(ROOT, "tests", "golden")
    files = sorted(os.path.join(gdir, f) for f in os.listdir(gdir) if f.endswith(".npz"))
    assert files, "no golden fixtures committed"
    return files


def test_golden_fixtures_match_reference(has_ref):
    """The committed vectors are still what the reference produces."""
    from golden_io import load_golden
    for f in _golden_files():
        b, (ca, cs), (aa, ast), groups = load_golden(f)
        ra, rs = ref.correlate(b)
        for k in ca:
            np.testing.assert_array_equal(ra[k], ca[k], err_msg=f"{f}:{k}")
        assert rs == cs
        ra2, rs2 = ref.analyze(b, groups[0], groups[1])
        for k in aa:
            np.testing.assert_array_equal(ra2[k], aa[k], err_msg=f"{f}:{k}")


def test_golden_fixtures_match_port():
    """Runs without the reference: the committed vectors pin the C port."""
    from golden_io import load_golden
    for f in _golden_files():
        b, (ca, cs), (aa, ast), groups = load_golden(f)
        corr, tabs = port.run(b, groups=groups)
        compare_correlation(b, corr, ca, cs)
        compare_tables(b, tabs, aa, ast)
