"""Every branch of the device trimmed mean (csrc/analyze.cu) against the C oracle
and the reference itself, bit for bit: register sorting networks of 8 / 16 / 32
samples, the local-memory fallback for 33..64 repetitions, the selection path
above 64, the exact-integer path for durations below 2^32 and the double path
above it, and occupancies that are unsorted across repetitions (the sort cannot
be skipped). The port is pinned to the reference on the same inputs in
tests/test_oracle.py (test_port_many_repetitions, test_port_durations_beyond_32_bits)."""
import numpy as np
import pytest

from oracle import port
from paper_1908_06869_b200 import _capi as capi
from paper_1908_06869_b200 import synth

pytestmark = pytest.mark.gpu


def _same_tables(a, b):
    assert (a.n_groups, a.n_layers, a.n_kernels, a.n_names) == (b.n_groups, b.n_layers, b.n_kernels, b.n_names)
    for k in a.cols:
        x, y = np.asarray(a.cols[k]), np.asarray(b.cols[k])
        assert x.shape == y.shape, k
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), k


def _check(engine, b, groups):
    _, want = port.run(b, groups=groups)
    corr, got = engine.run_host(b, groups=groups)
    _same_tables(got, want)
    from oracle import ref
    if ref.available():
        import parity
        ra, rs = ref.correlate(b)
        parity.compare_correlation(b, corr, ra, rs)
        aa, ast = ref.analyze(b, groups[0], groups[1])
        parity.compare_tables(b, got, aa, ast)


@pytest.mark.parametrize("runs", [3, 12, 20, 40, 80, 130])
def test_repetition_counts(engine, runs):
    b, gf, gr, gb = synth.c3(runs=runs, n_models=2, batches=(1, 8), seed=runs, min_layers=20,
                             max_layers=60 if runs <= 40 else 30)
    _check(engine, b, (gf, gr, gb))


def test_durations_beyond_32_bits_and_unsorted_occupancy(engine):
    b, gf, gr, gb = synth.c3(runs=20, n_models=2, batches=(1, 4), seed=5, min_layers=20, max_layers=60)
    rng = np.random.default_rng(9)
    execs = np.nonzero(((b.flags >> 2) & 3) == capi.KIND_EXEC)[0]
    # stretch a quarter of the executions past 2^32 ns (the kernel-duration path
    # falls back to doubles); execution intervals play no part in containment
    big = rng.choice(execs, size=execs.size // 4, replace=False)
    b.end_ns[big] += np.uint64(1) << np.uint64(33)
    # occupancies that differ between repetitions in random order
    b.occupancy[:] = rng.random(b.occupancy.size)
    _check(engine, b, (gf, gr, gb))
