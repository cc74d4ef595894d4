"""Full-size GPU checks (BASELINE configs 3 and 4) through size-independent
properties — the reference cannot hold these corpora in RAM at once — plus
exact parity against the reference on a random sample of C3's groups.

C3: 65 models x 8 batches x 20 iterations = 47.75 M spans (the bench workload).
C4: one long trace (synth.c4), 5 M layers = 38 M spans (the bench runs 28.6 M
layers; the properties do not depend on the size).
"""
import numpy as np
import pytest

from paper_1908_06869_b200 import synth

pytestmark = pytest.mark.gpu


def _roles(b):
    lvl, kind = b.flags & 3, (b.flags >> 2) & 3
    return lvl, kind


def _check_correlation_properties(b, corr):
    lvl, kind = _roles(b)
    layers = np.nonzero((lvl == 1) & (kind == 0))[0]
    launches = np.nonzero((lvl >= 2) & (kind == 1))[0]
    assert corr.n_failed == 0 and corr.n_orphans == 0 and corr.n_ambiguities == 0
    assert corr.n_layers == layers.size and corr.n_kernels == launches.size
    # every placed layer once, in timeline (= layer_index) order per trace
    assert np.array_equal(np.sort(corr.layer_row.astype(np.int64)), layers)
    # kernels: every launch once; its exec carries the same cid; the exec is an exec span
    kl = corr.kernel_launch_row.astype(np.int64)
    ke = corr.kernel_exec_row.astype(np.int64)
    assert np.array_equal(np.sort(kl), launches)
    assert np.array_equal(b.cid[kl], b.cid[ke])
    assert np.all(kind[ke] == 2)
    # CSR: each kernel's launch lies inside its layer's interval (closed containment)
    koff = corr.layer_kernel_off.astype(np.int64)
    assert koff[0] == 0 and koff[-1] == corr.n_kernels and np.all(np.diff(koff) >= 0)
    layer_of_k = np.repeat(np.arange(corr.n_layers), np.diff(koff))
    lr = corr.layer_row.astype(np.int64)[layer_of_k]
    assert np.all(b.begin_ns[lr] <= b.begin_ns[kl]) and np.all(b.end_ns[kl] <= b.end_ns[lr])
    # kernel durations and names come from the exec span
    assert np.array_equal(corr.kernel_dur, b.end_ns[ke] - b.begin_ns[ke])
    assert np.array_equal(corr.kernel_name, b.name_id[ke])
    return kl, ke


def test_c3_full_properties_and_sampled_parity(engine, has_ref):
    from oracle import ref
    import os
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from parity import compare_tables
    b, gf, gr, gb = synth.c3()
    assert b.n_spans > 47_000_000
    corr, tabs = engine.run_host(b, groups=(gf, gr, gb))
    _check_correlation_properties(b, corr)
    # analysis totals: u64 counters are exact sums of the first run's kernels
    G = len(gf)
    assert np.all(tabs.group_status == 0)
    goff = tabs.group_kernel_off.astype(np.int64)
    assert np.array_equal(tabs.m_count, np.diff(goff).astype(np.uint64))
    fl = tabs.k_flops.astype(np.uint64)
    sums = np.add.reduceat(fl, goff[:-1]) if tabs.n_kernels else np.zeros(G, np.uint64)
    assert np.array_equal(tabs.m_flops, sums)
    noff = tabs.group_name_off.astype(np.int64)
    ncount = np.add.reduceat(tabs.n_count.astype(np.uint64), noff[:-1])
    assert np.array_equal(ncount, np.diff(goff).astype(np.uint64))
    # a10 order: total latency descending within every group
    for g in range(0, G, 37):
        lat = tabs.n_lat[noff[g]:noff[g + 1]]
        assert np.all(np.diff(lat) <= 0)
    # exact parity with the reference on a random sample of groups
    rng = np.random.default_rng(12)
    for g in rng.choice(G, size=3, replace=False):
        t0, t1 = int(gf[g]), int(gf[g] + gr[g])
        sub = b.trace_slice(t0, t1)
        c2, t2 = engine.run_host(sub, groups=([0], [t1 - t0], [int(gb[g])]))
        aa, ast = ref.analyze(sub, [0], [t1 - t0])
        compare_tables(sub, t2, aa, ast)
        # and the full-batch tables of that group equal the per-group run bit for bit
        k0, k1 = int(goff[g]), int(goff[g + 1])
        assert np.array_equal(tabs.k_lat[k0:k1].view(np.uint64), t2.k_lat.view(np.uint64))
        assert tabs.m_lat[g] == t2.m_lat[0] and tabs.m_occ[g] == t2.m_occ[0]


def test_c4_long_trace_properties(engine):
    b = synth.c4(n_layers=5_000_000)
    assert b.n_spans > 35_000_000
    corr, tabs = engine.run_host(b)
    kl, ke = _check_correlation_properties(b, corr)
    # one run: integer latencies, so the model's kernel latency is the exact sum
    dur = (b.end_ns[ke] - b.begin_ns[ke]).astype(np.uint64)
    assert tabs.m_kern_lat[0] == float(int(dur.sum()))
    assert tabs.m_count[0] == corr.n_kernels
    lvl, kind = _roles(b)
    metric_rows = np.cumsum((b.flags & 0x40) != 0) - 1
    assert tabs.m_flops[0] == np.uint64(int(b.flops[metric_rows[ke]].astype(np.uint64).sum()))
    # a10 rows: every kernel counted once
    assert int(tabs.n_count.sum()) == corr.n_kernels
    # time-range shards agree with the single-GPU run
    from paper_1908_06869_b200 import timeshard
    starts = timeshard.choose_cuts(timeshard.quiescent_cuts(b), b.n_spans, 3)
    assert len(starts) == 3
