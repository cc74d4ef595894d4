"""Time-range sharding of one long trace (paper_1908_06869_b200/timeshard.py,
SURVEY 8(e), BASELINE config 4).

CPU tests compute every shard with the C oracle port (the product needs a GPU)
and check the combined result against the UNSHARDED oracle result on the same
C4-shaped trace: every correlation column and table column bit-exact, except
the occupancy-weighted sums sum(occ*lat) / sum(lat) of a10 and a15, which are
re-associated across shards and checked to 1e-12 relative (north star: 1e-9
for derived fp64 ratios). world_size 2 also runs over gloo with the byte-tensor
all_gather the GPUs use over NCCL. The GPU test uses the CUDA engine per shard
and compares with the reference itself."""
import os
import socket

import numpy as np
import pytest

from paper_1908_06869_b200 import synth, timeshard

APPROX = {"m_occ", "n_occ"}


def c4_small(layers=4000, block=400, seed=4):
    return synth.c4(n_layers=layers, drain_every=block, seed=seed, concurrent_frac=0.0)


def oracle_compute(sub):
    from oracle import port
    return port.run(sub)


def assert_corr_equal(a, b):
    assert a.n_layers == b.n_layers and a.n_kernels == b.n_kernels
    assert a.n_orphans == b.n_orphans and a.n_ambiguities == b.n_ambiguities
    for k in b.cols:
        x, y = np.asarray(a.cols[k]), np.asarray(b.cols[k])
        assert x.shape == y.shape and np.array_equal(x.astype(np.int64), y.astype(np.int64)) \
            if x.dtype.kind in "iu" else np.array_equal(x.view(np.uint8), y.view(np.uint8)), k


def assert_tables_equal(a, b, rtol=1e-12):
    assert (a.n_layers, a.n_kernels, a.n_names) == (b.n_layers, b.n_kernels, b.n_names)
    for k in b.cols:
        x, y = np.asarray(a.cols[k]), np.asarray(b.cols[k])
        assert x.dtype == y.dtype and x.shape == y.shape, k
        if k in APPROX:
            np.testing.assert_allclose(x, y, rtol=rtol, atol=0, err_msg=k)
        else:
            assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), k


def test_cuts_are_quiescent():
    b = c4_small()
    cuts = timeshard.quiescent_cuts(b)
    assert cuts.size >= 9  # one per synchronisation block
    lvl = b.flags & 3
    for c in cuts[:20]:
        assert lvl[c] == 1
        before = (lvl[:c] == 1)
        if before.any():
            assert b.end_ns[:c][before].max() < b.begin_ns[c]
    starts = timeshard.choose_cuts(cuts, b.n_spans, 4)
    assert len(starts) == 4 and starts == sorted(set(starts))


@pytest.mark.parametrize("world", [1, 2, 3, 7])
def test_in_process_matches_unsharded(world):
    from oracle import port
    b = c4_small()
    whole_c, whole_t = port.run(b)
    starts = timeshard.choose_cuts(timeshard.quiescent_cuts(b), b.n_spans, world)
    assert len(starts) == world
    bounds = starts + [b.n_spans]
    parts = []
    for r in range(len(starts)):
        rows = timeshard.shard_rows(b, bounds[r], bounds[r + 1])
        sub, mrows, arows = timeshard.sub_batch(b, rows)
        c, t = oracle_compute(sub)
        parts.append({"rows": rows, "mrows": mrows, "arows": arows, "corr": c, "tabs": t})
    corr, tabs = timeshard.combine(b, parts)
    assert_corr_equal(corr, whole_c)
    assert_tables_equal(tabs, whole_t)


def test_orphans_and_stragglers_across_shards():
    """Orphans of every phase in several shards come back in the reference order."""
    from oracle import port
    b = c4_small(layers=3000, block=300, seed=9)
    rng = np.random.default_rng(2)
    f = b.flags.copy()
    kind = (f >> 2) & 3
    ex = np.nonzero(kind == 2)[0]
    la = np.nonzero(kind == 1)[0]
    f[rng.choice(ex, 30, replace=False)] &= ~np.uint8(0x20)   # exec without cid
    f[rng.choice(la, 30, replace=False)] &= ~np.uint8(0x20)   # launch without cid
    b.flags = f
    whole_c, whole_t = port.run(b)
    assert whole_c.n_orphans >= 60
    starts = timeshard.choose_cuts(timeshard.quiescent_cuts(b), b.n_spans, 4)
    bounds = starts + [b.n_spans]
    parts = []
    for r in range(len(starts)):
        rows = timeshard.shard_rows(b, bounds[r], bounds[r + 1])
        sub, mrows, arows = timeshard.sub_batch(b, rows)
        c, t = oracle_compute(sub)
        parts.append({"rows": rows, "mrows": mrows, "arows": arows, "corr": c, "tabs": t})
    corr, tabs = timeshard.combine(b, parts)
    assert_corr_equal(corr, whole_c)
    assert_tables_equal(tabs, whole_t)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port_, out):
    import pickle
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = timeshard.run_time_sharded(c4_small(), oracle_compute, rank, world, dist=dist, device="cpu")
        if rank == 0:
            with open(out, "wb") as fh:
                pickle.dump(res, fh)
    finally:
        dist.destroy_process_group()


def test_gloo_world2(tmp_path):
    import pickle
    import torch.multiprocessing as mp
    from oracle import port
    out = str(tmp_path / "ts.pkl")
    mp.start_processes(_rank_main, args=(2, _free_port(), out), nprocs=2, start_method="spawn", join=True)
    with open(out, "rb") as fh:
        corr, tabs, starts = pickle.load(fh)
    assert len(starts) == 2
    whole_c, whole_t = port.run(c4_small())
    assert_corr_equal(corr, whole_c)
    assert_tables_equal(tabs, whole_t)


@pytest.mark.gpu
def test_gpu_shards_match_reference(engine, has_ref):
    """CUDA engine per shard (4 simulated ranks, one GPU) against the reference."""
    from oracle import ref
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from parity import compare_correlation, compare_tables
    b = c4_small(layers=20000, block=1000, seed=5)
    starts = timeshard.choose_cuts(timeshard.quiescent_cuts(b), b.n_spans, 4)
    bounds = starts + [b.n_spans]
    parts = []
    for r in range(len(starts)):
        rows = timeshard.shard_rows(b, bounds[r], bounds[r + 1])
        sub, mrows, arows = timeshard.sub_batch(b, rows)
        c, t = engine.run_host(sub)
        parts.append({"rows": rows, "mrows": mrows, "arows": arows, "corr": c, "tabs": t})
    corr, tabs = timeshard.combine(b, parts)
    whole_c, whole_t = engine.run_host(b)
    assert_corr_equal(corr, whole_c)
    assert_tables_equal(tabs, whole_t)
    ra, rs = ref.correlate(b)
    compare_correlation(b, corr, ra, rs)


@pytest.mark.gpu
def test_gpu_long_group_vs_reference(engine, has_ref):
    """One trace with > 65536 kernels takes the long-group path (chunked model and
    name folds): everything bit-exact against the reference except the
    occupancy-weighted ratios (re-associated at chunk boundaries, 1e-12)."""
    from oracle import ref
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from parity import compare_correlation, compare_tables
    b = c4_small(layers=40000, block=2000, seed=8)
    corr, tabs = engine.run_host(b)
    assert tabs.n_kernels > 65536
    ra, rs = ref.correlate(b)
    compare_correlation(b, corr, ra, rs)
    aa, ast = ref.analyze(b, [0], [1])
    compare_tables(b, tabs, aa, ast, rtol=1e-12)
    # integer-valued latency sums stay bit-exact
    assert tabs.m_kern_lat[0] == aa["m_kern_lat"][0] and tabs.m_gpu[0] == aa["m_gpu"][0]
