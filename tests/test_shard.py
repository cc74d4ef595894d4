"""Multi-rank sharding of correlate + analyze (paper_1908_06869_b200/shard.py).

CPU tests: world_size 2 over gloo, each rank computing its share with the C
oracle (the product needs a GPU); rank 0's gathered tables must equal the
unsharded oracle tables bit for bit. The GPU test runs the same path with the
CUDA engine as the per-rank compute (world_size 1 and 2 simulated in-process).
"""
import os
import socket

import numpy as np
import pytest

from paper_1908_06869_b200 import shard, synth


def _corpus():
    return synth.c3(runs=3, n_models=5, batches=(1, 4, 32), seed=7)


def _tables_equal(a, b):
    assert a.n_groups == b.n_groups
    assert set(a.cols) == set(b.cols)
    for k in a.cols:
        x, y = np.asarray(a.cols[k]), np.asarray(b.cols[k])
        assert x.dtype == y.dtype and x.shape == y.shape, k
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), k


def _oracle_compute(sub, groups):
    from oracle import port
    return port.run(sub, groups=groups)[1]


def test_assign_groups_covers_and_balances():
    rng = np.random.default_rng(3)
    w = rng.integers(1, 10_000, size=97)
    for world in (1, 2, 3, 8):
        r = shard.assign_groups(w, world)
        assert r.shape == w.shape and r.min() >= 0 and r.max() < world
        load = np.bincount(r, weights=w, minlength=world)
        assert load.sum() == w.sum()
        # LPT bound: max load <= mean + largest item
        assert load.max() <= w.sum() / world + w.max()
    assert np.array_equal(shard.assign_groups(w, 4), shard.assign_groups(w, 4))  # deterministic


def test_shard_single_process_matches_unsharded():
    b, gf, gr, gb = _corpus()
    groups = (gf, gr, gb)
    whole = _oracle_compute(b, groups)
    for world in (2, 3):
        ranks = shard.assign_groups(shard.group_spans(b, groups), world)
        parts = []
        for r in range(world):
            sub, lg, gids, base = shard.shard(b, groups, ranks, r)
            if sub is None:
                continue
            t = _oracle_compute(sub, lg)
            t.cols["l_row"] = shard._local_to_global_rows(t.cols["l_row"], sub, base)
            parts.append((t, gids))
        _tables_equal(shard.combine(parts, len(gf), 3), whole)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, gf, gr, gb = _corpus()
        tabs = shard.run_sharded(b, (gf, gr, gb), _oracle_compute, rank, world, dist=dist)
        if rank == 0:
            np.savez(out, n_groups=tabs.n_groups, **tabs.cols)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_gloo_world2_matches_unsharded(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "rank0.npz")
    mp.spawn(_rank_main, args=(2, _free_port(), out), nprocs=2, join=True)
    b, gf, gr, gb = _corpus()
    whole = _oracle_compute(b, (gf, gr, gb))
    z = np.load(out)
    from paper_1908_06869_b200.engine import Tables
    got = Tables(int(z["n_groups"]), {k: z[k] for k in z.files if k != "n_groups"})
    _tables_equal(got, whole)


@pytest.mark.gpu
def test_gpu_sharded_compute_matches_oracle(engine):
    b, gf, gr, gb = _corpus()
    groups = (gf, gr, gb)
    whole = _oracle_compute(b, groups)

    def gpu_compute(sub, g):
        return engine.run_host(sub, groups=g)[1]
    ranks = shard.assign_groups(shard.group_spans(b, groups), 2)
    parts = []
    for r in range(2):
        sub, lg, gids, base = shard.shard(b, groups, ranks, r)
        t = gpu_compute(sub, lg)
        t.cols["l_row"] = shard._local_to_global_rows(t.cols["l_row"], sub, base)
        parts.append((t, gids))
    _tables_equal(shard.combine(parts, len(gf), 3), whole)


@pytest.mark.gpu
def test_gpu_nccl_combine_reorders_groups(engine):
    """xsp_combine_tables over a world-1 NCCL communicator: the rank holds the
    groups in a permuted order (its sub-batch lists their traces in that order);
    the combine lays them out in global group order with l_row rebased to the
    original batch — the unsharded device tables bit for bit."""
    import torch
    from paper_1908_06869_b200.engine import DeviceBatch
    b, gf, gr, gb = synth.c3(runs=3, n_models=5, max_layers=120)
    groups = (gf, gr, gb)
    whole_c, whole_t = engine.run_host(b, groups=groups)
    G = len(gf)
    perm = np.random.default_rng(1).permutation(G)
    ranks = np.zeros(G, np.int64)
    parts, lfirst, bases, t = [], [], [], 0
    for g in perm:
        t0, t1 = int(gf[g]), int(gf[g] + gr[g])
        parts.append(b.trace_slice(t0, t1))
        bases.append(b.trace_span_off[t0:t1].astype(np.int64))
        lfirst.append(t)
        t += t1 - t0
    from paper_1908_06869_b200.columns import SpanBatch
    sub = SpanBatch.concat(parts)
    lgroups = (np.array(lfirst), np.asarray(gr)[perm], np.asarray(gb)[perm])
    engine.comm_init(1, 0)
    dev = DeviceBatch(sub)
    _, to = engine.run_device(dev, lgroups)
    rmap = torch.from_numpy(shard.l_row_map(sub, np.concatenate(bases)).view(np.int32)).cuda()
    out, sent = engine.combine_tables(to, perm, G, rmap.data_ptr())
    torch.cuda.synchronize()
    got = engine.tables_to_host(out)
    assert sent == 0  # rank 0 keeps its own tables
    for k in whole_t.cols:
        x, y = np.asarray(got.cols[k]), np.asarray(whole_t.cols[k])
        assert x.shape == y.shape and np.array_equal(x.view(np.uint8), y.view(np.uint8)), k
    del ranks
