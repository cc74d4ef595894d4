"""Packed host input (csrc/packed.cu, xsp_pack_host + xsp_run_host_packed): the
span columns cross PCIe as u32 deltas / durations / cid offsets with sparse
parent and cid lists and an escape list, and are rebuilt on the device. The
results must equal xsp_run_host's bit for bit — single-shot and chunked
pipeline, with escapes of every kind (trace / block starts, long durations,
wide cid ranges, backward begins) — and the wire bytes must shrink."""
import numpy as np
import pytest

from paper_1908_06869_b200 import synth

pytestmark = pytest.mark.gpu


def same(a, b):
    for k in b.cols:
        x, y = np.asarray(a.cols[k]), np.asarray(b.cols[k])
        assert x.shape == y.shape and np.array_equal(x.view(np.uint8), y.view(np.uint8)), k


def run_both(engine, b, groups, chunk=None, monkeypatch=None):
    if chunk is not None:
        monkeypatch.setenv("XSP_CHUNK_SPANS", str(chunk))
    c0, t0 = engine.run_host(b, groups=groups)
    h0, _ = engine.transfer_bytes()
    pk = engine.pack_host(b)
    c1, t1 = engine.run_host_packed(pk, b, groups=groups)
    h1, _ = engine.transfer_bytes()
    same(c1, c0)
    same(t1, t0)
    return h0, h1


@pytest.mark.parametrize("chunk", [None, 50_000])
def test_packed_equals_dense_c3(engine, monkeypatch, chunk):
    b, gf, gr, gb = synth.c3(runs=3, n_models=6, max_layers=400)
    h0, h1 = run_both(engine, b, (gf, gr, gb), chunk if chunk else 0, monkeypatch)
    assert h1 < 0.8 * h0, (h0, h1)


def test_packed_escapes(engine, monkeypatch):
    """Long durations, cids far apart, backward begins inside a trace (an
    out-of-order bundle is rejected the same way by both paths)."""
    from oracle import ref
    g = ref.Generator()
    for r in range(4):
        g.emit("resnet-like", batch=2, run_index=r, jitter_max=2000, jitter_seed=r + 3)
    g.random_nested(5, 2500).random_async(6, 300)
    b = g.batch()
    # cids spread over 2^40 within blocks; a few layers last > 2^32 ns
    has = (b.flags & 0x20) != 0
    b.cid = np.where(has, b.cid * np.uint64(1 << 20) + np.uint64(7), b.cid).astype(np.uint64)
    lay = np.nonzero((b.flags & 3) == 1)[0][::17]
    b.end_ns = b.end_ns.copy()
    b.end_ns[lay] += np.uint64(5 << 32)
    T = b.n_traces
    run_both(engine, b, (np.arange(T), np.ones(T), b.trace_batch), 0, monkeypatch)
    run_both(engine, b, (np.arange(T), np.ones(T), b.trace_batch), 3000, monkeypatch)


@pytest.mark.parametrize("chunk", [0, 50_000])
def test_host_outputs_rows_only(engine, monkeypatch, chunk):
    """XSP_HOST_OUT_ROWS: the four lookup columns stay on the device (NULL in
    the host result, fewer D2H bytes); every other column is unchanged and the
    lookups rebuilt from the span columns (engine.fill_lookups) equal the
    device's."""
    from paper_1908_06869_b200 import _capi as capi
    from paper_1908_06869_b200.engine import fill_lookups
    monkeypatch.setenv("XSP_CHUNK_SPANS", str(chunk))
    b, gf, gr, gb = synth.c3(runs=3, n_models=6, max_layers=400)
    pk = engine.pack_host(b)
    c0, t0 = engine.run_host_packed(pk, b, groups=(gf, gr, gb))
    _, d0 = engine.transfer_bytes()
    try:
        engine.set_host_outputs(capi.HOST_OUT_ROWS)
        co, _ = engine.run_host_packed(pk, b, groups=(gf, gr, gb), raw=True)
        assert not co.kernel_dur and not co.kernel_name and not co.kernel_occ and not co.layer_dur
        c1, t1 = engine.run_host_packed(pk, b, groups=(gf, gr, gb))
        _, d1 = engine.transfer_bytes()
        c2, _ = engine.run_host(b, groups=(gf, gr, gb))
    finally:
        engine.set_host_outputs(capi.HOST_OUT_ALL)
    lookups = ("layer_dur", "kernel_dur", "kernel_name", "kernel_occ")
    for k in lookups:
        assert c1.cols[k].size == 0 and c2.cols[k].size == 0, k
    skip = lambda c: type(c)(c.n_traces, c.n_failed, {k: v for k, v in c.cols.items() if k not in lookups})  # noqa
    same(skip(c1), skip(c0))
    same(skip(c2), skip(c0))
    same(t1, t0)
    kb = c0.n_kernels * 20 + c0.n_layers * 8
    assert d0 - d1 == kb, (d0, d1, kb)
    fill_lookups(c1, b)
    same(c1, c0)
    with pytest.raises(capi.XspError):
        engine.set_host_outputs(7)


def _bw_decode(col, n):
    """include/xsp.h xsp_bw_col, decoded with numpy (the wire format as documented)."""
    import ctypes as C
    nb = (n + 255) // 256
    w = np.ctypeslib.as_array(col.width, shape=(nb,)).copy()
    off = np.ctypeslib.as_array(col.boff, shape=(nb + 1,)).copy()
    data = np.frombuffer((C.c_uint8 * int(off[-1] + 8)).from_address(C.cast(col.data, C.c_void_p).value),
                         dtype=np.uint8)
    out = np.zeros(n, dtype=np.uint64)
    for b in range(nb):
        r0, r1 = b * 256, min(n, b * 256 + 256)
        wb = int(w[b])
        if wb:
            raw = data[off[b]:off[b] + wb * (r1 - r0)].reshape(r1 - r0, wb).astype(np.uint64)
            out[r0:r1] = (raw << (np.arange(wb, dtype=np.uint64) * np.uint64(8))).sum(axis=1, dtype=np.uint64)
    if col.base:
        base = np.ctypeslib.as_array(col.base, shape=(nb,)).copy()
        out += np.repeat(base, 256)[:n]
    return out


def test_packed_tables_wire_format(engine, monkeypatch):
    """The coded name / metric / layer columns decode (numpy, per the header's
    description) to the host columns; edge values: all-zero blocks (width 0),
    full 64-bit counters, negative alloc_bytes (two's complement), more than
    65536 distinct occupancies (dictionary off -> raw), and the device decode
    equals the raw upload bit for bit."""
    b, gf, gr, gb = synth.c3(runs=3, n_models=6, max_layers=400)
    b.flops = b.flops.copy()
    b.flops[:300] = 0
    b.flops[700] = np.uint64(0xFFFFFFFFFFFFFFFF)
    b.alloc_bytes = b.alloc_bytes.copy()
    b.alloc_bytes[5] = -12345
    pk = engine.pack_host(b)
    assert np.array_equal(_bw_decode(pk.name_bw, b.n_spans), b.name_id.astype(np.uint64))
    m, l_ = len(b.flops), len(b.alloc_bytes)
    assert np.array_equal(_bw_decode(pk.flops_bw, m), b.flops)
    assert np.array_equal(_bw_decode(pk.read_bw, m), b.dram_read)
    assert np.array_equal(_bw_decode(pk.write_bw, m), b.dram_write)
    assert np.array_equal(_bw_decode(pk.alloc_bw, l_).view(np.int64), b.alloc_bytes)
    assert np.array_equal(_bw_decode(pk.type_bw, l_), b.type_id.astype(np.uint64))
    assert pk.flops_bw.width[0] == 0
    # the u32 delta lists travel + 1 (the escape code wraps to 0)
    n, nc = b.n_spans, int(pk.n_cid)
    for bw, raw, cnt in ((pk.dbegin_bw, pk.dbegin, n), (pk.dur_bw, pk.dur, n), (pk.dcid_bw, pk.dcid, nc)):
        dec = (_bw_decode(bw, cnt) - np.uint64(1)).astype(np.uint32)
        assert np.array_equal(dec, np.ctypeslib.as_array(raw, shape=(cnt,))), cnt
    # per-block prefix counts of metric rows, layer rows, non-layer explicit parents
    nb = int(pk.n_blocks)
    f = b.flags
    lay = (f & 3) == 1
    for arr, pred in ((pk.blk_met0, (f & 0x40) != 0), (pk.blk_lay0, lay), (pk.blk_cpar0, ~lay & ((f & 0x10) != 0))):
        want = np.concatenate([[0], np.cumsum(pred)])[np.minimum(np.arange(nb + 1) * 256, n)]
        assert np.array_equal(np.ctypeslib.as_array(arr, shape=(nb + 1,)), want.astype(np.uint32))
    npar = int(pk.n_parent)
    assert pk.parent_bw.base and np.array_equal(_bw_decode(pk.parent_bw, npar),
                                                np.ctypeslib.as_array(pk.parent, shape=(npar,)))
    assert 0 < pk.occ_dict_n <= 256 and pk.occ_idx_bytes == 1
    d = np.ctypeslib.as_array(pk.occ_dict, shape=(pk.occ_dict_n,))
    ix = np.ctypeslib.as_array(pk.occ_idx, shape=(m,))
    assert np.array_equal(d[ix].view(np.uint64), b.occupancy.view(np.uint64))
    for chunk in (0, 40_000):
        run_both(engine, b, (gf, gr, gb), chunk, monkeypatch)
    # many distinct occupancies: raw fallback, still equal
    b.occupancy = np.random.default_rng(5).random(m)
    pk = engine.pack_host(b)
    assert pk.occ_dict_n == (0 if m > 65536 else pk.occ_dict_n)
    run_both(engine, b, (gf, gr, gb), 40_000, monkeypatch)


@pytest.mark.parametrize("chunk", [0, 50_000])
def test_packed_tables_off(engine, monkeypatch, chunk):
    """XSP_PACK_TABLES=0: name_id and the tables travel raw; results equal, and
    the coded form moves fewer bytes."""
    b, gf, gr, gb = synth.c3(runs=3, n_models=6, max_layers=400)
    h_coded = run_both(engine, b, (gf, gr, gb), chunk, monkeypatch)[1]
    monkeypatch.setenv("XSP_PACK_TABLES", "0")
    pk = engine.pack_host(b)
    assert not pk.name_bw.width and not pk.flops_bw.width and pk.occ_dict_n == 0 and not pk.dbegin_bw.width
    h_raw = run_both(engine, b, (gf, gr, gb), chunk, monkeypatch)[1]
    assert h_coded < h_raw, (h_coded, h_raw)


@pytest.mark.parametrize("model", ["minimal", "overlap", "async-straggler"])
def test_packed_small_reference_bundles(engine, monkeypatch, model):
    """Tiny bundles of the reference's generator models (one block or less,
    few or no metric rows) through both packed paths."""
    from oracle import ref
    b = ref.Generator().emit(model).batch()
    T = b.n_traces
    run_both(engine, b, (np.arange(T), np.ones(T), b.trace_batch), 0, monkeypatch)
