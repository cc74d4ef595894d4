"""Synthetic trace corpora at scale, vectorized (numpy).

The timeline follows the reference simulator's plan (simprof.cpp:203-343):
sequential layers starting at the run epoch (1000 ns), kernel launches packed
from the layer begin, each execution starting at max(device cursor, launch end)
on one device stream, correlation ids restarting at 1 per run, span ids in
record order (model, then per layer: layer, then launch/exec pairs), batch
scaling round(v * b^e) with exponents 0.9 / 1.0 / 1.0 (simprof.cpp:36-42), and
layers carrying their model span as explicit parent. Jitter stretches layer
bodies and executions by U[0, J] ns. The result is already in timeline order
(begin_ns, rank, span_id), i.e. a valid TraceBundle per trace.

Used by bench.py (C3: 65 models x 8 batch sizes x R iterations) and by tests.
Parity never depends on this generator matching simprof bit for bit: every
corpus is fed identically to the product and to the oracles.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

from . import _capi as capi
from .columns import SpanBatch

TYPES = ["Add", "Conv2D", "Mul", "Relu"]
KERNEL_VOCAB = [
    "volta_scudnn_128x64_relu_interior_nn_v1", "volta_scudnn_128x128_stridedB", "volta_sgemm_64x32",
    "volta_sgemm_128x64_nn", "winograd_kernel", "implicit_convolve_sgemm", "offset_kernel",
    "elementwise_add_kernel", "elementwise_mul_kernel", "relu_kernel", "bias_add_kernel",
    "batch_norm_fwd_kernel", "depthwise_conv_kernel", "reduce_mean_kernel", "softmax_kernel",
    "transpose_kernel", "fft2d_r2c_32x32", "fft2d_c2r_32x32", "gemv_kernel", "pooling_fwd_kernel",
    "concat_kernel", "pad_kernel", "cast_kernel", "scale_kernel", "copy_kernel",
    "maxwell_scudnn_winograd_128x128", "splitk_reduce_kernel", "conv2d_grouped_direct_kernel",
    "im2col_kernel", "col2im_kernel",
]
EPOCH_NS = 1000


@dataclass
class Model:
    name: str
    layer_ns: np.ndarray      # [L] host latency at batch 1
    alloc: np.ndarray         # [L]
    ltype: np.ndarray         # [L] index into TYPES
    kcount: np.ndarray        # [L] kernels per layer
    exec_ns: np.ndarray       # [K]
    launch_ns: np.ndarray     # [K]
    kname: np.ndarray         # [K] index into KERNEL_VOCAB
    flops: np.ndarray         # [K]
    dram_r: np.ndarray        # [K]
    dram_w: np.ndarray        # [K]
    occ: np.ndarray           # [K]


def make_models(n_models: int = 65, seed: int = 1, min_layers: int = 100, max_layers: int = 1500,
                max_kernels: int = 4) -> List[Model]:
    """C3 model family: L ~ U[min, max] layers, K ~ U{1..max_kernels} kernels per layer,
    layer types cycling Conv2D/Mul/Add/Relu."""
    rng = np.random.default_rng(seed)
    out = []
    for m in range(n_models):
        L = int(rng.integers(min_layers, max_layers + 1))
        kc = rng.integers(1, max_kernels + 1, L)
        K = int(kc.sum())
        ltype = np.array([[1, 2, 0, 3][i % 4] for i in range(L)], dtype=np.int64)
        out.append(Model(
            name=f"model_{m:02d}",
            layer_ns=rng.integers(300_000, 3_000_000, L),
            alloc=rng.integers(100_000, 30_000_000, L),
            ltype=ltype,
            kcount=kc,
            exec_ns=rng.integers(50_000, 2_000_000, K),
            launch_ns=rng.integers(3_000, 6_001, K),
            kname=rng.integers(0, len(KERNEL_VOCAB), K),
            flops=rng.integers(10_000_000, 10_000_000_000, K),
            dram_r=rng.integers(1_000_000, 100_000_000, K),
            dram_w=rng.integers(1_000_000, 100_000_000, K),
            occ=rng.integers(5, 96, K) / 100.0,
        ))
    return out


def scaled(v: np.ndarray, batch: int, exponent: float) -> np.ndarray:
    """scaled_quantity (simprof.cpp:36-42): round(v * batch^exponent), exact at batch 1."""
    if batch == 1:
        return v.astype(np.int64)
    return np.round(v.astype(np.float64) * float(batch) ** exponent).astype(np.int64)


def corpus(models: Sequence[Model], batches: Sequence[int], runs: int, jitter_ns: int = 1000,
           seed: int = 7) -> Tuple[SpanBatch, np.ndarray, np.ndarray, np.ndarray]:
    """All (model, batch) groups x `runs` iterations as one SpanBatch.

    Returns (batch, group_first_trace, group_runs, group_batch_size)."""
    rng = np.random.default_rng(seed)
    names = sorted({m.name for m in models} |
                   {f"{m.name}/layer{l:04d}/{TYPES[m.ltype[l]]}" for m in models for l in range(m.layer_ns.size)} |
                   set(KERNEL_VOCAB))
    nid = {n: i for i, n in enumerate(names)}
    vocab_ids = np.array([nid[n] for n in KERNEL_VOCAB], dtype=np.uint32)
    parts = {k: [] for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags", "name_id",
                             "flops", "dram_read", "dram_write", "occupancy", "alloc_bytes", "type_id")}
    lens, gfirst, gruns, gbatch, tbatch, trun = [], [], [], [], [], []
    ntr = 0
    for m in models:
        L, K = m.layer_ns.size, m.exec_ns.size
        layer_name_ids = np.array([nid[f"{m.name}/layer{l:04d}/{TYPES[m.ltype[l]]}"] for l in range(L)],
                                  dtype=np.uint32)
        lay_of_k = np.repeat(np.arange(L), m.kcount)
        # record order: model, then per layer [layer, (launch, exec) x K_l]
        first_k = np.concatenate([[0], np.cumsum(m.kcount)[:-1]])
        layer_sid = 2 + np.arange(L) + 2 * first_k
        k_in_layer = np.arange(K) - first_k[lay_of_k]
        launch_sid = layer_sid[lay_of_k] + 1 + 2 * k_in_layer
        exec_sid = launch_sid + 1
        # host sequence H: model, layers and their launches in record order
        nH = 1 + L + K
        h_is_layer = np.zeros(nH, dtype=bool)
        h_layer_pos = 1 + np.arange(L) + first_k  # position of layer l in H
        h_is_layer[h_layer_pos] = True
        h_launch_pos = 1 + lay_of_k + 1 + np.arange(K)  # = layer pos + 1 + k_in_layer
        h_launch_pos = h_layer_pos[lay_of_k] + 1 + k_in_layer
        for b in batches:
            lns = scaled(m.layer_ns, b, 0.9)
            ens = scaled(m.exec_ns, b, 0.9)
            fl = scaled(m.flops, b, 1.0)
            dr = scaled(m.dram_r, b, 1.0)
            dw = scaled(m.dram_w, b, 1.0)
            al = scaled(m.alloc, b, 1.0)
            gfirst.append(ntr)
            gruns.append(runs)
            gbatch.append(b)
            for r in range(runs):
                body = lns + (rng.integers(0, jitter_ns + 1, L) if jitter_ns else 0)
                lbeg = EPOCH_NS + np.concatenate([[0], np.cumsum(body)[:-1]])
                lend = lbeg + body
                kl = np.cumsum(m.launch_ns) - m.launch_ns  # exclusive over the whole model
                kl = kl - kl[first_k][lay_of_k]           # ... restarted per layer
                a_beg = lbeg[lay_of_k] + kl
                a_end = a_beg + m.launch_ns
                d = ens + (rng.integers(0, jitter_ns + 1, K) if jitter_ns else 0)
                S = np.cumsum(d)
                Sprev = S - d
                e_end = S + np.maximum.accumulate(np.maximum(a_end - Sprev, EPOCH_NS - Sprev))
                e_beg = e_end - d
                mend = int(lend[-1])
                # H columns
                hb = np.empty(nH, dtype=np.int64)
                he = np.empty(nH, dtype=np.int64)
                hsid = np.empty(nH, dtype=np.int64)
                hrank = np.full(nH, 3, dtype=np.int64)
                hb[0], he[0], hsid[0], hrank[0] = EPOCH_NS, mend, 1, 1
                hb[h_layer_pos], he[h_layer_pos], hsid[h_layer_pos], hrank[h_layer_pos] = lbeg, lend, layer_sid, 2
                hb[h_launch_pos], he[h_launch_pos], hsid[h_launch_pos] = a_beg, a_end, launch_sid
                # merge the exec stream (sorted by begin) into H by (begin, rank, span_id)
                lo = np.searchsorted(hb, e_beg, "left")
                hi = np.searchsorted(hb, e_beg, "right")
                before = lo.copy()
                for o in range(int((hi - lo).max()) if K else 0):
                    idx = np.minimum(lo + o, nH - 1)
                    before += ((lo + o) < hi) & ((hrank[idx] < 3) | (hsid[idx] < exec_sid))
                n = nH + K
                epos = np.arange(K) + before
                is_e = np.zeros(n, dtype=bool)
                is_e[epos] = True
                hpos = np.nonzero(~is_e)[0]
                # assemble
                sid = np.empty(n, dtype=np.uint64)
                beg = np.empty(n, dtype=np.uint64)
                end = np.empty(n, dtype=np.uint64)
                cid = np.zeros(n, dtype=np.uint64)
                par = np.zeros(n, dtype=np.uint64)
                flg = np.empty(n, dtype=np.uint8)
                nm = np.empty(n, dtype=np.uint32)
                sid[hpos], beg[hpos], end[hpos] = hsid, hb, he
                sid[epos], beg[epos], end[epos] = exec_sid, e_beg, e_end
                hflags = np.full(nH, capi.LEVEL_KERNEL | (capi.KIND_LAUNCH << 2) | capi.F_CID, dtype=np.uint8)
                hflags[0] = capi.LEVEL_MODEL
                hflags[h_layer_pos] = capi.LEVEL_LAYER | capi.F_PARENT
                flg[hpos] = hflags
                flg[epos] = capi.LEVEL_KERNEL | (capi.KIND_EXEC << 2) | capi.F_CID | capi.F_METRICS
                hcid = np.zeros(nH, dtype=np.uint64)
                hcid[h_launch_pos] = np.arange(1, K + 1)
                cid[hpos] = hcid
                cid[epos] = np.arange(1, K + 1)
                hpar = np.zeros(nH, dtype=np.uint64)
                hpar[h_layer_pos] = 1
                par[hpos] = hpar
                hname = np.empty(nH, dtype=np.uint32)
                hname[0] = nid[m.name]
                hname[h_layer_pos] = layer_name_ids
                hname[h_launch_pos] = vocab_ids[m.kname]
                nm[hpos] = hname
                nm[epos] = vocab_ids[m.kname]
                for k, v in (("span_id", sid), ("parent_id", par), ("begin_ns", beg), ("end_ns", end),
                             ("cid", cid), ("flags", flg), ("name_id", nm), ("flops", fl),
                             ("dram_read", dr), ("dram_write", dw), ("occupancy", m.occ),
                             ("alloc_bytes", al), ("type_id", m.ltype)):
                    parts[k].append(v)
                lens.append(n)
                tbatch.append(b)
                trun.append(r)
                ntr += 1
    off = np.zeros(ntr + 1, dtype=np.uint64)
    off[1:] = np.cumsum(lens)
    cols = {k: np.concatenate(v) for k, v in parts.items()}
    lv = (1 << capi.LEVEL_MODEL) | (1 << capi.LEVEL_LAYER) | (1 << capi.LEVEL_KERNEL)
    batch = SpanBatch(**cols, trace_span_off=off, trace_id=np.arange(ntr) + 1,
                      trace_levels=np.full(ntr, lv), trace_batch=np.array(tbatch),
                      trace_run=np.array(trun), trace_serialized=np.zeros(ntr),
                      names=[n.encode() for n in names], types=[t.encode() for t in TYPES],
                      system_name=b"tesla-v100-sxm2", peak_flops=15.7e12, mem_bw=900e9)
    return batch, np.array(gfirst), np.array(gruns), np.array(gbatch)


def c3(runs: int = 20, n_models: int = 65, batches=(1, 2, 4, 8, 16, 32, 64, 128), seed: int = 1,
       **kw):
    """BASELINE config 3: 65-model x 8-batch sweep (~50M spans at runs=20)."""
    return corpus(make_models(n_models, seed=seed, **kw), batches, runs, seed=seed + 1000)


def c4(n_layers: int = 1_000_000, seed: int = 4, streams: int = 4, drain_every: int = 0,
       long_frac: float = 0.01, long_max: int = 64, kernels: int = 3, concurrent_frac: float = 0.001,
       chunk_layers: int = 65536) -> SpanBatch:
    """BASELINE config 4: ONE long-running trace (model span + n_layers layers).

    * Layers run back to back; a layer has `kernels` launches, or U{8..long_max}
      for a `long_frac` share of "long" layers (deep nesting within the 3-level
      model), launches packed from the layer begin (simprof build_plan shape,
      simprof.cpp:203-271).
    * A `concurrent_frac` share of layers open a concurrent group of two: both
      layers begin at the group begin, both launch from it, and the next group
      starts at the later end (simprof.cpp:237-241). Their launches lie inside
      both layers, which makes them ambiguities (correlator.cpp:242-257).
    * Executions are spread over `streams` device streams (kernel k on stream
      k % streams), each stream a cursor: exec begin = max(stream cursor, launch
      end) (simprof.cpp:255-257). Executions of different streams overlap each
      other and run past the end of their layer into later layers
      ("interleaved streams"); the cursors carry across the whole trace.
    * drain_every > 0: every that many layers the host waits for all streams to
      drain (a synchronisation point). The default has none, so layer intervals
      and launch->exec pairs cross every instant of the trace.
    * Correlation ids increase in launch order; span ids follow record order.
    Generated in chunks of `chunk_layers` layers (the drain period when set).
    At n_layers = 28.6M the trace has ~200M spans."""
    rng = np.random.default_rng(seed)
    names = sorted({f"c4/layer/{t}" for t in TYPES} | {"c4_model"} | set(KERNEL_VOCAB))
    nid = {n: i for i, n in enumerate(names)}
    layer_name = np.array([nid[f"c4/layer/{t}"] for t in TYPES], dtype=np.uint32)
    vocab_ids = np.array([nid[n] for n in KERNEL_VOCAB], dtype=np.uint32)
    parts = {k: [] for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags", "name_id",
                             "flops", "dram_read", "dram_write", "occupancy", "alloc_bytes", "type_id")}
    t_now = EPOCH_NS                      # begin of the next layer group
    cursor = np.full(streams, EPOCH_NS, dtype=np.int64)  # device stream cursors
    next_sid = 2
    next_cid = 1
    k_total = 0                           # kernels so far (stream of kernel k = k % streams)
    KF = capi.LEVEL_KERNEL
    step = drain_every if drain_every > 0 else chunk_layers
    for b0 in range(0, n_layers, step):
        L = min(step, n_layers - b0)
        kc = np.full(L, kernels, dtype=np.int64)
        long = rng.random(L) < long_frac
        kc[long] = rng.integers(8, long_max + 1, int(long.sum()))
        K = int(kc.sum())
        first_k = np.concatenate([[0], np.cumsum(kc)[:-1]])
        lay_of_k = np.repeat(np.arange(L), kc)
        k_in_layer = np.arange(K) - first_k[lay_of_k]
        launch_ns = rng.integers(3_000, 6_001, K)
        # launches packed from the layer begin; the layer body covers them
        kl = np.cumsum(launch_ns) - launch_ns
        kl = kl - kl[first_k][lay_of_k]
        lsum = np.bincount(lay_of_k, weights=launch_ns, minlength=L).astype(np.int64)
        body = np.maximum(rng.integers(20_000, 400_000, L), lsum + 1_000)
        # concurrent groups of two layers (never across a chunk boundary)
        starts = np.ones(L, dtype=bool)
        if concurrent_frac > 0 and L > 1:
            pair = np.nonzero(rng.random(L - 1) < concurrent_frac)[0]
            pair = pair[np.concatenate([[True], np.diff(pair) > 1])] if pair.size else pair
            starts[pair + 1] = False
        gid = np.cumsum(starts) - 1
        gfirst = np.nonzero(starts)[0]
        gbody = np.maximum.reduceat(body, gfirst)
        gbeg = t_now + np.concatenate([[0], np.cumsum(gbody)[:-1]])
        lbeg = gbeg[gid]
        lend = lbeg + body
        a_beg = lbeg[lay_of_k] + kl
        a_end = a_beg + launch_ns
        d = rng.integers(5_000, 300_000, K)
        e_beg = np.empty(K, dtype=np.int64)
        for s in range(streams):
            idx = np.arange((s - k_total) % streams, K, streams)
            if idx.size == 0:
                continue
            ds = d[idx]
            S = np.cumsum(ds)
            Sprev = S - ds
            e_end_s = S + np.maximum.accumulate(np.maximum(a_end[idx] - Sprev, int(cursor[s]) - Sprev))
            e_beg[idx] = e_end_s - ds
            cursor[s] = int(e_end_s[-1])
        k_total += K
        e_end = e_beg + d
        # span ids in record order: per layer [layer, (launch, exec) x K_l]
        layer_sid = next_sid + np.arange(L) + 2 * first_k
        launch_sid = layer_sid[lay_of_k] + 1 + 2 * k_in_layer
        exec_sid = launch_sid + 1
        next_sid = int(layer_sid[-1] + 1 + 2 * kc[-1])
        cid = next_cid + np.arange(K)
        next_cid += K
        # timeline order (begin_ns, rank, span_id) of the chunk
        n = L + 2 * K
        beg = np.concatenate([lbeg, a_beg, e_beg])
        end = np.concatenate([lend, a_end, e_end])
        sid = np.concatenate([layer_sid, launch_sid, exec_sid])
        rank = np.concatenate([np.full(L, 2), np.full(2 * K, 3)])
        order = np.lexsort((sid, rank, beg))
        role = np.concatenate([np.zeros(L, np.int8), np.ones(K, np.int8), np.full(K, 2, np.int8)])[order]
        src = np.concatenate([np.arange(L), np.arange(K), np.arange(K)])[order]
        flg = np.empty(n, dtype=np.uint8)
        flg[role == 0] = capi.LEVEL_LAYER | capi.F_PARENT
        flg[role == 1] = KF | (capi.KIND_LAUNCH << 2) | capi.F_CID
        flg[role == 2] = KF | (capi.KIND_EXEC << 2) | capi.F_CID | capi.F_METRICS
        kname = rng.integers(0, len(KERNEL_VOCAB), K)
        ltype = (b0 + np.arange(L)) % 4
        nm = np.where(role == 0, layer_name[ltype[np.minimum(src, L - 1)]], vocab_ids[kname[np.minimum(src, K - 1)]])
        cc = np.where(role == 0, 0, cid[np.minimum(src, K - 1)]).astype(np.uint64)
        par = np.where(role == 0, 1, 0).astype(np.uint64)
        ex_src = src[role == 2]  # metric rows in span-row order
        parts["span_id"].append(sid[order].astype(np.uint64))
        parts["parent_id"].append(par)
        parts["begin_ns"].append(beg[order].astype(np.uint64))
        parts["end_ns"].append(end[order].astype(np.uint64))
        parts["cid"].append(cc)
        parts["flags"].append(flg)
        parts["name_id"].append(nm.astype(np.uint32))
        parts["flops"].append(rng.integers(10_000_000, 10_000_000_000, K)[ex_src])
        parts["dram_read"].append(rng.integers(1_000_000, 100_000_000, K)[ex_src])
        parts["dram_write"].append(rng.integers(1_000_000, 100_000_000, K)[ex_src])
        parts["occupancy"].append((rng.integers(5, 96, K) / 100.0)[ex_src])
        lay_src = src[role == 0]
        parts["alloc_bytes"].append(rng.integers(100_000, 30_000_000, L)[lay_src])
        parts["type_id"].append(ltype[lay_src].astype(np.uint32))
        t_now = int(lend.max())
        if drain_every > 0:
            # synchronisation point: the next block starts once every stream drained
            t_now = int(max(t_now, cursor.max())) + 1_000
            cursor[:] = t_now
    mend = int(max(t_now, cursor.max()))
    model = {"span_id": [1], "parent_id": [0], "begin_ns": [EPOCH_NS], "end_ns": [mend], "cid": [0],
             "flags": [capi.LEVEL_MODEL], "name_id": [nid["c4_model"]]}
    cols = {}
    for k, v in parts.items():
        if k in model:
            cols[k] = np.concatenate([np.asarray(model[k], dtype=v[0].dtype)] + v)
        else:
            cols[k] = np.concatenate(v)
    if not drain_every:
        # each chunk is in timeline order on its own, but executions of chunk c
        # may begin after the first layers of chunk c + 1: one stable re-sort
        cols = _timeline_order(cols)
    n = cols["span_id"].size
    lv = (1 << capi.LEVEL_MODEL) | (1 << capi.LEVEL_LAYER) | (1 << capi.LEVEL_KERNEL)
    return SpanBatch(**cols, trace_span_off=np.array([0, n], dtype=np.uint64), trace_id=np.array([1]),
                     trace_levels=np.array([lv]), trace_batch=np.array([1]), trace_run=np.array([0]),
                     trace_serialized=np.zeros(1), names=[x.encode() for x in names],
                     types=[t.encode() for t in TYPES], system_name=b"tesla-v100-sxm2",
                     peak_flops=15.7e12, mem_bw=900e9)


def _timeline_order(cols):
    """Stable re-sort of one trace's span columns by (begin_ns, rank, span_id)
    (span.cpp:112-127); metric / layer side tables follow their spans."""
    f = cols["flags"]
    lvl = f & 3
    rank = np.where(lvl == capi.LEVEL_MODEL, 1, np.where(lvl == capi.LEVEL_LAYER, 2, 3)).astype(np.uint8)
    order = np.lexsort((cols["span_id"], rank, cols["begin_ns"]))
    if np.array_equal(order, np.arange(order.size)):
        return cols
    met = (f & capi.F_METRICS) != 0
    lay = lvl == capi.LEVEL_LAYER
    mrow = np.cumsum(met) - 1
    lrow = np.cumsum(lay) - 1
    out = {k: cols[k][order] for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags", "name_id")}
    mo = mrow[order][met[order]]
    lo = lrow[order][lay[order]]
    for k in ("flops", "dram_read", "dram_write", "occupancy"):
        out[k] = cols[k][mo]
    for k in ("alloc_bytes", "type_id"):
        out[k] = cols[k][lo]
    return out


def _keep_levels(b: SpanBatch, mask: int) -> SpanBatch:
    """The spans of b whose level is in `mask` (timeline order kept), with their
    metric / layer-table rows; every trace's level set becomes `mask`."""
    lvl = b.flags & 3
    keep = ((1 << lvl.astype(np.int64)) & mask) != 0
    met = (b.flags & capi.F_METRICS) != 0
    lay = lvl == capi.LEVEL_LAYER
    off = b.trace_span_off.astype(np.int64)
    cnt = np.add.reduceat(keep.astype(np.int64), off[:-1]) if b.n_traces else np.zeros(0, np.int64)
    cnt[np.diff(off) == 0] = 0
    kw = {k: getattr(b, k)[keep] for k in ("span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags",
                                            "name_id")}
    mk = keep[met]
    lk = keep[lay]
    kw.update({k: getattr(b, k)[mk] for k in ("flops", "dram_read", "dram_write", "occupancy")})
    kw.update({k: getattr(b, k)[lk] for k in ("alloc_bytes", "type_id")})
    return SpanBatch(**kw, trace_span_off=np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint64),
                     trace_id=b.trace_id, trace_levels=np.full(b.n_traces, mask), trace_batch=b.trace_batch,
                     trace_run=b.trace_run, trace_serialized=b.trace_serialized, names=b.names, types=b.types,
                     system_name=b.system_name, peak_flops=b.peak_flops, mem_bw=b.mem_bw)


def leveled_corpus(models: Sequence[Model], runs: int = 10, layer_oh_ns: int = 20_000,
                   kernel_oh_ns: int = 8_000, seed: int = 11):
    """BASELINE config 2 at scale: every model profiled at the level sets {M},
    {M,L}, {M,L,G} (simprof emit_leveled_chain shape, simprof.cpp:300-340),
    `runs` repetitions each, batch 1. Profiling a level adds overhead to the
    host time of the levels above it: +layer_oh per layer under {M,L}, and
    +kernel_oh per kernel on top under {M,L,G}; a shallower run records only
    its levels. Returns (batch, level_sets) with level_sets[m] = [(mask, trace
    indices)] for model m (one LeveledRunGroup per model, leveled.cpp:56-84)."""
    parts, sets = [], []
    t0 = 0
    full = (1 << capi.LEVEL_MODEL) | (1 << capi.LEVEL_LAYER) | (1 << capi.LEVEL_KERNEL)
    for mi, m in enumerate(models):
        msets = []
        for mask, loh, koh in ((1 << capi.LEVEL_MODEL, 0, 0),
                               ((1 << capi.LEVEL_MODEL) | (1 << capi.LEVEL_LAYER), layer_oh_ns, 0),
                               (full, layer_oh_ns, kernel_oh_ns)):
            mm = Model(**{**m.__dict__, "layer_ns": m.layer_ns + loh + koh * m.kcount})
            b, _, _, _ = corpus([mm], [1], runs, seed=seed + 97 * mi + mask)
            b = _keep_levels(b, mask) if mask != full else b
            b.trace_id = np.full(b.n_traces, 1_000 + mi, np.uint64)  # one workload per model
            parts.append(b)
            msets.append((mask, list(range(t0, t0 + b.n_traces))))
            t0 += b.n_traces
        sets.append(msets)
    return SpanBatch.concat(parts), sets
