"""Comparison helpers: product results (C ABI) vs the reference oracle.

Integer / index outputs must match exactly. fp64 outputs are compared
bit-exactly by default (the reference's op order is reproduced); callers may
pass rtol (north star: derived fp64 ratios within 1e-9 relative).
"""
from __future__ import annotations

import numpy as np

GROUP_TEXT = {
    1: "analysis input holds no runs",
    2: "repetitions disagree on layer count",
    3: "repetitions disagree on kernel count of layer {i}",
    5: "trim fraction must lie in [0, 0.5)",
}


def _eq(a, b, what, rtol=0.0):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, f"{what}: shape {a.shape} != {b.shape}"
    if rtol and a.dtype.kind == "f":
        np.testing.assert_allclose(a, b, rtol=rtol, atol=0, equal_nan=True, err_msg=what)
    else:
        np.testing.assert_array_equal(a, b, err_msg=what)


def _rows(a, base):
    return np.asarray(a).astype(np.int64) + base


def compare_correlation(batch, corr, ref_arrays, ref_strings, t_base=0, row_base=0, whole=True):
    """corr (the product's result over `batch`) against the reference's result.
    whole=False: the reference ran on a slice of `batch`; its trace t is the
    product's trace t_base + t and its span rows are offset by row_base."""
    rs = ref_arrays
    T = len(rs["t_status"])
    if whole:
        assert corr.n_traces == batch.n_traces == T
    for tr in range(T):
        t = tr + t_base
        ref_ok = int(rs["t_status"][tr]) == 0
        gpu_msg = corr.error_message(batch, t)
        ref_msg = ref_strings["t_error"][tr].decode()
        assert gpu_msg == ref_msg, f"trace {t}: error {gpu_msg!r} != {ref_msg!r}"
        if not ref_ok:
            continue
        assert int(corr.trace_model_row[t]) == int(rs["t_model_row"][tr]) + row_base, f"trace {t} model row"
        rl0, rl1 = int(rs["t_layer_off"][tr]), int(rs["t_layer_off"][tr + 1])
        gl0, gl1 = int(corr.trace_layer_off[t]), int(corr.trace_layer_off[t + 1])
        _eq(corr.layer_row[gl0:gl1], _rows(rs["layer_row"][rl0:rl1], row_base), f"trace {t} layer rows")
        _eq(np.diff(corr.layer_kernel_off[gl0:gl1 + 1]), np.diff(rs["layer_kernel_off"][rl0:rl1 + 1]),
            f"trace {t} kernels per layer")
        # layer attributes (layer_type / alloc_bytes tags, correlator.cpp:197-202)
        attr = corr.layer_attr_row[gl0:gl1].astype(np.int64)
        _eq(batch.alloc_bytes[attr], rs["layer_alloc"][rl0:rl1], f"trace {t} alloc")
        types = [batch.types[i] for i in batch.type_id[attr]]
        assert types == ref_strings["layer_type"][rl0:rl1], f"trace {t} layer types"
        rk0, rk1 = int(rs["layer_kernel_off"][rl0]), int(rs["layer_kernel_off"][rl1])
        gk0, gk1 = int(corr.trace_kernel_off[t]), int(corr.trace_kernel_off[t + 1])
        _eq(corr.kernel_launch_row[gk0:gk1], _rows(rs["kernel_launch_row"][rk0:rk1], row_base),
            f"trace {t} launch rows")
        _eq(corr.kernel_exec_row[gk0:gk1], _rows(rs["kernel_exec_row"][rk0:rk1], row_base), f"trace {t} exec rows")
        mrow = corr.kernel_metric_row[gk0:gk1]
        has = mrow != 0xFFFFFFFF
        _eq(has.astype(np.uint8), rs["kernel_has_metrics"][rk0:rk1], f"trace {t} has_metrics")
        mr = mrow[has].astype(np.int64)
        _eq(batch.flops[mr], rs["kernel_flops"][rk0:rk1][has], f"trace {t} flops")
        _eq(batch.dram_read[mr], rs["kernel_read"][rk0:rk1][has], f"trace {t} reads")
        _eq(batch.dram_write[mr], rs["kernel_write"][rk0:rk1][has], f"trace {t} writes")
        _eq(batch.occupancy[mr], rs["kernel_occ"][rk0:rk1][has], f"trace {t} occupancy")
        # durations and names come from the exec span (correlator.hpp:80-86)
        ex = corr.kernel_exec_row[gk0:gk1].astype(np.int64)
        dur = np.where(batch.end_ns[ex] >= batch.begin_ns[ex], batch.end_ns[ex] - batch.begin_ns[ex], 0)
        _eq(corr.kernel_dur[gk0:gk1], dur, f"trace {t} kernel durations")
        _eq(corr.kernel_name[gk0:gk1], batch.name_id[ex], f"trace {t} kernel names")
        # orphans, in the reference's order, with the reference's reason text
        ro0, ro1 = int(rs["t_orphan_off"][tr]), int(rs["t_orphan_off"][tr + 1])
        go0, go1 = int(corr.trace_orphan_off[t]), int(corr.trace_orphan_off[t + 1])
        _eq(corr.orphan_row[go0:go1], _rows(rs["orphan_row"][ro0:ro1], row_base), f"trace {t} orphan rows")
        texts = [corr.orphan_text(batch, j) for j in range(go0, go1)]
        ref_texts = [x.decode() for x in ref_strings["orphan_text"][ro0:ro1]]
        assert texts == ref_texts, f"trace {t} orphan reasons {texts} != {ref_texts}"
        # ambiguities sorted by span_id with candidates sorted by span_id
        ra0, ra1 = int(rs["t_amb_off"][tr]), int(rs["t_amb_off"][tr + 1])
        ga0, ga1 = int(corr.trace_amb_off[t]), int(corr.trace_amb_off[t + 1])
        _eq(corr.amb_row[ga0:ga1], _rows(rs["amb_row"][ra0:ra1], row_base), f"trace {t} ambiguity rows")
        for q in range(ga1 - ga0):
            g0, g1 = int(corr.amb_cand_off[ga0 + q]), int(corr.amb_cand_off[ga0 + q + 1])
            r0, r1 = int(rs["amb_cand_off"][ra0 + q]), int(rs["amb_cand_off"][ra0 + q + 1])
            _eq(corr.amb_cand_row[g0:g1], _rows(rs["amb_cand_row"][r0:r1], row_base),
                f"trace {t} amb {q} candidates")


K_FIELDS = ["k_name", "k_layer", "k_lat", "k_flops", "k_read", "k_write", "k_occ", "k_ai", "k_tput"]
L_FIELDS = [("l_index", "l_index"), ("l_layer_lat", "l_layer_lat"), ("l_kern_lat", "l_kern_lat"),
            ("l_flops", "l_flops"), ("l_read", "l_read"), ("l_write", "l_write"), ("l_occ", "l_occ"),
            ("l_count", "l_count"), ("l_ai", "l_ai"), ("l_tput", "l_tput"), ("l_gpu", "l_kern_lat"),
            ("l_nongpu", "l_nongpu"), ("l_gpu_share", "l_gpu_share"),
            ("l_nongpu_share", "l_nongpu_share")]
N_FIELDS = ["n_name", "n_count", "n_lat", "n_pct", "n_flops", "n_read", "n_write", "n_occ", "n_ai",
            "n_tput"]
M_FIELDS = [("m_lat", "m_lat"), ("m_kern_lat", "m_kern_lat"), ("m_flops", "m_flops"),
            ("m_read", "m_read"), ("m_write", "m_write"), ("m_occ", "m_occ"), ("m_count", "m_count"),
            ("m_ai", "m_ai"), ("m_tput", "m_tput"), ("m_gpu", "m_gpu"), ("m_gpu_pct", "m_gpu_pct"),
            ("m_throughput", "m_throughput")]


def _bound(x):
    x = np.asarray(x).astype(np.int16)
    return np.where(x == 255, -1, x)


def compare_tables(batch, tabs, ref_arrays, ref_strings, rtol=0.0, g_base=0, whole=True):
    """tabs (the product's tables) against the reference's a5..a15; whole=False:
    the reference's group g is the product's group g_base + g."""
    ra = ref_arrays
    G = len(ref_strings["g_error"])
    if whole:
        assert G == tabs.n_groups
    rk = ra["g_kernel_off"] - ra["g_kernel_off"][0]
    rl = ra["g_layer_off"] - ra["g_layer_off"][0]
    rn = ra["g_name_off"] - ra["g_name_off"][0]
    for q in range(G):
        ref_err = ref_strings["g_error"][q].decode()
        g = q + g_base
        st = int(tabs.group_status[g])
        if ref_err:
            assert st != 0, f"group {g}: reference failed with {ref_err!r}, product did not"
            if st in GROUP_TEXT:
                assert GROUP_TEXT[st].format(i=int(tabs.group_err_arg[g])) == ref_err, (st, ref_err)
            continue
        assert st == 0, f"group {g}: product status {st}, reference ok"
        k0, k1 = int(tabs.group_kernel_off[g]), int(tabs.group_kernel_off[g + 1])
        assert k1 - k0 == int(rk[q + 1] - rk[q]), f"group {g}: kernel rows"
        for f in K_FIELDS:
            _eq(tabs.cols[f][k0:k1], ra[f][rk[q]:rk[q + 1]], f"group {g} {f}", rtol)
        _eq(_bound(tabs.k_bound[k0:k1]), _bound(ra["k_bound"][rk[q]:rk[q + 1]]), f"group {g} k_bound")
        # a9: classify() inclusion, values equal to a8's where included
        _eq(tabs.k_roofline_in[k0:k1], ra["k9_in"][rk[q]:rk[q + 1]], f"group {g} a9 inclusion")
        inc = ra["k9_in"][rk[q]:rk[q + 1]] == 1
        _eq(tabs.k_ai[k0:k1][inc], ra["k9_ai"][rk[q]:rk[q + 1]][inc], f"group {g} a9 ai", rtol)
        _eq(tabs.k_tput[k0:k1][inc], ra["k9_tput"][rk[q]:rk[q + 1]][inc], f"group {g} a9 tput", rtol)
        l0, l1 = int(tabs.group_layer_off[g]), int(tabs.group_layer_off[g + 1])
        assert l1 - l0 == int(rl[q + 1] - rl[q]), f"group {g}: layer rows"
        for rf, gf in L_FIELDS:
            _eq(tabs.cols[gf][l0:l1], ra[rf][rl[q]:rl[q + 1]], f"group {g} {rf}", rtol)
        _eq(_bound(tabs.l_bound[l0:l1]), _bound(ra["l_bound"][rl[q]:rl[q + 1]]), f"group {g} l_bound")
        _eq(tabs.l_flagged[l0:l1], ra["l_flagged"][rl[q]:rl[q + 1]], f"group {g} a13 flagged")
        _eq(tabs.l_roofline_in[l0:l1], ra["l14_in"][rl[q]:rl[q + 1]], f"group {g} a14 inclusion")
        _eq(batch.name_id[tabs.l_row[l0:l1].astype(np.int64)], ra["l_name"][rl[q]:rl[q + 1]],
            f"group {g} layer names")
        n0, n1 = int(tabs.group_name_off[g]), int(tabs.group_name_off[g + 1])
        assert n1 - n0 == int(rn[q + 1] - rn[q]), f"group {g}: a10 rows"
        for f in N_FIELDS:
            _eq(tabs.cols[f][n0:n1], ra[f][rn[q]:rn[q + 1]], f"group {g} {f}", rtol)
        _eq(_bound(tabs.n_bound[n0:n1]), _bound(ra["n_bound"][rn[q]:rn[q + 1]]), f"group {g} n_bound")
        for rf, gf in M_FIELDS:
            _eq(tabs.cols[gf][g:g + 1], ra[rf][q:q + 1], f"group {g} {rf}", rtol)
        _eq(_bound(tabs.m_bound[g:g + 1]), _bound(ra["m_bound"][q:q + 1]), f"group {g} m_bound")
        _eq(tabs.m_roofline_in[g:g + 1], ra["mr_in"][q:q + 1], f"group {g} model_roofline")
        # a5 / a6 / a7 by layer type (analysis.cpp:315-337)
        if "g_type_off" in ra and "group_type_off" in tabs.cols:
            ry = ra["g_type_off"] - ra["g_type_off"][0]
            y0, y1 = int(tabs.group_type_off[g]), int(tabs.group_type_off[g + 1])
            assert y1 - y0 == int(ry[q + 1] - ry[q]), f"group {g}: a5 rows"
            types = [batch.types[int(t)].decode() for t in tabs.y_type[y0:y1]]
            want = [x.decode() for x in ref_strings["y_type"][int(ry[q]):int(ry[q + 1])]]
            assert types == want, f"group {g} a5 types {types[:4]} != {want[:4]}"
            _eq(tabs.y_count[y0:y1], ra["y_count"][ry[q]:ry[q + 1]], f"group {g} a5 count")
            _eq(tabs.y_lat[y0:y1], ra["y_lat"][ry[q]:ry[q + 1]], f"group {g} a5 latency", rtol)
            _eq(tabs.y_alloc[y0:y1], ra["y_alloc"][ry[q]:ry[q + 1]], f"group {g} a7 alloc")


def topk_oracle(k_lat: np.ndarray, k_layer: np.ndarray, k: int) -> np.ndarray:
    """Top-k kernels per layer (north star (e)) restated over a8 rows: latency desc,
    kernel ordinal asc on ties; UINT32_MAX padding."""
    layers = int(k_layer.max()) + 1 if k_layer.size else 0
    out = np.full((layers, k), 0xFFFFFFFF, dtype=np.uint32)
    for li in range(layers):
        idx = np.nonzero(k_layer == li)[0]
        order = sorted(idx.tolist(), key=lambda j: (-k_lat[j], j))[:k]
        out[li, :len(order)] = order
    return out
