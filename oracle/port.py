"""TEST INFRASTRUCTURE — Python handle on the plain-C restatement (oracle/xsp_oracle.c).

It consumes the same SoA columns as the C ABI and fills the same result structs
(include/xsp.h) in host memory, so results diff directly against the product.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1908_06869_b200 import _capi as capi
from paper_1908_06869_b200.engine import CorrResult, Tables, _copy, _corr_counts, _tab_counts

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "lib", "libxsp_oracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(PORT_LIB):
            raise ImportError(f"{PORT_LIB} missing: run `make -C {HERE} port`")
        L = C.CDLL(PORT_LIB, mode=C.RTLD_LOCAL)
        L.xspo_correlate.argtypes = [C.POINTER(capi.SpanCols), C.POINTER(capi.Traces), C.POINTER(capi.CorrOut)]
        L.xspo_corr_free.argtypes = [C.POINTER(capi.CorrOut)]
        L.xspo_analyze.argtypes = [C.POINTER(capi.SpanCols), C.POINTER(capi.CorrOut), C.POINTER(capi.Groups),
                                   C.POINTER(capi.SystemSpec), C.POINTER(capi.AnalysisOpts),
                                   C.POINTER(capi.TablesOut)]
        L.xspo_tables_free.argtypes = [C.POINTER(capi.TablesOut)]
        _lib = L
    return _lib


def run(batch, groups=None, trim=0.2, noise=0.01, top_k=3, analyze=True):
    """correlate (+ analyze) with the C port; returns (CorrResult, Tables|None)."""
    from paper_1908_06869_b200.engine import Engine
    L = lib()
    cols, trs = batch.cols(), batch.traces()
    co = capi.CorrOut()
    L.xspo_correlate(C.byref(cols), C.byref(trs), C.byref(co))
    cc = _corr_counts(co)
    corr = CorrResult(co.n_traces, co.n_failed,
                      {n: _copy(getattr(co, n), t, cc[k]) for n, t, k in capi.CORR_FIELDS},
                      co.n_layers, co.n_kernels, co.n_orphans, co.n_ambiguities, co.n_candidates)
    tabs = None
    if analyze:
        if groups is None:
            T = batch.n_traces
            groups = (np.arange(T), np.ones(T), batch.trace_batch)
        g, keep = Engine.make_groups(*groups)
        spec = capi.SystemSpec(batch.peak_flops, batch.mem_bw)
        opts = Engine.make_opts(trim=trim, noise=noise, top_k=top_k)
        to = capi.TablesOut()
        L.xspo_analyze(C.byref(cols), C.byref(co), C.byref(g), C.byref(spec), C.byref(opts), C.byref(to))
        tc = _tab_counts(to, top_k)
        tabs = Tables(to.n_groups, {n: _copy(getattr(to, n), t, tc[k]) for n, t, k in capi.TABLE_FIELDS},
                      to.n_layers, to.n_kernels, to.n_names)
        L.xspo_tables_free(C.byref(to))
    L.xspo_corr_free(C.byref(co))
    return corr, tabs
