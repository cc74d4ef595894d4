"""CPU-side checks of the C-ABI boundary: the library loads, exports exactly what
include/xsp.h declares, its ctypes mirror has the C layout, and the product path
refuses to run without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_1908_06869_b200 import _capi as capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xsp.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*\s]+?)\b(xsp_\w+)\s*\(", text, re.M)))


def test_header_declares_the_api():
    fns = declared_functions()
    for f in ("xsp_ctx_create", "xsp_correlate", "xsp_analyze", "xsp_run_host", "xsp_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    lib = capi.load()
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (xsp_\w+)", out))
    declared = set(declared_functions())
    assert declared <= exported, f"missing: {declared - exported}"
    assert exported <= declared, f"undeclared exports: {exported - declared}"
    assert set(capi.EXPORTS) == declared
    assert lib.xsp_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def _c_layout():
    """sizeof/offsetof of the ABI structs as the C compiler sees them."""
    fields = {
        "xsp_span_cols": ["n_spans", "name_id", "n_metric_rows", "occupancy", "n_layer_rows", "type_id"],
        "xsp_traces": ["n_traces", "span_off", "levels"],
        "xsp_corr_out": ["n_failed", "n_candidates", "trace_status", "amb_cand_row"],
        "xsp_analysis_opts": ["noise_tolerance", "top_k"],
        "xsp_groups": ["n_groups", "batch_size"],
        "xsp_tables_out": ["n_names", "group_status", "l_topk", "m_roofline_in"],
    }
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "xsp.h"', "int main(void){"]
    for s, fs in fields.items():
        src.append(f'printf("{s} size %zu\\n", sizeof({s}));')
        for f in fs:
            src.append(f'printf("{s} {f} %zu\\n", offsetof({s}, {f}));')
    src.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write("\n".join(src))
        exe = os.path.join(d, "l")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    res = {}
    for line in out.splitlines():
        s, f, v = line.split()
        res[(s, f)] = int(v)
    return res


def test_ctypes_layout_matches_c():
    lay = _c_layout()
    m = {"xsp_span_cols": capi.SpanCols, "xsp_traces": capi.Traces, "xsp_corr_out": capi.CorrOut,
         "xsp_analysis_opts": capi.AnalysisOpts, "xsp_groups": capi.Groups,
         "xsp_tables_out": capi.TablesOut}
    for (s, f), v in lay.items():
        cls = m[s]
        if f == "size":
            assert C.sizeof(cls) == v, (s, C.sizeof(cls), v)
        else:
            assert getattr(cls, f).offset == v, (s, f, getattr(cls, f).offset, v)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1908_06869_b200 import Engine
    with pytest.raises(capi.XspError) as e:
        Engine(0)
    assert e.value.status == capi.XSP_E_NO_DEVICE
