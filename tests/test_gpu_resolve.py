"""GPU parity for resolve_with_serialized (correlator.cpp:379-456, SURVEY
§8(f)-2): xsp_resolve_serialized against the UNMODIFIED reference on
concurrent-branch traces and their serialized twins from the reference's own
simulator (simprof emit_run serialized=true), including the "serialized run is
itself ambiguous" fault."""
import numpy as np
import pytest

from oracle import ref
from paper_1908_06869_b200 import _capi as capi
from parity import compare_correlation

pytestmark = pytest.mark.gpu

CASES = [("overlap", 1), ("overlap", 2), ("overlap", 8), ("resnet-like", 1), ("minimal", 4)]


def pair_batches(cases, serialized_second=True):
    """One generator (one name table): every concurrent trace, then every twin."""
    g = ref.Generator()
    for m, b in cases:
        g.emit(m, batch=b)
    for m, b in cases:
        g.emit(m, batch=b, serialized=serialized_second)
    b = g.batch()
    k = len(cases)
    return b.trace_slice(0, k), b.trace_slice(k, 2 * k)


def test_resolve_matches_reference(engine, has_ref):
    orig, ser = pair_batches(CASES)
    first = engine.run_host(orig)[0]
    assert first.n_ambiguities > 0  # the overlap traces need the serialized twin
    corr = engine.resolve_serialized(orig, ser)
    ra, rs = ref.resolve(orig, ser)
    compare_correlation(orig, corr, ra, rs)
    assert corr.n_ambiguities == 0 and corr.n_failed == 0


def test_serialized_itself_ambiguous(engine, has_ref):
    orig, ser = pair_batches([("overlap", 1), ("resnet-like", 2)], serialized_second=False)
    corr = engine.resolve_serialized(orig, ser)
    ra, rs = ref.resolve(orig, ser)
    assert int(corr.trace_status[0]) == capi.T_SER_AMBIGUOUS
    assert corr.error_message(orig, 0) == rs["t_error"][0].decode()
    assert int(corr.trace_status[1]) == capi.T_OK
    assert rs["t_error"][1].decode() == ""
