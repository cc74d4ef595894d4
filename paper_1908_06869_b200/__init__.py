"""B200-native span correlation + analysis hot path of XSP (arXiv:1908.06869).

The product is lib/libxsp.so (hand-written sm_100a CUDA behind the C ABI in
include/xsp.h). This package is the Python host mirror used by tests and the
bench; the C++ drop-in for the reference's strata:: API lives in csrc/host/.
"""
from .columns import SpanBatch  # noqa: F401
from .engine import CorrResult, Engine, Tables  # noqa: F401

__all__ = ["SpanBatch", "Engine", "CorrResult", "Tables"]
