"""Regenerate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

    python tests/golden/make_golden.py

Each fixture stores its SoA input and the reference's correlate + a8..a15
outputs. Committed so parity can be checked where the reference is absent.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

import cases  # noqa: E402
from builders import KERNEL, MLG, MODEL, batch_of  # noqa: E402
from golden_io import save_golden  # noqa: E402
from oracle import ref  # noqa: E402


def emit(name, spec):
    g = ref.Generator()
    for kw in spec:
        g.emit(**kw)
    return g.batch()


def main():
    fixtures = {}
    # C1a shape: resnet-like x 10 jittered iterations in one group
    b = emit("c1", [dict(model="resnet-like", batch=1, run_index=r, jitter_max=1000, jitter_seed=r + 1)
                    for r in range(10)])
    fixtures["c1_resnet_x10"] = (b, ([0], [10], [1]))
    # criterion-10 shape: every fixture at batch 2, one group each
    g = ref.Generator()
    names = ["minimal", "resnet-like", "mobilenet-like", "overlap", "async-straggler", "overhead-chain"]
    for n in names:
        g.emit(n, batch=2)
    b = g.batch()
    fixtures["fixtures_b2"] = (b, (list(range(6)), [1] * 6, [2] * 6))
    # generators of the reference tests
    g = ref.Generator()
    for i in range(8):
        g.random_nested(99, 50 + 61 * i)
    g.random_async(7, 300)
    b = g.batch()
    T = b.n_traces
    fixtures["random_nested_async"] = (b, (list(range(T)), [1] * T, [1] * T))
    # known-answer edge cases + faults
    traces = [cases.nesting(), cases.layer_attrs(), cases.explicit_beats_containment(),
              cases.overlapping_layers(), cases.orphans(), cases.fusion(), cases.unmatched_async(),
              cases.mixed_orphan_order(), cases.dup_launch_cid(), cases.dup_exec_cid(),
              cases.no_model(), cases.two_models(), cases.skip_level()]
    levels = [MLG] * len(traces)
    levels[-1] = (1 << MODEL) | (1 << KERNEL)
    b = batch_of(traces, levels=levels)
    T = b.n_traces
    fixtures["edge_cases"] = (b, (list(range(T)), [1] * T, [1] * T))
    for name, (b, groups) in fixtures.items():
        corr = ref.correlate(b)
        an = ref.analyze(b, groups[0], groups[1])
        path = os.path.join(HERE, f"{name}.npz")
        save_golden(path, b, groups, corr, an)
        print(f"{path}: {b.n_spans} spans, {b.n_traces} traces, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
