"""Time sort_timeline on the per-trace shuffled C3 corpus (bench.measure_sort's
input) and report the varying key bits of its traces."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1908_06869_b200 import synth  # noqa: E402
from paper_1908_06869_b200.engine import DeviceBatch, Engine  # noqa: E402

b, gf, gr, gb = synth.c3()
off = b.trace_span_off
bits = []
for t in range(0, b.n_traces, 97):
    lo, hi = int(off[t]), int(off[t + 1])
    bits.append((int(b.begin_ns[lo:hi].max() - b.begin_ns[lo:hi].min()).bit_length(),
                 int(b.span_id[lo:hi].max() - b.span_id[lo:hi].min()).bit_length()))
print("begin bits / span_id bits (sample):", sorted(set(bits))[:10], "...")
eng = Engine(0)
dev = DeviceBatch(b, 0)
steps = int(os.environ.get("STEPS", "10"))
print(bench.measure_sort(eng, dev, b, steps, 0))
