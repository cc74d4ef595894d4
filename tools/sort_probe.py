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
# presorted input (the TraceBundle invariant): the order check alone
perm = torch.empty(b.n_spans, dtype=torch.int32, device="cuda:0")
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    assert eng.sort_timeline_device(dev, perm.data_ptr(), st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    eng.sort_timeline_device(dev, perm.data_ptr(), st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print({"presorted_ms": ms, "M spans/s": b.n_spans / ms / 1e3})
