"""Host-side cost of one device-resident step (C3): wall time of each API call
versus the device time of the work it enqueues (CUDA events)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1908_06869_b200 import synth  # noqa: E402
from paper_1908_06869_b200.engine import DeviceBatch, Engine  # noqa: E402

b, gf, gr, gb = synth.c3()
eng = Engine(0)
dev = DeviceBatch(b, 0)
groups = (gf, gr, gb)
for _ in range(3):
    co = eng.correlate_device(dev)
    eng.analyze_device(dev, co, groups)
torch.cuda.synchronize()
tc, ta, tg = [], [], []
for _ in range(10):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    t0 = time.perf_counter()
    e0.record()
    co = eng.correlate_device(dev)
    t1 = time.perf_counter()
    e1.record()
    eng.analyze_device(dev, co, groups)
    e2.record()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    tc.append((t1 - t0) * 1e3)
    ta.append((t2 - t1) * 1e3)
    tg.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
print("wall correlate ms", sorted(tc)[5], "analyze ms", sorted(ta)[5])
print("gpu  correlate ms", sorted(x[0] for x in tg)[5], "analyze ms", sorted(x[1] for x in tg)[5])
# python-side costs of building the call arguments
t0 = time.perf_counter()
for _ in range(100):
    dev.cols(); dev.traces(); eng.make_groups(*groups)
print("arg building us", (time.perf_counter() - t0) * 1e4)
