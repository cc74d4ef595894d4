"""Stage times of the device path on one long C4 trace (synth.c4)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1908_06869_b200 import synth  # noqa: E402
from paper_1908_06869_b200.engine import DeviceBatch, Engine  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
t = time.time()
b = synth.c4(n_layers=layers)
print("spans", b.n_spans, "gen s", round(time.time() - t, 1), flush=True)
eng = Engine(0)
dev = DeviceBatch(b, 0)
groups = ([0], [1], [1])
for _ in range(2):
    co = eng.correlate_device(dev)
    eng.analyze_device(dev, co, groups)
torch.cuda.synchronize()
eng.set_profiling(True)
eng.stage_reset()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    co = eng.correlate_device(dev)
    eng.analyze_device(dev, co, groups)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print("ms/step", round(ms, 3), "M spans/s", round(b.n_spans / ms / 1e3, 1))
print({k: round(v[0] / max(v[1], 1), 3) for k, v in eng.stage_times().items()})
