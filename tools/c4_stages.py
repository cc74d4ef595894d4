"""C4 stage breakdown on one GPU: python tools/c4_stages.py [layers] [concurrent_frac]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1908_06869_b200 import synth  # noqa: E402
from paper_1908_06869_b200.engine import DeviceBatch, Engine  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2_860_000
cf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.001
t = time.time()
b = synth.c4(n_layers=L, concurrent_frac=cf)
print(f"gen {time.time() - t:.1f}s, {b.n_spans} spans", flush=True)
eng = Engine(0)
dev = DeviceBatch(b, 0)
groups = ([0], [1], [1])
st = torch.cuda.current_stream().cuda_stream
co = eng.correlate_device(dev, stream=st)
print("layers", co.n_layers, "kernels", co.n_kernels, "orphans", co.n_orphans, "amb", co.n_ambiguities, flush=True)
eng.analyze_device(dev, co, groups, stream=st)
torch.cuda.synchronize()
eng.set_profiling(True)
eng.stage_reset()
t0 = time.time()
for _ in range(2):
    co = eng.correlate_device(dev, stream=st)
    eng.analyze_device(dev, co, groups, stream=st)
torch.cuda.synchronize()
ms = (time.time() - t0) / 2 * 1e3
s = eng.stage_times()
print(json.dumps({"ms_wall": ms, "spans": b.n_spans, "Gspans_s": b.n_spans / ms / 1e6,
                  "stages": {k: round(v[0] / max(v[1], 1), 3) for k, v in s.items()}}, indent=1))
