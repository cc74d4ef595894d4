"""Per-tile pass-1 timeline on C3 (XSP_P1_TRACE): where a tile's lifetime goes.

Slots per tile (csrc/correlate.cu k_pass1): 0 start, 1 tile staged, 2 aggregate
published, 5 prefix known (look-back warp), 3 phase 3 starts, 4 end, 6 look-back
steps, 7 spin polls. Prints percentiles of each phase in microseconds.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_06869_b200.engine import DeviceBatch, Engine  # noqa: E402
from paper_1908_06869_b200 import synth  # noqa: E402

b, gf, gr, gb = synth.c3()
eng = Engine(0)
dev = DeviceBatch(b, 0)
for _ in range(3):
    eng.correlate_device(dev)
path = "/tmp/p1trace.bin"
os.environ["XSP_P1_TRACE"] = path
eng.correlate_device(dev)
d = np.fromfile(path, dtype=np.uint64).reshape(-1, 16).astype(np.int64)
t0 = d[:, 0].min()
st, staged, agg, pre, p3, end = (d[:, k] - t0 for k in (0, 1, 2, 5, 3, 4))
pct = lambda x: " ".join(f"{np.percentile(x, q) / 1e3:7.2f}" for q in (5, 50, 95, 99))
print("tiles", len(d), "span of kernel (us)", (end.max() - st.min()) / 1e3)
print("phase                p5      p50     p95     p99 (us)")
print("load            ", pct(staged - st))
print("phase1+publish  ", pct(agg - staged))
print("wait prefix     ", pct(np.maximum(pre - agg, 0)))
print("barrier->p3     ", pct(p3 - np.maximum(pre, agg)))
print("phase3          ", pct(end - p3))
print("lifetime        ", pct(end - st))
print("lookback steps  ", np.percentile(d[:, 6], [50, 95, 99]), "spins", np.percentile(d[:, 7], [50, 95, 99]))
order = np.argsort(st)
conc = np.searchsorted(np.sort(st), end, side="left") - np.arange(len(d))
print("resident tiles (p50)", np.percentile(np.searchsorted(np.sort(st), end) - np.searchsorted(np.sort(st), st), 50))
lag = (pre - agg)
idx = np.arange(len(d))
print("start time vs tile index: slope us/tile", np.polyfit(idx, st, 1)[0] / 1e3)
print("prefix time vs tile index: slope us/tile", np.polyfit(idx, pre, 1)[0] / 1e3)
