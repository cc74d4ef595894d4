"""e2e (xsp_run_host) time per C3 step vs. pipeline chunk size (XSP_CHUNK_SPANS)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_06869_b200 import Engine, synth  # noqa: E402

b, gf, gr, gb = synth.c3()
hb = b.pinned()
eng = Engine(0)
for cs in [0, 24_000_000, 12_000_000, 6_000_000, 3_000_000, 1_500_000]:
    os.environ["XSP_CHUNK_SPANS"] = str(cs)
    eng.run_host(hb, groups=(gf, gr, gb), raw=True)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        eng.run_host(hb, groups=(gf, gr, gb), raw=True)
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"chunk {cs:>10d}: {min(ts):6.1f} ms (min of 3) {[round(x, 1) for x in ts]}", flush=True)
