"""GPU JSONL ingest phase breakdown: python tools/ingest_probe.py [models]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1908_06869_b200 import columns, synth  # noqa: E402
from paper_1908_06869_b200.engine import Engine  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 24
b, *_ = synth.c3(runs=1, n_models=m)
streams = [columns.to_jsonl(b, t) for t in range(b.n_traces)]
eng = Engine(0)
got, bad = eng.ingest_jsonl(streams)
assert bad == -1
os.environ["XSP_INGEST_TRACE"] = "1"
t = time.perf_counter()
eng.ingest_jsonl(streams)
print(f"total {1e3 * (time.perf_counter() - t):.1f} ms for {b.n_spans} spans, {sum(map(len, streams)) / 1e6:.0f} MB",
      flush=True)
