"""GPU JSONL ingest phase breakdown on page-locked text (as bench.py times it):
python tools/ingest_probe.py [models]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1908_06869_b200 import _capi as capi, columns, synth  # noqa: E402
from paper_1908_06869_b200.engine import Engine  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 24
b, *_ = synth.c3(runs=1, n_models=m)
streams = [columns.to_jsonl(b, t) for t in range(b.n_traces)]
raw = b"".join(streams)
off = np.zeros(len(streams) + 1, dtype=np.uint64)
off[1:] = np.cumsum([len(x) for x in streams])
pinned = torch.empty(len(raw), dtype=torch.uint8).pin_memory()
pinned.numpy()[:] = np.frombuffer(raw, dtype=np.uint8)
blob = C.cast(C.c_void_p(pinned.data_ptr()), C.c_char_p)
eng = Engine(0)


def call():
    out = capi.IngestOut()
    eng._check(eng.lib.xsp_ingest_jsonl(eng.ctx, blob, off.ctypes.data_as(capi.u64p), len(streams), C.byref(out),
                                        None))
    assert out.status == capi.INGEST_OK


for _ in range(3):
    call()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    call()
torch.cuda.synchronize()
ms = (time.perf_counter() - t) / 5 * 1e3
print(f"{ms:.2f} ms for {b.n_spans} spans, {len(raw) / 1e6:.0f} MB: {b.n_spans / ms / 1e3:.1f} M spans/s", flush=True)
os.environ["XSP_INGEST_TRACE"] = "1"
call()
