"""C3 end to end through xsp_run_host_packed vs xsp_run_host with chunk-size
variants: python tools/e2e_packed_probe.py [chunk_spans ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1908_06869_b200 import synth  # noqa: E402
from paper_1908_06869_b200.engine import Engine  # noqa: E402

b, gf, gr, gb = synth.c3()
hb = b.pinned()
eng = Engine(0)
from paper_1908_06869_b200 import _capi as capi  # noqa: E402
if os.environ.get("ROWS", "1") == "1":
    eng.set_host_outputs(capi.HOST_OUT_ROWS)  # the bench's e2e outputs
groups = (gf, gr, gb)
pk = eng.pack_host(hb)
for chunk in (sys.argv[1:] or ["6000000"]):
    os.environ["XSP_CHUNK_SPANS"] = chunk
    for name, fn in (("packed", lambda: eng.run_host_packed(pk, hb, groups=groups, raw=True)),):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) / 3 * 1e3
        h, d = eng.transfer_bytes()
        print(f"chunk {chunk} {name}: {ms:.1f} ms  {b.n_spans / ms / 1e3:.0f} M spans/s  h2d {h / 1e9:.2f} GB "
              f"({h / ms / 1e6:.1f} GB/s)  d2h {d / 1e9:.2f} GB", flush=True)
os.environ["XSP_CHUNK_SPANS"] = "12000000"
os.environ["XSP_PIPE_TRACE"] = "1"
eng.run_host_packed(pk, hb, groups=groups, raw=True)
torch.cuda.synchronize()
os.environ.pop("XSP_PIPE_TRACE", None)
# device stage times inside one packed call (work stream), vs the same with span_id copied
for zc in ("zero-copy span_id", "copied span_id"):
    if zc.startswith("copied"):
        os.environ["XSP_NO_ZERO_COPY"] = "1"
    eng.run_host_packed(pk, hb, groups=groups, raw=True)
    torch.cuda.synchronize()
    eng.set_profiling(True)
    eng.stage_reset()
    t = time.perf_counter()
    eng.run_host_packed(pk, hb, groups=groups, raw=True)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) * 1e3
    st = eng.stage_times()
    eng.set_profiling(False)
    print(zc, f"{ms:.1f} ms", {k: round(v[0], 3) for k, v in st.items()}, flush=True)
