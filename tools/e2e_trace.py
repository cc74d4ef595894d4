"""One traced xsp_run_host call on C3 (XSP_PIPE_TRACE host timeline per chunk)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_06869_b200 import Engine, synth  # noqa: E402

b, gf, gr, gb = synth.c3()
hb = b.pinned()
eng = Engine(0)
eng.run_host(hb, groups=(gf, gr, gb), raw=True)
eng.run_host(hb, groups=(gf, gr, gb), raw=True)
os.environ["XSP_PIPE_TRACE"] = "1"
eng.run_host(hb, groups=(gf, gr, gb), raw=True)
