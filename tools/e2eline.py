"""Print the C3 end-to-end lines of a bench.py JSON file: python tools/e2eline.py FILE"""
import json
import sys

d = json.load(open(sys.argv[1]))["c3"]
for k in ("e2e", "e2e_full", "e2e_dense"):
    e = d[k]
    print(k, round(e["value"]), "M spans/s", round(e["ms_per_step"], 2), "ms  h2d", e["h2d_bytes_per_step"],
          "d2h", e["d2h_bytes_per_step"])
print("c3 device", round(d["value"]), "M spans/s")
