"""Print the C3 line of a bench.py --c5-copies 0 run (stdin): value, ms, stage times."""
import json
import sys

d = json.loads(sys.stdin.read())["c3"]
print(round(d["value"]), round(d["ms_per_step"], 4), {k: round(v, 4) for k, v in d["stages_ms"].items()})
