"""Golden fixtures: inputs + the REFERENCE's outputs, stored as .npz so the GPU box
(where /root/reference does not exist) can check against them. Written by
tests/golden/make_golden.py from the unmodified reference (oracle/_ref)."""
import json

import numpy as np

from paper_1908_06869_b200 import SpanBatch
from paper_1908_06869_b200.columns import LAYER_COLS, METRIC_COLS, SPAN_COLS, TRACE_COLS


def _pack_strings(prefix, d, out):
    for k, lst in d.items():
        out[f"{prefix}.s.{k}"] = np.array(json.dumps([x.decode("latin-1") for x in lst]))


def _unpack_strings(prefix, z):
    res = {}
    for k in z.files:
        if k.startswith(prefix + ".s."):
            res[k[len(prefix) + 3:]] = [x.encode("latin-1") for x in json.loads(str(z[k]))]
    return res


def save_golden(path, batch, groups, corr_bag, an_bag):
    out = {}
    for k in list(SPAN_COLS) + list(METRIC_COLS) + list(LAYER_COLS) + list(TRACE_COLS):
        out[f"in.{k}"] = getattr(batch, k)
    _pack_strings("in", {"names": batch.names, "types": batch.types, "system_name": [batch.system_name]}, out)
    out["in.system"] = np.array([batch.peak_flops, batch.mem_bw])
    out["groups"] = np.array(groups, dtype=np.uint32)
    for prefix, (arrays, strings) in (("corr", corr_bag), ("an", an_bag)):
        for k, v in arrays.items():
            out[f"{prefix}.a.{k}"] = v
        _pack_strings(prefix, strings, out)
    np.savez_compressed(path, **out)


def load_golden(path):
    z = np.load(path, allow_pickle=False)
    kw = {k: z[f"in.{k}"] for k in list(SPAN_COLS) + list(METRIC_COLS) + list(LAYER_COLS) + list(TRACE_COLS)}
    s = _unpack_strings("in", z)
    b = SpanBatch(**kw, names=s["names"], types=s["types"], system_name=s["system_name"][0],
                  peak_flops=float(z["in.system"][0]), mem_bw=float(z["in.system"][1]))
    groups = z["groups"]

    def bag(prefix):
        arrays = {k[len(prefix) + 3:]: z[k] for k in z.files if k.startswith(prefix + ".a.")}
        return arrays, _unpack_strings(prefix, z)

    return b, bag("corr"), bag("an"), (groups[0], groups[1], groups[2])
