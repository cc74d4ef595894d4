"""profiles/traffic.json from an `ncu --set full` capture: per kernel (first
captured launch of each name) dram__bytes_read.sum + dram__bytes_write.sum and
duration, with the capture command and workload recorded.

  python tools/traffic_from_ncu.py REPORT.ncu-rep SPANS "capture description" "workload"
"""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(rep, spans, capture, workload):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = {}
    for row in rows[2:]:
        d = dict(zip(h, row))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0]
        if name in out:
            continue

        def val(k):
            u = units[h.index(k)]
            return float(d[k].replace(",", "")) * UNIT.get(u, 1)

        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        t = float(d["gpu__time_duration.sum"].replace(",", ""))
        tu = units[h.index("gpu__time_duration.sum")]
        us = {"ns": t / 1e3, "nsecond": t / 1e3, "us": t, "usecond": t, "ms": t * 1e3, "msecond": t * 1e3}[tu]
        out[name] = {"dram_bytes": int(rd + wr), "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
                     "duration_us": us, "spans": spans, "bytes_per_span": (rd + wr) / spans,
                     "capture": capture, "workload": workload}
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    for k, v in out.items():
        print(f"{k:24s} {v['dram_bytes'] / 1e6:9.1f} MB {v['duration_us']:8.1f} us "
              f"{v['dram_bytes'] / v['duration_us'] / 1e3:7.0f} GB/s")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4])
