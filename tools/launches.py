"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel:
launches, total us, DRAM MB read+write, GB/s."""
import csv
import sys
from collections import OrderedDict


def main(path, skip_ids=0):
    rows = OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if int(r["ID"]) < skip_ids:
            continue
        k = r["Kernel Name"].split("(")[0]
        key = (int(r["ID"]), k)
        d = rows.setdefault(key, {})
        v = float(r["Metric Value"].replace(",", ""))
        d[r["Metric Name"]] = v
    agg = OrderedDict()
    for (i, k), d in rows.items():
        a = agg.setdefault(k, [0, 0.0, 0.0])
        a[0] += 1
        t = d.get("gpu__time_duration.sum", 0.0)
        a[1] += t / 1e3  # ns -> us
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':40s} {'n':>4s} {'us':>10s} {'share':>6s} {'MB':>9s} {'GB/s':>7s}")
    for k, (n, us, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:40]:40s} {n:4d} {us:10.1f} {us / tot * 100:5.1f}% {b / 1e6:9.1f} {b / us / 1e3 if us else 0:7.0f}")
    print(f"total {tot:.1f} us, {sum(a[2] for a in agg.values()) / 1e6:.1f} MB")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
