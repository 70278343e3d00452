"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

python tools/ncu_launches.py gpurun_out/launches.csv
"""
import csv
import sys
from collections import OrderedDict


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    for k, (n, t) in agg.items():
        print(f"{k:60s} n={n:4d} total={t:10.1f} us  avg={t / n:9.1f} us  share={100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main()
