#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel count, total and mean time (our kernels only unless --all)."""
import collections
import csv
import sys

path = sys.argv[1]
show_all = "--all" in sys.argv
rows = list(csv.reader(open(path)))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        n = d["Kernel Name"].split("(")[0]
        if not show_all and "kwb" not in n:
            continue
        unit = d.get("Metric Unit", "ns")
        v = float(d["Metric Value"].replace(",", ""))
        v = v / 1e6 if unit == "ns" else (v / 1e3 if unit == "us" else v)
        agg.setdefault(n, []).append(v)
tot = sum(sum(v) for v in agg.values())
for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):10.3f} ms {100 * sum(v) / tot:5.1f}%  n={len(v):3d}  mean {sum(v) / len(v):8.3f} ms  {n}")
