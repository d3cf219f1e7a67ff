"""Summarise an ncu --csv launch list (gpu__time_duration) per kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[ui], 1.0)
    agg.setdefault(r[ki][:80], []).append(v * scale)
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"{len(v):4d} x {sum(v)/len(v):10.2f} us  {100*sum(v)/tot:5.1f}%  {k}")
