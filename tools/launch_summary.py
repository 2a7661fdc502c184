"""Summarise an ncu --csv launch list (gpu__time_duration.sum): total per kernel name.
python tools/launch_summary.py gpurun_out/x.csv"""
import csv
import sys
from collections import defaultdict

lines = open(sys.argv[1]).read().splitlines()
start = [n for n, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(list)
for r in rows[1:]:
    sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
    agg[r[ki].split("(")[0].replace("void ", "")[:70]].append(float(r[vi].replace(",", "")) * sc)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):10.1f} us {len(v):4d}x  {100 * sum(v) / tot:5.1f}%  {k}")
