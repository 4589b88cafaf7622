"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(list)
for r in rows[h + 1:]:
    if len(r) > vi:
        agg[r[ki].split("(")[0][:90]].append(float(r[vi].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):10.3f} us  x{len(v):3d}  {100 * sum(v) / tot:5.1f}%  {k}")
