"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
k, v = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[start + 1:]:
    agg[r[k].split("(")[0][-48:]].append(float(r[v].replace(",", "")))
tot = sum(sum(x) for x in agg.values())
for name, xs in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{name:48s} n={len(xs):3d} avg={sum(xs)/len(xs)/1e3:9.2f}us  share={sum(xs)/tot*100:5.1f}%")
