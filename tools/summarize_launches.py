"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi and r[vi]:
        agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")) / 1000.0)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':70s} {'n':>4s} {'mean_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:70s} {len(v):4d} {sum(v)/len(v):9.1f} {100*sum(v)/tot:5.1f}%")
