"""Summarise an ncu --metrics launch list (CSV): per kernel, launches, mean device time and its
share, and (when captured) DRAM read+write bytes per launch."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
mi = h.index("Metric Name") if "Metric Name" in h else None
ii = h.index("ID") if "ID" in h else None
vals = defaultdict(lambda: defaultdict(list))
for r in rows[hi + 1:]:
    if len(r) <= vi or not r[vi]:
        continue
    name = r[ki].split("(")[0][:70]
    metric = r[mi] if mi is not None else "gpu__time_duration.sum"
    vals[name][metric].append(float(r[vi].replace(",", "")))
tot = sum(sum(m.get("gpu__time_duration.sum", [])) for m in vals.values())
print(f"{'kernel':70s} {'n':>4s} {'mean_us':>9s} {'share':>6s} {'dram_MB':>9s}")
for k, m in sorted(vals.items(), key=lambda x: -sum(x[1].get("gpu__time_duration.sum", []))):
    t = m.get("gpu__time_duration.sum", [])
    n = len(t)
    rd, wr = m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", [])
    mb = (sum(rd) + sum(wr)) / max(n, 1) / 1e6 if rd else float("nan")
    print(f"{k:70s} {n:4d} {sum(t) / max(n, 1) / 1000:9.1f} {100 * sum(t) / max(tot, 1):5.1f}% {mb:9.1f}")
