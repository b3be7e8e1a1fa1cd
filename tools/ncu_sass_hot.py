"""Top SASS instructions by warp-stall samples from an .ncu-rep (source page)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
h = rows[hi]
ai, si, wi, ei = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[hi + 1:]:
    try:
        data.append((int(r[wi] or 0), r[ai], r[si], r[ei]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot)
for d in sorted(data, reverse=True)[:n]:
    print("%6d %5.1f%%  %s  %-70s %s" % (d[0], 100 * d[0] / tot, d[1][-5:], d[2][:70], d[3]))
