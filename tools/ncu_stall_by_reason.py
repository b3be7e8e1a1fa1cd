"""Top SASS instructions of one kernel by a given stall reason, from an .ncu-rep source page.
usage: python tools/ncu_stall_by_reason.py REP KERNEL_SUBSTR REASON [N]   (REASON e.g. stall_long_sb)"""
import csv
import io
import subprocess
import sys

rep, kpat, reason = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur, name = [], None, None
for r in rows:
    if r and r[0] == "Kernel Name":
        name = r[1]
        continue
    if "Address" in r and "Source" in r:
        cur = {"name": name, "h": r, "rows": []}
        blocks.append(cur)
        continue
    if cur is not None:
        cur["rows"].append(r)
for b in blocks:
    if kpat not in (b["name"] or ""):
        continue
    h = b["h"]
    ai, si, ri, ei = h.index("Address"), h.index("Source"), h.index(reason), h.index("Instructions Executed")
    tot = sum(int(r[ri] or 0) for r in b["rows"] if len(r) > ri and (r[ri] or "0").isdigit())
    print(b["name"][:90], reason, "total", tot)
    data = sorted(((int(r[ri]), r[ai], r[si], r[ei]) for r in b["rows"] if len(r) > ri and (r[ri] or "").isdigit()),
                  reverse=True)[:n]
    for v, a, s, e in data:
        print(f"{v:7d} {a:>8s} {s[:70]:70s} {e}")
    break
