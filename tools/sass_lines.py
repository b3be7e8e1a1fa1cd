"""Attribute ncu per-instruction execution counts / stall samples of a kernel to CUDA source lines.
usage: python tools/sass_lines.py REP.ncu-rep KERNEL_MANGLED_NAME_SUBSTR  (needs the current libpdssm.so)"""
import collections
import csv
import io
import os
import re
import subprocess
import sys

rep, kname = sys.argv[1], sys.argv[2]
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 40
lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2605_19150_b200", "libpdssm.so")
tmp = "/tmp/_cub"
os.makedirs(tmp, exist_ok=True)
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
# split per function
funcs = {}
cur = None
line = None
for l in dis.split("\n"):
    m = re.match(r"^\.text\.(\S+):", l)
    if m:
        cur = m.group(1)
        funcs[cur] = {}
        continue
    m = re.search(r'//## File ".*?([^/]+)", line (\d+)', l)
    if m:
        line = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m and cur:
        funcs[cur][int(m.group(1), 16)] = (line, m.group(2).strip())
fn = [f for f in funcs if kname in f]
assert fn, "function not found"
fmap = funcs[fn[0]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
# the report may hold several kernels: take the block whose kernel name matches
blocks = out.split('"Kernel Name"')
best = None
for b in blocks[1:]:
    first = b.split("\n", 1)[0]
    if kname.split("I")[-1][:6] and True:
        rows = list(csv.reader(io.StringIO('"Kernel Name"' + b)))
        name = rows[0][1] if len(rows[0]) > 1 else ""
        sel = sys.argv[4] if len(sys.argv) > 4 else None
        if (sel and sel in name) or (not sel and (("fwd" in kname and "fwd" in name) or ("bwd" in kname and "bwd" in name))):
            best = rows
            break
rows = best
hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
h = rows[hi]
ai, ei, wi = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
fi = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
data = []
for r in rows[hi + 1:]:
    try:
        data.append((int(r[ai], 16), int(r[ei] or 0), int(r[wi] or 0), int(r[fi] or 0) if fi is not None else 0))
    except (ValueError, IndexError):
        pass
base = min(d[0] for d in data)
byline = collections.defaultdict(lambda: [0, 0, 0, 0])
for addr, n, w, f in data:
    ln, ins = fmap.get(addr - base, ("?", "?"))
    byline[ln][0] += n
    byline[ln][1] += w
    byline[ln][2] += 1
    byline[ln][3] += f
tot = sum(v[0] for v in byline.values())
tw = sum(v[1] for v in byline.values()) or 1
tf = sum(v[3] for v in byline.values()) or 1
print(f"total warp-inst {tot}  samples {tw}  smem wavefronts {tf}")
key = 3 if os.environ.get("SORT") == "wf" else 0
for ln, (n, w, c, f) in sorted(byline.items(), key=lambda x: -x[1][key])[:topn]:
    print(f"{ln:32s} inst={n:11d} ({100*n/tot:5.1f}%) stall={100*w/tw:5.1f}% wf={f:10d} ({100*f/tf:5.1f}%) sass={c}")
