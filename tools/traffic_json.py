"""Write profiles/traffic_latest.json: dram read+write bytes per launch of the scan kernels
from an ncu --set full capture (bench.py reports it as roofline.traffic)."""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
prefix = sys.argv[3] if len(sys.argv) > 3 else ""   # e.g. "config4:" (merged into an existing file)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
k, rd, wr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
unit_rd, unit_wr = rows[1][rd], rows[1][wr]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = {}
for r in rows[2:]:
    name = r[k]
    key = "scan_fwd" if ("k_fwd_fused" in name or "k_fwd_seq" in name) else "scan_bwd" if ("k_bwd_fused" in name or "k_bwd_seq" in name) else None
    if key is None:
        continue
    b = float(r[rd].replace(",", "")) * scale.get(unit_rd, 1) + float(r[wr].replace(",", "")) * scale.get(unit_wr, 1)
    res.setdefault(key, []).append(b)
res = {prefix + key: sum(v) / len(v) for key, v in res.items()}
try:
    old = json.load(open(out))
except (OSError, ValueError):
    old = {}
old.update(res)
old.setdefault("sources", {})[prefix or "config2:"] = rep
old.pop("source", None)
with open(out, "w") as f:
    json.dump(old, f, indent=1)
print(json.dumps(res))
