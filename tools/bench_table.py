"""Markdown table of bench JSON lines (for DESIGN.md): config, dtype, tokens/s, step / fwd / bwd
median ms, step HBM fraction, dominant kernel and its fraction, seeds min-max, e2e."""
import json
import sys

print("| line | workload | dtype | M tok/s | step ms | fwd ms | bwd ms | step HBM frac | dominant (frac) | seeds M tok/s | e2e M tok/s |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for p in sys.argv[1:]:
    d = json.loads(open(p).read().strip().splitlines()[-1])
    s, r, c = d["step_hbm"], d["roofline"], d["config"]
    sd = d.get("seeds", {})
    e2e = d.get("e2e") or {}
    name = p.split("/")[-1].replace(".json", "")
    wl = c["workload"].split(":")[0] + (", recompute" if c.get("backward", "").startswith("recompute") else "")
    print(f"| {name} | {wl}, tau {c['tau']} | {d['dtype']} | {d['value'] / 1e6:.1f} | {s['step_ms_median']:.3f} | "
          f"{s['fwd_ms_median']:.3f} | {s['bwd_ms_median']:.3f} | {s['frac']:.2f} | {r['kernel']} ({r['frac']:.2f}) | "
          f"{sd.get('min', 0) / 1e6:.1f}-{sd.get('max', 0) / 1e6:.1f} | "
          f"{(e2e.get('value') or 0) / 1e6:.2f} |")
