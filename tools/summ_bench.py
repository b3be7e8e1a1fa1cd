"""One-line summaries of bench JSON lines (gpurun_out/*bench*.json)."""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as ex:
        print(p, "unreadable", ex)
        continue
    if "roofline" not in d:
        print(p, "value", d.get("value"), d.get("cpu_baseline", {}).get("value_1core"))
        continue
    s, r = d["step_hbm"], d["roofline"]
    print(f"{p.split('/')[-1]:28s} {d['value'] / 1e6:8.2f} Mtok/s  step {s['step_ms_median']:.4f} ms  "
          f"fwd {s['fwd_ms_median']:.4f} bwd {s['bwd_ms_median']:.4f}  step_frac {s['frac']:.3f}  "
          f"dom {r['kernel']} {r['frac']:.3f}  tau {d['config']['tau']}  seeds {[round(v / 1e6, 1) for v in d['seeds']['values']]}"
          f"  clocks {d['clocks'] and d['clocks']['sm_mhz']} e2e {d['e2e'] and round(d['e2e']['value'] / 1e6, 2)}")
