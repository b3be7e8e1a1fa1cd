"""Summarise an .ncu-rep (details page) for the kernels matching a pattern."""
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, si, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Value", "Metric Unit"))
keep = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis", "Scheduler Statistics",
        "Warp State Statistics", "Occupancy", "Launch Statistics")
seen = set()
for r in rows[1:]:
    if pat in r[ki] and r[si] in keep and (r[si], r[mi]) not in seen:
        seen.add((r[si], r[mi]))
        print(f"{r[si][:22]:22s} | {r[mi][:48]:48s} | {r[vi]} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_bytes.sum",
        "smsp__average_warp_latency_issue_stalled_barrier", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
for r in rr[2:]:
    if pat in r[hh.index("Kernel Name")]:
        for w in want:
            if w in hh:
                print(f"{w:60s} {r[hh.index(w)]} {rr[1][hh.index(w)]}")
# stall reasons
for r in rr[2:]:
    if pat in r[hh.index("Kernel Name")]:
        st = [(hh[i], r[i]) for i in range(len(hh)) if hh[i].startswith("smsp__average_warps_issue_stalled_") and hh[i].endswith("_per_issue_active.ratio")]
        st = sorted(((float(v), n) for n, v in st if v not in ("", "n/a")), reverse=True)[:8]
        for v, n in st:
            print(f"stall {n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v:.2f}")
