import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ii = h.index("ID")
out = {}
for r in rows[hi + 1:]:
    key = (r[ii], r[ki].split("(")[0].split("<")[0].split("::")[-1])
    out.setdefault(key, {})[r[mi]] = r[vi]
short = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "rdMB", "dram__bytes_write.sum": "wrMB",
         "lts__t_sector_hit_rate.pct": "l2hit", "smsp__inst_executed.sum": "Minst",
         "sm__inst_executed.avg.per_cycle_active": "ipc",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "Mwf_sh",
         "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "lsu%",
         "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "Mconf"}
scale = {"us": 1e-3, "rdMB": 1e-6, "wrMB": 1e-6, "Minst": 1e-6, "Mwf_sh": 1e-6, "Mconf": 1e-6}
for (i, k), m in out.items():
    parts = []
    for n, v in m.items():
        s = short.get(n, n)
        try:
            x = float(v.replace(",", "")) * scale.get(s, 1.0)
            parts.append(f"{s}={x:.4g}")
        except ValueError:
            parts.append(f"{s}={v}")
    print(k, " ".join(parts))
