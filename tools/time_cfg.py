"""Time fwd+bwd scan for an arbitrary shape on the given paths: python tools/time_cfg.py B H L N K c dtype [paths]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_19150_b200 as P
import synth

B, H, L, N, K, c = (int(x) for x in sys.argv[1:7])
bf16 = sys.argv[7] == "bf16"
paths = (sys.argv[8] if len(sys.argv) > 8 else "auto,fused").split(",")
inp = synth.scan_inputs(B, H, L, N, K, c, seed=3, dh=True, bf16=bf16)
d = {k: torch.from_numpy(v).cuda() for k, v in inp.items()}
d["dict_idx"] = d["dict_idx"].to(torch.int16)
if bf16:
    for k in ("diag", "bias", "dh"):
        d[k] = d[k].to(torch.bfloat16)
p = 2 if bf16 else 4
byt = (3 * c * N * p + 1 + 5 * c * N * p + 5) * B * H * L
for path in paths:
    if path == "auto":
        os.environ.pop("PDSSM_PATH", None)
    else:
        os.environ["PDSSM_PATH"] = path
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"])
    r = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"], dh=d["dh"])
    torch.cuda.synchronize()
    ts = []
    for i in range(6):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"])
        e1.record()
        r = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"], dh=d["dh"])
        e2.record()
        torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    ts = np.array(ts[2:]).mean(0)
    tot = ts.sum()
    print(f"{path:6s} tau {int(f['tau']):6d} fwd {ts[0]:.3f} bwd {ts[1]:.3f} ms  {B*L/tot/1e3:.1f} M tok/s  {byt/tot/1e6:.0f} GB/s",
          flush=True)
