"""Time the fwd / bwd scan of the headline workload on both kernel paths."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_19150_b200 as P
import synth

B, H, L, N, K, c = 16, 8, 2048, int(os.environ.get("N", 128)), 32, int(os.environ.get("C", 2))
tau = int(os.environ.get("TAU", 0))
inp = synth.scan_inputs(B, H, L, N, K, c, seed=2000, dh=True)
d = {k: torch.from_numpy(v).cuda() for k, v in inp.items()}
d["dict_idx"] = d["dict_idx"].to(torch.int16)
ref = None
for path in os.environ.get("PATHS", "fused,seq").split(","):
    os.environ["PDSSM_PATH"] = path
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], tau=tau)
    r = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"], dh=d["dh"])
    torch.cuda.synchronize()
    ts = []
    for i in range(10):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], tau=tau)
        e1.record()
        r = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"], dh=d["dh"])
        e2.record()
        torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    ts = np.array(ts[2:])
    print(path, "tau", f["tau"], "fwd ms %.3f bwd ms %.3f" % tuple(ts.mean(0)), flush=True)
    if ref is None:
        ref = (f["h"].clone(), r[0].clone(), r[1].clone(), r[2].clone())
    else:
        for name, a, b in zip(["h", "db", "dD", "g"], ref, (f["h"], r[0], r[1], r[2])):
            err = (a - b).abs().max().item() / max(a.abs().max().item(), 1e-30)
            print("  rel diff vs first path", name, "%.2e" % err)
