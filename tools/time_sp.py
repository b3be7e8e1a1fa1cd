"""Time the sequence-parallel segment summaries (pdssm_segment_summary / _bwd) of one rank's segment
at configs 3 and 5 with G = 8 (the per-rank work of bench.py --mode sp), default dispatch vs the
generic per-chunk kernels (PDSSM_PATH=generic): python tools/time_sp.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_19150_b200 as P
import synth


def timeit(fn, n=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for name, (B, H, L, N, K, c, pd) in {"config3_G8": (4, 8, 17984 // 8, 128, 32, 1, False),
                                      "config5_G8": (4, 4, 65536 // 8, 64, 16, 1, True)}.items():
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=5, per_dict=pd, dh=True)
    d = {k: torch.from_numpy(v).cuda() for k, v in inp.items()}
    d["dict_idx"] = d["dict_idx"].to(torch.int16)
    for path in ("default", "generic"):
        if path == "generic":
            os.environ["PDSSM_PATH"] = "generic"
        else:
            os.environ.pop("PDSSM_PATH", None)
        dims = P.make_dims(B, H, L, N, K, c=c, diag_mode=P.PER_DICT if pd else P.PER_STEP)
        f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], per_dict=pd)
        tf = timeit(lambda: P.segment_summary(d["kstar"], d["dict_idx"], d["diag"], d["bias"], dims))
        tb = timeit(lambda: P.segment_summary_bwd(d["kstar"], d["dict_idx"], d["diag"], f["chunk_state"], dims, dh=d["dh"]))
        print(f"{name} {path:8s} tau {f['tau']:5d}  summary fwd {tf * 1e3:8.1f} us  bwd {tb * 1e3:8.1f} us")
