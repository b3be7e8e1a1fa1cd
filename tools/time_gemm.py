"""Time the tensor-core select (a2/a3) and projection (a5) at config 2 (and the SIMT path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_19150_b200 as P

B, L, d_in, H, K, N, c = 16, 2048, 1024, 8, 32, 128, 2


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for dt in (torch.bfloat16, torch.float32):
    x = torch.randn(B, L, d_in, device="cuda").to(dt)
    S = (torch.rand(H, K, d_in, device="cuda") * 2 - 1).to(dt) / 32
    Bw = (torch.rand(H, c, N, d_in, device="cuda") * 2 - 1).to(dt) / 32
    out = torch.empty(B, H, L, c, N, device="cuda", dtype=dt)
    for path in ("auto", "generic"):
        if path == "generic":
            os.environ["PDSSM_PATH"] = "generic"
        else:
            os.environ.pop("PDSSM_PATH", None)
        ts = timeit(lambda: P.select(x, S))
        tp = timeit(lambda: P.project(x, Bw, out=out), n=5 if path == "generic" else 20)
        fs = 2.0 * B * L * H * K * d_in
        fp = 2.0 * B * L * H * c * N * d_in
        print(f"{str(dt):15s} {path:8s} select {ts*1e3:8.1f} us {fs/ts/1e9:7.1f} TF/s | project {tp*1e3:8.1f} us "
              f"{fp/tp/1e9:7.1f} TF/s", flush=True)
    os.environ.pop("PDSSM_PATH", None)
