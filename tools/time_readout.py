"""Time the a8 readout y = Re(C h) (pdssm_readout, tcgen05 3xTF32 / bf16) at the config-2 layer shape,
with the library variant / env switches of the caller: python tools/time_readout.py [f32|bf16]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_19150_b200 as P

B, L, H, N, c = 16, 2048, 8, 128, 2
Pp = N
dt = torch.bfloat16 if (len(sys.argv) > 1 and sys.argv[1] == "bf16") else torch.float32
g = torch.Generator(device="cuda").manual_seed(7)
h = torch.randn((B, H, L, c, N), device="cuda", generator=g).to(dt)
Cw = (torch.rand((H, c, Pp, N), device="cuda", generator=g) * 2 - 1) / N ** 0.5
y = torch.empty((B, L, H, Pp), device="cuda", dtype=dt)
dims = P.make_dims(B, H, L, N, 1, c=c, dtype=P.BF16 if dt == torch.bfloat16 else P.F32, p_out=Pp)
ws = torch.empty(max(P.workspace_bytes(dims, P.OP_READOUT), 256), dtype=torch.uint8, device="cuda")
for _ in range(3):
    P.readout(h, Cw, out=y, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
e0.record()
for _ in range(n):
    P.readout(h, Cw, out=y, ws=ws)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / n * 1e3
# parity on a sample of rows against a float64 product
hs = h[:2, :, :64].double().cpu()
hz = torch.complex(hs[..., 0, :], hs[..., 1, :])                     # [2][H][64][N]
Cz = torch.complex(Cw[:, 0].double().cpu(), Cw[:, 1].double().cpu())  # [H][P][N]
ref = torch.einsum("hpn,bhtn->bthp", Cz, hz).real
got = y[:2, :64].double().cpu()
err = float((got - ref).abs().max() / ref.abs().max())
byt = h.numel() * h.element_size() + y.numel() * y.element_size()
print(f"readout {dt} {us:.1f} us  {byt / us / 1e3:.0f} GB/s  rel_err {err:.2e}  variant={os.environ.get('PDSSM_LIB_VARIANT', '')} "
      f"wide={os.environ.get('PDSSM_READOUT_WIDE', '')}")
# per-kernel device durations (torch profiler, CUPTI): the GEMM alone vs the per-call weight split
try:
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            P.readout(h, Cw, out=y, ws=ws)
        torch.cuda.synchronize()
    for ev in prof.key_averages():
        if ev.device_type.name == "CUDA" or "pdssm" in ev.key:
            print(f"  {ev.key[:90]:90s} {ev.device_time_total / max(ev.count, 1):8.1f} us x{ev.count}")
except Exception as e:   # profiler unavailable: the wall-clock number above stands
    print("profiler:", e)
