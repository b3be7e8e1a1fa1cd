"""One launch each of the tcgen05 GEMM variants at the config-2 layer shape (B 16, L 2048,
d_in 1024, H 8, K 32, N 128, c 2, P 128), for an ncu capture of the tensor pipe:
select (fp32 3xTF32, bf16), projection (fp32, bf16), readout (fp32), D_t generator (fp32)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_19150_b200 as P  # noqa: E402

B, L, d_in, H, K, N, c, Pp = 16, 2048, 1024, 8, 32, 128, 2, 128
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(B, L, d_in, device="cuda", generator=g)
S = torch.randn(H, K, d_in, device="cuda", generator=g) / 32
Bw = torch.randn(H, c, N, d_in, device="cuda", generator=g) / 32
Cw = torch.randn(H, c, Pp, N, device="cuda", generator=g) / 12
bmag = torch.zeros(H, N, device="cuda")
for _ in range(2):   # warm-up (also the launches ncu skips with -s)
    P.select(x, S)
    P.select(x.bfloat16(), S.bfloat16())
    b = P.project(x, Bw)
    P.project(x.bfloat16(), Bw.bfloat16())
    P.readout(b, Cw)
    P.diag_gen(x, Bw, bmag)
torch.cuda.synchronize()
print("gemm driver done")
