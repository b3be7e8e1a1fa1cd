"""Graph-timed pdssm_dict_grad at the config-2 shape (PDSSM_LIB_VARIANT selects a variant build)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_19150_b200 as P

B, H, L, N, K, c = 16, 8, 2048, 128, 32, 2
g = torch.Generator(device="cuda").manual_seed(1)
ks = torch.randint(0, K, (B, H, L), device="cuda", generator=g).to(torch.uint8)
D = torch.randn((B, H, L, c, N), device="cuda", generator=g)
h = torch.randn((B, H, L, c, N), device="cuda", generator=g)
lam = torch.randn((B, H, L, c, N), device="cuda", generator=g)
M = torch.randn((H, K, N, N), device="cuda", generator=g)
dM = torch.empty_like(M)
dims = P.make_dims(B, H, L, N, K, c=c)
fn = lambda: P.dict_grad(M, ks, D, h, lam, 1.0, dims, out=dM)
for _ in range(3):
    fn()
torch.cuda.synchronize()
st = torch.cuda.Stream()
gr = torch.cuda.CUDAGraph()
with torch.cuda.stream(st), torch.cuda.graph(gr, stream=st):
    for _ in range(10):
        fn()
torch.cuda.synchronize()
gr.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
gr.replay()
e1.record()
torch.cuda.synchronize()
print(os.environ.get("PDSSM_LIB_VARIANT", "main"), "dict_grad us", e0.elapsed_time(e1) / 10 * 1e3)
