"""SequenceParallelScan(CudaOps) end to end on the GPU with two real processes (world size 2,
gloo; both ranks share cuda:0 and the all-gathers are staged through the host): segment
summary -> all-gather in rank order -> compose -> local scan, and the mirrored backward, against
the float64 oracle of the whole sequence (associativity PAPER.md:927-932).
Index maps bit-exact, floats within 1e-4 (per tensor and per (b, h))."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import synth
from parity import check

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, args, outdir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(WORLD))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    import paper_2605_19150_b200 as P
    from paper_2605_19150_b200.parallel import CudaOps, SequenceParallelScan, shard_range
    B, H, L, N, K, c, tau, seed = args
    torch.cuda.set_device(0)
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=seed, h0=True, dh=True)   # generated globally ...
    s, e = shard_range(L, WORLD, rank)                                       # ... then sliced
    seg = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, :, s:e])).cuda()
    kst, D, b, dh = seg(inp["kstar"]), seg(inp["diag"]), seg(inp["bias"]), seg(inp["dh"])
    di = torch.from_numpy(inp["dict_idx"]).cuda().to(torch.int16)
    h0 = torch.from_numpy(inp["h0"]).cuda()          # the global initial state, on every rank
    sp = SequenceParallelScan(CudaOps(N, K, c, tau=tau))
    out, ctx = sp.forward(kst, di, D, b, h0=h0)
    db, dD, g, dh0 = sp.backward(kst, di, D, out, ctx, dh)
    torch.cuda.synchronize()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), h=out["h"].cpu().numpy(), db=db.cpu().numpy(),
             dD=dD.cpu().numpy(), g=g.cpu().numpy(), dh0=dh0.cpu().numpy(),
             prefix_map=ctx["prefix_map"].cpu().numpy() if ctx["prefix_map"] is not None else np.zeros(0),
             s=s, e=e, tau=out["tau"])
    dist.destroy_process_group()


@pytest.mark.parametrize("args", [
    (2, 2, 301, 32, 8, 2, 0, 11),        # small B*H: the chunked fast path inside each segment
    (16, 8, 160, 128, 8, 2, 0, 12),      # B*H = 128: each segment's forward takes the single-chunk kernel
    (2, 3, 257, 64, 16, 1, 32, 13),      # explicit tau, ragged segments
])
def test_sequence_parallel_two_processes(args, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(_free_port(), args, str(tmp_path)), nprocs=WORLD, join=True)
    B, H, L, N, K, c, tau, seed = args
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=seed, h0=True, dh=True)
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, e, h0z = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "dh", "h0"))
    h = O.scan_forward(Pm, Dz, bz, h0z)
    db_r, dD_r, g_r, dh0_r = O.scan_backward(Pm, Dz, h, e, h0z)
    Pi, _ = O.prefix_maps(Pm, Dz)
    for r in range(WORLD):
        z = np.load(os.path.join(str(tmp_path), f"r{r}.npz"))
        s, e_ = int(z["s"]), int(z["e"])
        check("sp2_h", O.planes_to_complex(z["h"]), h[:, :, s:e_], 1e-4)
        check("sp2_db", O.planes_to_complex(z["db"]), db_r[:, :, s:e_], 1e-4)
        check("sp2_dD", O.planes_to_complex(z["dD"]), dD_r[:, :, s:e_], 1e-4)
        check("sp2_g", z["g"], g_r[:, :, s:e_], 1e-4)
        if r == 0:
            check("sp2_dh0", O.planes_to_complex(z["dh0"]), dh0_r, 1e-4)
        else:
            assert np.array_equal(z["prefix_map"].astype(np.int64), Pi[:, :, s - 1])   # bit-exact
