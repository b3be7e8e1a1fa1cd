"""Sequence-parallel summary algebra on the GPU: G virtual ranks in one process
run segment summary -> (gather) -> compose -> local scan, and must reproduce the
single-pass result (maps bit-exact, floats within 1e-4), forward and backward."""
import numpy as np
import pytest

import oracle as O
import synth
from parity import check

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_19150_b200 as mod
    return mod


@pytest.fixture(params=["auto", "generic"])
def path(request, monkeypatch):
    monkeypatch.setenv("PDSSM_PATH", request.param)
    return request.param


# (N, tau, L): short chunks (generic per-chunk summaries) and chunks of >= 128 steps at N = 64 / 128,
# whose summaries take the chunked single-CTA Phase A / A' kernels (pdssm_segment_summary(_bwd))
@pytest.mark.parametrize("G,c,N,tau,L", [(2, 2, 32, 32, 301), (4, 1, 32, 32, 301), (3, 2, 32, 32, 301),
                                         (3, 1, 64, 128, 1000), (2, 2, 128, 256, 1100), (4, 1, 128, 128, 900)])
def test_sp_virtual_ranks(P, G, c, N, tau, L, path):
    B, H, K = 2, 2, 8
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=40 + G, h0=True, dh=True)
    dev = {k: torch.from_numpy(v).cuda() for k, v in inp.items()}
    di = dev["dict_idx"].to(torch.int16)
    bounds = [(g * L // G, (g + 1) * L // G) for g in range(G)]
    seg = lambda t, s, e: t[:, :, s:e].contiguous()
    dims_g = []
    summ = []
    for (s, e) in bounds:
        dims = P.make_dims(B, H, e - s, N, K, c=c, tau=tau)
        dims_g.append(dims)
        summ.append(P.segment_summary(seg(dev["kstar"], s, e), di, seg(dev["diag"], s, e), seg(dev["bias"], s, e), dims))
    gathered = torch.cat(summ)          # what all_gather_into_tensor produces
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, h0z = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "h0"))
    h_ref = O.scan_forward(Pm, Dz, bz, h0z)
    Pi, _ = O.prefix_maps(Pm, Dz)
    e_ref = O.planes_to_complex(inp["dh"])
    db_ref, dD_ref, g_ref, dh0_ref = O.scan_backward(Pm, Dz, h_ref, e_ref, h0z)
    fwd_out = []
    for g, (s, e) in enumerate(bounds):
        carry, m = P.compose_carry(gathered, g, G, dims_g[g], h0=dev["h0"])
        if s > 0:
            assert np.array_equal(m.cpu().numpy().astype(np.int64), Pi[:, :, s - 1])
            check("sp_1", O.planes_to_complex(carry.cpu().numpy()), h_ref[:, :, s - 1], 1e-4)
        f = P.scan_fwd(seg(dev["kstar"], s, e), di, seg(dev["diag"], s, e), seg(dev["bias"], s, e), h0=carry, tau=tau)
        fwd_out.append((f, carry))
        check("sp_2", O.planes_to_complex(f["h"].cpu().numpy()), h_ref[:, :, s:e], 1e-4)
    # backward: per-rank beta' summaries, gathered, composed from the right
    betas = []
    for g, (s, e) in enumerate(bounds):
        f, carry = fwd_out[g]
        betas.append(P.segment_summary_bwd(seg(dev["kstar"], s, e), di, seg(dev["diag"], s, e), f["chunk_state"],
                                           dims_g[g], dh=seg(dev["dh"], s, e)))
    beta_all = torch.stack(betas)
    for g, (s, e) in enumerate(bounds):
        f, carry = fwd_out[g]
        lam_in = P.compose_lambda(gathered, beta_all, g, G, dims_g[g])
        db, dD, gs, dh0 = P.scan_bwd(seg(dev["kstar"], s, e), di, seg(dev["diag"], s, e), f["h"], f["chunk_state"],
                                     dims_g[g], dh=seg(dev["dh"], s, e), h0=carry, lam_in=lam_in)
        check("sp_3", O.planes_to_complex(db.cpu().numpy()), db_ref[:, :, s:e], 1e-4)
        check("sp_4", O.planes_to_complex(dD.cpu().numpy()), dD_ref[:, :, s:e], 1e-4)
        check("sp_5", gs.cpu().numpy(), g_ref[:, :, s:e], 1e-4)
        if g == 0:
            check("sp_6", O.planes_to_complex(dh0.cpu().numpy()), dh0_ref, 1e-4)
