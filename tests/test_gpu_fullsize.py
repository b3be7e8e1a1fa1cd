"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (the library
default path: one CTA per sequence at config 2), on sampled outputs the float64 oracle computes
one sequence at a time, plus properties that hold at any size (finite, run-to-run bitwise).
Sampled sequences are sliced out of the same seeded inputs the bench generates."""
import numpy as np
import pytest

import oracle as O
import synth
from parity import check, rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_19150_b200 as mod
    return mod


def sampled_check(inp, f, bwd, seqs, tol, bf16=False):
    """Oracle forward + backward of each sampled (b, h) sequence against the GPU's outputs.  bf16:
    the oracle's backward reads its own states rounded to bf16, as the kernel reads h_saved (R16)."""
    db, dD, g, _ = (None if t is None else t.float().cpu().numpy() for t in bwd)
    h_all = f["h"].float().cpu().numpy()
    c = inp["bias"].shape[-2]
    for (b, hh) in seqs:
        sl = lambda a: a[b:b + 1, hh:hh + 1]
        Pm = O.gather_P(inp["dict_idx"][hh:hh + 1], sl(inp["kstar"]))
        Dz, bz, e = (O.planes_to_complex(sl(inp[k])) for k in ("diag", "bias", "dh"))
        h = O.scan_forward(Pm, Dz, bz)
        hs = O.planes_to_complex(synth.round_bf16(O.complex_to_planes(h, c).astype(np.float32))) if bf16 else h
        db_r, dD_r, g_r, _ = O.scan_backward(Pm, Dz, hs, e)
        cp = lambda t: O.planes_to_complex(sl(t))
        check("h", cp(h_all), h, tol)
        check("db", cp(db), db_r, tol)
        check("dD", cp(dD), dD_r, tol)
        check("g", sl(g), g_r, tol)


def run(P, inp, bf16):
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()}
    d["dict_idx"] = d["dict_idx"].to(torch.int16)
    if bf16:
        for k in ("diag", "bias", "dh"):
            d[k] = d[k].to(torch.bfloat16)
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"])
    bwd = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"], dh=d["dh"])
    torch.cuda.synchronize()
    return d, f, bwd


def test_config2_bench_launch(P):
    """Config 2 (B 16, L 2048, H 8, N 128, K 32, complex fp32): the bench's exact shape and path."""
    B, H, L, N, K, c = 16, 8, 2048, 128, 32, 2
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=2000, dh=True)   # bench.py's default seed, rank 0
    d, f, bwd = run(P, inp, False)
    assert f["tau"] == L   # single-chunk path, as timed
    for t in (f["h"],) + tuple(x for x in bwd if x is not None):
        assert bool(torch.isfinite(t).all())
    # every one of the 128 sequences (the oracle needs ~25 ms per sequence)
    sampled_check(inp, f, bwd, [(b, hh) for b in range(B) for hh in range(H)], 1e-4)
    f2 = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"])
    b2 = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f2["h"], f2["chunk_state"], f2["dims"], dh=d["dh"])
    torch.cuda.synchronize()
    assert torch.equal(f["h"], f2["h"]) and torch.equal(bwd[0], b2[0]) and torch.equal(bwd[1], b2[1])
    assert torch.equal(bwd[2], b2[2])


def test_config2_dict_grad_sampled(P):
    """NEXT-1 dictionary gradient at config 2: G[h, k] for sampled (h, k) from the oracle's own scans
    over every sequence of head h."""
    B, H, L, N, K, c = 16, 8, 2048, 128, 32, 2
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=2000, dh=True)
    d, f, bwd = run(P, inp, False)
    M = torch.from_numpy(synth.dictionary(H, K, N, 2001)).cuda()
    dM, G = P.dict_grad(M, d["kstar"], d["diag"], f["h"], bwd[0], 1.0, f["dims"], want_G=True)
    torch.cuda.synchronize()
    hh = 5
    sl = lambda a: a[:, hh:hh + 1]
    Pm = O.gather_P(inp["dict_idx"][hh:hh + 1], sl(inp["kstar"]))
    Dz, bz, e = (O.planes_to_complex(sl(inp[k])) for k in ("diag", "bias", "dh"))
    h = O.scan_forward(Pm, Dz, bz)
    lam = O.scan_backward(Pm, Dz, h, e)[0]
    G_ref = O.dictionary_outer(sl(inp["kstar"]), lam, Dz, h, K)[0]
    assert rel(G[hh].cpu().numpy(), G_ref) <= 1e-4
    dM_ref = O.dictionary_grad(M[hh:hh + 1].cpu().numpy().astype(np.float64), G_ref[None], 1.0)[0]
    assert rel(dM[hh].cpu().numpy(), dM_ref) <= 1e-4


def test_config4_bf16_sampled(P):
    """Config 4 (B 32, H 32, L 4096, N 64, K 48, real bf16): 1024 sequences, several CTAs per SM."""
    B, H, L, N, K, c = 32, 32, 4096, 64, 48, 1
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=4000, dh=True, bf16=True)
    d, f, bwd = run(P, inp, True)
    # 128 of the 1024 sequences: every head, four batch rows each (strided)
    sampled_check(inp, f, bwd, [(b, hh) for hh in range(H) for b in (hh % 8, 8 + hh % 8, 16 + hh % 8, 31 - hh % 8)],
                  2e-2, bf16=True)


def test_config5_s5_full_length(P):
    """Config 5 (S_5 word problem, L = 65536, N 64, K 16, B 4, H 4, PER_DICT D = 1, b = 0,
    h0 = arange): exact permuted states at the end and exact final maps, every sequence."""
    dict_idx, _, _ = synth.s5_dictionary(64, 16, seed=5000)
    B, H, L, N = 4, 4, 65536, 64
    k = synth.kstar(B, H, L, 16, seed=5001)
    di = torch.from_numpy(np.tile(dict_idx[None], (H, 1, 1)).astype(np.int16)).cuda()
    diag = torch.ones((H, 16, 1, N), dtype=torch.float32, device="cuda")
    bias = torch.zeros((B, H, L, 1, N), dtype=torch.float32, device="cuda")
    h0 = torch.arange(N, dtype=torch.float32, device="cuda").view(1, 1, 1, N).repeat(B, H, 1, 1).contiguous()
    f = P.scan_fwd(torch.from_numpy(k).cuda(), di, diag, bias, h0=h0, per_dict=True, export_maps=True)
    torch.cuda.synchronize()
    # final composed map by the oracle's own fold (integer, exact)
    Pm = O.gather_P(np.tile(dict_idx[None], (H, 1, 1)), k)
    Pi, _ = O.prefix_maps(Pm, np.ones(Pm.shape))
    assert np.array_equal(f["maps"].cpu().numpy().astype(np.int64)[:, :, -1], Pi[:, :, -1])
    hlast = f["h"][:, :, -1, 0].cpu().numpy()
    expect = np.zeros((B, H, N))
    np.put_along_axis(expect, Pi[:, :, -1], np.arange(float(N))[None, None].repeat(B, 0).repeat(H, 1), axis=2)
    assert np.array_equal(hlast, expect)


def test_config3_sequence_parallel_full_length(P):
    """Config 3 (L = 17984, B 4, H 8, N 128, real fp32, temporally persistent k*): the sequence-
    parallel construction with G = 8 virtual ranks (segments of 2248 steps, ragged against tau)
    -- segment summaries, rank-ordered composition, local scans, and the mirrored backward (beta'
    summaries composed from the right into each segment's incoming adjoint) -- against the oracle
    on sampled sequences, and the composed carries' index maps bit-exact."""
    B, H, L, N, K, c, G = 4, 8, 17984, 128, 32, 1, 8
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=3000, h0=True, sticky=0.9, dh=True)
    dev = {k: torch.from_numpy(v).cuda() for k, v in inp.items()}
    di = dev["dict_idx"].to(torch.int16)
    bounds = [(g * L // G, (g + 1) * L // G) for g in range(G)]
    seg = lambda t, s, e: t[:, :, s:e].contiguous()
    dims_g = [P.make_dims(B, H, e - s, N, K, c=c) for (s, e) in bounds]
    gathered = torch.cat([P.segment_summary(seg(dev["kstar"], s, e), di, seg(dev["diag"], s, e),
                                            seg(dev["bias"], s, e), dims_g[g]) for g, (s, e) in enumerate(bounds)])
    hs, maps, fwd = [], [], []
    for g, (s, e) in enumerate(bounds):
        carry, m = P.compose_carry(gathered, g, G, dims_g[g], h0=dev["h0"])
        maps.append(m)
        f = P.scan_fwd(seg(dev["kstar"], s, e), di, seg(dev["diag"], s, e), seg(dev["bias"], s, e), h0=carry)
        fwd.append((f, carry))
        hs.append(f["h"])
    # the mirrored backward: per-segment beta' summaries, composed from the right (lam_in)
    betas = torch.stack([P.segment_summary_bwd(seg(dev["kstar"], s, e), di, seg(dev["diag"], s, e), fwd[g][0]["chunk_state"],
                                               dims_g[g], dh=seg(dev["dh"], s, e)) for g, (s, e) in enumerate(bounds)])
    dbs, gs = [], []
    for g, (s, e) in enumerate(bounds):
        f, carry = fwd[g]
        lam_in = P.compose_lambda(gathered, betas, g, G, dims_g[g])
        db, _, gg, _ = P.scan_bwd(seg(dev["kstar"], s, e), di, seg(dev["diag"], s, e), f["h"], f["chunk_state"], dims_g[g],
                                  dh=seg(dev["dh"], s, e), h0=carry, lam_in=lam_in, want_dh0=False)
        dbs.append(db)
        gs.append(gg)
    torch.cuda.synchronize()
    for (b, hh) in [(0, 0), (3, 7), (2, 4)]:
        sl = lambda a: a[b:b + 1, hh:hh + 1]
        Pm = O.gather_P(inp["dict_idx"][hh:hh + 1], sl(inp["kstar"]))
        Dz, bz, h0z = (O.planes_to_complex(sl(inp[k])) for k in ("diag", "bias", "h0"))
        h_ref = O.scan_forward(Pm, Dz, bz, h0z)
        Pi, _ = O.prefix_maps(Pm, np.ones(Pm.shape))
        got = np.concatenate([O.planes_to_complex(x[b:b + 1, hh:hh + 1].cpu().numpy()) for x in hs], axis=2)
        check("sp8_h", got, h_ref, 1e-4)
        db_r, _, g_r, _ = O.scan_backward(Pm, Dz, h_ref, O.planes_to_complex(sl(inp["dh"])), h0z)
        check("sp8_db", np.concatenate([O.planes_to_complex(x[b:b + 1, hh:hh + 1].cpu().numpy()) for x in dbs], axis=2),
              db_r, 1e-4)
        check("sp8_g", np.concatenate([x[b:b + 1, hh:hh + 1].cpu().numpy() for x in gs], axis=2), g_r, 1e-4)
        for g, (s, e) in enumerate(bounds):
            if s > 0:
                assert np.array_equal(maps[g][b, hh].cpu().numpy().astype(np.int64), Pi[0, 0, s - 1])
