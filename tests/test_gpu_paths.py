"""Path-coverage parity (GPU vs the float64 oracle, reading R19 bars via tests/parity.py):

* the ABI's extreme shapes: K = 256 (N = 32 and 128, chunked fast path and generic) and
  N = 1024 (generic);
* hypothesis-randomised small shapes (B, H, L, N, K, c, tau, dtype) through the default dispatch;
* a forward taken by the single-chunk kernel followed by a backward that takes another path,
  with an incoming adjoint;
* the sequence-parallel backward summary after a single-chunk forward (tau = 0, many sequences);
* the autograd glue with non-contiguous (permuted) inputs."""
import os

import numpy as np
import pytest

import oracle as O
import synth
from parity import TOL, check

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_19150_b200 as mod
    return mod


def to_dev(inp, bf16):
    d = {}
    for k, v in inp.items():
        t = torch.from_numpy(np.ascontiguousarray(v)).cuda()
        if k == "dict_idx":
            t = t.to(torch.int16)
        elif bf16 and k in ("bias", "dh", "diag"):
            t = t.to(torch.bfloat16)
        d[k] = t
    return d


def rounded(h, c, bf16):
    if not bf16:
        return h
    return O.planes_to_complex(synth.round_bf16(O.complex_to_planes(h, c).astype(np.float32)))


def fwd_bwd_check(P, B, H, L, N, K, c, tau, bf16=False, seed=0, h0=True):
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=seed, h0=h0, dh=True, bf16=bf16)
    d = to_dev(inp, bf16)
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=d.get("h0"), tau=tau, export_maps=True)
    db, dD, g, dh0 = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"],
                                dh=d["dh"], h0=d.get("h0"))
    torch.cuda.synchronize()
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, e = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "dh"))
    h0z = O.planes_to_complex(inp["h0"]) if h0 else None
    ch = O.scan_chunked(Pm, Dz, bz, f["tau"], h0z)
    tol = TOL["bf16" if bf16 else "f32"]
    cp = lambda t: O.planes_to_complex(t.float().cpu().numpy())
    check("h", cp(f["h"]), ch["h"], tol)
    assert np.array_equal(f["maps"].cpu().numpy().astype(np.int64), ch["maps"])
    db_r, dD_r, g_r, dh0_r = O.scan_backward(Pm, Dz, rounded(ch["h"], c, bf16), e, h0z)
    check("db", cp(db), db_r, tol)
    check("dD", cp(dD), dD_r, tol)
    check("g", g.cpu().numpy(), g_r, tol)
    check("dh0", cp(dh0), dh0_r, tol)


@pytest.mark.parametrize("path", ["auto", "generic"])
@pytest.mark.parametrize("N,c", [(32, 2), (128, 1)])
def test_dictionary_of_256_entries(P, N, c, path, monkeypatch):
    """K = 256 (the largest K of the paper, and the ABI maximum: k* is uint8)."""
    if path == "auto":
        monkeypatch.delenv("PDSSM_PATH", raising=False)    # the library's own dispatch for K = 256
    else:
        monkeypatch.setenv("PDSSM_PATH", "generic")
    fwd_bwd_check(P, 2, 2, 400, N, 256, c, 32, seed=N + c)


def test_state_1024(P, monkeypatch):
    """N = 1024, the ABI maximum (uint16 index maps)."""
    monkeypatch.setenv("PDSSM_PATH", "generic")
    fwd_bwd_check(P, 1, 2, 70, 1024, 8, 2, 16, seed=1024)
    fwd_bwd_check(P, 1, 1, 40, 1024, 3, 1, 40, seed=1025, bf16=True)


def test_hypothesis_random_shapes(P, monkeypatch):
    """Randomised small shapes through the library's default dispatch (seq / fused / generic)."""
    hyp = pytest.importorskip("hypothesis")
    from hypothesis import given, settings, HealthCheck
    from hypothesis import strategies as st

    monkeypatch.delenv("PDSSM_PATH", raising=False)

    @settings(max_examples=25, deadline=None, derandomize=True,
              suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])
    @given(B=st.integers(1, 3), H=st.integers(1, 3), L=st.integers(1, 300),
           N=st.sampled_from([1, 3, 8, 17, 32, 64, 96, 128, 130]), K=st.integers(1, 40), c=st.sampled_from([1, 2]),
           tau=st.sampled_from([0, 1, 5, 16, 64, 300]), bf16=st.booleans(), h0=st.booleans(),
           seed=st.integers(0, 10 ** 6))
    def run(B, H, L, N, K, c, tau, bf16, h0, seed):
        fwd_bwd_check(P, B, H, L, N, K, c, tau, bf16=bf16, seed=seed, h0=h0)

    run()


def test_single_chunk_forward_then_other_backward_path(P, monkeypatch):
    """The forward runs the single-chunk kernel (tau = L, EXPORT_MAPS off, h0 = 0: it composes no
    chunk aggregate), the backward is forced onto the chunked / generic kernels (the path a
    misaligned dh selects) with an incoming adjoint lam_in: they must not read the aggregate
    (dh0 comes from the chunk-0 replay)."""
    B, H, L, N, K, c = 2, 2, 160, 64, 8, 2
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=77, dh=True)
    d = to_dev(inp, False)
    monkeypatch.setenv("PDSSM_PATH", "seq")
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], tau=L)   # dims.chunk = L for every path
    assert f["tau"] == L
    rng = np.random.default_rng(3)
    lam = rng.standard_normal((B, H, c, N)).astype(np.float32)
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, e = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "dh"))
    h = O.scan_forward(Pm, Dz, bz)
    e_in = e.copy()
    e_in[:, :, -1] += O.planes_to_complex(lam)        # lam_in enters h_{L-1}
    db_r, dD_r, g_r, dh0_r = O.scan_backward(Pm, Dz, h, e_in)
    cp = lambda t: O.planes_to_complex(t.float().cpu().numpy())
    for path in ("seq", "fused", "generic"):
        monkeypatch.setenv("PDSSM_PATH", path)
        db, dD, g, dh0 = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"],
                                    dh=d["dh"], lam_in=torch.from_numpy(lam).cuda())
        torch.cuda.synchronize()
        check("db_" + path, cp(db), db_r, 1e-4)
        check("dD_" + path, cp(dD), dD_r, 1e-4)
        check("g_" + path, g.cpu().numpy(), g_r, 1e-4)
        check("dh0_" + path, cp(dh0), dh0_r, 1e-4)


def test_segment_summary_bwd_after_single_chunk_forward(P, monkeypatch):
    """Sequence-parallel backward summary of a segment whose forward took the single-chunk kernel
    (tau = 0 default with B*H large): beta' of the segment = dh0 of its local backward."""
    monkeypatch.delenv("PDSSM_PATH", raising=False)
    B, H, L, N, K, c = 16, 8, 96, 128, 8, 2
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=99, dh=True)
    d = to_dev(inp, False)
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"])
    assert f["tau"] == L                                  # the single-chunk path ran
    beta = P.segment_summary_bwd(d["kstar"], d["dict_idx"], d["diag"], f["chunk_state"], f["dims"], dh=d["dh"])
    torch.cuda.synchronize()
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, e = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "dh"))
    h = O.scan_forward(Pm, Dz, bz)
    dh0_r = O.scan_backward(Pm, Dz, h, e)[3]
    assert bool(torch.isfinite(beta).all())
    check("beta_prime", O.planes_to_complex(beta.cpu().numpy()), dh0_r, 1e-4)


def test_autograd_with_permuted_inputs(P):
    """diag / bias handed to the autograd glue as permuted (non-contiguous) views: the gradients
    must still be those of the logical tensors."""
    B, H, L, N, K, c = 2, 3, 50, 32, 4, 2
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=12, h0=True, dh=True)
    base_D = torch.from_numpy(np.ascontiguousarray(np.moveaxis(inp["diag"], 1, 2))).cuda()   # [B][L][H][c][N]
    base_b = torch.from_numpy(np.ascontiguousarray(np.moveaxis(inp["bias"], 1, 2))).cuda()
    base_D.requires_grad_(True)
    base_b.requires_grad_(True)
    h0 = torch.from_numpy(inp["h0"]).cuda().requires_grad_(True)
    diag = base_D.permute(0, 2, 1, 3, 4)          # logical [B][H][L][c][N], non-contiguous
    bias = base_b.permute(0, 2, 1, 3, 4)
    assert not diag.is_contiguous()
    kst = torch.from_numpy(inp["kstar"]).cuda()
    di = torch.from_numpy(inp["dict_idx"]).cuda().to(torch.int16)
    hs = P.scan(diag, bias, kst, di, h0=h0)
    dh = torch.from_numpy(inp["dh"]).cuda()
    (hs * dh).sum().backward()
    torch.cuda.synchronize()
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, e, h0z = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "dh", "h0"))
    h = O.scan_forward(Pm, Dz, bz, h0z)
    db_r, dD_r, _, dh0_r = O.scan_backward(Pm, Dz, h, e, h0z)
    gD = O.planes_to_complex(base_D.grad.permute(0, 2, 1, 3, 4).cpu().numpy())
    gb = O.planes_to_complex(base_b.grad.permute(0, 2, 1, 3, 4).cpu().numpy())
    check("autograd_dD", gD, dD_r, 1e-4)
    check("autograd_db", gb, db_r, 1e-4)
    check("autograd_dh0", O.planes_to_complex(h0.grad.cpu().numpy()), dh0_r, 1e-4)


def test_hypothesis_chunked_single_cta(P, monkeypatch):
    """Randomised shapes forced onto the chunked single-CTA path (PDSSM_PATH=seqc): ragged chunks,
    L = 1, one chunk, PER_STEP complex / real, fp32 / bf16, with and without h0."""
    pytest.importorskip("hypothesis")
    from hypothesis import given, settings, HealthCheck
    from hypothesis import strategies as st

    monkeypatch.setenv("PDSSM_PATH", "seqc")

    @settings(max_examples=20, deadline=None, derandomize=True,
              suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])
    @given(B=st.integers(1, 3), H=st.integers(1, 2), L=st.integers(1, 400), N=st.sampled_from([32, 64, 96, 128]),
           K=st.integers(1, 33), c=st.sampled_from([1, 2]), tau=st.integers(1, 200), bf16=st.booleans(),
           h0=st.booleans(), seed=st.integers(0, 10 ** 6))
    def run(B, H, L, N, K, c, tau, bf16, h0, seed):
        fwd_bwd_check(P, B, H, L, N, K, c, tau, bf16=bf16, seed=seed, h0=h0)

    run()
