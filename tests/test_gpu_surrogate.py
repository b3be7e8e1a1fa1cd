"""GPU parity of the NEXT-1 surrogate gradients (Prop. 2) through the C ABI
against the float64 oracle (oracle.selector_grad / dictionary_outer / dictionary_grad, pinned by
finite differences in test_oracle_pins.py).  The oracle side runs its own forward and backward
scans, so no GPU value enters the reference.  Bars (R19): max|gpu - oracle| /
max|oracle| <= 1e-4 (fp32) and 2e-2 (bf16) per tensor; for bf16 activations the oracle's
dictionary gradient reads its own lambda and h rounded to bf16, the activation-dtype tensors
the GPU kernel consumes (reading R16)."""
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


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - b)) / max(np.max(np.abs(b)), 1e-30))


@pytest.mark.parametrize("K,T", [(32, 1.0), (5, 0.5), (48, 0.1)])
def test_select_grad_parity(P, K, T):
    B, H, L = 2, 3, 77
    rng = np.random.default_rng(K)
    logits = rng.normal(size=(B, H, L, K)).astype(np.float32)
    ks = rng.integers(0, K, size=(B, H, L)).astype(np.uint8)
    g = rng.normal(size=(B, H, L)).astype(np.float32)
    d = P.select_grad(torch.from_numpy(logits).cuda(), torch.from_numpy(ks).cuda(), torch.from_numpy(g).cuda(), T)
    ref = O.selector_grad(logits.astype(np.float64), ks, g.astype(np.float64), T)
    assert rel(d.cpu().numpy(), ref) <= 1e-5
    # the argmax of the GPU's own select feeds it in practice; rows sum to 0
    assert np.max(np.abs(d.cpu().numpy().astype(np.float64).sum(-1))) <= 1e-5 * max(1.0, np.max(np.abs(ref)))


def run_dict_case(P, B, H, L, N, K, c, T, bf16=False, per_dict=False, unused_k=None, seed=0):
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=seed, h0=True, dh=True, per_dict=per_dict, bf16=bf16)
    M = synth.dictionary(H, K, N, seed + 1).astype(np.float32)
    if unused_k is not None:
        inp["kstar"][inp["kstar"] == unused_k] = (unused_k + 1) % K
    d = {}
    for k, v in inp.items():
        t = torch.from_numpy(np.ascontiguousarray(v)).cuda()
        if k == "dict_idx":
            t = t.to(torch.int16)
        elif k in ("bias", "dh") or (k == "diag" and not per_dict):
            if bf16:
                t = t.to(torch.bfloat16)
        d[k] = t
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=d["h0"], per_dict=per_dict)
    db, dD, g, dh0 = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"],
                                dh=d["dh"], h0=d["h0"])
    Mt = torch.from_numpy(M).cuda()
    dM, G = P.dict_grad(Mt, d["kstar"], d["diag"], f["h"], db, T, f["dims"], h0=d["h0"], want_G=True)
    torch.cuda.synchronize()
    # oracle: its own forward and backward from the same (rounded) inputs
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz = O.planes_to_complex(inp["diag"])
    if per_dict:
        Dz = O.gather_D_per_dict(Dz, inp["kstar"])
    bz, h0z, e = (O.planes_to_complex(inp[k]) for k in ("bias", "h0", "dh"))
    h = O.scan_forward(Pm, Dz, bz, h0z)
    lam = O.scan_backward(Pm, Dz, h, e, h0z)[0]
    if bf16:   # the kernel reads lambda (dbias) and h_saved in the activation dtype
        rnd = lambda z: O.planes_to_complex(synth.round_bf16(O.complex_to_planes(z, c).astype(np.float32)))
        lam, h = rnd(lam), rnd(h)
    G_ref = O.dictionary_outer(inp["kstar"], lam, Dz, h, K, h0=h0z)
    dM_ref = O.dictionary_grad(M.astype(np.float64), G_ref, T)
    return dM.cpu().numpy(), G.cpu().numpy(), dM_ref, G_ref, (Mt, d, f, db)


DICT_CASES = [
    # B, H, L, N, K, c, bf16, per_dict
    (2, 2, 300, 128, 32, 2, False, False),   # tcgen05 path, complex, ragged batches per entry
    (1, 2, 517, 128, 7, 1, False, False),    # tcgen05 path, real
    (2, 1, 200, 128, 6, 2, False, True),     # tcgen05 path, PER_DICT
    (2, 2, 150, 64, 16, 2, False, False),    # SIMT path
    (1, 1, 64, 8, 4, 2, False, False),       # config 1 (tiny), SIMT
    (1, 2, 100, 32, 5, 1, False, True),      # SIMT, PER_DICT, real
]


@pytest.mark.parametrize("case", DICT_CASES, ids=[str(c) for c in DICT_CASES])
@pytest.mark.parametrize("T", [1.0, 0.2])
def test_dict_grad_parity(P, case, T):
    B, H, L, N, K, c, bf16, pd = case
    dM, G, dM_ref, G_ref, _ = run_dict_case(P, B, H, L, N, K, c, T, bf16=bf16, per_dict=pd, seed=N + L)
    assert rel(G, G_ref) <= 1e-4
    assert rel(dM, dM_ref) <= 1e-4
    assert np.max(np.abs(dM.astype(np.float64).sum(axis=-2))) <= 1e-4 * max(1.0, np.max(np.abs(dM_ref)))


@pytest.mark.parametrize("N", [128, 64])
def test_dict_grad_bf16_and_unused_entry(P, N):
    B, H, L, K, c = 2, 2, 180, 8, 2
    dM, G, dM_ref, G_ref, _ = run_dict_case(P, B, H, L, N, K, c, 0.5, bf16=True, unused_k=3, seed=9)
    assert rel(G, G_ref) <= 2e-2
    assert rel(dM, dM_ref) <= 2e-2
    assert np.all(G[:, 3] == 0.0) and np.all(dM[:, 3] == 0.0)   # no step selected entry 3


def test_dict_grad_tc_matches_simt_and_is_deterministic(P, monkeypatch):
    B, H, L, N, K, c = 2, 2, 400, 128, 16, 2
    dM, G, dM_ref, G_ref, (Mt, d, f, db) = run_dict_case(P, B, H, L, N, K, c, 1.0, seed=3)
    dM2, G2 = P.dict_grad(Mt, d["kstar"], d["diag"], f["h"], db, 1.0, f["dims"], h0=d["h0"], want_G=True)
    assert torch.equal(dM2, torch.from_numpy(dM).cuda()) and torch.equal(G2, torch.from_numpy(G).cuda())
    monkeypatch.setenv("PDSSM_PATH", "generic")   # SIMT kernel at N = 128
    dM3, G3 = P.dict_grad(Mt, d["kstar"], d["diag"], f["h"], db, 1.0, f["dims"], h0=d["h0"], want_G=True)
    assert rel(G3.cpu().numpy(), G_ref) <= 1e-4
    assert rel(dM3.cpu().numpy(), dM_ref) <= 1e-4


def test_grad_argument_errors(P):
    dims = P.make_dims(1, 1, 4, 8, 2, c=1)
    z = torch.zeros(1, 1, 4, 2, device="cuda")
    ks = torch.zeros(1, 1, 4, dtype=torch.uint8, device="cuda")
    g = torch.zeros(1, 1, 4, device="cuda")
    with pytest.raises(P.PdssmError, match="ERR_RANGE"):
        P.select_grad(z, ks, g, 0.0)
    M = torch.zeros(1, 2, 8, 8, device="cuda")
    with pytest.raises(P.PdssmError, match="ERR_NULL"):
        P.dict_grad(M, ks, None, None, None, 1.0, dims)


def test_autograd_scan_matches_oracle(P):
    """The autograd glue (paper_2605_19150_b200.scan) routes a loss through pdssm_scan_bwd."""
    B, H, L, N, K, c = 2, 2, 90, 64, 6, 2
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=5, h0=True, dh=True)
    diag = torch.from_numpy(inp["diag"]).cuda().requires_grad_(True)
    bias = torch.from_numpy(inp["bias"]).cuda().requires_grad_(True)
    h0 = torch.from_numpy(inp["h0"]).cuda().requires_grad_(True)
    w = torch.from_numpy(inp["dh"]).cuda()
    ks = torch.from_numpy(inp["kstar"]).cuda()
    di = torch.from_numpy(inp["dict_idx"]).cuda().to(torch.int16)
    h = P.scan(diag, bias, ks, di, h0=h0)
    (h * w).sum().backward()
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, h0z, e = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "h0", "dh"))
    hr = O.scan_forward(Pm, Dz, bz, h0z)
    db_r, dD_r, _, dh0_r = O.scan_backward(Pm, Dz, hr, e, h0z)
    cp = lambda t: O.planes_to_complex(t.detach().cpu().numpy())
    rl = lambda a, b: float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
    assert rl(cp(h), hr) <= 1e-4
    assert rl(cp(bias.grad), db_r) <= 1e-4
    assert rl(cp(diag.grad), dD_r) <= 1e-4
    assert rl(cp(h0.grad), dh0_r) <= 1e-4


@pytest.mark.parametrize("c,N,bf16", [(2, 128, False), (1, 64, False), (2, 64, True)])
def test_layer_fwd_parity(P, c, N, bf16):
    """pdssm_layer_fwd (select -> b = Bx -> scan -> y = Re(Ch)) against the oracle chain.
    Integer-valued x, S make the selections exact (reading R18), so k* is compared bit for bit."""
    B, H, L, K, d_in, Pp = 2, 2, 200, 8, 64, 32
    x = synth.tokens_x(B, L, d_in, seed=N, integer=True)
    S = synth.selector(H, K, d_in, seed=N, integer=True)
    di = synth.random_maps(H, K, N, seed=N)
    Dk = synth.diag((H, K), N, c, seed=N)
    Bw = synth.projection_B(H, c, N, d_in, seed=N)
    C = synth.readout_C(H, Pp, N, c, seed=N)
    if bf16:
        Bw = synth.round_bf16(Bw)
        C = synth.round_bf16(C)          # the readout stages C in the activation dtype (R24)
    dt = torch.bfloat16 if bf16 else torch.float32
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    r = P.layer_fwd(cu(x).to(dt), cu(S).to(dt), cu(di).to(torch.int16), cu(Dk), cu(Bw).to(dt), C=cu(C), per_dict=True)
    torch.cuda.synchronize()
    ks_ref, _ = O.select(x.astype(np.float64), S.astype(np.float64))
    assert np.array_equal(r["kstar"].cpu().numpy(), ks_ref)
    Pm = O.gather_P(di, ks_ref)
    Dz = O.gather_D_per_dict(O.planes_to_complex(Dk), ks_ref)
    Bc = Bw[:, 0].astype(np.float64) + (1j * Bw[:, 1].astype(np.float64) if c == 2 else 0)
    h = O.scan_forward(Pm, Dz, O.project_b(x.astype(np.float64), Bc))
    Cc = C[:, 0].astype(np.float64) + (1j * C[:, 1].astype(np.float64) if c == 2 else 0)
    y = O.readout(h, Cc)
    tol = 2e-2 if bf16 else 1e-4
    hg = O.planes_to_complex(r["h"].float().cpu().numpy())
    check("layer_h", hg, h, tol)
    check("layer_y", r["y"].float().cpu().numpy(), y, tol, bh_axes=(0, 2))


@pytest.mark.parametrize("K", [100, 256])
def test_select_grad_warp_path(P, K):
    """K > 64 takes the warp-per-row kernel (logits in registers, KM = ceil(K / 32))."""
    B, H, L, T = 1, 2, 33, 0.7
    rng = np.random.default_rng(K + 1)
    logits = rng.normal(size=(B, H, L, K)).astype(np.float32)
    ks = rng.integers(0, K, size=(B, H, L)).astype(np.uint8)
    g = rng.normal(size=(B, H, L)).astype(np.float32)
    d = P.select_grad(torch.from_numpy(logits).cuda(), torch.from_numpy(ks).cuda(), torch.from_numpy(g).cuda(), T)
    ref = O.selector_grad(logits.astype(np.float64), ks, g.astype(np.float64), T)
    assert rel(d.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("N", [128, 64])
def test_dict_grad_first_steps_without_h0(P, N):
    """L = 1 (every selected step is t = 0, h_{-1} = h0 = 0 -> w = 0 -> G = 0) and L = 2 without h0."""
    for L in (1, 2):
        B, H, K, c = 3, 2, 4, 2
        inp = synth.scan_inputs(B, H, L, N, K, c, seed=L + N, dh=True)
        d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()}
        d["dict_idx"] = d["dict_idx"].to(torch.int16)
        M = torch.from_numpy(synth.dictionary(H, K, N, 3)).cuda()
        f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"])
        db = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"], dh=d["dh"])[0]
        dM, G = P.dict_grad(M, d["kstar"], d["diag"], f["h"], db, 1.0, f["dims"], want_G=True)
        torch.cuda.synchronize()
        Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
        Dz, bz, e = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "dh"))
        h = O.scan_forward(Pm, Dz, bz)
        lam = O.scan_backward(Pm, Dz, h, e)[0]
        G_ref = O.dictionary_outer(inp["kstar"], lam, Dz, h, K)
        if L == 1:
            assert np.all(G.cpu().numpy() == 0.0) and np.all(dM.cpu().numpy() == 0.0)
        else:
            assert rel(G.cpu().numpy(), G_ref) <= 1e-4
            assert rel(dM.cpu().numpy(), O.dictionary_grad(M.cpu().numpy().astype(np.float64), G_ref, 1.0)) <= 1e-4


@pytest.mark.parametrize("c,N,bf16,path", [(2, 128, False, "tc"), (1, 128, False, "tc"), (2, 64, True, "tc"),
                                            (2, 128, False, "generic"), (1, 24, False, "tc")])
def test_diag_gen_parity(P, c, N, bf16, path, monkeypatch):
    """NEXT-2 D_t generator (fused sigmoid / sincos epilogue, or projection + elementwise) vs the oracle."""
    if path == "generic":
        monkeypatch.setenv("PDSSM_PATH", "generic")
    B, H, L, d_in = 2, 3, 150, 64
    rng = np.random.default_rng(N + c)
    x = rng.normal(size=(B, L, d_in)).astype(np.float32)
    Wd = (rng.uniform(-1, 1, size=(H, c, N, d_in)) / np.sqrt(d_in)).astype(np.float32)
    bias = rng.normal(2.0, 1.0, size=(H, N)).astype(np.float32)
    if bf16:
        x, Wd = synth.round_bf16(x), synth.round_bf16(Wd)
    dt = torch.bfloat16 if bf16 else torch.float32
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    D = P.diag_gen(cu(x).to(dt), cu(Wd).to(dt), cu(bias))
    torch.cuda.synchronize()
    ref = O.diag_generator(x, Wd[:, 0], Wd[:, 1] if c == 2 else None, bias)
    got = O.planes_to_complex(D.float().cpu().numpy())
    assert float(np.max(np.abs(got - ref)) / np.max(np.abs(ref))) <= (2e-2 if bf16 else 1e-4)


def test_layer_fwd_with_generated_diag(P):
    """NEXT-2 chain with input-dependent D_t: pdssm_diag_gen -> pdssm_layer_fwd (PER_STEP), vs the oracle
    chain select -> D(u_t) -> b = Bx -> scan -> y."""
    B, H, L, N, K, c, d_in, Pp = 2, 2, 160, 128, 8, 2, 64, 16
    x = synth.tokens_x(B, L, d_in, seed=3, integer=True)
    S = synth.selector(H, K, d_in, seed=3, integer=True)
    di = synth.random_maps(H, K, N, seed=3)
    rng = np.random.default_rng(3)
    Wd = (rng.uniform(-1, 1, size=(H, c, N, d_in)) / (8 * np.sqrt(d_in))).astype(np.float32)
    bias = rng.normal(2.0, 1.0, size=(H, N)).astype(np.float32)
    Bw = synth.projection_B(H, c, N, d_in, seed=3)
    C = synth.readout_C(H, Pp, N, c, seed=3)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    D = P.diag_gen(cu(x), cu(Wd), cu(bias))
    r = P.layer_fwd(cu(x), cu(S), cu(di).to(torch.int16), D, cu(Bw), C=cu(C), per_dict=False)
    torch.cuda.synchronize()
    ks_ref, _ = O.select(x.astype(np.float64), S.astype(np.float64))
    assert np.array_equal(r["kstar"].cpu().numpy(), ks_ref)
    Dz = O.diag_generator(x, Wd[:, 0], Wd[:, 1], bias)
    h = O.scan_forward(O.gather_P(di, ks_ref), Dz, O.project_b(x.astype(np.float64), Bw[:, 0] + 1j * Bw[:, 1]))
    y = O.readout(h, C[:, 0] + 1j * C[:, 1])
    hg = O.planes_to_complex(r["h"].cpu().numpy())
    assert float(np.max(np.abs(hg - h)) / np.max(np.abs(h))) <= 1e-4
    assert rel(r["y"].cpu().numpy(), y) <= 1e-4


@pytest.mark.parametrize("N,K,bf16", [(128, 32, False), (64, 8, False), (128, 5, True), (32, 16, False)])
def test_soft_select_parity(P, N, K, bf16):
    """NEXT-3 PD-SSM soft generator (Eqs. 2-4) on tcgen05 with the column-hardmax epilogue vs the oracle.
    Argmax decisions are bit-exact wherever the float64 top-2 gap exceeds the GEMM's rounding bound
    (reading R18's margin rule); the rest (near ties) must be rare."""
    B, H, L = 2, 2, 100
    rng = np.random.default_rng(N + K)
    logits = (3 * rng.normal(size=(B, H, L, K))).astype(np.float32)
    M = synth.dictionary(H, K, N, seed=N + K)
    got = P.soft_select(torch.from_numpy(logits).cuda(), torch.from_numpy(M).cuda(), bf16=bf16)
    torch.cuda.synchronize()
    got = got.cpu().numpy().astype(np.int64)
    ref = O.soft_generator_P(logits.astype(np.float64), M.astype(np.float64))
    s = O.softmax_T(logits.astype(np.float64), 1.0)
    mix = np.einsum("bhtk,hkij->bhtij", s, M.astype(np.float64))
    srt = np.sort(mix, axis=-2)
    gap = srt[..., -1, :] - srt[..., -2, :]
    u = 2.0 ** -8 if bf16 else 2.0 ** -20
    bound = 4 * u * np.max(np.abs(M))
    clear = gap > bound
    assert np.array_equal(got[clear], ref[clear])
    if not bf16:   # bf16 operands (s, M rounded to 8 bits) leave more columns inside the margin
        assert np.mean(got != ref) <= 2e-3
    assert got.min() >= 0 and got.max() < N


@pytest.mark.parametrize("c,N,bf16,atm", [(2, 128, False, "1"), (1, 64, False, "1"), (2, 64, True, "1"),
                                          (2, 128, False, "0")])
def test_layer_fwd_gen_parity(P, c, N, bf16, atm, monkeypatch):
    """NEXT-2: selector + projection + D_t generator as one fused tcgen05 GEMM (pdssm_layer_fwd_gen),
    then the scan and the readout, against the oracle chain select -> project_b -> diag_generator ->
    scan_forward -> readout (R30).  Integer-valued x, S: the selections are exact (R18).
    atm "0": the fp32 fused GEMM with the token rows in shared memory instead of tensor memory."""
    monkeypatch.setenv("PDSSM_LAYER_ATM", atm)
    B, H, L, K, d_in, Pp = 2, 2, 150, 8, 64, 32
    x = synth.tokens_x(B, L, d_in, seed=N + 1, integer=True)
    S = synth.selector(H, K, d_in, seed=N + 1, integer=True)
    di = synth.random_maps(H, K, N, seed=N + 1)
    Bw = synth.projection_B(H, c, N, d_in, seed=N + 1)
    Wd = synth.projection_B(H, c, N, d_in, seed=N + 2) / 8.0
    bmag = np.random.default_rng(N).normal(2.0, 0.5, size=(H, N)).astype(np.float32)
    C = synth.readout_C(H, Pp, N, c, seed=N + 1)
    if bf16:
        Bw, Wd, C = synth.round_bf16(Bw), synth.round_bf16(Wd), synth.round_bf16(C)
    dt = torch.bfloat16 if bf16 else torch.float32
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    r = P.layer_fwd(cu(x).to(dt), cu(S).to(dt), cu(di).to(torch.int16), None, cu(Bw).to(dt), C=cu(C), Wd=cu(Wd).to(dt),
                    bias_mag=cu(bmag))
    torch.cuda.synchronize()
    ks_ref, _ = O.select(x.astype(np.float64), S.astype(np.float64))
    assert np.array_equal(r["kstar"].cpu().numpy(), ks_ref)
    Pm = O.gather_P(di, ks_ref)
    W = Wd.astype(np.float64)
    D = O.diag_generator(x.astype(np.float64), W[:, 0], W[:, 1] if c == 2 else None, bmag)
    if bf16:   # the generator writes D_t in the activation dtype, which the scan then reads (R16)
        D = O.planes_to_complex(synth.round_bf16(O.complex_to_planes(D, c).astype(np.float32)))
    Bc = Bw[:, 0].astype(np.float64) + (1j * Bw[:, 1].astype(np.float64) if c == 2 else 0)
    bz = O.project_b(x.astype(np.float64), Bc)
    if bf16:
        bz = O.planes_to_complex(synth.round_bf16(O.complex_to_planes(bz, c).astype(np.float32)))
    h = O.scan_forward(Pm, D, bz)
    Cc = C[:, 0].astype(np.float64) + (1j * C[:, 1].astype(np.float64) if c == 2 else 0)
    y = O.readout(h, Cc)
    tol = 2e-2 if bf16 else 1e-4
    check("gen_h", O.planes_to_complex(r["h"].float().cpu().numpy()), h, tol)
    check("gen_y", r["y"].float().cpu().numpy(), y, tol, bh_axes=(0, 2))


def test_layer_fwd_runs_one_fused_gemm(P):
    """The config-2-shaped layer call launches a single tcgen05 GEMM (EpiLayer: select + projection
    + D_t generator) before the scan, instead of three."""
    from torch.profiler import ProfilerActivity, profile
    B, H, L, K, d_in, N, c, Pp = 2, 8, 256, 32, 1024, 128, 2, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(B, L, d_in, device="cuda", generator=g)
    S = torch.randn(H, K, d_in, device="cuda", generator=g) / 32
    Bw = torch.randn(H, c, N, d_in, device="cuda", generator=g) / 32
    Wd = torch.randn(H, c, N, d_in, device="cuda", generator=g) / 32
    C = torch.randn(H, c, Pp, N, device="cuda", generator=g) / 12
    di = torch.randint(0, N, (H, K, N), device="cuda", generator=g).to(torch.int16)
    P.layer_fwd(x, S, di, None, Bw, C=C, Wd=Wd)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        P.layer_fwd(x, S, di, None, Bw, C=C, Wd=Wd)
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    gemms = [n for n in names if "k_gemm_tc" in n]
    assert any("EpiLayer" in n for n in gemms), gemms
    assert not any("EpiSelect" in n.split("EpiLayer")[0] or "EpiProject" in n.split("EpiLayer")[0] for n in gemms
                   if "EpiLayer" not in n)
