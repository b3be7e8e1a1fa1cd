"""GPU parity of the scan path (a4-a9) through the C ABI against the float64
oracle.  Bars (BASELINE.json north_star, R19): index maps and
integer outputs bit-exact; floats within max|gpu - oracle| / max|oracle|
<= 1e-4 (fp32) / 2e-2 (bf16), per tensor AND per (b, h) sequence (tests/parity.py).
bf16 runs: the oracle reads the bf16-rounded inputs, and its backward reads its own states
rounded to bf16 -- the activation-dtype h_saved the backward consumes (reading R16)."""
import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from parity import TOL, check, rel


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_19150_b200 as mod
    return mod


def saved_states(h, c, bf16):
    """The states the backward consumes: the oracle's own h, rounded to bf16 for bf16 runs (R16)."""
    if not bf16:
        return h
    return O.planes_to_complex(synth.round_bf16(O.complex_to_planes(h, c).astype(np.float32)))


def to_dev(inp, bf16):
    out = {}
    for k, v in inp.items():
        t = torch.from_numpy(np.ascontiguousarray(v)).cuda()
        if k == "dict_idx":
            t = t.to(torch.int16)
        elif k in ("diag_step", "bias", "dh", "diag") and bf16 and v.dtype == np.float32:
            t = t.to(torch.bfloat16)
        out[k] = t
    return out


def cpx(t):
    return O.planes_to_complex(t.float().cpu().numpy())


def run_case(P, B, H, L, N, K, c, tau, bf16=False, per_dict=False, h0=True, seed=0, sticky=0.0):
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=seed, h0=h0, dh=True, per_dict=per_dict, bf16=bf16, sticky=sticky)
    d = to_dev(inp, bf16)
    if per_dict:
        d["diag"] = torch.from_numpy(inp["diag"]).cuda()        # PER_DICT diag stays f32
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=d.get("h0"), tau=tau, per_dict=per_dict,
                   export_maps=True)
    db, dD, g, dh0 = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"],
                                dh=d["dh"], h0=d.get("h0"))
    torch.cuda.synchronize()
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz = O.planes_to_complex(inp["diag"])
    if per_dict:
        Dz = O.gather_D_per_dict(Dz, inp["kstar"])
    bz = O.planes_to_complex(inp["bias"])
    h0z = O.planes_to_complex(inp["h0"]) if h0 else None
    ch = O.scan_chunked(Pm, Dz, bz, f["tau"], h0z)
    e = O.planes_to_complex(inp["dh"])
    db_r, dD_r, g_r, dh0_r = O.scan_backward(Pm, Dz, saved_states(ch["h"], c, bf16), e, h0z)
    return inp, f, (db, dD, g, dh0), ch, (db_r, dD_r, g_r, dh0_r), Pm, Dz


CASES = [
    # B, H, L, N, K, c, tau
    (1, 1, 64, 8, 4, 2, 16),      # config 1 (tiny)
    (1, 1, 64, 8, 4, 1, 7),
    (2, 3, 65, 5, 3, 2, 64),
    (1, 2, 257, 32, 8, 2, 128),   # ragged last chunk
    (2, 1, 63, 64, 16, 1, 1),
    (1, 1, 1, 16, 4, 2, 0),       # L = 1
    (1, 2, 100, 120, 48, 2, 32),
    (2, 2, 300, 128, 32, 2, 0),   # headline N, default tau
    (1, 1, 50, 2, 2, 1, 1000),    # tau >= L
    (1, 1, 40, 1, 1, 2, 8),       # N = 1, K = 1
    (1, 1, 33, 200, 5, 1, 16),    # N not a multiple of 32
    (2, 3, 333, 64, 16, 2, 32),   # fused path shapes (N in {32, 64, 128})
    (3, 2, 190, 32, 7, 1, 17),
    (2, 2, 1000, 128, 32, 2, 32),
    (1, 2, 129, 128, 48, 1, 128),
]


FUSED_N = (32, 64, 128)


@pytest.fixture(params=["auto", "generic"])
def path(request, monkeypatch):
    monkeypatch.setenv("PDSSM_PATH", request.param)
    return request.param


def use_path(monkeypatch, path, N, tau):
    """'auto' on a fused-eligible shape is upgraded to 'fused' so the test proves the fast path ran."""
    if path == "auto" and N in FUSED_N and tau <= 256:
        monkeypatch.setenv("PDSSM_PATH", "fused")


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
@pytest.mark.parametrize("bf16", [False, True], ids=["f32", "bf16"])
def test_scan_fwd_bwd_parity(P, case, bf16, path, monkeypatch):
    B, H, L, N, K, c, tau = case
    use_path(monkeypatch, path, N, tau if tau else 64)
    inp, f, got, ch, ref, Pm, Dz = run_case(P, B, H, L, N, K, c, tau, bf16=bf16, seed=hash(case) % 1000)
    tol = TOL["bf16" if bf16 else "f32"]
    check("h", cpx(f["h"]), ch["h"], tol)
    # integer maps: bit-exact
    assert np.array_equal(f["maps"].cpu().numpy().astype(np.int64), ch["maps"])
    pi, d_bar, beta_bar, carry = P.chunk_state_views(f["chunk_state"], f["dims"])
    assert np.array_equal(pi.cpu().numpy().astype(np.int64), ch["pi_bar"])
    check("d_bar", O.planes_to_complex(d_bar.cpu().numpy()), ch["d_bar"], 1e-4)
    check("beta_bar", O.planes_to_complex(beta_bar.cpu().numpy()), ch["beta_bar"], 1e-4)
    check("carry", O.planes_to_complex(carry.cpu().numpy()), ch["carries"], 1e-4)
    db, dD, g, dh0 = got
    db_r, dD_r, g_r, dh0_r = ref
    check("db", cpx(db), db_r, tol)
    check("dD", cpx(dD), dD_r, tol)
    check("g", g.cpu().numpy(), g_r, tol)
    check("dh0", O.planes_to_complex(dh0.cpu().numpy()), dh0_r, tol)


@pytest.mark.parametrize("N", [16, 64])
def test_scan_per_dict_and_no_h0(P, N, path, monkeypatch):
    use_path(monkeypatch, path, N, 16)
    inp, f, got, ch, ref, Pm, Dz = run_case(P, 2, 2, 90, N, 5, 2, 16, per_dict=True, h0=False, seed=7)
    check("h", cpx(f["h"]), ch["h"], 1e-4)
    db, dD, g, dh0 = got
    db_r, dD_r, g_r, dh0_r = ref
    check("db", cpx(db), db_r, 1e-4)
    # PER_DICT ddiag = sum over steps selecting k of dD_t
    kst = inp["kstar"]
    H, K = 2, 5
    want = np.zeros((H, K, N), np.complex128)
    for h in range(H):
        for k in range(K):
            sel = kst[:, h, :] == k
            want[h, k] = dD_r[:, h][sel].sum(axis=0)
    check("dD_k", O.planes_to_complex(dD.cpu().numpy()), want, 1e-4)
    check("g", g.cpu().numpy(), g_r, 1e-4)


def test_determinism_bitwise(P, path, monkeypatch):
    use_path(monkeypatch, path, 64, 32)
    args = (2, 2, 200, 64, 16, 2, 32)
    _, f1, g1, *_ = run_case(P, *args, seed=3)
    _, f2, g2, *_ = run_case(P, *args, seed=3)
    assert torch.equal(f1["h"], f2["h"]) and torch.equal(f1["chunk_state"], f2["chunk_state"])
    for a, b in zip(g1, g2):
        assert torch.equal(a, b)


@pytest.mark.parametrize("tau", [1, 7, 64, 128])
def test_tau_invariance_of_final_outputs(P, tau, path, monkeypatch):
    use_path(monkeypatch, path, 32, 257)
    _, f, got, ch, ref, *_ = run_case(P, 1, 2, 257, 32, 8, 2, tau, seed=11)
    _, f0, got0, *_ = run_case(P, 1, 2, 257, 32, 8, 2, 257, seed=11)
    assert torch.equal(f["maps"][:, :, -1], f0["maps"][:, :, -1])
    assert rel(cpx(f["h"]), cpx(f0["h"])) <= 1e-4
    assert rel(cpx(got[0]), cpx(got0[0])) <= 1e-4


def test_fsa_emulation_exact(P, path):
    """Prop. 1 (App. D): states exactly one-hot, on the GPU."""
    from oracle import fsa
    import itertools
    for make in (fsa.parity, fsa.cyclic_z5, fsa.cycle_nav, fsa.even_pairs, fsa.mod_arith):
        A = make()
        dict_idx, dg, h0, C = A.compile()
        L = 6 if A.K <= 5 else 4
        words = np.array(list(itertools.product(range(A.K), repeat=L)), dtype=np.uint8)
        Bn = len(words)
        kst = torch.from_numpy(words[:, None, :].copy()).cuda()
        di = torch.from_numpy(dict_idx.astype(np.int16)).cuda()
        diag = torch.ones((1, A.K, 1, A.N), dtype=torch.float32, device="cuda")
        bias = torch.zeros((Bn, 1, L, 1, A.N), dtype=torch.float32, device="cuda")
        h0t = torch.from_numpy(np.tile(h0, (Bn, 1, 1, 1)).astype(np.float32)).cuda()
        for tau in (1, 2, 3, L):
            f = P.scan_fwd(kst, di, diag, bias, h0=h0t, tau=tau, per_dict=True, export_maps=True)
            h = f["h"].cpu().numpy()[:, 0, :, 0, :]
            runs = np.array([A.run(list(w)) for w in words])
            onehot = np.zeros((Bn, L, A.N), np.float32)
            np.put_along_axis(onehot, runs[:, :, None], 1.0, axis=2)
            assert np.array_equal(h, onehot), (A.name, tau)
            final_map = f["maps"].cpu().numpy()[:, 0, -1].astype(np.int64)
            for b in range(0, Bn, max(1, Bn // 50)):
                q = A.q_init
                assert final_map[b, q] == runs[b, -1]


def test_s5_word_problem_exact(P, path, monkeypatch):
    use_path(monkeypatch, path, 64, 64)
    """config 5 structure at reduced L: exact permuted arange states and exact maps."""
    dict_idx, perms5, blocks = synth.s5_dictionary(64, 16, seed=5000)
    B, H, L = 2, 2, 4096
    k = synth.kstar(B, H, L, 16, seed=5001)
    di = torch.from_numpy(np.tile(dict_idx[None], (H, 1, 1)).astype(np.int16)).cuda()
    kst = torch.from_numpy(k).cuda()
    diag = torch.ones((H, 16, 1, 64), dtype=torch.float32, device="cuda")
    bias = torch.zeros((B, H, L, 1, 64), dtype=torch.float32, device="cuda")
    h0 = torch.arange(64, dtype=torch.float32, device="cuda").view(1, 1, 1, 64).repeat(B, H, 1, 1).contiguous()
    f = P.scan_fwd(kst, di, diag, bias, h0=h0, tau=64, per_dict=True, export_maps=True)
    Pm = O.gather_P(np.tile(dict_idx[None], (H, 1, 1)), k)
    Pi, _ = O.prefix_maps(Pm, np.ones(Pm.shape))
    maps = f["maps"].cpu().numpy().astype(np.int64)
    for c in range(1, maps.shape[2] - 1):
        assert np.array_equal(maps[:, :, c], Pi[:, :, c * 64 - 1])
    assert np.array_equal(maps[:, :, -1], Pi[:, :, -1])
    hlast = f["h"].cpu().numpy()[:, :, -1, 0]
    expect = np.zeros((B, H, 64))
    np.put_along_axis(expect, Pi[:, :, -1], np.arange(64.0)[None, None].repeat(B, 0).repeat(H, 1), axis=2)
    assert np.array_equal(hlast, expect)


READOUT_CASES = [
    # N, c, P, L, bf16: P % 16 != 0 -> SIMT readout; P % 16 == 0 -> tcgen05 readout (3xTF32 / bf16)
    (16, 2, 8, 70, False),
    (32, 2, 48, 300, False),
    (32, 1, 16, 129, False),
    (16, 2, 32, 70, True),
    (64, 2, 128, 200, True),
    (64, 2, 128, 300, False),    # fp32, P % 64 == 0: pre-split weights, 64-column tiles, four stages
    (32, 1, 64, 129, False),
]


@pytest.mark.parametrize("rc", READOUT_CASES, ids=[str(r) for r in READOUT_CASES])
def test_readout_fused_and_dy_backward(P, rc, path, monkeypatch):
    N, c, Pp, L, bf16 = rc
    use_path(monkeypatch, path, N, 16)
    B, H, K = 2, 2, 4
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=21, h0=True, bf16=bf16)
    Cw = synth.readout_C(H, Pp, N, c, seed=21)
    if bf16:
        Cw = synth.round_bf16(Cw)          # the kernels stage C in the activation dtype (R24)
    d = to_dev(inp, bf16)
    Ct = torch.from_numpy(Cw).cuda()
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=d["h0"], C=Ct, tau=16, want_y=True)
    rng = np.random.default_rng(0)
    dy = rng.standard_normal((B, L, H, Pp)).astype(np.float32)
    if bf16:
        dy = synth.round_bf16(dy)
    dyt = torch.from_numpy(dy).cuda().to(torch.bfloat16 if bf16 else torch.float32)
    db, dD, g, dh0 = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"],
                                dy=dyt, C=Ct, h0=d["h0"])
    torch.cuda.synchronize()
    tol = TOL["bf16" if bf16 else "f32"]
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, h0z = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "h0"))
    h = O.scan_forward(Pm, Dz, bz, h0z)
    Cz = O.planes_to_complex(np.moveaxis(Cw, 1, -2))          # [H][P][N] complex
    y = O.readout(h, Cz)
    check("y", f["y"].float().cpu().numpy(), y, tol, bh_axes=(0, 2))
    e = O.readout_adjoint(dy, Cz)
    db_r, dD_r, g_r, dh0_r = O.scan_backward(Pm, Dz, saved_states(h, c, bf16), e, h0z)
    check("db", cpx(db), db_r, tol)
    check("dD", cpx(dD), dD_r, tol)
    check("g", g.cpu().numpy(), g_r, tol)


def test_check_finite_reports(P):
    B, H, L, N, K, c = 1, 1, 20, 8, 4, 1
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=2)
    d = to_dev(inp, False)
    P.check_device()
    bias = d["bias"].clone()
    bias[0, 0, 5, 0, 3] = float("nan")
    P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], bias, tau=8, check_finite=True)
    with pytest.raises(P.PdssmError) as ei:
        P.check_device()
    assert ei.value.status == 7
    k = d["kstar"].clone()
    k[0, 0, 3] = 200
    P.scan_fwd(k, d["dict_idx"], d["diag"], d["bias"], tau=8, check_finite=True)
    with pytest.raises(P.PdssmError) as ei:
        P.check_device()
    assert ei.value.status == 3
    P.check_device()      # cleared


# ---------------------------------------------------------------------------
# single-chunk path (tau >= L, C = 1): one CTA per sequence (csrc/k_scan_seq.cuh)
SEQ_CASES = [
    # B, H, L, N, K, c
    (2, 2, 300, 128, 32, 2),
    (1, 3, 129, 64, 16, 1),
    (2, 1, 77, 32, 5, 2),
    (1, 2, 1000, 96, 8, 2),
    (1, 1, 4500, 32, 4, 1),       # crosses the 4096-step k* window
    (3, 1, 1, 64, 3, 2),          # L = 1
]


@pytest.mark.parametrize("case", SEQ_CASES, ids=[str(c) for c in SEQ_CASES])
@pytest.mark.parametrize("bf16", [False, True], ids=["f32", "bf16"])
def test_seq_path_parity(P, case, bf16, monkeypatch):
    monkeypatch.setenv("PDSSM_PATH", "seq")
    B, H, L, N, K, c = case
    inp, f, got, ch, ref, Pm, Dz = run_case(P, B, H, L, N, K, c, 0, bf16=bf16, seed=L + N)
    assert f["tau"] == L
    tol = TOL["bf16" if bf16 else "f32"]
    check("h", cpx(f["h"]), ch["h"], tol)
    assert np.array_equal(f["maps"].cpu().numpy().astype(np.int64), ch["maps"])
    pi, d_bar, beta_bar, carry = P.chunk_state_views(f["chunk_state"], f["dims"])
    assert np.array_equal(pi.cpu().numpy().astype(np.int64), ch["pi_bar"])
    check("d_bar", O.planes_to_complex(d_bar.cpu().numpy()), ch["d_bar"], 1e-4)
    check("beta_bar", O.planes_to_complex(beta_bar.cpu().numpy()), ch["beta_bar"], 1e-4)
    check("carry", O.planes_to_complex(carry.cpu().numpy()), ch["carries"], 1e-4)
    db, dD, g, dh0 = got
    db_r, dD_r, g_r, dh0_r = ref
    check("db", cpx(db), db_r, tol)
    check("dD", cpx(dD), dD_r, tol)
    check("g", g.cpu().numpy(), g_r, tol)
    check("dh0", O.planes_to_complex(dh0.cpu().numpy()), dh0_r, tol)


@pytest.mark.parametrize("N", [64, 128])
def test_seq_path_per_dict_and_overflow(P, N, monkeypatch):
    """PER_DICT diagonals, and an entry whose preimage exceeds the 8-source records
    (a constant map: in-degree N) so the CSR fallback runs."""
    monkeypatch.setenv("PDSSM_PATH", "seq")
    B, H, L, K, c = 2, 2, 200, 6, 2
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=N + 7, h0=True, dh=True, per_dict=True)
    inp["dict_idx"][0, 1, :] = 3          # head 0, entry 1: every source -> state 3
    inp["dict_idx"][1, 2, : N // 2] = 0   # head 1, entry 2: in-degree N/2 at state 0
    d = to_dev(inp, False)
    d["diag"] = torch.from_numpy(inp["diag"]).cuda()
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=d["h0"], per_dict=True)
    db, dD, g, dh0 = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"],
                                dh=d["dh"], h0=d["h0"])
    torch.cuda.synchronize()
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz = O.gather_D_per_dict(O.planes_to_complex(inp["diag"]), inp["kstar"])
    bz, h0z, e = (O.planes_to_complex(inp[k]) for k in ("bias", "h0", "dh"))
    h = O.scan_forward(Pm, Dz, bz, h0z)
    check("h", cpx(f["h"]), h, 1e-4)
    db_r, dD_r, g_r, dh0_r = O.scan_backward(Pm, Dz, h, e, h0z)
    check("db", cpx(db), db_r, 1e-4)
    check("g", g.cpu().numpy(), g_r, 1e-4)
    # PER_DICT dD is reduced per entry: sum over the steps that selected it
    dDk = np.zeros((H, K, N), np.complex128)
    for b in range(B):
        for hh in range(H):
            np.add.at(dDk[hh], inp["kstar"][b, hh], dD_r[b, hh])
    check("dD_k", O.planes_to_complex(dD.cpu().numpy()), dDk, 1e-4)
    check("dh0", O.planes_to_complex(dh0.cpu().numpy()), dh0_r, 1e-4)


def test_seq_path_is_default_for_full_batches(P, monkeypatch):
    """B*H >= 0.6 * #SMs: the library default chunk is tau = L (single chunk)."""
    monkeypatch.delenv("PDSSM_PATH", raising=False)
    dims = P.make_dims(16, 8, 2048, 128, 32, c=2)
    assert P.default_chunk(dims) == 2048
    dims = P.make_dims(1, 2, 2048, 128, 32, c=2)
    assert P.default_chunk(dims) == 64


SEQ_NOMAPS_CASES = [
    # B, H, L, N, K, c   (single chunk, no EXPORT_MAPS: the production forward without aggregate chains)
    (2, 2, 300, 128, 32, 2),
    (1, 3, 129, 64, 16, 1),
    (2, 1, 77, 32, 5, 2),
    (1, 1, 64, 32, 4, 2),
    (1, 2, 2048, 128, 32, 2),
]


@pytest.mark.parametrize("case", SEQ_NOMAPS_CASES, ids=[str(c) for c in SEQ_NOMAPS_CASES])
@pytest.mark.parametrize("bf16", [False, True], ids=["f32", "bf16"])
def test_seq_no_maps_parity(P, case, bf16, monkeypatch):
    """Single-chunk scan as the bench runs it (no EXPORT_MAPS): states and the backward against the oracle."""
    monkeypatch.setenv("PDSSM_PATH", "seq")
    B, H, L, N, K, c = case
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=L + 3 * N, h0=True, dh=True, bf16=bf16)
    d = to_dev(inp, bf16)
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=d["h0"])
    assert f["tau"] == L
    db, dD, g, dh0 = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"],
                                dh=d["dh"], h0=d["h0"])
    torch.cuda.synchronize()
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, h0z, e = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "h0", "dh"))
    h = O.scan_forward(Pm, Dz, bz, h0z)
    tol = TOL["bf16" if bf16 else "f32"]
    check("h", cpx(f["h"]), h, tol)
    db_r, dD_r, g_r, dh0_r = O.scan_backward(Pm, Dz, saved_states(h, c, bf16), e, h0z)
    check("db", cpx(db), db_r, tol)
    check("dD", cpx(dD), dD_r, tol)
    check("g", g.cpu().numpy(), g_r, tol)
    check("dh0", O.planes_to_complex(dh0.cpu().numpy()), dh0_r, tol)
    # run-to-run bitwise determinism
    f2 = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=d["h0"])
    assert torch.equal(f["h"], f2["h"])


def test_seq_no_maps_per_dict_and_overflow(P, monkeypatch):
    monkeypatch.setenv("PDSSM_PATH", "seq")
    B, H, L, N, K, c = 2, 2, 257, 64, 6, 2
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=91, h0=True, dh=True, per_dict=True)
    inp["dict_idx"][0, 1, :] = 5
    d = to_dev(inp, False)
    d["diag"] = torch.from_numpy(inp["diag"]).cuda()
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=d["h0"], per_dict=True)
    torch.cuda.synchronize()
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz = O.gather_D_per_dict(O.planes_to_complex(inp["diag"]), inp["kstar"])
    h = O.scan_forward(Pm, Dz, O.planes_to_complex(inp["bias"]), O.planes_to_complex(inp["h0"]))
    check("h", cpx(f["h"]), h, 1e-4)


PAIRED_CASES = [
    # B, H, L, N, K, c, bf16: N = 64, B even, B*H > #SMs -> two sequences of a head per CTA
    (20, 8, 300, 64, 48, 1, True),
    (20, 8, 77, 64, 16, 2, False),
    (38, 4, 129, 64, 5, 1, False),
]


@pytest.mark.parametrize("case", PAIRED_CASES, ids=[str(c) for c in PAIRED_CASES])
@pytest.mark.parametrize("pair_bwd", [False, True], ids=["bwd_single", "bwd_paired"])
def test_seq_paired_sequences_per_cta(P, case, pair_bwd, monkeypatch):
    """Single-chunk kernels with two sequences (batch rows b, b+1) of one head per CTA (the config-4
    launch shape of the forward; the paired backward is opt-in, PDSSM_SEQ_PAIR_BWD): every sequence
    against the oracle, and bitwise run-to-run repeatability."""
    monkeypatch.delenv("PDSSM_PATH", raising=False)
    if pair_bwd:
        monkeypatch.setenv("PDSSM_SEQ_PAIR_BWD", "1")
    else:
        monkeypatch.delenv("PDSSM_SEQ_PAIR_BWD", raising=False)
    B, H, L, N, K, c, bf16 = case
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=B + L, dh=True, bf16=bf16)
    d = to_dev(inp, bf16)
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"])
    assert f["tau"] == L
    db, dD, g, _ = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"], dh=d["dh"],
                              want_dh0=False)
    torch.cuda.synchronize()
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, e = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "dh"))
    h = O.scan_forward(Pm, Dz, bz)
    tol = TOL["bf16" if bf16 else "f32"]
    check("paired_h", cpx(f["h"]), h, tol)
    db_r, dD_r, g_r, _ = O.scan_backward(Pm, Dz, saved_states(h, c, bf16), e)
    check("paired_db", cpx(db), db_r, tol)
    check("paired_dD", cpx(dD), dD_r, tol)
    check("paired_g", g.cpu().numpy(), g_r, tol)
    f2 = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"])
    torch.cuda.synchronize()
    assert torch.equal(f["h"], f2["h"])


SEQC_CASES = [
    # B, H, L, N, K, c, tau, bf16, per_dict: chunked single-CTA path (k_fwd_seq / k_bwd_seq MODE 1 / 2)
    (1, 2, 1000, 128, 32, 2, 300, False, False),    # tau > the warp-per-chunk cap: the library's choice
    (1, 2, 1000, 128, 32, 2, 300, True, False),
    (2, 2, 777, 64, 16, 1, 96, False, False),       # forced (PDSSM_PATH=seqc), ragged last chunk
    (2, 1, 500, 32, 5, 2, 128, False, True),        # PER_DICT
    (1, 3, 333, 96, 8, 2, 100, False, False),       # N = 96 (runtime N)
]


@pytest.mark.parametrize("case", SEQC_CASES, ids=[str(c) for c in SEQC_CASES])
def test_seqc_chunked_single_cta_path(P, case, monkeypatch):
    """One CTA per (sequence, chunk): Phase A (chunk aggregates from a zero state) -> Phase B (carries,
    maps) -> Phase C (replay), and the mirrored backward; every output against the oracle, chunk-level
    intermediates against the float64 chunked oracle at the same tau, maps bit-exact."""
    B, H, L, N, K, c, tau, bf16, pd = case
    monkeypatch.setenv("PDSSM_PATH", "seqc")
    inp, f, got, ch, ref, Pm, Dz = run_case(P, B, H, L, N, K, c, tau, bf16=bf16, per_dict=pd, seed=L + tau)
    assert f["tau"] == tau
    tol = TOL["bf16" if bf16 else "f32"]
    check("seqc_h", cpx(f["h"]), ch["h"], tol)
    assert np.array_equal(f["maps"].cpu().numpy().astype(np.int64), ch["maps"])
    pi, d_bar, beta_bar, carry = P.chunk_state_views(f["chunk_state"], f["dims"])
    assert np.array_equal(pi.cpu().numpy().astype(np.int64), ch["pi_bar"])
    check("seqc_d_bar", O.planes_to_complex(d_bar.cpu().numpy()), ch["d_bar"], 1e-4)
    check("seqc_beta_bar", O.planes_to_complex(beta_bar.cpu().numpy()), ch["beta_bar"], 1e-4)
    check("seqc_carry", O.planes_to_complex(carry.cpu().numpy()), ch["carries"], 1e-4)
    db, dD, g, dh0 = got
    db_r, dD_r, g_r, dh0_r = ref
    check("seqc_db", cpx(db), db_r, tol)
    check("seqc_g", g.cpu().numpy(), g_r, tol)
    check("seqc_dh0", O.planes_to_complex(dh0.cpu().numpy()), dh0_r, tol)
    if pd:
        dDk = np.zeros((H, K, N), np.complex128)
        for b in range(B):
            for hh in range(H):
                np.add.at(dDk[hh], inp["kstar"][b, hh], dD_r[b, hh])
        check("seqc_dD_k", O.planes_to_complex(dD.cpu().numpy()), dDk, tol)
    else:
        check("seqc_dD", cpx(dD), dD_r, tol)


def test_default_chunk_policy(P, monkeypatch):
    """Library default tau (R20): one CTA per sequence when the sequences fill most SMs (config 2
    fp32 and bf16, config 4); the chunked single-CTA path with ~2.8 chunks per SM for few, long
    sequences (configs 3 and 5); the warp-per-chunk path (tau 64) when chunks would be short."""
    monkeypatch.delenv("PDSSM_PATH", raising=False)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    d = lambda B, H, L, N, K, c, dt: P.default_chunk(P.make_dims(B, H, L, N, K, c=c, dtype=dt))
    assert d(16, 8, 2048, 128, 32, 2, P.F32) == 2048
    assert d(16, 8, 2048, 128, 32, 2, P.BF16) == 2048
    assert d(32, 32, 4096, 64, 48, 1, P.BF16) == 4096
    chunks = lambda S: -(-28 * sms // (10 * S))
    assert d(4, 8, 17984, 128, 32, 1, P.F32) == -(-17984 // chunks(32))
    assert d(4, 4, 65536, 64, 16, 1, P.F32) == -(-65536 // chunks(16))
    assert d(1, 2, 300, 128, 32, 2, P.F32) == 64
