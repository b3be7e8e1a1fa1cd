"""Recompute mode of the backward (include/pdssm.h pdssm_scan_bwd with h_saved_opt = NULL):
the states are replayed per chunk from bias + the chunk carries of chunk_state, so the
forward's O(L N) states need not be kept.  Parity against the float64
oracle (reading R19 bars, per tensor and per (b, h)), and agreement with the saved-state
backward."""
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


def dev_inputs(inp, bf16, per_dict):
    d = {}
    for k, v in inp.items():
        t = torch.from_numpy(np.ascontiguousarray(v)).cuda()
        if k == "dict_idx":
            t = t.to(torch.int16)
        elif bf16 and k in ("bias", "dh") or (bf16 and k == "diag" and not per_dict):
            t = t.to(torch.bfloat16)
        d[k] = t
    return d


RC_CASES = [
    # B, H, L, N, K, c, tau, bf16, per_dict, h0
    (2, 2, 300, 128, 32, 2, 64, False, False, True),     # config-2 state size, ragged last chunk
    (1, 3, 257, 64, 16, 1, 32, False, False, False),
    (2, 1, 100, 5, 3, 2, 7, False, False, True),         # N not a multiple of 32, tiny chunks
    (1, 2, 129, 200, 8, 2, 16, False, False, True),      # N = 200
    (2, 2, 190, 32, 7, 2, 190, False, False, True),      # one chunk (tau = L)
    (1, 1, 1, 16, 4, 2, 8, False, False, True),          # L = 1
    (2, 2, 300, 128, 32, 2, 64, True, False, True),      # bf16
    (1, 2, 200, 64, 6, 2, 32, False, True, True),        # PER_DICT
    (1, 1, 64, 1024, 4, 1, 16, False, False, True),      # N = 1024 (the ABI maximum)
]


@pytest.mark.parametrize("case", RC_CASES, ids=[str(c) for c in RC_CASES])
@pytest.mark.parametrize("path", ["auto", "generic"])
def test_recompute_backward_parity(P, case, path, monkeypatch):
    """auto: one CTA per sequence (k_bwd_seq_rc) where N % 32 == 0 and N <= 128, else the generic
    per-(sequence, chunk) kernel; generic: always the latter."""
    B, H, L, N, K, c, tau, bf16, pd, use_h0 = case
    if path == "generic":
        monkeypatch.setenv("PDSSM_PATH", "generic")
    else:
        monkeypatch.delenv("PDSSM_PATH", raising=False)
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=L + N + tau, h0=use_h0, dh=True, per_dict=pd, bf16=bf16)
    d = dev_inputs(inp, bf16, pd)
    h0 = d.get("h0")
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=h0, tau=tau, per_dict=pd)
    assert f["tau"] == min(tau, L)
    db, dD, g, dh0 = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], None, f["chunk_state"], f["dims"],
                                dh=d["dh"], h0=h0, bias=d["bias"])
    torch.cuda.synchronize()
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz = O.planes_to_complex(inp["diag"])
    if pd:
        Dz = O.gather_D_per_dict(Dz, inp["kstar"])
    bz, e = O.planes_to_complex(inp["bias"]), O.planes_to_complex(inp["dh"])
    h0z = O.planes_to_complex(inp["h0"]) if use_h0 else None
    h = O.scan_forward(Pm, Dz, bz, h0z)
    # recompute mode replays the states in f32: the oracle's backward reads its exact states
    db_r, dD_r, g_r, dh0_r = O.scan_backward(Pm, Dz, h, e, h0z)
    tol = TOL["bf16" if bf16 else "f32"]
    cp = lambda t: O.planes_to_complex(t.float().cpu().numpy())
    check("rc_db", cp(db), db_r, tol)
    check("rc_g", g.cpu().numpy(), g_r, tol)
    check("rc_dh0", cp(dh0), dh0_r, tol)
    if pd:
        dDk = np.zeros((H, K, N), np.complex128)
        for b in range(B):
            for hh in range(H):
                np.add.at(dDk[hh], inp["kstar"][b, hh], dD_r[b, hh])
        check("rc_dD_k", cp(dD), dDk, tol)
    else:
        check("rc_dD", cp(dD), dD_r, tol)


def test_recompute_matches_saved_backward(P):
    """Same forward, both backward modes (the generic saved-state kernels and the recompute kernel):
    every output agrees to f32 rounding (different summation orders, and recomputed vs stored states)."""
    B, H, L, N, K, c, tau = 2, 2, 333, 64, 16, 2, 48
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=5, h0=True, dh=True)
    d = dev_inputs(inp, False, False)
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=d["h0"], tau=tau)
    import os
    old = os.environ.get("PDSSM_PATH")
    os.environ["PDSSM_PATH"] = "generic"     # the saved-state three-phase backward
    try:
        a = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"], dh=d["dh"],
                       h0=d["h0"])
    finally:
        if old is None:
            del os.environ["PDSSM_PATH"]
        else:
            os.environ["PDSSM_PATH"] = old
    b = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], None, f["chunk_state"], f["dims"], dh=d["dh"], h0=d["h0"],
                   bias=d["bias"])
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert float((x - y).abs().max()) <= 1e-5 * float(x.abs().max())


def test_recompute_rejects_long_chunks(P):
    B, H, L, N, K, c = 1, 1, 4096, 128, 4, 2
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=1, dh=True)
    d = dev_inputs(inp, False, False)
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], tau=L)
    with pytest.raises(P.PdssmError, match="UNSUPPORTED"):
        P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], None, f["chunk_state"], f["dims"], dh=d["dh"],
                   bias=d["bias"])
