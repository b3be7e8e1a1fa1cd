"""Pins of the float64 oracle against things the paper and the mathematics fix
(not against the oracle itself): dense matrix products built from the App. D
definition, closed forms, FSA emulation vs independent interpreters (Prop. 1),
S_5 group products via sympy, central finite differences, brute-force argmax.
All CPU (`-m "not gpu"`)."""
import itertools
import math

import numpy as np
import pytest

import oracle as O
from oracle import fsa
import synth

RNG = np.random.default_rng(1234)


def crand(*shape, rng=RNG):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def dense_from_def(P, D):
    """A = sum_j D[j] e_{P[j]} e_j^T -- the column-one-hot matrix of PAPER.md:143
    / the App. D sum of outer products, built independently."""
    N = len(P)
    A = np.zeros((N, N), dtype=np.complex128)
    for j in range(N):
        ej = np.zeros(N)
        ej[j] = 1.0
        ei = np.zeros(N)
        ei[P[j]] = 1.0
        A += D[j] * np.outer(ei, ej)
    return A


# ---------------------------------------------------------------- a1 sparsify
def test_sparsify_bruteforce_and_ties():
    M = RNG.standard_normal((2, 3, 7, 7))
    M[0, 0, :, 3] = 0.5          # all-equal column -> 0
    M[1, 2, 2, 5] = M[1, 2, 4, 5] = 10.0   # tie between rows 2 and 4 -> 2
    idx = O.sparsify(M)
    for h, k, j in itertools.product(range(2), range(3), range(7)):
        best, arg = -np.inf, -1
        for i in range(7):
            if M[h, k, i, j] > best:        # strict: first max wins
                best, arg = M[h, k, i, j], i
        assert idx[h, k, j] == arg
    assert idx[0, 0, 3] == 0 and idx[1, 2, 5] == 2


def test_sparsify_diag_is_identity_and_nan_raises():
    M = np.tile(np.eye(6) * 3.0 - 1.0, (1, 2, 1, 1))
    assert (O.sparsify(M) == np.arange(6)).all()
    M[0, 1, 2, 2] = np.nan
    with pytest.raises(ValueError):
        O.sparsify(M)


# ---------------------------------------------------------------- a2/a3 select
def test_select_integer_exact_and_ties():
    x = synth.tokens_x(2, 9, 5, seed=3, tie_dense=True)
    S = synth.selector(3, 4, 5, seed=3, tie_dense=True)
    k, logits = O.select(x, S)
    for b, h, t in itertools.product(range(2), range(3), range(9)):
        row = [sum(int(S[h, kk, d]) * int(x[b, t, d]) for d in range(5)) for kk in range(4)]
        assert list(logits[b, h, t]) == row
        m = max(row)
        assert k[b, h, t] == row.index(m)        # first maximum
    assert (logits == np.round(logits)).all()


def test_argmax_nan_rule():
    v = np.array([[np.nan, 1.0, 1.0], [np.nan, np.nan, np.nan], [-np.inf, -np.inf, 0.0],
                  [-np.inf, -np.inf, -np.inf], [np.nan, -np.inf, 2.0]])
    assert list(O.argmax_smallest(v)) == [1, 0, 2, 0, 2]


def test_gather_P_definition():
    d = synth.random_maps(2, 5, 6, seed=9)
    k = synth.kstar(3, 2, 4, 5, seed=9)
    P = O.gather_P(d, k)
    for b, h, t in itertools.product(range(3), range(2), range(4)):
        assert (P[b, h, t] == d[h, k[b, h, t]]).all()


# ---------------------------------------------------------------- PD algebra
def test_pd_apply_matches_dense_definition():
    for N in (1, 2, 5, 8):
        for _ in range(20):
            P = RNG.integers(0, N, N)
            D = crand(N)
            h = crand(N)
            assert np.allclose(O.pd_apply(P, D, h), dense_from_def(P, D) @ h, atol=1e-13)
    # SPEC.md:101 collapsing map -> [a+b, 0]; SPEC.md:137 placement [[0,3],[2,0]]
    assert np.allclose(O.pd_apply([0, 0], [1, 1], np.array([2.0, 5.0])), [7.0, 0.0])
    assert np.allclose(O.pd_apply([1, 0], [2, 3], np.array([1.0, 10.0])), np.array([[0, 3], [2, 0]]) @ [1.0, 10.0])


def test_pd_transpose_adjoint_identity():
    for N in (2, 5, 8):
        P = RNG.integers(0, N, N)
        D = crand(N)
        x, g = crand(N), crand(N)
        lhs = np.sum(np.real(np.conj(O.pd_apply(P, D, x)) * g))   # real inner product
        rhs = np.sum(np.real(np.conj(x) * O.pd_apply_transpose(P, D, g)))
        assert abs(lhs - rhs) < 1e-12
        # equals the conjugate-transposed dense matrix
        assert np.allclose(O.pd_apply_transpose(P, D, g), dense_from_def(P, D).conj().T @ g)
    assert np.allclose(O.pd_apply_transpose([0, 0], [1, 1], np.array([3.0, 4.0])), [3.0, 3.0])


def test_pd_compose_closure_associativity():
    N = 7
    for _ in range(20):
        P1, P2, P3 = (RNG.integers(0, N, N) for _ in range(3))
        D1, D2, D3 = crand(N), crand(N), crand(N)
        pi, d = O.pd_compose(P2, D2, P1, D1)
        assert np.allclose(dense_from_def(pi, d), dense_from_def(P2, D2) @ dense_from_def(P1, D1))
        a = O.pd_compose(P3, D3, *O.pd_compose(P2, D2, P1, D1))
        b = O.pd_compose(*O.pd_compose(P3, D3, P2, D2), P1, D1)
        assert (a[0] == b[0]).all() and np.allclose(a[1], b[1])
    sw = np.array([1, 0])
    pi, d = O.pd_compose(sw, np.ones(2), sw, np.ones(2))
    assert (pi == [0, 1]).all() and (d == 1).all()


# ---------------------------------------------------------------- forward scan
@pytest.mark.parametrize("c", [1, 2])
def test_scan_forward_matches_dense_recurrence(c):
    B, H, L, N = 2, 2, 23, 6
    P = RNG.integers(0, N, (B, H, L, N))
    D = crand(B, H, L, N) if c == 2 else RNG.standard_normal((B, H, L, N)) + 0j
    b = crand(B, H, L, N) if c == 2 else RNG.standard_normal((B, H, L, N)) + 0j
    h0 = crand(B, H, N)
    h = O.scan_forward(P, D, b, h0)
    for bb, hh in itertools.product(range(B), range(H)):
        cur = h0[bb, hh]
        for t in range(L):
            cur = dense_from_def(P[bb, hh, t], D[bb, hh, t]) @ cur + b[bb, hh, t]
            assert np.allclose(h[bb, hh, t], cur, atol=1e-12, rtol=1e-12)


def test_scan_closed_forms():
    B, H, L, N = 1, 2, 17, 5
    ident = np.tile(np.arange(N), (B, H, L, 1))
    cvec = crand(B, H, N)
    h0 = crand(B, H, N)
    b = np.repeat(cvec[:, :, None, :], L, axis=2)
    h = O.scan_forward(ident, np.ones((B, H, L, N)), b, h0)
    for t in range(L):                       # h_t = h0 + (t+1) c
        assert np.allclose(h[:, :, t], h0 + (t + 1) * cvec, atol=1e-12)
    # L = 1
    P = RNG.integers(0, N, (B, H, 1, N))
    D = crand(B, H, 1, N)
    b1 = crand(B, H, 1, N)
    h1 = O.scan_forward(P, D, b1, h0)
    for hh in range(H):
        assert np.allclose(h1[0, hh, 0], dense_from_def(P[0, hh, 0], D[0, hh, 0]) @ h0[0, hh] + b1[0, hh, 0])
    # permutations with D = 1, b = 0: h_t[Pi_t[j]] = h0[j] exactly
    Pp = np.stack([[RNG.permutation(N) for _ in range(L)] for _ in range(H)])[None]
    h0r = np.arange(N, dtype=float)[None, None].repeat(H, 1)
    hp = O.scan_forward(Pp, np.ones((1, H, L, N)), np.zeros((1, H, L, N)), h0r)
    Pi, rho = O.prefix_maps(Pp, np.ones((1, H, L, N)))
    for hh, t in itertools.product(range(H), range(L)):
        expect = np.zeros(N)
        expect[Pi[0, hh, t]] = np.arange(N)
        assert (hp[0, hh, t].real == expect).all()
    assert (rho == 1).all()


def test_scan_linearity_and_head_independence():
    B, H, L, N = 1, 3, 12, 5
    P = RNG.integers(0, N, (B, H, L, N))
    D = crand(B, H, L, N)
    b1, b2 = crand(B, H, L, N), crand(B, H, L, N)
    a, bcoef = 0.7 - 0.2j, -1.3
    lhs = O.scan_forward(P, D, a * b1 + bcoef * b2)
    rhs = a * O.scan_forward(P, D, b1) + bcoef * O.scan_forward(P, D, b2)
    assert np.allclose(lhs, rhs, atol=1e-12)
    b3 = b1.copy()
    b3[:, 1] = 0
    h3 = O.scan_forward(P, D, b3)
    h1 = O.scan_forward(P, D, b1)
    assert (h3[:, 0] == h1[:, 0]).all() and (h3[:, 2] == h1[:, 2]).all()


def test_prefix_maps_are_dense_products():
    B, H, L, N = 1, 1, 9, 6
    P = RNG.integers(0, N, (B, H, L, N))
    D = crand(B, H, L, N)
    Pi, rho = O.prefix_maps(P, D)
    M = np.eye(N, dtype=np.complex128)
    for t in range(L):
        M = dense_from_def(P[0, 0, t], D[0, 0, t]) @ M
        assert np.allclose(dense_from_def(Pi[0, 0, t], rho[0, 0, t]), M, atol=1e-12)


# ---------------------------------------------------------------- chunked (Alg. 1)
@pytest.mark.parametrize("tau", [1, 2, 5, 7, 23, 64])
def test_chunked_equals_sequential(tau):
    B, H, L, N = 2, 2, 23, 6
    P = RNG.integers(0, N, (B, H, L, N))
    D = crand(B, H, L, N) * 0.8
    b = crand(B, H, L, N)
    h0 = crand(B, H, N)
    seq = O.scan_forward(P, D, b, h0)
    ch = O.scan_chunked(P, D, b, tau, h0)
    assert np.allclose(ch["h"], seq, atol=1e-12)
    Pi, rho = O.prefix_maps(P, D)
    bounds = O.chunk_bounds(L, tau)
    for c, (s, e) in enumerate(bounds):
        # carry = true state before the chunk; maps = composed map before the chunk
        want = h0 if s == 0 else seq[:, :, s - 1]
        assert np.allclose(ch["carries"][:, :, c], want, atol=1e-12)
        if s > 0:
            assert (ch["maps"][:, :, c] == Pi[:, :, s - 1]).all()
        else:
            assert (ch["maps"][:, :, 0] == np.arange(N)).all()
        # aggregate = dense product of the chunk's matrices and local replay
        for bb, hh in itertools.product(range(B), range(H)):
            M = np.eye(N, dtype=np.complex128)
            beta = np.zeros(N, np.complex128)
            for t in range(s, e):
                A = dense_from_def(P[bb, hh, t], D[bb, hh, t])
                M = A @ M
                beta = A @ beta + b[bb, hh, t]
            assert np.allclose(dense_from_def(ch["pi_bar"][bb, hh, c], ch["d_bar"][bb, hh, c]), M, atol=1e-12)
            assert np.allclose(ch["beta_bar"][bb, hh, c], beta, atol=1e-12)
    assert (ch["maps"][:, :, -1] == Pi[:, :, -1]).all()
    assert np.allclose(ch["final"], seq[:, :, -1], atol=1e-12)


# ---------------------------------------------------------------- FSA (Prop. 1)
FSAS = [(fsa.parity, fsa.interp_parity, 8), (fsa.cyclic_z5, fsa.interp_z5, 6),
        (fsa.cycle_nav, fsa.interp_cycle_nav, 7), (fsa.even_pairs, fsa.interp_even_pairs, 8),
        (fsa.mod_arith, fsa.interp_mod_arith, 5)]


@pytest.mark.parametrize("make,interp,maxlen", FSAS, ids=[f[0].__name__ for f in FSAS])
def test_fsa_emulation_exact(make, interp, maxlen):
    A = make()
    dict_idx, dg, h0, C = A.compile()
    for L in range(1, maxlen + 1):
        words = np.array(list(itertools.product(range(A.K), repeat=L)), dtype=np.int64)
        # delta table vs independent interpreter (final label)
        for w in words[:: max(1, len(words) // 400)]:
            assert A.label[A.run(list(w))[-1]] == interp(list(w))
        Bn = len(words)
        kst = words[:, None, :].astype(np.uint8)
        P = O.gather_P(dict_idx, kst)
        D = np.ones((Bn, 1, L, A.N))
        h = O.scan_forward(P, D, np.zeros((Bn, 1, L, A.N)), np.tile(h0, (Bn, 1, 1)))
        runs = np.array([A.run(list(w)) for w in words])
        onehot = np.zeros((Bn, L, A.N))
        np.put_along_axis(onehot, runs[:, :, None], 1.0, axis=2)
        assert (h[:, 0].real == onehot).all() and (h.imag == 0).all()
        y = O.readout(h, C[None].astype(np.complex128))
        lab = A.label[runs]
        assert (np.argmax(y[:, :, 0], axis=-1) == lab).all()


def test_fsa_scatter_is_load_bearing():
    """the gather reading of App. E (x[i] = D[q] x[q], q = P[i]) does not keep
    states one-hot for non-injective delta."""
    A = fsa.mod_arith()
    dict_idx, _, h0, _ = A.compile()
    tokens = [7, 0]          # '*' then 0: collapse
    h = h0.copy()
    for s in tokens:
        h = h[dict_idx[0, s].astype(np.int64)]
    assert h.sum() != 1.0            # gather reading loses the one-hot state
    hs = O.scan_forward(O.gather_P(dict_idx, np.array([[tokens]], np.uint8)), np.ones((1, 1, 2, A.N)),
                        np.zeros((1, 1, 2, A.N)), h0[None, None])
    assert hs[0, 0, -1].real.sum() == 1.0 and hs[0, 0, -1].real[A.run(tokens)[-1]] == 1.0


def test_s5_word_problem_against_sympy():
    from sympy.combinatorics import Permutation, PermutationGroup
    dict_idx, perms5, blocks = synth.s5_dictionary(N=64, K=16, seed=5000)
    G = PermutationGroup([Permutation(list(p)) for p in perms5])
    assert G.order() == 120
    L = 300
    k = synth.kstar(1, 1, L, 16, seed=5003)
    P = O.gather_P(dict_idx[None], k)
    Pi, rho = O.prefix_maps(P, np.ones(P.shape))
    # sympy: applying p_0 then p_1 ... : composed = p_{L-1} o ... o p_0
    total = Permutation(list(range(5)))
    for t in range(L):
        total = total * Permutation(list(perms5[k[0, 0, t]]))   # sympy: apply left factor first
        img = total.array_form
        for blk in blocks[:3]:
            for a in range(5):
                assert Pi[0, 0, t, blk[a]] == blk[img[a]]
    # states: h0 = arange, D = 1, b = 0 -> exact permuted arange
    h0 = np.arange(64, dtype=float)[None, None]
    h = O.scan_forward(P, np.ones(P.shape), np.zeros(P.shape), h0)
    expect = np.zeros(64)
    expect[Pi[0, 0, -1]] = np.arange(64)
    assert (h[0, 0, -1].real == expect).all()


# ---------------------------------------------------------------- backward (App. C)
def _loss_setup(c, seed):
    rng = np.random.default_rng(seed)
    B, H, L, N = 1, 2, 7, 5
    P = rng.integers(0, N, (B, H, L, N))
    if c == 2:
        D = (rng.standard_normal((B, H, L, N)) + 1j * rng.standard_normal((B, H, L, N))) * 0.6
        b = rng.standard_normal((B, H, L, N)) + 1j * rng.standard_normal((B, H, L, N))
        h0 = rng.standard_normal((B, H, N)) + 1j * rng.standard_normal((B, H, N))
        W = rng.standard_normal((B, H, L, N)) + 1j * rng.standard_normal((B, H, L, N))
    else:
        D = rng.standard_normal((B, H, L, N)) * 0.6 + 0j
        b = rng.standard_normal((B, H, L, N)) + 0j
        h0 = rng.standard_normal((B, H, N)) + 0j
        W = rng.standard_normal((B, H, L, N)) + 0j
    return P, D, b, h0, W


def _loss(P, D, b, h0, W):
    h = O.scan_forward(P, D, b, h0)
    return float(np.sum(np.real(np.conj(W) * h)))     # dl/dh packed = W


@pytest.mark.parametrize("c", [1, 2])
def test_backward_finite_differences(c):
    P, D, b, h0, W = _loss_setup(c, 7 + c)
    h = O.scan_forward(P, D, b, h0)
    db, dD, g, dh0 = O.scan_backward(P, D, h, W, h0)
    eps = 1e-6
    comps = [1.0, 1j] if c == 2 else [1.0]

    def fd(arr_name, idx, unit):
        args = dict(P=P, D=D.copy(), b=b.copy(), h0=h0.copy(), W=W)
        args[arr_name] = args[arr_name].copy()
        args[arr_name][idx] += eps * unit
        lp = _loss(**args)
        args[arr_name][idx] -= 2 * eps * unit
        lm = _loss(**args)
        return (lp - lm) / (2 * eps)

    for idx in [(0, 0, 0, 1), (0, 1, 3, 4), (0, 0, 6, 2), (0, 1, 5, 0)]:
        for u in comps:
            want_b = fd("b", idx, u)
            want_D = fd("D", idx, u)
            got_b = db[idx].real if u == 1.0 else db[idx].imag
            got_D = dD[idx].real if u == 1.0 else dD[idx].imag
            assert abs(got_b - want_b) < 1e-6 * max(1, abs(want_b))
            assert abs(got_D - want_D) < 1e-6 * max(1, abs(want_D))
    for idx in [(0, 0, 1), (0, 1, 4)]:
        for u in comps:
            want = fd("h0", idx, u)
            got = dh0[idx].real if u == 1.0 else dh0[idx].imag
            assert abs(got - want) < 1e-6 * max(1, abs(want))
    # g_t = d loss / d s for A_t -> (1+s) A_t  (the selected matrix's scale)
    for (bb, hh, t) in [(0, 0, 0), (0, 1, 4), (0, 0, 6)]:
        Dp, Dm = D.copy(), D.copy()
        Dp[bb, hh, t] *= (1 + eps)
        Dm[bb, hh, t] *= (1 - eps)
        want = (_loss(P, Dp, b, h0, W) - _loss(P, Dm, b, h0, W)) / (2 * eps)
        assert abs(g[bb, hh, t] - want) < 1e-6 * max(1, abs(want))


def test_readout_and_adjoint():
    rng = np.random.default_rng(5)
    B, H, L, N, Pp = 1, 2, 3, 4, 3
    h = rng.standard_normal((B, H, L, N)) + 1j * rng.standard_normal((B, H, L, N))
    C = rng.standard_normal((H, Pp, N)) + 1j * rng.standard_normal((H, Pp, N))
    y = O.readout(h, C)
    for bb, hh, t, p in itertools.product(range(B), range(H), range(L), range(Pp)):
        want = sum(C[hh, p, j].real * h[bb, hh, t, j].real - C[hh, p, j].imag * h[bb, hh, t, j].imag for j in range(N))
        assert abs(y[bb, t, hh, p] - want) < 1e-12
    dy = rng.standard_normal(y.shape)
    e = O.readout_adjoint(dy, C)
    eps = 1e-6
    for idx in [(0, 0, 0, 1), (0, 1, 2, 3)]:
        for u in (1.0, 1j):
            hp, hm = h.copy(), h.copy()
            hp[idx] += eps * u
            hm[idx] -= eps * u
            want = (np.sum(dy * O.readout(hp, C)) - np.sum(dy * O.readout(hm, C))) / (2 * eps)
            got = e[idx].real if u == 1.0 else e[idx].imag
            assert abs(got - want) < 1e-6


@pytest.mark.parametrize("tau", [1, 3, 7, 30])
def test_backward_chunked_equals_sequential(tau):
    P, D, b, h0, W = _loss_setup(2, 11)
    h = O.scan_forward(P, D, b, h0)
    db, dD, g, dh0 = O.scan_backward(P, D, h, W, h0)
    pi_bar, d_bar, _ = O.chunk_aggregates(P, D, b, tau)
    r = O.scan_backward_chunked(P, D, W, pi_bar, d_bar, tau)
    assert np.allclose(r["lam"], db, atol=1e-12)
    assert np.allclose(r["dh0"], dh0, atol=1e-12)
    # mu_c = lambda at the chunk's last step minus its direct term
    for c, (s, e) in enumerate(O.chunk_bounds(P.shape[2], tau)):
        assert np.allclose(r["mu"][:, :, c], db[:, :, e - 1] - W[:, :, e - 1], atol=1e-12)


# ---------------------------------------------------------------- SP summaries
def test_segment_summaries_compose_to_carries():
    B, H, L, N = 1, 2, 40, 6
    P = RNG.integers(0, N, (B, H, L, N))
    D = crand(B, H, L, N) * 0.7
    b = crand(B, H, L, N)
    h0 = crand(B, H, N)
    seq = O.scan_forward(P, D, b, h0)
    Pi, _ = O.prefix_maps(P, D)
    G = 4
    segs = [(g * L // G, (g + 1) * L // G) for g in range(G)]
    summ = [O.segment_summary(P[:, :, s:e], D[:, :, s:e], b[:, :, s:e]) for s, e in segs]
    pis, ds, betas = zip(*summ)
    for g, (s, e) in enumerate(segs):
        carry, m = O.compose_summaries(pis, ds, betas, g, h0)
        want = h0 if s == 0 else seq[:, :, s - 1]
        assert np.allclose(carry, want, atol=1e-12)
        if s > 0:
            assert (m == Pi[:, :, s - 1]).all()


def test_project_b_one_hot_columns_and_per_dict_gather():
    rng = np.random.default_rng(8)
    H, N, d_in = 2, 4, 5
    Bw = rng.standard_normal((H, N, d_in)) + 1j * rng.standard_normal((H, N, d_in))
    x = np.zeros((1, d_in, d_in))
    x[0] = np.eye(d_in)                      # token t is the one-hot e_t
    b = O.project_b(x, Bw)
    for h, t in itertools.product(range(H), range(d_in)):
        assert np.array_equal(b[0, h, t], Bw[h, :, t])
    Dk = rng.standard_normal((H, 3, N)) + 0j
    k = synth.kstar(2, H, 6, 3, seed=1)
    Dt = O.gather_D_per_dict(Dk, k)
    for bb, h, t in itertools.product(range(2), range(H), range(6)):
        assert np.array_equal(Dt[bb, h, t], Dk[h, k[bb, h, t]])


# ---------------------------------------------------------------------------
# NEXT-1: Prop. 2 surrogate gradients (App. C :814-841)
# The pins differentiate, by central finite differences, the relaxed functionals the
# straight-through estimator linearises (hardmax -> tempered softmax),
# written here directly (softmax + inner products), not the oracle's Jacobian formulas.
def _test_softmax(z, T, axis):
    e = np.exp((z - z.max(axis=axis, keepdims=True)) / T)
    return e / e.sum(axis=axis, keepdims=True)


@pytest.mark.parametrize("T", [1.0, 0.3])
def test_selector_grad_finite_differences(T):
    rng = np.random.default_rng(71)
    B, H, L, K = 2, 2, 5, 6
    z = rng.normal(size=(B, H, L, K))
    ks = rng.integers(0, K, size=(B, H, L))
    g = rng.normal(size=(B, H, L))

    def f(zz):   # sum_t g_t softmax_T(z_t)[k*_t]: the activated coordinate of v_t^soft
        s = _test_softmax(zz, T, -1)
        return float(np.sum(g * np.take_along_axis(s, ks[..., None], -1)[..., 0]))

    got = O.selector_grad(z, ks, g, T)
    eps = 1e-6
    fd = np.zeros_like(z)
    for idx in itertools.product(*(range(n) for n in z.shape)):
        zp, zm = z.copy(), z.copy()
        zp[idx] += eps
        zm[idx] -= eps
        fd[idx] = (f(zp) - f(zm)) / (2 * eps)
    assert np.max(np.abs(got - fd)) <= 1e-7 * max(1.0, np.max(np.abs(fd)))
    # softmax-Jacobian rows sum to zero; g = 0 (lambda = 0) gives zero
    assert np.allclose(got.sum(-1), 0.0, atol=1e-12)
    assert np.all(O.selector_grad(z, ks, np.zeros_like(g), T) == 0.0)


def test_selector_grad_two_way_closed_form():
    """K = 2, equal logits, k* = 0: s = (1/2, 1/2), so dl/dz = g (1/2)((1,0) - (1/2,1/2)) / T = g/T (1/4, -1/4)."""
    g, T = 1.7, 0.5
    got = O.selector_grad(np.zeros((1, 1, 1, 2)), np.zeros((1, 1, 1), np.int64), np.full((1, 1, 1), g), T)
    assert np.allclose(got[0, 0, 0], [g / T / 4, -g / T / 4], rtol=0, atol=1e-15)


@pytest.mark.parametrize("c", [1, 2])
def test_dictionary_outer_is_dP_of_linear_functional(c):
    """G_k = d/dP_k of sum_t Re<lambda_t, P_{k*_t} D_t h_{t-1}>, with P_k a free dense matrix
    (linear in P, so central differences are exact up to rounding)."""
    rng = np.random.default_rng(72 + c)
    B, H, L, N, K = 2, 2, 7, 4, 3
    cz = (lambda *s: rng.normal(size=s) + 1j * rng.normal(size=s)) if c == 2 else (lambda *s: rng.normal(size=s) + 0j)
    lam, D, h, h0 = cz(B, H, L, N), cz(B, H, L, N), cz(B, H, L, N), cz(B, H, N)
    ks = rng.integers(0, K, size=(B, H, L))
    hprev = np.concatenate([h0[:, :, None], h[:, :, :-1]], axis=2)

    def f(Pd):   # Pd [H,K,N,N] dense
        tot = 0.0
        for b in range(B):
            for hh in range(H):
                for t in range(L):
                    v = Pd[hh, ks[b, hh, t]] @ (D[b, hh, t] * hprev[b, hh, t])
                    tot += float(np.real(np.vdot(lam[b, hh, t], v)))
        return tot

    G = O.dictionary_outer(ks, lam, D, h, K, h0=h0)
    P0 = rng.normal(size=(H, K, N, N))
    fd = np.zeros_like(P0)
    for idx in itertools.product(*(range(n) for n in P0.shape)):
        Pp, Pm = P0.copy(), P0.copy()
        Pp[idx] += 0.5
        Pm[idx] -= 0.5
        fd[idx] = f(Pp) - f(Pm)
    assert np.max(np.abs(G - fd)) <= 1e-10 * max(1.0, np.max(np.abs(fd)))


@pytest.mark.parametrize("T", [1.0, 0.25])
def test_dictionary_grad_finite_differences(T):
    """dM = d/dM of sum_t Re<lambda_t, softmax_T(M_{k*_t}) D_t h_{t-1}>, the column softmax
    replacing the column hardmax of Eq. 5 with lambda, D, h held fixed."""
    rng = np.random.default_rng(73)
    B, H, L, N, K = 2, 1, 6, 4, 3
    lam = rng.normal(size=(B, H, L, N)) + 1j * rng.normal(size=(B, H, L, N))
    D = rng.normal(size=(B, H, L, N)) + 1j * rng.normal(size=(B, H, L, N))
    h = rng.normal(size=(B, H, L, N)) + 1j * rng.normal(size=(B, H, L, N))
    ks = np.array([[[0, 1, 0, 0, 1, 0]], [[1, 1, 0, 0, 0, 1]]])   # entry 2 never selected
    hprev = np.concatenate([np.zeros((B, H, 1, N)), h[:, :, :-1]], axis=2)
    M = rng.normal(size=(H, K, N, N))

    def f(MM):
        S = _test_softmax(MM, T, -2)   # column-wise (softmax over rows i of each column j)
        tot = 0.0
        for b in range(B):
            for t in range(L):
                v = S[0, ks[b, 0, t]] @ (D[b, 0, t] * hprev[b, 0, t])
                tot += float(np.real(np.vdot(lam[b, 0, t], v)))
        return tot

    got = O.dictionary_grad(M, O.dictionary_outer(ks, lam, D, h, K), T)
    eps = 1e-6
    fd = np.zeros_like(M)
    for idx in itertools.product(*(range(n) for n in M.shape)):
        Mp, Mm = M.copy(), M.copy()
        Mp[idx] += eps
        Mm[idx] -= eps
        fd[idx] = (f(Mp) - f(Mm)) / (2 * eps)
    assert np.max(np.abs(got - fd)) <= 1e-7 * max(1.0, np.max(np.abs(fd)))
    assert np.allclose(got.sum(axis=-2), 0.0, atol=1e-12)   # every column sums to zero
    assert np.all(got[0, 2] == 0.0)                           # an unselected entry gets no gradient


# ---------------------------------------------------------------------------
# NEXT-2: D_t generator (SPEC.md:367 form; reading R30)
def test_diag_generator_special_cases():
    rng = np.random.default_rng(81)
    B, H, L, N, d = 2, 2, 5, 6, 4
    x = rng.normal(size=(B, L, d))
    Wm, Wp = rng.normal(size=(H, N, d)), rng.normal(size=(H, N, d))
    beta = rng.normal(size=(H, N))
    # zero weights: D = sigmoid(bias) exactly (real, in (0, 1)); sigmoid(0) = 1/2
    D0 = O.diag_generator(x, np.zeros_like(Wm), np.zeros_like(Wp), beta)
    assert np.allclose(D0.imag, 0.0) and np.allclose(D0.real, np.broadcast_to((1 / (1 + np.exp(-beta)))[None, :, None, :], D0.shape))
    assert np.allclose(O.diag_generator(x, np.zeros_like(Wm)), 0.5)
    # |D| < 1 always (the stability bound of SURVEY §8(d)); real mode = the magnitude of complex mode
    D = O.diag_generator(x, Wm, Wp, beta)
    assert np.all(np.abs(D) < 1.0)
    assert np.allclose(np.abs(D), O.diag_generator(x, Wm, None, beta).real)
    # doubling the phase weights squares the unit phase: D2 = |D| (D / |D|)^2
    D2 = O.diag_generator(x, Wm, 2 * Wp, beta)
    assert np.allclose(D2, np.abs(D) * (D / np.abs(D)) ** 2)
    # the phase weights act linearly on x: flipping x's sign conjugates the phase
    Dn = O.diag_generator(-x, np.zeros_like(Wm), Wp, np.zeros((H, N)))
    Dp = O.diag_generator(x, np.zeros_like(Wm), Wp, np.zeros((H, N)))
    assert np.allclose(Dn, np.conj(Dp))


def test_diag_generator_one_hot_tokens_pick_a_weight_column():
    """A one-hot token x_t = e_m reduces the generator to column m of the weights:
    D[b,h,t,n] = sigmoid(W_mag[h,n,m] + bias[h,n]) * exp(i W_phase[h,n,m]) (SPEC.md:367 form,
    PAPER.md:133, :211; reading R30).  Chosen phase weights pin the phase coefficient to exactly 1
    (pi/2 -> i, pi -> -1, 1 rad -> cos 1 + i sin 1) and the contraction index to d."""
    H, N, d = 2, 3, 4
    L = d
    x = np.eye(d)[None]                                   # token t is e_t (B = 1, L = d)
    Wm = np.arange(H * N * d, dtype=np.float64).reshape(H, N, d) / 10.0 - 1.0
    Wp = np.zeros((H, N, d))
    Wp[0, 0, :] = [np.pi / 2, np.pi, 1.0, -np.pi / 3]
    Wp[1, 2, :] = [0.25, -0.5, 2.0, 3.0]
    beta = np.array([[0.5, -0.25, 0.0], [1.0, 0.0, -2.0]])
    D = O.diag_generator(x, Wm, Wp, beta)
    for h in range(H):
        for n in range(N):
            for t in range(L):
                mag = 1.0 / (1.0 + math.exp(-(Wm[h, n, t] + beta[h, n])))
                want = complex(mag * math.cos(Wp[h, n, t]), mag * math.sin(Wp[h, n, t]))
                assert abs(D[0, h, t, n] - want) <= 1e-15
    mag00 = 1.0 / (1.0 + math.exp(-(Wm[0, 0, 0] + beta[0, 0])))
    assert abs(D[0, 0, 0, 0] - 1j * mag00) <= 1e-15          # phase pi/2: purely imaginary
    mag01 = 1.0 / (1.0 + math.exp(-(Wm[0, 0, 1] + beta[0, 0])))
    assert abs(D[0, 0, 1, 0] + mag01) <= 1e-15               # phase pi: negative real


# ---------------------------------------------------------------------------
# NEXT-3: PD-SSM soft generator (Eqs. 2-4)
def test_soft_generator_reduces_to_the_hard_path():
    rng = np.random.default_rng(91)
    B, H, L, N, K = 2, 2, 7, 6, 4
    M = rng.normal(size=(H, K, N, N))
    z = rng.normal(size=(B, H, L, K))
    # a (numerically) one-hot softmax selects one entry: Eq. 4 of M_{k*} = the Flash path (Eqs. 5-8)
    P_soft = O.soft_generator_P(z * 1e4, M)
    P_hard = O.gather_P(O.sparsify(M), O.argmax_smallest(z, axis=-1))
    assert np.array_equal(P_soft, P_hard)
    # K = 1: every step is the sparsified single matrix; identical entries: s does not matter
    P1 = O.soft_generator_P(z[..., :1], M[:, :1])
    assert np.array_equal(P1, np.broadcast_to(O.sparsify(M[:, :1])[:, 0][None, :, None, :], P1.shape))
    Msame = np.repeat(M[:, :1], K, axis=1)
    assert np.array_equal(O.soft_generator_P(z, Msame), np.broadcast_to(O.sparsify(M[:, :1])[:, 0][None, :, None, :], P1.shape))
    # a genuine mixture differs from the hard path somewhere (the relaxation is not the selection)
    assert not np.array_equal(O.soft_generator_P(z, M), O.gather_P(O.sparsify(M), O.argmax_smallest(z, axis=-1)))
