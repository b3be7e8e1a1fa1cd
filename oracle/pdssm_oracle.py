"""Float64 sequential oracle for the Flash PD-SSM hot path.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``): never imported by the
product package.  Plain NumPy, float64 / complex128, no blocking or fusion
beyond what the cited passage states.

Notation:  x_t input token, h_t hidden state (N per
head), P_t index map (uint16[N]), D_t diagonal, b_t = B x_t drive, k*_t the
selected dictionary entry.  Complex tensors are handled here as complex128
arrays ``[..., N]``; the boundary format is split planes ``[..., c, N]``
(c=1 real, c=2 re/im) and is converted by ``planes_to_complex`` /
``complex_to_planes``.

Convention (reading R1, scatter / column-one-hot):
    A_t = P_t D_t  with  A_t[P_t[j], j] = D_t[j]
    (A_t h)[i] = sum_{j : P_t[j] = i} D_t[j] h[j]      (ascending j)
which is the matrix of PAPER.md:143 (column_hardmax -> one-hot column) and of
the Prop. 1 construction PAPER.md:854 (A(sigma) = sum_q enc(delta(q,sigma)) enc(q)^T).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "planes_to_complex", "complex_to_planes",
    "sparsify", "selector_logits", "argmax_smallest", "select", "gather_P",
    "gather_D_per_dict", "project_b",
    "pd_apply", "pd_apply_transpose", "pd_compose",
    "scan_forward", "readout", "readout_adjoint",
    "prefix_maps", "chunk_bounds", "chunk_aggregates", "chunk_carries",
    "exclusive_prefix_maps", "scan_chunked",
    "scan_backward", "scan_backward_chunked",
    "segment_summary", "compose_summaries",
    "softmax_T", "selector_grad", "dictionary_outer", "dictionary_grad",
    "diag_generator", "soft_generator_P",
]


# ----------------------------------------------------------------------------
# representation helpers (no method arithmetic)
# ----------------------------------------------------------------------------
def planes_to_complex(a):
    """[..., c, N] real planes (c=1 real, c=2 re/im) -> complex128 [..., N]."""
    a = np.asarray(a, dtype=np.float64)
    if a.shape[-2] == 1:
        return a[..., 0, :].astype(np.complex128)
    return a[..., 0, :] + 1j * a[..., 1, :]


def complex_to_planes(z, c):
    """complex128 [..., N] -> float64 [..., c, N]."""
    z = np.asarray(z)
    if c == 1:
        return np.real(z)[..., None, :].astype(np.float64)
    return np.stack([np.real(z), np.imag(z)], axis=-2).astype(np.float64)


# ----------------------------------------------------------------------------
# a1: dictionary sparsification  (Eq. 5; App. E.2.1)
# ----------------------------------------------------------------------------
def sparsify(M):
    """dict_idx[h,k,j] = argmax_i M[h,k,i,j], ties -> smallest i (reading R7).

    ``M`` is the dense dictionary [H][K][N][N] (row i, column j)
    "M_k^sparse[j] = argmax(M_k[:,j])".  NaN raises.
    """
    M = np.asarray(M, dtype=np.float64)
    if np.isnan(M).any():
        raise ValueError("sparsify: NaN in dictionary")
    H, K, N, N2 = M.shape
    assert N == N2
    out = np.zeros((H, K, N), dtype=np.uint16)
    for h in range(H):
        for k in range(K):
            # np.argmax returns the first (smallest) index among equal maxima
            out[h, k] = np.argmax(M[h, k], axis=0)
    return out


# ----------------------------------------------------------------------------
# a2/a3: selector logits and hard selection (Eqs. 6-7)
# ----------------------------------------------------------------------------
def selector_logits(x, S):
    """logits[b,h,t,k] = sum_d S[h,k,d] x[b,t,d]   (Eq. 6)."""
    x = np.asarray(x, dtype=np.float64)
    S = np.asarray(S, dtype=np.float64)
    return np.einsum("hkd,btd->bhtk", S, x)


def argmax_smallest(v, axis=-1):
    """argmax with ties -> smallest index; NaN treated as -inf (reading R8)."""
    v = np.asarray(v, dtype=np.float64)
    v = np.where(np.isnan(v), -np.inf, v)
    return np.argmax(v, axis=axis)


def select(x, S):
    """k*[b,h,t] = argmax_k (S x_t)_k  (Eq. 7; 0-based, R6)."""
    logits = selector_logits(x, S)
    return argmax_smallest(logits, axis=-1).astype(np.uint8), logits


def gather_P(dict_idx, kstar):
    """P[b,h,t,:] = dict_idx[h, k*[b,h,t], :]   (Eq. 8)."""
    dict_idx = np.asarray(dict_idx)
    kstar = np.asarray(kstar).astype(np.int64)
    B, H, L = kstar.shape
    N = dict_idx.shape[-1]
    P = np.zeros((B, H, L, N), dtype=np.uint16)
    for h in range(H):
        P[:, h] = dict_idx[h][kstar[:, h]]
    return P


def gather_D_per_dict(Dk, kstar):
    """PER_DICT diagonal: D_t = D_k[h, k*]  (reading R3; complex128 [H][K][N])."""
    Dk = np.asarray(Dk)
    kstar = np.asarray(kstar).astype(np.int64)
    B, H, L = kstar.shape
    out = np.zeros((B, H, L, Dk.shape[-1]), dtype=Dk.dtype)
    for h in range(H):
        out[:, h] = Dk[h][kstar[:, h]]
    return out


def project_b(x, Bw):
    """b_t = B x_t per head  (Eq. 1 B(u_t)u_t with static B).

    x [B][L][d_in] real, Bw complex128 [H][N][d_in] -> complex128 [B][H][L][N].
    """
    return np.einsum("hnd,btd->bhtn", np.asarray(Bw), np.asarray(x, dtype=np.float64))


# ----------------------------------------------------------------------------
# PD algebra (scatter convention R1)
# ----------------------------------------------------------------------------
def pd_apply(P, D, h):
    """(P D) h : out[P[j]] += D[j] h[j] for j ascending."""
    out = np.zeros_like(np.asarray(h, dtype=np.complex128))
    for j in range(len(P)):
        out[P[j]] += D[j] * h[j]
    return out


def pd_apply_transpose(P, D, g):
    """(P D)^T g under the real-linear split inner product (reading R13):
    out[j] = conj(D[j]) g[P[j]]."""
    g = np.asarray(g, dtype=np.complex128)
    return np.conj(np.asarray(D)) * g[np.asarray(P, dtype=np.int64)]


def pd_compose(P2, D2, P1, D1):
    """(P2 D2)(P1 D1) = (pi, d) with pi[j] = P2[P1[j]], d[j] = D2[P1[j]] D1[j]
    (App. E.2 accumulator update)."""
    P1 = np.asarray(P1, dtype=np.int64)
    P2 = np.asarray(P2, dtype=np.int64)
    return P2[P1].astype(np.uint16), np.asarray(D2)[P1] * np.asarray(D1)


# ----------------------------------------------------------------------------
# a6-a8: forward recurrence, Eq. 1, scatter form
# ----------------------------------------------------------------------------
def scan_forward(P, D, b, h0=None):
    """h_t = P_t D_t h_{t-1} + b_t, t = 0..L-1, h_{-1} = h0 (or 0; reading R5).

    P [B][H][L][N] ints, D, b complex128 [B][H][L][N].  Returns h complex128
    [B][H][L][N].  Collisions are summed in ascending j (reading R17), then b
    is added (SURVEY O5 order).
    """
    P = np.asarray(P, dtype=np.int64)
    D = np.asarray(D, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    B, H, L, N = P.shape
    h = np.zeros((B, H, L, N), dtype=np.complex128)
    prev = np.zeros((B, H, N), dtype=np.complex128) if h0 is None else np.asarray(h0, np.complex128).copy()
    for bb in range(B):
        for hh in range(H):
            hp = prev[bb, hh]
            for t in range(L):
                new = np.zeros(N, dtype=np.complex128)
                # np.add.at is unbuffered and processes j in ascending order
                np.add.at(new, P[bb, hh, t], D[bb, hh, t] * hp)
                new = new + b[bb, hh, t]
                h[bb, hh, t] = new
                hp = new
    return h


def readout(h, C):
    """y_t = Re(C_h h_t)  (Eq. 1 y_t = C x_t, psi = Re; skip
    term excluded, reading R4).  h complex [B][H][L][N], C complex [H][P][N]
    -> y float64 [B][L][H][P]."""
    y = np.einsum("hpn,bhtn->bthp", np.asarray(C, np.complex128), np.asarray(h, np.complex128))
    return np.real(y)


def readout_adjoint(dy, C):
    """Direct state gradient of y = Re(C h):  e_t = conj(C)^T dy_t (packed
    re + i im, reading R13).  dy [B][L][H][P] -> complex [B][H][L][N]."""
    return np.einsum("hpn,bthp->bhtn", np.conj(np.asarray(C, np.complex128)), np.asarray(dy, np.float64))


# ----------------------------------------------------------------------------
# O7: composed maps, chunk aggregates, carries (Alg. 1)
# ----------------------------------------------------------------------------
def prefix_maps(P, D):
    """Pi_t[j] = P_t[Pi_{t-1}[j]], rho_t[j] = D_t[Pi_{t-1}[j]] rho_{t-1}[j],
    Pi_{-1} = id, rho_{-1} = 1.  Returns (Pi, rho) with
    shapes [B][H][L][N]."""
    P = np.asarray(P, dtype=np.int64)
    D = np.asarray(D, dtype=np.complex128)
    B, H, L, N = P.shape
    Pi = np.zeros((B, H, L, N), dtype=np.int64)
    rho = np.zeros((B, H, L, N), dtype=np.complex128)
    for bb in range(B):
        for hh in range(H):
            pi = np.arange(N)
            r = np.ones(N, dtype=np.complex128)
            for t in range(L):
                r = D[bb, hh, t][pi] * r
                pi = P[bb, hh, t][pi]
                Pi[bb, hh, t] = pi
                rho[bb, hh, t] = r
    return Pi, rho


def chunk_bounds(L, tau):
    """Chunks [c*tau, min((c+1)*tau, L)), C = ceil(L/tau) (reading R11)."""
    C = -(-L // tau)
    return [(c * tau, min((c + 1) * tau, L)) for c in range(C)]


def chunk_aggregates(P, D, b, tau):
    """Phase A of Alg. 1 (Kernel A PAPER.md:1020-1046) in
    scatter form: per chunk, from identity (pi=j, d=1, beta=0), for each step
    pi <- P_t[pi], d <- D_t[pi_old] d, beta <- A_t beta + b_t.
    Returns (pi_bar [B][H][C][N] int, d_bar, beta_bar complex [B][H][C][N])."""
    P = np.asarray(P, dtype=np.int64)
    D = np.asarray(D, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    B, H, L, N = P.shape
    bounds = chunk_bounds(L, tau)
    C = len(bounds)
    pi_bar = np.zeros((B, H, C, N), dtype=np.int64)
    d_bar = np.zeros((B, H, C, N), dtype=np.complex128)
    beta_bar = np.zeros((B, H, C, N), dtype=np.complex128)
    for bb in range(B):
        for hh in range(H):
            for c, (s, e) in enumerate(bounds):
                pi = np.arange(N)
                d = np.ones(N, dtype=np.complex128)
                beta = np.zeros(N, dtype=np.complex128)
                for t in range(s, e):
                    d = D[bb, hh, t][pi] * d
                    pi = P[bb, hh, t][pi]
                    nb = np.zeros(N, dtype=np.complex128)
                    np.add.at(nb, P[bb, hh, t], D[bb, hh, t] * beta)
                    beta = nb + b[bb, hh, t]
                pi_bar[bb, hh, c] = pi
                d_bar[bb, hh, c] = d
                beta_bar[bb, hh, c] = beta
    return pi_bar, d_bar, beta_bar


def chunk_carries(pi_bar, d_bar, beta_bar, h0=None):
    """Phase B (Kernel B :1069-1081): carry_0 = h0 (R5),
    carry_{c+1} = Abar_c carry_c + beta_bar_c with Abar_c = (pi_bar_c, d_bar_c)
    applied as a scatter.  Returns carries [B][H][C][N] (state entering chunk c)
    and the final state [B][H][N]."""
    pi_bar = np.asarray(pi_bar, dtype=np.int64)
    B, H, C, N = pi_bar.shape
    carries = np.zeros((B, H, C, N), dtype=np.complex128)
    final = np.zeros((B, H, N), dtype=np.complex128)
    for bb in range(B):
        for hh in range(H):
            cur = np.zeros(N, np.complex128) if h0 is None else np.asarray(h0, np.complex128)[bb, hh].copy()
            for c in range(C):
                carries[bb, hh, c] = cur
                nxt = np.zeros(N, dtype=np.complex128)
                np.add.at(nxt, pi_bar[bb, hh, c], d_bar[bb, hh, c] * cur)
                cur = nxt + beta_bar[bb, hh, c]
            final[bb, hh] = cur
    return carries, final


def exclusive_prefix_maps(pi_bar):
    """maps[c] = Pi before chunk c (maps[0] = id), maps[C] = final map Pi_{L-1}
    (reading R12; composition by gather PAPER.md:1040).  [B][H][C+1][N]."""
    pi_bar = np.asarray(pi_bar, dtype=np.int64)
    B, H, C, N = pi_bar.shape
    maps = np.zeros((B, H, C + 1, N), dtype=np.int64)
    for bb in range(B):
        for hh in range(H):
            m = np.arange(N)
            for c in range(C):
                maps[bb, hh, c] = m
                m = pi_bar[bb, hh, c][m]
            maps[bb, hh, C] = m
    return maps


def scan_chunked(P, D, b, tau, h0=None):
    """Alg. 1 three-phase recurrence with the replay form of Phase C (reading
    R10).  Returns dict with h, pi_bar, d_bar, beta_bar,
    carries, maps, final."""
    P = np.asarray(P, dtype=np.int64)
    D = np.asarray(D, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    B, H, L, N = P.shape
    pi_bar, d_bar, beta_bar = chunk_aggregates(P, D, b, tau)
    carries, final = chunk_carries(pi_bar, d_bar, beta_bar, h0)
    h = np.zeros((B, H, L, N), dtype=np.complex128)
    for bb in range(B):
        for hh in range(H):
            for c, (s, e) in enumerate(chunk_bounds(L, tau)):
                cur = carries[bb, hh, c]
                for t in range(s, e):
                    nxt = np.zeros(N, dtype=np.complex128)
                    np.add.at(nxt, P[bb, hh, t], D[bb, hh, t] * cur)
                    cur = nxt + b[bb, hh, t]
                    h[bb, hh, t] = cur
    return dict(h=h, pi_bar=pi_bar, d_bar=d_bar, beta_bar=beta_bar,
                carries=carries, maps=exclusive_prefix_maps(pi_bar), final=final)


# ----------------------------------------------------------------------------
# a9: backward (reverse, transposed) scan  (App. C; Prop. 2 :210-222)
# ----------------------------------------------------------------------------
def scan_backward(P, D, h, e, h0=None):
    """Adjoint of the forward recurrence, real-linear split gradients packed as
    G = dl/dRe + i dl/dIm (reading R13):

        lambda_{L-1} = e_{L-1}
        lambda_{t-1} = e_{t-1} + A_t^T lambda_t,  (A_t^T mu)[j] = conj(D_t[j]) mu[P_t[j]]
        db_t   = lambda_t
        dD_t[j] = conj(h_{t-1}[j]) lambda_t[P_t[j]]          (h_{-1} = h0)
        g_t    = sum_j Re(conj(lambda_t[P_t[j]]) D_t[j] h_{t-1}[j])
        dh0    = A_0^T lambda_0

    ``e`` is the direct state gradient dl/dh_t (dh, or readout_adjoint(dy)).
    g_t is dl/dP_t ("dl/dx_t (D_t x_{t-1})^T") contracted with P_t
    (reading R14).  Returns (db, dD, g, dh0)."""
    P = np.asarray(P, dtype=np.int64)
    D = np.asarray(D, dtype=np.complex128)
    h = np.asarray(h, dtype=np.complex128)
    e = np.asarray(e, dtype=np.complex128)
    B, H, L, N = P.shape
    db = np.zeros((B, H, L, N), dtype=np.complex128)
    dD = np.zeros((B, H, L, N), dtype=np.complex128)
    g = np.zeros((B, H, L), dtype=np.float64)
    dh0 = np.zeros((B, H, N), dtype=np.complex128)
    for bb in range(B):
        for hh in range(H):
            lam = e[bb, hh, L - 1].copy()
            for t in range(L - 1, -1, -1):
                if t > 0:
                    hprev = h[bb, hh, t - 1]
                elif h0 is not None:
                    hprev = np.asarray(h0, np.complex128)[bb, hh]
                else:
                    hprev = np.zeros(N, np.complex128)
                db[bb, hh, t] = lam
                lam_at_P = lam[P[bb, hh, t]]
                dD[bb, hh, t] = np.conj(hprev) * lam_at_P
                g[bb, hh, t] = np.sum(np.real(np.conj(lam_at_P) * D[bb, hh, t] * hprev))
                back = np.conj(D[bb, hh, t]) * lam_at_P
                if t > 0:
                    lam = e[bb, hh, t - 1] + back
                else:
                    dh0[bb, hh] = back
    return db, dD, g, dh0


def scan_backward_chunked(P, D, e, pi_bar, d_bar, tau):
    """Chunk-level backward quantities (transposed Alg. 1):
        lam_loc : reverse scan inside chunk c with zero incoming
        beta'_c = A_{s_c}^T lam_loc_{s_c}
        mu_{C-1} = 0, mu_{c-1} = beta'_c + Abar_c^T mu_c,
            (Abar_c^T mu)[j] = conj(d_bar_c[j]) mu[pi_bar_c[j]]   (forward aggregate reused)
        lambda_t (t in chunk c) = reverse scan from lambda_{e_c} = e_{e_c} + mu_c
        dh0 = beta'_0 + Abar_0^T mu_0
    Returns dict(lam [B][H][L][N], beta_p [B][H][C][N], mu [B][H][C][N], dh0)."""
    P = np.asarray(P, dtype=np.int64)
    D = np.asarray(D, dtype=np.complex128)
    e = np.asarray(e, dtype=np.complex128)
    pi_bar = np.asarray(pi_bar, dtype=np.int64)
    d_bar = np.asarray(d_bar, dtype=np.complex128)
    B, H, L, N = P.shape
    bounds = chunk_bounds(L, tau)
    C = len(bounds)
    beta_p = np.zeros((B, H, C, N), np.complex128)
    mu = np.zeros((B, H, C, N), np.complex128)
    lam_all = np.zeros((B, H, L, N), np.complex128)
    dh0 = np.zeros((B, H, N), np.complex128)
    for bb in range(B):
        for hh in range(H):
            # local reverse scans
            for c, (s, en) in enumerate(bounds):
                lam = e[bb, hh, en - 1].copy()
                for t in range(en - 1, s, -1):
                    lam = e[bb, hh, t - 1] + np.conj(D[bb, hh, t]) * lam[P[bb, hh, t]]
                beta_p[bb, hh, c] = np.conj(D[bb, hh, s]) * lam[P[bb, hh, s]]
            # reverse carries
            m = np.zeros(N, np.complex128)
            for c in range(C - 1, -1, -1):
                mu[bb, hh, c] = m
                m = beta_p[bb, hh, c] + np.conj(d_bar[bb, hh, c]) * m[pi_bar[bb, hh, c]]
            dh0[bb, hh] = m
            # replay
            for c, (s, en) in enumerate(bounds):
                lam = e[bb, hh, en - 1] + mu[bb, hh, c]
                lam_all[bb, hh, en - 1] = lam
                for t in range(en - 1, s, -1):
                    lam = e[bb, hh, t - 1] + np.conj(D[bb, hh, t]) * lam[P[bb, hh, t]]
                    lam_all[bb, hh, t - 1] = lam
    return dict(lam=lam_all, beta_p=beta_p, mu=mu, dh0=dh0)


# ----------------------------------------------------------------------------
# sequence parallelism: segment summaries (the chunk algebra with chunk = segment)
# ----------------------------------------------------------------------------
def segment_summary(P, D, b):
    """Summary (pi, d, beta) of one segment = its Phase-A aggregate with a single
    chunk spanning the segment ("the PD-SSM composition operator is
    associative")."""
    L = np.asarray(P).shape[2]
    pi, d, beta = chunk_aggregates(P, D, b, L)
    return pi[:, :, 0], d[:, :, 0], beta[:, :, 0]


def compose_summaries(pis, ds, betas, rank, h0=None):
    """carry into segment ``rank`` = S_{rank-1} o ... o S_0 applied to h0, and the
    prefix map Pi before the segment (composition order = rank order)."""
    B, H, N = np.asarray(pis[0]).shape
    cur = np.zeros((B, H, N), np.complex128) if h0 is None else np.asarray(h0, np.complex128).copy()
    m = np.tile(np.arange(N), (B, H, 1))
    for g in range(rank):
        nxt = np.zeros((B, H, N), np.complex128)
        for bb in range(B):
            for hh in range(H):
                np.add.at(nxt[bb, hh], np.asarray(pis[g], np.int64)[bb, hh], np.asarray(ds[g])[bb, hh] * cur[bb, hh])
                m[bb, hh] = np.asarray(pis[g], np.int64)[bb, hh][m[bb, hh]]
        cur = nxt + np.asarray(betas[g])
    return cur, m


# ----------------------------------------------------------------------------
# NEXT-1: Prop. 2 surrogate gradients (derivation App. C
# PAPER.md:814-841).  Slope-annealed straight-through estimation: each hardmax of
# the forward is a tempered softmax in the backward.
# ----------------------------------------------------------------------------
def softmax_T(z, T, axis=-1):
    """Tempered softmax softmax_T(z) = exp(z / T) / sum exp(z / T) along ``axis``
    ("softmax_tau ... the tempered softmax function")."""
    z = np.asarray(z, dtype=np.float64) / float(T)
    z = z - z.max(axis=axis, keepdims=True)
    ez = np.exp(z)
    return ez / ez.sum(axis=axis, keepdims=True)


def selector_grad(logits, kstar, g, T):
    """Selector surrogate gradient, Prop. 2 second expression (App. C
    Eq. grad_k):

        dl/dk(u_t) = (dl/dx_t (P_t D_t x_{t-1})^T) dsoftmax_T(k(u_t))/dk(u_t)

    The first factor, contracted with the activated entry only ("uses the activated
    forward state"), is the scalar g_t of scan_backward (reading R14):
    dl/dv_t = g_t e_{k*}.  Through the softmax Jacobian ds_j/dz_k = s_j (delta_jk - s_k) / T:

        dlogits[b,h,t,k] = g_t s_{k*} (delta_{k,k*} - s_k) / T,   s = softmax_T(logits[b,h,t,:])

    logits [B,H,L,K], kstar [B,H,L], g [B,H,L] -> [B,H,L,K] float64."""
    logits = np.asarray(logits, dtype=np.float64)
    K = logits.shape[-1]
    s = softmax_T(logits, T, axis=-1)
    ks = np.asarray(kstar, dtype=np.int64)[..., None]
    s_k = np.take_along_axis(s, ks, axis=-1)
    onehot = (np.arange(K) == ks).astype(np.float64)
    return np.asarray(g, dtype=np.float64)[..., None] * s_k * (onehot - s) / float(T)


def dictionary_outer(kstar, lam, D, h, K, h0=None):
    """Outer-product sums of Prop. 2's first expression before the softmax Jacobian
    (App. C: dl/dP_t = dl/dx_t (D_t x_{t-1})^T, summed over the
    steps t with k*(u_t) = k):

        G[h,k,i,j] = sum_{b,t : k*[b,h,t] = k} Re(conj(lambda_t[i]) (D_t h_{t-1})[j])

    (real-linear split gradient of a real matrix entry, reading R13; h_{-1} = h0).
    lam = db of scan_backward, D, h complex [B,H,L,N] (h the forward states) -> [H,K,N,N]."""
    lam = np.asarray(lam, dtype=np.complex128)
    D = np.asarray(D, dtype=np.complex128)
    h = np.asarray(h, dtype=np.complex128)
    B, H, L, N = lam.shape
    first = np.zeros((B, H, 1, N), np.complex128) if h0 is None else np.asarray(h0, np.complex128)[:, :, None, :]
    hprev = np.concatenate([first, h[:, :, :-1]], axis=2)
    w = D * hprev
    ks = np.asarray(kstar, dtype=np.int64)
    G = np.zeros((H, K, N, N), dtype=np.float64)
    for hh in range(H):
        for k in range(K):
            sel = ks[:, hh, :] == k                      # [B, L]
            lk = lam[:, hh][sel]                          # [n_k, N]
            wk = w[:, hh][sel]
            G[hh, k] = np.real(np.conj(lk).T @ wk)        # sum over the selected steps
    return G


def dictionary_grad(M, G, T):
    """Dictionary surrogate gradient, Prop. 2 first expression (App. C
    Eq. grad_M): the outer-product sum G_k pushed through the
    Jacobian of the tempered softmax of M_k, taken column-wise as the column hardmax
    it replaces (Eq. 5; column one-hot; reading A15):

        sigma_j = softmax_T(M_k[:, j]),   dM_k[:, j] = (diag(sigma_j) - sigma_j sigma_j^T) / T  G_k[:, j]

    M, G [H,K,N,N] -> [H,K,N,N] float64."""
    sig = softmax_T(M, T, axis=-2)                       # softmax over the rows i of column j
    G = np.asarray(G, dtype=np.float64)
    proj = (sig * G).sum(axis=-2, keepdims=True)         # sigma_j^T G[:, j]
    return sig * (G - proj) / float(T)


# ----------------------------------------------------------------------------
# NEXT-2: the input-dependent diagonal D_t = D(u_t) (form fixed by
# SPEC.md:367, reading R30): magnitude sigmoid(w^mag u_t + bias^mag) times phase exp(i w^phase u_t)
# ----------------------------------------------------------------------------
def diag_generator(x, W_mag, W_phase=None, bias_mag=None):
    """D[b,h,t,n] = sigmoid((W_mag[h] x_t)[n] + bias_mag[h,n]) * exp(i (W_phase[h] x_t)[n])
    (real mode, W_phase None: the magnitude alone).  x [B][L][d_in]; W_mag, W_phase [H][N][d_in];
    bias_mag [H][N] or None -> complex128 [B][H][L][N]."""
    x = np.asarray(x, dtype=np.float64)
    a = np.einsum("hnd,btd->bhtn", np.asarray(W_mag, np.float64), x)
    if bias_mag is not None:
        a = a + np.asarray(bias_mag, np.float64)[None, :, None, :]
    mag = 1.0 / (1.0 + np.exp(-a))
    if W_phase is None:
        return mag.astype(np.complex128)
    th = np.einsum("hnd,btd->bhtn", np.asarray(W_phase, np.float64), x)
    return mag * np.exp(1j * th)


# ----------------------------------------------------------------------------
# NEXT-3: the PD-SSM (soft) generator Flash PD-SSM replaces (Eqs. 2-4)
# ----------------------------------------------------------------------------
def soft_generator_P(logits, M):
    """P(u_t) of PD-SSM: s = softmax(S u_t) (Eq. 2), M(u_t) = sum_k s_k M_k (Eq. 3),
    P_{:,j} = column_hardmax(M_{:,j}(u_t)) (Eq. 4), as the index map of the one-hot column
    (smallest row on ties, reading R7).  Materialises the L N^2 mixture the paper names as the
    bottleneck.  logits [B,H,L,K] (= S u_t), M [H,K,N,N] -> int [B,H,L,N]."""
    s = softmax_T(logits, 1.0, axis=-1)
    mix = np.einsum("bhtk,hkij->bhtij", s, np.asarray(M, np.float64))
    return argmax_smallest(mix, axis=-2)
