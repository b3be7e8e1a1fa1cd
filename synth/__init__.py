"""Seeded synthetic input generators shared by the oracle tests, the GPU
parity tests and bench.py.

This module holds NONE of the method's arithmetic (no selection, no scan, no
argmax): it only draws random inputs with the shapes and distributions of the
paper's workloads (recipe in DESIGN.md "Synthetic inputs").
Random numbers the method itself would draw are not needed (the method is
deterministic).

Every tensor gets its own child stream of ``numpy.random.SeedSequence(seed)``
(spawn order: M, S, x, D, b, h0, dh, kstar, dict), so a tensor's values do not
depend on which other tensors were requested.
"""
from __future__ import annotations

import numpy as np

_STREAMS = ["M", "S", "x", "D", "b", "h0", "dh", "kstar", "dict", "C", "Bw", "Dk"]

# BASELINE.json configs (SURVEY §8(d) "Per-config workloads")
CONFIGS = {
    1: dict(name="tiny", B=1, H=1, L=64, N=8, K=4, c=2, d_in=16, tau=16),
    2: dict(name="fig1", B=16, H=8, L=2048, N=128, K=32, c=2, d_in=1024, tau=0),
    3: dict(name="long_ts", B=4, H=8, L=17984, N=128, K=32, c=1, d_in=6, tau=0),
    4: dict(name="hybrid_llm", B=32, H=32, L=4096, N=64, K=48, c=1, d_in=2048, tau=0),
    5: dict(name="s5", B=4, H=4, L=65536, N=64, K=16, c=1, d_in=16, tau=0),
}


def _rng(seed, stream):
    ss = np.random.SeedSequence(seed)
    child = ss.spawn(len(_STREAMS))[_STREAMS.index(stream)]
    return np.random.Generator(np.random.PCG64(child))


def round_bf16(a):
    """Round float32 values to the nearest bfloat16 (ties to even), returned as
    float32 holding bf16-representable values (reading R16: the oracle reads
    back the rounded values)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def to_bf16_bits(a):
    """float32 (bf16-representable) -> uint16 bf16 bit patterns."""
    a = round_bf16(a)
    return (a.view(np.uint32) >> 16).astype(np.uint16)


def dictionary(H, K, N, seed):
    """Dense dictionary M[H][K][N][N] ~ U(-1/sqrt(N), 1/sqrt(N))."""
    r = _rng(seed, "M")
    lim = 1.0 / np.sqrt(N)
    return r.uniform(-lim, lim, size=(H, K, N, N)).astype(np.float32)


def random_maps(H, K, N, seed):
    """dict_idx[H][K][N] uniform random maps: the distribution of the column
    argmax of an iid continuous matrix (each column's argmax is uniform and
    independent), drawn directly so no argmax is computed here."""
    r = _rng(seed, "dict")
    return r.integers(0, N, size=(H, K, N)).astype(np.uint16)


def selector(H, K, d_in, seed, integer=False, tie_dense=False):
    """S[H][K][d_in] ~ U(+-1/sqrt(d_in)); integer=True: ints in [-8, 8];
    tie_dense: values in {-1,0,1} (reading R18)."""
    r = _rng(seed, "S")
    if tie_dense:
        return r.integers(-1, 2, size=(H, K, d_in)).astype(np.float32)
    if integer:
        return r.integers(-8, 9, size=(H, K, d_in)).astype(np.float32)
    lim = 1.0 / np.sqrt(d_in)
    return r.uniform(-lim, lim, size=(H, K, d_in)).astype(np.float32)


def tokens_x(B, L, d_in, seed, integer=False, tie_dense=False, walk=False):
    """x[B][L][d_in] ~ N(0,1); integer: ints in [-8,8]; walk: cumsum of
    N(0, 0.1) per channel (EigenWorms-like, config 3)."""
    r = _rng(seed, "x")
    if tie_dense:
        return r.integers(-1, 2, size=(B, L, d_in)).astype(np.float32)
    if integer:
        return r.integers(-8, 9, size=(B, L, d_in)).astype(np.float32)
    if walk:
        return np.cumsum(r.normal(0.0, 0.1, size=(B, L, d_in)), axis=1).astype(np.float32)
    return r.standard_normal(size=(B, L, d_in), dtype=np.float32)


def kstar(B, H, L, K, seed, sticky=0.0):
    """k*[B][H][L] uint8 drawn uniformly; sticky>0 repeats the previous entry
    with that probability (temporally persistent selections, config 3)."""
    r = _rng(seed, "kstar")
    k = r.integers(0, K, size=(B, H, L)).astype(np.uint8)
    if sticky > 0:
        keep = r.random(size=(B, H, L)) < sticky
        for t in range(1, L):
            k[:, :, t] = np.where(keep[:, :, t], k[:, :, t - 1], k[:, :, t])
    return k


def diag(shape_lead, N, c, seed, stream="D"):
    """Diagonal planes [*shape_lead, c, N]: |D| = sigmoid(a), a ~ N(2,1); complex
    phase theta ~ U[-pi, pi).  Stable: |D| < 1."""
    r = _rng(seed, stream)
    a = r.normal(2.0, 1.0, size=tuple(shape_lead) + (N,))
    mag = 1.0 / (1.0 + np.exp(-a))
    if c == 1:
        return mag[..., None, :].astype(np.float32)
    th = r.uniform(-np.pi, np.pi, size=tuple(shape_lead) + (N,))
    return np.stack([mag * np.cos(th), mag * np.sin(th)], axis=-2).astype(np.float32)


def normal_planes(shape_lead, N, c, seed, stream):
    r = _rng(seed, stream)
    return r.standard_normal(size=tuple(shape_lead) + (c, N), dtype=np.float32)


def scan_inputs(B, H, L, N, K, c, seed, h0=False, per_dict=False, sticky=0.0, dh=False, bf16=False):
    """Scan-level inputs: dict_idx, kstar, diag (PER_STEP
    [B][H][L][c][N] or PER_DICT [H][K][c][N]), bias b [B][H][L][c][N], optional
    h0 [B][H][c][N] and dh [B][H][L][c][N].  float32 (bf16-rounded if bf16)."""
    out = dict(dict_idx=random_maps(H, K, N, seed), kstar=kstar(B, H, L, K, seed, sticky))
    if per_dict:
        out["diag"] = diag((H, K), N, c, seed, "Dk")
    else:
        out["diag"] = diag((B, H, L), N, c, seed, "D")
    out["bias"] = normal_planes((B, H, L), N, c, seed, "b")
    if h0:
        out["h0"] = normal_planes((B, H), N, c, seed, "h0")
    if dh:
        out["dh"] = normal_planes((B, H, L), N, c, seed, "dh")
    if bf16:
        for k in ("diag", "bias", "dh"):
            if k in out:
                out[k] = round_bf16(out[k])
    return out


def _rng_row(seed, stream, b):
    """Stream of batch row b of tensor `stream`: rows are independent of each other, so any
    contiguous block of a global batch can be generated alone (bench.py: inputs are generated
    globally and each rank draws only its own rows)."""
    ss = np.random.SeedSequence(seed, spawn_key=(_STREAMS.index(stream), int(b)))
    return np.random.Generator(np.random.PCG64(ss))


def scan_inputs_rows(B, H, L, N, K, c, seed, rows=None, h0=False, per_dict=False, sticky=0.0, dh=False,
                     bf16=False):
    """scan_inputs of a global batch of B rows, generated row by row: `rows` = (b0, b1) returns
    only rows b0..b1-1 (the same values those rows have in the full batch).  Same distributions
    as scan_inputs; the dictionary is global."""
    b0, b1 = (0, B) if rows is None else rows
    n = b1 - b0
    out = dict(dict_idx=random_maps(H, K, N, seed))
    ks = np.empty((n, H, L), np.uint8)
    bias = np.empty((n, H, L, c, N), np.float32)
    D = None if per_dict else np.empty((n, H, L, c, N), np.float32)
    dhv = np.empty((n, H, L, c, N), np.float32) if dh else None
    h0v = np.empty((n, H, c, N), np.float32) if h0 else None
    for i, b in enumerate(range(b0, b1)):
        r = _rng_row(seed, "kstar", b)
        k = r.integers(0, K, size=(H, L)).astype(np.uint8)
        if sticky > 0:
            keep = r.random(size=(H, L)) < sticky
            for t in range(1, L):
                k[:, t] = np.where(keep[:, t], k[:, t - 1], k[:, t])
        ks[i] = k
        if D is not None:
            r = _rng_row(seed, "D", b)
            a = r.normal(2.0, 1.0, size=(H, L, N))
            mag = 1.0 / (1.0 + np.exp(-a))
            if c == 1:
                D[i, :, :, 0] = mag
            else:
                th = r.uniform(-np.pi, np.pi, size=(H, L, N))
                D[i, :, :, 0] = mag * np.cos(th)
                D[i, :, :, 1] = mag * np.sin(th)
        bias[i] = _rng_row(seed, "b", b).standard_normal(size=(H, L, c, N), dtype=np.float32)
        if dhv is not None:
            dhv[i] = _rng_row(seed, "dh", b).standard_normal(size=(H, L, c, N), dtype=np.float32)
        if h0v is not None:
            h0v[i] = _rng_row(seed, "h0", b).standard_normal(size=(H, c, N), dtype=np.float32)
    out["kstar"] = ks
    out["diag"] = diag((H, K), N, c, seed, "Dk") if per_dict else D
    out["bias"] = bias
    if dhv is not None:
        out["dh"] = dhv
    if h0v is not None:
        out["h0"] = h0v
    if bf16:
        for k in ("diag", "bias", "dh"):
            if k in out and not (k == "diag" and per_dict):
                out[k] = round_bf16(out[k])
    return out


def projection_B(H, c, N, d_in, seed):
    """Bw[H][c][N][d_in] ~ U(+-1/sqrt(d_in)) (plane 0 real part, 1 imaginary)."""
    r = _rng(seed, "Bw")
    lim = 1.0 / np.sqrt(d_in)
    return r.uniform(-lim, lim, size=(H, c, N, d_in)).astype(np.float32)


def readout_C(H, P, N, c, seed):
    """C[H][c][P][N] ~ U(+-1/sqrt(N))."""
    r = _rng(seed, "C")
    lim = 1.0 / np.sqrt(N)
    return r.uniform(-lim, lim, size=(H, c, P, N)).astype(np.float32)


def s5_dictionary(N=64, K=16, seed=5000):
    """Config-5 dictionary: K elements of S_5 (including the transposition
    (0 1) and the 5-cycle (0 1 2 3 4), which generate S_5), each acting on
    floor(N/5) disjoint 5-point blocks relabelled by a fixed random bijection;
    the N mod 5 leftover points are fixed.  Returns (dict_idx [K][N] uint16,
    perms5 [K][5] image lists, blocks list of 5-point index arrays)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    perms = [np.array([1, 0, 2, 3, 4]), np.array([1, 2, 3, 4, 0])]
    seen = {tuple(p) for p in perms}
    while len(perms) < K:
        p = rng.permutation(5)
        if tuple(p) not in seen:
            seen.add(tuple(p))
            perms.append(p)
    order = rng.permutation(N)
    blocks = [order[5 * i:5 * i + 5] for i in range(N // 5)]
    dict_idx = np.tile(np.arange(N), (K, 1))
    for k, p in enumerate(perms):
        for blk in blocks:
            for a in range(5):
                dict_idx[k, blk[a]] = blk[p[a]]
    return dict_idx.astype(np.uint16), np.stack(perms), blocks
