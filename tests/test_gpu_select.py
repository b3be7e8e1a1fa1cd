"""GPU parity of a1-a4 (sparsify, selector logits, hard selection, P gather)
through the C ABI.  Integer results bit-exact; float-data selections checked
with the margin rule of DESIGN.md reading R18."""
import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_19150_b200 as mod
    return mod


@pytest.fixture(params=["generic", "auto"])
def path(request, monkeypatch):
    """generic: SIMT logits + argmax kernel; auto: tcgen05 logits with the argmax (and the
    P gather) fused into the TMEM epilogue wherever the shape allows it."""
    if request.param == "generic":
        monkeypatch.setenv("PDSSM_PATH", "generic")
    else:
        monkeypatch.delenv("PDSSM_PATH", raising=False)
    return request.param


@pytest.mark.parametrize("H,K,N", [(1, 4, 8), (2, 3, 5), (8, 32, 128), (2, 5, 1000), (1, 1, 1)])
def test_sparsify_bit_exact(P, H, K, N):
    M = synth.dictionary(H, K, N, seed=N)
    if N >= 5:
        M[0, 0, :, 2] = 0.25                     # all-equal column -> 0
        M[0, -1, 1, 3] = M[0, -1, 4, 3] = 9.0     # tie -> 1
    got = P.sparsify(torch.from_numpy(M).cuda()).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, O.sparsify(M))


def test_sparsify_nan_reported(P):
    M = synth.dictionary(1, 2, 8, seed=1)
    M[0, 1, 3, 3] = np.nan
    P.check_device()
    P.sparsify(torch.from_numpy(M).cuda(), check_finite=True)
    with pytest.raises(P.PdssmError):
        P.check_device()


@pytest.mark.parametrize("shape", [(1, 64, 16, 1, 4, 8), (2, 33, 40, 3, 7, 5), (2, 130, 1024, 8, 32, 128),
                                   (1, 70, 2048, 4, 48, 64)])
@pytest.mark.parametrize("mode", ["integer", "tie_dense"])
@pytest.mark.parametrize("bf16", [False, True])
def test_select_integer_bit_exact(P, path, shape, mode, bf16):
    B, L, d_in, H, K, N = shape
    kw = {mode: True}
    x = synth.tokens_x(B, L, d_in, seed=L, **kw)
    S = synth.selector(H, K, d_in, seed=L, **kw)
    di = synth.random_maps(H, K, N, seed=L)
    dt = torch.bfloat16 if bf16 else torch.float32          # |values| <= 8: exact in bf16 / tf32 too
    k, Pm, lg = P.select(torch.from_numpy(x).cuda().to(dt), torch.from_numpy(S).cuda().to(dt),
                         torch.from_numpy(di.astype(np.int16)).cuda(), want_P=True, want_logits=True)
    k_ref, lg_ref = O.select(x, S)
    assert np.array_equal(lg.cpu().numpy().astype(np.float64), lg_ref)     # exact integers
    assert np.array_equal(k.cpu().numpy(), k_ref)
    assert np.array_equal(Pm.cpu().numpy().astype(np.int64), O.gather_P(di, k_ref).astype(np.int64))


@pytest.mark.parametrize("bf16", [False, True])
def test_select_float_margin_rule(P, path, bf16):
    """Reading R18 on float data at the config-2 layer shape (d_in 1024, H 8, K 32; 65536
    positions): every position whose float64 top-2 gap exceeds gamma matches bit for bit; the
    positions that do not match are counted and must be near-ties (gap <= gamma) and at most
    1e-4 of all positions."""
    B, L, d_in, H, K = 4, 2048, 1024, 8, 32
    x = synth.tokens_x(B, L, d_in, seed=5)
    S = synth.selector(H, K, d_in, seed=5)
    if bf16:
        x, S = synth.round_bf16(x), synth.round_bf16(S)
    xt = torch.from_numpy(x).cuda()
    St = torch.from_numpy(S).cuda()
    if bf16:
        xt, St = xt.to(torch.bfloat16), St.to(torch.bfloat16)
    k, _, lg = P.select(xt, St, want_logits=True)
    k = k.cpu().numpy()
    k_ref, lg_ref = O.select(x, S)
    # argmax stage bit-exact on the GPU's own logits
    assert np.array_equal(k, O.argmax_smallest(lg.cpu().numpy()))
    # margin rule: positions with a float64 top-2 gap above gamma must match
    srt = np.sort(lg_ref, axis=-1)
    gap = srt[..., -1] - srt[..., -2]
    absum = np.einsum("hkd,btd->bhtk", np.abs(S.astype(np.float64)), np.abs(x.astype(np.float64)))
    k1 = np.argsort(lg_ref, axis=-1)[..., -1:]
    k2 = np.argsort(lg_ref, axis=-1)[..., -2:-1]
    # u_in: 0 for bf16 inputs (products exact) and for the fp32 SIMT path; 2^-20 bounds the
    # 3xTF32 split of the tensor-core fp32 path (dropped lo*lo term + lo truncation)
    u_in = 2.0 ** -20 if (path == "auto" and not bf16) else 0.0
    gamma = (u_in + d_in * 2.0 ** -24) * (np.take_along_axis(absum, k1, -1)[..., 0] + np.take_along_axis(absum, k2, -1)[..., 0])
    sure = gap > gamma
    assert np.array_equal(k[sure], k_ref[sure])
    # near-ties (gap <= gamma): the GPU's pick must be within gamma of the exact maximum
    chosen = np.take_along_axis(lg_ref, k[..., None].astype(np.int64), -1)[..., 0]
    assert np.all(srt[..., -1][~sure] - chosen[~sure] <= gamma[~sure])
    # the mismatching positions are near-ties, and few: <= 1e-4 of all positions
    mismatch = k != k_ref
    assert not np.any(mismatch & sure)
    assert int(mismatch.sum()) <= 1e-4 * mismatch.size, (int(mismatch.sum()), int((~sure).sum()), mismatch.size)
    assert np.max(np.abs(lg.cpu().numpy() - lg_ref)) <= 1e-4 * np.max(np.abs(lg_ref))


@pytest.mark.parametrize("K", [32, 7])
def test_select_nan_never_wins(P, path, K):
    """Reading R8: a NaN logit never wins; a token whose logits are all NaN selects 0."""
    B, L, d_in, H = 1, 150, 64, 2
    x = synth.tokens_x(B, L, d_in, seed=3, integer=True)
    S = synth.selector(H, K, d_in, seed=3, integer=True)
    S[0, 3, 5] = np.nan                 # logit k=3 of head 0 is NaN at every token
    x[0, 7, :] = np.nan                 # token 7: every logit NaN
    k, _, _ = P.select(torch.from_numpy(x).cuda(), torch.from_numpy(S).cuda())
    k_ref, _ = O.select(x, S)
    assert np.array_equal(k.cpu().numpy(), k_ref)
    assert np.all(k.cpu().numpy()[0, :, 7] == 0)
