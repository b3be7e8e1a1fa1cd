"""GPU parity of a5, the projection b_t = B x_t feeding the scan (Eq. 1,
PAPER.md:94-95, :970), through the C ABI, on the tensor-core path (tcgen05:
bf16 kind::f16, fp32 3xTF32) and the SIMT path, against oracle.project_b.
Tolerance: reading R19 (max abs error / max |oracle| <= 1e-4 fp32, 2e-2 bf16)."""
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
    if request.param == "generic":
        monkeypatch.setenv("PDSSM_PATH", "generic")
    else:
        monkeypatch.delenv("PDSSM_PATH", raising=False)
    return request.param


# (B, L, d_in, H, c, N): tensor-core shapes (ragged token tail, multi-tile columns)
# and SIMT-only shapes (c*N % 16 != 0, d_in row pitch not 16-byte aligned)
CASES = [(1, 64, 16, 1, 1, 16), (2, 130, 1024, 8, 2, 128), (1, 200, 2048, 4, 1, 64), (2, 33, 40, 3, 2, 5),
         (1, 50, 6, 2, 1, 32), (3, 129, 64, 2, 2, 64)]


@pytest.mark.parametrize("shape", CASES)
@pytest.mark.parametrize("bf16", [False, True])
def test_project_parity(P, path, shape, bf16):
    B, L, d_in, H, c, N = shape
    x = synth.tokens_x(B, L, d_in, seed=L + d_in)
    Bw = synth.projection_B(H, c, N, d_in, seed=L + d_in)
    if bf16:
        x, Bw = synth.round_bf16(x), synth.round_bf16(Bw)
    Bc = Bw[:, 0].astype(np.float64) + (1j * Bw[:, 1].astype(np.float64) if c == 2 else 0.0)
    ref = O.project_b(x.astype(np.float64), Bc)            # complex [B][H][L][N]
    ref_planes = np.stack([ref.real, ref.imag], axis=3)[:, :, :, :c]
    dt = torch.bfloat16 if bf16 else torch.float32
    xt = torch.from_numpy(x).cuda().to(dt)
    Bt = torch.from_numpy(Bw).cuda().to(dt)
    got = P.project(xt, Bt).float().cpu().numpy().astype(np.float64)
    assert got.shape == (B, H, L, c, N)
    tol = 2e-2 if bf16 else 1e-4
    err = np.max(np.abs(got - ref_planes)) / max(np.max(np.abs(ref_planes)), 1e-30)
    assert err <= tol, err


def test_project_integer_exact(P, path):
    """Integer-valued x, B (|.| <= 8): every product and partial sum is an exact fp32
    integer, so both paths must reproduce the oracle bit for bit."""
    B, L, d_in, H, c, N = 2, 160, 256, 2, 2, 32
    x = synth.tokens_x(B, L, d_in, seed=9, integer=True)
    Bw = np.rint(synth.projection_B(H, c, N, d_in, seed=9) * 8 * np.sqrt(d_in)).astype(np.float32)
    ref = O.project_b(x.astype(np.float64), Bw[:, 0].astype(np.float64) + 1j * Bw[:, 1].astype(np.float64))
    for dt in (torch.float32, torch.bfloat16):
        got = P.project(torch.from_numpy(x).cuda().to(dt), torch.from_numpy(Bw).cuda().to(dt))
        g = got.float().cpu().numpy().astype(np.float64)
        if dt == torch.bfloat16:   # bf16 output rounding of exact integers < 2^8 is exact only below 256
            ok = np.abs(ref.real) < 256
            assert np.array_equal(g[:, :, :, 0][ok], ref.real[ok])
        else:
            assert np.array_equal(g[:, :, :, 0], ref.real)
            assert np.array_equal(g[:, :, :, 1], ref.imag)


def test_project_validation(P):
    x = torch.zeros((1, 4, 8), device="cuda")
    Bw = torch.zeros((1, 1, 8, 8), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(TypeError):
        P.project(x, Bw)


@pytest.mark.parametrize("shape", [(2, 2, 300, 2, 64, 32), (1, 3, 129, 1, 32, 16), (2, 1, 70, 2, 16, 5),
                                   (1, 8, 256, 2, 128, 128), (2, 2, 700, 2, 128, 128), (1, 2, 384, 1, 128, 96)])
@pytest.mark.parametrize("bf16", [False, True])
@pytest.mark.parametrize("variant", ["", "PDSSM_READOUT_MT2", "PDSSM_READOUT_NARROW", "PDSSM_READOUT_ATM=0"])
def test_readout_standalone(P, path, shape, bf16, variant, monkeypatch):
    """a8 readout y_t = Re(C_h h_t) (Eq. 1) on given states, against oracle.readout."""
    if variant:   # the other tilings of the fp32 tensor-core readout (MT = 2 row tiles, 64-column tiles, A in smem)
        if bf16:
            pytest.skip("fp32 pre-split variants")
        name, _, val = variant.partition("=")
        monkeypatch.setenv(name, val or "1")
    B, H, L, c, N, Pp = shape
    rng = np.random.default_rng(L + N)
    h = rng.standard_normal((B, H, L, c, N)).astype(np.float32)
    if bf16:
        h = synth.round_bf16(h)
    Cw = synth.readout_C(H, Pp, N, c, seed=L)
    dt = torch.bfloat16 if bf16 else torch.float32
    y = P.readout(torch.from_numpy(h).cuda().to(dt), torch.from_numpy(Cw).cuda())
    hz = O.planes_to_complex(h)                              # [B][H][L][N]
    Cz = O.planes_to_complex(np.moveaxis(Cw, 1, -2))         # [H][P][N]
    ref = O.readout(hz, Cz)
    tol = 2e-2 if bf16 else 1e-4
    err = np.max(np.abs(y.float().cpu().numpy() - ref)) / np.max(np.abs(ref))
    assert err <= tol, err
