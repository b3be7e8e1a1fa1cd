"""CPU-only checks of the C-ABI library: it loads, exports every symbol the
header declares, and validates arguments synchronously (before any CUDA call,
so no GPU is needed)."""
import ctypes

import pytest

import paper_2605_19150_b200 as P


def dims(**kw):
    base = dict(B=2, H=3, L=100, N=16, K=4, c=2, dtype=P.F32, tau=0)
    base.update(kw)
    return P.make_dims(**base)


def test_all_header_symbols_exported():
    syms = P.header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(P.lib, s), s
    assert P.lib.pdssm_version().startswith(b"pdssm")


def test_status_strings():
    for code, name in P.STATUS.items():
        assert P.lib.pdssm_status_string(code).decode() == name


def test_sizes_and_default_chunk():
    d = dims(tau=7)
    assert P.default_chunk(d) == 7
    d = dims(tau=1000)          # tau > L is clamped to L
    assert P.default_chunk(d) == 100
    d = dims()
    tau = P.default_chunk(d)
    assert tau >= 1
    Cch = -(-100 // tau)
    assert P.lib.pdssm_chunk_state_bytes(ctypes.byref(d)) >= 6 * Cch * 16 * 2 + 3 * 6 * Cch * 2 * 16 * 4
    offs = (ctypes.c_size_t * 4)()
    assert P.lib.pdssm_chunk_state_offsets(ctypes.byref(d), offs) == 0
    assert offs[0] == 0 and offs[1] < offs[2] < offs[3]
    assert all(o % 256 == 0 for o in offs)
    for op in (P.OP_FWD, P.OP_BWD, P.OP_SEGMENT):
        assert P.workspace_bytes(d, op) > 0
    assert P.lib.pdssm_summary_bytes(ctypes.byref(d)) == 16 * 2 + 2 * 2 * 16 * 4


@pytest.mark.parametrize("bad,code", [
    (dict(B=0), 2), (dict(N=0), 2), (dict(N=1025), 2), (dict(K=257), 2), (dict(c=3), 2),
    (dict(dtype=7), 5), (dict(tau=-1), 2),
])
def test_invalid_dims_rejected(bad, code):
    d = dims(**bad)
    assert P.workspace_bytes(d, P.OP_FWD) == 0
    st = P.lib.pdssm_scan_fwd(None, None, None, None, None, None, None, None, None, None,
                              ctypes.byref(d), None, 0, None)
    assert st == code
    assert len(P.lib.pdssm_last_error()) > 0


def test_null_and_workspace_and_alignment_checks():
    d = dims()
    p = ctypes.c_void_p(0x10000)     # never dereferenced: validation fails first
    # missing required pointers
    assert P.lib.pdssm_scan_fwd(None, p, p, p, None, None, p, None, p, None, ctypes.byref(d), p, 1 << 30, None) == 1
    # no outputs requested
    assert P.lib.pdssm_scan_fwd(p, p, p, p, None, None, None, None, p, None, ctypes.byref(d), p, 1 << 30, None) == 1
    # workspace too small
    assert P.lib.pdssm_scan_fwd(p, p, p, p, None, None, p, None, p, None, ctypes.byref(d), p, 1, None) == 6
    # misaligned bias
    q = ctypes.c_void_p(0x10001)
    assert P.lib.pdssm_scan_fwd(p, p, p, q, None, None, p, None, p, None, ctypes.byref(d), p, 1 << 30, None) == 4
    # readout without C
    assert P.lib.pdssm_scan_fwd(p, p, p, p, None, None, None, p, p, None, ctypes.byref(d), p, 1 << 30, None) == 1
    # backward requires h_saved or (recompute mode) the bias
    assert P.lib.pdssm_scan_bwd(p, p, p, None, None, None, p, None, None, None, None, p, p, None, None,
                                ctypes.byref(d), p, 1 << 30, None) == 1
    # recompute mode with a chunk too long for shared memory -> ERR_UNSUPPORTED (9)
    dr = dims(N=128, L=4096, c=2, tau=4096)
    assert P.lib.pdssm_scan_bwd(p, p, p, None, p, None, p, None, None, None, None, p, p, None, None,
                                ctypes.byref(dr), p, 1 << 30, None) == 9
    # select requires d_in >= 1
    assert P.lib.pdssm_select(p, p, None, p, None, None, ctypes.byref(d), p, 1 << 30, None) == 2
    ds = dims(d_in=8)
    assert P.lib.pdssm_select(p, p, None, p, p, None, ctypes.byref(ds), p, 1 << 30, None) == 1   # P needs dict
    # compose: rank out of range
    assert P.lib.pdssm_compose_carry(p, 4, 4, None, p, None, ctypes.byref(d), None) == 2
    assert P.lib.pdssm_compose_lambda(p, p, -1, 4, p, ctypes.byref(d), None) == 2
    assert P.lib.pdssm_sparsify(None, p, ctypes.byref(d), None) == 1


def test_dims_struct_layout():
    assert ctypes.sizeof(P.Dims) == 80


def test_next_rows_validate_before_any_cuda_call():
    """NEXT-1/2/3 entry points: synchronous argument validation (no GPU needed)."""
    fake = ctypes.c_void_p(4096)   # never dereferenced: every case fails validation first
    d = dims(N=16, K=4)
    # selector gradient: NULL -> ERR_NULL (1), temperature <= 0 -> ERR_RANGE (3)
    assert P.lib.pdssm_select_grad(None, fake, fake, 1.0, fake, ctypes.byref(d), None) == 1
    assert P.lib.pdssm_select_grad(fake, fake, fake, 0.0, fake, ctypes.byref(d), None) == 3
    assert P.lib.pdssm_select_grad(fake, fake, fake, float("nan"), fake, ctypes.byref(d), None) == 3
    # dictionary gradient: NULL -> 1; N > 128 -> ERR_UNSUPPORTED (9)
    assert P.lib.pdssm_dict_grad(None, fake, fake, fake, None, fake, 1.0, fake, None, ctypes.byref(d), None) == 1
    big = dims(N=200, K=4)
    assert P.lib.pdssm_dict_grad(fake, fake, fake, fake, None, fake, 1.0, fake, None, ctypes.byref(big), None) == 9
    # soft generator: N not a multiple of 16 -> 9; too little workspace -> ERR_WORKSPACE (6)
    odd = dims(N=24, K=4)
    assert P.lib.pdssm_soft_select(fake, fake, fake, ctypes.byref(odd), fake, 1 << 30, None) == 9
    assert P.lib.pdssm_soft_select(fake, fake, fake, ctypes.byref(d), fake, 16, None) == 6
    assert P.workspace_bytes(d, P.OP_SOFT) >= 3 * 2 * 100 * 8 * 4 + 3 * 16 * 16 * 8 * 4
    # layer forward and D generator: d_in must be >= 1 -> ERR_SHAPE (2)
    assert P.lib.pdssm_layer_fwd(fake, fake, fake, fake, fake, None, None, fake, None, None, fake,
                                 ctypes.byref(d), fake, 1 << 30, None) == 2
    assert P.lib.pdssm_diag_gen(fake, fake, None, fake, ctypes.byref(d), None) == 2
    dl = P.make_dims(2, 3, 100, 16, 4, c=2, d_in=32)
    assert P.workspace_bytes(dl, P.OP_LAYER) >= 2 * 3 * 100 * 2 * 16 * 4
