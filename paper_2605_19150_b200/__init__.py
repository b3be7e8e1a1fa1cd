"""Flash PD-SSM hot path on B200 (sm_100a): thin Python binding of libpdssm.so.

Argument marshalling only -- every step of the path runs in the CUDA kernels
behind the C ABI declared in ``include/pdssm.h``.  PyTorch provides device
memory and the current stream.  There is no CPU fallback: importing this
package fails loudly if ``libpdssm.so`` is missing, and every call raises
``PdssmError`` on a non-zero status.

Complex tensors cross the boundary as real tensors with an explicit plane
axis ``[..., c, N]`` (c = 1 real, c = 2 re/im), never as torch.complex64.
"""
from __future__ import annotations

import ctypes
import os
import re

__all__ = [
    "PdssmError", "Dims", "lib", "sparsify", "select", "scan_fwd", "scan_bwd",
    "segment_summary", "compose_carry", "segment_summary_bwd", "compose_lambda",
    "check_device", "chunk_state_views", "select_grad", "dict_grad", "scan", "layer_fwd", "layer_fwd_gen", "diag_gen", "soft_select", "default_chunk", "workspace_bytes",
    "F32", "BF16", "PER_STEP", "PER_DICT", "CHECK_FINITE", "EXPORT_MAPS",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpdssm.so")
if os.environ.get("PDSSM_LIB_VARIANT"):   # tuning experiments: variants/<name>.so built by tools/build_variant.sh
    LIB_PATH = os.path.join(_HERE, "variants", os.environ["PDSSM_LIB_VARIANT"] + ".so")

F32, BF16 = 0, 1
PER_STEP, PER_DICT = 0, 1
CHECK_FINITE, DETERMINISTIC, SAVE_STATES, EXPORT_MAPS = 1, 2, 4, 8
OP_SELECT, OP_FWD, OP_BWD, OP_SEGMENT, OP_READOUT, OP_LAYER, OP_SOFT = 0, 1, 2, 3, 4, 5, 6

STATUS = {0: "PDSSM_OK", 1: "PDSSM_ERR_NULL", 2: "PDSSM_ERR_SHAPE", 3: "PDSSM_ERR_RANGE",
          4: "PDSSM_ERR_ALIGN", 5: "PDSSM_ERR_DTYPE", 6: "PDSSM_ERR_WORKSPACE",
          7: "PDSSM_ERR_NONFINITE", 8: "PDSSM_ERR_CUDA", 9: "PDSSM_ERR_UNSUPPORTED"}


class PdssmError(RuntimeError):
    def __init__(self, status, message):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {message}")


class Dims(ctypes.Structure):
    """Mirror of ``pdssm_dims`` (include/pdssm.h)."""
    _fields_ = [("batch", ctypes.c_int64), ("heads", ctypes.c_int64), ("len", ctypes.c_int64),
                ("state", ctypes.c_int64), ("dict", ctypes.c_int64), ("d_in", ctypes.c_int64),
                ("p_out", ctypes.c_int64), ("chunk", ctypes.c_int32), ("is_complex", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("diag_mode", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, sz, i32, u32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32, ctypes.c_uint32
    D = ctypes.POINTER(Dims)
    sig = {
        "pdssm_default_chunk": (i32, [D]),
        "pdssm_workspace_bytes": (sz, [D, ctypes.c_int]),
        "pdssm_chunk_state_bytes": (sz, [D]),
        "pdssm_chunk_state_offsets": (ctypes.c_int, [D, ctypes.POINTER(ctypes.c_size_t)]),
        "pdssm_summary_bytes": (sz, [D]),
        "pdssm_sparsify": (ctypes.c_int, [vp, vp, D, vp]),
        "pdssm_select": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, D, vp, sz, vp]),
        "pdssm_project": (ctypes.c_int, [vp, vp, vp, D, vp]),
        "pdssm_readout": (ctypes.c_int, [vp, vp, vp, D, vp, sz, vp]),
        "pdssm_scan_fwd": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, D, vp, sz, vp]),
        "pdssm_scan_bwd": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, D, vp, sz, vp]),
        "pdssm_segment_summary": (ctypes.c_int, [vp, vp, vp, vp, vp, D, vp, sz, vp]),
        "pdssm_compose_carry": (ctypes.c_int, [vp, i32, i32, vp, vp, vp, D, vp]),
        "pdssm_segment_summary_bwd": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, D, vp, sz, vp]),
        "pdssm_compose_lambda": (ctypes.c_int, [vp, vp, i32, i32, vp, D, vp]),
        "pdssm_select_grad": (ctypes.c_int, [vp, vp, vp, ctypes.c_float, vp, D, vp]),
        "pdssm_soft_select": (ctypes.c_int, [vp, vp, vp, D, vp, sz, vp]),
        "pdssm_diag_gen": (ctypes.c_int, [vp, vp, vp, vp, D, vp]),
        "pdssm_layer_fwd": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, D, vp, sz, vp]),
        "pdssm_layer_fwd_gen": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, D, vp, sz, vp]),
        "pdssm_dict_grad": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, ctypes.c_float, vp, vp, D, vp]),
        "pdssm_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "pdssm_last_error": (ctypes.c_char_p, []),
        "pdssm_version": (ctypes.c_char_p, []),
        "pdssm_check_device": (ctypes.c_int, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


lib = _load()


def header_symbols():
    """Function names declared in include/pdssm.h (for the export test)."""
    hdr = os.path.join(os.path.dirname(_HERE), "include", "pdssm.h")
    txt = open(hdr).read()
    return sorted(set(re.findall(r"\b(pdssm_[a-z_]+)\s*\(", txt)))


def _check(status):
    if status != 0:
        raise PdssmError(status, lib.pdssm_last_error().decode())


# ---------------------------------------------------------------- torch glue
def _torch():
    import torch
    return torch


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dtype_code(t):
    torch = _torch()
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise TypeError(f"act tensors must be float32 or bfloat16, got {t.dtype}")


def _act_dtype(code):
    torch = _torch()
    return torch.bfloat16 if code == BF16 else torch.float32


def _contig(t, name):
    if t is not None and (not t.is_cuda or not t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous CUDA tensor")
    return t


def make_dims(B, H, L, N, K, c=1, dtype=F32, tau=0, diag_mode=PER_STEP, d_in=0, p_out=0, flags=0):
    return Dims(batch=B, heads=H, len=L, state=N, dict=K, d_in=d_in, p_out=p_out, chunk=tau,
                is_complex=c, dtype=dtype, diag_mode=diag_mode, flags=flags, reserved=0)


def default_chunk(dims):
    return lib.pdssm_default_chunk(ctypes.byref(dims))


def workspace_bytes(dims, op):
    return lib.pdssm_workspace_bytes(ctypes.byref(dims), op)


def _workspace(dims, op, device):
    torch = _torch()
    n = workspace_bytes(dims, op)
    return torch.empty(max(n, 256), dtype=torch.uint8, device=device), max(n, 256)


def chunk_state_views(chunk_state, dims):
    """Typed views (pi_bar, d_bar, beta_bar, carry) of a chunk_state buffer."""
    torch = _torch()
    offs = (ctypes.c_size_t * 4)()
    _check(lib.pdssm_chunk_state_offsets(ctypes.byref(dims), offs))
    S = dims.batch * dims.heads
    C = -(-dims.len // default_chunk(dims))
    N, c = dims.state, dims.is_complex
    pi = chunk_state[offs[0]:offs[0] + S * C * N * 2].view(torch.int16).view(dims.batch, dims.heads, C, N)
    f = [chunk_state[o:o + S * C * c * N * 4].view(torch.float32).view(dims.batch, dims.heads, C, c, N)
         for o in offs[1:]]
    return pi, f[0], f[1], f[2]


# ---------------------------------------------------------------- entry points
def sparsify(M, check_finite=False):
    """a1: dict_idx[h,k,j] = argmax_i M[h,k,i,j]  (Eq. 5)."""
    torch = _torch()
    _contig(M, "M")
    H, K, N, _ = M.shape
    dims = make_dims(1, H, 1, N, K, flags=CHECK_FINITE if check_finite else 0)
    out = torch.empty((H, K, N), dtype=torch.int16, device=M.device)
    _check(lib.pdssm_sparsify(_ptr(M), _ptr(out), ctypes.byref(dims), _stream()))
    return out


def select(x, S, dict_idx=None, want_P=False, want_logits=False, check_finite=False):
    """a2-a4: k* = argmax_k S x_t per head (Eqs. 6-8)."""
    torch = _torch()
    _contig(x, "x"), _contig(S, "S"), _contig(dict_idx, "dict_idx")
    B, L, d_in = x.shape
    H, K, _ = S.shape
    N = dict_idx.shape[-1] if dict_idx is not None else 1
    dims = make_dims(B, H, L, N, K, dtype=_dtype_code(x), d_in=d_in, flags=CHECK_FINITE if check_finite else 0)
    kstar = torch.empty((B, H, L), dtype=torch.uint8, device=x.device)
    P = torch.empty((B, H, L, N), dtype=torch.int16, device=x.device) if want_P else None
    logits = torch.empty((B, H, L, K), dtype=torch.float32, device=x.device) if want_logits else None
    ws, wsb = _workspace(dims, OP_SELECT, x.device)
    _check(lib.pdssm_select(_ptr(x), _ptr(S), _ptr(dict_idx), _ptr(kstar), _ptr(P), _ptr(logits),
                            ctypes.byref(dims), _ptr(ws), wsb, _stream()))
    return kstar, P, logits


def project(x, Bw, out=None):
    """a5: b_t = B x_t in the scan layout (Eq. 1).

    x [B][L][d_in], Bw [H][c][N][d_in] (same dtype) -> b [B][H][L][c][N]."""
    torch = _torch()
    _contig(x, "x"), _contig(Bw, "Bw")
    B, L, d_in = x.shape
    H, c, N, _ = Bw.shape
    if Bw.dtype != x.dtype:
        raise TypeError("x and Bw must have the same dtype")
    dims = make_dims(B, H, L, N, 1, c=c, dtype=_dtype_code(x), d_in=d_in)
    b = out if out is not None else torch.empty((B, H, L, c, N), dtype=x.dtype, device=x.device)
    _check(lib.pdssm_project(_ptr(x), _ptr(Bw), _ptr(b), ctypes.byref(dims), _stream()))
    return b


def readout(h, C, out=None, ws=None):
    """a8: y_t = Re(C_h h_t) (Eq. 1).  h [B][H][L][c][N], C f32 [H][c][P][N]
    -> y [B][L][H][P] in h's dtype."""
    torch = _torch()
    _contig(h, "h"), _contig(C, "C")
    B, H, L, c, N = h.shape
    Pp = C.shape[2]
    dims = make_dims(B, H, L, N, 1, c=c, dtype=_dtype_code(h), p_out=Pp)
    y = out if out is not None else torch.empty((B, L, H, Pp), dtype=h.dtype, device=h.device)
    if ws is None:
        ws, wsb = _workspace(dims, OP_READOUT, h.device)
    else:
        wsb = ws.numel()
    _check(lib.pdssm_readout(_ptr(h), _ptr(C), _ptr(y), ctypes.byref(dims), _ptr(ws), wsb, _stream()))
    return y


def scan_fwd(kstar, dict_idx, diag, bias, h0=None, C=None, tau=0, per_dict=False, want_h=True,
             want_y=False, export_maps=False, check_finite=False, out=None):
    """a6-a8: forward chunked scan (Alg. 1) + optional fused readout.

    Returns dict(h, y, chunk_state, maps, dims).  ``out`` may pass preallocated
    tensors (keys h, y, chunk_state, maps, ws) to keep the call allocation-free."""
    torch = _torch()
    for n, t in (("kstar", kstar), ("dict_idx", dict_idx), ("diag", diag), ("bias", bias), ("h0", h0), ("C", C)):
        _contig(t, n)
    B, H, L = kstar.shape
    K, N = dict_idx.shape[-2:]
    c = bias.shape[-2]
    P = C.shape[-2] if C is not None else 0
    flags = (CHECK_FINITE if check_finite else 0) | (EXPORT_MAPS if export_maps else 0)
    dims = make_dims(B, H, L, N, K, c=c, dtype=_dtype_code(bias), tau=tau,
                     diag_mode=PER_DICT if per_dict else PER_STEP, p_out=P, flags=flags)
    out = dict(out or {})
    dev = bias.device
    tau_eff = default_chunk(dims)
    Cch = -(-L // tau_eff)
    h = out.get("h") if want_h else None
    if want_h and h is None:
        h = torch.empty((B, H, L, c, N), dtype=bias.dtype, device=dev)
    y = out.get("y") if want_y else None
    if want_y and y is None:
        y = torch.empty((B, L, H, P), dtype=bias.dtype, device=dev)
    cs = out.get("chunk_state")
    if cs is None:
        cs = torch.empty(lib.pdssm_chunk_state_bytes(ctypes.byref(dims)), dtype=torch.uint8, device=dev)
    maps = out.get("maps") if export_maps else None
    if export_maps and maps is None:
        maps = torch.empty((B, H, Cch + 1, N), dtype=torch.int16, device=dev)
    ws = out.get("ws")
    wsb = workspace_bytes(dims, OP_FWD)
    if ws is None or ws.numel() < wsb:
        ws, wsb = _workspace(dims, OP_FWD, dev)
    else:
        wsb = ws.numel()
    _check(lib.pdssm_scan_fwd(_ptr(kstar), _ptr(dict_idx), _ptr(diag), _ptr(bias), _ptr(h0), _ptr(C), _ptr(h),
                              _ptr(y), _ptr(cs), _ptr(maps), ctypes.byref(dims), _ptr(ws), wsb, _stream()))
    return dict(h=h, y=y, chunk_state=cs, maps=maps, dims=dims, tau=tau_eff)


def scan_bwd(kstar, dict_idx, diag, h_saved, chunk_state, dims, dh=None, dy=None, C=None, h0=None,
             lam_in=None, want_g=True, want_dh0=True, out=None, bias=None):
    """a9: reverse transposed scan -> (dbias, ddiag, gsel, dh0) (App. C).
    h_saved=None with bias=b_t: recompute mode (states replayed per chunk from chunk_state)."""
    torch = _torch()
    for n, t in (("kstar", kstar), ("dict_idx", dict_idx), ("diag", diag), ("h_saved", h_saved), ("bias", bias),
                 ("chunk_state", chunk_state), ("dh", dh), ("dy", dy), ("C", C), ("h0", h0), ("lam_in", lam_in)):
        _contig(t, n)
    B, H, L = kstar.shape
    N, c = dims.state, dims.is_complex
    dev = chunk_state.device
    out = dict(out or {})
    act = h_saved if h_saved is not None else bias
    db = out.get("dbias")
    if db is None:
        db = torch.empty_like(act)
    dD = out.get("ddiag")
    if dD is None:
        dD = torch.empty(diag.shape, dtype=torch.float32 if dims.diag_mode == PER_DICT else act.dtype, device=dev)
    g = out.get("gsel") if want_g else None
    if want_g and g is None:
        g = torch.empty((B, H, L), dtype=torch.float32, device=dev)
    dh0 = out.get("dh0") if want_dh0 else None
    if want_dh0 and dh0 is None:
        dh0 = torch.empty((B, H, c, N), dtype=torch.float32, device=dev)
    ws = out.get("ws")
    wsb = workspace_bytes(dims, OP_BWD)
    if ws is None or ws.numel() < wsb:
        ws, wsb = _workspace(dims, OP_BWD, dev)
    else:
        wsb = ws.numel()
    _check(lib.pdssm_scan_bwd(_ptr(kstar), _ptr(dict_idx), _ptr(diag), _ptr(h_saved), _ptr(bias), _ptr(h0),
                              _ptr(chunk_state),
                              _ptr(dh), _ptr(dy), _ptr(C), _ptr(lam_in), _ptr(db), _ptr(dD), _ptr(g), _ptr(dh0),
                              ctypes.byref(dims), _ptr(ws), wsb, _stream()))
    return db, dD, g, dh0


def soft_select(logits, M, bf16=False, out=None, ws=None):
    """NEXT-3 PD-SSM soft generator (Eqs. 2-4): P_t = column_hardmax(sum_k softmax(logits)_k M_k) -> int16 [B,H,L,N].
    bf16=True runs the mixture GEMM in bf16 (kind::f16), else 3xTF32."""
    torch = _torch()
    B, H, L, K = logits.shape
    N = M.shape[-1]
    dims = make_dims(B, H, L, N, K, dtype=BF16 if bf16 else F32)
    P = torch.empty((B, H, L, N), dtype=torch.int16, device=logits.device) if out is None else out
    wsb = workspace_bytes(dims, OP_SOFT)
    if ws is None or ws.numel() < wsb:
        ws, wsb = _workspace(dims, OP_SOFT, logits.device)
    else:
        wsb = ws.numel()
    _check(lib.pdssm_soft_select(_ptr(_contig(logits, "logits")), _ptr(_contig(M, "M")), _ptr(P), ctypes.byref(dims),
                                 _ptr(ws), wsb, _stream()))
    return P


def diag_gen(x, Wd, bias=None, out=None):
    """NEXT-2 D_t generator: D = sigmoid(W_mag x + bias) exp(i W_phase x) -> act [B,H,L,c,N] (PER_STEP diag)."""
    torch = _torch()
    for n, t in (("x", x), ("Wd", Wd), ("bias", bias)):
        _contig(t, n)
    B, L, d_in = x.shape
    H, c, N, _ = Wd.shape
    dims = make_dims(B, H, L, N, 1, c=c, dtype=_dtype_code(x), d_in=d_in)
    D = torch.empty((B, H, L, c, N), dtype=x.dtype, device=x.device) if out is None else out
    _check(lib.pdssm_diag_gen(_ptr(x), _ptr(Wd), _ptr(bias), _ptr(D), ctypes.byref(dims), _stream()))
    return D


def layer_fwd(x, S, dict_idx, diag, Bw, C=None, h0=None, per_dict=True, want_h=True, out=None, Wd=None,
              bias_mag=None):
    """Layer-level forward (select -> b = Bx -> scan -> y = Re(Ch)) with the north_star argument list.
    Wd (with diag=None): the D_t generator weights [H][c][N][d_in] (+ bias_mag [H][N]) fused into the
    same GEMM as the selector and the projection (pdssm_layer_fwd_gen; PER_STEP).
    Returns dict(kstar, h, y, chunk_state, dims)."""
    torch = _torch()
    for n, t in (("x", x), ("S", S), ("dict_idx", dict_idx), ("diag", diag), ("Bw", Bw), ("C", C), ("h0", h0),
                 ("Wd", Wd), ("bias_mag", bias_mag)):
        _contig(t, n)
    if Wd is not None:
        per_dict = False
    B, L, d_in = x.shape
    H, c, N, _ = Bw.shape
    K = S.shape[1]
    P = C.shape[-2] if C is not None else 0
    dims = make_dims(B, H, L, N, K, c=c, dtype=_dtype_code(x), diag_mode=PER_DICT if per_dict else PER_STEP,
                     d_in=d_in, p_out=P)
    out = dict(out or {})
    dev = x.device
    ks = out.get("kstar")
    if ks is None:
        ks = torch.empty((B, H, L), dtype=torch.uint8, device=dev)
    h = out.get("h") if want_h else None
    if want_h and h is None:
        h = torch.empty((B, H, L, c, N), dtype=x.dtype, device=dev)
    y = out.get("y")
    if C is not None and y is None:
        y = torch.empty((B, L, H, P), dtype=x.dtype, device=dev)
    cs = out.get("chunk_state")
    if cs is None:
        cs = torch.empty(lib.pdssm_chunk_state_bytes(ctypes.byref(dims)), dtype=torch.uint8, device=dev)
    ws = out.get("ws")
    wsb = workspace_bytes(dims, OP_LAYER)
    if ws is None or ws.numel() < wsb:
        ws, wsb = _workspace(dims, OP_LAYER, dev)
    else:
        wsb = ws.numel()
    if Wd is not None:
        _check(lib.pdssm_layer_fwd_gen(_ptr(x), _ptr(S), _ptr(dict_idx), _ptr(Wd), _ptr(bias_mag), _ptr(Bw), _ptr(C),
                                       _ptr(h0), _ptr(ks), _ptr(h), _ptr(y), _ptr(cs), ctypes.byref(dims), _ptr(ws), wsb,
                                       _stream()))
    else:
        _check(lib.pdssm_layer_fwd(_ptr(x), _ptr(S), _ptr(dict_idx), _ptr(diag), _ptr(Bw), _ptr(C), _ptr(h0), _ptr(ks),
                                   _ptr(h), _ptr(y), _ptr(cs), ctypes.byref(dims), _ptr(ws), wsb, _stream()))
    return dict(kstar=ks, h=h, y=y, chunk_state=cs, dims=dims)


def select_grad(logits, kstar, gsel, temp, out=None):
    """NEXT-1 selector surrogate gradient (Prop. 2): -> dlogits f32 [B,H,L,K]."""
    torch = _torch()
    B, H, L, K = logits.shape
    dims = make_dims(B, H, L, 1, K)
    out = torch.empty_like(logits) if out is None else out
    _check(lib.pdssm_select_grad(_ptr(_contig(logits, "logits")), _ptr(_contig(kstar, "kstar")), _ptr(_contig(gsel, "gsel")),
                                 float(temp), _ptr(out), ctypes.byref(dims), _stream()))
    return out


def dict_grad(M, kstar, diag, h_saved, dbias, temp, dims, h0=None, want_G=False, out=None):
    """NEXT-1 dictionary surrogate gradient (Prop. 2): -> (dM, G or None), f32 [H,K,N,N]."""
    torch = _torch()
    dM = torch.empty_like(M) if out is None else out
    G = torch.empty_like(M) if want_G else None
    _check(lib.pdssm_dict_grad(_ptr(_contig(M, "M")), _ptr(kstar), _ptr(diag), _ptr(h_saved), _ptr(h0), _ptr(dbias),
                               float(temp), _ptr(dM), _ptr(G), ctypes.byref(dims), _stream()))
    return dM, G


def summary_bytes(dims):
    return lib.pdssm_summary_bytes(ctypes.byref(dims))


def segment_summary(kstar, dict_idx, diag, bias, dims, out=None):
    torch = _torch()
    S = dims.batch * dims.heads
    sb = summary_bytes(dims)
    if out is None:
        out = torch.empty(S * sb, dtype=torch.uint8, device=bias.device)
    ws, wsb = _workspace(dims, OP_SEGMENT, bias.device)
    _check(lib.pdssm_segment_summary(_ptr(kstar), _ptr(dict_idx), _ptr(diag), _ptr(bias), _ptr(out),
                                     ctypes.byref(dims), _ptr(ws), wsb, _stream()))
    return out


def summary_views(summaries, dims, G=1):
    """(pi [G][B][H][N] int16, d [G][B][H][c][N], beta [G][B][H][c][N]) views of gathered summaries."""
    torch = _torch()
    sb = summary_bytes(dims)
    N, c = dims.state, dims.is_complex
    npad = (N + 7) // 8 * 8
    blk = summaries.view(G, dims.batch, dims.heads, sb)
    pi = blk[..., :npad * 2].contiguous().view(torch.int16)[..., :N]
    d = blk[..., npad * 2:npad * 2 + c * N * 4].contiguous().view(torch.float32).view(G, dims.batch, dims.heads, c, N)
    beta = blk[..., npad * 2 + c * N * 4:].contiguous().view(torch.float32).view(G, dims.batch, dims.heads, c, N)
    return pi, d, beta


def compose_carry(summaries, rank, G, dims, h0=None, want_map=True):
    torch = _torch()
    B, H, N, c = dims.batch, dims.heads, dims.state, dims.is_complex
    carry = torch.empty((B, H, c, N), dtype=torch.float32, device=summaries.device)
    m = torch.empty((B, H, N), dtype=torch.int16, device=summaries.device) if want_map else None
    _check(lib.pdssm_compose_carry(_ptr(summaries), rank, G, _ptr(h0), _ptr(carry), _ptr(m), ctypes.byref(dims),
                                   _stream()))
    return carry, m


def segment_summary_bwd(kstar, dict_idx, diag, chunk_state, dims, dh=None, dy=None, C=None):
    torch = _torch()
    B, H, N, c = dims.batch, dims.heads, dims.state, dims.is_complex
    beta = torch.empty((B, H, c, N), dtype=torch.float32, device=chunk_state.device)
    ws, wsb = _workspace(dims, OP_SEGMENT, chunk_state.device)
    _check(lib.pdssm_segment_summary_bwd(_ptr(kstar), _ptr(dict_idx), _ptr(diag), _ptr(chunk_state), _ptr(dh),
                                         _ptr(dy), _ptr(C), _ptr(beta), ctypes.byref(dims), _ptr(ws), wsb,
                                         _stream()))
    return beta


def compose_lambda(fwd_summaries, beta_bwd, rank, G, dims):
    torch = _torch()
    B, H, N, c = dims.batch, dims.heads, dims.state, dims.is_complex
    lam = torch.empty((B, H, c, N), dtype=torch.float32, device=beta_bwd.device)
    _check(lib.pdssm_compose_lambda(_ptr(fwd_summaries), _ptr(beta_bwd), rank, G, _ptr(lam), ctypes.byref(dims),
                                    _stream()))
    return lam


def check_device():
    """Synchronise and read/clear the device error word (PDSSM_CHECK_FINITE)."""
    _check(lib.pdssm_check_device(_stream()))


# ---------------------------------------------------------------- autograd glue
_SCAN_FN = None


def _scan_fn():
    """torch.autograd.Function over pdssm_scan_fwd / pdssm_scan_bwd (built lazily so the
    binding imports without touching autograd)."""
    global _SCAN_FN
    if _SCAN_FN is not None:
        return _SCAN_FN
    torch = _torch()

    class _Scan(torch.autograd.Function):
        @staticmethod
        def forward(ctx, diag, bias, h0, kstar, dict_idx, per_dict):
            # the backward must see exactly the (contiguous) tensors the forward consumed
            diag_c, bias_c = diag.contiguous(), bias.contiguous()
            h0_c = None if h0 is None else h0.contiguous()
            kstar_c, dict_c = kstar.contiguous(), dict_idx.contiguous()
            f = scan_fwd(kstar_c, dict_c, diag_c, bias_c, h0=h0_c, per_dict=per_dict)
            ctx.save_for_backward(kstar_c, dict_c, diag_c, f["h"], f["chunk_state"], h0_c)
            ctx.dims = f["dims"]
            return f["h"]

        @staticmethod
        def backward(ctx, dh):
            kstar, dict_idx, diag, h, cs, h0 = ctx.saved_tensors
            db, dD, _, dh0 = scan_bwd(kstar, dict_idx, diag, h, cs, ctx.dims, dh=dh.contiguous(), h0=h0,
                                      want_g=False, want_dh0=h0 is not None)
            return dD, db, dh0, None, None, None

    _SCAN_FN = _Scan
    return _Scan


def scan(diag, bias, kstar, dict_idx, h0=None, per_dict=False):
    """Differentiable h = scan(D, b; k*, dict) (Eq. 1 with the hard selection held fixed, PAPER.md:94-101,
    :222): gradients flow to diag (PER_STEP: per step; PER_DICT: summed per entry), bias and h0 through
    the reverse transposed scan (App. C).  Complex tensors use the [..., c, N] plane layout."""
    return _scan_fn().apply(diag, bias, h0, kstar, dict_idx, per_dict)
