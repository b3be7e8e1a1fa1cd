"""NEXT-4: the multi-head Flash PD-SSM block (Fig. 5) around the hot path.

The mixer of one layer, per head h (H heads of state N, dictionary of K dense N x N matrices):

  k*_t   = argmax_k (S_h u_t)_k                          (Eqs. 6-7)       pdssm_select (tcgen05 + argmax)
  P_t    = column_argmax(M_{h,k*_t})                     (Eqs. 5, 8)      pdssm_sparsify, once per step
  D_t    = sigmoid(W_mag u_t + b_mag) exp(i W_phase u_t) (reading R30)
  b_t    = B_h u_t                                        (Eq. 1)
  h_t    = P_t D_t h_{t-1} + b_t                          (Eq. 1)          pdssm_scan_fwd / pdssm_scan_bwd
  y_t    = Re(C_h h_t)                                    (Eq. 1, psi = Re)

with the straight-through surrogate gradients of Prop. 2 for the two argmaxes:
dlogits from pdssm_select_grad (NEXT-1) and dM from pdssm_dict_grad (NEXT-1), both fed by the
scan backward's g_t and lambda_t.  The block follows the Mamba pattern the paper cites (pre-norm
residual, input projection to (u, z), gate silu(z), output projection).

The hot path (selection, sparsification, scan, surrogate gradients) runs in libpdssm.so; the
dense projections, the norm, the D_t generator's elementwise maps and the optimizer are plain
PyTorch (they are outside the hot path).  Everything is float32 (the complex state as re/im
planes, c = 2)."""
from __future__ import annotations

import math

import torch
import torch.nn as nn
import torch.nn.functional as F

import paper_2605_19150_b200 as P


class _FlashPDSSMFn(torch.autograd.Function):
    """h = scan(select(u; S), sparsify(M), D, b) with Prop. 2's surrogate gradients."""

    @staticmethod
    def forward(ctx, u, S, M, diag, bias, temp):
        dict_idx = P.sparsify(M)
        kstar, _, logits = P.select(u, S, dict_idx, want_logits=True)
        f = P.scan_fwd(kstar, dict_idx, diag, bias)
        ctx.save_for_backward(u, S, M, diag, kstar, dict_idx, logits, f["h"], f["chunk_state"])
        ctx.dims = f["dims"]
        ctx.temp = float(temp)
        ctx.mark_non_differentiable(kstar)
        return f["h"], kstar

    @staticmethod
    def backward(ctx, dh, _dk):
        u, S, M, diag, kstar, dict_idx, logits, h, cs = ctx.saved_tensors
        db, dD, g, _ = P.scan_bwd(kstar, dict_idx, diag, h, cs, ctx.dims, dh=dh.contiguous(), want_dh0=False)
        dlog = P.select_grad(logits, kstar, g, ctx.temp)          # [B][H][L][K]
        dS = torch.einsum("bhtk,btd->hkd", dlog, u)
        du = torch.einsum("bhtk,hkd->btd", dlog, S)
        dM, _ = P.dict_grad(M, kstar, diag, h, db, ctx.temp, ctx.dims)
        return du, dS, dM, dD, db, None


class FlashPDSSMMixer(nn.Module):
    """One multi-head Flash PD-SSM layer d_model -> d_model (complex state, c = 2)."""

    def __init__(self, d_model, heads, state, dict_size):
        super().__init__()
        H, N, K, d = heads, state, dict_size, d_model
        if d % H:
            raise ValueError("d_model must be divisible by heads")
        self.H, self.N, self.K, self.P = H, N, K, d // H
        u = lambda *s, lim: nn.Parameter(torch.empty(*s).uniform_(-lim, lim))
        self.S = u(H, K, d, lim=1 / math.sqrt(d))                   # selector (Eq. 6)
        self.M = u(H, K, N, N, lim=1 / math.sqrt(N))                # dense dictionary (Eq. 5)
        self.W_mag = u(H, N, d, lim=1 / math.sqrt(d))
        self.b_mag = nn.Parameter(torch.full((H, N), 2.0))          # |D| ~ sigmoid(2) = 0.88 at init
        self.W_phase = u(H, N, d, lim=1 / math.sqrt(d))
        self.Bw = u(H, 2, N, d, lim=1 / math.sqrt(d))
        self.C = u(H, 2, self.P, N, lim=1 / math.sqrt(N))
        self.temp = 1.0                                             # annealed by the trainer

    def forward(self, u):
        u = u.contiguous()
        mag = torch.sigmoid(torch.einsum("btd,hnd->bhtn", u, self.W_mag) + self.b_mag[None, :, None, :])
        th = torch.einsum("btd,hnd->bhtn", u, self.W_phase)
        diag = torch.stack([mag * torch.cos(th), mag * torch.sin(th)], dim=3).contiguous()   # [B][H][L][2][N]
        bias = torch.einsum("btd,hcnd->bhtcn", u, self.Bw).contiguous()
        h, _ = _FlashPDSSMFn.apply(u, self.S, self.M, diag, bias, self.temp)
        y = torch.einsum("bhtn,hpn->bthp", h[:, :, :, 0], self.C[:, 0]) - \
            torch.einsum("bhtn,hpn->bthp", h[:, :, :, 1], self.C[:, 1])       # Re(C h)
        return y.reshape(u.shape[0], u.shape[1], -1)


class RMSNorm(nn.Module):
    def __init__(self, d, eps=1e-6):
        super().__init__()
        self.w = nn.Parameter(torch.ones(d))
        self.eps = eps

    def forward(self, x):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + self.eps) * self.w


class FlashPDSSMBlock(nn.Module):
    """Pre-norm residual block: x + out_proj(mixer(u) * silu(z)), (u, z) = in_proj(norm(x))."""

    def __init__(self, d_model, heads, state, dict_size):
        super().__init__()
        self.norm = RMSNorm(d_model)
        self.in_proj = nn.Linear(d_model, 2 * d_model, bias=False)
        self.mixer = FlashPDSSMMixer(d_model, heads, state, dict_size)
        self.out_proj = nn.Linear(d_model, d_model, bias=False)

    def forward(self, x):
        u, z = self.in_proj(self.norm(x)).chunk(2, dim=-1)
        return x + self.out_proj(self.mixer(u) * F.silu(z))


class FSAClassifier(nn.Module):
    """Token embedding -> n_layers Flash PD-SSM blocks -> norm -> linear head on the last token
    (the state-tracking setup of PAPER.md:303-313: predict the final state)."""

    def __init__(self, vocab, classes, d_model=128, heads=4, dict_size=None, n_layers=2):
        super().__init__()
        state = d_model // heads                                    # total state size = d_model
        K = dict_size or max(2, int(round(math.sqrt(d_model))))     # K = sqrt(D) rule
        self.embed = nn.Embedding(vocab, d_model)
        self.blocks = nn.ModuleList([FlashPDSSMBlock(d_model, heads, state, K) for _ in range(n_layers)])
        self.norm = RMSNorm(d_model)
        self.head = nn.Linear(d_model, classes)

    def set_temperature(self, t):
        for b in self.blocks:
            b.mixer.temp = float(t)

    def forward(self, tokens):
        x = self.embed(tokens)
        for b in self.blocks:
            x = b(x)
        return self.head(self.norm(x)[:, -1])
