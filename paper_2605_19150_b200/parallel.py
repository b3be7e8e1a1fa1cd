"""Multi-GPU host logic of the path; one process per GPU.

Two ways the scan shards:

* batch x head ("weak" in bench.py): the (b, h) sequences are independent (heads share
  nothing; the dictionary is read-only), so rank r owns a contiguous
  block of the flattened S = B*H sequences -- no collective on the data path.
* sequence parallel (long L): rank g owns steps [g*L/G, (g+1)*L/G) of every sequence.
  Forward: local segment summary (pi, d, beta) -- the segment's Alg. 1 aggregate with a
  single chunk ("the PD-SSM composition operator is associative") --> one
  all-gather in rank order --> compose summaries 0..g-1 onto h0 --> local scan from that
  carry.  Backward: mirrored; the segment's beta' summaries are gathered and composed
  from the right through the forward (pi, d) (the transposed aggregate is a gather).

The compute steps are delegated to an ``ops`` object (``CudaOps`` below: the C-ABI
library); the partition, the exchange and the rank ordering live here, so the same code
runs the multi-process CPU tests (gloo) and the GPUs (NCCL).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n, world, rank):
    """Contiguous block [s, e) of n units for `rank` of `world`; block sizes differ by at
    most one, earlier ranks take the larger blocks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    q, r = divmod(n, world)
    s = rank * q + min(rank, r)
    return s, s + q + (1 if rank < r else 0)


def all_gather_rank_order(t, group=None):
    """[world, *t.shape]: every rank's tensor, in rank order (NCCL: one
    all_gather_into_tensor; other backends: all_gather into a list)."""
    world = dist.get_world_size(group)
    t = t.contiguous()
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * t.numel(),), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.reshape(-1), group=group)
        return out.view(world, *t.shape)
    # gloo (CPU tests, or several ranks sharing one GPU): stage device tensors through the host
    src = t.cpu() if t.is_cuda else t
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src, group=group)
    return torch.stack(parts).to(t.device)


def shard_sequences(t, world, rank):
    """Batch x head shard of a [B][H][...] tensor: rank's contiguous block of the
    flattened S = B*H sequences, as [S_r][...]."""
    S = t.shape[0] * t.shape[1]
    s, e = shard_range(S, world, rank)
    return t.reshape(S, *t.shape[2:])[s:e]


class SequenceParallelScan:
    """One rank's segment of a sequence-parallel scan.  Inputs are the rank's time slice
    [B][H][L_g]...; ``ops`` provides segment_summary, compose_carry, scan_fwd,
    segment_summary_bwd, compose_lambda and scan_bwd (see CudaOps)."""

    def __init__(self, ops, group=None):
        self.ops = ops
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def forward(self, kstar, dict_idx, diag, bias, h0=None):
        summ = self.ops.segment_summary(kstar, dict_idx, diag, bias)
        gathered = all_gather_rank_order(summ, self.group)
        carry, prefix_map = self.ops.compose_carry(gathered, self.rank, self.world, h0)
        out = self.ops.scan_fwd(kstar, dict_idx, diag, bias, carry)
        return out, {"gathered": gathered, "carry": carry, "prefix_map": prefix_map}

    def backward(self, kstar, dict_idx, diag, fwd_out, ctx, dh):
        beta = self.ops.segment_summary_bwd(kstar, dict_idx, diag, fwd_out, dh)
        beta_all = all_gather_rank_order(beta, self.group)
        lam_in = self.ops.compose_lambda(ctx["gathered"], beta_all, self.rank, self.world)
        return self.ops.scan_bwd(kstar, dict_idx, diag, fwd_out, dh, ctx["carry"], lam_in)


class CudaOps:
    """The C-ABI library as SequenceParallelScan ops (device tensors, one rank = one GPU)."""

    def __init__(self, N, K, c, tau=0, per_dict=False):
        import paper_2605_19150_b200 as P
        self.P, self.N, self.K, self.c, self.tau, self.pd = P, N, K, c, tau, per_dict

    def _dims(self, kstar):
        B, H, L = kstar.shape
        return self.P.make_dims(B, H, L, self.N, self.K, c=self.c, tau=self.tau,
                                diag_mode=self.P.PER_DICT if self.pd else self.P.PER_STEP)

    def segment_summary(self, kstar, dict_idx, diag, bias):
        self._seg_dims = self._dims(kstar)   # every rank's segment has the same B, H, N, c
        return self.P.segment_summary(kstar, dict_idx, diag, bias, self._seg_dims)

    def compose_carry(self, gathered, rank, world, h0):
        return self.P.compose_carry(gathered.reshape(-1), rank, world, self._seg_dims, h0=h0)

    def scan_fwd(self, kstar, dict_idx, diag, bias, carry):
        return self.P.scan_fwd(kstar, dict_idx, diag, bias, h0=carry, tau=self.tau, per_dict=self.pd)

    def segment_summary_bwd(self, kstar, dict_idx, diag, fwd_out, dh):
        return self.P.segment_summary_bwd(kstar, dict_idx, diag, fwd_out["chunk_state"], fwd_out["dims"], dh=dh)

    def compose_lambda(self, gathered, beta_all, rank, world):
        return self.P.compose_lambda(gathered.reshape(-1), beta_all, rank, world, self._seg_dims)

    def scan_bwd(self, kstar, dict_idx, diag, fwd_out, dh, carry, lam_in):
        return self.P.scan_bwd(kstar, dict_idx, diag, fwd_out["h"], fwd_out["chunk_state"], fwd_out["dims"], dh=dh,
                               h0=carry, lam_in=lam_in)
