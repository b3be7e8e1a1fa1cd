"""Multi-process (world size 2, gloo, CPU) tests of the multi-GPU host logic in
paper_2605_19150_b200/parallel.py: the partition, the all-gather in
rank order and the summary composition order.  The per-rank compute is the float64
oracle (test infrastructure), so these run without a GPU; on GPUs the same
SequenceParallelScan drives the C-ABI library over NCCL (tests/test_gpu_sp.py covers
the device summary algebra)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleOps:
    """SequenceParallelScan ops on the CPU oracle.  Segment inputs are passed as
    (P maps, None, D complex, b complex); summaries travel as float64 tensors
    [B][H][5N] = (pi, Re d, Im d, Re beta, Im beta)."""

    def segment_summary(self, Pm, _unused, Dz, bz):
        pi, d, beta = O.segment_summary(Pm, Dz, bz)
        return torch.from_numpy(np.concatenate([np.asarray(pi, np.float64), d.real, d.imag, beta.real, beta.imag], -1))

    @staticmethod
    def _unpack(gathered):
        g = gathered.numpy()
        N = g.shape[-1] // 5
        pis = g[..., :N].astype(np.int64)
        ds = g[..., N:2 * N] + 1j * g[..., 2 * N:3 * N]
        betas = g[..., 3 * N:4 * N] + 1j * g[..., 4 * N:]
        return pis, ds, betas

    def compose_carry(self, gathered, rank, world, h0):
        pis, ds, betas = self._unpack(gathered)
        return O.compose_summaries(list(pis), list(ds), list(betas), rank, h0)

    def scan_fwd(self, Pm, _unused, Dz, bz, carry):
        return O.scan_forward(Pm, Dz, bz, carry)

    def segment_summary_bwd(self, Pm, _unused, Dz, h, e):
        # beta' = A_{s}^T lambda^loc_{s}: the reverse scan's dh0 with zero incoming adjoint
        bp = O.scan_backward(Pm, Dz, h, e)[3]
        return torch.from_numpy(np.concatenate([bp.real, bp.imag], -1))

    def compose_lambda(self, gathered, beta_all, rank, world):
        pis, ds, _ = self._unpack(gathered)
        bp = beta_all.numpy()
        N = bp.shape[-1] // 2
        bp = bp[..., :N] + 1j * bp[..., N:]
        B, H = pis.shape[1:3]
        mu = np.zeros((B, H, N), np.complex128)   # adjoint entering the last segment
        for g in range(world - 1, rank, -1):      # mu_{g-1} = beta'_g + Abar_g^T mu_g
            nxt = np.empty_like(mu)
            for b in range(B):
                for h in range(H):
                    nxt[b, h] = bp[g, b, h] + O.pd_apply_transpose(pis[g, b, h], ds[g, b, h], mu[b, h])
            mu = nxt
        return mu

    def scan_bwd(self, Pm, _unused, Dz, h, e, carry, lam_in):
        e2 = np.array(e, np.complex128)
        e2[:, :, -1] += lam_in
        return O.scan_backward(Pm, Dz, h, e2, carry)


def _global_inputs(L, c, seed):
    B, H, N, K = 2, 3, 16, 5
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=seed, h0=True, dh=True)
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, h0, e = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "h0", "dh"))
    return Pm, Dz, bz, h0, e


def _init(rank, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)


def _sp_worker(rank, port, L, c):
    from paper_2605_19150_b200.parallel import SequenceParallelScan, shard_range
    _init(rank, port)
    try:
        Pm, Dz, bz, h0, e = _global_inputs(L, c, seed=70 + L)
        h_ref = O.scan_forward(Pm, Dz, bz, h0)
        Pi, _ = O.prefix_maps(Pm, Dz)
        db_r, dD_r, g_r, dh0_r = O.scan_backward(Pm, Dz, h_ref, e, h0)
        s, t = shard_range(L, WORLD, rank)
        seg = lambda a: a[:, :, s:t]
        sp = SequenceParallelScan(OracleOps())
        h, ctx = sp.forward(seg(Pm), None, seg(Dz), seg(bz), h0)
        if s > 0:
            assert np.array_equal(ctx["prefix_map"], Pi[:, :, s - 1])       # integer maps: exact
            assert np.max(np.abs(ctx["carry"] - h_ref[:, :, s - 1])) <= 1e-10 * np.max(np.abs(h_ref))
        else:
            assert np.array_equal(ctx["carry"], h0)
        assert np.max(np.abs(h - h_ref[:, :, s:t])) <= 1e-10 * np.max(np.abs(h_ref))
        db, dD, g, dh0 = sp.backward(seg(Pm), None, seg(Dz), h, ctx, seg(e))
        sc = lambda a: 1e-10 * max(np.max(np.abs(a)), 1e-30)
        assert np.max(np.abs(db - db_r[:, :, s:t])) <= sc(db_r)
        assert np.max(np.abs(dD - dD_r[:, :, s:t])) <= sc(dD_r)
        assert np.max(np.abs(g - g_r[:, :, s:t])) <= sc(g_r)
        if rank == 0:
            assert np.max(np.abs(dh0 - dh0_r)) <= sc(dh0_r)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _bh_worker(rank, port, L):
    from paper_2605_19150_b200.parallel import all_gather_rank_order, shard_sequences
    _init(rank, port)
    try:
        Pm, Dz, bz, h0, e = _global_inputs(L, 2, seed=90)
        h_ref = O.scan_forward(Pm, Dz, bz, h0)
        mine = [shard_sequences(a, WORLD, rank)[None] for a in (Pm, Dz, bz, h0)]   # [1][S_r][...]
        h = O.scan_forward(*mine)[0]
        got = all_gather_rank_order(torch.from_numpy(np.stack([h.real, h.imag])))   # [G][2][S_r][L][N]
        full = np.concatenate([got[r, 0].numpy() + 1j * got[r, 1].numpy() for r in range(WORLD)], 0)
        assert np.array_equal(full, h_ref.reshape(-1, *h_ref.shape[2:]))     # same per-sequence arithmetic
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L,c", [(37, 2), (64, 1), (5, 2)])
def test_sequence_parallel_world2_gloo(L, c):
    mp.spawn(_sp_worker, args=(_free_port(), L, c), nprocs=WORLD, join=True)


def test_batch_head_shards_world2_gloo():
    mp.spawn(_bh_worker, args=(_free_port(), 23), nprocs=WORLD, join=True)


def test_shard_range_partitions():
    from paper_2605_19150_b200.parallel import shard_range
    for n in (0, 1, 5, 8, 2048, 17984):
        for w in (1, 2, 3, 4, 8):
            blocks = [shard_range(n, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
            sizes = [e - s for s, e in blocks]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
