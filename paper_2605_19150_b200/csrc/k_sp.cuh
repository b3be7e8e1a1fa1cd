// Sequence-parallel summary algebra: the chunk aggregates of Alg. 1 lifted to
// per-rank segments (associativity of (A2,b2) o (A1,b1) = (A2 A1, A2 b1 + b2),
// PAPER.md:927-932).  All compositions run in fixed (ascending) order so every
// rank derives bit-identical carries from the same gathered summaries.
#pragma once
#include "k_scan_fwd.cuh"

namespace pdssm {

struct SummaryView {
    // one (b,h) block: pi u16[npad] | d f32[NC][N] | beta f32[NC][N]
    char* base;
    size_t block_bytes;
    int npad;
    __device__ __forceinline__ uint16_t* pi(size_t blk) const {
        return reinterpret_cast<uint16_t*>(base + blk * block_bytes);
    }
    __device__ __forceinline__ float* d(size_t blk) const {
        return reinterpret_cast<float*>(base + blk * block_bytes + (size_t)npad * 2);
    }
    template <int NC>
    __device__ __forceinline__ float* beta(size_t blk, int N) const {
        return d(blk) + NC * N;
    }
};

// Fold the C chunk aggregates of each sequence (ascending c) into one summary:
//   R <- agg_c o R :  pi <- pi_c[pi],  d <- d_c[pi] d,  beta <- Abar_c beta + beta_c
template <int NC>
__global__ void k_fold_aggregates(ChunkStateView cs, SummaryView out, int N, int C_ch) {
    extern __shared__ float smem[];
    float* wsh = smem;                                          // [NC][N]
    uint16_t* psh = reinterpret_cast<uint16_t*>(smem + NC * N);  // [N]
    const int s = blockIdx.x;
    const int j = threadIdx.x;
    const bool act = j < N;
    int pi = j;
    cpx d{1.f, 0.f}, beta{0.f, 0.f};
    for (int c = 0; c < C_ch; ++c) {
        const size_t ci = (size_t)s * C_ch + c;
        cpx dc{0.f, 0.f}, bc{0.f, 0.f};
        if (act) {
            dc.re = cs.d[ci * NC * N + j];
            bc.re = cs.beta[ci * NC * N + j];
            if (NC == 2) { dc.im = cs.d[ci * NC * N + N + j]; bc.im = cs.beta[ci * NC * N + N + j]; }
            psh[j] = cs.pi[ci * N + j];
            cpx w = cmul(dc, beta);
            wsh[j] = w.re;
            if (NC == 2) wsh[N + j] = w.im;
            // stash d_c for the gather at pi
        }
        __syncthreads();
        if (act) {
            cpx acc{0.f, 0.f};
            for (int q = 0; q < N; ++q)
                if (psh[q] == j) { acc.re += wsh[q]; if (NC == 2) acc.im += wsh[N + q]; }
            const size_t cpi = ci * NC * N + pi;
            cpx dpi{cs.d[cpi], NC == 2 ? cs.d[cpi + N] : 0.f};
            d = cmul(dpi, d);
            pi = psh[pi];
            beta = cadd(acc, bc);
        }
        __syncthreads();
    }
    if (act) {
        out.pi(s)[j] = (uint16_t)pi;
        out.d(s)[j] = d.re;
        out.template beta<NC>(s, N)[j] = beta.re;
        if (NC == 2) {
            out.d(s)[N + j] = d.im;
            out.template beta<NC>(s, N)[N + j] = beta.im;
        }
    }
}

// carry into segment `rank`: carry = S_{rank-1} o ... o S_0 (h0); map likewise.
template <int NC>
__global__ void k_compose_carry(SummaryView sums, int rank, int S_per_rank, const float* __restrict__ h0,
                                float* __restrict__ carry_out, uint16_t* __restrict__ map_out, int N) {
    extern __shared__ float smem[];
    float* wsh = smem;
    uint16_t* psh = reinterpret_cast<uint16_t*>(smem + NC * N);
    const int s = blockIdx.x;
    const int j = threadIdx.x;
    const bool act = j < N;
    cpx cur{0.f, 0.f};
    if (act && h0) {
        cur.re = h0[(size_t)s * NC * N + j];
        if (NC == 2) cur.im = h0[(size_t)s * NC * N + N + j];
    }
    int m = j;
    for (int g = 0; g < rank; ++g) {
        const size_t blk = (size_t)g * S_per_rank + s;
        cpx dg{0.f, 0.f}, bg{0.f, 0.f};
        if (act) {
            dg.re = sums.d(blk)[j];
            bg.re = sums.template beta<NC>(blk, N)[j];
            if (NC == 2) { dg.im = sums.d(blk)[N + j]; bg.im = sums.template beta<NC>(blk, N)[N + j]; }
            psh[j] = sums.pi(blk)[j];
            cpx w = cmul(dg, cur);
            wsh[j] = w.re;
            if (NC == 2) wsh[N + j] = w.im;
        }
        __syncthreads();
        if (act) {
            cpx acc{0.f, 0.f};
            for (int q = 0; q < N; ++q)
                if (psh[q] == j) { acc.re += wsh[q]; if (NC == 2) acc.im += wsh[N + q]; }
            m = psh[m];
            cur = cadd(acc, bg);
        }
        __syncthreads();
    }
    if (act) {
        carry_out[(size_t)s * NC * N + j] = cur.re;
        if (NC == 2) carry_out[(size_t)s * NC * N + N + j] = cur.im;
        if (map_out) map_out[(size_t)s * N + j] = (uint16_t)m;
    }
}

// adjoint entering segment `rank`: mu = 0; for g = G-1 .. rank+1: mu = beta'_g + Abar_g^T mu
template <int NC>
__global__ void k_compose_lambda(SummaryView fwd, const float* __restrict__ beta_bwd, int rank, int G,
                                 int S_per_rank, float* __restrict__ lam_out, int N) {
    extern __shared__ float smem[];
    float* msh = smem;
    const int s = blockIdx.x;
    const int j = threadIdx.x;
    const bool act = j < N;
    cpx mu{0.f, 0.f};
    for (int g = G - 1; g > rank; --g) {
        const size_t blk = (size_t)g * S_per_rank + s;
        if (act) {
            msh[j] = mu.re;
            if (NC == 2) msh[N + j] = mu.im;
        }
        __syncthreads();
        if (act) {
            const int pj = fwd.pi(blk)[j];
            cpx dg{fwd.d(blk)[j], NC == 2 ? fwd.d(blk)[N + j] : 0.f};
            cpx bp{beta_bwd[blk * NC * N + j], NC == 2 ? beta_bwd[blk * NC * N + N + j] : 0.f};
            cpx mP{msh[pj], NC == 2 ? msh[N + pj] : 0.f};
            mu = cadd(bp, cmulc(dg, mP));
        }
        __syncthreads();
    }
    if (act) {
        lam_out[(size_t)s * NC * N + j] = mu.re;
        if (NC == 2) lam_out[(size_t)s * NC * N + N + j] = mu.im;
    }
}

}  // namespace pdssm
