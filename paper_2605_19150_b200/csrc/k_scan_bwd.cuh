// Backward (reverse, transposed) chunked scan.  The paper gives no backward
// kernel (only App. C PAPER.md:818-823 and Prop. 2); this is
// the transposed Algorithm 1:
//   lambda_{t-1} = e_{t-1} + A_t^T lambda_t,  (A_t^T mu)[j] = conj(D_t[j]) mu[P_t[j]]
// which is a pure gather -- no collisions.  Chunk summaries:
//   Phase A': beta'_c = A_{s_c}^T lambda_loc_{s_c}   (reverse local scan, zero incoming)
//   Phase B': mu_{C-1} = lam_in, mu_{c-1} = beta'_c + Abar_c^T mu_c  (forward (pi_bar, d_bar) reused)
//   Phase C': replay lambda from e_{e_c} + mu_c, emit db, dD, g.
#pragma once
#include "k_scan_fwd.cuh"

namespace pdssm {

template <typename TE, int NC>
__device__ __forceinline__ cpx load_e(const TE* e, size_t off, int N, int j) {
    if (e == nullptr) return cpx{0.f, 0.f};
    return load_plane<TE, NC>(e, off, N, j);
}

// Phase A': reverse local scan of chunk c from zero incoming adjoint.
template <typename T, typename TE, int NC, bool PERDICT>
__global__ void k_bwd_phaseA(const uint8_t* __restrict__ kstar, const uint16_t* __restrict__ dict_idx,
                             const T* __restrict__ diag, const float* __restrict__ diag_dict,
                             const TE* __restrict__ e, float* __restrict__ betap, int H, int L, int N, int K,
                             int tau, int C_ch) {
    extern __shared__ float smem[];
    float* lsh = smem;  // [2][NC][N]
    const int item = blockIdx.x;
    const int s = item / C_ch, c = item % C_ch, h = s % H;
    const int t0 = c * tau, t1 = min(t0 + tau, L);
    const int j = threadIdx.x;
    const bool act = j < N;
    cpx lam{0.f, 0.f};
    if (act) lam = load_e<TE, NC>(e, ((size_t)s * L + (t1 - 1)) * NC * N, N, j);
    for (int t = t1 - 1; t >= t0; --t) {
        const int buf = (t1 - 1 - t) & 1;
        float* l_b = lsh + buf * NC * N;
        if (act) {
            l_b[j] = lam.re;
            if (NC == 2) l_b[N + j] = lam.im;
        }
        __syncthreads();
        if (act) {
            const int k = load_k(kstar, (size_t)s * L + t, K, 0);
            const size_t off = ((size_t)s * L + t) * NC * N;
            const int pj = clamp_idx(__ldg(dict_idx + (size_t)(h * K + k) * N + j), N, 0);
            cpx lamP{l_b[pj], NC == 2 ? l_b[N + pj] : 0.f};
            cpx Dj = load_diag<T, NC, PERDICT>(diag, diag_dict, off, h, k, K, N, j);
            cpx back = cmulc(Dj, lamP);
            if (t > t0) {
                lam = cadd(load_e<TE, NC>(e, off - (size_t)NC * N, N, j), back);
            } else {
                const size_t ci = (size_t)s * C_ch + c;
                betap[ci * NC * N + j] = back.re;
                if (NC == 2) betap[ci * NC * N + N + j] = back.im;
            }
        }
    }
}

// Phase B': reverse carry chain per sequence (mu_{c-1} for c >= 1).  With dh0 given it also
// takes the final step dh0 = beta'_0 + Abar_0^T mu_0 (pdssm_segment_summary_bwd's beta'; the full
// backward instead takes dh0 from the chunk-0 replay of Phase C', so it never reads Abar_0).
template <int NC>
__global__ void k_bwd_phaseB(ChunkStateView cs, const float* __restrict__ betap, const float* __restrict__ lam_in,
                             float* __restrict__ mu_out, float* __restrict__ dh0, int N, int C_ch) {
    extern __shared__ float smem[];
    float* msh = smem;  // [NC][N]
    const int s = blockIdx.x;
    const int j = threadIdx.x;
    const bool act = j < N;
    cpx mu{0.f, 0.f};
    if (act && lam_in) {
        mu.re = lam_in[(size_t)s * NC * N + j];
        if (NC == 2) mu.im = lam_in[(size_t)s * NC * N + N + j];
    }
    const int c_last = dh0 ? 0 : 1;
    for (int c = C_ch - 1; c >= 0; --c) {
        const size_t ci = (size_t)s * C_ch + c;
        if (act) {
            mu_out[ci * NC * N + j] = mu.re;
            if (NC == 2) mu_out[ci * NC * N + N + j] = mu.im;
            msh[j] = mu.re;
            if (NC == 2) msh[N + j] = mu.im;
        }
        __syncthreads();
        if (c < c_last) break;
        if (act) {
            cpx bp{betap[ci * NC * N + j], NC == 2 ? betap[ci * NC * N + N + j] : 0.f};
            if (c == C_ch - 1 && !lam_in) {
                mu = bp;   // mu_{C-1} = 0: the Abar^T term vanishes (and the aggregate is not read)
            } else {
                const int pj = min((int)cs.pi[ci * N + j], N - 1);
                cpx db{cs.d[ci * NC * N + j], NC == 2 ? cs.d[ci * NC * N + N + j] : 0.f};
                cpx mP{msh[pj], NC == 2 ? msh[N + pj] : 0.f};
                mu = cadd(bp, cmulc(db, mP));
            }
        }
        __syncthreads();
    }
    if (act && dh0) {
        dh0[(size_t)s * NC * N + j] = mu.re;
        if (NC == 2) dh0[(size_t)s * NC * N + N + j] = mu.im;
    }
}

// Phase C': replay lambda from e_{e_c} + mu_c and emit the gradients.
//   db_t = lambda_t, dD_t[j] = conj(h_{t-1}[j]) lambda_t[P_t[j]],
//   g_t = sum_j Re(conj(lambda_t[P_t[j]]) D_t[j] h_{t-1}[j])   (warp shuffles +
//   per-warp partials summed in warp order: deterministic)
template <typename T, typename TE, int NC, bool PERDICT>
__global__ void k_bwd_phaseC(const uint8_t* __restrict__ kstar, const uint16_t* __restrict__ dict_idx,
                             const T* __restrict__ diag, const float* __restrict__ diag_dict,
                             const T* __restrict__ hsaved, const float* __restrict__ h0,
                             const TE* __restrict__ e, const float* __restrict__ mu_in, T* __restrict__ dbias,
                             T* __restrict__ ddiag, float* __restrict__ ddiag_f32, float* __restrict__ gsel,
                             float* __restrict__ dh0, int H, int L, int N, int K, int tau, int C_ch) {
    extern __shared__ float smem[];
    const int nw = blockDim.x / 32;
    float* lsh = smem;                   // [2][NC][N]
    float* gpart = smem + 2 * NC * N;    // ring [64][nw] of per-warp partials of g
    const int item = blockIdx.x;
    const int s = item / C_ch, c = item % C_ch, h = s % H;
    const int t0 = c * tau, t1 = min(t0 + tau, L);
    const int j = threadIdx.x;
    const int lane = j & 31, w = j >> 5;
    const bool act = j < N;
    const size_t ci = (size_t)s * C_ch + c;
    cpx lam{0.f, 0.f};
    if (act) {
        lam = load_e<TE, NC>(e, ((size_t)s * L + (t1 - 1)) * NC * N, N, j);
        lam.re += mu_in[ci * NC * N + j];
        if (NC == 2) lam.im += mu_in[ci * NC * N + N + j];
    }
    for (int t = t1 - 1; t >= t0; --t) {
        const int buf = (t1 - 1 - t) & 1;
        float* l_b = lsh + buf * NC * N;
        const size_t off = ((size_t)s * L + t) * NC * N;
        if (act) {
            l_b[j] = lam.re;
            if (NC == 2) l_b[N + j] = lam.im;
            stact(dbias + off + j, lam.re);
            if (NC == 2) stact(dbias + off + N + j, lam.im);
        }
        __syncthreads();
        const int q = t1 - 1 - t;            // reverse step count within the chunk
        if (gsel && q > 0 && (q & 31) == 0 && j < 32) {
            // flush steps [q-32, q): their partials were written before this barrier
            const int qq = q - 32 + j;
            float acc = 0.f;
            for (int ww = 0; ww < nw; ++ww) acc += gpart[(qq & 63) * nw + ww];
            gsel[(size_t)s * L + (t1 - 1 - qq)] = acc;
        }
        float gval = 0.f;
        if (act) {
            const int k = load_k(kstar, (size_t)s * L + t, K, 0);
            const int pj = clamp_idx(__ldg(dict_idx + (size_t)(h * K + k) * N + j), N, 0);
            cpx lamP{l_b[pj], NC == 2 ? l_b[N + pj] : 0.f};
            cpx Dj = load_diag<T, NC, PERDICT>(diag, diag_dict, off, h, k, K, N, j);
            cpx hp{0.f, 0.f};
            if (t > 0) {
                hp = load_plane<T, NC>(hsaved, off - (size_t)NC * N, N, j);
            } else if (h0) {
                hp.re = h0[(size_t)s * NC * N + j];
                if (NC == 2) hp.im = h0[(size_t)s * NC * N + N + j];
            }
            cpx dD = cmulc(hp, lamP);
            if (PERDICT) {
                ddiag_f32[off + j] = dD.re;
                if (NC == 2) ddiag_f32[off + N + j] = dD.im;
            } else {
                stact(ddiag + off + j, dD.re);
                if (NC == 2) stact(ddiag + off + N + j, dD.im);
            }
            cpx prod = cmul(Dj, hp);
            gval = lamP.re * prod.re + lamP.im * prod.im;
            if (t > t0) lam = cadd(load_e<TE, NC>(e, off - (size_t)NC * N, N, j), cmulc(Dj, lamP));
            else if (t == 0 && dh0) {   // chunk 0 ends at t = 0: dh0 = A_0^T lambda_0 (no e_{-1})
                const cpx d0 = cmulc(Dj, lamP);
                dh0[(size_t)s * NC * N + j] = d0.re;
                if (NC == 2) dh0[(size_t)s * NC * N + N + j] = d0.im;
            }
        }
        for (int o = 16; o > 0; o >>= 1) gval += __shfl_xor_sync(0xffffffffu, gval, o);
        if (lane == 0) gpart[(q & 63) * nw + w] = gval;
    }
    __syncthreads();
    if (gsel) {
        const int nsteps = t1 - t0;
        const int qlast = ((nsteps - 1) / 32) * 32;
        for (int qq = qlast + j; qq < nsteps; qq += blockDim.x) {
            float acc = 0.f;
            for (int ww = 0; ww < nw; ++ww) acc += gpart[(qq & 63) * nw + ww];
            gsel[(size_t)s * L + (t1 - 1 - qq)] = acc;
        }
    }
}

// Phase C' in recompute mode (pdssm_scan_bwd with h_saved_opt = NULL; include/pdssm.h):
// the forward states are not kept between the passes.  Each (sequence, chunk) item first
// replays its chunk forward from the chunk's carry (Alg. 1 Phase C: the
// carries in chunk_state are the only O(C N) state the forward leaves), h_t -> shared memory
// (tau x c x N f32), then runs the reverse pass of k_bwd_phaseC reading h_{t-1} from there
// (h_{s_c - 1} = carry_c, which is h0 at c = 0).  Same gradients, no O(L N) activation memory.
template <typename T, typename TE, int NC, bool PERDICT>
__global__ void k_bwd_phaseC_rc(const uint8_t* __restrict__ kstar, const uint16_t* __restrict__ dict_idx,
                                const uint16_t* __restrict__ pstart, const uint16_t* __restrict__ psrc,
                                const T* __restrict__ diag, const float* __restrict__ diag_dict,
                                const T* __restrict__ bias, ChunkStateView cs, const TE* __restrict__ e,
                                const float* __restrict__ mu_in, T* __restrict__ dbias, T* __restrict__ ddiag,
                                float* __restrict__ ddiag_f32, float* __restrict__ gsel, float* __restrict__ dh0, int H, int L, int N, int K,
                                int tau, int C_ch) {
    extern __shared__ float smem[];
    const int nw = blockDim.x / 32;
    float* vsh = smem;                          // [2][NC][N]: forward exchange, then lambda rows
    float* gpart = smem + 2 * NC * N;           // ring [64][nw] of per-warp partials of g
    float* hbuf = gpart + 64 * nw;              // [tau][NC][N] recomputed states of this chunk
    const int item = blockIdx.x;
    const int s = item / C_ch, c = item % C_ch, h = s % H;
    const int t0 = c * tau, t1 = min(t0 + tau, L);
    const int j = threadIdx.x;
    const int lane = j & 31, w = j >> 5;
    const bool act = j < N;
    const size_t ci = (size_t)s * C_ch + c;
    cpx carry{0.f, 0.f};
    if (act) {
        carry.re = cs.carry[ci * NC * N + j];
        if (NC == 2) carry.im = cs.carry[ci * NC * N + N + j];
    }
    // ---- forward replay of the chunk (the scatter as a gather over the preimage plan)
    {
        cpx cur = carry;
        for (int t = t0; t < t1; ++t) {
            const int buf = (t - t0) & 1;
            const int k = load_k(kstar, (size_t)s * L + t, K, 0);
            const size_t off = ((size_t)s * L + t) * NC * N;
            float* v_b = vsh + buf * NC * N;
            cpx bj{0.f, 0.f};
            if (act) {
                cpx Dj = load_diag<T, NC, PERDICT>(diag, diag_dict, off, h, k, K, N, j);
                bj = load_plane<T, NC>(bias, off, N, j);
                cpx v = cmul(Dj, cur);
                v_b[j] = v.re;
                if (NC == 2) v_b[N + j] = v.im;
            }
            __syncthreads();
            if (act) {
                cur = cadd(scatter_gather<NC>(v_b, pstart, psrc, h * K + k, N, j), bj);
                float* hr = hbuf + (size_t)(t - t0) * NC * N;
                hr[j] = cur.re;
                if (NC == 2) hr[N + j] = cur.im;
            }
        }
        __syncthreads();   // the exchange rows are reused by the reverse pass
    }
    // ---- reverse pass (k_bwd_phaseC with h_{t-1} from hbuf)
    cpx lam{0.f, 0.f};
    if (act) {
        lam = load_e<TE, NC>(e, ((size_t)s * L + (t1 - 1)) * NC * N, N, j);
        lam.re += mu_in[ci * NC * N + j];
        if (NC == 2) lam.im += mu_in[ci * NC * N + N + j];
    }
    for (int t = t1 - 1; t >= t0; --t) {
        const int buf = (t1 - 1 - t) & 1;
        float* l_b = vsh + buf * NC * N;
        const size_t off = ((size_t)s * L + t) * NC * N;
        if (act) {
            l_b[j] = lam.re;
            if (NC == 2) l_b[N + j] = lam.im;
            stact(dbias + off + j, lam.re);
            if (NC == 2) stact(dbias + off + N + j, lam.im);
        }
        __syncthreads();
        const int q = t1 - 1 - t;
        if (gsel && q > 0 && (q & 31) == 0 && j < 32) {
            const int qq = q - 32 + j;
            float acc = 0.f;
            for (int ww = 0; ww < nw; ++ww) acc += gpart[(qq & 63) * nw + ww];
            gsel[(size_t)s * L + (t1 - 1 - qq)] = acc;
        }
        float gval = 0.f;
        if (act) {
            const int k = load_k(kstar, (size_t)s * L + t, K, 0);
            const int pj = clamp_idx(__ldg(dict_idx + (size_t)(h * K + k) * N + j), N, 0);
            cpx lamP{l_b[pj], NC == 2 ? l_b[N + pj] : 0.f};
            cpx Dj = load_diag<T, NC, PERDICT>(diag, diag_dict, off, h, k, K, N, j);
            cpx hp = carry;
            if (t > t0) {
                const float* hr = hbuf + (size_t)(t - 1 - t0) * NC * N;
                hp.re = hr[j];
                hp.im = NC == 2 ? hr[N + j] : 0.f;
            }
            cpx dD = cmulc(hp, lamP);
            if (PERDICT) {
                ddiag_f32[off + j] = dD.re;
                if (NC == 2) ddiag_f32[off + N + j] = dD.im;
            } else {
                stact(ddiag + off + j, dD.re);
                if (NC == 2) stact(ddiag + off + N + j, dD.im);
            }
            cpx prod = cmul(Dj, hp);
            gval = lamP.re * prod.re + lamP.im * prod.im;
            if (t > t0) lam = cadd(load_e<TE, NC>(e, off - (size_t)NC * N, N, j), cmulc(Dj, lamP));
            else if (t == 0 && dh0) {   // chunk 0 ends at t = 0: dh0 = A_0^T lambda_0 (no e_{-1})
                const cpx d0 = cmulc(Dj, lamP);
                dh0[(size_t)s * NC * N + j] = d0.re;
                if (NC == 2) dh0[(size_t)s * NC * N + N + j] = d0.im;
            }
        }
        for (int o = 16; o > 0; o >>= 1) gval += __shfl_xor_sync(0xffffffffu, gval, o);
        if (lane == 0) gpart[(q & 63) * nw + w] = gval;
    }
    __syncthreads();
    if (gsel) {
        const int nsteps = t1 - t0;
        const int qlast = ((nsteps - 1) / 32) * 32;
        for (int qq = qlast + j; qq < nsteps; qq += blockDim.x) {
            float acc = 0.f;
            for (int ww = 0; ww < nw; ++ww) acc += gpart[(qq & 63) * nw + ww];
            gsel[(size_t)s * L + (t1 - 1 - qq)] = acc;
        }
    }
}

// shared memory of k_bwd_phaseC_rc (host and device agree)
__host__ __device__ inline size_t rc_smem_bytes(int tau, int nc, int N, int threads) {
    return ((size_t)2 * nc * N + (size_t)64 * (threads / 32) + (size_t)tau * nc * N) * 4;
}

// e_t = dh_t + conj(C_h)^T dy_t  (readout adjoint, reading R13) into f32 scratch.
template <typename T, int NC>
__global__ void k_bwd_prepare_e(const T* __restrict__ dh, const T* __restrict__ dy, const float* __restrict__ Cw,
                                float* __restrict__ e, int H, int L, int N, int P) {
    extern __shared__ float smem[];
    const int t = blockIdx.x % L;
    const int s = blockIdx.x / L;
    const int h = s % H, b = s / H;
    for (int p = threadIdx.x; p < P; p += blockDim.x) smem[p] = dy ? ldact(dy + (((size_t)b * L + t) * H + h) * P + p) : 0.f;
    __syncthreads();
    const size_t off = ((size_t)s * L + t) * NC * N;
    for (int q = threadIdx.x; q < NC * N; q += blockDim.x) {
        const int pl = q / N, j = q % N;
        float acc = dh ? ldact(dh + off + q) : 0.f;
        if (dy) {
            const float* cp = Cw + ((size_t)(h * NC + pl) * P) * N + j;
            float sgn = pl == 0 ? 1.f : -1.f;   // conj(C): re part +, im part -
            for (int p = 0; p < P; ++p) acc += sgn * __ldg(cp + (size_t)p * N) * smem[p];
        }
        e[off + q] = acc;
    }
}

// PER_DICT: ddiag[h][k][pl][j] = sum over (b, t) with k*[b,h,t] = k of dD (fixed order).
// PER_DICT: dD_k = sum over the steps that selected entry k of the per-step dD_t (f32 scratch),
// deterministically in two stages.  Stage 1: one CTA per (sequence, slice of RD_SLICE steps,
// tile of RD_COLS columns of the c N plane); thread q owns column q and accumulates per entry
// in shared memory (its own column: no conflicts), ascending t.  Stage 2: one thread per (h, k,
// column) sums the partials over (b, slice) in ascending order.
constexpr int RD_SLICE = 512;
constexpr int RD_COLS = 128;

inline size_t reduce_dict_ws_bytes(int64_t S, int64_t L, int64_t K, int64_t cN) {
    const int64_t ns = (L + RD_SLICE - 1) / RD_SLICE;
    return (((size_t)S * ns * K * cN * 4) + 255) & ~(size_t)255;
}

static __global__ void __launch_bounds__(RD_COLS) k_reduce_dict_partial(const uint8_t* __restrict__ kstar,
                                                                 const float* __restrict__ dD,
                                                                 float* __restrict__ part, int L, int K, int cN) {
    extern __shared__ float acc[];   // [K][RD_COLS]
    const int ns = (L + RD_SLICE - 1) / RD_SLICE;
    const int ntile = (cN + RD_COLS - 1) / RD_COLS;
    const int tile = blockIdx.x % ntile;
    const int sl = (blockIdx.x / ntile) % ns;
    const size_t s = blockIdx.x / ((size_t)ntile * ns);
    const int q = tile * RD_COLS + threadIdx.x;
    const bool act = q < cN;
    for (int k = 0; k < K; ++k) acc[k * RD_COLS + threadIdx.x] = 0.f;
    const int t0 = sl * RD_SLICE, t1 = min(t0 + RD_SLICE, L);
    if (act) {
        const float* src = dD + ((size_t)s * L + t0) * cN + q;
        for (int t = t0; t < t1; ++t, src += cN) {
            int k = __ldg(kstar + (size_t)s * L + t);
            if (k >= K) k = K - 1;
            acc[k * RD_COLS + threadIdx.x] += __ldg(src);
        }
    }
    if (act) {
        float* dst = part + (((size_t)s * ns + sl) * K) * cN + q;
        for (int k = 0; k < K; ++k) dst[(size_t)k * cN] = acc[k * RD_COLS + threadIdx.x];
    }
}

static __global__ void k_reduce_dict_final(const float* __restrict__ part, float* __restrict__ ddiag, int B, int H, int L, int K,
                                    int cN) {
    const int ns = (L + RD_SLICE - 1) / RD_SLICE;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // over H * K * cN
    if (idx >= (int64_t)H * K * cN) return;
    const int q = (int)(idx % cN);
    const int k = (int)((idx / cN) % K);
    const int h = (int)(idx / ((int64_t)cN * K));
    float acc = 0.f;
    for (int b = 0; b < B; ++b) {
        const size_t s = (size_t)b * H + h;
        for (int sl = 0; sl < ns; ++sl) acc += part[(((size_t)s * ns + sl) * K + k) * cN + q];
    }
    ddiag[idx] = acc;
}


}  // namespace pdssm
