// Forward chunked scan, the three phases of Algorithm 1 (
// Kernels A/B/C PAPER.md:1020-1095) in the column-one-hot SCATTER convention
// (reading R1):  (A_t v)[i] = sum_{j : P_t[j] = i} D_t[j] v[j].
//
// The scatter is executed as a deterministic gather over a per-dictionary-entry
// preimage list ("plan"): target i sums v[j] over j in pre_k(i), ascending j
// (reading R17) -- no float atomics, bitwise run-to-run reproducible.
//
// One CTA per (sequence, chunk) item, one thread per state j (blockDim >= N),
// c = NC planes.  Generic path used for every shape; the fused single-pass
// kernel (k_scan_fused.cuh) is the fast path for the headline shapes.
#pragma once
#include "pdssm_common.cuh"

namespace pdssm {

struct ChunkStateView {
    uint16_t* pi;    // [S][C][N]
    float* d;        // [S][C][NC][N]
    float* beta;     // [S][C][NC][N]
    float* carry;    // [S][C][NC][N]
};

// ---------------------------------------------------------------------------
// plan: preimage lists of every dictionary entry (counting sort, deterministic)
//   pstart[e][i] = #{j : P[j] < i} (i = 0..N),  psrc[e][pstart[e][P[j]] + rank_j] = j
// with rank_j = #{j' < j : P[j'] = P[j]}; e = h*K + k.
// ---------------------------------------------------------------------------
static __global__ void k_build_plan(const uint16_t* __restrict__ dict_idx, uint16_t* __restrict__ pstart,
                             uint16_t* __restrict__ psrc, int N, uint32_t flags) {
    extern __shared__ uint16_t sP[];
    const int e = blockIdx.x;
    const uint16_t* P = dict_idx + (size_t)e * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        uint16_t p = P[j];
        if (p >= N) {
            if (flags & PDSSM_CHECK_FINITE) report(ERRBIT_RANGE);
            p = (uint16_t)(N - 1);
        }
        sP[j] = p;
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= N; i += blockDim.x) {
        int cnt = 0;
        for (int j = 0; j < N; ++j) cnt += (sP[j] < i);
        pstart[(size_t)e * (N + 1) + i] = (uint16_t)cnt;
    }
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        const int pj = sP[j];
        int pos = 0;
        for (int q = 0; q < N; ++q) pos += (sP[q] < pj) || (sP[q] == pj && q < j);
        psrc[(size_t)e * N + pos] = (uint16_t)j;
    }
}

__device__ __forceinline__ int load_k(const uint8_t* kstar, size_t idx, int K, uint32_t flags) {
    int k = __ldg(kstar + idx);
    if (k >= K) {
        if (flags & PDSSM_CHECK_FINITE) report(ERRBIT_RANGE);
        k = K - 1;
    }
    return k;
}

__device__ __forceinline__ int clamp_idx(int p, int N, uint32_t flags) {
    if (p >= N) {
        if (flags & PDSSM_CHECK_FINITE) report(ERRBIT_RANGE);
        p = N - 1;
    }
    return p;
}

template <typename T, int NC, bool PERDICT>
__device__ __forceinline__ cpx load_diag(const T* diag, const float* diag_dict, size_t step_off, int h, int k,
                                         int K, int N, int j) {
    cpx r{0.f, 0.f};
    if (PERDICT) {
        const float* p = diag_dict + ((size_t)(h * K + k) * NC) * N + j;
        r.re = __ldg(p);
        if (NC == 2) r.im = __ldg(p + N);
    } else {
        const T* p = diag + step_off + j;
        r.re = ldact(p);
        if (NC == 2) r.im = ldact(p + N);
    }
    return r;
}

template <typename T, int NC>
__device__ __forceinline__ cpx load_plane(const T* base, size_t step_off, int N, int j) {
    cpx r{0.f, 0.f};
    const T* p = base + step_off + j;
    r.re = ldact(p);
    if (NC == 2) r.im = ldact(p + N);
    return r;
}

__device__ __forceinline__ void check_cpx(cpx v, uint32_t flags) {
    if ((flags & PDSSM_CHECK_FINITE) && !(finite_f(v.re) && finite_f(v.im))) report(ERRBIT_NONFINITE);
}

// One scatter step  out = A_t v + b  executed as a gather over the preimage list.
//   vsh: this step's v = D_t (.) state for all j (smem, already synchronised)
template <int NC>
__device__ __forceinline__ cpx scatter_gather(const float* vsh, const uint16_t* __restrict__ pstart,
                                              const uint16_t* __restrict__ psrc, int e, int N, int i) {
    const int st = __ldg(pstart + (size_t)e * (N + 1) + i);
    const int en = __ldg(pstart + (size_t)e * (N + 1) + i + 1);
    cpx acc{0.f, 0.f};
    for (int q = st; q < en; ++q) {
        const int j = __ldg(psrc + (size_t)e * N + q);
        acc.re += vsh[j];
        if (NC == 2) acc.im += vsh[N + j];
    }
    return acc;
}

// ---------------------------------------------------------------------------
// Phase A: per (sequence, chunk) aggregate from identity (PAPER.md:883-896,
// Kernel A PAPER.md:1020-1046):  pi <- P_t[pi], d <- D_t[pi_old] d,
// beta <- A_t beta + b_t.
// ---------------------------------------------------------------------------
template <typename T, int NC, bool PERDICT>
__global__ void k_fwd_phaseA(const uint8_t* __restrict__ kstar, const uint16_t* __restrict__ dict_idx,
                             const uint16_t* __restrict__ pstart, const uint16_t* __restrict__ psrc,
                             const T* __restrict__ diag, const float* __restrict__ diag_dict,
                             const T* __restrict__ bias, ChunkStateView cs, int H, int L, int N, int K,
                             int tau, int C_ch, uint32_t flags) {
    extern __shared__ float smem[];
    float* Dsh = smem;                 // [2][NC][N]
    float* vsh = smem + 2 * NC * N;    // [2][NC][N]
    const int item = blockIdx.x;
    const int s = item / C_ch, c = item % C_ch, h = s % H;
    const int t0 = c * tau, t1 = min(t0 + tau, L);
    const int j = threadIdx.x;
    const bool act = j < N;
    int pi = act ? j : 0;
    cpx d{1.f, 0.f}, beta{0.f, 0.f};
    for (int t = t0; t < t1; ++t) {
        const int buf = (t - t0) & 1;
        const int k = load_k(kstar, (size_t)s * L + t, K, flags);
        const size_t off = ((size_t)s * L + t) * NC * N;
        float* D_b = Dsh + buf * NC * N;
        float* v_b = vsh + buf * NC * N;
        cpx bj{0.f, 0.f};
        if (act) {
            cpx Dj = load_diag<T, NC, PERDICT>(diag, diag_dict, off, h, k, K, N, j);
            bj = load_plane<T, NC>(bias, off, N, j);
            check_cpx(Dj, flags);
            check_cpx(bj, flags);
            cpx v = cmul(Dj, beta);
            D_b[j] = Dj.re;
            v_b[j] = v.re;
            if (NC == 2) { D_b[N + j] = Dj.im; v_b[N + j] = v.im; }
        }
        __syncthreads();
        if (act) {
            cpx Dpi{D_b[pi], NC == 2 ? D_b[N + pi] : 0.f};
            d = cmul(Dpi, d);
            pi = clamp_idx(__ldg(dict_idx + (size_t)(h * K + k) * N + pi), N, flags);
            cpx acc = scatter_gather<NC>(v_b, pstart, psrc, h * K + k, N, j);
            beta = cadd(acc, bj);
        }
    }
    if (act) {
        const size_t ci = (size_t)s * C_ch + c;
        cs.pi[ci * N + j] = (uint16_t)pi;
        cs.d[ci * NC * N + j] = d.re;
        cs.beta[ci * NC * N + j] = beta.re;
        if (NC == 2) {
            cs.d[ci * NC * N + N + j] = d.im;
            cs.beta[ci * NC * N + N + j] = beta.im;
        }
    }
}

// ---------------------------------------------------------------------------
// Phase B: carry chain per sequence (Kernel B :1069-1081)
//   carry_0 = h0 (reading R5), carry_{c+1} = Abar_c carry_c + beta_bar_c,
//   maps: Pi_0 = id, Pi_{c+1} = pi_bar_c[Pi_c].
// The collision-heavy scatter with pi_bar is summed in ascending j.
// ---------------------------------------------------------------------------
template <int NC>
__global__ void k_fwd_phaseB(ChunkStateView cs, const float* __restrict__ h0, uint16_t* __restrict__ maps,
                             float* __restrict__ final_out, int N, int C_ch) {
    extern __shared__ float smem[];
    float* wsh = smem;                                   // [NC][N]
    uint16_t* psh = reinterpret_cast<uint16_t*>(smem + NC * N);   // [N]
    const int s = blockIdx.x;
    const int j = threadIdx.x;
    const bool act = j < N;
    cpx carry{0.f, 0.f};
    if (act && h0) {
        carry.re = h0[(size_t)s * NC * N + j];
        if (NC == 2) carry.im = h0[(size_t)s * NC * N + N + j];
    }
    int m = j;
    for (int c = 0; c < C_ch; ++c) {
        const size_t ci = (size_t)s * C_ch + c;
        cpx db{0.f, 0.f}, bb{0.f, 0.f};
        if (act) {
            cs.carry[ci * NC * N + j] = carry.re;
            if (NC == 2) cs.carry[ci * NC * N + N + j] = carry.im;
            if (maps) maps[((size_t)s * (C_ch + 1) + c) * N + j] = (uint16_t)m;
            db.re = cs.d[ci * NC * N + j];
            bb.re = cs.beta[ci * NC * N + j];
            if (NC == 2) { db.im = cs.d[ci * NC * N + N + j]; bb.im = cs.beta[ci * NC * N + N + j]; }
            cpx w = cmul(db, carry);
            wsh[j] = w.re;
            if (NC == 2) wsh[N + j] = w.im;
            psh[j] = cs.pi[ci * N + j];
        }
        __syncthreads();
        if (act) {
            cpx acc{0.f, 0.f};
            for (int q = 0; q < N; ++q) {
                if (psh[q] == j) {
                    acc.re += wsh[q];
                    if (NC == 2) acc.im += wsh[N + q];
                }
            }
            m = psh[m];
            carry = cadd(acc, bb);
        }
        __syncthreads();
    }
    if (act) {
        if (maps) maps[((size_t)s * (C_ch + 1) + C_ch) * N + j] = (uint16_t)m;
        if (final_out) {
            final_out[(size_t)s * NC * N + j] = carry.re;
            if (NC == 2) final_out[(size_t)s * NC * N + N + j] = carry.im;
        }
    }
}

// ---------------------------------------------------------------------------
// Phase C: replay each chunk from its carry (PAPER.md:905-913 in the replay
// form of Kernel C; reading R10) and write h_t.
// ---------------------------------------------------------------------------
template <typename T, int NC, bool PERDICT>
__global__ void k_fwd_phaseC(const uint8_t* __restrict__ kstar, const uint16_t* __restrict__ pstart,
                             const uint16_t* __restrict__ psrc, const T* __restrict__ diag,
                             const float* __restrict__ diag_dict, const T* __restrict__ bias,
                             ChunkStateView cs, T* __restrict__ hout, int H, int L, int N, int K, int tau,
                             int C_ch, uint32_t flags) {
    extern __shared__ float smem[];
    float* vsh = smem;  // [2][NC][N]
    const int item = blockIdx.x;
    const int s = item / C_ch, c = item % C_ch, h = s % H;
    const int t0 = c * tau, t1 = min(t0 + tau, L);
    const int j = threadIdx.x;
    const bool act = j < N;
    cpx cur{0.f, 0.f};
    const size_t ci = (size_t)s * C_ch + c;
    if (act) {
        cur.re = cs.carry[ci * NC * N + j];
        if (NC == 2) cur.im = cs.carry[ci * NC * N + N + j];
    }
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
            cpx acc = scatter_gather<NC>(v_b, pstart, psrc, h * K + k, N, j);
            cur = cadd(acc, bj);
            stact(hout + off + j, cur.re);
            if (NC == 2) stact(hout + off + N + j, cur.im);
        }
    }
}

// ---------------------------------------------------------------------------
// Readout y_t = Re(C_h h_t) (Eq. 1 with psi = Re).
//   h [B][H][L][NC][N] (act), C f32 [H][NC][P][N], y act [B][L][H][P]
// one CTA per (b, h, t); thread p.
// ---------------------------------------------------------------------------
template <typename T, int NC>
__global__ void k_readout(const T* __restrict__ hs, const float* __restrict__ Cw, T* __restrict__ y, int H,
                          int L, int N, int P) {
    extern __shared__ float smem[];
    const int t = blockIdx.x % L;
    const int s = blockIdx.x / L;
    const int h = s % H, b = s / H;
    const size_t off = ((size_t)s * L + t) * NC * N;
    for (int q = threadIdx.x; q < NC * N; q += blockDim.x) smem[q] = ldact(hs + off + q);
    __syncthreads();
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
        const float* cre = Cw + ((size_t)(h * NC) * P + p) * N;
        float acc = 0.f;
        for (int j = 0; j < N; ++j) acc += __ldg(cre + j) * smem[j];
        if (NC == 2) {
            const float* cim = Cw + ((size_t)(h * NC + 1) * P + p) * N;
            for (int j = 0; j < N; ++j) acc -= __ldg(cim + j) * smem[N + j];
        }
        stact(y + (((size_t)b * L + t) * H + h) * P + p, acc);
    }
}

}  // namespace pdssm
