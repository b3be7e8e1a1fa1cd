// a1 sparsification (Eq. 5; App. E.2.1) and the
// generic (SIMT) selection path (Eqs. 6-8).
// Every argmax: strict '>' while scanning ascending indices -> ties go to the
// smallest index, NaN never wins (treated as -inf), all-NaN -> 0 (readings R7, R8).
#pragma once
#include "pdssm_common.cuh"

namespace pdssm {

// dict_idx[h][k][j] = argmax_i M[h][k][i][j]; one CTA per (h,k), thread per column j
// (coalesced: for fixed i the warp reads a contiguous row segment).
static __global__ void k_sparsify(const float* __restrict__ M, uint16_t* __restrict__ dict_idx, int N, uint32_t flags) {
    const int e = blockIdx.x;
    const float* Me = M + (size_t)e * N * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        float best = -INFINITY;
        int arg = 0;
        for (int i = 0; i < N; ++i) {
            const float v = __ldg(Me + (size_t)i * N + j);
            if ((flags & PDSSM_CHECK_FINITE) && isnan(v)) report(ERRBIT_NONFINITE);
            if (v > best) {
                best = v;
                arg = i;
            }
        }
        dict_idx[(size_t)e * N + j] = (uint16_t)arg;
    }
}

// Selector logits, SIMT tiled GEMM: logits[(b,h,t)][k] = sum_d S[h][k][d] x[b][t][d].
// Tile 64 tokens x 64 (h,k) columns x 32 d; 256 threads, 4x4 outputs each.
// fp32 accumulation in ascending-d order of 32-wide slabs.
template <typename T>
__global__ void __launch_bounds__(256) k_select_logits_simt(const T* __restrict__ x, const T* __restrict__ S,
                                                            float* __restrict__ logits, int B, int L, int H,
                                                            int K, int d_in, uint32_t flags) {
    constexpr int TM = 64, TN = 64, TK = 32;
    __shared__ float xs[TK][TM + 4];
    __shared__ float ss[TK][TN + 4];
    const int M = B * L, NN = H * K;
    const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN;
    const int tid = threadIdx.x;
    const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
    float acc[4][4] = {};
    for (int d0 = 0; d0 < d_in; d0 += TK) {
        for (int q = tid; q < TM * TK; q += 256) {
            const int r = q / TK, dd = q % TK;
            const int m = m0 + r, d = d0 + dd;
            float v = 0.f;
            if (m < M && d < d_in) {
                v = ldact(x + (size_t)m * d_in + d);
                if ((flags & PDSSM_CHECK_FINITE) && !isfinite(v)) report(ERRBIT_NONFINITE);
            }
            xs[dd][r] = v;
        }
        for (int q = tid; q < TN * TK; q += 256) {
            const int r = q / TK, dd = q % TK;
            const int n = n0 + r, d = d0 + dd;
            float v = 0.f;
            if (n < NN && d < d_in) v = ldact(S + (size_t)n * d_in + d);
            ss[dd][r] = v;
        }
        __syncthreads();
#pragma unroll 8
        for (int dd = 0; dd < TK; ++dd) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = xs[dd][tm + i];
#pragma unroll
            for (int i = 0; i < 4; ++i) b[i] = ss[dd][tn + i];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(a[i], b[q], acc[i][q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + tm + i;
        if (m >= M) continue;
        const int b = m / L, t = m % L;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int n = n0 + tn + q;
            if (n >= NN) continue;
            const int h = n / K, k = n % K;
            logits[(((size_t)b * H + h) * L + t) * K + k] = acc[i][q];
        }
    }
}

// a5 generic path (shapes TMA cannot take): b[b][h][t][w] = sum_d x[b][t][d] Bw[h][w][d],
// w = (c, n); same SIMT tiling as the selector logits.
template <typename T>
__global__ void __launch_bounds__(256) k_project_simt(const T* __restrict__ x, const T* __restrict__ Bw,
                                                      T* __restrict__ out, int B, int L, int H, int cN, int d_in) {
    constexpr int TM = 64, TN = 64, TK = 32;
    __shared__ float xs[TK][TM + 4];
    __shared__ float ws[TK][TN + 4];
    const int M = B * L, NN = H * cN;
    const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN;
    const int tid = threadIdx.x;
    const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
    float acc[4][4] = {};
    for (int d0 = 0; d0 < d_in; d0 += TK) {
        for (int q = tid; q < TM * TK; q += 256) {
            const int r = q / TK, dd = q % TK;
            const int m = m0 + r, d = d0 + dd;
            xs[dd][r] = (m < M && d < d_in) ? ldact(x + (size_t)m * d_in + d) : 0.f;
        }
        for (int q = tid; q < TN * TK; q += 256) {
            const int r = q / TK, dd = q % TK;
            const int n = n0 + r, d = d0 + dd;
            ws[dd][r] = (n < NN && d < d_in) ? ldact(Bw + (size_t)n * d_in + d) : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int dd = 0; dd < TK; ++dd) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = xs[dd][tm + i];
#pragma unroll
            for (int i = 0; i < 4; ++i) b[i] = ws[dd][tn + i];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(a[i], b[q], acc[i][q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + tm + i;
        if (m >= M) continue;
        const int b = m / L, t = m % L;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int n = n0 + tn + q;
            if (n >= NN) continue;
            const int h = n / cN, w = n % cN;
            stact(out + (((size_t)b * H + h) * L + t) * cN + w, acc[i][q]);
        }
    }
}

// k*[b,h,t] = argmax_k logits (smallest index on ties, NaN never wins); optional P gather.
static __global__ void k_select_argmax(const float* __restrict__ logits, const uint16_t* __restrict__ dict_idx,
                                uint8_t* __restrict__ kstar, uint16_t* __restrict__ P, int64_t rows, int H, int L,
                                int N, int K) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;   // row = (b*H + h)*L + t
    if (r >= rows) return;
    const float* lg = logits + r * K;
    // warp-parallel argmax over K with lexicographic (value, -index) compare
    float best = -INFINITY;
    int arg = K;   // sentinel: no candidate yet
    for (int k = threadIdx.x; k < K; k += 32) {
        const float v = lg[k];
        if (v > best) {   // strict: NaN and -inf never become candidates
            best = v;
            arg = k;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (ob > best || (ob == best && oa < arg)) {
            best = ob;
            arg = oa;
        }
    }
    if (arg >= K) arg = 0;   // all NaN
    if (threadIdx.x == 0) kstar[r] = (uint8_t)arg;
    if (P) {
        const int h = (int)((r / L) % H);
        const uint16_t* src = dict_idx + ((size_t)h * K + arg) * N;
        for (int j = threadIdx.x; j < N; j += 32) P[r * N + j] = src[j];
    }
}

}  // namespace pdssm
