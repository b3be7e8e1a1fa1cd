// NEXT-1: Prop. 2 surrogate gradients (App. C).
// Slope-annealed straight-through estimation: each hardmax of the forward is a tempered
// softmax in the backward.  Both consume the backward scan's outputs:
//
//   selector   dlogits[b,h,t,k] = g_t s_{k*} (delta_{k,k*} - s_k) / T,  s = softmax_T(logits[b,h,t,:])
//              (g_t = gsel of pdssm_scan_bwd, reading R14)
//   dictionary G[h,k,i,j] = sum_{b,t: k*=k} Re(conj(lambda_t[i]) (D_t h_{t-1})[j])
//              dM[h,k,:,j] = (diag sigma_j - sigma_j sigma_j^T) / T  G[h,k,:,j],
//              sigma_j = softmax_T(M[h,k,:,j])   (column-wise; reading A15)
//
// The dictionary outer-product sum is the one dense contraction of the backward: per
// (h, k) a 128 x 128 x (c * #steps selecting k) GEMM with the K dimension gathered from the
// steps that selected k.  k_dict_grad_tc runs it on tcgen05 (kind::tf32, 3xTF32 split,
// fp32 accumulator in TMEM): every CTA streams its head's k* row in order, compacts the
// positions selecting its entry (a stable, deterministic order), stages each batch of rows
// straight into the K-major SWIZZLE_128B operand layout (lambda as A with the state index i
// as the M row; w = D (.) h_{t-1} as B with j as the N row; K = (step, plane)), and one
// thread issues the MMAs while the other threads stage the next batch (two buffers).
// The softmax Jacobian runs in the epilogue (TMEM -> shared tile -> one thread per column).
#pragma once
#include "pdssm_common.cuh"
#include "k_gemm_tc.cuh"

namespace pdssm {
namespace sg {

// ----------------------------------------------------------------------------- selector
// one warp per SG_ROWS consecutive (b, h, t) rows of K <= 256 logits, held in registers
// (lane owns k = lane + 32 m); all rows' loads are issued before any reduction.
constexpr int SG_ROWS = 4;
template <int KM>   // ceil(K / 32) logits per lane
__global__ void k_select_grad(const float* __restrict__ logits, const uint8_t* __restrict__ kstar,
                              const float* __restrict__ gsel, float* __restrict__ dlogits, int64_t rows, int K,
                              float invT) {
    const int lane = threadIdx.x & 31;
    const int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * SG_ROWS;
    if (r0 >= rows) return;
    float v[SG_ROWS][KM], gr[SG_ROWS];
    int ks[SG_ROWS];
#pragma unroll
    for (int q = 0; q < SG_ROWS; ++q) {
        const int64_t r = r0 + q;
        const bool ok = r < rows;
        ks[q] = ok ? min((int)kstar[r], K - 1) : 0;
        gr[q] = ok ? gsel[r] : 0.f;
#pragma unroll
        for (int m = 0; m < KM; ++m) {
            const int k = lane + 32 * m;
            v[q][m] = (ok && k < K) ? logits[r * K + k] * invT : -INFINITY;
        }
    }
#pragma unroll
    for (int q = 0; q < SG_ROWS; ++q) {
        const int64_t r = r0 + q;
        float mx = -INFINITY;
#pragma unroll
        for (int m = 0; m < KM; ++m) mx = fmaxf(mx, v[q][m]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float sum = 0.f;
#pragma unroll
        for (int m = 0; m < KM; ++m) {
            v[q][m] = lane + 32 * m < K ? expf(v[q][m] - mx) : 0.f;
            sum += v[q][m];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const float rs = 1.f / sum;
        float eks = 0.f;   // exp of the selected logit: lane ks % 32, slot ks / 32
#pragma unroll
        for (int m = 0; m < KM; ++m) {
            const float e = __shfl_sync(0xffffffffu, v[q][m], ks[q] & 31);
            if ((ks[q] >> 5) == m) eks = e;
        }
        const float coef = gr[q] * eks * rs * invT;
        if (r < rows) {
#pragma unroll
            for (int m = 0; m < KM; ++m) {
                const int k = lane + 32 * m;
                if (k < K) dlogits[r * K + k] = coef * ((k == ks[q] ? 1.f : 0.f) - v[q][m] * rs);
            }
        }
    }
}

// small K (<= KP, KP in {32, 64}): one THREAD per row, the row's logits in registers
// (fixed-order serial reductions): ~10x fewer warp instructions than the warp-per-row form.
template <int KP>
__global__ void __launch_bounds__(128) k_select_grad_row(const float* __restrict__ logits, const uint8_t* __restrict__ kstar,
                                                         const float* __restrict__ gsel, float* __restrict__ dlogits,
                                                         int64_t rows, int K, float invT) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* z = logits + r * K;
    const int ks = min((int)kstar[r], K - 1);
    const float gr = gsel[r];
    float v[KP];
    const bool vec = (K & 3) == 0;   // 16-byte rows
    if (vec) {
#pragma unroll
        for (int k = 0; k < KP; k += 4) {
            if (k < K) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(z + k));
                v[k] = q.x; v[k + 1] = q.y; v[k + 2] = q.z; v[k + 3] = q.w;
            } else {
                v[k] = v[k + 1] = v[k + 2] = v[k + 3] = -INFINITY;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < KP; ++k) v[k] = k < K ? __ldg(z + k) : -INFINITY;
    }
    float mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
        v[k] *= invT;
        mx = fmaxf(mx, v[k]);
    }
    float sum = 0.f, eks = 0.f;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
        v[k] = k < K ? expf(v[k] - mx) : 0.f;
        sum += v[k];
        if (k == ks) eks = v[k];
    }
    const float rs = 1.f / sum;
    const float coef = gr * eks * rs * invT;
    float* o = dlogits + r * K;
    if (vec) {
#pragma unroll
        for (int k = 0; k < KP; k += 4)
            if (k < K)
                *reinterpret_cast<float4*>(o + k) =
                    make_float4(coef * ((k == ks ? 1.f : 0.f) - v[k] * rs), coef * ((k + 1 == ks ? 1.f : 0.f) - v[k + 1] * rs),
                                coef * ((k + 2 == ks ? 1.f : 0.f) - v[k + 2] * rs), coef * ((k + 3 == ks ? 1.f : 0.f) - v[k + 3] * rs));
    } else {
#pragma unroll
        for (int k = 0; k < KP; ++k)
            if (k < K) o[k] = coef * ((k == ks ? 1.f : 0.f) - v[k] * rs);
    }
}

// ----------------------------------------------------------------------------- dictionary
struct DictArgs {
    const float* M;         // [H][K][N][N]
    const uint8_t* kstar;   // [B][H][L]
    const void* diag;       // PER_STEP act [B][H][L][c][N]
    const float* diag_dict; // PER_DICT f32 [H][K][c][N]
    const void* hsaved;     // act [B][H][L][c][N]
    const float* h0;        // f32 [B][H][c][N] or null
    const void* lam;        // act [B][H][L][c][N]  (dbias of pdssm_scan_bwd)
    float* dM;              // [H][K][N][N]
    float* G;               // [H][K][N][N] or null
    int B, H, L, N, K;
    float invT;
};

template <typename T>
__device__ __forceinline__ float ld_act(const T* p) {
    if constexpr (std::is_same<T, float>::value) return __ldg(p);
    else return __bfloat162float(*p);
}

// Stable in-order compaction of the positions p = b*L + t of head h with k*[b,h,t] == k:
// appends to q[*qn ...] (shared), scanning [pos, pos + blockDim.x).  Returns the new count.
__device__ __forceinline__ int compact_chunk(const DictArgs& a, int h, int k, int64_t pos, int* q, int qn, int* wcnt) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, NWp = blockDim.x >> 5;
    const int64_t p = pos + tid;
    const int64_t BL = (int64_t)a.B * a.L;
    bool m = false;
    if (p < BL) {
        const int64_t b = p / a.L, t = p - b * a.L;
        m = min((int)a.kstar[(b * a.H + h) * a.L + t], a.K - 1) == k;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, m);
    if (lane == 0) wcnt[w] = __popc(bal);
    __syncthreads();
    int before = 0, tot = 0;
    for (int x = 0; x < NWp; ++x) {
        const int c = wcnt[x];
        before += x < w ? c : 0;
        tot += c;
    }
    if (m) q[qn + before + __popc(bal & ((1u << lane) - 1u))] = (int)p;
    __syncthreads();
    return qn + tot;
}

// drop the first nb entries of the queue (qn - nb < blockDim.x: one entry per thread)
__device__ __forceinline__ void pop_queue(int* q, int qn, int nb) {
    const int x = threadIdx.x;
    const int v = x < qn - nb ? q[x + nb] : 0;
    __syncthreads();
    if (x < qn - nb) q[x] = v;
    __syncthreads();
}

// softmax Jacobian epilogue for one (h, k): Gs [N][N+1] shared (G[i][j]); one thread per column
__device__ __forceinline__ void jacobian_epilogue(const DictArgs& a, int h, int k, const float* Gs) {
    const int N = a.N;
    const size_t base = ((size_t)h * a.K + k) * N * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        const float* Mc = a.M + base + j;
        float mx = -INFINITY;
        for (int i = 0; i < N; ++i) mx = fmaxf(mx, Mc[(size_t)i * N] * a.invT);
        float sum = 0.f;
        for (int i = 0; i < N; ++i) sum += expf(Mc[(size_t)i * N] * a.invT - mx);
        const float rs = 1.f / sum;
        float proj = 0.f;
        for (int i = 0; i < N; ++i) proj += expf(Mc[(size_t)i * N] * a.invT - mx) * rs * Gs[i * (N + 1) + j];
        for (int i = 0; i < N; ++i) {
            const float g = Gs[i * (N + 1) + j];
            const float sg = expf(Mc[(size_t)i * N] * a.invT - mx) * rs;
            a.dM[base + (size_t)i * N + j] = sg * (g - proj) * a.invT;
            if (a.G) a.G[base + (size_t)i * N + j] = g;
        }
    }
}

// w_t[j] = D_t[j] h_{t-1}[j] (complex; NC = 1: real) and lambda_t[j] for position p, plane pl
template <typename T, int NC, bool PD>
__device__ __forceinline__ void row_vals(const DictArgs& a, int h, int k, int64_t p, int n, float& lr, float& li,
                                         float& wr, float& wi) {
    const int N = a.N;
    const int64_t b = p / a.L, t = p - b * a.L;
    const size_t s = (size_t)b * a.H + h;
    const size_t off = (s * a.L + t) * NC * N + n;
    const T* lam = static_cast<const T*>(a.lam);
    lr = ld_act(lam + off);
    li = NC == 2 ? ld_act(lam + off + N) : 0.f;
    float dr, di = 0.f;
    if constexpr (PD) {
        const float* dk = a.diag_dict + ((size_t)h * a.K + k) * NC * N + n;
        dr = dk[0];
        if constexpr (NC == 2) di = dk[N];
    } else {
        const T* D = static_cast<const T*>(a.diag);
        dr = ld_act(D + off);
        if constexpr (NC == 2) di = ld_act(D + off + N);
    }
    float hr = 0.f, hi = 0.f;
    if (t > 0) {
        const T* hs = static_cast<const T*>(a.hsaved);
        hr = ld_act(hs + off - NC * N);
        if constexpr (NC == 2) hi = ld_act(hs + off - NC * N + N);
    } else if (a.h0) {
        hr = a.h0[s * NC * N + n];
        if constexpr (NC == 2) hi = a.h0[s * NC * N + N + n];
    }
    wr = dr * hr - di * hi;
    wi = dr * hi + di * hr;
}

// Generic SIMT kernel (any N <= 128): CTA per (h, k), G in shared memory, one batch of
// 32 rows at a time; each thread owns the entries e = tid + blockDim.x * m.
template <typename T, int NC, bool PD>
__global__ void __launch_bounds__(256) k_dict_grad_simt(DictArgs a) {
    extern __shared__ __align__(16) float sm[];
    const int N = a.N;
    const int h = blockIdx.x / a.K, k = blockIdx.x % a.K;
    constexpr int RB = 32;
    float* Gs = sm;                                  // [N][N+1]
    float* ls = Gs + (size_t)N * (N + 1);            // [RB][NC][N]
    float* ws = ls + (size_t)RB * NC * N;            // [RB][NC][N]
    int* q = reinterpret_cast<int*>(ws + (size_t)RB * NC * N);   // [RB + 256]
    int* wcnt = q + RB + 256;                        // [8]
    for (int e = threadIdx.x; e < N * (N + 1); e += blockDim.x) Gs[e] = 0.f;
    const int64_t BL = (int64_t)a.B * a.L;
    int64_t pos = 0;
    int qn = 0;
    __syncthreads();
    while (true) {
        while (qn < RB && pos < BL) {
            qn = compact_chunk(a, h, k, pos, q, qn, wcnt);
            pos += blockDim.x;
        }
        const int nb = min(qn, RB);
        if (nb == 0) break;
        for (int x = threadIdx.x; x < nb * N; x += blockDim.x) {
            const int r = x / N, n = x - r * N;
            float lr, li, wr, wi;
            row_vals<T, NC, PD>(a, h, k, q[r], n, lr, li, wr, wi);
            ls[(r * NC) * N + n] = lr;
            ws[(r * NC) * N + n] = wr;
            if constexpr (NC == 2) {
                ls[(r * NC + 1) * N + n] = li;
                ws[(r * NC + 1) * N + n] = wi;
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
            const int i = e / N, j = e - i * N;
            float acc = Gs[i * (N + 1) + j];
            for (int r = 0; r < nb; ++r) {
#pragma unroll
                for (int pl = 0; pl < NC; ++pl) acc += ls[(r * NC + pl) * N + i] * ws[(r * NC + pl) * N + j];
            }
            Gs[i * (N + 1) + j] = acc;
        }
        __syncthreads();
        pop_queue(q, qn, nb);   // (q is not read by the MMA)
        qn -= nb;
    }
    jacobian_epilogue(a, h, k, Gs);
}

// tcgen05 kernel, N = 128: CTA per (h, k), 256 threads.  Per batch, RB = 32 / NC steps give
// one 128-byte K slab: K index kk = r * NC + plane.
constexpr int TC_N = 128;
constexpr int TC_SLAB = TC_N * 128;        // bytes of one 128-row x 128-byte operand tile
constexpr int TC_STAGE = 4 * TC_SLAB;      // A hi, A lo, B hi, B lo (one operand stage)
constexpr int TC_THREADS = 512;
constexpr int TC_PAIRS = TC_N * 8 / TC_THREADS;   // (row n, 16-byte chunk) pairs per thread per batch
constexpr int TC_PPT = 4;                  // k* positions per thread per compaction window
constexpr int TC_WIN = TC_PPT * TC_THREADS;
constexpr int TC_QCAP = TC_WIN + 64;       // queue capacity (window + carried-over rows)
// two operand stages | queue | window sums | mbarriers | TMEM slot.  The epilogue's G tile
// [N][N+1] and M tile [N][N] reuse the operand stages.
constexpr size_t TC_OFF_Q = 2 * (size_t)TC_STAGE;
constexpr size_t TC_OFF_WSUM = TC_OFF_Q + 4 * (size_t)TC_QCAP;
constexpr size_t TC_OFF_BAR = TC_OFF_WSUM + 4 * (size_t)(TC_THREADS / 32);
__host__ __device__ constexpr size_t tc_smem_bytes() { return 1024 + TC_OFF_BAR + 64; }
static_assert(TC_OFF_Q >= 4 * (size_t)(TC_N * (TC_N + 1) + TC_N * TC_N) - 1024, "epilogue tiles must fit");
static_assert(1024 + 3 * 4 * (size_t)TC_THREADS <= 4 * (size_t)TC_QCAP, "Jacobian partials must fit after the M tile");
static_assert(1024 + TC_OFF_BAR + 64 <= 227 * 1024, "shared memory budget");

// byte offset of (row n, 16-byte chunk ch) in a K-major SWIZZLE_128B tile (8-row atoms of 1024 B)
__device__ __forceinline__ uint32_t sw128(int n, int ch) { return (uint32_t)((n >> 3) * 1024 + (n & 7) * 128 + ((ch ^ (n & 7)) << 4)); }

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
// hi = x truncated to tf32 (the top 10 mantissa bits: one LOP3, where cvt.rna costs a slow-path
// conversion) and lo = x - hi (exact) at the same swizzled offset of the hi / lo tiles; the
// 3xTF32 products keep ~2^-20 relative accuracy (lo's own truncation and lo*lo are dropped)
__device__ __forceinline__ uint32_t tf32_trunc(float x) { return __float_as_uint(x) & 0xffffe000u; }
__device__ __forceinline__ void split_store(uint32_t hi, uint32_t lo, uint32_t off, float x0, float x1, float x2, float x3) {
    const uint32_t h0 = tf32_trunc(x0), h1 = tf32_trunc(x1), h2 = tf32_trunc(x2), h3 = tf32_trunc(x3);
    sts128(hi + off, h0, h1, h2, h3);
    sts128(lo + off, __float_as_uint(x0 - __uint_as_float(h0)), __float_as_uint(x1 - __uint_as_float(h1)),
           __float_as_uint(x2 - __uint_as_float(h2)), __float_as_uint(x3 - __uint_as_float(h3)));
}

// Stable compaction of a window of TC_WIN positions [pos, pos + TC_WIN) (TC_PPT consecutive
// per thread, all loads in flight together) appended to q[qn ...] as row codes: the row
// R = (b H + h) L + t of a step with t > 0, or -(b H + h) - 1 for t = 0.  Returns the new count.
__device__ __forceinline__ int compact_window(const DictArgs& a, int h, int k, int64_t pos, int* q, int qn, int* wsum) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t BL = (int64_t)a.B * a.L;
    const int64_t p0 = pos + TC_PPT * (int64_t)tid;
    // one 32-bit division per thread (B * L < 2^31), then carry t across sequence ends
    int b = (int)(p0 / a.L), t = (int)(p0 - (int64_t)b * a.L);
    uint32_t bits = 0;
    int code[TC_PPT];
#pragma unroll
    for (int u = 0; u < TC_PPT; ++u) {
        code[u] = 0;
        if (p0 + u < BL) {
            const int sq = b * a.H + h;
            bits |= (uint32_t)(min((int)a.kstar[(int64_t)sq * a.L + t], a.K - 1) == k) << u;
            code[u] = t > 0 ? sq * a.L + t : -sq - 1;
        }
        if (++t == a.L) {
            t = 0;
            ++b;
        }
    }
    const int c = __popc(bits);
    int inc = c;   // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    int before = inc - c, tot = 0;
    for (int x = 0; x < TC_THREADS / 32; ++x) {
        const int v = wsum[x];
        before += x < w ? v : 0;
        tot += v;
    }
    int o = qn + before;
#pragma unroll
    for (int u = 0; u < TC_PPT; ++u)
        if (bits >> u & 1u) q[o++] = code[u];
    __syncthreads();
    return qn + tot;
}

// Raw operand values of one batch for this thread: TC_PAIRS (row n, chunk) pairs x 12 values
// (NC = 2: 2 steps x {lr, li, Dr, Di, hr, hi};  NC = 1: 4 steps x {l, D, h}).  Rows are the
// row codes of compact_window (no division here).
template <typename T, int NC, bool PD>
__device__ __forceinline__ void load_raw(const DictArgs& a, int h, int k, const int* rows, int nb,
                                         float (&raw)[TC_PAIRS][12]) {
    constexpr int N = TC_N;
#pragma unroll
    for (int m = 0; m < TC_PAIRS; ++m) {
        const int x = threadIdx.x + TC_THREADS * m;
        const int n = x & (N - 1), ch = x >> 7;
        constexpr int RPC = 4 / NC;   // steps per 16-byte chunk
#pragma unroll
        for (int u = 0; u < RPC; ++u) {
            const int r = RPC * ch + u;
            float* v = &raw[m][u * 3 * NC];
#ifdef DG_NOLOAD   // timing experiment only: constant operands, no global loads
            if (r < nb) {
#pragma unroll
                for (int z = 0; z < 3 * NC; ++z) v[z] = 0.5f + (float)(rows[r] & 7);
            } else
#else
            if (r < nb) {
                const int c = rows[r];
                const bool first = c < 0;
                const size_t sq = first ? (size_t)(-c - 1) : 0;
                const size_t R = first ? sq * (size_t)a.L : (size_t)c;
                const size_t off = R * NC * N + n;
                const T* lam = static_cast<const T*>(a.lam);
                v[0] = ld_act(lam + off);
                if constexpr (NC == 2) v[1] = ld_act(lam + off + N);
                float* dv = v + NC;
                if constexpr (PD) {
                    const float* dk = a.diag_dict + ((size_t)h * a.K + k) * NC * N + n;
                    dv[0] = __ldg(dk);
                    if constexpr (NC == 2) dv[1] = __ldg(dk + N);
                } else {
                    const T* D = static_cast<const T*>(a.diag);
                    dv[0] = ld_act(D + off);
                    if constexpr (NC == 2) dv[1] = ld_act(D + off + N);
                }
                float* hv = v + 2 * NC;
                if (!first) {
                    const T* hs = static_cast<const T*>(a.hsaved);
                    hv[0] = ld_act(hs + off - NC * N);
                    if constexpr (NC == 2) hv[1] = ld_act(hs + off - NC * N + N);
                } else if (a.h0) {
                    hv[0] = __ldg(a.h0 + sq * NC * N + n);
                    if constexpr (NC == 2) hv[1] = __ldg(a.h0 + sq * NC * N + N + n);
                } else {
                    hv[0] = 0.f;
                    if constexpr (NC == 2) hv[1] = 0.f;
                }
            } else
#endif
            {
#pragma unroll
                for (int z = 0; z < 3 * NC; ++z) v[z] = 0.f;
            }
        }
    }
}

// raw -> (lambda, w = D (.) h_{t-1}) -> tf32 hi/lo into the K-major SWIZZLE_128B operand tiles
template <int NC>
__device__ __forceinline__ void convert_store(const float (&raw)[TC_PAIRS][12], uint32_t st) {
#pragma unroll
    for (int m = 0; m < TC_PAIRS; ++m) {
        const int x = threadIdx.x + TC_THREADS * m;
        const int n = x & (TC_N - 1), ch = x >> 7;
        float lv[4], wv[4];
        if constexpr (NC == 2) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float* v = &raw[m][6 * u];
                lv[2 * u] = v[0];
                lv[2 * u + 1] = v[1];
                wv[2 * u] = v[2] * v[4] - v[3] * v[5];
                wv[2 * u + 1] = v[2] * v[5] + v[3] * v[4];
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float* v = &raw[m][3 * u];
                lv[u] = v[0];
                wv[u] = v[1] * v[2];
            }
        }
        const uint32_t off = sw128(n, ch);
        split_store(st, st + TC_SLAB, off, lv[0], lv[1], lv[2], lv[3]);
        split_store(st + 2 * TC_SLAB, st + 3 * TC_SLAB, off, wv[0], wv[1], wv[2], wv[3]);
    }
}

template <typename T, int NC, bool PD>
__global__ void __launch_bounds__(TC_THREADS, 1) k_dict_grad_tc(DictArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    constexpr int N = TC_N;
    constexpr int RB = 32 / NC;                // steps per K slab
    const int h = blockIdx.x / a.K, k = blockIdx.x % a.K;
    int* q = reinterpret_cast<int*>(smem + TC_OFF_Q);          // queue of row codes
    int* wsum = reinterpret_cast<int*>(smem + TC_OFF_WSUM);
    uint64_t* done = reinterpret_cast<uint64_t*>(smem + TC_OFF_BAR);   // [2] MMA completion per operand stage
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 2);
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        tc::mbar_init(done, 1);
        tc::mbar_init(done + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::su32(tslot)), "r"(128)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t id_ = tc::idesc(2u, N);   // kind::tf32, M = 128, N = 128
    const int64_t BL = (int64_t)a.B * a.L;
    int64_t pos = 0;
    int qh = 0, qn = 0;
    auto refill = [&]() {   // >= 2 RB rows queued (or the head's positions exhausted)
        while (qn - qh < 2 * RB && pos < BL) {
            const int rem = qn - qh;   // < 2 RB <= blockDim
            const int v = tid < rem ? q[qh + tid] : 0;
            __syncthreads();
            if (tid < rem) q[tid] = v;
            qn = rem;
            qh = 0;
            qn = compact_window(a, h, k, pos, q, qn, wsum);   // (syncs before reading q)
            pos += TC_WIN;
        }
    };
    // three batches of raw values in registers, rotated by role (no copies: a register copy
    // of a pending load would wait for it): batch n is converted while n+1 and n+2 are in flight
    float R0[TC_PAIRS][12], R1[TC_PAIRS][12], R2[TC_PAIRS][12];
    int nbs[3];
    refill();
    nbs[0] = min(qn - qh, RB);
    if (nbs[0] > 0) load_raw<T, NC, PD>(a, h, k, q + qh, nbs[0], R0);
    qh += nbs[0];
    refill();
    nbs[1] = min(qn - qh, RB);
    if (nbs[1] > 0) load_raw<T, NC, PD>(a, h, k, q + qh, nbs[1], R1);
    qh += nbs[1];
    int nbatch = 0;
    auto iter = [&](float (&cur)[TC_PAIRS][12], float (&ld)[TC_PAIRS][12], const int ic, const int il) -> bool {
        if (nbs[ic] == 0) return false;
        refill();
        nbs[il] = min(qn - qh, RB);
        if (nbs[il] > 0) load_raw<T, NC, PD>(a, h, k, q + qh, nbs[il], ld);   // two batches ahead
        qh += nbs[il];
        const int s = nbatch & 1;
        uint8_t* st = smem + (size_t)s * TC_STAGE;
#ifndef DG_NOMMA
        if (nbatch >= 2) tc::mbar_wait(done + s, (uint32_t)((nbatch - 2) >> 1) & 1u);   // MMAs of batch n-2 read it
#endif
#ifndef DG_NOCONVERT   // timing experiments only
        convert_store<NC>(cur, tc::su32(st));
#endif
#ifndef DG_NOFENCE
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA reads
#endif
        __syncthreads();
#ifdef DG_NOMMA   // timing experiment only
        if (false) {
#else
        if (tid == 0) {
#endif
            tc::fence_after();
            const uint64_t ah = tc::sdesc(tc::su32(st)), al = tc::sdesc(tc::su32(st + TC_SLAB));
            const uint64_t bh = tc::sdesc(tc::su32(st + 2 * TC_SLAB)), bl = tc::sdesc(tc::su32(st + 3 * TC_SLAB));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {   // 8 tf32 (32 bytes) of K per instruction
                const uint32_t acc0 = (nbatch | kk) != 0;
                tc::Kind<float>::mma(tmem, al + 2 * kk, bh + 2 * kk, id_, acc0);
                tc::Kind<float>::mma(tmem, ah + 2 * kk, bl + 2 * kk, id_, 1u);
                tc::Kind<float>::mma(tmem, ah + 2 * kk, bh + 2 * kk, id_, 1u);
            }
            tc::commit(done + s);
        }
        ++nbatch;
        return true;
    };
    while (iter(R0, R2, 0, 2) && iter(R1, R0, 1, 0) && iter(R2, R1, 2, 1)) {
    }
    // drain: the last batch's commit covers every earlier MMA
#ifndef DG_NOMMA
    if (nbatch > 0) tc::mbar_wait(done + ((nbatch - 1) & 1), (uint32_t)((nbatch - 1) >> 1) & 1u);
#endif
    tc::fence_after();
    __syncthreads();
    float* Gs = reinterpret_cast<float*>(smem);   // [N][N+1] over the (now idle) operand stages
    if (warp < 4) {
        const int i = warp * 32 + (tid & 31);
        for (int j0 = 0; j0 < N; j0 += 16) {
            float v[16];
            if (nbatch > 0) {
                tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)j0, v);
            } else {
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = 0.f;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) Gs[i * (N + 1) + j0 + u] = v[u];
        }
    }
    // the dictionary tile M[h][k] next to it (row-major, read row-wise by the column threads)
    float* Ms = Gs + N * (N + 1);
    {
        const float4* src = reinterpret_cast<const float4*>(a.M + ((size_t)h * a.K + k) * N * N);
        for (int x = tid; x < N * N / 4; x += TC_THREADS) reinterpret_cast<float4*>(Ms)[x] = __ldg(src + x);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128) : "memory");
    }
    // softmax Jacobian over the 512 threads: thread (q, j) = tid / N, tid % N owns rows
    // [q N/4, (q+1) N/4) of column j; the four partial max / sums / projections combine in a
    // fixed order (q = 0..3) through shared memory, so the result is run-to-run identical
#ifndef DG_NOEPI
    {
        constexpr int QN = TC_THREADS / N;   // 4 row quarters
        constexpr int RQ = N / QN;
        float* part = reinterpret_cast<float*>(smem + TC_OFF_Q + 1024);   // [3][QN][N] (after Ms)
        const int j = tid % N, qq = tid / N, i0 = qq * RQ;
        float mx = -INFINITY;
        for (int i = i0; i < i0 + RQ; ++i) mx = fmaxf(mx, Ms[i * N + j] * a.invT);
        part[qq * N + j] = mx;
        __syncthreads();
        mx = part[j];
#pragma unroll
        for (int x = 1; x < QN; ++x) mx = fmaxf(mx, part[x * N + j]);
        float sum = 0.f, pr = 0.f;
        for (int i = i0; i < i0 + RQ; ++i) {
            const float e = expf(Ms[i * N + j] * a.invT - mx);
            sum += e;
            pr += e * Gs[i * (N + 1) + j];
        }
        part[(QN + qq) * N + j] = sum;
        part[(2 * QN + qq) * N + j] = pr;
        __syncthreads();
        sum = part[QN * N + j];
        pr = part[2 * QN * N + j];
#pragma unroll
        for (int x = 1; x < QN; ++x) {
            sum += part[(QN + x) * N + j];
            pr += part[(2 * QN + x) * N + j];
        }
        const float rs = 1.f / sum;
        const float proj = pr * rs;
        const size_t base = ((size_t)h * a.K + k) * N * N;
        for (int i = i0; i < i0 + RQ; ++i) {
            const float g = Gs[i * (N + 1) + j];
            const float sg = expf(Ms[i * N + j] * a.invT - mx) * rs;
            a.dM[base + (size_t)i * N + j] = sg * (g - proj) * a.invT;
            if (a.G) a.G[base + (size_t)i * N + j] = g;
        }
    }
#endif
}

// NEXT-2 D_t generator, SIMT fallback: the projection writes raw (a, theta) planes, then
// this kernel applies sigmoid / sincos in place.  rows = B*H*L in [B][H][L] order.
template <typename T>
__global__ void k_diag_activate(T* __restrict__ D, const float* __restrict__ bias, int64_t rows, int H, int L, int N,
                                int nc) {
    const int64_t total = rows * N;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / N;
        const int n = (int)(i - r * N);
        const int h = (int)((r / L) % H);
        T* row = D + r * (int64_t)nc * N;
        const float mag = 1.f / (1.f + expf(-(ldact(row + n) + (bias ? bias[(size_t)h * N + n] : 0.f))));
        if (nc == 2) {
            float sn, cs;
            sincosf(ldact(row + N + n), &sn, &cs);
            stact(row + n, mag * cs);
            stact(row + N + n, mag * sn);
        } else {
            stact(row + n, mag);
        }
    }
}

// NEXT-3 staging for the soft generator GEMM: s = softmax(logits) per (b, h, t) into the per-head
// K-major operand [H][B*L][Kp] (zero-padded to Kp), and the dictionary transposed to
// Mt[H][j * N + i][Kp] = M[H][k][i][j].
template <typename T>
__global__ void k_soft_stage_s(const float* __restrict__ logits, T* __restrict__ s, int64_t BL, int H, int L, int K, int Kp) {
    // one warp per (b, h, t) row: lanes own k = lane + 32 m (coalesced row reads and writes)
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // (b, h, t) row
    if (r >= BL * H) return;
    const int64_t b = r / ((int64_t)H * L), rem = r - b * H * L;
    const int h = (int)(rem / L);
    const int64_t t = rem - (int64_t)h * L;
    const float* z = logits + r * K;
    float mx = -INFINITY;
    for (int k = lane; k < K; k += 32) mx = fmaxf(mx, z[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int k = lane; k < K; k += 32) sum += expf(z[k] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float rs = 1.f / sum;
    T* o = s + ((size_t)h * BL + b * L + t) * Kp;
    for (int k = lane; k < Kp; k += 32) stact(o + k, k < K ? expf(z[k] - mx) * rs : 0.f);
}
template <typename T>
__global__ void k_soft_stage_M(const float* __restrict__ M, T* __restrict__ Mt, int H, int K, int N, int Kp) {
    const int64_t total = (int64_t)H * N * N * Kp;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(x % Kp);
        const int64_t rest = x / Kp;   // (h, j, i)
        const int i = (int)(rest % N), j = (int)((rest / N) % N), h = (int)(rest / ((int64_t)N * N));
        stact(Mt + x, k < K ? M[(((size_t)h * K + k) * N + i) * N + j] : 0.f);
    }
}

}  // namespace sg
}  // namespace pdssm
