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
// one warp per (b, h, t) row of K logits
__global__ void k_select_grad(const float* __restrict__ logits, const uint8_t* __restrict__ kstar,
                              const float* __restrict__ gsel, float* __restrict__ dlogits, int64_t rows, int K,
                              float invT) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= rows) return;
    const float* z = logits + r * K;
    float mx = -INFINITY;
    for (int k = lane; k < K; k += 32) mx = fmaxf(mx, z[k] * invT);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int k = lane; k < K; k += 32) sum += expf(z[k] * invT - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const int ks = min((int)kstar[r], K - 1);
    const float rs = 1.f / sum;
    const float sk = expf(z[ks] * invT - mx) * rs;
    const float coef = gsel[r] * sk * invT;
    for (int k = lane; k < K; k += 32) {
        const float s = expf(z[k] * invT - mx) * rs;
        dlogits[r * K + k] = coef * ((k == ks ? 1.f : 0.f) - s);
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
constexpr int TC_STAGE = 4 * TC_SLAB;      // A hi, A lo, B hi, B lo
constexpr int TC_THREADS = 256;
__host__ __device__ constexpr size_t tc_smem_bytes() { return 1024 + 2 * (size_t)TC_STAGE + 4 * (32 + 256) + 64 + 64; }

// byte offset of (row n, 16-byte chunk ch) in a K-major SWIZZLE_128B tile (8-row atoms of 1024 B)
__device__ __forceinline__ uint32_t sw128(int n, int ch) { return (uint32_t)((n >> 3) * 1024 + (n & 7) * 128 + ((ch ^ (n & 7)) << 4)); }

__device__ __forceinline__ void split_store(uint8_t* hi, uint8_t* lo, uint32_t off, float x0, float x1, float x2, float x3) {
    const uint32_t h0 = tc::tf32_rna(x0), h1 = tc::tf32_rna(x1), h2 = tc::tf32_rna(x2), h3 = tc::tf32_rna(x3);
    *reinterpret_cast<uint4*>(hi + off) = make_uint4(h0, h1, h2, h3);
    *reinterpret_cast<float4*>(lo + off) = make_float4(x0 - __uint_as_float(h0), x1 - __uint_as_float(h1),
                                                       x2 - __uint_as_float(h2), x3 - __uint_as_float(h3));
}

template <typename T, int NC, bool PD>
__global__ void __launch_bounds__(TC_THREADS, 1) k_dict_grad_tc(DictArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    constexpr int N = TC_N;
    constexpr int RB = 32 / NC;                // steps per K slab
    const int h = blockIdx.x / a.K, k = blockIdx.x % a.K;
    int* q = reinterpret_cast<int*>(smem + 2 * TC_STAGE);      // [RB + 256] queue
    int* wcnt = q + 32 + 256;                                  // [8]
    uint64_t* done = reinterpret_cast<uint64_t*>(wcnt + 16);   // [2] MMA completion per buffer
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
    int qn = 0, nbatch = 0;
    while (true) {
        while (qn < RB && pos < BL) {
            qn = compact_chunk(a, h, k, pos, q, qn, wcnt);
            pos += blockDim.x;
        }
        const int nb = min(qn, RB);
        if (nb == 0) break;
        const int s = nbatch & 1;
        uint8_t* st = smem + (size_t)s * TC_STAGE;
        if (nbatch >= 2) tc::mbar_wait(done + s, (uint32_t)((nbatch - 2) >> 1) & 1u);   // MMAs of batch n-2 read it
        // stage: pair x = (n, chunk); chunk ch holds kk = 4ch..4ch+3 = (row, plane) pairs
        for (int x = tid; x < N * 8; x += TC_THREADS) {
            const int n = x & (N - 1), ch = x >> 7;
            float lv[4], wv[4];
            if constexpr (NC == 2) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int r = 2 * ch + u;
                    float lr = 0.f, li = 0.f, wr = 0.f, wi = 0.f;
                    if (r < nb) row_vals<T, NC, PD>(a, h, k, q[r], n, lr, li, wr, wi);
                    lv[2 * u] = lr;
                    lv[2 * u + 1] = li;
                    wv[2 * u] = wr;
                    wv[2 * u + 1] = wi;
                }
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int r = 4 * ch + u;
                    float lr = 0.f, li, wr = 0.f, wi;
                    if (r < nb) row_vals<T, NC, PD>(a, h, k, q[r], n, lr, li, wr, wi);
                    lv[u] = lr;
                    wv[u] = wr;
                }
            }
            const uint32_t off = sw128(n, ch);
            split_store(st, st + TC_SLAB, off, lv[0], lv[1], lv[2], lv[3]);
            split_store(st + 2 * TC_SLAB, st + 3 * TC_SLAB, off, wv[0], wv[1], wv[2], wv[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA reads
        __syncthreads();
        if (tid == 0) {
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
        pop_queue(q, qn, nb);   // (q is not read by the MMA)
        qn -= nb;
        ++nbatch;
    }
    // drain: the last batch's commit covers every earlier MMA
    if (nbatch > 0) tc::mbar_wait(done + ((nbatch - 1) & 1), (uint32_t)((nbatch - 1) >> 1) & 1u);
    tc::fence_after();
    float* Gs = reinterpret_cast<float*>(smem);   // [N][N+1] over the (now idle) operand buffers
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
    tc::fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128) : "memory");
    }
    jacobian_epilogue(a, h, k, Gs);
}

}  // namespace sg
}  // namespace pdssm
