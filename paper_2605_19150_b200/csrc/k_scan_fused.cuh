// Fused single-pass chunked scan for sm_100a (fast path of pdssm_scan_fwd /
// pdssm_scan_bwd).  Algorithm 1 re-blocked for B200:
//
//  * one WARP per (sequence, chunk) item; lane l owns the NPL = N/32 contiguous
//    states [l*NPL, l*NPL+NPL) so every HBM access is a coalesced 16-byte
//    vector per lane and intra-step exchange needs only __syncwarp;
//  * Phase A (aggregate), the carry hand-off and Phase C (replay) run in ONE
//    launch: a warp finishes Phase A, waits for its predecessor's carry
//    (chained look-back over per-(sequence, chunk) flags, dynamic tickets in
//    chunk-major order guarantee forward progress), publishes its own carry,
//    then replays the chunk.  The replay re-reads D_t / b_t while they are
//    still L2-resident (measured 18 TB/s L2 vs 6.9 TB/s HBM read, tools/l2bw.cu),
//    so HBM sees each input once: the algorithmic byte count of SURVEY §8(d);
//  * the scatter (A_t v)[i] = sum_{j : P_t[j] = i} D_t[j] v[j] runs as a
//    gather over a per-dictionary-entry, per-lane padded preimage list
//    ("fused plan", built once per call, MU sources per target inline, longer
//    preimages fall back to the CSR plan) -- deterministic, no float atomics;
//  * the backward is the transposed scan (pure gather) with the same
//    structure in reverse chunk order, reusing the forward (pi_bar, d_bar).
#pragma once
#include <type_traits>

#include "k_scan_fwd.cuh"

namespace pdssm {
namespace fused {

constexpr int WARPS = 4;          // warps (= concurrent items) per CTA
constexpr int MU = 6;             // inline preimage capacity per target

// ------------------------------------------------------------------ vector IO
template <typename T, int NPL>
__device__ __forceinline__ void vld(const T* __restrict__ p, float (&o)[NPL]) {
    if constexpr (std::is_same<T, float>::value) {
        if constexpr (NPL == 4) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(p));
            o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
        } else if constexpr (NPL == 2) {
            const float2 v = __ldg(reinterpret_cast<const float2*>(p));
            o[0] = v.x; o[1] = v.y;
        } else {
            o[0] = __ldg(p);
        }
    } else {
        if constexpr (NPL == 4) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
            o[0] = __uint_as_float(v.x << 16); o[1] = __uint_as_float(v.x & 0xffff0000u);
            o[2] = __uint_as_float(v.y << 16); o[3] = __uint_as_float(v.y & 0xffff0000u);
        } else if constexpr (NPL == 2) {
            const uint32_t v = __ldg(reinterpret_cast<const unsigned int*>(p));
            o[0] = __uint_as_float(v << 16); o[1] = __uint_as_float(v & 0xffff0000u);
        } else {
            o[0] = __bfloat162float(__ldg(p));
        }
    }
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);   // .x = a (low half)
    return *reinterpret_cast<const uint32_t*>(&v);
}

template <typename T, int NPL>
__device__ __forceinline__ void vst(T* __restrict__ p, const float (&v)[NPL]) {
    if constexpr (std::is_same<T, float>::value) {
        if constexpr (NPL == 4) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        else if constexpr (NPL == 2) *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
        else *p = v[0];
    } else {
        if constexpr (NPL == 4) *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]));
        else if constexpr (NPL == 2) *reinterpret_cast<uint32_t*>(p) = pack_bf16x2(v[0], v[1]);
        else *p = __float2bfloat16_rn(v[0]);
    }
}

// coherent (L2) loads for data produced by other warps during this launch
template <int NPL>
__device__ __forceinline__ void vld_cg(const float* p, float (&o)[NPL]) {
    if constexpr (NPL == 4) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(p));
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else if constexpr (NPL == 2) {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(p));
        o[0] = v.x; o[1] = v.y;
    } else {
        o[0] = __ldcg(p);
    }
}

template <int NPL>
__device__ __forceinline__ void vst_f(float* p, const float (&v)[NPL]) { vst<float, NPL>(p, v); }

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_flag(const uint32_t* p) {
    while (ld_acquire(p) == 0u) __nanosleep(20);
}

// per-step own-state planes: x[NC][NPL]
template <int NC, int NPL>
struct Planes {
    float v[NC][NPL];
};

template <typename T, int NC, int NPL>
__device__ __forceinline__ void load_planes(const T* __restrict__ base, Planes<NC, NPL>& o, int N) {
    vld<T, NPL>(base, o.v[0]);
    if constexpr (NC == 2) vld<T, NPL>(base + N, o.v[1]);
}

template <typename T, int NC, int NPL>
__device__ __forceinline__ void store_planes(T* __restrict__ base, const Planes<NC, NPL>& o, int N) {
    vst<T, NPL>(base, o.v[0]);
    if constexpr (NC == 2) vst<T, NPL>(base + N, o.v[1]);
}

template <int NC>
struct SVal;   // smem exchange value
template <> struct SVal<1> { using type = float; };
template <> struct SVal<2> { using type = float2; };

template <int NC>
__device__ __forceinline__ typename SVal<NC>::type mk(float re, float im) {
    if constexpr (NC == 2) return make_float2(re, im);
    else { (void)im; return re; }
}
template <int NC>
__device__ __forceinline__ float re_of(typename SVal<NC>::type v) {
    if constexpr (NC == 2) return v.x; else return v;
}
template <int NC>
__device__ __forceinline__ float im_of(typename SVal<NC>::type v) {
    if constexpr (NC == 2) return v.y; else { (void)v; return 0.f; }
}

// store this lane's NPL exchange values (contiguous) into an smem row
template <int NC, int NPL>
__device__ __forceinline__ void sts_row(typename SVal<NC>::type* row, int lane, const float (&re)[NPL],
                                        const float (&im)[NPL]) {
#pragma unroll
    for (int u = 0; u < NPL; ++u) row[lane * NPL + u] = mk<NC>(re[u], im[u]);
}

// ------------------------------------------------------------------ fused plan
// For entry e = h*K + k and lane l: rec[e][l][u*MU + q] = q-th source (ascending)
// of target i = l*NPL + u, padded with the sentinel N; hdr[e] = M_0 | M_1<<8 |
// M_2<<16 | M_3<<24 where M_u = max over lanes of the in-degree of slot u
// (warp-uniform trip counts); bit 31 of ovf[e] set if some M_u > MU.
template <int NPL>
__global__ void k_build_fused_plan(const uint16_t* __restrict__ dict_idx, uint8_t* __restrict__ rec,
                                   uint32_t* __restrict__ hdr, int N) {
    extern __shared__ uint16_t sP[];
    __shared__ int smax[8];
    const int e = blockIdx.x;
    const uint16_t* P = dict_idx + (size_t)e * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) sP[j] = min((int)P[j], N - 1);
    if (threadIdx.x < 8) smax[threadIdx.x] = 0;
    __syncthreads();
    constexpr int RB = NPL * MU;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int l = i / NPL, u = i % NPL;
        int q = 0;
        for (int j = 0; j < N; ++j) {
            if (sP[j] == i) {
                if (q < MU) rec[((size_t)e * 32 + l) * RB + u * MU + q] = (uint8_t)j;
                ++q;
            }
        }
        for (int qq = q; qq < MU; ++qq) rec[((size_t)e * 32 + l) * RB + u * MU + qq] = (uint8_t)N;
        atomicMax(&smax[u], q);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t h = 0;
        bool ovf = false;
        for (int u = 0; u < NPL; ++u) {
            h |= (uint32_t)min(smax[u], 255) << (8 * u);
            ovf |= smax[u] > MU;
        }
        hdr[2 * e] = h;
        hdr[2 * e + 1] = ovf ? 1u : 0u;
    }
}

// record bytes of one (entry, lane): NPL*MU bytes, read as 32-bit words
template <int NPL>
struct Rec {
    static constexpr int W = (NPL * MU + 3) / 4;
    uint32_t w[W];
};

template <int NPL>
__device__ __forceinline__ void load_rec(const uint8_t* __restrict__ rec, int e, int lane, Rec<NPL>& r) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(rec + ((size_t)e * 32 + lane) * (NPL * MU));
#pragma unroll
    for (int i = 0; i < Rec<NPL>::W; ++i) r.w[i] = __ldg(p + i);
}

template <int NPL>
__device__ __forceinline__ int rec_byte(const Rec<NPL>& r, int idx) {   // idx compile-time after unroll
    return (r.w[idx >> 2] >> (8 * (idx & 3))) & 0xff;
}

// acc[u] += sum_{q < M_u} vbuf[src_q] for the lane's NPL targets
template <int NC, int NPL>
__device__ __forceinline__ void gather_sum(const typename SVal<NC>::type* vbuf, const Rec<NPL>& r, uint32_t hdr,
                                           float (&are)[NPL], float (&aim)[NPL]) {
#pragma unroll
    for (int u = 0; u < NPL; ++u) {
        const int M = (hdr >> (8 * u)) & 0xff;
#pragma unroll
        for (int q = 0; q < MU; ++q) {
            if (q < M) {
                const auto v = vbuf[rec_byte<NPL>(r, u * MU + q)];
                are[u] += re_of<NC>(v);
                if constexpr (NC == 2) aim[u] += im_of<NC>(v);
            }
        }
    }
}

// slow path for entries with a preimage longer than MU: CSR plan (k_build_plan)
template <int NC, int NPL>
__device__ __forceinline__ void gather_sum_csr(const typename SVal<NC>::type* vbuf, const uint16_t* __restrict__ pstart,
                                               const uint16_t* __restrict__ psrc, int e, int N, int lane,
                                               float (&are)[NPL], float (&aim)[NPL]) {
#pragma unroll
    for (int u = 0; u < NPL; ++u) {
        const int i = lane * NPL + u;
        const int st = __ldg(pstart + (size_t)e * (N + 1) + i);
        const int en = __ldg(pstart + (size_t)e * (N + 1) + i + 1);
        for (int q = st; q < en; ++q) {
            const auto v = vbuf[__ldg(psrc + (size_t)e * N + q)];
            are[u] += re_of<NC>(v);
            if constexpr (NC == 2) aim[u] += im_of<NC>(v);
        }
    }
}

struct FusedArgs {
    const uint8_t* kstar;
    const uint16_t* dict_idx;
    const uint16_t* pstart;
    const uint16_t* psrc;
    const uint8_t* rec;
    const uint32_t* hdr;
    const void* diag;        // PER_STEP act tensor
    const float* diag_dict;  // PER_DICT f32 [H][K][NC][N]
    const void* bias;        // fwd: b_t ; bwd: e (direct gradient)
    const void* hsaved;      // bwd
    const float* h0;
    const float* lam_in;     // bwd
    ChunkStateView cs;
    uint16_t* maps;          // fwd (optional)
    void* out0;              // fwd: h ; bwd: dbias
    void* out1;              // bwd: ddiag (act, PER_STEP) or f32 scratch (PER_DICT)
    float* gsel;             // bwd
    float* dh0;              // bwd
    float* mu;               // bwd: [S][C][NC][N]
    uint32_t* ctrl;          // [0] ticket counter, [1..S*C] flags
    int H, L, N, K, tau, C, S;
    uint32_t flags;
};

template <typename T, int NC, int NPL, bool PD>
__device__ __forceinline__ void load_diag_own(const FusedArgs& a, size_t step_off, int h, int k, int lane,
                                              Planes<NC, NPL>& D) {
    if constexpr (PD) {
        const float* p = a.diag_dict + ((size_t)(h * a.K + k) * NC) * a.N + lane * NPL;
        vld<float, NPL>(p, D.v[0]);
        if constexpr (NC == 2) vld<float, NPL>(p + a.N, D.v[1]);
    } else {
        load_planes<T, NC, NPL>(static_cast<const T*>(a.diag) + step_off + lane * NPL, D, a.N);
    }
}

// ============================================================================
// forward
// ============================================================================
template <typename T, int NC, int NPL, bool PD>
__global__ void __launch_bounds__(WARPS * 32) k_fwd_fused(FusedArgs a) {
    using SV = typename SVal<NC>::type;
    constexpr int NMAX = 32 * NPL;
    __shared__ SV s_v[WARPS][2][NMAX + 1];   // v = D (.) state, + zero sentinel
    __shared__ SV s_d[WARPS][2][NMAX];       // D_t staged for the pi-gather; chain scratch
    __shared__ uint16_t s_key[WARPS][NMAX];
    __shared__ int s_cnt[WARPS][NMAX];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = a.N;
    SV* vb[2] = {s_v[w][0], s_v[w][1]};
    if (lane == 0) { vb[0][N] = mk<NC>(0.f, 0.f); vb[1][N] = mk<NC>(0.f, 0.f); }
    const int total = a.S * a.C;
    const T* bias = static_cast<const T*>(a.bias);
    T* hout = static_cast<T*>(a.out0);
    while (true) {
        __syncwarp();
        int ticket = 0;
        if (lane == 0) ticket = atomicAdd(a.ctrl, 1u);
        ticket = __shfl_sync(0xffffffffu, ticket, 0);
        if (ticket >= total) break;
        const int c = ticket / a.S, s = ticket - c * a.S, h = s % a.H;
        const int t0 = c * a.tau, t1 = min(t0 + a.tau, a.L);
        const size_t ci = (size_t)s * a.C + c;
        const size_t row = (size_t)NC * N;
        // ---------------- Phase A: aggregate from identity
        int pi[NPL];
        float dre[NPL], dim[NPL], bre[NPL], bim[NPL];
#pragma unroll
        for (int u = 0; u < NPL; ++u) { pi[u] = lane * NPL + u; dre[u] = 1.f; dim[u] = 0.f; bre[u] = 0.f; bim[u] = 0.f; }
        {
            Planes<NC, NPL> Dn, Bn;
            int kn = load_k(a.kstar, (size_t)s * a.L + t0, a.K, a.flags);
            load_diag_own<T, NC, NPL, PD>(a, ((size_t)s * a.L + t0) * row, h, kn, lane, Dn);
            load_planes<T, NC, NPL>(bias + ((size_t)s * a.L + t0) * row + lane * NPL, Bn, N);
            for (int t = t0; t < t1; ++t) {
                const int buf = (t - t0) & 1;
                const int k = kn;
                Planes<NC, NPL> D = Dn, Bv = Bn;
                if (t + 1 < t1) {
                    kn = load_k(a.kstar, (size_t)s * a.L + t + 1, a.K, a.flags);
                    load_diag_own<T, NC, NPL, PD>(a, ((size_t)s * a.L + t + 1) * row, h, kn, lane, Dn);
                    load_planes<T, NC, NPL>(bias + ((size_t)s * a.L + t + 1) * row + lane * NPL, Bn, N);
                }
                const int e = h * a.K + k;
                const uint32_t hd = __ldg(a.hdr + 2 * e);
                const uint32_t ovf = __ldg(a.hdr + 2 * e + 1);
                Rec<NPL> r;
                load_rec<NPL>(a.rec, e, lane, r);
                float vre[NPL], vim[NPL], Dim_[NPL];
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const float di = NC == 2 ? D.v[NC - 1][u] : 0.f;
                    Dim_[u] = di;
                    vre[u] = D.v[0][u] * bre[u] - di * bim[u];
                    vim[u] = D.v[0][u] * bim[u] + di * bre[u];
                }
                sts_row<NC, NPL>(vb[buf], lane, vre, vim);
                sts_row<NC, NPL>(s_d[w][buf], lane, D.v[0], Dim_);
                __syncwarp();
                // pi / d update: d <- D_t[pi] d, pi <- P_t[pi]
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const SV dp = s_d[w][buf][pi[u]];
                    const float nr = re_of<NC>(dp) * dre[u] - im_of<NC>(dp) * dim[u];
                    const float ni = re_of<NC>(dp) * dim[u] + im_of<NC>(dp) * dre[u];
                    dre[u] = nr; dim[u] = ni;
                    pi[u] = clamp_idx(__ldg(a.dict_idx + (size_t)e * N + pi[u]), N, a.flags);
                }
                // beta <- A_t beta + b_t
                float are[NPL], aim[NPL];
#pragma unroll
                for (int u = 0; u < NPL; ++u) { are[u] = 0.f; aim[u] = 0.f; }
                if (ovf) gather_sum_csr<NC, NPL>(vb[buf], a.pstart, a.psrc, e, N, lane, are, aim);
                else gather_sum<NC, NPL>(vb[buf], r, hd, are, aim);
#pragma unroll
                for (int u = 0; u < NPL; ++u) { bre[u] = are[u] + Bv.v[0][u]; bim[u] = NC == 2 ? aim[u] + Bv.v[NC - 1][u] : 0.f; }
            }
        }
        // publish the aggregate (chunk_state sections 0-2)
        {
            float tmp[NPL];
#pragma unroll
            for (int u = 0; u < NPL; ++u) a.cs.pi[ci * N + lane * NPL + u] = (uint16_t)pi[u];
            vst_f<NPL>(a.cs.d + ci * row + lane * NPL, dre);
            vst_f<NPL>(a.cs.beta + ci * row + lane * NPL, bre);
            if constexpr (NC == 2) {
                vst_f<NPL>(a.cs.d + ci * row + N + lane * NPL, dim);
                vst_f<NPL>(a.cs.beta + ci * row + N + lane * NPL, bim);
            }
            (void)tmp;
        }
        // ---------------- carry hand-off: carry_c (wait) -> carry_{c+1} (publish)
        float cre[NPL], cim[NPL];
        if (c == 0) {
#pragma unroll
            for (int u = 0; u < NPL; ++u) { cre[u] = 0.f; cim[u] = 0.f; }
            if (a.h0) {
                vld<float, NPL>(a.h0 + (size_t)s * row + lane * NPL, cre);
                if constexpr (NC == 2) vld<float, NPL>(a.h0 + (size_t)s * row + N + lane * NPL, cim);
            }
            vst_f<NPL>(a.cs.carry + ci * row + lane * NPL, cre);
            if constexpr (NC == 2) vst_f<NPL>(a.cs.carry + ci * row + N + lane * NPL, cim);
        } else {
            wait_flag(a.ctrl + 1 + ci);
            vld_cg<NPL>(a.cs.carry + ci * row + lane * NPL, cre);
            if constexpr (NC == 2) vld_cg<NPL>(a.cs.carry + ci * row + N + lane * NPL, cim);
        }
        int mp[NPL];   // exclusive prefix map before this chunk (maps export)
        if (a.maps) {
            if (c == 0) {
#pragma unroll
                for (int u = 0; u < NPL; ++u) mp[u] = lane * NPL + u;
            } else {
#pragma unroll
                for (int u = 0; u < NPL; ++u) mp[u] = __ldcg(a.maps + ((size_t)s * (a.C + 1) + c) * N + lane * NPL + u);
            }
        }
        {
            // carry_{c+1}[i] = beta_bar[i] + sum_{j : pi[j] = i} d[j] carry_c[j]
            // deterministic: unique targets stored, colliding groups reduced by a
            // fixed xor-butterfly per distinct key (ballot loop)
            __syncwarp();            // Phase A's last smem reads are done
            SV* obuf = s_d[w][1];    // [N] result
            uint16_t* key = s_key[w];
            int* cnt = s_cnt[w];
            float wr[NPL], wi[NPL];
#pragma unroll
            for (int u = 0; u < NPL; ++u) {
                wr[u] = dre[u] * cre[u] - dim[u] * cim[u];
                wi[u] = dre[u] * cim[u] + dim[u] * cre[u];
                key[lane * NPL + u] = (uint16_t)pi[u];
                obuf[lane * NPL + u] = mk<NC>(0.f, 0.f);
                cnt[lane * NPL + u] = 0;
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < NPL; ++u) atomicAdd(&cnt[pi[u]], 1);   // integer: order-independent
            __syncwarp();
            // unique targets are stored directly; colliding ones are reduced below
            bool pend[NPL];
            uint32_t anyp = 0;
#pragma unroll
            for (int u = 0; u < NPL; ++u) {
                pend[u] = cnt[pi[u]] > 1;
                if (!pend[u]) obuf[pi[u]] = mk<NC>(wr[u], wi[u]);
                anyp |= pend[u];
            }
            __syncwarp();
            uint32_t bal = __ballot_sync(0xffffffffu, anyp);
            while (bal) {
                const int leader = __ffs(bal) - 1;
                int mykey = N;
#pragma unroll
                for (int u = NPL - 1; u >= 0; --u) if (pend[u]) mykey = pi[u];
                const int K0 = __shfl_sync(0xffffffffu, mykey, leader);
                float pr = 0.f, pim = 0.f;
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    if (pend[u] && pi[u] == K0) { pr += wr[u]; pim += wi[u]; pend[u] = false; }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    pr += __shfl_xor_sync(0xffffffffu, pr, o);
                    if constexpr (NC == 2) pim += __shfl_xor_sync(0xffffffffu, pim, o);
                }
                if (lane == 0) obuf[K0] = mk<NC>(pr, pim);
                anyp = 0;
#pragma unroll
                for (int u = 0; u < NPL; ++u) anyp |= pend[u];
                bal = __ballot_sync(0xffffffffu, anyp);
            }
            __syncwarp();
            if (c + 1 < a.C) {
                float nr[NPL], ni[NPL];
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const SV o = obuf[lane * NPL + u];
                    nr[u] = re_of<NC>(o) + bre[u];
                    ni[u] = im_of<NC>(o) + bim[u];
                }
                const size_t cn = ci + 1;
                vst_f<NPL>(a.cs.carry + cn * row + lane * NPL, nr);
                if constexpr (NC == 2) vst_f<NPL>(a.cs.carry + cn * row + N + lane * NPL, ni);
                if (a.maps) {
#pragma unroll
                    for (int u = 0; u < NPL; ++u)
                        a.maps[((size_t)s * (a.C + 1) + c + 1) * N + lane * NPL + u] = key[mp[u]];
                }
                __threadfence();
                __syncwarp();
                if (lane == 0) st_release(a.ctrl + 1 + cn, 1u);
            } else if (a.maps) {
#pragma unroll
                for (int u = 0; u < NPL; ++u) a.maps[((size_t)s * (a.C + 1) + c + 1) * N + lane * NPL + u] = key[mp[u]];
            }
            if (a.maps) {
#pragma unroll
                for (int u = 0; u < NPL; ++u) a.maps[((size_t)s * (a.C + 1) + c) * N + lane * NPL + u] = (uint16_t)mp[u];
            }
            __syncwarp();
        }
        // ---------------- Phase C: replay from carry_c (L2-resident re-read)
        {
            Planes<NC, NPL> Dn, Bn;
            int kn = load_k(a.kstar, (size_t)s * a.L + t0, a.K, 0);
            load_diag_own<T, NC, NPL, PD>(a, ((size_t)s * a.L + t0) * row, h, kn, lane, Dn);
            load_planes<T, NC, NPL>(bias + ((size_t)s * a.L + t0) * row + lane * NPL, Bn, N);
            for (int t = t0; t < t1; ++t) {
                const int buf = (t - t0) & 1;
                const int k = kn;
                Planes<NC, NPL> D = Dn, Bv = Bn;
                if (t + 1 < t1) {
                    kn = load_k(a.kstar, (size_t)s * a.L + t + 1, a.K, 0);
                    load_diag_own<T, NC, NPL, PD>(a, ((size_t)s * a.L + t + 1) * row, h, kn, lane, Dn);
                    load_planes<T, NC, NPL>(bias + ((size_t)s * a.L + t + 1) * row + lane * NPL, Bn, N);
                }
                const int e = h * a.K + k;
                const uint32_t hd = __ldg(a.hdr + 2 * e);
                const uint32_t ovf = __ldg(a.hdr + 2 * e + 1);
                Rec<NPL> r;
                load_rec<NPL>(a.rec, e, lane, r);
                float vre[NPL], vim[NPL];
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const float di = NC == 2 ? D.v[NC - 1][u] : 0.f;
                    vre[u] = D.v[0][u] * cre[u] - di * cim[u];
                    vim[u] = D.v[0][u] * cim[u] + di * cre[u];
                }
                sts_row<NC, NPL>(vb[buf], lane, vre, vim);
                __syncwarp();
                float are[NPL], aim[NPL];
#pragma unroll
                for (int u = 0; u < NPL; ++u) { are[u] = 0.f; aim[u] = 0.f; }
                if (ovf) gather_sum_csr<NC, NPL>(vb[buf], a.pstart, a.psrc, e, N, lane, are, aim);
                else gather_sum<NC, NPL>(vb[buf], r, hd, are, aim);
                Planes<NC, NPL> hn;
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    cre[u] = are[u] + Bv.v[0][u];
                    cim[u] = NC == 2 ? aim[u] + Bv.v[NC - 1][u] : 0.f;
                    hn.v[0][u] = cre[u];
                    if constexpr (NC == 2) hn.v[NC - 1][u] = cim[u];
                }
                store_planes<T, NC, NPL>(hout + ((size_t)s * a.L + t) * row + lane * NPL, hn, N);
            }
        }
    }
}

// ============================================================================
// backward (transposed scan, reverse chunk order)
// ============================================================================
template <typename T, typename TE, int NC, int NPL, bool PD>
__global__ void __launch_bounds__(WARPS * 32) k_bwd_fused(FusedArgs a) {
    using SV = typename SVal<NC>::type;
    constexpr int NMAX = 32 * NPL;
    __shared__ SV s_l[WARPS][2][NMAX];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = a.N;
    const int total = a.S * a.C;
    const TE* ein = static_cast<const TE*>(a.bias);
    const T* hs = static_cast<const T*>(a.hsaved);
    T* dbias = static_cast<T*>(a.out0);
    const size_t row = (size_t)NC * N;
    while (true) {
        __syncwarp();
        int ticket = 0;
        if (lane == 0) ticket = atomicAdd(a.ctrl, 1u);
        ticket = __shfl_sync(0xffffffffu, ticket, 0);
        if (ticket >= total) break;
        const int cr = ticket / a.S, s = ticket - cr * a.S, h = s % a.H;
        const int c = a.C - 1 - cr;
        const int t0 = c * a.tau, t1 = min(t0 + a.tau, a.L);
        const size_t ci = (size_t)s * a.C + c;
        auto load_e = [&](int t, Planes<NC, NPL>& E) {
            if (ein) load_planes<TE, NC, NPL>(ein + ((size_t)s * a.L + t) * row + lane * NPL, E, N);
            else {
#pragma unroll
                for (int p = 0; p < NC; ++p)
#pragma unroll
                    for (int u = 0; u < NPL; ++u) E.v[p][u] = 0.f;
            }
        };
        auto load_P = [&](int k, int (&P)[NPL]) {
            const uint16_t* p = a.dict_idx + (size_t)(h * a.K + k) * N + lane * NPL;
            if constexpr (NPL == 4) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
                P[0] = v.x & 0xffff; P[1] = v.x >> 16; P[2] = v.y & 0xffff; P[3] = v.y >> 16;
            } else if constexpr (NPL == 2) {
                const uint32_t v = __ldg(reinterpret_cast<const unsigned int*>(p));
                P[0] = v & 0xffff; P[1] = v >> 16;
            } else {
                P[0] = __ldg(p);
            }
#pragma unroll
            for (int u = 0; u < NPL; ++u) P[u] = min(P[u], N - 1);
        };
        // ---------------- Phase A': reverse local scan, zero incoming
        float lre[NPL], lim[NPL], bpre[NPL], bpim[NPL];
        {
            Planes<NC, NPL> E;
            load_e(t1 - 1, E);
#pragma unroll
            for (int u = 0; u < NPL; ++u) { lre[u] = E.v[0][u]; lim[u] = NC == 2 ? E.v[NC - 1][u] : 0.f; }
            Planes<NC, NPL> Dn, En;
            int kn = load_k(a.kstar, (size_t)s * a.L + (t1 - 1), a.K, 0);
            load_diag_own<T, NC, NPL, PD>(a, ((size_t)s * a.L + (t1 - 1)) * row, h, kn, lane, Dn);
            if (t1 - 1 > t0) load_e(t1 - 2, En);
            for (int t = t1 - 1; t >= t0; --t) {
                const int buf = (t1 - 1 - t) & 1;
                const int k = kn;
                Planes<NC, NPL> D = Dn, Ep = En;
                if (t - 1 >= t0) {
                    kn = load_k(a.kstar, (size_t)s * a.L + t - 1, a.K, 0);
                    load_diag_own<T, NC, NPL, PD>(a, ((size_t)s * a.L + t - 1) * row, h, kn, lane, Dn);
                    if (t - 2 >= t0) load_e(t - 2, En);
                }
                int P[NPL];
                load_P(k, P);
                sts_row<NC, NPL>(s_l[w][buf], lane, lre, lim);
                __syncwarp();
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const SV lp = s_l[w][buf][P[u]];
                    const float dr = D.v[0][u], di = NC == 2 ? D.v[NC - 1][u] : 0.f;
                    // conj(D) * lamP
                    const float br = dr * re_of<NC>(lp) + di * im_of<NC>(lp);
                    const float bi = dr * im_of<NC>(lp) - di * re_of<NC>(lp);
                    if (t > t0) { lre[u] = Ep.v[0][u] + br; lim[u] = (NC == 2 ? Ep.v[NC - 1][u] : 0.f) + bi; }
                    else { bpre[u] = br; bpim[u] = bi; }
                }
            }
        }
        // ---------------- chain: mu_c (wait) -> mu_{c-1} = beta'_c + Abar_c^T mu_c (publish)
        float mre[NPL], mim[NPL];
        if (c == a.C - 1) {
#pragma unroll
            for (int u = 0; u < NPL; ++u) { mre[u] = 0.f; mim[u] = 0.f; }
            if (a.lam_in) {
                vld<float, NPL>(a.lam_in + (size_t)s * row + lane * NPL, mre);
                if constexpr (NC == 2) vld<float, NPL>(a.lam_in + (size_t)s * row + N + lane * NPL, mim);
            }
        } else {
            wait_flag(a.ctrl + 1 + ci);
            vld_cg<NPL>(a.mu + ci * row + lane * NPL, mre);
            if constexpr (NC == 2) vld_cg<NPL>(a.mu + ci * row + N + lane * NPL, mim);
        }
        {
            __syncwarp();            // Phase A''s last smem reads are done
            sts_row<NC, NPL>(s_l[w][0], lane, mre, mim);
            __syncwarp();
            float nr[NPL], ni[NPL];
#pragma unroll
            for (int u = 0; u < NPL; ++u) {
                const int j = lane * NPL + u;
                const int pj = min((int)a.cs.pi[ci * N + j], N - 1);
                const float dr = a.cs.d[ci * row + j], di = NC == 2 ? a.cs.d[ci * row + N + j] : 0.f;
                const SV mp = s_l[w][0][pj];
                nr[u] = bpre[u] + dr * re_of<NC>(mp) + di * im_of<NC>(mp);
                ni[u] = bpim[u] + dr * im_of<NC>(mp) - di * re_of<NC>(mp);
            }
            if (c > 0) {
                const size_t cp = ci - 1;
                vst_f<NPL>(a.mu + cp * row + lane * NPL, nr);
                if constexpr (NC == 2) vst_f<NPL>(a.mu + cp * row + N + lane * NPL, ni);
                __threadfence();
                __syncwarp();
                if (lane == 0) st_release(a.ctrl + 1 + cp, 1u);
            } else if (a.dh0) {
                vst_f<NPL>(a.dh0 + (size_t)s * row + lane * NPL, nr);
                if constexpr (NC == 2) vst_f<NPL>(a.dh0 + (size_t)s * row + N + lane * NPL, ni);
            }
            __syncwarp();
        }
        // ---------------- Phase C': replay, emit db, dD, g
        {
            Planes<NC, NPL> E;
            load_e(t1 - 1, E);
#pragma unroll
            for (int u = 0; u < NPL; ++u) { lre[u] = E.v[0][u] + mre[u]; lim[u] = (NC == 2 ? E.v[NC - 1][u] : 0.f) + mim[u]; }
            Planes<NC, NPL> Dn, En, Hn;
            int kn = load_k(a.kstar, (size_t)s * a.L + (t1 - 1), a.K, 0);
            load_diag_own<T, NC, NPL, PD>(a, ((size_t)s * a.L + (t1 - 1)) * row, h, kn, lane, Dn);
            if (t1 - 1 > t0) load_e(t1 - 2, En);
            auto load_h = [&](int t, Planes<NC, NPL>& Hp) {   // h_{t-1}
                if (t > 0) load_planes<T, NC, NPL>(hs + ((size_t)s * a.L + t - 1) * row + lane * NPL, Hp, N);
                else {
#pragma unroll
                    for (int p = 0; p < NC; ++p)
#pragma unroll
                        for (int u = 0; u < NPL; ++u) Hp.v[p][u] = 0.f;
                    if (a.h0) {
                        vld<float, NPL>(a.h0 + (size_t)s * row + lane * NPL, Hp.v[0]);
                        if constexpr (NC == 2) vld<float, NPL>(a.h0 + (size_t)s * row + N + lane * NPL, Hp.v[1]);
                    }
                }
            };
            load_h(t1 - 1, Hn);
            for (int t = t1 - 1; t >= t0; --t) {
                const int buf = (t1 - 1 - t) & 1;
                const int k = kn;
                Planes<NC, NPL> D = Dn, Ep = En, Hp = Hn;
                if (t - 1 >= t0) {
                    kn = load_k(a.kstar, (size_t)s * a.L + t - 1, a.K, 0);
                    load_diag_own<T, NC, NPL, PD>(a, ((size_t)s * a.L + t - 1) * row, h, kn, lane, Dn);
                    if (t - 2 >= t0) load_e(t - 2, En);
                    load_h(t - 1, Hn);
                }
                int P[NPL];
                load_P(k, P);
                const size_t off = ((size_t)s * a.L + t) * row + lane * NPL;
                {
                    Planes<NC, NPL> Lv;
#pragma unroll
                    for (int u = 0; u < NPL; ++u) { Lv.v[0][u] = lre[u]; if constexpr (NC == 2) Lv.v[NC - 1][u] = lim[u]; }
                    store_planes<T, NC, NPL>(dbias + off, Lv, N);
                }
                sts_row<NC, NPL>(s_l[w][buf], lane, lre, lim);
                __syncwarp();
                Planes<NC, NPL> dD;
                float gv = 0.f;
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const SV lp = s_l[w][buf][P[u]];
                    const float lr = re_of<NC>(lp), li = im_of<NC>(lp);
                    const float dr = D.v[0][u], di = NC == 2 ? D.v[NC - 1][u] : 0.f;
                    const float hr = Hp.v[0][u], hi = NC == 2 ? Hp.v[NC - 1][u] : 0.f;
                    // dD = conj(h) * lamP
                    dD.v[0][u] = hr * lr + hi * li;
                    if constexpr (NC == 2) dD.v[NC - 1][u] = hr * li - hi * lr;
                    // g += Re(conj(lamP) * D * h)
                    const float pr = dr * hr - di * hi, pim = dr * hi + di * hr;
                    gv += lr * pr + li * pim;
                    if (t > t0) {
                        lre[u] = Ep.v[0][u] + dr * lr + di * li;
                        lim[u] = (NC == 2 ? Ep.v[NC - 1][u] : 0.f) + dr * li - di * lr;
                    }
                }
                if constexpr (PD) store_planes<float, NC, NPL>(static_cast<float*>(a.out1) + off, dD, N);
                else store_planes<T, NC, NPL>(static_cast<T*>(a.out1) + off, dD, N);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) gv += __shfl_xor_sync(0xffffffffu, gv, o);
                if (a.gsel && lane == 0) a.gsel[(size_t)s * a.L + t] = gv;
            }
        }
    }
}

}  // namespace fused

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------
inline size_t fused_plan_bytes(int64_t H, int64_t K, int NPL) {
    return (((size_t)H * K * 32 * NPL * fused::MU + 255) & ~(size_t)255) + (((size_t)H * K * 8 + 255) & ~(size_t)255);
}

inline size_t fused_ctrl_bytes(int64_t S, int C) { return (((size_t)(1 + S * C) * 4 + 255) & ~(size_t)255); }

inline size_t fused_ws_bytes(int64_t S, int C) { return fused_ctrl_bytes(S, C); }

inline int fused_npl(int64_t N) {
    if (N == 32) return 1;
    if (N == 64) return 2;
    if (N == 128) return 4;
    return 0;
}

inline int fused_grid(int total_items) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const int ctas_per_sm = 2;
    int g = sms * ctas_per_sm;
    const int need = (total_items + fused::WARPS - 1) / fused::WARPS;
    return g < need ? g : need;
}

}  // namespace pdssm
