// Fused single-pass chunked scan for sm_100a (fast path of pdssm_scan_fwd /
// pdssm_scan_bwd).  Algorithm 1 re-blocked for B200:
//
//  * one WARP per (sequence, chunk) item; lane l owns the NPL = N/32 contiguous
//    states [l*NPL, l*NPL+NPL), so all own-state traffic is 16-byte vectors and
//    the intra-step exchange needs only __syncwarp;
//  * every per-step input row (D_t, b_t or e_{t-1}, h_{t-1}, the selected index
//    row P_{k*_t}, the preimage records and header of entry k*_t) is streamed
//    into a per-warp shared-memory ring by 1-D TMA bulk copies
//    (cp.async.bulk + mbarrier complete_tx), PF steps ahead of use, so a step
//    never waits on a global load;
//  * Phase A (aggregate), the carry hand-off and Phase C (replay) run in ONE
//    launch: a warp finishes Phase A, waits for its predecessor's carry
//    (chained look-back over per-(sequence, chunk) flags; dynamic tickets in
//    chunk-major order guarantee forward progress), publishes its own carry,
//    then replays the chunk.  The ring runs over the concatenated Phase A /
//    Phase C step list, so the replay's re-read (L2-resident: measured 18 TB/s
//    L2 vs 6.9 TB/s HBM, tools/l2bw.cu) is in flight during the carry wait, and
//    HBM sees each input once -- the algorithmic byte count of SURVEY §8(d);
//  * the scatter (A_t v)[i] = sum_{j : P_t[j] = i} D_t[j] v[j] is a gather over
//    a per-dictionary-entry, per-lane padded preimage list ("fused plan", MU
//    inline sources per target, longer preimages fall back to the CSR plan):
//    deterministic, no float atomics;
//  * the backward is the transposed scan (a pure gather) with the same
//    structure in reverse chunk order, reusing the forward (pi_bar, d_bar).
#pragma once
#include <type_traits>

#include "k_scan_fwd.cuh"

namespace pdssm {
namespace fused {

constexpr int MU = 6;         // inline preimage capacity per target
constexpr int TAUMAX = 256;   // fused-path chunk-length cap (k* staged in smem)
#ifndef PDSSM_PF_FWD
#define PDSSM_PF_FWD 3
#endif
#ifndef PDSSM_PF_BWD
#define PDSSM_PF_BWD 2
#endif
constexpr int PF_FWD = PDSSM_PF_FWD;     // ring slots (groups of Layout::G steps) per warp
constexpr int PF_BWD = PDSSM_PF_BWD;

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

// the same from shared memory
template <typename T, int NPL>
__device__ __forceinline__ void sld(const T* p, float (&o)[NPL]) {
    if constexpr (std::is_same<T, float>::value) {
        if constexpr (NPL == 4) {
            const float4 v = *reinterpret_cast<const float4*>(p);
            o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
        } else if constexpr (NPL == 2) {
            const float2 v = *reinterpret_cast<const float2*>(p);
            o[0] = v.x; o[1] = v.y;
        } else {
            o[0] = *p;
        }
    } else {
        if constexpr (NPL == 4) {
            const uint2 v = *reinterpret_cast<const uint2*>(p);
            o[0] = __uint_as_float(v.x << 16); o[1] = __uint_as_float(v.x & 0xffff0000u);
            o[2] = __uint_as_float(v.y << 16); o[3] = __uint_as_float(v.y & 0xffff0000u);
        } else if constexpr (NPL == 2) {
            const uint32_t v = *reinterpret_cast<const uint32_t*>(p);
            o[0] = __uint_as_float(v << 16); o[1] = __uint_as_float(v & 0xffff0000u);
        } else {
            o[0] = __bfloat162float(*p);
        }
    }
}

template <typename T>
__device__ __forceinline__ float sld1(const T* p) {
    if constexpr (std::is_same<T, float>::value) return *p;
    else return __bfloat162float(*p);
}

// NPL uint16 index values from shared memory (clamped into [0, N))
template <int NPL>
__device__ __forceinline__ void sld_idx(const uint16_t* p, int N, int (&P)[NPL]) {
    if constexpr (NPL == 4) {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        P[0] = v.x & 0xffff; P[1] = v.x >> 16; P[2] = v.y & 0xffff; P[3] = v.y >> 16;
    } else if constexpr (NPL == 2) {
        const uint32_t v = *reinterpret_cast<const uint32_t*>(p);
        P[0] = v & 0xffff; P[1] = v >> 16;
    } else {
        P[0] = *p;
    }
#pragma unroll
    for (int u = 0; u < NPL; ++u) P[u] = min(P[u], N - 1);
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

// per-step own-state planes: x[NC][NPL]
template <int NC, int NPL>
struct Planes {
    float v[NC][NPL];
};

template <typename T, int NC, int NPL>
__device__ __forceinline__ void store_planes(T* __restrict__ base, const Planes<NC, NPL>& o, int N) {
    vst<T, NPL>(base, o.v[0]);
    if constexpr (NC == 2) vst<T, NPL>(base + N, o.v[1]);
}

// streamed output stores with an L2 evict_first policy (never re-read in this launch)
template <typename T, int NPL>
__device__ __forceinline__ void vst_stream(T* p, const float (&v)[NPL], uint64_t pol) {
    if constexpr (std::is_same<T, float>::value && NPL == 4) {
        asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v[0]), "f"(v[1]),
                     "f"(v[2]), "f"(v[3]), "l"(pol)
                     : "memory");
    } else if constexpr (std::is_same<T, float>::value && NPL == 2) {
        asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v[0]), "f"(v[1]), "l"(pol)
                     : "memory");
    } else if constexpr (std::is_same<T, float>::value) {
        asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v[0]), "l"(pol) : "memory");
    } else if constexpr (NPL == 4) {
        asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(pack_bf16x2(v[0], v[1])),
                     "r"(pack_bf16x2(v[2], v[3])), "l"(pol)
                     : "memory");
    } else if constexpr (NPL == 2) {
        asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(pack_bf16x2(v[0], v[1])), "l"(pol)
                     : "memory");
    } else {
        vst<T, NPL>(p, v);
    }
}
template <typename T, int NC, int NPL>
__device__ __forceinline__ void store_planes_stream(T* __restrict__ base, const Planes<NC, NPL>& o, int N,
                                                    uint64_t pol) {
    vst_stream<T, NPL>(base, o.v[0], pol);
    if constexpr (NC == 2) vst_stream<T, NPL>(base + N, o.v[1], pol);
}

// ------------------------------------------------------------------ chain flags
// Producer: data stores, __threadfence (every lane), __syncwarp, st.release flag.
// Consumer: relaxed polling (no L1 invalidation per poll), then one acquire fence.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_flag(const uint32_t* p) {
    while (ld_relaxed(p) == 0u) __nanosleep(32);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// ------------------------------------------------------------------ TMA ring primitives
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_1d(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}
// L2 eviction-priority policies (createpolicy) and the cache-hinted bulk copy:
// Phase-A rows are kept (evict_last) for the replay's re-read, replay rows and all
// streamed outputs are evict_first, so the replay working set stays L2-resident.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_1d_hint(void* dst, const void* src, uint32_t bytes, uint64_t* b, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------------ exchange values
template <int NC> struct SVal;
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
// Exchange-buffer position of state i (N = 32 * NPL): lane l owns states l*NPL + u in
// registers, and slot u of every lane forms one contiguous 32-element row, so the
// owners' stores and read-backs are conflict-free (one wavefront per 128 B).  The
// zero sentinel sits at position N.
template <int NPL>
__host__ __device__ constexpr int xpos(int i) { return NPL == 1 ? i : (i % NPL) * 32 + i / NPL; }

template <int NC, int NPL>
__device__ __forceinline__ void sts_row(typename SVal<NC>::type* row, int lane, const float (&re)[NPL],
                                        const float (&im)[NPL]) {
#pragma unroll
    for (int u = 0; u < NPL; ++u) row[u * 32 + lane] = mk<NC>(re[u], im[u]);
}

// ------------------------------------------------------------------ fused plan
// The gather that realises the scatter (A_t v)[i] = sum_{j : P_t[j] = i} v[j] is
// balanced per dictionary entry: targets are ranked by in-degree (descending,
// ties by index) and rank r is computed by lane r % 32 in slot u = r / 32, so the
// warp-uniform trip count of slot u, M_u = max in-degree inside the slot, is
// small (random maps, N = 128: sum_u M_u = 7.0 on average vs 14.1 for the
// natural i -> (i / NPL, i % NPL) assignment).  The computing lane writes the
// target's sum to the exchange buffer; the owner of state i reads it back.
// Record of (entry e, lane l), 32 bytes: byte u (< NPL) = target of slot u, then
// per slot u its sources (ascending j) at REC_SOFF[u], at most REC_SCAP[u] of them,
// padded with the sentinel N (a zero slot of the exchange buffer).
// hdr[e] = {M_0 | M_1<<8 | M_2<<16 | M_3<<24, ovf, e, 0}; ovf != 0 if some slot
// exceeds its capacity (then the CSR plan is used for that step).
// Fixed per-slot capacities (unconditional, branch-free gathers; the zero sentinel pads):
// slot 0 holds the highest in-degrees (<= 6), slot 1 <= 2, slots 2-3 <= 1 -- the
// in-degree profile of random maps; entries that do not fit take the CSR path.
// Record entries are uint16 BYTE offsets into the exchange buffer (index * element
// size), so a gather is one extract + one add + one LDS.
__host__ __device__ constexpr int rec_scap(int u) { return u == 0 ? 6 : u == 1 ? 2 : 1; }
__host__ __device__ constexpr int rec_soff(int u) { return u == 0 ? 4 : u == 1 ? 10 : u == 2 ? 12 : 13; }   // in u16 units

template <int NPL>
struct Rec {
    static constexpr int B = 32;   // record bytes per lane: 4 target + 10 source u16 offsets (+2 pad)
    static constexpr int W = B / 4;
    uint32_t w[W];
};

// Records of one entry are stored as two 512-byte halves [2][32 lanes][16 B] so that a
// warp reads its records with two conflict-free 16-byte loads; u16 field idx of lane l:
__device__ __forceinline__ uint16_t& rec_u16(uint8_t* entry, int l, int idx) {
    return reinterpret_cast<uint16_t*>(entry + (idx >> 3) * 512 + l * 16)[idx & 7];
}
template <int NPL>
__device__ __forceinline__ void rec_load(const uint8_t* entry, int lane, Rec<NPL>& r) {
    const uint4 lo = *reinterpret_cast<const uint4*>(entry + lane * 16);
    const uint4 hi = *reinterpret_cast<const uint4*>(entry + 512 + lane * 16);
    r.w[0] = lo.x; r.w[1] = lo.y; r.w[2] = lo.z; r.w[3] = lo.w;
    r.w[4] = hi.x; r.w[5] = hi.y; r.w[6] = hi.z; r.w[7] = hi.w;
}

template <int NPL>
__global__ void k_build_fused_plan(const uint16_t* __restrict__ dict_idx, uint8_t* __restrict__ rec,
                                   uint32_t* __restrict__ hdr, uint16_t* __restrict__ pclamp, int N, int sv,
                                   uint32_t flags) {
    extern __shared__ uint16_t sP[];   // [N] clamped row, then [N] in-degrees
    __shared__ int smax[8];
    __shared__ int sovf;
    uint16_t* sdeg = sP + N;
    const int e = blockIdx.x;
    const uint16_t* P = dict_idx + (size_t)e * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        int p = P[j];
        if (p >= N) {
            if (flags & PDSSM_CHECK_FINITE) report(ERRBIT_RANGE);
            p = N - 1;
        }
        sP[j] = (uint16_t)p;
        pclamp[(size_t)e * N + j] = (uint16_t)p;   // clamped index rows used by the fused kernels
    }
    if (threadIdx.x < 8) smax[threadIdx.x] = 0;
    if (threadIdx.x == 0) sovf = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        int d = 0;
        for (int j = 0; j < N; ++j) d += sP[j] == i;
        sdeg[i] = (uint16_t)d;
    }
    __syncthreads();
    constexpr int RB = Rec<NPL>::B;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int di = sdeg[i];
        int rank = 0;
        for (int i2 = 0; i2 < N; ++i2) {
            const int d2 = sdeg[i2];
            rank += (d2 > di) || (d2 == di && i2 < i);
        }
        const int l = rank % 32, u = rank / 32;
        uint8_t* re = rec + (size_t)e * 32 * RB;
        rec_u16(re, l, u) = (uint16_t)(xpos<NPL>(i) * sv);
        int q = 0;
        for (int j = 0; j < N; ++j) {
            if (sP[j] == i) {
                if (q < rec_scap(u)) rec_u16(re, l, rec_soff(u) + q) = (uint16_t)(xpos<NPL>(j) * sv);
                ++q;
            }
        }
        for (int qq = q; qq < rec_scap(u); ++qq) rec_u16(re, l, rec_soff(u) + qq) = (uint16_t)(N * sv);
        atomicMax(&smax[u], q);
        if (q > rec_scap(u)) sovf = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t h = 0;
        for (int u = 0; u < NPL; ++u) h |= (uint32_t)min(smax[u], rec_scap(u)) << (8 * u);   // informative
        hdr[4 * e] = h;
        hdr[4 * e + 1] = sovf ? 1u : 0u;
        hdr[4 * e + 2] = (uint32_t)e;   // entry index (CSR fallback)
        hdr[4 * e + 3] = 0u;
    }
}

template <int NPL>
__device__ __forceinline__ uint32_t rec_off(const Rec<NPL>& r, int idx) {   // u16 entry idx (compile-time)
    return (idx & 1) ? (r.w[idx >> 1] >> 16) : (r.w[idx >> 1] & 0xffffu);
}

// Balanced, branch-free gather: sum over the slot's (padded) source list, written
// to s[target_u].  Padding reads the zero slot v[N] (a broadcast, no conflict).
template <int NC, int NPL>
__device__ __forceinline__ void gather_sorted(const typename SVal<NC>::type* vbuf, typename SVal<NC>::type* sbuf,
                                              const Rec<NPL>& r) {
#pragma unroll
    for (int u = 0; u < NPL; ++u) {
        using SVT = typename SVal<NC>::type;
        const char* vb = reinterpret_cast<const char*>(vbuf);
        const SVT v0 = *reinterpret_cast<const SVT*>(vb + rec_off<NPL>(r, rec_soff(u)));
        float ar = re_of<NC>(v0), ai = im_of<NC>(v0);
#pragma unroll
        for (int q = 1; q < rec_scap(u); ++q) {
            const SVT v = *reinterpret_cast<const SVT*>(vb + rec_off<NPL>(r, rec_soff(u) + q));
            ar += re_of<NC>(v);
            if constexpr (NC == 2) ai += im_of<NC>(v);
        }
        *reinterpret_cast<SVT*>(reinterpret_cast<char*>(sbuf) + rec_off<NPL>(r, u)) = mk<NC>(ar, ai);
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
            const auto v = vbuf[xpos<NPL>(__ldg(psrc + (size_t)e * N + q))];
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
    const uint16_t* pclamp;  // fwd: clamped copy of dict_idx (fused plan)
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
    float* mu;               // bwd: [S][C][NC][N]  mu_c, adjoint entering chunk c from later chunks
    float* betap;            // bwd: [S][C][NC][N]  beta'_c, the chunk's transposed aggregate
    uint32_t* ctrl;          // [0] ticket counter, [1..S*C] flags
    int H, L, N, K, tau, C, S;
    uint32_t flags;
    int debug_nochain;       // timing experiments only (PDSSM_DEBUG_NOCHAIN): skip the carry wait
    int smem_tables;         // 1: the CTA's home-head tables live in shared memory
};


// x <- Abar x + beta for one chunk aggregate (pi, d, beta) held as this lane's NPL
// source slices: out[i] = beta[i] + sum_{j : pi[j] = i} d[j] x[j].  Unique targets are
// stored directly; colliding groups are reduced by a fixed xor-butterfly per distinct
// key (ballot loop) -- deterministic, no float atomics.  Optionally composes the
// index map m <- pi[m] (gather through the key row).
template <int NC, int NPL>
__device__ __forceinline__ void apply_aggregate(int lane, int N, uint16_t* key, int* cnt, typename SVal<NC>::type* obuf,
                                                const int (&pi)[NPL], const float (&dre)[NPL], const float (&dim)[NPL],
                                                const float (&bre)[NPL], const float (&bim)[NPL], float (&xr)[NPL],
                                                float (&xi)[NPL], int* mp) {
    __syncwarp();   // previous users of key / cnt / obuf are done
    float wr[NPL], wi[NPL];
#pragma unroll
    for (int u = 0; u < NPL; ++u) {
        wr[u] = dre[u] * xr[u] - dim[u] * xi[u];
        wi[u] = dre[u] * xi[u] + dim[u] * xr[u];
        key[lane * NPL + u] = (uint16_t)pi[u];
        obuf[lane * NPL + u] = mk<NC>(0.f, 0.f);
        cnt[lane * NPL + u] = 0;
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < NPL; ++u) atomicAdd(&cnt[pi[u]], 1);   // integer counts: order-independent
    __syncwarp();
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
        for (int u = NPL - 1; u >= 0; --u)
            if (pend[u]) mykey = pi[u];
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
#pragma unroll
    for (int u = 0; u < NPL; ++u) {
        const auto o = obuf[lane * NPL + u];
        xr[u] = re_of<NC>(o) + bre[u];
        xi[u] = im_of<NC>(o) + bim[u];
        if (mp) mp[u] = key[mp[u]];
    }
    __syncwarp();   // the buffers alias the exchange rows of the next phase
}


__host__ __device__ constexpr size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

// ============================================================================
// CTA = WARPS independent consumer warps, one CTA per SM (persistent).
//  * head affinity: warps of CTA i take tickets of head h = i mod H first (per-head
//    ticket counters), so the head's small per-entry tables (index rows, preimage
//    records, headers) stay L1-resident and are read with plain loads;
//  * each warp streams its per-step rows (D_t, b_t / e_{t-1}, h_{t-1}) into a
//    private ring of PF slots of G consecutive steps with 1-D TMA bulk copies
//    (one copy per stream per slot: G rows are contiguous in HBM), issued by the
//    warp itself once per G steps, PF*G steps ahead, across item boundaries.
// ============================================================================
#ifndef PDSSM_WARPS_FWD
#define PDSSM_WARPS_FWD 11
#endif
#ifndef PDSSM_WARPS_BWD
#define PDSSM_WARPS_BWD 11
#endif
#ifndef PDSSM_G_FWD
#define PDSSM_G_FWD 2
#endif
#ifndef PDSSM_G_BWD
#define PDSSM_G_BWD 2
#endif
constexpr int WARPS_FWD = PDSSM_WARPS_FWD;   // consumer warps (= items in flight) per CTA: the minimum
constexpr int WARPS_BWD = PDSSM_WARPS_BWD;   // the host launches (fused_warps); one CTA per SM
#ifndef PDSSM_WARPS_MAX
#define PDSSM_WARPS_MAX 15
#endif
constexpr int WARPS_MAX = PDSSM_WARPS_MAX;   // launch bound: 480 threads -> <= 136 registers (the kernels use <= 127)

template <typename T, int NC, int NPL, bool PD, bool BWD, int ESZ = (int)sizeof(T)>
struct Layout {
    static constexpr int WARPS = BWD ? WARPS_BWD : WARPS_FWD;
    static constexpr int THREADS = WARPS * 32;
    static constexpr int G = BWD ? PDSSM_G_BWD : PDSSM_G_FWD;  // steps per ring slot
    static constexpr int N = 32 * NPL;
    static constexpr int ROW = NC * N * (int)sizeof(T);      // one D / b / h row (act dtype)
    static constexpr int EROW = NC * N * ESZ;                 // one e row (bwd)
    static constexpr int DG = PD ? 0 : G * ROW;               // D rows per slot (PER_DICT: none)
    static constexpr int OFF_B = DG;                          // fwd b rows
    static constexpr int OFF_E = DG;                          // bwd e rows
    static constexpr int OFF_H = DG + G * EROW;           // bwd h rows
    static constexpr int SLOT = (int)al16(BWD ? OFF_H + G * ROW : OFF_B + G * ROW);
    static constexpr int PF = BWD ? PF_BWD : PF_FWD;          // slots in flight
    static constexpr int SV = NC == 2 ? 8 : 4;
    static constexpr size_t w_ring = 0;
    static constexpr size_t w_bar = al16(w_ring + (size_t)PF * SLOT);
    static constexpr size_t w_x = al16(w_bar + (size_t)PF * 8);              // exchange [2][N+1]
    static constexpr size_t x_end = al16(w_x + (size_t)2 * (N + 1) * SV);
    // fwd chain buffers (apply_aggregate runs between the phases, when the exchange rows
    // are idle): complex -- result [N] over the second row, keys u16 [N] and counts int [N]
    // over the first row below its zero sentinel; real -- separate
    static constexpr bool ALIAS = NC == 2;
    static constexpr size_t w_ob = ALIAS ? w_x + (size_t)(N + 1) * SV : x_end;
    static constexpr size_t w_key = ALIAS ? w_x : al16(w_ob + (BWD ? 0 : (size_t)N * SV));
    static constexpr size_t w_cnt = ALIAS ? w_x + (size_t)N * 2 : al16(w_key + (BWD ? 0 : (size_t)N * 2));
    static constexpr size_t w_k = ALIAS ? x_end : al16(w_cnt + (BWD ? 0 : (size_t)N * 4));   // k* of the chunk [TAUMAX]
    static constexpr size_t w_g = al16(w_k + TAUMAX);                        // bwd g partials [32][33]
    static constexpr size_t w_bytes = al16(w_g + (BWD ? 32 * 33 * 4 : 0));
    static constexpr size_t bytes = (size_t)WARPS * w_bytes;
    // CTA-shared tables of the home head (after the warps' blocks), K entries:
    //   P rows u16 [K][N] (clamped), fwd: records [K][32][Rec::B] and headers [K][4] u32,
    //   PER_DICT: diagonal rows f32 [K][NC][N]
    static constexpr size_t t_P = 0;
    __host__ __device__ static constexpr size_t t_rec(int K) { return al16(t_P + (size_t)K * N * 2); }
    __host__ __device__ static constexpr size_t t_hdr(int K) { return al16(t_rec(K) + (BWD ? 0 : (size_t)K * 32 * Rec<NPL>::B)); }
    __host__ __device__ static constexpr size_t t_dk(int K) { return al16(t_hdr(K) + (BWD ? 0 : (size_t)K * 16)); }
    __host__ __device__ static constexpr size_t t_bytes(int K) { return al16(t_dk(K) + (PD ? (size_t)K * NC * N * 4 : 0)); }
};

// CTA-cooperative copy of the home head's tables into shared memory
template <typename LY, bool BWD, bool PD, int NC, int NPL>
__device__ __forceinline__ void load_tables(const FusedArgs& a, uint8_t* tb, int h) {
    const int K = a.K, N = a.N;
    uint16_t* sP = reinterpret_cast<uint16_t*>(tb + LY::t_P);
    const uint16_t* gP = a.dict_idx + (size_t)h * K * N;
    // fwd: natural state indices (the pi composition indexes D rows); bwd: exchange positions
    for (int i = threadIdx.x; i < K * N; i += blockDim.x) {
        const int p = min((int)__ldg(gP + i), N - 1);
        sP[i] = (uint16_t)(BWD ? xpos<NPL>(p) : p);
    }
    if constexpr (!BWD) {
        const uint4* gr = reinterpret_cast<const uint4*>(a.rec + (size_t)h * K * 32 * Rec<NPL>::B);
        uint4* sr = reinterpret_cast<uint4*>(tb + LY::t_rec(K));
        const int nr = K * 32 * Rec<NPL>::B / 16;
        for (int i = threadIdx.x; i < nr; i += blockDim.x) sr[i] = __ldg(gr + i);
        const uint4* gh = reinterpret_cast<const uint4*>(a.hdr + (size_t)h * K * 4);
        uint4* sh = reinterpret_cast<uint4*>(tb + LY::t_hdr(K));
        for (int i = threadIdx.x; i < K; i += blockDim.x) sh[i] = __ldg(gh + i);
    }
    if constexpr (PD) {
        const float* gd = a.diag_dict + (size_t)h * K * NC * N;
        float* sd = reinterpret_cast<float*>(tb + LY::t_dk(K));
        for (int i = threadIdx.x; i < K * NC * N; i += blockDim.x) sd[i] = __ldg(gd + i);
    }
}

template <bool PD, typename T>
using DType = typename std::conditional<PD, float, T>::type;

struct Item {
    int ticket, c, s, h, t0, t1, n;
};

// per-head tickets: ticket in [0, B*C): chunk-major (reverse for the backward)
__device__ __forceinline__ Item make_item(const FusedArgs& a, int h, int ticket, bool reverse) {
    Item it;
    it.ticket = ticket;
    const int B = a.S / a.H;
    const int cr = ticket / B;
    const int b = ticket - cr * B;
    it.h = h;
    it.s = b * a.H + h;
    it.c = reverse ? a.C - 1 - cr : cr;
    it.t0 = it.c * a.tau;
    it.t1 = min(it.t0 + a.tau, a.L);
    it.n = it.t1 - it.t0;
    return it;
}

// next item of head h for this warp (per-head ticket counter)
__device__ __forceinline__ bool next_item(const FusedArgs& a, int h, int lane, bool reverse, Item& it) {
    const int per_head = (a.S / a.H) * a.C;
    int t = 0;
    if (lane == 0) t = (int)atomicAdd(a.ctrl + h, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t < per_head) {
        it = make_item(a, h, t, reverse);
        return true;
    }
    return false;
}

__device__ __forceinline__ uint32_t* flag_ptr(const FusedArgs& a, size_t ci) { return a.ctrl + a.H + ci; }

// item k* bytes, prefetched one item ahead: lane i holds bytes i, i+32, ...
struct KPre {
    uint32_t b[TAUMAX / 32];
};
__device__ __forceinline__ void kpre_load(const FusedArgs& a, KPre& kp, const Item& it, int lane) {
#pragma unroll
    for (int i = 0; i < TAUMAX / 32; ++i) {
        const int idx = lane + 32 * i;
        kp.b[i] = idx < it.n ? (uint32_t)__ldg(a.kstar + (size_t)it.s * a.L + it.t0 + idx) : 0u;
    }
}
__device__ __forceinline__ void kpre_store(const FusedArgs& a, const KPre& kp, uint8_t* sk, int n, int lane,
                                           bool check) {
#pragma unroll
    for (int i = 0; i < TAUMAX / 32; ++i) {
        const int idx = lane + 32 * i;
        if (idx < n) {
            int k = (int)kp.b[i];
            if (k >= a.K) {
                if (check && (a.flags & PDSSM_CHECK_FINITE)) report(ERRBIT_RANGE);
                k = a.K - 1;
            }
            sk[idx] = (uint8_t)k;
        }
    }
}

// ---------------------------------------------------------------------------
// ring fill cursor: virtual group stream of the current item, then the next one.
// An item has 2*ng groups (Phase A groups, then Phase C groups), ng = ceil(n/G).
// ---------------------------------------------------------------------------
struct FillCursor {
    Item it[2];        // [0] item being filled, [1] the one after (if known)
    bool valid[2];
    int g;             // next virtual group of it[0]
    uint32_t q;        // total fills issued (slot = q % PF)
};

template <typename T, typename TE, int NC, int NPL, bool PD, bool BWD>
__device__ __forceinline__ void issue_fill(const FusedArgs& a, const Item& it, int g, uint8_t* ring, uint64_t* bars,
                                           int slot, uint64_t pol_last, uint64_t pol_first) {
    using LY = Layout<T, NC, NPL, PD, BWD, (int)sizeof(TE)>;
    constexpr int N = LY::N;
    constexpr size_t row = (size_t)NC * N;
    const size_t seq0 = (size_t)it.s * a.L;
    const int ng = (it.n + LY::G - 1) / LY::G;
    const bool phC = g >= ng;
    const int gi = phC ? g - ng : g;
    const int v0 = gi * LY::G;
    const int len = min(LY::G, it.n - v0);
    uint8_t* dst = ring + (size_t)slot * LY::SLOT;
    uint64_t* bar = bars + slot;
    // WAR on the slot: its previous contents were consumed (generic-proxy reads whose
    // values were used) before this lane reached here, in program order after __syncwarp
    const uint64_t pol = phC ? pol_first : pol_last;
    if constexpr (!BWD) {
        const int t = it.t0 + v0;   // rows t .. t+len-1 at slot offsets 0..len-1
        mbar_expect_tx(bar, (uint32_t)((PD ? 0 : len * LY::ROW) + len * LY::ROW));
        if constexpr (!PD) tma_1d_hint(dst, static_cast<const T*>(a.diag) + (seq0 + t) * row, len * LY::ROW, bar, pol);
        tma_1d_hint(dst + LY::OFF_B, static_cast<const T*>(a.bias) + (seq0 + t) * row, len * LY::ROW, bar, pol);
    } else {
        // steps v0..v0+len-1 are times t_hi = t1-1-v0 down to t_lo = t_hi-len+1; the row
        // of time t sits at slot offset (t - t_lo) for D, e_{t-1} and h_{t-1}
        const int t_hi = it.t1 - 1 - v0;
        const int t_lo = t_hi - len + 1;
        const TE* ein = static_cast<const TE*>(a.bias);
        const int e_first = max(t_lo - 1, it.t0);   // e_{t-1} needed for t > t0
        const int e_cnt = ein ? max(0, t_hi - 1 - e_first + 1) : 0;
        const int h_first = max(t_lo - 1, 0);       // h_{t-1} needed for t > 0 (Phase C' only)
        const int h_cnt = phC ? max(0, t_hi - 1 - h_first + 1) : 0;
        mbar_expect_tx(bar, (uint32_t)((PD ? 0 : len * LY::ROW) + e_cnt * LY::EROW + h_cnt * LY::ROW));
        if constexpr (!PD) tma_1d_hint(dst, static_cast<const T*>(a.diag) + (seq0 + t_lo) * row, len * LY::ROW, bar, pol);
        if (e_cnt > 0)
            tma_1d_hint(dst + LY::OFF_E + (size_t)(e_first - (t_lo - 1)) * LY::EROW, ein + (seq0 + e_first) * row,
                        e_cnt * LY::EROW, bar, pol);
        if (h_cnt > 0)
            tma_1d_hint(dst + LY::OFF_H + (size_t)(h_first - (t_lo - 1)) * LY::ROW,
                        static_cast<const T*>(a.hsaved) + (seq0 + h_first) * row, h_cnt * LY::ROW, bar, pol_first);
    }
}

// issue fills while fewer than PF are outstanding ahead of `consumed`
template <typename T, typename TE, int NC, int NPL, bool PD, bool BWD>
__device__ __forceinline__ void pump(const FusedArgs& a, FillCursor& fc, uint32_t consumed, uint8_t* ring,
                                     uint64_t* bars, int lane, uint64_t pol_last, uint64_t pol_first) {
    using LY = Layout<T, NC, NPL, PD, BWD, (int)sizeof(TE)>;
    constexpr int PF = LY::PF;
    while (fc.q < consumed + PF) {
        if (!fc.valid[0]) break;
        const int ng = (fc.it[0].n + LY::G - 1) / LY::G;
        if (fc.g >= 2 * ng) {
            if (!fc.valid[1]) break;
            fc.it[0] = fc.it[1];
            fc.valid[1] = false;
            fc.g = 0;
            continue;
        }
        if (lane == 0 && !(a.debug_nochain & 2))
            issue_fill<T, TE, NC, NPL, PD, BWD>(a, fc.it[0], fc.g, ring, bars, (int)(fc.q % PF), pol_last, pol_first);
        ++fc.g;
        ++fc.q;
    }
}

// ============================================================================
// forward
// ============================================================================
template <typename T, int NC, int NPL, bool PD>
__global__ void __launch_bounds__(WARPS_MAX * 32, 1) k_fwd_fused(FusedArgs a) {
    using SV = typename SVal<NC>::type;
    using LY = Layout<T, NC, NPL, PD, false>;
    using DT = DType<PD, T>;
    constexpr int PF = LY::PF;
    extern __shared__ __align__(128) uint8_t smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* base = smem + (size_t)w * LY::w_bytes;
    uint8_t* ring = base + LY::w_ring;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + LY::w_bar);
    SV* xb = reinterpret_cast<SV*>(base + LY::w_x);
    SV* obuf = reinterpret_cast<SV*>(base + LY::w_ob);
    uint16_t* key = reinterpret_cast<uint16_t*>(base + LY::w_key);
    int* cnt = reinterpret_cast<int*>(base + LY::w_cnt);
    uint8_t* sk = base + LY::w_k;
    constexpr int N = LY::N;
    constexpr size_t row = (size_t)NC * N;
    if (lane == 0) {
        for (int i = 0; i < PF; ++i) mbar_init(bars + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        xb[N] = mk<NC>(0.f, 0.f);
        xb[(N + 1) + N] = mk<NC>(0.f, 0.f);
    }
    __syncwarp();
    // one scatter step: z = A_t-scatter of v (own slices in, own target sums out).
    // v -> vbuf, sync, balanced gather -> sbuf[target], sync, own sums <- sbuf.
    SV* vbuf = xb;
    SV* sbuf = xb + (N + 1);
    auto scatter_step = [&](const float (&vr)[NPL], const float (&vi)[NPL], const Rec<NPL>& r, const uint4& hd, int e,
                            float (&zr)[NPL], float (&zi)[NPL]) {
        sts_row<NC, NPL>(vbuf, lane, vr, vi);
        __syncwarp();
        if (hd.y) {
            float cr[NPL], ci[NPL];
#pragma unroll
            for (int u = 0; u < NPL; ++u) { cr[u] = 0.f; ci[u] = 0.f; }
            gather_sum_csr<NC, NPL>(vbuf, a.pstart, a.psrc, e, N, lane, cr, ci);
            sts_row<NC, NPL>(sbuf, lane, cr, ci);
        } else {
            gather_sorted<NC, NPL>(vbuf, sbuf, r);
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < NPL; ++u) {
            const SV z = sbuf[u * 32 + lane];
            zr[u] = re_of<NC>(z);
            zi[u] = im_of<NC>(z);
        }
    };
    const uint64_t pol_out = policy_evict_first();
    const uint64_t pol_last = policy_evict_last();
    uint8_t* tbl = smem + (size_t)(blockDim.x >> 5) * LY::w_bytes;   // after every warp's block
    FillCursor fc;
    fc.q = 0;
    uint32_t consumed = 0;        // groups consumed
    // heads of this CTA: blockIdx % H when grid = (SMs / H) * H >= H, else blockIdx, + grid, ...
    for (int head = blockIdx.x % a.H; head < a.H; head += gridDim.x) {
    __syncthreads();
    load_tables<LY, false, PD, NC, NPL>(a, tbl, head);
    __syncthreads();
    fc.valid[0] = next_item(a, head, lane, false, fc.it[0]);
    fc.valid[1] = false;
    fc.g = 0;
    KPre kp;
    if (fc.valid[0]) kpre_load(a, kp, fc.it[0], lane);
    bool have = fc.valid[0];
    Item it = fc.it[0];
    while (have) {
        // the item after this one (ticket prefetch) so the ring can run across items
        Item nx;
        const bool has_next = next_item(a, head, lane, false, nx);
        if (has_next) { fc.it[1] = nx; fc.valid[1] = true; }
        const int c = it.c, s = it.s, h = it.h, n = it.n;
        const int ng = (n + LY::G - 1) / LY::G;
        const size_t ci = (size_t)s * a.C + c;
        __syncwarp();
        kpre_store(a, kp, sk, n, lane, true);
        if (has_next) kpre_load(a, kp, nx, lane);
        __syncwarp();
        pump<T, T, NC, NPL, PD, false>(a, fc, consumed, ring, bars, lane, pol_last, pol_out);
        // per-entry tables of this head, in shared memory
        const uint16_t* prow_base = reinterpret_cast<const uint16_t*>(tbl + LY::t_P);
        const uint8_t* rec_base = tbl + LY::t_rec(a.K);
        const uint32_t* hdr_base = reinterpret_cast<const uint32_t*>(tbl + LY::t_hdr(a.K));
        const float* dk_base = reinterpret_cast<const float*>(tbl + LY::t_dk(a.K));
        // ---------------- Phase A: aggregate from identity
        int pi[NPL];
        float dre[NPL], dim[NPL], bre[NPL], bim[NPL];
#pragma unroll
        for (int u = 0; u < NPL; ++u) { pi[u] = lane * NPL + u; dre[u] = 1.f; dim[u] = 0.f; bre[u] = 0.f; bim[u] = 0.f; }
        // per-step table prefetch (L1): record words + header of entry k*_{v+1}
        Rec<NPL> rn;
        uint4 hn;
        {
            const int k0 = sk[0];
            rec_load<NPL>(rec_base + (size_t)k0 * 32 * Rec<NPL>::B, lane, rn);
            hn = *reinterpret_cast<const uint4*>(hdr_base + 4 * k0);
        }
        for (int gi = 0; gi < ng; ++gi) {
            const int slot = consumed % PF;
            if (!(a.debug_nochain & 2)) mbar_wait(bars + slot, (consumed / PF) & 1);
            const uint8_t* sp = ring + (size_t)slot * LY::SLOT;
            const int len = min(LY::G, n - gi * LY::G);
#pragma unroll
            for (int i = 0; i < LY::G; ++i) {
                if (i >= len) break;
                const int v = gi * LY::G + i;
                const int k = sk[v];
                const Rec<NPL> r = rn;
                const uint4 hd = hn;
                {
                    const int kn = sk[v + 1 < n ? v + 1 : v];
                    rec_load<NPL>(rec_base + (size_t)kn * 32 * Rec<NPL>::B, lane, rn);
                    hn = *reinterpret_cast<const uint4*>(hdr_base + 4 * kn);
                }
                Planes<NC, NPL> D, Bv;
                const DT* Dp;
                if constexpr (PD) Dp = dk_base + (size_t)k * NC * N;
                else Dp = reinterpret_cast<const T*>(sp) + (size_t)i * row;
                sld<DT, NPL>(Dp + lane * NPL, D.v[0]);
                if constexpr (NC == 2) sld<DT, NPL>(Dp + N + lane * NPL, D.v[1]);
                const T* Bp = reinterpret_cast<const T*>(sp + LY::OFF_B) + (size_t)i * row;
                sld<T, NPL>(Bp + lane * NPL, Bv.v[0]);
                if constexpr (NC == 2) sld<T, NPL>(Bp + N + lane * NPL, Bv.v[1]);
                if (a.flags & PDSSM_CHECK_FINITE) {
#pragma unroll
                    for (int u = 0; u < NPL; ++u) {
                        check_cpx(cpx{D.v[0][u], D.v[NC - 1][u]}, a.flags);
                        check_cpx(cpx{Bv.v[0][u], Bv.v[NC - 1][u]}, a.flags);
                    }
                }
                // pi / d update: d <- D_t[pi] d, pi <- P_t[pi]
                const uint16_t* prow = prow_base + (size_t)k * N;
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    float pr, pm;
                    pr = sld1<DT>(Dp + pi[u]);
                    pm = NC == 2 ? sld1<DT>(Dp + N + pi[u]) : 0.f;
                    const float nr = pr * dre[u] - pm * dim[u];
                    const float ni = pr * dim[u] + pm * dre[u];
                    dre[u] = nr; dim[u] = ni;
                    pi[u] = prow[pi[u]];   // rows are pre-clamped (plan build / table load)
                }
                float vre[NPL], vim[NPL];
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const float di = NC == 2 ? D.v[NC - 1][u] : 0.f;
                    vre[u] = D.v[0][u] * bre[u] - di * bim[u];
                    vim[u] = D.v[0][u] * bim[u] + di * bre[u];
                }
                float zr[NPL], zi[NPL];
                scatter_step(vre, vim, r, hd, h * a.K + k, zr, zi);
#pragma unroll
                for (int u = 0; u < NPL; ++u) { bre[u] = zr[u] + Bv.v[0][u]; bim[u] = NC == 2 ? zi[u] + Bv.v[NC - 1][u] : 0.f; }
            }
            // slot fully read (the syncwarp of the group's last step orders every lane's reads
            // except this step's pi-gathers, which the next syncwarp covers)
            __syncwarp();
            ++consumed;
            pump<T, T, NC, NPL, PD, false>(a, fc, consumed, ring, bars, lane, pol_last, pol_out);
        }
        // publish the aggregate (chunk_state sections 0-2), then flag = 1 ("aggregate ready")
#pragma unroll
        for (int u = 0; u < NPL; ++u) a.cs.pi[ci * N + lane * NPL + u] = (uint16_t)pi[u];
        vst_f<NPL>(a.cs.d + ci * row + lane * NPL, dre);
        vst_f<NPL>(a.cs.beta + ci * row + lane * NPL, bre);
        if constexpr (NC == 2) {
            vst_f<NPL>(a.cs.d + ci * row + N + lane * NPL, dim);
            vst_f<NPL>(a.cs.beta + ci * row + N + lane * NPL, bim);
        }
        if (c + 1 < a.C) {
            __threadfence();
            __syncwarp();
            if (lane == 0) st_release(flag_ptr(a, ci), 1u);
        }
        // ---------------- decoupled look-back for carry_c: fold the aggregates of the chunks
        // between the nearest predecessor that already published its inclusive carry
        // (flag 2) and this chunk.  The fold repeats exactly the chain's arithmetic
        // carry_{m+1} = Abar_m carry_m + beta_bar_m, so the result does not depend on
        // which predecessor was found (bitwise deterministic).
        float cre[NPL], cim[NPL];
        int mp[NPL];                 // exclusive prefix map before this chunk (maps export)
        {
            int mP = -1;             // carry_{mP+1} is known; -1: carry_0 = h0
            if (c > 0 && !(a.debug_nochain & 1)) {
                while (true) {
                    const int m = c - 1 - lane;
                    const uint32_t f = m >= 0 ? ld_relaxed(flag_ptr(a, (size_t)s * a.C + m)) : 2u;
                    const uint32_t b2 = __ballot_sync(0xffffffffu, f == 2u);
                    const uint32_t b0 = __ballot_sync(0xffffffffu, f == 0u);
                    if (b2) {
                        const int first = __ffs(b2) - 1;
                        if ((b0 & ((1u << first) - 1u)) == 0u) { mP = c - 1 - first; break; }
                    }
                    __nanosleep(64);
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else if (c > 0) {
                mP = c - 1;
            }
            if (mP < 0) {
#pragma unroll
                for (int u = 0; u < NPL; ++u) { cre[u] = 0.f; cim[u] = 0.f; mp[u] = lane * NPL + u; }
                if (a.h0) {
                    vld<float, NPL>(a.h0 + (size_t)s * row + lane * NPL, cre);
                    if constexpr (NC == 2) vld<float, NPL>(a.h0 + (size_t)s * row + N + lane * NPL, cim);
                }
            } else {
                const size_t cm = (size_t)s * a.C + mP + 1;
                vld_cg<NPL>(a.cs.carry + cm * row + lane * NPL, cre);
                if constexpr (NC == 2) vld_cg<NPL>(a.cs.carry + cm * row + N + lane * NPL, cim);
                if (a.maps) {
#pragma unroll
                    for (int u = 0; u < NPL; ++u)
                        mp[u] = __ldcg(a.maps + ((size_t)s * (a.C + 1) + mP + 1) * N + lane * NPL + u);
                }
            }
            for (int m = mP + 1; m < c; ++m) {
                const size_t cm = (size_t)s * a.C + m;
                int pk[NPL];
                float pdr[NPL], pdi[NPL], pbr[NPL], pbi[NPL];
#pragma unroll
                for (int u = 0; u < NPL; ++u) { pk[u] = min((int)__ldcg(a.cs.pi + cm * N + lane * NPL + u), N - 1); pdi[u] = 0.f; pbi[u] = 0.f; }
                vld_cg<NPL>(a.cs.d + cm * row + lane * NPL, pdr);
                vld_cg<NPL>(a.cs.beta + cm * row + lane * NPL, pbr);
                if constexpr (NC == 2) {
                    vld_cg<NPL>(a.cs.d + cm * row + N + lane * NPL, pdi);
                    vld_cg<NPL>(a.cs.beta + cm * row + N + lane * NPL, pbi);
                }
                apply_aggregate<NC, NPL>(lane, N, key, cnt, obuf, pk, pdr, pdi, pbr, pbi, cre, cim, a.maps ? mp : nullptr);
            }
            if (c > 0 && mP + 1 < c) {   // carry_c computed here (duplicates of the chain's value are bitwise equal)
                vst_f<NPL>(a.cs.carry + ci * row + lane * NPL, cre);
                if constexpr (NC == 2) vst_f<NPL>(a.cs.carry + ci * row + N + lane * NPL, cim);
            }
            if (c == 0) {
                vst_f<NPL>(a.cs.carry + ci * row + lane * NPL, cre);
                if constexpr (NC == 2) vst_f<NPL>(a.cs.carry + ci * row + N + lane * NPL, cim);
            }
            if (a.maps) {
#pragma unroll
                for (int u = 0; u < NPL; ++u) a.maps[((size_t)s * (a.C + 1) + c) * N + lane * NPL + u] = (uint16_t)mp[u];
            }
        }
        // ---------------- inclusive carry_{c+1} = Abar_c carry_c + beta_bar_c, flag = 2
        {
            float nr[NPL], ni[NPL];
            int mq[NPL];
#pragma unroll
            for (int u = 0; u < NPL; ++u) { nr[u] = cre[u]; ni[u] = cim[u]; mq[u] = mp[u]; }
            apply_aggregate<NC, NPL>(lane, N, key, cnt, obuf, pi, dre, dim, bre, bim, nr, ni, a.maps ? mq : nullptr);
            if (c + 1 < a.C) {
                const size_t cn = ci + 1;
                vst_f<NPL>(a.cs.carry + cn * row + lane * NPL, nr);
                if constexpr (NC == 2) vst_f<NPL>(a.cs.carry + cn * row + N + lane * NPL, ni);
            }
            if (a.maps) {
#pragma unroll
                for (int u = 0; u < NPL; ++u) a.maps[((size_t)s * (a.C + 1) + c + 1) * N + lane * NPL + u] = (uint16_t)mq[u];
            }
            if (c + 1 < a.C) {
                __threadfence();
                __syncwarp();
                if (lane == 0) st_release(flag_ptr(a, ci), 2u);
            }
            __syncwarp();
        }
        // ---------------- Phase C: replay from carry_c (its slots were prefetched meanwhile)
        T* hout = static_cast<T*>(a.out0) + ((size_t)s * a.L + it.t0) * row + lane * NPL;
        {
            const int k0 = sk[0];
            rec_load<NPL>(rec_base + (size_t)k0 * 32 * Rec<NPL>::B, lane, rn);
            hn = *reinterpret_cast<const uint4*>(hdr_base + 4 * k0);
        }
        for (int gi = 0; gi < ng; ++gi) {
            const int slot = consumed % PF;
            if (!(a.debug_nochain & 2)) mbar_wait(bars + slot, (consumed / PF) & 1);
            const uint8_t* sp = ring + (size_t)slot * LY::SLOT;
            const int len = min(LY::G, n - gi * LY::G);
#pragma unroll
            for (int i = 0; i < LY::G; ++i) {
                if (i >= len) break;
                const int v = gi * LY::G + i;
                const int k = sk[v];
                const Rec<NPL> r = rn;
                const uint4 hd = hn;
                {
                    const int kn = sk[v + 1 < n ? v + 1 : v];
                    rec_load<NPL>(rec_base + (size_t)kn * 32 * Rec<NPL>::B, lane, rn);
                    hn = *reinterpret_cast<const uint4*>(hdr_base + 4 * kn);
                }
                Planes<NC, NPL> D, Bv;
                if constexpr (PD) {
                    const float* Dp = dk_base + (size_t)k * NC * N;
                    sld<float, NPL>(Dp + lane * NPL, D.v[0]);
                    if constexpr (NC == 2) sld<float, NPL>(Dp + N + lane * NPL, D.v[1]);
                } else {
                    const T* Dp = reinterpret_cast<const T*>(sp) + (size_t)i * row;
                    sld<T, NPL>(Dp + lane * NPL, D.v[0]);
                    if constexpr (NC == 2) sld<T, NPL>(Dp + N + lane * NPL, D.v[1]);
                }
                const T* Bp = reinterpret_cast<const T*>(sp + LY::OFF_B) + (size_t)i * row;
                sld<T, NPL>(Bp + lane * NPL, Bv.v[0]);
                if constexpr (NC == 2) sld<T, NPL>(Bp + N + lane * NPL, Bv.v[1]);
                float vre[NPL], vim[NPL];
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const float di = NC == 2 ? D.v[NC - 1][u] : 0.f;
                    vre[u] = D.v[0][u] * cre[u] - di * cim[u];
                    vim[u] = D.v[0][u] * cim[u] + di * cre[u];
                }
                float zr[NPL], zi[NPL];
                scatter_step(vre, vim, r, hd, h * a.K + k, zr, zi);
                Planes<NC, NPL> hv;
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    cre[u] = zr[u] + Bv.v[0][u];
                    cim[u] = NC == 2 ? zi[u] + Bv.v[NC - 1][u] : 0.f;
                    hv.v[0][u] = cre[u];
                    if constexpr (NC == 2) hv.v[NC - 1][u] = cim[u];
                }
                store_planes_stream<T, NC, NPL>(hout, hv, N, pol_out);
                hout += row;
            }
            __syncwarp();
            ++consumed;
            pump<T, T, NC, NPL, PD, false>(a, fc, consumed, ring, bars, lane, pol_last, pol_out);
        }
        have = has_next;
        it = nx;
    }
    }   // head loop
}

// ============================================================================
// backward (transposed scan, reverse chunk order)
// ============================================================================
template <typename T, typename TE, int NC, int NPL, bool PD>
__global__ void __launch_bounds__(WARPS_MAX * 32, 1) k_bwd_fused(FusedArgs a) {
    using SV = typename SVal<NC>::type;
    using LY = Layout<T, NC, NPL, PD, true, (int)sizeof(TE)>;
    constexpr int PF = LY::PF;
    extern __shared__ __align__(128) uint8_t smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* base = smem + (size_t)w * LY::w_bytes;
    uint8_t* ring = base + LY::w_ring;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + LY::w_bar);
    SV* xb = reinterpret_cast<SV*>(base + LY::w_x);
    uint8_t* sk = base + LY::w_k;
    float* gbuf = reinterpret_cast<float*>(base + LY::w_g);   // [32][33] per-lane g partials
    constexpr int N = LY::N;
    constexpr size_t row = (size_t)NC * N;
    const TE* ein = static_cast<const TE*>(a.bias);
    if (lane == 0) {
        for (int i = 0; i < PF; ++i) mbar_init(bars + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint64_t pol_out = policy_evict_first();
    const uint64_t pol_last = policy_evict_last();
    uint8_t* tbl = smem + (size_t)(blockDim.x >> 5) * LY::w_bytes;   // after every warp's block
    FillCursor fc;
    fc.q = 0;
    uint32_t consumed = 0;
    for (int head = blockIdx.x % a.H; head < a.H; head += gridDim.x) {
    __syncthreads();
    load_tables<LY, true, PD, NC, NPL>(a, tbl, head);
    __syncthreads();
    fc.valid[0] = next_item(a, head, lane, true, fc.it[0]);
    fc.valid[1] = false;
    fc.g = 0;
    KPre kp;
    if (fc.valid[0]) kpre_load(a, kp, fc.it[0], lane);
    bool have = fc.valid[0];
    Item it = fc.it[0];
    while (have) {
        Item nx;
        const bool has_next = next_item(a, head, lane, true, nx);
        if (has_next) { fc.it[1] = nx; fc.valid[1] = true; }
        const int c = it.c, s = it.s, h = it.h, t0 = it.t0, t1 = it.t1, n = it.n;
        const int ng = (n + LY::G - 1) / LY::G;
        const size_t ci = (size_t)s * a.C + c;
        const size_t seq0 = (size_t)s * a.L;
        __syncwarp();
        kpre_store(a, kp, sk, n, lane, false);
        if (has_next) kpre_load(a, kp, nx, lane);
        __syncwarp();
        pump<T, TE, NC, NPL, PD, true>(a, fc, consumed, ring, bars, lane, pol_last, pol_out);
        const uint16_t* prow_base = reinterpret_cast<const uint16_t*>(tbl + LY::t_P) + lane * NPL;
        const float* dk_base = reinterpret_cast<const float*>(tbl + LY::t_dk(a.K));
        // index row slice of entry k: raw words loaded one step ahead, decoded at use
        auto load_P = [&](int k) -> uint2 {
            const uint16_t* p = prow_base + (size_t)k * N;
            if constexpr (NPL == 4) return *reinterpret_cast<const uint2*>(p);
            else if constexpr (NPL == 2) return make_uint2(*reinterpret_cast<const unsigned int*>(p), 0u);
            else return make_uint2((uint32_t)*p, 0u);
        };
        auto decode_P = [&](uint2 vv, int (&P)[NPL]) {
            if constexpr (NPL == 4) { P[0] = vv.x & 0xffff; P[1] = vv.x >> 16; P[2] = vv.y & 0xffff; P[3] = vv.y >> 16; }
            else if constexpr (NPL == 2) { P[0] = vv.x & 0xffff; P[1] = vv.x >> 16; }
            else { P[0] = vv.x; }   // table rows hold clamped exchange positions
        };
        auto load_D = [&](const uint8_t* sp, int ro, int k, Planes<NC, NPL>& D) {
            if constexpr (PD) {
                const float* Dp = dk_base + (size_t)k * NC * N + lane * NPL;
                sld<float, NPL>(Dp, D.v[0]);
                if constexpr (NC == 2) sld<float, NPL>(Dp + N, D.v[1]);
            } else {
                const T* Dp = reinterpret_cast<const T*>(sp) + (size_t)ro * row + lane * NPL;
                sld<T, NPL>(Dp, D.v[0]);
                if constexpr (NC == 2) sld<T, NPL>(Dp + N, D.v[1]);
            }
        };
        auto load_e_direct = [&](int t, float (&er)[NPL], float (&ei)[NPL]) {
#pragma unroll
            for (int u = 0; u < NPL; ++u) { er[u] = 0.f; ei[u] = 0.f; }
            if (ein) {
                vld<TE, NPL>(ein + (seq0 + t) * row + lane * NPL, er);
                if constexpr (NC == 2) vld<TE, NPL>(ein + (seq0 + t) * row + N + lane * NPL, ei);
            }
        };
        // ---------------- Phase A': reverse local scan from zero incoming adjoint
        float lre[NPL], lim[NPL], bpre[NPL], bpim[NPL];
        load_e_direct(t1 - 1, lre, lim);
        uint2 Pn = load_P(sk[n - 1]);
        for (int gi = 0; gi < ng; ++gi) {
            const int slot = consumed % PF;
            if (!(a.debug_nochain & 2)) mbar_wait(bars + slot, (consumed / PF) & 1);
            const uint8_t* sp = ring + (size_t)slot * LY::SLOT;
            const int len = min(LY::G, n - gi * LY::G);
#pragma unroll
            for (int i = 0; i < LY::G; ++i) {
                if (i >= len) break;
                const int v = gi * LY::G + i;
                const int t = t1 - 1 - v;
                const int ro = len - 1 - i;           // row offset of time t in the slot
                const int k = sk[t - t0];
                int P[NPL];
                decode_P(Pn, P);
                if (t > t0) Pn = load_P(sk[t - 1 - t0]);
                Planes<NC, NPL> D;
                load_D(sp, ro, k, D);
                float er[NPL], ei[NPL];
#pragma unroll
                for (int u = 0; u < NPL; ++u) { er[u] = 0.f; ei[u] = 0.f; }
                if (ein && t > t0) {
                    const TE* ep = reinterpret_cast<const TE*>(sp + LY::OFF_E) + (size_t)ro * row + lane * NPL;
                    sld<TE, NPL>(ep, er);
                    if constexpr (NC == 2) sld<TE, NPL>(ep + N, ei);
                }
                SV* lb = xb + (v & 1) * (N + 1);
                sts_row<NC, NPL>(lb, lane, lre, lim);
                __syncwarp();
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const SV lp = lb[P[u]];
                    const float dr = D.v[0][u], di = NC == 2 ? D.v[NC - 1][u] : 0.f;
                    lre[u] = er[u] + dr * re_of<NC>(lp) + di * im_of<NC>(lp);   // e_{t-1} + conj(D) lamP
                    lim[u] = ei[u] + dr * im_of<NC>(lp) - di * re_of<NC>(lp);
                }
            }
            ++consumed;
            pump<T, TE, NC, NPL, PD, true>(a, fc, consumed, ring, bars, lane, pol_last, pol_out);
        }
#pragma unroll
        for (int u = 0; u < NPL; ++u) { bpre[u] = lre[u]; bpim[u] = lim[u]; }   // beta'_c (e term was zero at t0)
        // publish beta'_c (the chunk's aggregate for the transposed scan), flag = 1
        if (c > 0) {
            vst_f<NPL>(a.betap + ci * row + lane * NPL, bpre);
            if constexpr (NC == 2) vst_f<NPL>(a.betap + ci * row + N + lane * NPL, bpim);
            __threadfence();
            __syncwarp();
            if (lane == 0) st_release(flag_ptr(a, ci), 1u);
        }
        // ---------------- decoupled look-forward for mu_c (adjoint entering this chunk's last
        // step from the chunks after it): fold beta'_m + Abar_m^T (.) of the successors
        // between this chunk and the nearest one that already published its inclusive
        // value (flag 2: mu_{m-1} ready).  Same arithmetic as the chain: deterministic.
        // Abar_m^T is a pure gather that reuses the forward (pi_bar, d_bar).
        auto applyT = [&](const int (&pk)[NPL], const float (&dr)[NPL], const float (&di)[NPL], const float (&br)[NPL],
                          const float (&bi)[NPL], float (&xr)[NPL], float (&xi)[NPL]) {
            SV* xbuf = xb;
            __syncwarp();
            sts_row<NC, NPL>(xbuf, lane, xr, xi);
            __syncwarp();
#pragma unroll
            for (int u = 0; u < NPL; ++u) {
                const SV xp = xbuf[xpos<NPL>(pk[u])];
                xr[u] = br[u] + dr[u] * re_of<NC>(xp) + di[u] * im_of<NC>(xp);   // beta' + conj(d) x[pi]
                xi[u] = bi[u] + dr[u] * im_of<NC>(xp) - di[u] * re_of<NC>(xp);
            }
        };
        auto load_fwd_agg = [&](size_t cm, int (&pk)[NPL], float (&dr)[NPL], float (&di)[NPL]) {
#pragma unroll
            for (int u = 0; u < NPL; ++u) { pk[u] = min((int)__ldg(a.cs.pi + cm * N + lane * NPL + u), N - 1); di[u] = 0.f; }
            vld<float, NPL>(a.cs.d + cm * row + lane * NPL, dr);
            if constexpr (NC == 2) vld<float, NPL>(a.cs.d + cm * row + N + lane * NPL, di);
        };
        float mre[NPL], mim[NPL];
        {
            int mP = a.C;            // mu_{mP-1} is known; C: mu_{C-1} = lam_in
            if (c + 1 < a.C && !(a.debug_nochain & 1)) {
                while (true) {
                    const int m = c + 1 + lane;
                    const uint32_t f = m < a.C ? ld_relaxed(flag_ptr(a, (size_t)s * a.C + m)) : 2u;
                    const uint32_t b2 = __ballot_sync(0xffffffffu, f == 2u);
                    const uint32_t b0 = __ballot_sync(0xffffffffu, f == 0u);
                    if (b2) {
                        const int first = __ffs(b2) - 1;
                        if ((b0 & ((1u << first) - 1u)) == 0u) { mP = c + 1 + first; break; }
                    }
                    __nanosleep(64);
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else if (c + 1 < a.C) {
                mP = c + 1;
            }
            if (mP >= a.C) {
#pragma unroll
                for (int u = 0; u < NPL; ++u) { mre[u] = 0.f; mim[u] = 0.f; }
                if (a.lam_in) {
                    vld<float, NPL>(a.lam_in + (size_t)s * row + lane * NPL, mre);
                    if constexpr (NC == 2) vld<float, NPL>(a.lam_in + (size_t)s * row + N + lane * NPL, mim);
                }
            } else {
                const size_t cm = (size_t)s * a.C + mP - 1;
                vld_cg<NPL>(a.mu + cm * row + lane * NPL, mre);
                if constexpr (NC == 2) vld_cg<NPL>(a.mu + cm * row + N + lane * NPL, mim);
            }
            for (int m = mP - 1; m > c; --m) {
                const size_t cm = (size_t)s * a.C + m;
                int pk[NPL];
                float dr[NPL], di[NPL], br[NPL], bi[NPL];
                load_fwd_agg(cm, pk, dr, di);
#pragma unroll
                for (int u = 0; u < NPL; ++u) bi[u] = 0.f;
                vld_cg<NPL>(a.betap + cm * row + lane * NPL, br);
                if constexpr (NC == 2) vld_cg<NPL>(a.betap + cm * row + N + lane * NPL, bi);
                applyT(pk, dr, di, br, bi, mre, mim);
            }
        }
        // ---------------- inclusive mu_{c-1} = beta'_c + Abar_c^T mu_c, flag = 2 (c > 0).  Chunk 0's
        // dh0 = A_0^T lambda_0 falls out of its replay below, so Abar_0 is never read (a chunk_state
        // written by the single-chunk forward carries no aggregate unless maps were exported).
        if (c > 0) {
            int pk[NPL];
            float dr[NPL], di[NPL], nr[NPL], ni[NPL];
            load_fwd_agg(ci, pk, dr, di);
#pragma unroll
            for (int u = 0; u < NPL; ++u) { nr[u] = mre[u]; ni[u] = mim[u]; }
            applyT(pk, dr, di, bpre, bpim, nr, ni);
            const size_t cp = ci - 1;
            vst_f<NPL>(a.mu + cp * row + lane * NPL, nr);
            if constexpr (NC == 2) vst_f<NPL>(a.mu + cp * row + N + lane * NPL, ni);
            __threadfence();
            __syncwarp();
            if (lane == 0) st_release(flag_ptr(a, ci), 2u);
        }
        __syncwarp();   // the exchange-row reads above (applyT) precede the replay's writes
        // ---------------- Phase C': replay, emit db, dD, g
        {
            float er0[NPL], ei0[NPL];
            load_e_direct(t1 - 1, er0, ei0);
#pragma unroll
            for (int u = 0; u < NPL; ++u) { lre[u] = er0[u] + mre[u]; lim[u] = ei0[u] + mim[u]; }
        }
        T* dbp = static_cast<T*>(a.out0) + (seq0 + t1 - 1) * row + lane * NPL;
        T* ddp = PD ? nullptr : static_cast<T*>(a.out1) + (seq0 + t1 - 1) * row + lane * NPL;
        float* ddf = PD ? static_cast<float*>(a.out1) + (seq0 + t1 - 1) * row + lane * NPL : nullptr;
        Pn = load_P(sk[n - 1]);
        for (int gi = 0; gi < ng; ++gi) {
            const int slot = consumed % PF;
            if (!(a.debug_nochain & 2)) mbar_wait(bars + slot, (consumed / PF) & 1);
            const uint8_t* sp = ring + (size_t)slot * LY::SLOT;
            const int len = min(LY::G, n - gi * LY::G);
#pragma unroll
            for (int i = 0; i < LY::G; ++i) {
                if (i >= len) break;
                const int v = gi * LY::G + i;
                const int t = t1 - 1 - v;
                const int ro = len - 1 - i;
                const int k = sk[t - t0];
                int P[NPL];
                decode_P(Pn, P);
                if (t > t0) Pn = load_P(sk[t - 1 - t0]);
                Planes<NC, NPL> D, Hp;
                load_D(sp, ro, k, D);
                float er[NPL], ei[NPL];
#pragma unroll
                for (int u = 0; u < NPL; ++u) { er[u] = 0.f; ei[u] = 0.f; }
                if (ein && t > t0) {
                    const TE* ep = reinterpret_cast<const TE*>(sp + LY::OFF_E) + (size_t)ro * row + lane * NPL;
                    sld<TE, NPL>(ep, er);
                    if constexpr (NC == 2) sld<TE, NPL>(ep + N, ei);
                }
                if (t > 0) {
                    const T* hp = reinterpret_cast<const T*>(sp + LY::OFF_H) + (size_t)ro * row + lane * NPL;
                    sld<T, NPL>(hp, Hp.v[0]);
                    if constexpr (NC == 2) sld<T, NPL>(hp + N, Hp.v[1]);
                } else {
#pragma unroll
                    for (int p = 0; p < NC; ++p)
#pragma unroll
                        for (int u = 0; u < NPL; ++u) Hp.v[p][u] = 0.f;
                    if (a.h0) {
                        vld<float, NPL>(a.h0 + (size_t)s * row + lane * NPL, Hp.v[0]);
                        if constexpr (NC == 2) vld<float, NPL>(a.h0 + (size_t)s * row + N + lane * NPL, Hp.v[1]);
                    }
                }
                {
                    Planes<NC, NPL> Lv;
#pragma unroll
                    for (int u = 0; u < NPL; ++u) { Lv.v[0][u] = lre[u]; if constexpr (NC == 2) Lv.v[NC - 1][u] = lim[u]; }
                    store_planes_stream<T, NC, NPL>(dbp, Lv, N, pol_out);
                }
                SV* lb = xb + (v & 1) * (N + 1);
                sts_row<NC, NPL>(lb, lane, lre, lim);
                __syncwarp();
                Planes<NC, NPL> dD;
                float gv = 0.f;
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const SV lp = lb[P[u]];
                    const float lr = re_of<NC>(lp), li = im_of<NC>(lp);
                    const float dr = D.v[0][u], di = NC == 2 ? D.v[NC - 1][u] : 0.f;
                    const float hr = Hp.v[0][u], hi = NC == 2 ? Hp.v[NC - 1][u] : 0.f;
                    dD.v[0][u] = hr * lr + hi * li;                       // conj(h) * lamP
                    if constexpr (NC == 2) dD.v[NC - 1][u] = hr * li - hi * lr;
                    const float pr = dr * hr - di * hi, pim = dr * hi + di * hr;
                    gv += lr * pr + li * pim;                             // Re(conj(lamP) D h)
                    lre[u] = er[u] + dr * lr + di * li;                   // e_{t-1} + conj(D) lamP
                    lim[u] = ei[u] + dr * li - di * lr;
                }
                if constexpr (PD) { store_planes_stream<float, NC, NPL>(ddf, dD, N, pol_out); ddf -= row; }
                else { store_planes_stream<T, NC, NPL>(ddp, dD, N, pol_out); ddp -= row; }
                dbp -= row;
                // g_t = sum over lanes of gv: park the partial, reduce 32 steps at a time
                gbuf[(v & 31) * 33 + lane] = gv;
                if ((v & 31) == 31 || v == n - 1) {
                    __syncwarp();
                    if (a.gsel && lane <= (v & 31)) {
                        float acc = 0.f;
#pragma unroll 8
                        for (int q = 0; q < 32; ++q) acc += gbuf[lane * 33 + q];
                        a.gsel[seq0 + (t1 - 1 - (v - (v & 31) + lane))] = acc;
                    }
                    __syncwarp();
                }
            }
            __syncwarp();
            ++consumed;
            pump<T, TE, NC, NPL, PD, true>(a, fc, consumed, ring, bars, lane, pol_last, pol_out);
        }
        if (c == 0 && a.dh0) {   // after t = 0 (no e_{-1} term): lambda = A_0^T lambda_0 = dh0
            vst_f<NPL>(a.dh0 + (size_t)s * row + lane * NPL, lre);
            if constexpr (NC == 2) vst_f<NPL>(a.dh0 + (size_t)s * row + N + lane * NPL, lim);
        }
        have = has_next;
        it = nx;
    }
    }   // head loop
}

}  // namespace fused


// ---------------------------------------------------------------------------
// host-side sizing helpers
// ---------------------------------------------------------------------------
inline size_t fused_rec_bytes(int64_t H, int64_t K) {
    return (((size_t)H * K * 32 * fused::Rec<4>::B) + 255) & ~(size_t)255;   // NPL = 4 is the largest record
}
inline size_t fused_hdr_bytes(int64_t H, int64_t K) { return (((size_t)H * K * 16) + 255) & ~(size_t)255; }
inline size_t fused_pclamp_bytes(int64_t H, int64_t K, int64_t N) { return (((size_t)H * K * N * 2) + 255) & ~(size_t)255; }
inline size_t fused_plan_bytes(int64_t H, int64_t K, int64_t N) { return fused_rec_bytes(H, K) + fused_hdr_bytes(H, K) + fused_pclamp_bytes(H, K, N); }

// [0, H): per-head ticket counters; then one flag per (sequence, chunk)
inline size_t fused_ctrl_bytes(int64_t S, int C, int64_t H) { return (((size_t)(H + S * C) * 4 + 255) & ~(size_t)255); }

inline int fused_npl(int64_t N) {
    if (N == 32) return 1;
    if (N == 64) return 2;
    if (N == 128) return 4;
    return 0;
}

// SM count of the current device, cached per device ordinal (a process may drive several GPUs)
inline int num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
    if (dev >= 64) {
        int s = 0;
        return cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && s > 0 ? s : 148;
    }
    if (!cache[dev]) {
        int s = 0;
        if (cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || s <= 0) s = 148;
        cache[dev] = s;
    }
    return cache[dev];
}

// persistent grid, one CTA per SM: the same number of CTAs for every head (CTA i serves
// head i mod H) when H <= #SMs, else #SMs CTAs that walk the heads i, i + grid, ...
inline int fused_grid(int64_t H) {
    const int sms = num_sms();
    if (H > sms) return sms;
    return (int)((sms / H) * H);
}

}  // namespace pdssm
