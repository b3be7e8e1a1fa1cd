// Dense contractions of the path on the 5th-generation tensor cores (tcgen05):
//   a2/a3  selector logits  logits[(b,t)][(h,k)] = sum_d x[b,t,d] S[h,k,d]   (Eq. 6)
//          with the hard-selection argmax fused into the TMEM epilogue      (Eq. 7)
//          and the optional P_t = dict_idx[h][k*] gather                    (Eq. 8)
//   a5     projection       b[b,h,t,(c,n)] = sum_d x[b,t,d] B[h,c,n,d]       (Eq. 1 b_t = B u_t,
//          PAPER.md:94-95, :970), written straight into the scan layout [B][H][L][c][N].
//
// One CTA computes a BM x BN tile (BM = 128 tokens, BN <= 256 output columns):
//   warp 0 (one lane)  TMA producer: 128-byte K slabs of x and of the weight rows into a
//                      STAGES-deep ring (SWIZZLE_128B, full/empty mbarriers);
//   warp 1 (one lane)  MMA issuer: tcgen05.mma cta_group::1, M=128, N=BN, K = 32 bytes per
//                      instruction (bf16: kind::f16, K=16; fp32: kind::tf32, K=8), fp32
//                      accumulators in TMEM; tcgen05.commit frees ring slots;
//   warp 2             TMEM allocator (BN columns rounded to a power of two);
//   warps 4-7          epilogue: warp 4+q reads TMEM lanes 32q..32q+31 (= tile rows) with
//                      tcgen05.ld 32x32b and applies the fused epilogue.
// Operands are K-major (the HBM layouts of x, S and B), so no transposes are needed.
#pragma once
#include "pdssm_common.cuh"

#include <cuda.h>

namespace pdssm {
namespace tc {

constexpr int BM = 128;
constexpr int ROWB = 128;   // K bytes per ring slot row = one 128-byte swizzle atom
constexpr int THREADS = 512;   // 0 TMA, 1 MMA, 2 TMEM, 4-7 epilogue, 8-15 tf32 split
constexpr int NCONV = 8;       // converter warps

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra TC_WAIT_%=;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
        : "memory");
}
// L2 prefetch of a tensor box (no shared-memory destination): the producer runs one tile ahead so
// that the ring's TMA loads of A hit L2 instead of DRAM (the ring holds only a few stages: the
// DRAM latency x bandwidth product of one SM does not fit in it)
__device__ __forceinline__ void tma_pf_2d(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_pf_3d(const CUtensorMap* map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
#ifndef PDSSM_TC_PREFETCH
#define PDSSM_TC_PREFETCH 0   // measured: readout fp32 +4%, bf16 +15% slower; fp32 projection 4% faster
#endif
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major SWIZZLE_128B: rows of 128 B, 8-row atoms
// 1024 B apart (SBO), LBO unused (1), version 1 (sm_100), layout type 2.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;
    d |= (uint64_t)(1024u >> 4) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)2u << 61;
    return d;
}
// Instruction descriptor: D f32, A/B format fmt (1 = bf16 under kind::f16, 2 = tf32 under
// kind::tf32), both K-major, N = n, M = 128.
__host__ __device__ constexpr uint32_t idesc(uint32_t fmt, int n) {
    return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

template <typename T>
struct Kind;
template <>
struct Kind<__nv_bfloat16> {
    static constexpr uint32_t FMT = 1;
    __device__ static void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
            "l"(a), "l"(b), "r"(id), "r"(acc)
            : "memory");
    }
};
template <>
struct Kind<float> {
    static constexpr uint32_t FMT = 2;
    __device__ static void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
            "l"(a), "l"(b), "r"(id), "r"(acc)
            : "memory");
    }
};

// D (+)= A B with A from tensor memory (tf32, K-major rows = TMEM lanes), B from shared memory
__device__ __forceinline__ void mma_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
// 16 consecutive 32-bit columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}

// 16 consecutive accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__host__ __device__ constexpr int tmem_cols(int bn) { return bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256; }

// --------------------------------------------------------------------------- epilogues
// a3 (+a4): per row (token) and head, k* = smallest argmax_k of the K fp32 logits
// (strict '>' over ascending k: ties -> smallest index, NaN never wins, all-NaN -> 0;
// readings R7/R8); optional logits and P rows.
struct EpiSelect {
    uint8_t* kstar;
    float* logits;             // [B][H][L][K] or null
    const uint16_t* dict_idx;  // [H][K][N] (P gather) or null
    uint16_t* P;               // [B][H][L][N] or null
    int64_t M;                 // B * L
    int L, H, K, N;
    uint32_t flags;
    // P row copy (16-byte vectors when the rows allow it)
    __device__ void copy_P(int h, int k, size_t r) const {
        const uint16_t* src = dict_idx + ((size_t)h * K + k) * N;
        uint16_t* dst = P + r * N;
        if ((N & 7) == 0 && ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(dict_idx)) & 15) == 0) {
            for (int j = 0; j < N; j += 8) *reinterpret_cast<uint4*>(dst + j) = __ldg(reinterpret_cast<const uint4*>(src + j));
        } else {
            for (int j = 0; j < N; ++j) dst[j] = __ldg(src + j);
        }
    }
    __device__ void operator()(uint32_t taddr, int64_t m, int n0, int bn, int z) const {
        (void)z;
        const bool valid = m < M;
        const int64_t b = valid ? m / L : 0, t = valid ? m - b * L : 0;
        const int h0 = n0 / K;
        if ((K & 15) == 0) {
            // whole 16-column groups per head: NaN -> -inf at the leaves, then a
            // (value desc, index asc) tree per group and a strict '>' across groups --
            // the same winner as the sequential rule (ties -> smallest k, NaN never wins,
            // no finite value -> 0)
            const int nh = bn / K;
            for (int hh = 0; hh < nh; ++hh) {
                const int h = h0 + hh;
                const bool live = valid && h < H;
                float best = -INFINITY;
                int arg = 0;
                for (int q = 0; q < K; q += 16) {
                    float v[16];
                    tmem_ld16(taddr + (uint32_t)(hh * K + q), v);
                    if (live) {
                        if (flags & PDSSM_CHECK_FINITE) {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (!isfinite(v[i])) report(ERRBIT_NONFINITE);
                        }
                        if (logits) {
                            float* lp = logits + (((size_t)b * H + h) * L + t) * K + q;
                            if ((reinterpret_cast<uintptr_t>(logits) & 15) == 0) {
#pragma unroll
                                for (int i = 0; i < 16; i += 4)
                                    *reinterpret_cast<float4*>(lp + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                            } else {
#pragma unroll
                                for (int i = 0; i < 16; ++i) lp[i] = v[i];
                            }
                        }
                    }
                    float w[16];
                    int ix[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        w[i] = isnan(v[i]) ? -INFINITY : v[i];
                        ix[i] = q + i;
                    }
#pragma unroll
                    for (int st = 1; st < 16; st *= 2)
#pragma unroll
                        for (int i = 0; i < 16; i += 2 * st)
                            if (w[i + st] > w[i]) {   // right operand has the larger index
                                w[i] = w[i + st];
                                ix[i] = ix[i + st];
                            }
                    if (w[0] > best || q == 0) {
                        best = w[0];
                        arg = ix[0];
                    }
                }
                if (live) {
                    const size_t r = ((size_t)b * H + h) * L + t;
                    kstar[r] = (uint8_t)arg;
                    if (P) copy_P(h, arg, r);
                }
            }
            return;
        }
        // general K: sequential scan over the tile's columns
        float best = -INFINITY;
        int arg = K, kk = 0, hh = 0;
        for (int c0 = 0; c0 < bn; c0 += 16) {
            float v[16];
            tmem_ld16(taddr + (uint32_t)c0, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float x = v[i];
                const int h = h0 + hh;
                if (valid && h < H) {
                    if ((flags & PDSSM_CHECK_FINITE) && !isfinite(x)) report(ERRBIT_NONFINITE);
                    if (logits) logits[(((size_t)b * H + h) * L + t) * K + kk] = x;
                }
                if (x > best) {
                    best = x;
                    arg = kk;
                }
                if (++kk == K) {
                    if (valid && h < H) {
                        const int k = arg >= K ? 0 : arg;
                        const size_t r = ((size_t)b * H + h) * L + t;
                        kstar[r] = (uint8_t)k;
                        if (P) copy_P(h, k, r);
                    }
                    ++hh;
                    kk = 0;
                    best = -INFINITY;
                    arg = K;
                }
            }
        }
    }
};

// a5: column j = (h, c, n) of the tile -> b[b][h][t][c][n] (activation dtype TO)
template <typename TO>
struct EpiProject {
    TO* out;
    int64_t M;
    int L, H, cN;
    int64_t NN;   // H * cN
    __device__ void operator()(uint32_t taddr, int64_t m, int n0, int bn, int z) const {
        (void)z;
        const bool valid = m < M;
        const int64_t b = valid ? m / L : 0, t = valid ? m - b * L : 0;
        for (int c0 = 0; c0 < bn; c0 += 16) {
            float v[16];
            tmem_ld16(taddr + (uint32_t)c0, v);
            const int64_t j = (int64_t)n0 + c0;
            if (!valid || j >= NN) continue;
            const int64_t h = j / cN, w = j - h * cN;
            TO* dst = out + (((size_t)b * H + h) * L + t) * cN + w;
            if constexpr (std::is_same<TO, float>::value) {
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            } else {
                uint32_t p[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const __nv_bfloat162 q = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
                    p[i] = *reinterpret_cast<const uint32_t*>(&q);
                }
                reinterpret_cast<uint4*>(dst)[0] = make_uint4(p[0], p[1], p[2], p[3]);
                reinterpret_cast<uint4*>(dst)[1] = make_uint4(p[4], p[5], p[6], p[7]);
            }
        }
    }
};

// NEXT-2 D_t generator (SPEC.md:367 form, reading R30): one tile = one head's c*N columns
// [a_0..a_{N-1} | theta_0..theta_{N-1}] of a token row; the epilogue writes
// D[b][h][t][c][n] = sigmoid(a + bias[h][n]) (cos theta, sin theta)   (c = 1: the magnitude)
// ns (0 = N): states per tile -- a tile of nc * ns columns holds [a_s0..a_{s0+ns-1} | theta_s0..]
// of the head's states s0 .. s0 + ns - 1 (tile jt = n0 / (nc ns): head jt / (N / ns), s0 = ns (jt % (N / ns))).
template <typename TO>
struct EpiDiag {
    TO* out;
    const float* bias;   // [H][N] or null
    int64_t M;
    int L, H, N, nc;
    int ns = 0;
    __device__ void operator()(uint32_t taddr, int64_t m, int n0, int bn, int z) const {
        (void)z;
        (void)bn;
        const bool valid = m < M;
        const int64_t b = valid ? m / L : 0, t = valid ? m - b * L : 0;
        const int cN = nc * N;
        const int S = ns ? ns : N;
        const int jt = n0 / (nc * S);
        const int h = jt / (N / S), s0 = (jt % (N / S)) * S;
        TO* dst = out + (((size_t)b * H + h) * L + t) * cN + s0;
        for (int c0 = 0; c0 < S; c0 += 16) {
            float a[16], th[16];
            tmem_ld16(taddr + (uint32_t)c0, a);
            if (nc == 2) tmem_ld16(taddr + (uint32_t)(c0 + S), th);
            if (!valid) continue;
            float re[16], im[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float mag = 1.f / (1.f + expf(-(a[i] + (bias ? bias[(size_t)h * N + s0 + c0 + i] : 0.f))));
                if (nc == 2) {
                    float sn, cs;
                    sincosf(th[i], &sn, &cs);
                    re[i] = mag * cs;
                    im[i] = mag * sn;
                } else {
                    re[i] = mag;
                    im[i] = 0.f;
                }
            }
            st16_act(dst + c0, re);
            if (nc == 2) st16_act(dst + N + c0, im);
        }
    }
    template <typename T2>
    __device__ static void st16_act(T2* d, const float (&v)[16]) {
        if constexpr (std::is_same<T2, float>::value) {
#pragma unroll
            for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(d + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        } else {
            uint32_t p[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const __nv_bfloat162 q = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
                p[i] = *reinterpret_cast<const uint32_t*>(&q);
            }
            reinterpret_cast<uint4*>(d)[0] = make_uint4(p[0], p[1], p[2], p[3]);
            reinterpret_cast<uint4*>(d)[1] = make_uint4(p[4], p[5], p[6], p[7]);
        }
    }
};

// NEXT-2 fused layer GEMM: one launch over the stacked weight rows [S (padded to n_sel) | B
// (n_prj) | W_d (optional)] of the layer (api_gemm.cu layer_gemm): every tile reads the same x
// slabs (consecutive tiles of one token block run concurrently and share them through L2), and
// the tile's column range picks its epilogue -- the argmax of Eq. 7, the projection of Eq. 1, or
// the D_t generator (R30).  bn divides n_sel and n_prj, and equals nc * ns for the D range.
template <typename TO>
struct EpiLayer {
    EpiSelect sel;
    EpiProject<TO> prj;
    EpiDiag<TO> dg;
    int n_sel, n_prj;
    __device__ void operator()(uint32_t taddr, int64_t m, int n0, int bn, int z) const {
        if (n0 < n_sel) sel(taddr, m, n0, bn, z);
        else if (n0 < n_sel + n_prj) prj(taddr, m, n0 - n_sel, bn, z);
        else dg(taddr, m, n0 - n_sel - n_prj, bn, z);
    }
};

// NEXT-3 PD-SSM soft generator (Eqs. 2-4): the tile holds the mixture
// M(u_t)[i][j] = sum_k s_k M_k[i][j] of one head for bn / N columns j (column index j * N + i,
// i fastest); the epilogue takes the column hardmax over i (smallest i on ties, NaN never
// wins, all-NaN -> 0) and writes P[b][h][t][j] -- the L N^2 mixture is never stored.
struct EpiColArgmax {
    uint16_t* P;   // [B][H][L][N]
    int64_t M;     // B * L
    int L, H, N, h;
    __device__ void operator()(uint32_t taddr, int64_t m, int n0, int bn, int z) const {
        (void)z;
        const bool valid = m < M;
        const int64_t b = valid ? m / L : 0, t = valid ? m - b * L : 0;
        uint16_t* dst = P + (((size_t)b * H + h) * L + t) * N;
        for (int j0 = 0; j0 < bn; j0 += N) {
            float best = -INFINITY;
            int arg = N;
            for (int c0 = 0; c0 < N; c0 += 16) {
                float v[16];
                tmem_ld16(taddr + (uint32_t)(j0 + c0), v);
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (v[q] > best) {
                        best = v[q];
                        arg = c0 + q;
                    }
            }
            if (valid) dst[(n0 + j0) / N] = (uint16_t)(arg >= N ? 0 : arg);
        }
    }
};

// store 16 consecutive fp32 values as TO (16-byte vector stores; dst 16-byte aligned)
template <typename TO>
__device__ __forceinline__ void st16(TO* dst, const float (&v)[16]) {
    if constexpr (std::is_same<TO, float>::value) {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else {
        uint32_t p[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const __nv_bfloat162 q = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            p[i] = *reinterpret_cast<const uint32_t*>(&q);
        }
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(p[0], p[1], p[2], p[3]);
        reinterpret_cast<uint4*>(dst)[1] = make_uint4(p[4], p[5], p[6], p[7]);
    }
}

// a8 readout y_t = Re(C_h h_t) = C_re h_re - C_im h_im (Eq. 1): tile rows are
// the steps t of one sequence z = b*H + h, columns the readout rows p -> y[b][t][h][p]
template <typename TO>
struct EpiReadout {
    TO* y;
    int L, H, P;
    // tcgen05.ld gives thread = row (its 16 columns): stored directly (fp32), every warp store would
    // write 32 rows 4 KB apart in 16-byte half sectors.  Each 32-column slice goes through a per-warp shared tile
    // instead and leaves as 4 rows x 128 contiguous bytes per warp store (full sectors).
    __device__ void operator()(uint32_t taddr, int64_t t, int n0, int bn, int z) const {
        if constexpr (!std::is_same<TO, float>::value) {   // bf16: 16 columns = one 32-byte sector per row
            const bool valid = t < L;
            const int b = z / H, h = z - (z / H) * H;
            for (int c0 = 0; c0 < bn; c0 += 16) {
                float v[16];
                tmem_ld16(taddr + (uint32_t)c0, v);
                const int p = n0 + c0;
                if (valid && p < P) st16<TO>(y + (((size_t)b * L + t) * H + h) * P + p, v);
            }
            return;
        }
        __shared__ float stile[4][32][33];   // [epilogue warp][row][column] (+1: conflict-free)
        const int lane = threadIdx.x & 31;
        float(*tl)[33] = stile[(threadIdx.x >> 5) & 3];
        const int b = z / H, h = z - (z / H) * H;
        const int64_t tw = t - lane;   // first row of this warp
        for (int c0 = 0; c0 < bn; c0 += 32) {
            const int nc = bn - c0 < 32 ? bn - c0 : 32;   // 16 or 32 (bn % 16 == 0)
            float v[16];
            tmem_ld16(taddr + (uint32_t)c0, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) tl[lane][i] = v[i];
            if (nc > 16) {
                tmem_ld16(taddr + (uint32_t)(c0 + 16), v);
#pragma unroll
                for (int i = 0; i < 16; ++i) tl[lane][16 + i] = v[i];
            }
            __syncwarp();
            const int cc = (lane & 7) * 4;
            const int p = n0 + c0 + cc;
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int rr = it * 4 + (lane >> 3);
                const int64_t tr = tw + rr;
#ifndef PDSSM_EXP_NOSTORE   // timing experiment only (no output)
                if (tr < L && cc < nc && p < P) {
                    TO* dst = y + (((size_t)b * L + tr) * H + h) * P + p;
                    *reinterpret_cast<float4*>(dst) = make_float4(tl[rr][cc], tl[rr][cc + 1], tl[rr][cc + 2], tl[rr][cc + 3]);
                }
#endif
            }
            __syncwarp();
        }
    }
};

// readout adjoint (bwd with dy): e_t = dh_t + conj(C)^T dy_t per head (reading R13), rows
// m = b*L + t, columns w = (c, n) of head z -> e[b][z][t][w] (fp32 scratch of the scan)
template <typename TI>
struct EpiAdjoint {
    float* e;
    const TI* dh;   // or null
    int64_t M;
    int L, H, cN;
    __device__ void operator()(uint32_t taddr, int64_t m, int n0, int bn, int z) const {
        const bool valid = m < M;
        const int64_t b = valid ? m / L : 0, t = valid ? m - b * L : 0;
        for (int c0 = 0; c0 < bn; c0 += 16) {
            float v[16];
            tmem_ld16(taddr + (uint32_t)c0, v);
            const int w = n0 + c0;
            if (!valid || w >= cN) continue;
            const size_t off = (((size_t)b * H + z) * L + t) * cN + w;
            if (dh) {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] += ldact(dh + off + i);
            }
            st16<float>(e + off, v);
        }
    }
};

// How a CTA finds its A rows and B rows (the operand maps are 2-D or 3-D):
//  mode 0: A rows m0 = blockIdx.x*BM of a 2-D map; B rows n0.
//  mode 1: A is 3-D (K, rows, Z): z = blockIdx.x / tiles, m0 = (blockIdx.x % tiles)*BM;
//          B rows (z % zmod)*brows + n0 (per-head weights stacked in one 2-D map).
//  mode 2: A is 3-D (K, Z, rows) with box (EK, 1, BM): z = blockIdx.z, m0 = blockIdx.x*BM;
//          B rows z*brows + n0.
struct TileMap {
    int mode, tiles, zmod, brows;
};

// --------------------------------------------------------------------------- kernel
// SPLIT (fp32 operands): 3xTF32.  Each landed fp32 slab is split in shared memory by the
// epilogue warps (idle during the main loop) into hi = tf32_rna(a) (in place) and
// lo = a - hi (a twin slab at the same swizzled offsets); the MMA warp then issues
// lo*hi + hi*lo + hi*hi per K step, which keeps the products to ~2^-21 relative
// (plain TF32 would be 2^-11), i.e. fp32-grade logits and projections.
#ifndef PDSSM_TC_RAWHI
#define PDSSM_TC_RAWHI 1
#endif
__device__ __forceinline__ uint32_t tf32_rna(float a) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(a));
    return r;
}

template <typename T, int STAGES, bool SPLIT, int MT = 1, bool ATM = false>
struct Smem {
    // A rows (MT row tiles of BM) then B rows (ATM: then the B lo rows; the A lo parts live in TMEM)
    __host__ __device__ static constexpr size_t slot(int bn) { return (size_t)(MT * BM + bn * (ATM ? 2 : 1)) * ROWB; }
    __host__ __device__ static constexpr size_t ring(int bn) { return (size_t)STAGES * slot(bn) * (SPLIT && !ATM ? 2 : 1); }
    __host__ __device__ static constexpr size_t bytes(int bn) { return 1024 + ring(bn) + 8 * (3 * STAGES + 4) + 16; }
};

// Persistent: grid = min(#tiles, #SMs); CTA c takes tiles c, c + grid, ...  Tiles are
// numbered with the column tile fastest (consecutive tiles share the A rows in L2).  TMEM
// holds two accumulators (2 x 256 columns), so the epilogue of tile j overlaps the main loop
// of tile j+1 (tmem_full / tmem_empty barriers).  Warps: 0 TMA, 1 MMA, 2 TMEM allocator,
// 4-7 epilogue, 8-15 tf32 split (SPLIT only).
struct TileGrid {
    int gx, gy, gz;   // tiles along the A rows (x), the output columns (y), the z batch
};

// BPRE (with SPLIT): the weights B arrive pre-split in global memory (mB = tf32 hi part, mBlo = the
// lo part, written once per call by the host path), so the converter warps split only the A rows
// of each slab -- half the shared-memory traffic of the split (readout: B = the readout weights).
// MT = 2 (bn <= 128): a tile is 2 x BM rows sharing every B slab (two MMAs per K step into the two
// 128-column halves of the tile's accumulator): half the B traffic per output (the readout reloads
// its per-head weights for every tile: B was 2/3 of its L2 -> SM bytes at MT = 1).
// ATM (with SPLIT, BPRE, MT = 1, bn <= 128): the A operand is read from TENSOR memory.  The tf32
// MMAs at N = 128 read 8 KB of shared operands per 64-cycle instruction -- the whole shared-memory
// bandwidth, three times per K step with the 3xTF32 split; with A (raw hi and lo, written by the
// converter warps with tcgen05.st straight from the landed slab) in TMEM, only B is read from shared
// memory.  TMEM: accumulators 2 x 128 columns, then STAGES x (32 hi + 32 lo) A columns.
template <typename T, int STAGES, bool SPLIT, class Epi, bool BPRE = false, int MT = 1, bool ATM = false>
__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
              const __grid_constant__ CUtensorMap mBlo, int nk, int bn, TileMap tm, TileGrid tg, Epi epi) {
    static_assert(!BPRE || SPLIT, "pre-split weights only with the 3xTF32 split");
    static_assert(MT == 1 || MT == 2, "row tiles per CTA tile");
    static_assert(!ATM || (SPLIT && BPRE && MT == 1 && 256 + STAGES * 64 <= 512), "A in TMEM: readout shape");
    constexpr uint32_t ACCS = ATM ? 128 : 256;   // accumulator stride (columns)
    constexpr uint32_t ACOL = 256;               // ATM: first A column
    using SM = Smem<T, STAGES, SPLIT, MT, ATM>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const size_t SLOT = SM::slot(bn);                  // multiple of 1024 (bn % 8 == 0)
    auto hi = [&](int s) { return smem + (size_t)s * SLOT; };
    auto lo = [&](int s) { return smem + (size_t)(STAGES + s) * SLOT; };
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::ring(bn));
    uint64_t* conv = full + STAGES;
    uint64_t* empty = conv + STAGES;
    uint64_t* tfull = empty + STAGES;     // [2]
    uint64_t* tempty = tfull + 2;         // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t NCOLS = 512;       // two accumulators of up to 256 columns
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(conv + s, NCONV);   // one arrival per converter warp
            mbar_init(empty + s, 1);
        }
        for (int q = 0; q < 2; ++q) {
            mbar_init(tfull + q, 1);
            mbar_init(tempty + q, 4);  // one arrival per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mB)) : "memory");
        if constexpr (BPRE) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBlo)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(NCOLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tslot;
    const int ntiles = tg.gx * tg.gy * tg.gz;
    // tile id -> (A row m0, output column n0, z, weight row brow)
    auto coords = [&](int id, int64_t& m0, int& n0, int& z, int& brow) {
        const int by = id % tg.gy;
        const int rest = id / tg.gy;
        const int bx = rest % tg.gx;
        const int bz = rest / tg.gx;
        n0 = by * bn;
        if (tm.mode == 1) {
            z = bx / tm.tiles;
            m0 = (int64_t)(bx - z * tm.tiles) * (BM * MT);
            brow = (z % tm.zmod) * tm.brows + n0;
        } else if (tm.mode == 2) {
            z = bz;
            m0 = (int64_t)bx * (BM * MT);
            brow = z * tm.brows + n0;
        } else {
            z = 0;
            m0 = (int64_t)bx * (BM * MT);
            brow = n0;
        }
    };
    constexpr int EK = ROWB / (int)sizeof(T);   // elements of K per slab row
    if (warp == 0) {
        if (lane == 0) {
            // (programmatic dependent launch) everything this kernel reads or writes in global memory
            // is ordered after the producer's first load, hence after the previous launch completed
            asm volatile("griddepcontrol.wait;" ::: "memory");
            const uint32_t bytes = (uint32_t)(SLOT + (BPRE && !ATM ? (size_t)bn * ROWB : 0));
            int kg = 0;
            for (int id = blockIdx.x; id < ntiles; id += gridDim.x) {
                int64_t m0;
                int n0, z, brow;
                coords(id, m0, n0, z, brow);
                int64_t m0n = 0;
                int n0n = 0, zn = 0, brown = 0;
                const int idn = id + (int)gridDim.x;   // this CTA's next tile
                const bool pfn = PDSSM_TC_PREFETCH && idn < ntiles;
                if (pfn) coords(idn, m0n, n0n, zn, brown);
                for (int kb = 0; kb < nk; ++kb, ++kg) {
                    const int s = kg % STAGES;
                    if (pfn) {   // the next tile's A slab kb -> L2
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            const int mr = (int)m0n + mt * BM;
                            if (tm.mode == 1) tma_pf_3d(&mA, kb * EK, mr, zn);
                            else if (tm.mode == 2) tma_pf_3d(&mA, kb * EK, zn, mr);
                            else tma_pf_2d(&mA, kb * EK, mr);
                        }
                    }
                    if (kg >= STAGES) mbar_wait(empty + s, (uint32_t)((kg / STAGES) + 1) & 1u);
                    mbar_expect_tx(full + s, bytes);
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        uint8_t* da = hi(s) + (size_t)mt * BM * ROWB;
                        const int mr = (int)m0 + mt * BM;
                        if (tm.mode == 1) tma_3d(da, &mA, kb * EK, mr, z, full + s);
                        else if (tm.mode == 2) tma_3d(da, &mA, kb * EK, z, mr, full + s);
                        else tma_2d(da, &mA, kb * EK, mr, full + s);
                    }
                    tma_2d(hi(s) + (size_t)MT * BM * ROWB, &mB, kb * EK, brow, full + s);
                    if constexpr (ATM) tma_2d(hi(s) + (size_t)(BM + bn) * ROWB, &mBlo, kb * EK, brow, full + s);
                    else if constexpr (BPRE) tma_2d(lo(s) + (size_t)MT * BM * ROWB, &mBlo, kb * EK, brow, full + s);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t id_ = idesc(Kind<T>::FMT, bn);
            int kg = 0, j = 0;
            for (int id = blockIdx.x; id < ntiles; id += gridDim.x, ++j) {
                const int acc = j & 1;
                if (j >= 2) mbar_wait(tempty + acc, (uint32_t)((j / 2) - 1) & 1u);   // epilogue drained it
                fence_after();
                const uint32_t tacc = tmem + (uint32_t)acc * ACCS;
                for (int kb = 0; kb < nk; ++kb, ++kg) {
                    const int s = kg % STAGES;
                    mbar_wait((SPLIT ? conv : full) + s, (uint32_t)(kg / STAGES) & 1u);
                    fence_after();
                    const uint64_t bh = sdesc(su32(hi(s) + (size_t)MT * BM * ROWB));
                    const uint64_t bl = sdesc(su32(ATM ? hi(s) + (size_t)(BM + bn) * ROWB : lo(s) + (size_t)MT * BM * ROWB));
                    if constexpr (ATM) {
                        const uint32_t ah = tmem + ACOL + (uint32_t)s * 64, al = ah + 32;
#pragma unroll
                        for (int k = 0; k < ROWB / 32; ++k) {   // 8 tf32 columns of A per instruction
                            const uint32_t acc0 = (kb | k) != 0;
                            mma_ta(tacc, al + 8 * k, bh + 2 * k, id_, acc0);
                            mma_ta(tacc, ah + 8 * k, bl + 2 * k, id_, 1u);
                            mma_ta(tacc, ah + 8 * k, bh + 2 * k, id_, 1u);
                        }
                        commit(empty + s);
                        continue;
                    }
#pragma unroll
                    for (int k = 0; k < ROWB / 32; ++k) {   // 32 bytes of K per instruction
                        const uint32_t acc0 = (kb | k) != 0;
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            const uint64_t ah = sdesc(su32(hi(s) + (size_t)mt * BM * ROWB));
                            const uint64_t al = sdesc(su32(lo(s) + (size_t)mt * BM * ROWB));
                            const uint32_t tm_ = tacc + (uint32_t)(mt * 128);
                            if constexpr (SPLIT) {
#ifndef PDSSM_EXP_ONEMMA   // timing experiment only (plain TF32)
                                Kind<T>::mma(tm_, al + 2 * k, bh + 2 * k, id_, acc0);
                                Kind<T>::mma(tm_, ah + 2 * k, bl + 2 * k, id_, 1u);
#endif
                                Kind<T>::mma(tm_, ah + 2 * k, bh + 2 * k, id_, 1u);
                            } else {
                                Kind<T>::mma(tm_, ah + 2 * k, bh + 2 * k, id_, acc0);
                            }
                        }
                    }
                    commit(empty + s);
                }
                commit(tfull + acc);
            }
        }
        __syncwarp();
    } else if (warp >= 4 && warp < 8) {
        const int q = warp - 4;
        int j = 0;
        for (int id = blockIdx.x; id < ntiles; id += gridDim.x, ++j) {
            const int acc = j & 1;
            int64_t m0;
            int n0, z, brow;
            coords(id, m0, n0, z, brow);
            mbar_wait(tfull + acc, (uint32_t)(j / 2) & 1u);
            fence_after();
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
                epi(tmem + (uint32_t)acc * ACCS + (uint32_t)(mt * 128) + ((uint32_t)(32 * q) << 16), m0 + mt * BM + 32 * q + lane,
                    n0, bn, z);
            fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(tempty + acc)) : "memory");
        }
    } else if (warp >= 8) {
        if constexpr (ATM) {
            // converters -> TMEM: warp 8 + q and 12 + q serve the tile rows 32q..32q+31 (their TMEM lane
            // quarter), K elements 0..15 and 16..31 of each landed slab; raw fp32 = hi (the MMA
            // truncates to tf32), lo = a - trunc(a).  The A columns of stage s are rewritten only after
            // full[s] completed again, i.e. after the MMAs that read them committed (empty[s]).
            const int q = warp & 3, hk = (warp - 8) >> 2;
            const int m = 32 * q + lane;   // this thread's tile row
            int kg = 0;
            for (int id = blockIdx.x; id < ntiles; id += gridDim.x) {
                for (int kb = 0; kb < nk; ++kb, ++kg) {
                    const int s = kg % STAGES;
                    mbar_wait(full + s, (uint32_t)(kg / STAGES) & 1u);
                    const uint8_t* rowp = hi(s) + (size_t)m * ROWB;
                    uint32_t rh[16], rl[16];
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {   // 16-byte chunk 4 hk + cc of the SWIZZLE_128B row
                        const int c = 4 * hk + cc;
                        const float4 a = *reinterpret_cast<const float4*>(rowp + ((c ^ (m & 7)) << 4));
                        const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t bits = __float_as_uint(av[u]);
                            rh[4 * cc + u] = bits;
                            rl[4 * cc + u] = __float_as_uint(av[u] - __uint_as_float(bits & 0xffffe000u));
                        }
                    }
                    const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + ACOL + (uint32_t)s * 64 + (uint32_t)(16 * hk);
                    tmem_st16(ta, rh);
                    tmem_st16(ta + 32, rl);
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    fence_before();
                    __syncwarp();
                    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(conv + s)) : "memory");
                }
            }
        } else if constexpr (SPLIT) {
            // converters: split every landed slab (the producer reused slot s only after the
            // MMAs of its previous round completed, and full[s] completes after that reuse)
            const int ct = threadIdx.x - 256;
            const int nchunks = (BPRE ? MT * BM : MT * BM + bn) * (ROWB / 16);   // BPRE: the B rows arrive split
            int kg = 0;
            for (int id = blockIdx.x; id < ntiles; id += gridDim.x) {
                for (int kb = 0; kb < nk; ++kb, ++kg) {
                    const int s = kg % STAGES;
                    mbar_wait(full + s, (uint32_t)(kg / STAGES) & 1u);
                    float4* ph = reinterpret_cast<float4*>(hi(s));
                    float4* pl = reinterpret_cast<float4*>(lo(s));
#ifdef PDSSM_EXP_NOCONV   // timing experiment only (lo parts left as they are)
                    for (int i = ct; i < 0; i += NCONV * 32) {
#else
                    for (int i = ct; i < nchunks; i += NCONV * 32) {
#endif
                        const float4 a = ph[i];
#if PDSSM_TC_RAWHI
                        // hi stays the raw fp32 slab: kind::tf32 reads only its top 19 bits (truncation),
                        // so lo = a - trunc(a) (exact) is the only store -- half the split's shared traffic
                        pl[i] = make_float4(a.x - __uint_as_float(__float_as_uint(a.x) & 0xffffe000u),
                                            a.y - __uint_as_float(__float_as_uint(a.y) & 0xffffe000u),
                                            a.z - __uint_as_float(__float_as_uint(a.z) & 0xffffe000u),
                                            a.w - __uint_as_float(__float_as_uint(a.w) & 0xffffe000u));
#else
                        const uint32_t h0 = tf32_rna(a.x), h1 = tf32_rna(a.y), h2 = tf32_rna(a.z), h3 = tf32_rna(a.w);
                        ph[i] = make_float4(__uint_as_float(h0), __uint_as_float(h1), __uint_as_float(h2), __uint_as_float(h3));
                        pl[i] = make_float4(a.x - __uint_as_float(h0), a.y - __uint_as_float(h1), a.z - __uint_as_float(h2),
                                            a.w - __uint_as_float(h3));
#endif
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA reads
                    __syncwarp();
                    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(conv + s)) : "memory");
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(NCOLS) : "memory");
    }
}

}  // namespace tc
}  // namespace pdssm
