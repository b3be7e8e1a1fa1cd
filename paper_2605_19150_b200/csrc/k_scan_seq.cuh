// Single-chunk scan (tau >= L, C = 1): one CTA per (b, h) sequence, thread i owns state i.
//
// Alg. 1 with one chunk per sequence needs no Phase A aggregate and
// no inter-chunk carry: the replay from carry_0 = h0 IS the scan.  When B*H fills the
// GPU (config 2: 128 sequences on 148 SMs) this reads every step's D_t, b_t once
// (evict-first TMA stream) instead of twice, and each step is one CTA barrier:
//
//   v_t = D_t (.) h_{t-1}   (own state, registers)   -> vbuf[t&1][i]      (STS, conflict-free)
//   __syncthreads()                                   (double-buffered vbuf: one barrier/step)
//   h_t[i] = b_t[i] + sum_{j : P_t[j] = i} v_t[j]    (the column-one-hot scatter, reading R1,
//                                                      as a gather over the preimage of i)
//
// The preimage of i under entry k is a per-(k, i) record of up to 8 source indices (u8,
// ascending, padded with the zero slot N); the warp-uniform trip count is the warp's
// maximum in-degree of entry k.  Entries with an in-degree > 8 take the CSR plan.
// AGG (PDSSM_EXPORT_MAPS): the chunk aggregate (pi_bar, d_bar, beta_bar) of the single chunk
// and the final map are composed alongside (thread-local gathers).
//
// Backward (reverse, transposed; App. C): thread j owns source j;
//   lbuf[t&1][j] = lambda_t;  __syncthreads();  lp = lambda_t[P_t[j]]  (a pure gather)
//   dD_t[j] = conj(h_{t-1}[j]) lp;  g_t = sum_j Re(conj(lp) D_t[j] h_{t-1}[j]);
//   lambda_{t-1}[j] = e_{t-1}[j] + conj(D_t[j]) lp.
#pragma once
#include "pdssm_common.cuh"
#include "k_scan_fwd.cuh"
#include "k_scan_fused.cuh"

namespace pdssm {
namespace seq {

constexpr int CAP = 8;       // record slots per (entry, target) (u8 sources, padded with the zero slot N)
#ifndef PDSSM_SEQ_GCAP
#define PDSSM_SEQ_GCAP 8
#endif
constexpr int GCAP = PDSSM_SEQ_GCAP;   // sources gathered inline (<= CAP); longer preimages take the CSR plan
static_assert(GCAP == 6 || GCAP == 8, "gather capacity");
constexpr int LMAX = 16384;  // k* of the whole sequence is staged in shared memory
constexpr int MAXN = 128;    // states per CTA (one thread each)
constexpr int WM_OVF = 15;   // trip-count code of an overflowing entry

__host__ __device__ constexpr size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }

// shared-memory carve-up (host and device agree)
// SPC sequences of one head share a CTA (and its per-head tables): the ring slot holds, per
// stream, SPC blocks of G rows; the exchange rows, k* staging and g tiles are per sequence.
struct Layout {
    size_t ring, bars, x, x2, kb, rec, wm, ovf, prow, dk, gs, bytes;
    int slot;     // bytes per ring slot
    size_t xs;    // bytes of one sequence's exchange rows (two rows of N + 1 values)
    size_t kbs;   // bytes of one sequence's k* staging
    size_t gss;   // bytes of one sequence's g tiles
    __host__ __device__ Layout(int N, int K, int R, int G, int NC, int esz, int esz_e, bool PD, bool AGG, bool BWD, int L,
                               int SPC = 1) {
        const int row = NC * N * esz, erow = NC * N * esz_e;
        const int NW = N / 32;
        slot = (int)a16((size_t)SPC * (BWD ? (size_t)(PD ? 0 : G * row) + (size_t)G * erow + (size_t)G * row
                                           : (size_t)(PD ? 0 : G * row) + (size_t)G * row));
        size_t o = 0;
        ring = o; o = a16(o + (size_t)R * slot);
        bars = o; o = a16(o + (size_t)(2 * R + 1) * 8);   // full[R], empty[R], then the table barrier
        const int sv = NC == 2 ? 8 : 4;
        xs = a16((size_t)2 * (N + 1) * sv);
        x = o; o = a16(o + (size_t)SPC * xs);
        x2 = o; o = a16(o + (AGG ? (size_t)SPC * xs : 0));
        kbs = a16((size_t)L + 2 + 15);   // + slack: the row starts at the k* address mod 16 (stage_k)
        kb = o; o = a16(o + (size_t)SPC * kbs);
        rec = o; o = a16(o + (BWD ? 0 : (size_t)K * N * 8));
        wm = o; o = a16(o + (BWD ? 0 : (size_t)K * NW));
        ovf = o; o = a16(o + (BWD ? 0 : (size_t)K));
        prow = o; o = a16(o + ((AGG || BWD) ? (size_t)K * N * 2 : 0));
        dk = o; o = a16(o + (PD ? (size_t)K * NC * N * 4 : 0));
        gss = BWD ? a16(((size_t)32 * (N + 1) + (size_t)32 * NW) * 4) : 0;
        gs = o; o = a16(o + (size_t)SPC * gss);
        bytes = o;
    }
};

struct SeqArgs {
    const uint8_t* kstar;
    const uint16_t* dict_idx;   // [H][K][N] (clamped on load)
    const uint8_t* rec;         // [H][K][N][8] preimage records (fwd)
    const uint8_t* wm;          // [H][K][NW] warp trip counts (fwd)
    const uint8_t* ovf;         // [H][K] 1 = some preimage longer than CAP (fwd)
    const uint16_t* pstart;     // CSR plan (overflow entries)
    const uint16_t* psrc;
    const void* diag;           // PER_STEP act rows
    const float* diag_dict;     // PER_DICT f32 [H][K][NC][N]
    const void* bias;           // fwd: b_t ; bwd: e_t (act or f32)
    const void* hsaved;         // bwd
    const float* h0;
    const float* lam_in;        // bwd
    ChunkStateView cs;          // C = 1
    uint16_t* maps;             // fwd [S][2][N] (EXPORT_MAPS)
    void* out0;                 // fwd: h ; bwd: dbias
    void* out1;                 // bwd: ddiag (act) or f32 scratch (PER_DICT)
    float* gsel;                // bwd
    float* dh0;                 // bwd
    int H, L, N, K, R, G;
    int spc;                    // sequences per CTA (the host requires B % spc == 0)
    int tau, C;                 // chunk modes (MODE != 0): chunk length and chunks per sequence
    float* mu;                  // bwd MODE 2: incoming adjoint mu_c [S][C][NC][N] (k_bwd_phaseB)
    float* betap;               // bwd MODE 1: beta'_c out [S][C][NC][N]
    uint32_t flags;
};

// per (entry, target) preimage records: sources ascending, padded with N; wm = warp max
// in-degree (<= CAP); ovf = an in-degree above CAP occurred
// The same launch writes the CSR plan of k_build_plan (pstart / psrc: preimage lists in
// ascending source order) used by entries that overflow the records.
static __global__ void k_build_seq_plan(const uint16_t* __restrict__ dict_idx, uint8_t* __restrict__ rec,
                                 uint8_t* __restrict__ wm, uint8_t* __restrict__ ovf, uint16_t* __restrict__ pstart,
                                 uint16_t* __restrict__ psrc, int N, uint32_t flags) {
    extern __shared__ uint16_t sP[];
    __shared__ int sovf;
    asm volatile("griddepcontrol.launch_dependents;");   // the forward scan may start its prologue
    const int e = blockIdx.x;
    const int i = threadIdx.x;   // blockDim.x == N (multiple of 32)
    if (i == 0) sovf = 0;
    int p = dict_idx[(size_t)e * N + i];
    if (p >= N) {
        if (flags & PDSSM_CHECK_FINITE) report(ERRBIT_RANGE);
        p = N - 1;
    }
    sP[i] = (uint16_t)p;
    __syncthreads();
    // the record in a register (byte q = q-th source; a local array indexed by d would live
    // in local memory)
    unsigned long long r = 0x0101010101010101ull * (unsigned long long)(uint8_t)N;
    int d = 0, below = 0, rank = 0;
    const int pi = sP[i];
    for (int j = 0; j < N; ++j) {
        const int pj = sP[j];
        if (pj == i) {
            if (d < GCAP) r = (r & ~(0xffull << (8 * d))) | ((unsigned long long)j << (8 * d));
            ++d;
        }
        below += pj < i;                              // pstart[i] = #{j : P[j] < i}
        rank += (pj < pi) || (pj == pi && j < i);      // position of source i in the CSR order
    }
    pstart[(size_t)e * (N + 1) + i] = (uint16_t)below;
    if (i == 0) pstart[(size_t)e * (N + 1) + N] = (uint16_t)N;
    psrc[(size_t)e * N + rank] = (uint16_t)i;
    reinterpret_cast<unsigned long long*>(rec)[(size_t)e * N + i] = r;   // (CAP == 8 bytes, aligned)
    int m = d < GCAP ? d : GCAP;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (d > GCAP) sovf = 1;
    __syncthreads();
    // warp trip count; WM_OVF marks an entry with a preimage longer than CAP (CSR fallback)
    if ((i & 31) == 0) wm[(size_t)e * (N / 32) + (i >> 5)] = (uint8_t)(sovf ? WM_OVF : m);
    if (i == 0) ovf[e] = (uint8_t)sovf;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fused::smem_u32(b)) : "memory");
}

// ---- prologue staging (global -> shared, every thread of the CTA).  The prologue is latency
// bound: each thread issues all of its loads of a pass before its first store, so a table costs
// one HBM round trip per pass instead of one per element (an element-wise loop cost ~15 us of the
// ~190 us config-2 forward).  src and dst 16-byte aligned; f transforms each loaded word.  U is
// small (the staging registers count against the kernel's peak); the largest table, the forward's
// preimage records, goes by one bulk copy instead (stage_rec).
template <int U = 4, typename F>
__device__ __forceinline__ void stage16(const uint4* __restrict__ src, uint4* dst, int n4, F&& f) {
    const int nt = blockDim.x;
    for (int x0 = threadIdx.x; x0 < n4; x0 += U * nt) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (x0 + u * nt < n4) v[u] = __ldg(src + x0 + u * nt);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (x0 + u * nt < n4) dst[x0 + u * nt] = f(v[u]);
    }
}
struct Ident {
    __device__ uint4 operator()(uint4 v) const { return v; }
};
__device__ __forceinline__ bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }
// the staged k* row of a sequence starts at (its global address mod 16) inside its buffer, so the
// bulk of it moves as aligned 16-byte words (the buffers carry 16 bytes of slack)
__device__ __forceinline__ int kshift(const uint8_t* g) { return (int)((uintptr_t)g & 15); }

// k* of one sequence (L bytes at src) -> kbuf + kshift(src), clamped to K - 1 (reported under
// CHECK_FINITE), zero-padded by two; returns the staged row
__device__ __forceinline__ uint8_t* stage_k(const uint8_t* src, int K, uint32_t flags, uint8_t* kbuf, int L) {
    uint8_t* kb = kbuf + kshift(src);
    const int tid = threadIdx.x;
    const int head = min(L, (16 - kshift(src)) & 15);
    const int n4 = (L - head) >> 4, tail0 = head + n4 * 16;
    bool bad = false;
    auto fixb = [&](int k) {
        if (k >= K) {
            bad = true;
            k = K - 1;
        }
        return (uint8_t)k;
    };
    if (tid < head) kb[tid] = fixb(src[tid]);
    if (tid < L - tail0) kb[tail0 + tid] = fixb(src[tail0 + tid]);
    if (tid < 2) kb[L + tid] = 0;
    const uint32_t kx4 = (uint32_t)(K & 255) * 0x01010101u, km4 = (uint32_t)((K - 1) & 255) * 0x01010101u;
    auto fixw = [&](uint32_t w) {
        if (K < 256 && __vcmpgeu4(w, kx4)) {
            bad = true;
            w = __vminu4(w, km4);
        }
        return w;
    };
    stage16(reinterpret_cast<const uint4*>(src + head), reinterpret_cast<uint4*>(kb + head), n4, [&](uint4 v) {
        return make_uint4(fixw(v.x), fixw(v.y), fixw(v.z), fixw(v.w));
    });
    if (bad && (flags & PDSSM_CHECK_FINITE)) report(ERRBIT_RANGE);
    return kb;
}
__device__ __forceinline__ void stage_k(const SeqArgs& a, uint8_t* kbuf, size_t base, int L) {
    stage_k(a.kstar + base, a.K, a.flags, kbuf, L);
}
// P_k rows of head h ([K][N] u16, clamped to N - 1) -> prow
__device__ __forceinline__ void stage_prow(const uint16_t* src, uint16_t* prow, int KN, int N) {
    if (aligned16(src) && (KN & 7) == 0) {
        const uint32_t m2 = (uint32_t)(N - 1) * 0x10001u;
        stage16(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(prow), KN >> 3, [&](uint4 v) {
            return make_uint4(__vminu2(v.x, m2), __vminu2(v.y, m2), __vminu2(v.z, m2), __vminu2(v.w, m2));
        });
    } else {
        for (int x = threadIdx.x; x < KN; x += blockDim.x) prow[x] = (uint16_t)min((int)__ldg(src + x), N - 1);
    }
}
// the forward's preimage records of head h (n = K * N records of CAP bytes): one bulk copy by
// thread 0 completing on tbar (initialised, arrival count 1) when the source is 16-byte aligned,
// else an element loop (visible after the caller's next __syncthreads); either way tbar's phase 0
// completes, so the consumers wait on it unconditionally
__device__ __forceinline__ void stage_rec(const uint8_t* src, uint2* rec, int n, uint64_t* tbar) {
    const uint32_t bytes = (uint32_t)n * CAP;
    if (aligned16(src)) {
        if (threadIdx.x == 0) {
            fused::mbar_expect_tx(tbar, bytes);
            fused::tma_1d(rec, src, bytes, tbar);
        }
    } else {
        for (int x = threadIdx.x; x < n; x += blockDim.x) rec[x] = __ldg(reinterpret_cast<const uint2*>(src) + x);
        if (threadIdx.x == 0) mbar_arrive(tbar);
    }
}
// f32 table (n floats) -> shared
__device__ __forceinline__ void stage_f32(const float* src, float* dst, int n) {
    if (aligned16(src) && (n & 3) == 0) {
        stage16(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), n >> 2, Ident{});
    } else {
        for (int x = threadIdx.x; x < n; x += blockDim.x) dst[x] = __ldg(src + x);
    }
}

// global row of local step 0 of batch row b, head h, chunk start tb
__device__ __forceinline__ size_t seq0_of(const SeqArgs& a, int b, int h, int tb) { return (size_t)(b * a.H + h) * a.L + tb; }

// the N compute threads synchronise on named barrier 1 (the producer warp never joins)
__device__ __forceinline__ void compute_sync(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }
// producer warp (one elected lane): keeps the ring R groups ahead; a slot is refilled
// once the compute threads released it (empty barrier, one arrival per consumed group)
template <typename F>
__device__ __forceinline__ void produce(uint64_t* bars, int R, int ngroups, F&& issue) {
    if ((threadIdx.x & 31) != 0) return;
    for (int g = 0; g < ngroups; ++g) {
        const int slot = g % R;
        if (g >= R) fused::mbar_wait(bars + R + slot, (uint32_t)((g / R) - 1) & 1u);
        issue(g, slot);
    }
}

// shared-space addresses base + sv * byte_q(w), q = 0..3, pinned before whatever volatile
// asm follows (the barrier): the compiler may not sink them onto the post-barrier path
__device__ __forceinline__ void gather_addr4(uint32_t w, uint32_t base, uint32_t sv, uint32_t (&a)[4]) {
    asm volatile(
        "{\n\t.reg .b32 t0, t1, t2, t3;\n\t"
        "prmt.b32 t0, %4, 0, 0x4440;\n\t"
        "prmt.b32 t1, %4, 0, 0x4441;\n\t"
        "prmt.b32 t2, %4, 0, 0x4442;\n\t"
        "prmt.b32 t3, %4, 0, 0x4443;\n\t"
        "mad.lo.u32 %0, t0, %6, %5;\n\t"
        "mad.lo.u32 %1, t1, %6, %5;\n\t"
        "mad.lo.u32 %2, t2, %6, %5;\n\t"
        "mad.lo.u32 %3, t3, %6, %5;\n\t}"
        : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
        : "r"(w), "r"(base), "r"(sv));
}
template <int NC>
__device__ __forceinline__ void lds_sv(uint32_t addr, float& re, float& im) {
    if constexpr (NC == 2) {
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(re), "=f"(im) : "r"(addr));
    } else {
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(re) : "r"(addr));
        im = 0.f;
    }
}

// slot q of the gather, issued only when q < m (m: the warp's maximum in-degree, warp-uniform):
// a predicated load, no branch; re / im keep their zero otherwise.  Slots past m would all read
// the zero slot -- one shared-memory wavefront per warp and slot for nothing.
template <int NC>
__device__ __forceinline__ void lds_sv_pred(uint32_t addr, int q, int m, float& re, float& im) {
    if constexpr (NC == 2) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %3, %4;\n\t@p ld.shared.v2.f32 {%0, %1}, [%2];\n\t}"
                     : "+f"(re), "+f"(im)
                     : "r"(addr), "r"(q), "r"(m));
    } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %2, %3;\n\t@p ld.shared.f32 %0, [%1];\n\t}"
                     : "+f"(re)
                     : "r"(addr), "r"(q), "r"(m));
    }
}
#ifndef PDSSM_SEQ_PRED
#define PDSSM_SEQ_PRED 0   // measured slower (config 2 fwd 0.185 -> 0.27 ms): the zero-slot reads stay
#endif

// packed fp32x2 add (sm_100a FADD2): the complex gather tree and the bias add in half the instructions
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    float2 r;
    asm("{.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tadd.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}

template <typename T>
__device__ __forceinline__ void st_stream(T* p, float v, uint64_t pol) {
    if constexpr (std::is_same<T, float>::value) {
        asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol));
    } else {
        const __nv_bfloat16 b = __float2bfloat16_rn(v);
        asm volatile("st.global.L2::cache_hint.b16 [%0], %1, %2;" ::"l"(p), "h"(*reinterpret_cast<const uint16_t*>(&b)),
                     "l"(pol));
    }
}

#ifndef PDSSM_SEQ_DEFER_STORE
#define PDSSM_SEQ_DEFER_STORE 1   // measured: config 2 forward 0.185 -> 0.175 ms (fp32), 0.203 -> 0.187 ms (bf16)
#endif
// forward: h_{t-1} is stored at step t right after the gather loads are issued (off the chain)
// instead of right after it is computed
constexpr bool SEQ_DEFER_STORE = PDSSM_SEQ_DEFER_STORE != 0;
#ifndef PDSSM_SEQ_BWD_EARLY_STS
#define PDSSM_SEQ_BWD_EARLY_STS 0
#endif
constexpr bool SEQ_BWD_EARLY_STS = PDSSM_SEQ_BWD_EARLY_STS != 0;
#ifndef PDSSM_SEQ_SKEW
#define PDSSM_SEQ_SKEW 1   // measured: config 2 forward 0.175 -> 0.172 ms (fp32), 0.188 -> 0.179 ms (bf16)
#endif
constexpr bool SEQ_SKEW = PDSSM_SEQ_SKEW != 0;
#ifndef PDSSM_SEQ_EARLY_ADDR
#define PDSSM_SEQ_EARLY_ADDR 0
#endif
// forward (no maps, no tiers): the gather addresses of step t+1 are computed during step t, from a
// record loaded a step earlier, instead of between h_t and the store of v_{t+1} (on the chain)
constexpr bool SEQ_EARLY_ADDR = PDSSM_SEQ_EARLY_ADDR != 0;
constexpr int SEQ_G = 16;    // backward: steps per ring slot (one TMA group)
#ifndef PDSSM_SEQ_GF
#define PDSSM_SEQ_GF 32
#endif
constexpr int SEQ_GF = PDSSM_SEQ_GF;   // forward: steps per ring slot

// ============================================================================ forward
// Step t (r = t mod 8 is compile-time inside a full group, so ring rows, the exchange
// parity and pointer offsets are immediates; in-order issue: nothing waits on a load
// issued in the same step except the gather itself):
//   gather offsets (record read a step earlier) ; v_t = D_t h_{t-1} -> STS ; BARRIER ;
//   8 gather loads (zero slot past the in-degree: branch-free) ; refill (group start) ;
//   operands of step t+1 (record, trip code, D, b) and k*_{t+2} ; pairwise sum ;
//   h_t = sum + b_t ; streaming store.
// NN: the state count as a compile-time constant (0 = runtime a.N): every row offset, ring
// position and exchange address of an unrolled group becomes an immediate.
// SPC > 1 (N <= 64): SPC sequences (b, b+1, ...) of the same head h share the CTA, its per-head
// tables, the producer warp and the step barrier; blockIdx.x = p * H + h serves batch rows
// p * SPC .. p * SPC + SPC - 1.  GF: steps per TMA group.
// TIER: warp-uniform two-tier gather (4 slots when the warp's in-degree <= 4, else 8): fewer
// instructions per step, for the issue-bound launches (several CTAs per SM).
// MODE (one CTA per (sequence, chunk), SPC = 1; the chunked single-CTA path, "seqc"):
//   0  the whole sequence (tau = L);
//   1  Alg. 1 Phase A of chunk c: replay from a zero state without storing, composing (pi, d)
//      thread-locally; the final state is beta_bar_c -> chunk_state (pi_bar, d_bar, beta_bar);
//   2  Alg. 1 Phase C of chunk c: replay from carry_c (chunk_state, k_fwd_phaseB) storing h.
template <typename T, int NC, bool PD, bool AGG, bool CHECK, int NN, int SPC = 1, int GF = SEQ_GF, bool TIER = false,
          int MODE = 0>
__global__ void __launch_bounds__(MAXN + 32, 1) k_fwd_seq(SeqArgs a) {
    using SV = typename fused::SVal<NC>::type;
    constexpr int G = GF;
    constexpr int SVB = (int)sizeof(SV);
    constexpr bool CHUNK = MODE != 0;
    constexpr bool COMPOSE = AGG || MODE == 1;   // (pi, d) composed alongside
    static_assert(!CHUNK || (SPC == 1 && !AGG), "chunk modes: one sequence per CTA, maps from k_fwd_phaseB");
    extern __shared__ __align__(128) uint8_t smem[];
    const int C = CHUNK ? a.C : 1;
    const int cidx = CHUNK ? (int)(blockIdx.x % C) : 0;
    const int tb = cidx * (CHUNK ? a.tau : 0);                    // first step of the chunk
    const int N = NN ? NN : a.N, K = a.K, L = CHUNK ? min(a.tau, a.L - tb) : a.L, R = a.R;
    const int i = threadIdx.x, NW = N >> 5;
    const int sblk = CHUNK ? (int)(blockIdx.x / C) : (int)blockIdx.x;
    const int h = sblk % a.H, pidx = sblk / a.H;
    const int sub = (SPC > 1 && i < SPC * N) ? i / N : 0;   // this thread's sequence within the CTA
    const int il = i - sub * N;                             // its state
    const int w = il >> 5;                                  // its warp within the sequence
    const int s = (pidx * SPC + sub) * a.H + h;
    const Layout Ly(N, K, R, G, NC, (int)sizeof(T), (int)sizeof(T), PD, COMPOSE, false, CHUNK ? a.tau : L, SPC);
    uint8_t* ring = smem + Ly.ring;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Ly.bars);
    char* xbc = reinterpret_cast<char*>(smem + Ly.x + sub * Ly.xs);
    char* xbc2 = reinterpret_cast<char*>(smem + Ly.x2 + sub * Ly.xs);
    uint8_t* kb = smem + Ly.kb + sub * Ly.kbs + kshift(a.kstar + seq0_of(a, pidx * SPC + sub, h, tb));
    uint2* rec = reinterpret_cast<uint2*>(smem + Ly.rec);
    uint8_t* wm = smem + Ly.wm;
    uint16_t* prow = reinterpret_cast<uint16_t*>(smem + Ly.prow);
    float* dk = reinterpret_cast<float*>(smem + Ly.dk);
    const size_t row = (size_t)NC * N;
    const size_t seq0 = (size_t)s * a.L + tb;   // global row of local step 0
    const int ngroups = (L + G - 1) / G;
    const uint64_t pol = fused::policy_evict_first();
    // The sequence's k* first: it does not depend on the plan launch that precedes this
    // kernel, which may still be running (programmatic dependent launch); wait for it only
    // before the tables it writes are read.
    for (int j = 0; j < SPC; ++j) stage_k(a, smem + Ly.kb + j * Ly.kbs, seq0_of(a, pidx * SPC + j, h, tb), L);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int my_ovf = 0;
    if (i == 0) {
        for (int q = 0; q < 2 * R + 1; ++q) fused::mbar_init(bars + q, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    stage_rec(a.rec + (size_t)h * K * N * CAP, rec, K * N, bars + 2 * R);
    {   // the other one-time tables of head h
        for (int x = i; x < K * NW; x += blockDim.x) {
            const uint8_t v = a.wm[(size_t)h * K * NW + x];
            wm[x] = v;
            my_ovf |= v == WM_OVF;   // does any entry of this head need the CSR plan?
        }
        if constexpr (COMPOSE) stage_prow(a.dict_idx + (size_t)h * K * N, prow, K * N, N);
        if constexpr (PD) stage_f32(a.diag_dict + (size_t)h * K * NC * N, dk, K * NC * N);
    }
    const int XB = (N + 1) * SVB;   // bytes of one exchange row (N values + the zero slot)
    if (il == 0 && i < SPC * N) {   // the zero slots of this sequence's exchange rows
        *reinterpret_cast<SV*>(xbc + N * SVB) = fused::mk<NC>(0.f, 0.f);
        *reinterpret_cast<SV*>(xbc + XB + N * SVB) = fused::mk<NC>(0.f, 0.f);
        if constexpr (AGG) {
            *reinterpret_cast<SV*>(xbc2 + N * SVB) = fused::mk<NC>(0.f, 0.f);
            *reinterpret_cast<SV*>(xbc2 + XB + N * SVB) = fused::mk<NC>(0.f, 0.f);
        }
    }
    const bool any_ovf = __syncthreads_or(my_ovf) != 0;
    const int ROWB = (int)(row * sizeof(T));
    const int OFF_B = PD ? 0 : SPC * G * ROWB;   // slot: [D rows of seq 0..SPC-1][b rows of seq 0..SPC-1]
    const int SUBOFF = sub * G * ROWB;           // this sequence's block inside each stream
    auto issue = [&](int g, int slot) {   // producer lane 0: rows of steps [gG, gG+len) -> slot
        const int t = g * G, len = min(G, L - t);
        uint8_t* dst = ring + (size_t)slot * Ly.slot;
        fused::mbar_expect_tx(bars + slot, (uint32_t)(SPC * ((PD ? 0 : len * ROWB) + len * ROWB)));
        for (int j = 0; j < SPC; ++j) {
            const size_t sj0 = (size_t)((pidx * SPC + j) * a.H + h) * a.L + tb;
            if constexpr (!PD)
                fused::tma_1d_hint(dst + j * G * ROWB, static_cast<const T*>(a.diag) + (sj0 + t) * row, len * ROWB,
                                   bars + slot, pol);
            fused::tma_1d_hint(dst + OFF_B + j * G * ROWB, static_cast<const T*>(a.bias) + (sj0 + t) * row, len * ROWB,
                               bars + slot, pol);
        }
    };
    if (i >= SPC * N) {   // producer warp
        produce(bars, R, ngroups, issue);
        return;
    }
    float hr = 0.f, hi = 0.f;
    if constexpr (MODE == 2) {   // carry_c of this chunk
        const size_t ci = (size_t)s * C + cidx;
        hr = a.cs.carry[ci * row + il];
        if constexpr (NC == 2) hi = a.cs.carry[ci * row + N + il];
    } else if (MODE == 0 && a.h0) {
        hr = a.h0[(size_t)s * row + il];
        if constexpr (NC == 2) hi = a.h0[(size_t)s * row + N + il];
    }
    float br = 0.f, bi = 0.f, dr = 1.f, di = 0.f;
    int pi = il;
    T* hout = static_cast<T*>(a.out0) + seq0 * row + il;
    // operands of the current step
    int k, k1, m;
    uint2 rc;
    float Dr, Di, Br, Bi;
    auto load_ops = [&](const uint8_t* rp, int k_) {
        if constexpr (PD) {
            Dr = dk[(size_t)k_ * row + il];
            Di = NC == 2 ? dk[(size_t)k_ * row + N + il] : 0.f;
        } else {
            const T* Dp = reinterpret_cast<const T*>(rp);
            Dr = ldact_s(Dp + il);
            Di = NC == 2 ? ldact_s(Dp + N + il) : 0.f;
        }
        const T* Bp = reinterpret_cast<const T*>(rp + OFF_B);
        Br = ldact_s(Bp + il);
        Bi = NC == 2 ? ldact_s(Bp + N + il) : 0.f;
    };
    int slot = 0;
    uint32_t ph = 0;
    const uint8_t* sb = ring + SUBOFF;   // this sequence's rows in the current group's slot
    fused::mbar_wait(bars + 2 * R, 0);   // the records (stage_rec)
    fused::mbar_wait(bars, 0);
    k = kb[0];
    k1 = kb[1];
    rc = rec[(size_t)k * N + il];
    m = wm[k * NW + w];
    load_ops(sb, k);
    // (on by default at N = 64 only: measured config 5 forward 0.469 -> 0.447 ms, config 2 (N = 128)
    // 0.175 -> 0.181 ms)
    constexpr bool EARLY = (SEQ_EARLY_ADDR || NN == 64) && !AGG && !TIER;
    uint32_t gan[CAP];   // EARLY: this step's gather addresses (computed during the previous step)
    uint2 rcn = rc;      // EARLY: the record of the next step
    auto addr8 = [&](uint2 rc_, char* vb_, uint32_t (&a_)[CAP]) {
        uint32_t lo[4], hi4[4];
        const uint32_t vb_s = fused::smem_u32(vb_);
        gather_addr4(rc_.x, vb_s, SVB, lo);
        gather_addr4(rc_.y, vb_s, SVB, hi4);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            a_[q] = lo[q];
            a_[4 + q] = hi4[q];
        }
    };
    if constexpr (EARLY) {
        addr8(rc, xbc, gan);              // step 0 (parity 0)
        rcn = rec[(size_t)k1 * N + il];   // step 1
    }
    auto step = [&](const int r, const int g, const int t, auto ovfv) {
        constexpr bool OVF = decltype(ovfv)::value;
        char* vbc = xbc + (t & 1) * XB;
        char* vbc2 = xbc2 + (t & 1) * XB;
        uint32_t off[CAP];
#pragma unroll
        for (int q = 0; q < CAP; ++q) off[q] = __byte_perm(q < 4 ? rc.x : rc.y, 0u, 0x4440u + (uint32_t)(q & 3)) * SVB;
        uint32_t ga[CAP];   // shared addresses of this step's gather, computed before the barrier
        if constexpr (EARLY) {
#pragma unroll
            for (int q = 0; q < CAP; ++q) ga[q] = gan[q];
        } else {
            uint32_t lo[4], hi4[4] = {0u, 0u, 0u, 0u};
            const uint32_t vb_s = fused::smem_u32(vbc);
            gather_addr4(rc.x, vb_s, SVB, lo);
            if (!TIER || AGG || m > 4) gather_addr4(rc.y, vb_s, SVB, hi4);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                ga[q] = lo[q];
                ga[4 + q] = hi4[q];
            }
        }
        if constexpr (CHECK) {
            check_cpx(cpx{Dr, Di}, a.flags);
            check_cpx(cpx{Br, Bi}, a.flags);
        }
        *reinterpret_cast<SV*>(vbc + il * SVB) = fused::mk<NC>(Dr * hr - Di * hi, Dr * hi + Di * hr);
        if constexpr (AGG) *reinterpret_cast<SV*>(vbc2 + il * SVB) = fused::mk<NC>(Dr * br - Di * bi, Dr * bi + Di * br);
        const int mc = m, kc = k;
        const float bcr = Br, bci = Bi;
        const uint8_t* rpc = sb + r * ROWB;
#ifndef FWD_EXP_NOBAR   // timing experiment only: no exchange barrier (wrong results)
        compute_sync(SPC * N);
#endif
        SV v[CAP];
#if defined(FWD_EXP_SLOTS)   // timing experiment only: FWD_EXP_SLOTS gather slots (wrong results)
#pragma unroll
        for (int q = 0; q < CAP; ++q) {
            float re = 0.f, im = 0.f;
            if (q < FWD_EXP_SLOTS) lds_sv<NC>(ga[q], re, im);
            v[q] = fused::mk<NC>(re, im);
        }
#else
        const bool tier4 = TIER && !AGG && mc <= 4;   // warp-uniform
        if (tier4) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float re, im;
                lds_sv<NC>(ga[q], re, im);
                v[q] = fused::mk<NC>(re, im);
            }
        } else {
#pragma unroll
            for (int q = 0; q < CAP; ++q) {
                float re = 0.f, im = 0.f;
                if (q < GCAP) {   // (compile-time: slots past GCAP hold the zero slot)
                    if (PDSSM_SEQ_PRED && q > 0 && !AGG) lds_sv_pred<NC>(ga[q], q, mc, re, im);
                    else lds_sv<NC>(ga[q], re, im);
                }
                v[q] = fused::mk<NC>(re, im);
            }
        }
#endif
        if constexpr (SEQ_DEFER_STORE && MODE != 1) {   // h_{t-1}, stored while the gather is in flight
            if (t > 0) {
                st_stream<T>(hout, hr, pol);
                if constexpr (NC == 2) st_stream<T>(hout + N, hi, pol);
                hout += row;
            }
        }
        if (r == 0 && i == 0 && g >= 1) {   // every compute thread is done with the previous group's slot
            mbar_arrive(bars + R + (slot == 0 ? R - 1 : slot - 1));
        }
        // operands of step t+1 (consumed a step later)
        if (r < G - 1) {
            k = k1;
            if constexpr (!EARLY) rc = rec[(size_t)k * N + il];
            m = wm[k * NW + w];
            load_ops(sb + (r + 1) * ROWB, k);
        } else if (g + 1 < ngroups) {
            if (++slot == R) {
                slot = 0;
                ph ^= 1u;
            }
            sb = ring + (size_t)slot * Ly.slot + SUBOFF;
            fused::mbar_wait(bars + slot, ph);
            k = k1;
            if constexpr (!EARLY) rc = rec[(size_t)k * N + il];
            m = wm[k * NW + w];
            load_ops(sb, k);
        }
        if constexpr (EARLY) {   // addresses of step t+1 from its record (loaded a step ago); record of t+2
            addr8(rcn, xbc + ((t + 1) & 1) * XB, gan);
            rc = rcn;
        }
        k1 = kb[t + 2];
        if constexpr (EARLY) rcn = rec[(size_t)k1 * N + il];
        // pairwise sum of the 8 slots (sources past the in-degree read the zero slot)
        auto sum8 = [&](const SV (&x)[CAP], float& sr, float& si) {
            if constexpr (NC == 2) {   // packed: same pairwise order, FADD2
                float2 t = add2(add2(x[0], x[1]), add2(x[2], x[3]));
                t = add2(t, GCAP == 6 ? add2(x[4], x[5]) : add2(add2(x[4], x[5]), add2(x[6], x[7])));
                sr = t.x;
                si = t.y;
            } else if constexpr (GCAP == 6) {
                sr = ((fused::re_of<NC>(x[0]) + fused::re_of<NC>(x[1])) + (fused::re_of<NC>(x[2]) + fused::re_of<NC>(x[3]))) +
                     (fused::re_of<NC>(x[4]) + fused::re_of<NC>(x[5]));
                si = ((fused::im_of<NC>(x[0]) + fused::im_of<NC>(x[1])) + (fused::im_of<NC>(x[2]) + fused::im_of<NC>(x[3]))) +
                     (fused::im_of<NC>(x[4]) + fused::im_of<NC>(x[5]));
            } else {
                sr = ((fused::re_of<NC>(x[0]) + fused::re_of<NC>(x[1])) + (fused::re_of<NC>(x[2]) + fused::re_of<NC>(x[3]))) +
                     ((fused::re_of<NC>(x[4]) + fused::re_of<NC>(x[5])) + (fused::re_of<NC>(x[6]) + fused::re_of<NC>(x[7])));
                si = ((fused::im_of<NC>(x[0]) + fused::im_of<NC>(x[1])) + (fused::im_of<NC>(x[2]) + fused::im_of<NC>(x[3]))) +
                     ((fused::im_of<NC>(x[4]) + fused::im_of<NC>(x[5])) + (fused::im_of<NC>(x[6]) + fused::im_of<NC>(x[7])));
            }
        };
        float ar, ai, cr = 0.f, ci = 0.f;
        // SKEW (8 slots, no maps): the later-arriving slots enter last and b_t early --
        // (((v0+v1)+(v2+v3)) + (v4+v5)) + b, then + (v6+v7): two adds after the last gather load instead
        // of four (a fixed order too; not the balanced tree of the other variants)
        // (complex only: real scans measured slower with it -- config 4 0.641 -> 0.707 ms, config 5 +1%)
        constexpr bool SKEW = SEQ_SKEW && NC == 2 && GCAP == 8 && !AGG;
        bool with_b = false;
#if !defined(FWD_EXP_SLOTS)
        if constexpr (SKEW) {
            if (!tier4) {
                float2 t = add2(add2(add2(v[0], v[1]), add2(v[2], v[3])), add2(v[4], v[5]));
                t = add2(add2(t, make_float2(bcr, bci)), add2(v[6], v[7]));
                ar = t.x;
                ai = t.y;
                with_b = true;
            } else {
                ar = (fused::re_of<NC>(v[0]) + fused::re_of<NC>(v[1])) + (fused::re_of<NC>(v[2]) + fused::re_of<NC>(v[3]));
                ai = (fused::im_of<NC>(v[0]) + fused::im_of<NC>(v[1])) + (fused::im_of<NC>(v[2]) + fused::im_of<NC>(v[3]));
            }
        } else if (tier4) {
            ar = (fused::re_of<NC>(v[0]) + fused::re_of<NC>(v[1])) + (fused::re_of<NC>(v[2]) + fused::re_of<NC>(v[3]));
            ai = (fused::im_of<NC>(v[0]) + fused::im_of<NC>(v[1])) + (fused::im_of<NC>(v[2]) + fused::im_of<NC>(v[3]));
        } else {
            sum8(v, ar, ai);
        }
#else
        sum8(v, ar, ai);
#endif
        if constexpr (AGG) {
#pragma unroll
            for (int q = 0; q < CAP; ++q) v[q] = *reinterpret_cast<const SV*>(vbc2 + off[q]);
            sum8(v, cr, ci);
        }
        if (OVF && mc == WM_OVF) {   // preimage longer than CAP: CSR plan (rare, warp-uniform)
            ar = ai = cr = ci = 0.f;
            with_b = false;
            const SV* vb = reinterpret_cast<const SV*>(vbc);
            const SV* vb2 = reinterpret_cast<const SV*>(vbc2);
            const size_t e = (size_t)h * K + kc;
            const int st = __ldg(a.pstart + e * (N + 1) + il), en = __ldg(a.pstart + e * (N + 1) + il + 1);
            for (int q = st; q < en; ++q) {
                const int j = __ldg(a.psrc + e * N + q);
                ar += fused::re_of<NC>(vb[j]);
                ai += fused::im_of<NC>(vb[j]);
                if constexpr (AGG) {
                    cr += fused::re_of<NC>(vb2[j]);
                    ci += fused::im_of<NC>(vb2[j]);
                }
            }
        }
        if constexpr (NC == 2) {
            const float2 hv = with_b ? make_float2(ar, ai) : add2(make_float2(ar, ai), make_float2(bcr, bci));
            hr = hv.x;
            hi = hv.y;
        } else {
            hr = with_b ? ar : ar + bcr;
            hi = 0.f;
        }
        if constexpr (MODE != 1 && !SEQ_DEFER_STORE) {
            st_stream<T>(hout, hr, pol);
            if constexpr (NC == 2) st_stream<T>(hout + N, hi, pol);
            hout += row;
        }
        if constexpr (AGG) {
            br = cr + bcr;
            bi = NC == 2 ? ci + bci : 0.f;
        }
        if constexpr (COMPOSE) {
            // pi / d composition: d <- D_t[pi] d, pi <- P_t[pi]
            float pr, pm = 0.f;
            if constexpr (PD) {
                pr = dk[(size_t)kc * row + pi];
                if constexpr (NC == 2) pm = dk[(size_t)kc * row + N + pi];
            } else {
                const T* Dp = reinterpret_cast<const T*>(rpc);
                pr = ldact_s(Dp + pi);
                if constexpr (NC == 2) pm = ldact_s(Dp + N + pi);
            }
            const float nr = pr * dr - pm * di, ni = pr * di + pm * dr;
            dr = nr;
            di = ni;
            pi = prow[(size_t)kc * N + pi];
        }
    };
    auto run = [&](auto ovfv) {
        constexpr bool OVF = decltype(ovfv)::value;
        for (int g = 0; g < ngroups; ++g) {
            const int t0 = g * G;
            if (!OVF && t0 + G <= L) {
#pragma unroll
                for (int r = 0; r < G; ++r) step(r, g, t0 + r, ovfv);
            } else {   // ragged last group, or a head with CSR-overflow entries (rare): not unrolled
                for (int r = 0; r < min(G, L - t0); ++r) step(r, g, t0 + r, ovfv);
            }
        }
    };
    if (any_ovf) run(std::true_type{});
    else run(std::false_type{});
    if constexpr (SEQ_DEFER_STORE && MODE != 1) {   // the last state
        st_stream<T>(hout, hr, pol);
        if constexpr (NC == 2) st_stream<T>(hout + N, hi, pol);
    }
    if constexpr (MODE == 1) {   // the chunk's aggregate: beta_bar is the replay from zero
        const size_t ci = (size_t)s * C + cidx;
        a.cs.pi[ci * N + il] = (uint16_t)pi;
        a.cs.d[ci * row + il] = dr;
        a.cs.beta[ci * row + il] = hr;
        if constexpr (NC == 2) {
            a.cs.d[ci * row + N + il] = di;
            a.cs.beta[ci * row + N + il] = hi;
        }
        return;
    }
    if constexpr (MODE == 2) return;
    // chunk_state of the single chunk: carry_0 = h0; aggregate (pi_bar, d_bar, beta_bar)
    {
        a.cs.carry[(size_t)s * row + il] = a.h0 ? a.h0[(size_t)s * row + il] : 0.f;
        if constexpr (NC == 2) a.cs.carry[(size_t)s * row + N + il] = a.h0 ? a.h0[(size_t)s * row + N + il] : 0.f;
        if constexpr (AGG) {
            a.cs.pi[(size_t)s * N + il] = (uint16_t)pi;
            a.cs.d[(size_t)s * row + il] = dr;
            a.cs.beta[(size_t)s * row + il] = br;
            if constexpr (NC == 2) {
                a.cs.d[(size_t)s * row + N + il] = di;
                a.cs.beta[(size_t)s * row + N + il] = bi;
            }
            if (a.maps) {
                a.maps[((size_t)s * 2) * N + il] = (uint16_t)il;
                a.maps[((size_t)s * 2 + 1) * N + il] = (uint16_t)pi;
            }
        }
    }
}

// ============================================================================ backward
// Step t (descending; rr = position from the top of the 8-step group, compile-time in a
// full group): db_t store ; lambda_t -> STS ; BARRIER ; lp = lambda_t[P_t[j]] (P_t[j]
// read a step earlier) ; refill ; operands of step t-1 (D, e, h from the ring row, P) ;
// lambda_{t-1} = e_{t-1} + conj(D_t) lp ; dD_t store ; this thread's g_t term -> tile.
// SPC > 1 (N <= 64): SPC sequences of one head per CTA, as in k_fwd_seq.
// MODE (chunked single-CTA path, one CTA per (sequence, chunk), SPC = 1):
//   0  the whole sequence;
//   1  Phase A' of chunk c: reverse local scan from a zero incoming adjoint, nothing stored but
//      beta'_c = A_{s_c}^T lambda_loc_{s_c} -> a.betap (no h rows are read);
//   2  Phase C' of chunk c: replay from lambda_{e_c} = e_{e_c} + mu_c (k_bwd_phaseB), emitting
//      db, dD, g (and dh0 at chunk 0).
template <typename T, typename TE, int NC, bool PD, int NN, int SPC = 1, int GB = SEQ_G, int MODE = 0>
__global__ void __launch_bounds__(MAXN + 32, 1) k_bwd_seq(SeqArgs a) {
    using SV = typename fused::SVal<NC>::type;
    constexpr int G = GB;
    static_assert(32 % G == 0, "g_t is reduced every 32 steps: G must divide 32");
    constexpr int SVB = (int)sizeof(SV);
    constexpr bool CHUNK = MODE != 0;
    constexpr bool EMIT = MODE != 1;   // db, dD, g stored (and h rows read)
    // early exchange store of lambda (below): on for the whole-sequence kernel (config 2 bf16 backward
    // 0.191 -> 0.182 ms, config 4 0.668 -> 0.629 ms), off in the chunk modes (config 5 measured slower)
    constexpr bool BES = SEQ_BWD_EARLY_STS || MODE == 0;
    static_assert(!CHUNK || SPC == 1, "chunk modes: one sequence per CTA");
    extern __shared__ __align__(128) uint8_t smem[];
    const int C = CHUNK ? a.C : 1;
    const int cidx = CHUNK ? (int)(blockIdx.x % C) : 0;
    const int tb = cidx * (CHUNK ? a.tau : 0);
    const int N = NN ? NN : a.N, K = a.K, L = CHUNK ? min(a.tau, a.L - tb) : a.L, R = a.R;
    const int jt = threadIdx.x;
    const int sblk = CHUNK ? (int)(blockIdx.x / C) : (int)blockIdx.x;
    const int h = sblk % a.H, pidx = sblk / a.H;
    const int sub = (SPC > 1 && jt < SPC * N) ? jt / N : 0;
    const int j = jt - sub * N;                           // this thread's source state
    const int s = (pidx * SPC + sub) * a.H + h;
    const Layout Ly(N, K, R, G, NC, (int)sizeof(T), (int)sizeof(TE), PD, false, true, CHUNK ? a.tau : L, SPC);
    uint8_t* ring = smem + Ly.ring;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Ly.bars);
    char* xbc = reinterpret_cast<char*>(smem + Ly.x + sub * Ly.xs);
    uint8_t* kb = smem + Ly.kb + sub * Ly.kbs + kshift(a.kstar + seq0_of(a, pidx * SPC + sub, h, tb));
    uint16_t* prow = reinterpret_cast<uint16_t*>(smem + Ly.prow);
    float* dk = reinterpret_cast<float*>(smem + Ly.dk);
    float* gs = reinterpret_cast<float*>(smem + Ly.gs + sub * Ly.gss);   // [32][N+1] g terms, then [32][NW] partials
    const size_t row = (size_t)NC * N;
    const size_t seq0 = (size_t)s * a.L + tb;   // global row of local step 0
    const int ngroups = (L + G - 1) / G;
    const uint64_t pol = fused::policy_evict_first();
    const TE* ein = static_cast<const TE*>(a.bias);
    for (int q = 0; q < SPC; ++q) stage_k(a, smem + Ly.kb + q * Ly.kbs, seq0_of(a, pidx * SPC + q, h, tb), L);
    stage_prow(a.dict_idx + (size_t)h * K * N, prow, K * N, N);
    if constexpr (PD) stage_f32(a.diag_dict + (size_t)h * K * NC * N, dk, K * NC * N);
    if (jt == 0) {
        for (int q = 0; q < 2 * R; ++q) fused::mbar_init(bars + q, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int ROWB = (int)(row * sizeof(T)), EROWB = (int)(row * sizeof(TE));
    // slot: [D rows of seq 0..SPC-1][e rows ...][h rows ...], G rows per sequence and stream
    const int OFF_E = PD ? 0 : SPC * G * ROWB, OFF_H = OFF_E + SPC * G * EROWB;
    const int SUB_D = sub * G * ROWB, SUB_E = sub * G * EROWB;
    // group g: times t_hi = L-1-gG down to t_lo; D_t at row t - t_lo, e_{t-1} and h_{t-1} likewise
    auto issue = [&](int g, int slot) {
        const int t_hi = L - 1 - g * G, t_lo = max(t_hi - G + 1, 0), len = t_hi - t_lo + 1;
        uint8_t* dst = ring + (size_t)slot * Ly.slot;
        const int f_first = max(t_lo - 1, 0);                 // e_{t-1} rows needed for local t >= 1
        const int f_cnt = max(0, t_hi - 1 - f_first + 1);
        const int f_off = f_first - (t_lo - 1);
        // h_{t-1} rows: also the row before a chunk that does not start the sequence
        const int h_first = (tb > 0) ? t_lo - 1 : f_first;
        const int h_cnt = EMIT ? max(0, t_hi - 1 - h_first + 1) : 0;
        const int h_off = h_first - (t_lo - 1);
        fused::mbar_expect_tx(bars + slot,
                              (uint32_t)(SPC * ((PD ? 0 : len * ROWB) + (ein ? f_cnt * EROWB : 0) + h_cnt * ROWB)));
        for (int q = 0; q < SPC; ++q) {
            const size_t sq0 = (size_t)((pidx * SPC + q) * a.H + h) * a.L + tb;
            if constexpr (!PD)
                fused::tma_1d_hint(dst + q * G * ROWB, static_cast<const T*>(a.diag) + (sq0 + t_lo) * row, len * ROWB,
                                   bars + slot, pol);
            if (ein && f_cnt > 0)
                fused::tma_1d_hint(dst + OFF_E + q * G * EROWB + (size_t)f_off * EROWB, ein + (sq0 + f_first) * row,
                                   f_cnt * EROWB, bars + slot, pol);
            if (h_cnt > 0)
                fused::tma_1d_hint(dst + OFF_H + q * G * ROWB + (size_t)h_off * ROWB,
                                   static_cast<const T*>(a.hsaved) + (sq0 + h_first) * row, h_cnt * ROWB, bars + slot, pol);
        }
    };
    if (jt >= SPC * N) {   // producer warp
        produce(bars, R, ngroups, issue);
        return;
    }
    float lr = 0.f, li = 0.f;   // lambda_{L-1} = e_{L-1} + lam_in
    if (ein) {
        lr = ldact_s(ein + (seq0 + L - 1) * row + j);
        if constexpr (NC == 2) li = ldact_s(ein + (seq0 + L - 1) * row + N + j);
    }
    if constexpr (MODE == 0) {
        if (a.lam_in) {
            lr += a.lam_in[(size_t)s * row + j];
            if constexpr (NC == 2) li += a.lam_in[(size_t)s * row + N + j];
        }
    } else if (MODE == 2) {   // mu_c: the adjoint entering this chunk from the chunks after it
        const size_t ci = (size_t)s * C + cidx;
        lr += a.mu[ci * row + j];
        if constexpr (NC == 2) li += a.mu[ci * row + N + j];
    }
    float h0r = 0.f, h0i = 0.f;
    if (a.h0) {
        h0r = a.h0[(size_t)s * row + j];
        if constexpr (NC == 2) h0i = a.h0[(size_t)s * row + N + j];
    }
    T* dbp = static_cast<T*>(a.out0) + (seq0 + L - 1) * row + j;
    T* ddp = PD ? nullptr : static_cast<T*>(a.out1) + (seq0 + L - 1) * row + j;
    float* ddf = PD ? static_cast<float*>(a.out1) + (seq0 + L - 1) * row + j : nullptr;
    int p;
    float Dr, Di, er, ei, hr, hi;
    int slot = 0;
    uint32_t ph = 0;
    const uint8_t* sb = ring;
    fused::mbar_wait(bars, 0);
    // explicit row loads: (slot base, row index) -> operands of time t
    auto load_row = [&](const uint8_t* sb_, int ro, int t, int k_) {
        p = prow[(size_t)k_ * N + j];
        if constexpr (PD) {
            Dr = dk[(size_t)k_ * row + j];
            Di = NC == 2 ? dk[(size_t)k_ * row + N + j] : 0.f;
        } else {
            const T* Dp = reinterpret_cast<const T*>(sb_ + SUB_D + ro * ROWB);
            Dr = ldact_s(Dp + j);
            Di = NC == 2 ? ldact_s(Dp + N + j) : 0.f;
        }
        if (t > 0) {
            if (ein) {
                const TE* ep = reinterpret_cast<const TE*>(sb_ + OFF_E + SUB_E + ro * EROWB);
                er = ldact_s(ep + j);
                ei = NC == 2 ? ldact_s(ep + N + j) : 0.f;
            } else {
                er = ei = 0.f;
            }
            const T* hp = reinterpret_cast<const T*>(sb_ + OFF_H + SUB_D + ro * ROWB);
            hr = ldact_s(hp + j);
            hi = NC == 2 ? ldact_s(hp + N + j) : 0.f;
        } else {
            er = ei = 0.f;   // (a chunk's first step: its lambda_{-1} term belongs to the chunk before)
            if (EMIT && tb > 0) {
                const T* hp = reinterpret_cast<const T*>(sb_ + OFF_H + SUB_D + ro * ROWB);
                hr = ldact_s(hp + j);
                hi = NC == 2 ? ldact_s(hp + N + j) : 0.f;
            } else {
                hr = h0r;
                hi = h0i;
            }
        }
    };
    {
        const int t_lo0 = max(L - G, 0);
        load_row(sb, L - 1 - t_lo0, L - 1, kb[L - 1]);
    }
    int km1 = L > 1 ? kb[L - 2] : 0;   // k* of step t-1
    // BWD_EARLY_STS: lambda_{t-1} goes to its exchange row as soon as it is computed (step t, after
    // that step's barrier: every thread is done reading that buffer, last read at step t+1), and
    // db_{t-1} = lambda_{t-1} is stored at step t-1 while its gather load is in flight -- the stores of
    // db / dD no longer sit between lambda_{t-1} and its exchange store
    if constexpr (BES)   // lambda_{L-1}
        *reinterpret_cast<SV*>(xbc + ((L - 1) & 1) * (N * SVB) + j * SVB) = fused::mk<NC>(lr, li);
    auto step = [&](const int rr, const int g, const int t, const int t_lo, const bool inner) {
        // inner: full group with t_lo > 0 -> rows of step t-1 are compile-time, t-1 > 0
        const int v = L - 1 - t;
        if constexpr (EMIT && !BES) {
            st_stream<T>(dbp, lr, pol);                       // db_t = lambda_t
            if constexpr (NC == 2) st_stream<T>(dbp + N, li, pol);
            dbp -= row;
        }
        char* lbc = xbc + (t & 1) * (N * SVB);
        if constexpr (!BES) *reinterpret_cast<SV*>(lbc + j * SVB) = fused::mk<NC>(lr, li);
        const float Dcr = Dr, Dci = Di, ecr = er, eci = ei, hcr = hr, hci = hi;
        uint32_t la;   // shared address of lambda_t[P_t[j]], computed before the barrier
        asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(la) : "r"(p), "r"(SVB), "r"(fused::smem_u32(lbc)));
        compute_sync(SPC * N);
        SV lpv;
        {
            float re, im;
            lds_sv<NC>(la, re, im);
            lpv = fused::mk<NC>(re, im);
        }
        if constexpr (EMIT && BES) {   // db_t = lambda_t, off the chain
            st_stream<T>(dbp, lr, pol);
            if constexpr (NC == 2) st_stream<T>(dbp + N, li, pol);
            dbp -= row;
        }
        if (rr == 0 && jt == 0 && g >= 1) {   // every compute thread is done with the previous group's slot
            mbar_arrive(bars + R + (slot == 0 ? R - 1 : slot - 1));
        }
        // g_t of the previous 32 steps (v = 8 g + rr, so only the first step of every 4th group)
        if (EMIT && rr == 0 && (g % (32 / G)) == 0 && g > 0 && a.gsel) {
            const int q = j & 31, part = j >> 5, NP = N >> 5;
            const float* gr = gs + (size_t)q * (N + 1);
            float acc = 0.f;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
            int x = part;
            for (; x + 3 * NP < N; x += 4 * NP) {
                a0 += gr[x];
                a1 += gr[x + NP];
                a2 += gr[x + 2 * NP];
                a3 += gr[x + 3 * NP];
            }
            for (; x < N; x += NP) a0 += gr[x];
            acc = (a0 + a1) + (a2 + a3);
            float* red = gs + (size_t)32 * (N + 1);
            red[part * 32 + q] = acc;
            compute_sync(SPC * N);
            if (j < 32) {
                float tot = 0.f;
                for (int x = 0; x < NP; ++x) tot += red[x * 32 + j];
                a.gsel[seq0 + (L - 1 - (v - 32 + j))] = tot;
            }
            compute_sync(SPC * N);
        }
        // operands of step t-1 (consumed a step later)
        if (inner && rr < G - 1) {
            load_row(sb, G - 2 - rr, 1, km1);
            km1 = kb[t - 2];
        } else if (t > 0) {
            if (t - 1 >= t_lo) {
                load_row(sb, t - 1 - t_lo, t - 1, km1);
            } else {
                if (++slot == R) {
                    slot = 0;
                    ph ^= 1u;
                }
                sb = ring + (size_t)slot * Ly.slot;
                fused::mbar_wait(bars + slot, ph);
                const int tlo_n = max(t_lo - G, 0);
                load_row(sb, t - 1 - tlo_n, t - 1, km1);
            }
            km1 = t >= 2 ? kb[t - 2] : 0;
        }
        // (real scans, NC = 1: the imaginary terms are spelled out away -- x * 0 does not fold in IEEE
        // arithmetic, so the complex expressions would cost ~6 instructions per step for nothing)
        const float pr = fused::re_of<NC>(lpv), pm = fused::im_of<NC>(lpv);
        if constexpr (NC == 2) {
            lr = ecr + Dcr * pr + Dci * pm;               // lambda_{t-1} = e_{t-1} + conj(D_t) lp
            li = eci + Dcr * pm - Dci * pr;
        } else {
            lr = ecr + Dcr * pr;
            li = 0.f;
        }
        if constexpr (BES)
            if (t > 0) *reinterpret_cast<SV*>(xbc + ((t - 1) & 1) * (N * SVB) + j * SVB) = fused::mk<NC>(lr, li);
        if constexpr (EMIT) {
            const float ddr = NC == 2 ? hcr * pr + hci * pm : hcr * pr;   // dD_t = conj(h_{t-1}) lp
            const float ddi = NC == 2 ? hcr * pm - hci * pr : 0.f;
            if constexpr (PD) {
                ddf[0] = ddr;
                if constexpr (NC == 2) ddf[N] = ddi;
                ddf -= row;
            } else {
                st_stream<T>(ddp, ddr, pol);
                if constexpr (NC == 2) st_stream<T>(ddp + N, ddi, pol);
                ddp -= row;
            }
            if constexpr (NC == 2) {
                const float qr = Dcr * hcr - Dci * hci, qi = Dcr * hci + Dci * hcr;
                gs[(size_t)(v & 31) * (N + 1) + j] = pr * qr + pm * qi;   // this thread's term of g_t
            } else {
                gs[(size_t)(v & 31) * (N + 1) + j] = pr * (Dcr * hcr);
            }
        }
    };
    for (int g = 0; g < ngroups; ++g) {
        const int t_hi = L - 1 - g * G, t_lo = max(t_hi - G + 1, 0);
        if (t_hi - t_lo + 1 == G && t_lo > 0) {
#pragma unroll
            for (int rr = 0; rr < G; ++rr) step(rr, g, t_hi - rr, t_lo, true);
        } else {
            for (int rr = 0; rr <= t_hi - t_lo; ++rr) step(rr, g, t_hi - rr, t_lo, false);
        }
    }
    compute_sync(SPC * N);
    if (EMIT && a.gsel) {   // the last (L % 32 or 32) steps
        const int v0 = ((L - 1) / 32) * 32;
        for (int x = j; x < 32 && v0 + x < L; x += N) {
            const float* gr = gs + (size_t)x * (N + 1);
            float acc = 0.f;
            for (int y = 0; y < N; ++y) acc += gr[y];
            a.gsel[seq0 + (L - 1 - (v0 + x))] = acc;
        }
    }
    // after the chunk's first step (no e term): lambda = A_{s_c}^T lambda_{s_c}
    if constexpr (MODE == 1) {   // beta'_c
        const size_t ci = (size_t)s * C + cidx;
        a.betap[ci * row + j] = lr;
        if constexpr (NC == 2) a.betap[ci * row + N + j] = li;
    } else if (a.dh0 && cidx == 0) {   // the sequence's first step: dh0 = A_0^T lambda_0
        a.dh0[(size_t)s * row + j] = lr;
        if constexpr (NC == 2) a.dh0[(size_t)s * row + N + j] = li;
    }
}

}  // namespace seq
}  // namespace pdssm
