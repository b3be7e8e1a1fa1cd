// Internal host-side helpers shared by the library's translation units (not part of the ABI).
// The library is split into several .cu files that nvcc compiles in parallel
// (paper_2605_19150_b200/_build.py); this header holds the dims/geometry logic, the
// workspace carve-up and the declarations of the per-file launchers.
#pragma once
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <mutex>
#include <string>
#include <type_traits>
#include <utility>

#include "pdssm_common.cuh"
#include "k_scan_seq.cuh"   // + k_scan_fwd.cuh, k_scan_fused.cuh (Args and Layout types)
#include "k_scan_bwd.cuh"   // reduce_dict_ws_bytes
#include "k_scan_rc.cuh"    // RcArgs

namespace pdssm {
namespace api {

// records the message for pdssm_last_error (thread-local) and returns s (pdssm_api.cu)
pdssm_status fail(pdssm_status s, const char* fmt, ...);

struct Geo {
    int64_t B, H, L, N, K, S, d_in, P;
    int tau, C, nc, dtype, diag_mode;
    uint32_t flags;
    size_t act;   // bytes per act element
};

constexpr uint32_t kKnownFlags = PDSSM_CHECK_FINITE | PDSSM_DETERMINISTIC | PDSSM_SAVE_STATES | PDSSM_EXPORT_MAPS;

// single-chunk (tau = L) scan kernels: one CTA of N threads per sequence
inline bool seq_shape_ok(int64_t N, int64_t K, int64_t L, int nc, size_t act) {
    (void)nc; (void)act;
    return N % 32 == 0 && N <= seq::MAXN && (size_t)K * N * 8 <= 64 * 1024 && L <= seq::LMAX;
}
// SM count of the current device (cached per device ordinal)
inline int num_sms_dev() { return num_sms(); }
inline bool env_path_is(const char* v) {
    const char* p = getenv("PDSSM_PATH");
    return p && strcmp(p, v) == 0;
}

// Library default chunk length (reading R20: tuning only).  When the B*H sequences
// alone fill most of the SMs, one chunk per sequence (tau = L) runs the single-pass
// CTA-per-sequence kernels; otherwise tau = 64 (chunked, decoupled look-back).
inline int default_tau(const pdssm_dims* d) {
    const int64_t S = d->batch * d->heads;
    const int64_t sms = num_sms_dev();
    const bool forced_chunked = env_path_is("fused") || env_path_is("generic");
    const size_t act = d->dtype == PDSSM_BF16 ? 2 : 4;
    if (forced_chunked || d->len > (int64_t)1 << 30) return 64;
    // one CTA per sequence when the sequences fill most SMs
    if (seq_shape_ok(d->state, d->dict, d->len, d->is_complex, act) && (env_path_is("seq") || S * 10 >= sms * 6))
        return (int)d->len;
    // otherwise the chunked single-CTA path ("seqc"): two passes per chunk, but the per-step chain of
    // a chunk is tau steps long instead of L, and with small TMA groups (seqc_group) two or three
    // (sequence, chunk) CTAs share an SM and interleave their chains.  ~2.8 chunks per SM measured
    // best (tau sweeps, profiles/r02s_*: config 3 tau 1384 -> 92 M tok/s vs 60 for the
    // warp-per-chunk path; config 5 tau 2521 -> 247 vs 197 M tok/s at 2 chunks per SM).
    const int64_t C = ceil_div(28 * sms, 10 * S);
    const int64_t tau = std::max<int64_t>(ceil_div(d->len, C), 1);
    if (seq_shape_ok(d->state, d->dict, std::min<int64_t>(tau, d->len), d->is_complex, act) &&
        (env_path_is("seqc") || tau >= 256))
        return (int)tau;
    return 64;
}

inline pdssm_status geo_of(const pdssm_dims* d, Geo* g) {
    if (!d) return fail(PDSSM_ERR_NULL, "dims is NULL");
    if (d->batch < 1 || d->heads < 1 || d->len < 1)
        return fail(PDSSM_ERR_SHAPE, "batch, heads, len must be >= 1 (got %lld, %lld, %lld)", (long long)d->batch,
                    (long long)d->heads, (long long)d->len);
    if (d->state < 1 || d->state > 1024) return fail(PDSSM_ERR_SHAPE, "state N must be in [1, 1024] (got %lld)", (long long)d->state);
    if (d->dict < 1 || d->dict > 256) return fail(PDSSM_ERR_SHAPE, "dict K must be in [1, 256] (got %lld)", (long long)d->dict);
    if (d->is_complex != 1 && d->is_complex != 2) return fail(PDSSM_ERR_SHAPE, "is_complex must be 1 or 2");
    if (d->dtype != PDSSM_F32 && d->dtype != PDSSM_BF16) return fail(PDSSM_ERR_DTYPE, "unknown dtype %d", d->dtype);
    if (d->diag_mode != PDSSM_DIAG_PER_STEP && d->diag_mode != PDSSM_DIAG_PER_DICT)
        return fail(PDSSM_ERR_DTYPE, "unknown diag_mode %d", d->diag_mode);
    if (d->flags & ~kKnownFlags) return fail(PDSSM_ERR_DTYPE, "unknown flag bits 0x%x", d->flags & ~kKnownFlags);
    if (d->reserved != 0) return fail(PDSSM_ERR_DTYPE, "reserved must be 0");
    if (d->chunk < 0) return fail(PDSSM_ERR_SHAPE, "chunk must be >= 0");
    if (d->p_out < 0 || d->d_in < 0) return fail(PDSSM_ERR_SHAPE, "p_out, d_in must be >= 0");
    g->B = d->batch; g->H = d->heads; g->L = d->len; g->N = d->state; g->K = d->dict;
    g->S = g->B * g->H; g->d_in = d->d_in; g->P = d->p_out;
    g->tau = d->chunk ? d->chunk : default_tau(d);
    if (g->tau > g->L) g->tau = (int)g->L;
    g->C = (int)ceil_div(g->L, g->tau);
    if ((int64_t)g->S * g->C > (int64_t)1 << 31) return fail(PDSSM_ERR_SHAPE, "too many (sequence, chunk) items");
    g->nc = d->is_complex; g->dtype = d->dtype; g->diag_mode = d->diag_mode; g->flags = d->flags;
    g->act = d->dtype == PDSSM_BF16 ? 2 : 4;
    return PDSSM_OK;
}

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Bump {
    char* base;
    size_t off = 0;
    explicit Bump(void* p) : base(static_cast<char*>(p)) {}
    template <typename T> T* take(size_t bytes) {
        T* r = reinterpret_cast<T*>(base ? base + off : nullptr);
        off += align256(bytes);
        return r;
    }
};

inline size_t plan_bytes(const Geo& g) {
    return align256((size_t)g.H * g.K * (g.N + 1) * 2) + align256((size_t)g.H * g.K * g.N * 2);
}
inline size_t cs_pi_bytes(const Geo& g) { return align256((size_t)g.S * g.C * g.N * 2); }
inline size_t cs_f_bytes(const Geo& g) { return align256((size_t)g.S * g.C * g.nc * g.N * 4); }
inline size_t chunk_state_bytes_g(const Geo& g) { return cs_pi_bytes(g) + 3 * cs_f_bytes(g); }
inline size_t seq_f_bytes(const Geo& g) { return align256((size_t)g.S * g.L * g.nc * g.N * 4); }
// single-chunk plan: preimage records [H][K][N][8], warp trip counts, overflow flags
inline size_t seq_rec_bytes(const Geo& g) { return align256((size_t)g.H * g.K * g.N * 8); }
inline size_t seq_wm_bytes(const Geo& g) { return align256((size_t)g.H * g.K * (g.N / 32 > 0 ? g.N / 32 : 1)); }
inline size_t seq_ovf_bytes(const Geo& g) { return align256((size_t)g.H * g.K); }
inline size_t seq_plan_bytes(const Geo& g) { return seq_rec_bytes(g) + seq_wm_bytes(g) + seq_ovf_bytes(g); }
// readout weights staged in act dtype (Cp or CT), H*P*c*N elements
inline size_t readout_w_bytes(const Geo& g) {   // fp32: hi part + tf32 lo part (pre-split weights)
    return g.P > 0 ? align256((size_t)g.H * g.P * g.nc * g.N * g.act) * (g.act == 4 ? 2 : 1) : 0;
}
// the lo part of the pre-split fp32 readout weights inside the readout workspace (else NULL)
inline float* readout_lo_part(const Geo& g, void* wbuf) {
    return g.act == 4 && g.P <= 128 ? reinterpret_cast<float*>(static_cast<char*>(wbuf) +
                                                                 align256((size_t)g.H * g.P * g.nc * g.N * 4))
                                    : nullptr;
}
inline size_t seq_act_bytes(const Geo& g) { return align256((size_t)g.S * g.L * g.nc * g.N * g.act); }
// NEXT-2 fused layer GEMM: stacked weight rows [S | pad | B | W_d] (upper bound), fp32 adds the tf32 lo part
inline int64_t layer_w_rows(const Geo& g) { return g.H * g.K + 256 + 2 * g.H * g.nc * g.N; }
inline size_t layer_w_bytes(const Geo& g) {
    return g.d_in > 0 ? align256((size_t)layer_w_rows(g) * g.d_in * g.act) + (g.act == 4 ? align256((size_t)layer_w_rows(g) * g.d_in * 4) : 0)
                      : 0;
}
inline int npad8(int64_t N) { return (int)((N + 7) & ~7); }
inline size_t summary_block_bytes(const Geo& g) { return (size_t)npad8(g.N) * 2 + (size_t)2 * g.nc * g.N * 4; }

inline ChunkStateView cs_view(const Geo& g, void* p) {
    char* b = static_cast<char*>(p);
    ChunkStateView v;
    v.pi = reinterpret_cast<uint16_t*>(b);
    v.d = reinterpret_cast<float*>(b + cs_pi_bytes(g));
    v.beta = reinterpret_cast<float*>(b + cs_pi_bytes(g) + cs_f_bytes(g));
    v.carry = reinterpret_cast<float*>(b + cs_pi_bytes(g) + 2 * cs_f_bytes(g));
    return v;
}

inline size_t ws_bytes_g(const Geo& g, int op) {
    switch (op) {
        case PDSSM_OP_SELECT:
            return align256((size_t)g.S * g.L * g.K * 4);
        case PDSSM_OP_FWD:
            return plan_bytes(g) + (g.P > 0 ? seq_act_bytes(g) + readout_w_bytes(g) : 0) +
                   fused_plan_bytes(g.H, g.K, g.N) + fused_ctrl_bytes(g.S, g.C, g.H) + seq_plan_bytes(g);
        case PDSSM_OP_BWD:
            return 2 * cs_f_bytes(g) + (g.P > 0 ? seq_f_bytes(g) + readout_w_bytes(g) : 0) +
                   (g.diag_mode == PDSSM_DIAG_PER_DICT ? seq_f_bytes(g) + reduce_dict_ws_bytes(g.S, g.L, g.K, g.nc * g.N)
                                                        : 0) +
                   fused_ctrl_bytes(g.S, g.C, g.H) + plan_bytes(g) + seq_plan_bytes(g);
        case PDSSM_OP_READOUT:
            return readout_w_bytes(g);
        case PDSSM_OP_SOFT: {   // s [H][B L][Kp] and Mt [H][N^2][Kp] in the act dtype
            const int64_t kp = (g.K + 7) / 8 * 8;
            return align256((size_t)g.H * g.B * g.L * kp * g.act) + align256((size_t)g.H * g.N * g.N * kp * g.act);
        }
        case PDSSM_OP_LAYER: {   // b_t, D_t (generator), stacked weights of the fused layer GEMM, scan ws
            const size_t sel = align256((size_t)g.S * g.L * g.K * 4), fwd = ws_bytes_g(g, PDSSM_OP_FWD);
            return 2 * seq_act_bytes(g) + layer_w_bytes(g) + (sel > fwd ? sel : fwd);
        }
        case PDSSM_OP_SEGMENT: {
            size_t fwd = plan_bytes(g) + chunk_state_bytes_g(g) + seq_plan_bytes(g);
            size_t bwd = 2 * cs_f_bytes(g) + (g.P > 0 ? seq_f_bytes(g) + readout_w_bytes(g) : 0);
            return fwd > bwd ? fwd : bwd;
        }
        default:
            return 0;
    }
}

inline bool misaligned(const void* p, size_t a) { return p && (reinterpret_cast<uintptr_t>(p) % a) != 0; }

inline pdssm_status cuda_check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return PDSSM_OK;
}

inline int threads_for(int64_t N) { return (int)((N + 31) / 32 * 32); }

template <typename F>
inline pdssm_status with_nc(int nc, F&& f) {
    if (nc == 1) return f(std::integral_constant<int, 1>{});
    return f(std::integral_constant<int, 2>{});
}

template <typename F>
inline pdssm_status with_act(int dtype, F&& f) {
    if (dtype == PDSSM_BF16) return f(__nv_bfloat16{});
    return f(float{});
}

template <typename F>
inline pdssm_status with_pd(int mode, F&& f) {
    if (mode == PDSSM_DIAG_PER_DICT) return f(std::true_type{});
    return f(std::false_type{});
}

inline pdssm_status set_smem(const void* fn, size_t bytes) {
    if (bytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    }
    return PDSSM_OK;
}

// ------------------------------------------------------------------ fused fast path
// PDSSM_PATH=generic forces the three-phase kernels (used by the tests to cover both).
inline bool path_generic_forced() {
    const char* p = getenv("PDSSM_PATH");
    return p && strcmp(p, "generic") == 0;
}
// PDSSM_PATH=fused makes the fused path mandatory (tests): a shape it cannot take is an error
inline bool path_fused_forced() {
    const char* p = getenv("PDSSM_PATH");
    return p && strcmp(p, "fused") == 0;
}
// ---------------------------------------------------------------------------
// single-chunk path: plan, sizing, launches
// ---------------------------------------------------------------------------

constexpr size_t kSeqSmemBudget = 200 * 1024;
// CTAs of the single-chunk kernels per SM when sequences outnumber the SMs (config 4's backward
// measured 0.72 ms at 4 per SM in two waves against 0.78 ms at 7 per SM in one: issue-bound)
constexpr int kSeqMaxPerSm = 4;
constexpr int kSeqG = seq::SEQ_G;     // backward group
constexpr int kSeqGF = seq::SEQ_GF;   // forward group
// group of the chunked single-CTA kernels (fwd and bwd): small, so that the rings of two or more
// (sequence, chunk) CTAs fit one SM and their step chains interleave (measured, config 3 / 5:
// 8 steps at N = 128, 16 at N = 64; the single-chunk kernels' 32 / 16 allow one CTA per SM)
constexpr int kSeqcG128 = 8, kSeqcG64 = 16;
inline int seqc_group(int64_t N) { return N == 64 ? kSeqcG64 : kSeqcG128; }   // (as instantiated)

// Sequences per CTA of the single-chunk kernels: with N <= 64 and more sequences than SMs, two
// sequences (batch rows b, b + 1) of one head share a CTA, its per-head tables, producer warp and
// step barrier -- the per-sequence shared memory shrinks, so every CTA is resident in one wave
// (config 4: 1024 sequences as 512 CTAs, 4 per SM).
inline int seq_spc(const Geo& g) {
    return (g.N <= 64 && g.N % 32 == 0 && g.B % 2 == 0 && g.S > (int64_t)num_sms_dev()) ? 2 : 1;
}
// steps per TMA group: the paired variants use shorter groups to fit 4 CTAs per SM
inline int seq_group(bool bwd, int spc) { return bwd ? (spc > 1 ? 8 : kSeqG) : (spc > 1 ? 16 : kSeqGF); }

// ring depth R for this shape (0: the layout does not fit).  When there are more CTAs than
// SMs, the budget is split so that ceil(#CTAs / #SMs) CTAs (up to 4) fit per SM.
// Lk: the steps one CTA covers (g.L, or tau for the chunked single-CTA path); ctas: CTAs launched
inline int seq_ring(const Geo& g, bool bwd, bool agg, size_t esz_e, int spc = 1, int64_t Lk = 0, int64_t ctas_in = 0,
                    int G_in = 0) {
    const int G = G_in > 0 ? G_in : seq_group(bwd, spc);
    if (Lk <= 0) Lk = g.L;
    const int ngroups = (int)ceil_div(Lk, G);
    const int64_t ctas = ctas_in > 0 ? ctas_in : g.S / spc;
    int cap = kSeqMaxPerSm;   // PDSSM_SEQ_MAX_PER_SM: tuning experiments only
    if (const char* e = getenv("PDSSM_SEQ_MAX_PER_SM")) cap = std::max(1, std::min(8, atoi(e)));
    const int64_t want = std::min<int64_t>(std::max<int64_t>(ceil_div(ctas, num_sms_dev()), 1), cap);
    // the largest ring at the wanted occupancy; if even two slots do not fit there, fewer CTAs per SM
    // (down to one): occupancy degrades, applicability does not depend on the batch size
    for (int64_t per_sm = want; per_sm >= 1; --per_sm) {
        const size_t budget = std::min<size_t>(kSeqSmemBudget, (size_t)(226 * 1024) / (size_t)per_sm - 1024);
        int best = 0;
        for (int R = 2; R <= 16 && R <= ngroups + 1; ++R) {
            seq::Layout ly((int)g.N, (int)g.K, R, G, g.nc, (int)g.act, (int)esz_e, g.diag_mode == PDSSM_DIAG_PER_DICT,
                           agg, bwd, (int)Lk, spc);
            if (ly.bytes <= budget) best = R;
        }
        if (best == 0 && ngroups <= 1) {
            seq::Layout ly((int)g.N, (int)g.K, 2, G, g.nc, (int)g.act, (int)esz_e, g.diag_mode == PDSSM_DIAG_PER_DICT, agg,
                           bwd, (int)Lk, spc);
            if (ly.bytes <= budget) best = 2;
        }
        if (best >= 2) return best;
    }
    return 0;
}

// chunked single-CTA path: one CTA per (sequence, chunk) with the single-chunk kernels' step
// (k_fwd_seq / k_bwd_seq MODE 1 / 2) around the generic Phase B / B' carry kernels
inline bool seqc_applicable(const Geo& g, std::initializer_list<const void*> ptrs) {
    if (g.C <= 1 || env_path_is("fused") || env_path_is("generic") || env_path_is("seq")) return false;
    if (!env_path_is("seqc") && g.tau <= fused::TAUMAX) return false;   // short chunks: the warp-per-chunk path
    if (!seq_shape_ok(g.N, g.K, g.tau, g.nc, g.act)) return false;
    for (const void* p : ptrs)
        if (misaligned(p, 16)) return false;
    const int64_t ctas = g.S * g.C;
    const int G = seqc_group(g.N);
    return seq_ring(g, false, true, g.act, 1, g.tau, ctas, G) >= 2 && seq_ring(g, true, false, 4, 1, g.tau, ctas, G) >= 2 &&
           seq_ring(g, true, false, g.act, 1, g.tau, ctas, G) >= 2;
}

// the chunked single-CTA Phase A (k_fwd_seq MODE 1) for the sequence-parallel segment summary: chunks of
// >= 128 steps (shorter ones keep the generic per-chunk kernel), 16-byte aligned rows, a ring that fits
inline bool seqc_phaseA_ok(const Geo& g, std::initializer_list<const void*> ptrs) {
    if (env_path_is("generic") || g.tau < 128 || !seq_shape_ok(g.N, g.K, g.tau, g.nc, g.act)) return false;
    for (const void* p : ptrs)
        if (misaligned(p, 16)) return false;
    return seq_ring(g, false, true, g.act, 1, g.tau, g.S * g.C, seqc_group(g.N)) >= 2;
}

// its backward counterpart (k_bwd_seq MODE 1, beta'_c), adjoint rows of esz_e bytes
inline bool seqc_phaseA_bwd_ok(const Geo& g, size_t esz_e, std::initializer_list<const void*> ptrs) {
    if (env_path_is("generic") || g.tau < 128 || !seq_shape_ok(g.N, g.K, g.tau, g.nc, g.act)) return false;
    for (const void* p : ptrs)
        if (misaligned(p, 16)) return false;
    return seq_ring(g, true, false, esz_e, 1, g.tau, g.S * g.C, seqc_group(g.N)) >= 2;
}

inline bool seq_applicable(const Geo& g, std::initializer_list<const void*> ptrs) {
    if (g.C != 1 || env_path_is("fused") || env_path_is("generic")) return false;
    if (!seq_shape_ok(g.N, g.K, g.L, g.nc, g.act)) return false;
    for (const void* p : ptrs)
        if (misaligned(p, 16)) return false;
    return seq_ring(g, false, true, g.act) >= 2 && seq_ring(g, true, false, 4) >= 2;
}

inline pdssm_status seq_set_smem(const void* f, size_t bytes) {
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return PDSSM_OK;
}

// ---------------------------------------------------------------------------
// launchers defined in the other translation units
// ---------------------------------------------------------------------------
// api_seq_fwd.cu / api_seq_bwd.cu: single-chunk path (one CTA per sequence)
pdssm_status fwd_seq(const Geo& g, seq::SeqArgs& sa, uint8_t* rec, uint8_t* wm, uint8_t* ovf, cudaStream_t st);
pdssm_status bwd_seq_run(const Geo& g, seq::SeqArgs& sa, bool e_f32, cudaStream_t st);
// chunked single-CTA path (MODE 1 / phase B / MODE 2)
pdssm_status fwd_seqc(const Geo& g, seq::SeqArgs& sa, uint8_t* rec, uint8_t* wm, uint8_t* ovf, cudaStream_t st,
                      bool phaseA_only = false);
pdssm_status bwd_seqc_run(const Geo& g, seq::SeqArgs& sa, bool e_f32, cudaStream_t st, bool phaseA_only = false);
// api_seq_bwd.cu: recompute-mode backward, one CTA per sequence (k_scan_rc.cuh)
bool bwd_seq_rc_applicable(const Geo& g, std::initializer_list<const void*> ptrs);
pdssm_status bwd_seq_rc_run(const Geo& g, seq::RcArgs& ra, bool e_f32, uint8_t* rec, uint8_t* wm, uint8_t* ovf,
                            cudaStream_t st);
// api_fused.cu: chunked warp-per-item path with decoupled look-back
bool fused_applicable(const Geo& g, std::initializer_list<const void*> ptrs);
pdssm_status fwd_fused(const Geo& g, fused::FusedArgs& fa, uint8_t* rec, uint32_t* hdr, cudaStream_t st);
pdssm_status bwd_fused_run(const Geo& g, fused::FusedArgs& fa, bool e_f32, cudaStream_t st);
// api_gemm.cu: readout y = Re(C h) after the scan, and the backward's e = dh + conj(C)^T dy
pdssm_status readout_run(const Geo& g, const void* h, const float* C, void* y, void* wbuf, cudaStream_t st);
pdssm_status prepare_e_run(const Geo& g, const void* dh, const void* dy, const float* C, float* e, void* wbuf,
                           cudaStream_t st);

// device error words: one per translation unit (internal linkage, pdssm_common.cuh);
// each reader copies its unit's word out and clears it
cudaError_t errword_core(uint32_t* w);
cudaError_t errword_seq_fwd(uint32_t* w);
cudaError_t errword_seq_bwd(uint32_t* w);
cudaError_t errword_fused(uint32_t* w);
cudaError_t errword_gemm(uint32_t* w);
cudaError_t errword_grad(uint32_t* w);

}  // namespace api
}  // namespace pdssm

#define PDSSM_DEFINE_ERRWORD(name)                                                       \
    cudaError_t pdssm::api::errword_##name(uint32_t* w) {                                 \
        cudaError_t e = cudaMemcpyFromSymbol(w, pdssm::g_err_word, sizeof(uint32_t));     \
        if (e != cudaSuccess) return e;                                                  \
        const uint32_t z = 0;                                                            \
        return cudaMemcpyToSymbol(pdssm::g_err_word, &z, sizeof(uint32_t));              \
    }
