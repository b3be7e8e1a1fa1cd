// libpdssm.so: single-chunk backward scan launcher (k_bwd_seq, csrc/k_scan_seq.cuh).
#include "api_internal.cuh"
#include "k_scan_rc.cuh"

using namespace pdssm;
using namespace pdssm::api;

namespace pdssm {
namespace api {

constexpr int SEQ_G_ = seq::SEQ_G;

template <typename TE>
pdssm_status bwd_seq(const Geo& g, seq::SeqArgs& sa, cudaStream_t st) {
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        using TEE = typename std::conditional<std::is_same<TE, void>::value, T, TE>::type;
        // paired sequences per CTA (seq_spc) measured slower for the backward at config 4 (0.86 vs
        // 0.72 ms: 16 compute warps per SM make it issue-bound); kept selectable via PDSSM_SEQ_PAIR_BWD
        int spc = (g.N == 64 && getenv("PDSSM_SEQ_PAIR_BWD")) ? seq_spc(g) : 1;
        sa.R = seq_ring(g, true, false, sizeof(TEE), spc);
        if (spc > 1 && sa.R < 2) {
            spc = 1;
            sa.R = seq_ring(g, true, false, sizeof(TEE), 1);
        }
        sa.G = seq_group(true, spc);
        sa.spc = spc;
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            return with_pd(g.diag_mode, [&](auto pdv) {
                constexpr bool PD = decltype(pdv)::value;
                seq::Layout ly((int)g.N, (int)g.K, sa.R, sa.G, NC, (int)sizeof(T), (int)sizeof(TEE), PD, false, true,
                               (int)g.L, spc);
                auto kern = g.N == 128 ? seq::k_bwd_seq<T, TEE, NC, PD, 128>
                            : g.N == 64 ? (spc == 2 ? seq::k_bwd_seq<T, TEE, NC, PD, 64, 2, 8> : seq::k_bwd_seq<T, TEE, NC, PD, 64>)
                                        : seq::k_bwd_seq<T, TEE, NC, PD, 0>;
                pdssm_status rr = seq_set_smem((const void*)kern, ly.bytes);
                if (rr) return rr;
                kern<<<(unsigned)(g.S / spc), (unsigned)(spc * g.N) + 32, ly.bytes, st>>>(sa);   // + producer warp
                return cuda_check("bwd_seq");
            });
        });
    });
}

// e_f32: the direct state gradient e is the f32 buffer prepared from dy (else dh in the act dtype)
pdssm_status bwd_seq_run(const Geo& g, seq::SeqArgs& sa, bool e_f32, cudaStream_t st) {
    return e_f32 ? bwd_seq<float>(g, sa, st) : bwd_seq<void>(g, sa, st);
}


// recompute-mode backward, one CTA per sequence (k_scan_rc.cuh); 0 rings: does not fit
int rc_ring(const Geo& g, size_t esz_e) {
    int best = 0;
    for (int R = 2; R <= 8; ++R) {
        seq::RcLayout ly((int)g.N, (int)g.K, R, g.nc, (int)g.act, (int)esz_e, g.diag_mode == PDSSM_DIAG_PER_DICT, (int)g.L,
                         g.tau);
        if (ly.bytes <= kSeqSmemBudget) best = R;
    }
    return best;
}

bool bwd_seq_rc_applicable(const Geo& g, std::initializer_list<const void*> ptrs) {
    if (env_path_is("generic") || env_path_is("fused")) return false;
    if (g.N % 32 != 0 || g.N > seq::MAXN || (size_t)g.K * g.N * 8 > 64 * 1024 || g.L > seq::LMAX) return false;
    for (const void* p : ptrs)
        if (misaligned(p, 16)) return false;
    return rc_ring(g, 4) >= 2 && rc_ring(g, g.act) >= 2;
}

pdssm_status bwd_seq_rc_run(const Geo& g, seq::RcArgs& ra, bool e_f32, uint8_t* rec, uint8_t* wm, uint8_t* ovf,
                            cudaStream_t st) {
    seq::k_build_seq_plan<<<(unsigned)(g.H * g.K), (unsigned)g.N, (size_t)g.N * 2, st>>>(
        ra.dict_idx, rec, wm, ovf, const_cast<uint16_t*>(ra.pstart), const_cast<uint16_t*>(ra.psrc), (int)g.N, g.flags);
    pdssm_status r = cuda_check("build_seq_plan");
    if (r) return r;
    ra.rec = rec;
    ra.wm = wm;
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            return with_pd(g.diag_mode, [&](auto pdv) {
                constexpr bool PD = decltype(pdv)::value;
                auto go = [&](auto ev) -> pdssm_status {
                    using TE = decltype(ev);
                    ra.R = rc_ring(g, sizeof(TE));
                    seq::RcLayout ly((int)g.N, (int)g.K, ra.R, NC, (int)sizeof(T), (int)sizeof(TE), PD, (int)g.L, g.tau);
                    auto kern = seq::k_bwd_seq_rc<T, TE, NC, PD>;
                    pdssm_status rr = seq_set_smem((const void*)kern, ly.bytes);
                    if (rr) return rr;
                    kern<<<(unsigned)g.S, (unsigned)g.N + 32, ly.bytes, st>>>(ra);
                    return cuda_check("bwd_seq_rc");
                };
                return e_f32 ? go(float{}) : go(T{});
            });
        });
    });
}


// chunked single-CTA path: Phase A' (MODE 1: beta'_c) -> Phase B' (mu chain through the forward
// aggregates: k_bwd_phaseB) -> Phase C' (MODE 2: replay from e + mu_c, emitting the gradients)
template <typename TE>
pdssm_status bwd_seqc(const Geo& g, seq::SeqArgs& sa, cudaStream_t st, bool phaseA_only) {
    const int64_t ctas = g.S * g.C;
    sa.G = seqc_group(g.N);
    sa.spc = 1;
    sa.tau = g.tau;
    sa.C = g.C;
    const int thr = threads_for(g.N);
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        using TEE = typename std::conditional<std::is_same<TE, void>::value, T, TE>::type;
        sa.R = seq_ring(g, true, false, sizeof(TEE), 1, g.tau, ctas, sa.G);
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            return with_pd(g.diag_mode, [&](auto pdv) {
                constexpr bool PD = decltype(pdv)::value;
                seq::Layout ly((int)g.N, (int)g.K, sa.R, sa.G, NC, (int)sizeof(T), (int)sizeof(TEE), PD, false, true, g.tau,
                               1);
                auto kA = g.N == 128 ? seq::k_bwd_seq<T, TEE, NC, PD, 128, 1, kSeqcG128, 1>
                          : g.N == 64 ? seq::k_bwd_seq<T, TEE, NC, PD, 64, 1, kSeqcG64, 1>
                                      : seq::k_bwd_seq<T, TEE, NC, PD, 0, 1, kSeqcG128, 1>;
                auto kC = g.N == 128 ? seq::k_bwd_seq<T, TEE, NC, PD, 128, 1, kSeqcG128, 2>
                          : g.N == 64 ? seq::k_bwd_seq<T, TEE, NC, PD, 64, 1, kSeqcG64, 2>
                                      : seq::k_bwd_seq<T, TEE, NC, PD, 0, 1, kSeqcG128, 2>;
                pdssm_status rr = seq_set_smem((const void*)kA, ly.bytes);
                if (rr) return rr;
                kA<<<(unsigned)ctas, (unsigned)g.N + 32, ly.bytes, st>>>(sa);
                if ((rr = cuda_check("bwd_seqc_A")) || phaseA_only) return rr;   // (sequence-parallel summary)
                k_bwd_phaseB<NC><<<(unsigned)g.S, thr, (size_t)NC * g.N * 4, st>>>(sa.cs, sa.betap, sa.lam_in, sa.mu,
                                                                                     nullptr, (int)g.N, g.C);
                if ((rr = cuda_check("bwd_seqc_B"))) return rr;
                if ((rr = seq_set_smem((const void*)kC, ly.bytes))) return rr;
                kC<<<(unsigned)ctas, (unsigned)g.N + 32, ly.bytes, st>>>(sa);
                return cuda_check("bwd_seqc_C");
            });
        });
    });
}

pdssm_status bwd_seqc_run(const Geo& g, seq::SeqArgs& sa, bool e_f32, cudaStream_t st, bool phaseA_only) {
    return e_f32 ? bwd_seqc<float>(g, sa, st, phaseA_only) : bwd_seqc<void>(g, sa, st, phaseA_only);
}

}  // namespace api
}  // namespace pdssm

PDSSM_DEFINE_ERRWORD(seq_bwd)
