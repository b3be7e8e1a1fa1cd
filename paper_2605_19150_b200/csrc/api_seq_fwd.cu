// libpdssm.so: single-chunk forward scan launcher (k_fwd_seq, csrc/k_scan_seq.cuh).
#include "api_internal.cuh"

using namespace pdssm;
using namespace pdssm::api;

namespace pdssm {
namespace api {

constexpr int SEQ_GF_ = seq::SEQ_GF;

pdssm_status fwd_seq(const Geo& g, seq::SeqArgs& sa, uint8_t* rec, uint8_t* wm, uint8_t* ovf, cudaStream_t st) {
    seq::k_build_seq_plan<<<(unsigned)(g.H * g.K), (unsigned)g.N, (size_t)g.N * 2, st>>>(
        sa.dict_idx, rec, wm, ovf, const_cast<uint16_t*>(sa.pstart), const_cast<uint16_t*>(sa.psrc), (int)g.N, g.flags);
    pdssm_status r = cuda_check("build_seq_plan");
    if (r) return r;
    // the single chunk's aggregate is composed only on request: no backward reads it (dh0 comes
    // from the chunk-0 replay, PDSSM_EXPORT_MAPS exports it for tests and SP)
    const bool agg = (g.flags & PDSSM_EXPORT_MAPS) != 0;
    const bool chk = (g.flags & PDSSM_CHECK_FINITE) != 0;
    // paired sequences per CTA: production variant (no maps, no checks) at N = 64 only
    int spc = (agg || chk || g.N != 64) ? 1 : seq_spc(g);
    sa.R = seq_ring(g, false, agg, g.act, spc);
    if (spc > 1 && sa.R < 2) {
        spc = 1;
        sa.R = seq_ring(g, false, agg, g.act, 1);
    }
    sa.G = seq_group(false, spc);
    sa.spc = spc;
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            return with_pd(g.diag_mode, [&](auto pdv) {
                constexpr bool PD = decltype(pdv)::value;
                auto go = [&](auto aggv, auto chkv) {
                    constexpr bool AGG = decltype(aggv)::value;
                    constexpr bool CHK = decltype(chkv)::value;
                    seq::Layout ly((int)g.N, (int)g.K, sa.R, sa.G, NC, (int)sizeof(T), (int)sizeof(T), PD, AGG, false,
                                   (int)g.L, spc);
                    // compile-time N for the production variants (no maps, no checks)
                    auto kern = seq::k_fwd_seq<T, NC, PD, AGG, CHK, 0>;
                    if constexpr (!AGG && !CHK) {
                        if (g.N == 128)
                            kern = getenv("PDSSM_SEQ_TIER") ? seq::k_fwd_seq<T, NC, PD, false, false, 128, 1, SEQ_GF_, true>
                                                            : seq::k_fwd_seq<T, NC, PD, false, false, 128>;
                        else if (g.N == 64)
                            kern = spc == 2 ? (getenv("PDSSM_SEQ_NO_TIER") ? seq::k_fwd_seq<T, NC, PD, false, false, 64, 2, 16>
                                                                          : seq::k_fwd_seq<T, NC, PD, false, false, 64, 2, 16, true>)
                                            : seq::k_fwd_seq<T, NC, PD, false, false, 64>;
                    }
                    pdssm_status rr = seq_set_smem((const void*)kern, ly.bytes);
                    if (rr) return rr;
                    // programmatic dependent launch: the prologue overlaps the plan kernel's tail
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3((unsigned)(g.S / spc));
                    cfg.blockDim = dim3((unsigned)(spc * g.N) + 32);   // + producer warp
                    cfg.dynamicSmemBytes = ly.bytes;
                    cfg.stream = st;
                    cudaLaunchAttribute attr[1];
                    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    attr[0].val.programmaticStreamSerializationAllowed = 1;
                    cfg.attrs = attr;
                    cfg.numAttrs = 1;
                    cudaError_t le = cudaLaunchKernelEx(&cfg, kern, sa);
                    if (le != cudaSuccess) return fail(PDSSM_ERR_CUDA, "fwd_seq launch: %s", cudaGetErrorString(le));
                    return cuda_check("fwd_seq");
                };
                if (agg) return chk ? go(std::true_type{}, std::true_type{}) : go(std::true_type{}, std::false_type{});
                return chk ? go(std::false_type{}, std::true_type{}) : go(std::false_type{}, std::false_type{});
            });
        });
    });
}


// chunked single-CTA path: Phase A (MODE 1, every chunk's aggregate) -> Phase B (carries and, under
// EXPORT_MAPS, the exclusive prefix maps: k_fwd_phaseB) -> Phase C (MODE 2, replay storing h)
pdssm_status fwd_seqc(const Geo& g, seq::SeqArgs& sa, uint8_t* rec, uint8_t* wm, uint8_t* ovf, cudaStream_t st,
                      bool phaseA_only) {
    seq::k_build_seq_plan<<<(unsigned)(g.H * g.K), (unsigned)g.N, (size_t)g.N * 2, st>>>(
        sa.dict_idx, rec, wm, ovf, const_cast<uint16_t*>(sa.pstart), const_cast<uint16_t*>(sa.psrc), (int)g.N, g.flags);
    pdssm_status r = cuda_check("build_seq_plan");
    if (r) return r;
    const int64_t ctas = g.S * g.C;
    sa.G = seqc_group(g.N);
    sa.spc = 1;
    sa.tau = g.tau;
    sa.C = g.C;
    const int thr = threads_for(g.N);
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            return with_pd(g.diag_mode, [&](auto pdv) {
                constexpr bool PD = decltype(pdv)::value;
                auto launch = [&](auto kern, bool compose, const char* what) -> pdssm_status {
                    sa.R = seq_ring(g, false, compose, g.act, 1, g.tau, ctas, sa.G);
                    seq::Layout ly((int)g.N, (int)g.K, sa.R, sa.G, NC, (int)sizeof(T), (int)sizeof(T), PD, compose, false,
                                   g.tau, 1);
                    pdssm_status rr = seq_set_smem((const void*)kern, ly.bytes);
                    if (rr) return rr;
                    kern<<<(unsigned)ctas, (unsigned)g.N + 32, ly.bytes, st>>>(sa);
                    return cuda_check(what);
                };
                auto kA = g.N == 128 ? seq::k_fwd_seq<T, NC, PD, false, false, 128, 1, kSeqcG128, false, 1>
                          : g.N == 64 ? seq::k_fwd_seq<T, NC, PD, false, false, 64, 1, kSeqcG64, false, 1>
                                      : seq::k_fwd_seq<T, NC, PD, false, false, 0, 1, kSeqcG128, false, 1>;
                auto kC = g.N == 128 ? seq::k_fwd_seq<T, NC, PD, false, false, 128, 1, kSeqcG128, false, 2>
                          : g.N == 64 ? seq::k_fwd_seq<T, NC, PD, false, false, 64, 1, kSeqcG64, false, 2>
                                      : seq::k_fwd_seq<T, NC, PD, false, false, 0, 1, kSeqcG128, false, 2>;
                pdssm_status rr = launch(kA, true, "fwd_seqc_A");
                if (rr || phaseA_only) return rr;   // (the sequence-parallel summary needs the aggregates only)
                k_fwd_phaseB<NC><<<(unsigned)g.S, thr, (size_t)NC * g.N * 4 + (size_t)g.N * 2 + 16, st>>>(
                    sa.cs, sa.h0, sa.maps, nullptr, (int)g.N, g.C);
                if ((rr = cuda_check("fwd_seqc_B"))) return rr;
                return launch(kC, false, "fwd_seqc_C");
            });
        });
    });
}

}  // namespace api
}  // namespace pdssm

PDSSM_DEFINE_ERRWORD(seq_fwd)
