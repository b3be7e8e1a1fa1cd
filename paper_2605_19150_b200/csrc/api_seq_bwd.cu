// libpdssm.so: single-chunk backward scan launcher (k_bwd_seq, csrc/k_scan_seq.cuh).
#include "api_internal.cuh"

using namespace pdssm;
using namespace pdssm::api;

namespace pdssm {
namespace api {

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

}  // namespace api
}  // namespace pdssm

PDSSM_DEFINE_ERRWORD(seq_bwd)
