// libpdssm.so: chunked warp-per-item scan launchers (k_fwd_fused / k_bwd_fused, csrc/k_scan_fused.cuh).
#include "api_internal.cuh"

using namespace pdssm;
using namespace pdssm::api;

namespace pdssm {
namespace api {

template <typename F>
pdssm_status with_npl(int npl, F&& f) {
    if (npl == 1) return f(std::integral_constant<int, 1>{});
    if (npl == 2) return f(std::integral_constant<int, 2>{});
    return f(std::integral_constant<int, 4>{});
}

// Warps (items in flight) per CTA of a fused-kernel layout: as many as the shared memory holds
// beside the head's tables, up to fused::WARPS_MAX (0: not even FUSED_MIN_WARPS fit).  More warps
// hide more of the per-step latency (15 vs the fixed 11 of round 1: config 3 +10%, config 5 +6%).
constexpr int FUSED_MIN_WARPS = 4;
// Complex fp32 layouts stay at the round-1 count (11): more items in flight measured slower there
// (config 2 at tau 64: 0.41 vs 0.34 ms forward -- the chunk replay's L2 reuse suffers).
template <class LY>
int fused_warps_of(int64_t K) {
    const size_t lim = 227 * 1024, tb = LY::t_bytes((int)K);
    if (tb >= lim) return 0;
    const int cap = LY::ROW >= 2 * 128 * 4 ? fused::WARPS_FWD : fused::WARPS_MAX;
    const int w = (int)std::min<size_t>((lim - tb) / LY::w_bytes, (size_t)cap);
    return w >= FUSED_MIN_WARPS ? w : 0;
}

template <bool BWD>
int fused_warps(const Geo& g, int esz) {
    int r = 0;
    with_npl(fused_npl(g.N), [&](auto nv) {
        constexpr int NPL = decltype(nv)::value;
        return with_act(g.dtype, [&](auto tv) {
            using T = decltype(tv);
            return with_nc(g.nc, [&](auto ncv) {
                constexpr int NC = decltype(ncv)::value;
                return with_pd(g.diag_mode, [&](auto pdv) {
                    constexpr bool PD = decltype(pdv)::value;
                    if (esz == 4) r = fused_warps_of<fused::Layout<T, NC, NPL, PD, BWD, 4>>(g.K);
                    else r = fused_warps_of<fused::Layout<T, NC, NPL, PD, BWD, (int)sizeof(T)>>(g.K);
                    return PDSSM_OK;
                });
            });
        });
    });
    return r;
}

bool fused_applicable(const Geo& g, std::initializer_list<const void*> ptrs) {
    if (path_generic_forced() || fused_npl(g.N) == 0 || g.tau > fused::TAUMAX) return false;
    for (const void* p : ptrs)
        if (misaligned(p, 16)) return false;
    return fused_warps<false>(g, (int)g.act) > 0 && fused_warps<true>(g, 4) > 0 && fused_warps<true>(g, (int)g.act) > 0;
}


template <typename K>
pdssm_status launch_fused(K kernel, const fused::FusedArgs& fa_in, size_t smem, int threads, const Geo& g,
                          cudaStream_t st, const char* what) {
    fused::FusedArgs fa = fa_in;
    fa.smem_tables = 1;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "%s attribute: %s", what, cudaGetErrorString(e));
    // timing experiments only: bit 0 skips the carry wait, bit 1 skips the TMA ring (results invalid)
    fa.debug_nochain = getenv("PDSSM_DEBUG_NOCHAIN") ? atoi(getenv("PDSSM_DEBUG_NOCHAIN")) : 0;
    kernel<<<fused_grid(g.H), threads, smem, st>>>(fa);
    return cuda_check(what);
}

pdssm_status fwd_fused(const Geo& g, fused::FusedArgs& fa, uint8_t* rec, uint32_t* hdr, cudaStream_t st) {
    const int npl = fused_npl(g.N);
    return with_npl(npl, [&](auto nv) {
        constexpr int NPL = decltype(nv)::value;
        fused::k_build_fused_plan<NPL><<<(unsigned)(g.H * g.K), threads_for(g.N), (size_t)g.N * 4, st>>>(
            fa.dict_idx, rec, hdr, const_cast<uint16_t*>(fa.pclamp), (int)g.N, g.nc == 2 ? 8 : 4, g.flags);
        pdssm_status r = cuda_check("build_fused_plan");
        if (r) return r;
        cudaError_t e = cudaMemsetAsync(fa.ctrl, 0, fused_ctrl_bytes(g.S, g.C, g.H), st);
        if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "memset ctrl: %s", cudaGetErrorString(e));
        return with_act(g.dtype, [&](auto tv) {
            using T = decltype(tv);
            return with_nc(g.nc, [&](auto ncv) {
                constexpr int NC = decltype(ncv)::value;
                return with_pd(g.diag_mode, [&](auto pdv) {
                    constexpr bool PD = decltype(pdv)::value;
                    using WS = fused::Layout<T, NC, NPL, PD, false>;
                    const int nw = fused_warps_of<WS>(g.K);
                    return launch_fused(fused::k_fwd_fused<T, NC, NPL, PD>, fa, nw * WS::w_bytes + WS::t_bytes((int)g.K),
                                        nw * 32, g, st, "fwd_fused");
                });
            });
        });
    });
}

template <typename TE>
pdssm_status bwd_fused(const Geo& g, fused::FusedArgs& fa, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(fa.ctrl, 0, fused_ctrl_bytes(g.S, g.C, g.H), st);
    if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "memset ctrl: %s", cudaGetErrorString(e));
    return with_npl(fused_npl(g.N), [&](auto nv) {
        constexpr int NPL = decltype(nv)::value;
        return with_act(g.dtype, [&](auto tv) {
            using T = decltype(tv);
            return with_nc(g.nc, [&](auto ncv) {
                constexpr int NC = decltype(ncv)::value;
                return with_pd(g.diag_mode, [&](auto pdv) {
                    constexpr bool PD = decltype(pdv)::value;
                    using TEE = typename std::conditional<std::is_same<TE, void>::value, T, TE>::type;
                    using WS = fused::Layout<T, NC, NPL, PD, true, (int)sizeof(TEE)>;
                    const int nw = fused_warps_of<WS>(g.K);
                    return launch_fused(fused::k_bwd_fused<T, TEE, NC, NPL, PD>, fa, nw * WS::w_bytes + WS::t_bytes((int)g.K),
                                        nw * 32, g, st, "bwd_fused");
                });
            });
        });
    });
}

pdssm_status bwd_fused_run(const Geo& g, fused::FusedArgs& fa, bool e_f32, cudaStream_t st) {
    return e_f32 ? bwd_fused<float>(g, fa, st) : bwd_fused<void>(g, fa, st);
}

}  // namespace api
}  // namespace pdssm

PDSSM_DEFINE_ERRWORD(fused)
