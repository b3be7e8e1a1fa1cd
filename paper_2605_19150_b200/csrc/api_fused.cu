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

// shared memory (warp blocks + the head's tables) of the fused kernels for these dims
template <bool BWD>
size_t fused_smem(const Geo& g, int esz) {
    size_t r = 0;
    with_npl(fused_npl(g.N), [&](auto nv) {
        constexpr int NPL = decltype(nv)::value;
        return with_act(g.dtype, [&](auto tv) {
            using T = decltype(tv);
            return with_nc(g.nc, [&](auto ncv) {
                constexpr int NC = decltype(ncv)::value;
                return with_pd(g.diag_mode, [&](auto pdv) {
                    constexpr bool PD = decltype(pdv)::value;
                    if (esz == 4) {
                        using LY = fused::Layout<T, NC, NPL, PD, BWD, 4>;
                        r = LY::bytes + LY::t_bytes((int)g.K);
                    } else {
                        using LY = fused::Layout<T, NC, NPL, PD, BWD, (int)sizeof(T)>;
                        r = LY::bytes + LY::t_bytes((int)g.K);
                    }
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
    const size_t lim = 227 * 1024;
    if (fused_smem<false>(g, (int)g.act) > lim || fused_smem<true>(g, 4) > lim || fused_smem<true>(g, (int)g.act) > lim)
        return false;
    return true;
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
                    return launch_fused(fused::k_fwd_fused<T, NC, NPL, PD>, fa, WS::bytes + WS::t_bytes((int)g.K),
                                        WS::THREADS, g, st, "fwd_fused");
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
                    return launch_fused(fused::k_bwd_fused<T, TEE, NC, NPL, PD>, fa, WS::bytes + WS::t_bytes((int)g.K),
                                        WS::THREADS, g, st, "bwd_fused");
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
