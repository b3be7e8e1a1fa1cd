// libpdssm.so: NEXT-1 surrogate gradients (Prop. 2): pdssm_select_grad, pdssm_dict_grad.
#include "api_internal.cuh"
#include "k_surrogate.cuh"

using namespace pdssm;
using namespace pdssm::api;

PDSSM_DEFINE_ERRWORD(grad)

extern "C" {

// ---------------------------------------------------------------------------
// NEXT-1: Prop. 2 surrogate gradients (k_surrogate.cuh)
// ---------------------------------------------------------------------------
pdssm_status pdssm_select_grad(const float* logits, const uint8_t* kstar, const float* gsel, float temp,
                               float* dlogits, const pdssm_dims* dims, pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (!logits || !kstar || !gsel || !dlogits) return fail(PDSSM_ERR_NULL, "select_grad: logits, kstar, gsel, dlogits are required");
    if (!(temp > 0.f) || !std::isfinite(temp)) return fail(PDSSM_ERR_RANGE, "select_grad: temperature must be finite and > 0");
    if (misaligned(logits, 4) || misaligned(gsel, 4) || misaligned(dlogits, 4)) return fail(PDSSM_ERR_ALIGN, "select_grad: misaligned");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t rows = g.S * g.L;
    if (g.K <= 64 && !misaligned(logits, 16) && !misaligned(dlogits, 16)) {
        auto kr = g.K <= 32 ? sg::k_select_grad_row<32> : sg::k_select_grad_row<64>;
        kr<<<(unsigned)ceil_div(rows, 128), 128, 0, st>>>(logits, kstar, gsel, dlogits, rows, (int)g.K, 1.f / temp);
        return cuda_check("select_grad");
    }
    const int km = (int)ceil_div(g.K, 32);
    auto kern = km == 1 ? sg::k_select_grad<1> : km == 2 ? sg::k_select_grad<2> : km <= 4 ? sg::k_select_grad<4>
                                                                                        : sg::k_select_grad<8>;
    kern<<<(unsigned)ceil_div(rows, 8 * sg::SG_ROWS), 256, 0, st>>>(logits, kstar, gsel, dlogits, rows, (int)g.K, 1.f / temp);
    return cuda_check("select_grad");
}

pdssm_status pdssm_dict_grad(const float* M, const uint8_t* kstar, const void* diag, const void* h_saved,
                             const float* h0_opt, const void* dbias, float temp, float* dM, float* G_opt,
                             const pdssm_dims* dims, pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (!M || !kstar || !diag || !h_saved || !dbias || !dM)
        return fail(PDSSM_ERR_NULL, "dict_grad: M, kstar, diag, h_saved, dbias, dM are required");
    if (!(temp > 0.f) || !std::isfinite(temp)) return fail(PDSSM_ERR_RANGE, "dict_grad: temperature must be finite and > 0");
    if (g.N > 128) return fail(PDSSM_ERR_UNSUPPORTED, "dict_grad: state N must be <= 128 (got %lld)", (long long)g.N);
    if (g.S * g.L > ((int64_t)1 << 31) - 1) return fail(PDSSM_ERR_SHAPE, "dict_grad: B * L too large");
    const bool pd = g.diag_mode == PDSSM_DIAG_PER_DICT;
    if (misaligned(M, 4) || misaligned(dM, 4) || misaligned(G_opt, 4) || misaligned(h0_opt, 4) ||
        misaligned(diag, pd ? 4 : g.act) || misaligned(h_saved, g.act) || misaligned(dbias, g.act))
        return fail(PDSSM_ERR_ALIGN, "dict_grad: misaligned");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    sg::DictArgs a{};
    a.M = M;
    a.kstar = kstar;
    a.diag = pd ? nullptr : diag;
    a.diag_dict = pd ? static_cast<const float*>(diag) : nullptr;
    a.hsaved = h_saved;
    a.h0 = h0_opt;
    a.lam = dbias;
    a.dM = dM;
    a.G = G_opt;
    a.B = (int)g.B; a.H = (int)g.H; a.L = (int)g.L; a.N = (int)g.N; a.K = (int)g.K;
    a.invT = 1.f / temp;
    const unsigned grid = (unsigned)(g.H * g.K);
    const bool tc = g.N == sg::TC_N && !env_path_is("generic") && !misaligned(M, 16);   // (float4 M-tile loads)
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            return with_pd(g.diag_mode, [&](auto pdv) {
                constexpr bool PD = decltype(pdv)::value;
                if (tc) {
                    auto kern = sg::k_dict_grad_tc<T, NC, PD>;
                    const size_t bytes = sg::tc_smem_bytes();
                    pdssm_status rr = seq_set_smem((const void*)kern, bytes);
                    if (rr) return rr;
                    kern<<<grid, sg::TC_THREADS, bytes, st>>>(a);
                    return cuda_check("dict_grad_tc");
                }
                auto kern = sg::k_dict_grad_simt<T, NC, PD>;
                const size_t bytes = ((size_t)g.N * (g.N + 1) + (size_t)2 * 32 * NC * g.N) * 4 + (32 + 256 + 8) * 4;
                pdssm_status rr = seq_set_smem((const void*)kern, bytes);
                if (rr) return rr;
                kern<<<grid, 256, bytes, st>>>(a);
                return cuda_check("dict_grad_simt");
            });
        });
    });
}

}  // extern "C"
