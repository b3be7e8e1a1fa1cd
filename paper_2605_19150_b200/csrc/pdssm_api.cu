// C ABI of libpdssm.so (declarations and contracts: include/pdssm.h).
// Validation is synchronous and happens before any CUDA call; every kernel is
// enqueued on the caller's stream; nothing is allocated.
// This unit: dims/workspace queries, status, sparsify, the generic three-phase scan, the
// scan_fwd / scan_bwd dispatch, sequence-parallel summaries, layer_fwd.  The other units
// (api_seq_fwd.cu, api_seq_bwd.cu, api_fused.cu, api_gemm.cu, api_grad.cu) hold the
// launchers of the remaining kernel families.
#include "api_internal.cuh"
#include "k_scan_bwd.cuh"
#include "k_select.cuh"
#include "k_sp.cuh"

using namespace pdssm;
using namespace pdssm::api;

namespace {
thread_local std::string g_last_error;
}  // namespace

pdssm_status pdssm::api::fail(pdssm_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

PDSSM_DEFINE_ERRWORD(core)

namespace pdssm {
namespace api {

// ------------------------------------------------------------------ plan
pdssm_status launch_plan(const Geo& g, const uint16_t* dict_idx, uint16_t* pstart, uint16_t* psrc,
                         cudaStream_t st) {
    int thr = threads_for(g.N);
    if (thr > 1024) thr = 1024;
    k_build_plan<<<(unsigned)(g.H * g.K), thr, (size_t)g.N * 2, st>>>(dict_idx, pstart, psrc, (int)g.N, g.flags);
    return cuda_check("build_plan");
}

// ------------------------------------------------------------------ forward phases
pdssm_status fwd_three_phase(const Geo& g, const uint8_t* kstar, const uint16_t* dict_idx, const uint16_t* pstart,
                             const uint16_t* psrc, const void* diag, const void* bias, const float* h0,
                             ChunkStateView cs, uint16_t* maps, void* hout, bool phaseC, cudaStream_t st) {
    const int thr = threads_for(g.N);
    const unsigned items = (unsigned)(g.S * g.C);
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            return with_pd(g.diag_mode, [&](auto pdv) {
                constexpr bool PD = decltype(pdv)::value;
                const T* dg = PD ? nullptr : static_cast<const T*>(diag);
                const float* dd = PD ? static_cast<const float*>(diag) : nullptr;
                size_t smA = (size_t)4 * NC * g.N * 4;
                k_fwd_phaseA<T, NC, PD><<<items, thr, smA, st>>>(kstar, dict_idx, pstart, psrc, dg, dd,
                                                                 static_cast<const T*>(bias), cs, (int)g.H, (int)g.L,
                                                                 (int)g.N, (int)g.K, g.tau, g.C, g.flags);
                pdssm_status r = cuda_check("fwd_phaseA");
                if (r) return r;
                size_t smB = (size_t)NC * g.N * 4 + (size_t)g.N * 2 + 16;
                k_fwd_phaseB<NC><<<(unsigned)g.S, thr, smB, st>>>(cs, h0, maps, nullptr, (int)g.N, g.C);
                r = cuda_check("fwd_phaseB");
                if (r || !phaseC) return r;
                size_t smC = (size_t)2 * NC * g.N * 4;
                k_fwd_phaseC<T, NC, PD><<<items, thr, smC, st>>>(kstar, pstart, psrc, dg, dd,
                                                                 static_cast<const T*>(bias), cs,
                                                                 static_cast<T*>(hout), (int)g.H, (int)g.L,
                                                                 (int)g.N, (int)g.K, g.tau, g.C, g.flags);
                return cuda_check("fwd_phaseC");
            });
        });
    });
}

// PER_DICT dD_k: two-stage deterministic reduction of the per-step f32 dD_t (k_scan_bwd.cuh)
pdssm_status reduce_dict(const Geo& g, const uint8_t* kstar, const float* dDbuf, float* ddiag, float* part,
                         cudaStream_t st) {
    const int cN = g.nc * (int)g.N;
    const int64_t ns = ceil_div(g.L, RD_SLICE), ntile = ceil_div(cN, RD_COLS);
    const size_t sm = (size_t)g.K * RD_COLS * 4;
    pdssm_status r = set_smem((const void*)k_reduce_dict_partial, sm);
    if (r) return r;
    k_reduce_dict_partial<<<(unsigned)(g.S * ns * ntile), RD_COLS, sm, st>>>(kstar, dDbuf, part, (int)g.L, (int)g.K, cN);
    if ((r = cuda_check("reduce_dict_partial"))) return r;
    const int64_t n = g.H * g.K * cN;
    k_reduce_dict_final<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(part, ddiag, (int)g.B, (int)g.H, (int)g.L, (int)g.K, cN);
    return cuda_check("reduce_dict_final");
}

}  // namespace api
}  // namespace pdssm

extern "C" {

int32_t pdssm_default_chunk(const pdssm_dims* dims) {
    Geo g;
    if (geo_of(dims, &g)) return 0;
    return g.tau;
}

size_t pdssm_workspace_bytes(const pdssm_dims* dims, int op) {
    Geo g;
    if (geo_of(dims, &g)) return 0;
    return ws_bytes_g(g, op);
}

size_t pdssm_chunk_state_bytes(const pdssm_dims* dims) {
    Geo g;
    if (geo_of(dims, &g)) return 0;
    return chunk_state_bytes_g(g);
}

pdssm_status pdssm_chunk_state_offsets(const pdssm_dims* dims, size_t offsets[4]) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (!offsets) return fail(PDSSM_ERR_NULL, "offsets is NULL");
    offsets[0] = 0;
    offsets[1] = cs_pi_bytes(g);
    offsets[2] = cs_pi_bytes(g) + cs_f_bytes(g);
    offsets[3] = cs_pi_bytes(g) + 2 * cs_f_bytes(g);
    return PDSSM_OK;
}

size_t pdssm_summary_bytes(const pdssm_dims* dims) {
    Geo g;
    if (geo_of(dims, &g)) return 0;
    return summary_block_bytes(g);
}

const char* pdssm_status_string(pdssm_status s) {
    switch (s) {
        case PDSSM_OK: return "PDSSM_OK";
        case PDSSM_ERR_NULL: return "PDSSM_ERR_NULL";
        case PDSSM_ERR_SHAPE: return "PDSSM_ERR_SHAPE";
        case PDSSM_ERR_RANGE: return "PDSSM_ERR_RANGE";
        case PDSSM_ERR_ALIGN: return "PDSSM_ERR_ALIGN";
        case PDSSM_ERR_DTYPE: return "PDSSM_ERR_DTYPE";
        case PDSSM_ERR_WORKSPACE: return "PDSSM_ERR_WORKSPACE";
        case PDSSM_ERR_NONFINITE: return "PDSSM_ERR_NONFINITE";
        case PDSSM_ERR_CUDA: return "PDSSM_ERR_CUDA";
        case PDSSM_ERR_UNSUPPORTED: return "PDSSM_ERR_UNSUPPORTED";
    }
    return "PDSSM_UNKNOWN";
}

const char* pdssm_last_error(void) { return g_last_error.c_str(); }

const char* pdssm_version(void) { return "pdssm-b200 0.1 (sm_100a)"; }

pdssm_status pdssm_check_device(pdssm_stream_t stream) {
    cudaError_t e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "cudaStreamSynchronize: %s", cudaGetErrorString(e));
    uint32_t w = 0;
    cudaError_t (*readers[])(uint32_t*) = {errword_core, errword_seq_fwd, errword_seq_bwd, errword_fused, errword_gemm,
                                           errword_grad};
    for (auto rd : readers) {
        uint32_t wi = 0;
        e = rd(&wi);
        if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "read/clear error word: %s", cudaGetErrorString(e));
        w |= wi;
    }
    if (w & ERRBIT_NONFINITE) return fail(PDSSM_ERR_NONFINITE, "device reported NaN/Inf input");
    if (w & ERRBIT_RANGE) return fail(PDSSM_ERR_RANGE, "device reported an out-of-range index");
    return PDSSM_OK;
}

pdssm_status pdssm_sparsify(const float* M, uint16_t* dict_idx, const pdssm_dims* dims, pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (!M || !dict_idx) return fail(PDSSM_ERR_NULL, "sparsify: M and dict_idx are required");
    if (misaligned(M, 4) || misaligned(dict_idx, 2)) return fail(PDSSM_ERR_ALIGN, "sparsify: misaligned pointer");
    int thr = threads_for(g.N);
    if (thr > 1024) thr = 1024;
    k_sparsify<<<(unsigned)(g.H * g.K), thr, 0, reinterpret_cast<cudaStream_t>(stream)>>>(M, dict_idx, (int)g.N,
                                                                                          g.flags);
    return cuda_check("sparsify");
}


static pdssm_status common_scan_checks(const Geo& g, const void* kstar, const void* dict_idx, const void* diag) {
    if (!kstar || !dict_idx || !diag) return fail(PDSSM_ERR_NULL, "kstar, dict_idx and diag are required");
    if (misaligned(dict_idx, 2)) return fail(PDSSM_ERR_ALIGN, "dict_idx misaligned");
    if (misaligned(diag, g.diag_mode == PDSSM_DIAG_PER_DICT ? 4 : g.act)) return fail(PDSSM_ERR_ALIGN, "diag misaligned");
    return PDSSM_OK;
}

pdssm_status pdssm_scan_fwd(const uint8_t* kstar, const uint16_t* dict_idx, const void* diag, const void* bias,
                            const float* h0_opt, const float* C_opt, void* h_out_opt, void* y_opt, void* chunk_state,
                            uint16_t* maps_opt, const pdssm_dims* dims, void* ws, size_t ws_bytes,
                            pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if ((r = common_scan_checks(g, kstar, dict_idx, diag))) return r;
    if (!bias) return fail(PDSSM_ERR_NULL, "scan_fwd: bias is required");
    if (!chunk_state) return fail(PDSSM_ERR_WORKSPACE, "scan_fwd: chunk_state is required");
    if (!h_out_opt && !y_opt) return fail(PDSSM_ERR_NULL, "scan_fwd: need h_out_opt and/or y_opt");
    if (y_opt && (!C_opt || g.P < 1)) return fail(PDSSM_ERR_NULL, "scan_fwd: y_opt needs C_opt and p_out >= 1");
    if ((g.flags & PDSSM_EXPORT_MAPS) && !maps_opt) return fail(PDSSM_ERR_NULL, "scan_fwd: EXPORT_MAPS needs maps_opt");
    if (misaligned(bias, g.act) || misaligned(h_out_opt, g.act) || misaligned(y_opt, g.act) || misaligned(h0_opt, 4) ||
        misaligned(C_opt, 4) || misaligned(chunk_state, 16) || misaligned(maps_opt, 2))
        return fail(PDSSM_ERR_ALIGN, "scan_fwd: misaligned pointer");
    const size_t need = ws_bytes_g(g, PDSSM_OP_FWD);
    if (!ws || ws_bytes < need) return fail(PDSSM_ERR_WORKSPACE, "scan_fwd: workspace too small (need %zu)", need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Bump bump(ws);
    uint16_t* pstart = bump.take<uint16_t>((size_t)g.H * g.K * (g.N + 1) * 2);
    uint16_t* psrc = bump.take<uint16_t>((size_t)g.H * g.K * g.N * 2);
    void* hscratch = g.P > 0 ? bump.take<char>(seq_act_bytes(g)) : nullptr;
    void* wbuf = g.P > 0 ? bump.take<char>(readout_w_bytes(g)) : nullptr;
    uint8_t* frec = bump.take<uint8_t>(fused_rec_bytes(g.H, g.K));
    uint32_t* fhdr = bump.take<uint32_t>(fused_hdr_bytes(g.H, g.K));
    uint16_t* fpcl = bump.take<uint16_t>(fused_pclamp_bytes(g.H, g.K, g.N));
    uint32_t* ctrl = bump.take<uint32_t>(fused_ctrl_bytes(g.S, g.C, g.H));
    uint8_t* srec = bump.take<uint8_t>(seq_rec_bytes(g));
    uint8_t* swm = bump.take<uint8_t>(seq_wm_bytes(g));
    uint8_t* sovf = bump.take<uint8_t>(seq_ovf_bytes(g));
    void* hout = h_out_opt ? h_out_opt : hscratch;
    ChunkStateView cs = cs_view(g, chunk_state);
    uint16_t* maps = (g.flags & PDSSM_EXPORT_MAPS) ? maps_opt : nullptr;
    const bool use_seq = seq_applicable(g, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, bias, hout});
    // the single-CTA paths build their records and the CSR plan in one launch (fwd_seq / fwd_seqc)
    const bool seqc_fwd = !use_seq && seqc_applicable(g, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, bias, hout});
    if (!use_seq && !seqc_fwd && (r = launch_plan(g, dict_idx, pstart, psrc, st))) return r;
    if (env_path_is("seq") && !use_seq)
        return fail(PDSSM_ERR_UNSUPPORTED, "scan_fwd: PDSSM_PATH=seq but the single-chunk path does not apply");
    const bool use_seqc = !use_seq && seqc_applicable(g, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, bias, hout});
    const bool use_fused = !use_seq && !use_seqc && fused_applicable(
        g, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, bias, hout, h0_opt, chunk_state, maps});
    if (use_seqc) {
        seq::SeqArgs sa{};
        sa.kstar = kstar; sa.dict_idx = dict_idx; sa.rec = srec; sa.wm = swm; sa.ovf = sovf; sa.pstart = pstart;
        sa.psrc = psrc;
        sa.diag = g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr;
        sa.diag_dict = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<const float*>(diag) : nullptr;
        sa.bias = bias; sa.h0 = h0_opt; sa.cs = cs; sa.maps = maps; sa.out0 = hout;
        sa.H = (int)g.H; sa.L = (int)g.L; sa.N = (int)g.N; sa.K = (int)g.K; sa.flags = g.flags;
        if ((r = fwd_seqc(g, sa, srec, swm, sovf, st))) return r;
    } else if (use_seq) {
        seq::SeqArgs sa{};
        sa.kstar = kstar; sa.dict_idx = dict_idx; sa.rec = srec; sa.wm = swm; sa.ovf = sovf; sa.pstart = pstart;
        sa.psrc = psrc;
        sa.diag = g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr;
        sa.diag_dict = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<const float*>(diag) : nullptr;
        sa.bias = bias; sa.h0 = h0_opt; sa.cs = cs; sa.maps = maps; sa.out0 = hout;
        sa.H = (int)g.H; sa.L = (int)g.L; sa.N = (int)g.N; sa.K = (int)g.K; sa.flags = g.flags;
        if ((r = fwd_seq(g, sa, srec, swm, sovf, st))) return r;
    } else if (use_fused) {
        fused::FusedArgs fa{};
        fa.kstar = kstar; fa.dict_idx = dict_idx; fa.pstart = pstart; fa.psrc = psrc; fa.rec = frec; fa.hdr = fhdr;
        fa.pclamp = fpcl;
        fa.diag = g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr;
        fa.diag_dict = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<const float*>(diag) : nullptr;
        fa.bias = bias; fa.h0 = h0_opt; fa.cs = cs; fa.maps = maps; fa.out0 = hout; fa.ctrl = ctrl;
        fa.H = (int)g.H; fa.L = (int)g.L; fa.N = (int)g.N; fa.K = (int)g.K; fa.tau = g.tau; fa.C = g.C;
        fa.S = (int)g.S; fa.flags = g.flags;
        if ((r = fwd_fused(g, fa, frec, fhdr, st))) return r;
    } else if (path_fused_forced()) {
        return fail(PDSSM_ERR_UNSUPPORTED, "scan_fwd: PDSSM_PATH=fused but the fused path does not apply to these dims");
    } else {
        if ((r = fwd_three_phase(g, kstar, dict_idx, pstart, psrc, diag, bias, h0_opt, cs, maps, hout, true, st)))
            return r;
    }
    if (y_opt) r = readout_run(g, hout, C_opt, y_opt, wbuf, st);
    return r;
}

pdssm_status pdssm_scan_bwd(const uint8_t* kstar, const uint16_t* dict_idx, const void* diag, const void* h_saved,
                            const void* bias_opt, const float* h0_opt, const void* chunk_state, const void* dh_opt,
                            const void* dy_opt,
                            const float* C_opt, const float* lam_in_opt, void* dbias, void* ddiag, float* gsel,
                            float* dh0_opt, const pdssm_dims* dims, void* ws, size_t ws_bytes,
                            pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if ((r = common_scan_checks(g, kstar, dict_idx, diag))) return r;
    if (!h_saved && !bias_opt) return fail(PDSSM_ERR_NULL, "scan_bwd: h_saved (or bias_opt, recompute mode) is required");
    const bool recompute = h_saved == nullptr;   // replay the states from bias + chunk_state carries
    if (!chunk_state) return fail(PDSSM_ERR_WORKSPACE, "scan_bwd: chunk_state is required");
    if (!dbias || !ddiag) return fail(PDSSM_ERR_NULL, "scan_bwd: dbias and ddiag are required");
    if (dy_opt && (!C_opt || g.P < 1)) return fail(PDSSM_ERR_NULL, "scan_bwd: dy_opt needs C_opt and p_out >= 1");
    if (recompute && rc_smem_bytes(g.tau, g.nc, (int)g.N, threads_for(g.N)) > (size_t)(220 * 1024))
        return fail(PDSSM_ERR_UNSUPPORTED,
                    "scan_bwd: recompute mode keeps one chunk of states in shared memory: need chunk * c * N * 4 <= "
                    "~200 KB (chunk %d, c %d, N %lld); pass a smaller dims.chunk to both passes",
                    g.tau, g.nc, (long long)g.N);
    if (misaligned(h_saved, g.act) || misaligned(bias_opt, g.act) || misaligned(dh_opt, g.act) || misaligned(dy_opt, g.act) || misaligned(dbias, g.act) ||
        misaligned(ddiag, g.diag_mode == PDSSM_DIAG_PER_DICT ? 4 : g.act) || misaligned(gsel, 4) ||
        misaligned(dh0_opt, 4) || misaligned(h0_opt, 4) || misaligned(lam_in_opt, 4) || misaligned(C_opt, 4) ||
        misaligned(chunk_state, 16))
        return fail(PDSSM_ERR_ALIGN, "scan_bwd: misaligned pointer");
    const size_t need = ws_bytes_g(g, PDSSM_OP_BWD);
    if (!ws || ws_bytes < need) return fail(PDSSM_ERR_WORKSPACE, "scan_bwd: workspace too small (need %zu)", need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Bump bump(ws);
    float* betap = bump.take<float>(cs_f_bytes(g));
    float* mu = bump.take<float>(cs_f_bytes(g));
    float* ebuf = g.P > 0 ? bump.take<float>(seq_f_bytes(g)) : nullptr;
    void* wbuf = g.P > 0 ? bump.take<char>(readout_w_bytes(g)) : nullptr;
    float* dDbuf = g.diag_mode == PDSSM_DIAG_PER_DICT ? bump.take<float>(seq_f_bytes(g)) : nullptr;
    float* rdpart = g.diag_mode == PDSSM_DIAG_PER_DICT
                        ? bump.take<float>(reduce_dict_ws_bytes(g.S, g.L, g.K, g.nc * g.N)) : nullptr;
    uint32_t* ctrl = bump.take<uint32_t>(fused_ctrl_bytes(g.S, g.C, g.H));
    uint16_t* pstart = bump.take<uint16_t>((size_t)g.H * g.K * (g.N + 1) * 2);   // recompute: forward plan
    uint16_t* psrc = bump.take<uint16_t>((size_t)g.H * g.K * g.N * 2);
    uint8_t* srec = bump.take<uint8_t>(seq_rec_bytes(g));   // recompute (one CTA per sequence): gather records
    uint8_t* swm = bump.take<uint8_t>(seq_wm_bytes(g));
    uint8_t* sovf = bump.take<uint8_t>(seq_ovf_bytes(g));
    ChunkStateView cs = cs_view(g, const_cast<void*>(chunk_state));
    const int thr = threads_for(g.N);
    const unsigned items = (unsigned)(g.S * g.C);
    if (recompute && bwd_seq_rc_applicable(g, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, bias_opt, dh_opt,
                                                ebuf, dbias, g.diag_mode == PDSSM_DIAG_PER_STEP ? ddiag : nullptr})) {
        if (dy_opt && (r = prepare_e_run(g, dh_opt, dy_opt, C_opt, ebuf, wbuf, st))) return r;
        seq::RcArgs ra{};
        ra.kstar = kstar; ra.dict_idx = dict_idx; ra.pstart = pstart; ra.psrc = psrc;
        ra.diag = g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr;
        ra.diag_dict = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<const float*>(diag) : nullptr;
        ra.bias = bias_opt; ra.e = dy_opt ? static_cast<const void*>(ebuf) : dh_opt; ra.lam_in = lam_in_opt; ra.cs = cs;
        ra.dbias = dbias; ra.ddiag = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<void*>(dDbuf) : ddiag;
        ra.gsel = gsel; ra.dh0 = dh0_opt;
        ra.H = (int)g.H; ra.L = (int)g.L; ra.N = (int)g.N; ra.K = (int)g.K; ra.tau = g.tau; ra.C = g.C; ra.flags = g.flags;
        if ((r = bwd_seq_rc_run(g, ra, dy_opt != nullptr, srec, swm, sovf, st))) return r;
        if (g.diag_mode == PDSSM_DIAG_PER_DICT)
            return reduce_dict(g, kstar, dDbuf, static_cast<float*>(ddiag), rdpart, st);
        return PDSSM_OK;
    }
    const bool use_seq = !recompute && seq_applicable(g, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, h_saved, dh_opt, ebuf});
    const bool use_seqc = !recompute && !use_seq &&
        seqc_applicable(g, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, h_saved, dh_opt, ebuf, dbias,
                            g.diag_mode == PDSSM_DIAG_PER_STEP ? ddiag : nullptr});
    if (use_seqc) {
        if (dy_opt && (r = prepare_e_run(g, dh_opt, dy_opt, C_opt, ebuf, wbuf, st))) return r;
        seq::SeqArgs sa{};
        sa.kstar = kstar; sa.dict_idx = dict_idx;
        sa.diag = g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr;
        sa.diag_dict = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<const float*>(diag) : nullptr;
        sa.bias = dy_opt ? static_cast<const void*>(ebuf) : dh_opt;
        sa.hsaved = h_saved; sa.h0 = h0_opt; sa.lam_in = lam_in_opt; sa.cs = cs;
        sa.out0 = dbias; sa.out1 = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<void*>(dDbuf) : ddiag;
        sa.gsel = gsel; sa.dh0 = dh0_opt; sa.mu = mu; sa.betap = betap;
        sa.H = (int)g.H; sa.L = (int)g.L; sa.N = (int)g.N; sa.K = (int)g.K; sa.flags = g.flags;
        if ((r = bwd_seqc_run(g, sa, dy_opt != nullptr, st))) return r;
        if (g.diag_mode == PDSSM_DIAG_PER_DICT)
            return reduce_dict(g, kstar, dDbuf, static_cast<float*>(ddiag), rdpart, st);
        return PDSSM_OK;
    }
    if (env_path_is("seq") && !use_seq)
        return fail(PDSSM_ERR_UNSUPPORTED, "scan_bwd: PDSSM_PATH=seq but the single-chunk path does not apply");
    const bool use_fused = !use_seq && !recompute &&
        fused_applicable(g, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, h_saved, dh_opt, h0_opt, lam_in_opt,
                             dbias, g.diag_mode == PDSSM_DIAG_PER_STEP ? ddiag : nullptr, dh0_opt, chunk_state});
    if (!use_fused && !use_seq && !recompute && path_fused_forced())
        return fail(PDSSM_ERR_UNSUPPORTED, "scan_bwd: PDSSM_PATH=fused but the fused path does not apply to these dims");
    if (use_seq) {
        if (dy_opt && (r = prepare_e_run(g, dh_opt, dy_opt, C_opt, ebuf, wbuf, st))) return r;
        seq::SeqArgs sa{};
        sa.kstar = kstar; sa.dict_idx = dict_idx;
        sa.diag = g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr;
        sa.diag_dict = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<const float*>(diag) : nullptr;
        sa.bias = dy_opt ? static_cast<const void*>(ebuf) : dh_opt;
        sa.hsaved = h_saved; sa.h0 = h0_opt; sa.lam_in = lam_in_opt; sa.cs = cs;
        sa.out0 = dbias; sa.out1 = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<void*>(dDbuf) : ddiag;
        sa.gsel = gsel; sa.dh0 = dh0_opt;
        sa.H = (int)g.H; sa.L = (int)g.L; sa.N = (int)g.N; sa.K = (int)g.K; sa.flags = g.flags;
        r = bwd_seq_run(g, sa, dy_opt != nullptr, st);
        if (r) return r;
        if (g.diag_mode == PDSSM_DIAG_PER_DICT) {
            r = with_nc(g.nc, [&](auto ncv) {
                constexpr int NC = decltype(ncv)::value;
                return reduce_dict(g, kstar, dDbuf, static_cast<float*>(ddiag), rdpart, st);
            });
        }
        return r;
    }
    if (use_fused) {
        if (dy_opt && (r = prepare_e_run(g, dh_opt, dy_opt, C_opt, ebuf, wbuf, st))) return r;
        fused::FusedArgs fa{};
        fa.kstar = kstar; fa.dict_idx = dict_idx;
        fa.diag = g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr;
        fa.diag_dict = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<const float*>(diag) : nullptr;
        fa.bias = dy_opt ? static_cast<const void*>(ebuf) : dh_opt;
        fa.hsaved = h_saved; fa.h0 = h0_opt; fa.lam_in = lam_in_opt; fa.cs = cs;
        fa.out0 = dbias; fa.out1 = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<void*>(dDbuf) : ddiag;
        fa.gsel = gsel; fa.dh0 = dh0_opt; fa.mu = mu; fa.betap = betap; fa.ctrl = ctrl;
        fa.H = (int)g.H; fa.L = (int)g.L; fa.N = (int)g.N; fa.K = (int)g.K; fa.tau = g.tau; fa.C = g.C;
        fa.S = (int)g.S; fa.flags = g.flags;
        r = bwd_fused_run(g, fa, dy_opt != nullptr, st);
        if (r) return r;
        if (g.diag_mode == PDSSM_DIAG_PER_DICT) {
            r = with_nc(g.nc, [&](auto ncv) {
                constexpr int NC = decltype(ncv)::value;
                return reduce_dict(g, kstar, dDbuf, static_cast<float*>(ddiag), rdpart, st);
            });
        }
        return r;
    }
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            return with_pd(g.diag_mode, [&](auto pdv) -> pdssm_status {
                constexpr bool PD = decltype(pdv)::value;
                const T* dg = PD ? nullptr : static_cast<const T*>(diag);
                const float* dd = PD ? static_cast<const float*>(diag) : nullptr;
                auto run = [&](auto ev) -> pdssm_status {
                    using TE = decltype(ev);
                    const TE* e = nullptr;
                    if (std::is_same<TE, float>::value && dy_opt) e = reinterpret_cast<const TE*>(ebuf);
                    else if (dh_opt) e = reinterpret_cast<const TE*>(dh_opt);
                    size_t smA = (size_t)2 * NC * g.N * 4;
                    k_bwd_phaseA<T, TE, NC, PD><<<items, thr, smA, st>>>(kstar, dict_idx, dg, dd, e, betap, (int)g.H,
                                                                         (int)g.L, (int)g.N, (int)g.K, g.tau, g.C);
                    pdssm_status rr = cuda_check("bwd_phaseA");
                    if (rr) return rr;
                    // dh0 comes from the chunk-0 replay (Phase C'), not from Abar_0
                    k_bwd_phaseB<NC><<<(unsigned)g.S, thr, (size_t)NC * g.N * 4, st>>>(cs, betap, lam_in_opt, mu,
                                                                                         nullptr, (int)g.N, g.C);
                    if ((rr = cuda_check("bwd_phaseB"))) return rr;
                    const int nw = thr / 32;
                    if (recompute) {
                        if ((rr = launch_plan(g, dict_idx, pstart, psrc, st))) return rr;
                        const size_t smR = rc_smem_bytes(g.tau, NC, (int)g.N, thr);
                        if ((rr = set_smem((const void*)k_bwd_phaseC_rc<T, TE, NC, PD>, smR))) return rr;
                        k_bwd_phaseC_rc<T, TE, NC, PD><<<items, thr, smR, st>>>(
                            kstar, dict_idx, pstart, psrc, dg, dd, static_cast<const T*>(bias_opt), cs, e, mu,
                            static_cast<T*>(dbias), PD ? nullptr : static_cast<T*>(ddiag), dDbuf, gsel, dh0_opt,
                            (int)g.H, (int)g.L, (int)g.N, (int)g.K, g.tau, g.C);
                        if ((rr = cuda_check("bwd_phaseC_rc"))) return rr;
                        if (PD) {
                            if ((rr = reduce_dict(g, kstar, dDbuf, static_cast<float*>(ddiag), rdpart, st))) return rr;
                        }
                        return PDSSM_OK;
                    }
                    size_t smC = (size_t)2 * NC * g.N * 4 + (size_t)64 * nw * 4;
                    if ((rr = set_smem((const void*)k_bwd_phaseC<T, TE, NC, PD>, smC))) return rr;
                    k_bwd_phaseC<T, TE, NC, PD><<<items, thr, smC, st>>>(
                        kstar, dict_idx, dg, dd, static_cast<const T*>(h_saved), h0_opt, e, mu, static_cast<T*>(dbias),
                        PD ? nullptr : static_cast<T*>(ddiag), dDbuf, gsel, dh0_opt, (int)g.H, (int)g.L, (int)g.N,
                        (int)g.K, g.tau, g.C);
                    if ((rr = cuda_check("bwd_phaseC"))) return rr;
                    if (PD) {
                        if ((rr = reduce_dict(g, kstar, dDbuf, static_cast<float*>(ddiag), rdpart, st))) return rr;
                    }
                    return PDSSM_OK;
                };
                if (dy_opt) {
                    pdssm_status rr = prepare_e_run(g, dh_opt, dy_opt, C_opt, ebuf, wbuf, st);
                    if (rr) return rr;
                    return run(float{});
                }
                return run(T{});
            });
        });
    });
}

pdssm_status pdssm_segment_summary(const uint8_t* kstar, const uint16_t* dict_idx, const void* diag,
                                   const void* bias, void* summary_out, const pdssm_dims* dims, void* ws,
                                   size_t ws_bytes, pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if ((r = common_scan_checks(g, kstar, dict_idx, diag))) return r;
    if (!bias || !summary_out) return fail(PDSSM_ERR_NULL, "segment_summary: bias and summary_out are required");
    if (misaligned(bias, g.act) || misaligned(summary_out, 16)) return fail(PDSSM_ERR_ALIGN, "segment_summary: misaligned");
    const size_t need = ws_bytes_g(g, PDSSM_OP_SEGMENT);
    if (!ws || ws_bytes < need) return fail(PDSSM_ERR_WORKSPACE, "segment_summary: workspace too small (need %zu)", need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Bump bump(ws);
    uint16_t* pstart = bump.take<uint16_t>((size_t)g.H * g.K * (g.N + 1) * 2);
    uint16_t* psrc = bump.take<uint16_t>((size_t)g.H * g.K * g.N * 2);
    void* csmem = bump.take<char>(chunk_state_bytes_g(g));
    uint8_t* srec = bump.take<uint8_t>(seq_rec_bytes(g));
    uint8_t* swm = bump.take<uint8_t>(seq_wm_bytes(g));
    uint8_t* sovf = bump.take<uint8_t>(seq_ovf_bytes(g));
    // The summary is the fold of chunk aggregates, whatever the chunking (Alg. 1's composition is
    // associative): chunks shorter than 128 steps are merged to 128 here so that the
    // chunked single-CTA kernel takes them (fewer chunks: the caller's chunk_state-sized workspace fits)
    Geo gs = g;
    if (gs.tau < 128 && gs.L > gs.tau) {
        gs.tau = (int)std::min<int64_t>(128, gs.L);
        gs.C = (int)ceil_div(gs.L, gs.tau);
    }
    if (!seqc_phaseA_ok(gs, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, bias})) gs = g;
    ChunkStateView cs = cs_view(gs, csmem);
    if (seqc_phaseA_ok(gs, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, bias})) {
        // the chunk aggregates by the chunked single-CTA kernel (Phase A only; its plan launch also
        // writes the CSR lists): one read of the segment at the single-chunk kernels' step rate
        seq::SeqArgs sa{};
        sa.kstar = kstar; sa.dict_idx = dict_idx; sa.rec = srec; sa.wm = swm; sa.ovf = sovf; sa.pstart = pstart;
        sa.psrc = psrc;
        sa.diag = g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr;
        sa.diag_dict = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<const float*>(diag) : nullptr;
        sa.bias = bias; sa.h0 = nullptr; sa.cs = cs; sa.maps = nullptr; sa.out0 = nullptr;
        sa.H = (int)g.H; sa.L = (int)g.L; sa.N = (int)g.N; sa.K = (int)g.K; sa.flags = g.flags;
        if ((r = fwd_seqc(gs, sa, srec, swm, sovf, st, true))) return r;
    } else {
        if ((r = launch_plan(g, dict_idx, pstart, psrc, st))) return r;
        if ((r = fwd_three_phase(g, kstar, dict_idx, pstart, psrc, diag, bias, nullptr, cs, nullptr, nullptr, false, st)))
            return r;
    }
    SummaryView sv{static_cast<char*>(summary_out), summary_block_bytes(g), npad8(g.N)};
    return with_nc(g.nc, [&](auto ncv) {
        constexpr int NC = decltype(ncv)::value;
        k_fold_aggregates<NC><<<(unsigned)g.S, threads_for(g.N), (size_t)NC * g.N * 4 + g.N * 2 + 16, st>>>(
            cs, sv, (int)g.N, gs.C);
        return cuda_check("fold_aggregates");
    });
}

pdssm_status pdssm_compose_carry(const void* summaries, int32_t rank, int32_t G, const float* h0_opt, float* carry_out,
                                 uint16_t* map_out_opt, const pdssm_dims* dims, pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (!summaries || !carry_out) return fail(PDSSM_ERR_NULL, "compose_carry: summaries and carry_out are required");
    if (G < 1 || rank < 0 || rank >= G) return fail(PDSSM_ERR_SHAPE, "compose_carry: need 0 <= rank < G");
    if (misaligned(summaries, 16) || misaligned(carry_out, 4) || misaligned(h0_opt, 4) || misaligned(map_out_opt, 2))
        return fail(PDSSM_ERR_ALIGN, "compose_carry: misaligned");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    SummaryView sv{static_cast<char*>(const_cast<void*>(summaries)), summary_block_bytes(g), npad8(g.N)};
    return with_nc(g.nc, [&](auto ncv) {
        constexpr int NC = decltype(ncv)::value;
        k_compose_carry<NC><<<(unsigned)g.S, threads_for(g.N), (size_t)NC * g.N * 4 + g.N * 2 + 16, st>>>(
            sv, rank, (int)g.S, h0_opt, carry_out, map_out_opt, (int)g.N);
        return cuda_check("compose_carry");
    });
}

pdssm_status pdssm_segment_summary_bwd(const uint8_t* kstar, const uint16_t* dict_idx, const void* diag,
                                       const void* chunk_state, const void* dh_opt, const void* dy_opt,
                                       const float* C_opt, float* beta_out, const pdssm_dims* dims, void* ws,
                                       size_t ws_bytes, pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if ((r = common_scan_checks(g, kstar, dict_idx, diag))) return r;
    if (!chunk_state || !beta_out) return fail(PDSSM_ERR_NULL, "segment_summary_bwd: chunk_state and beta_out required");
    if (dy_opt && (!C_opt || g.P < 1)) return fail(PDSSM_ERR_NULL, "segment_summary_bwd: dy_opt needs C_opt");
    if (misaligned(dh_opt, g.act) || misaligned(dy_opt, g.act) || misaligned(beta_out, 4) || misaligned(chunk_state, 16))
        return fail(PDSSM_ERR_ALIGN, "segment_summary_bwd: misaligned");
    const size_t need = ws_bytes_g(g, PDSSM_OP_SEGMENT);
    if (!ws || ws_bytes < need) return fail(PDSSM_ERR_WORKSPACE, "segment_summary_bwd: workspace too small (need %zu)", need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Bump bump(ws);
    float* betap = bump.take<float>(cs_f_bytes(g));
    float* mu = bump.take<float>(cs_f_bytes(g));
    float* ebuf = g.P > 0 ? bump.take<float>(seq_f_bytes(g)) : nullptr;
    void* wbuf = g.P > 0 ? bump.take<char>(readout_w_bytes(g)) : nullptr;
    ChunkStateView cs = cs_view(g, const_cast<void*>(chunk_state));
    const int thr = threads_for(g.N);
    const unsigned items = (unsigned)(g.S * g.C);
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            return with_pd(g.diag_mode, [&](auto pdv) -> pdssm_status {
                constexpr bool PD = decltype(pdv)::value;
                const T* dg = PD ? nullptr : static_cast<const T*>(diag);
                const float* dd = PD ? static_cast<const float*>(diag) : nullptr;
                auto run = [&](auto ev) -> pdssm_status {
                    using TE = decltype(ev);
                    const TE* e = nullptr;
                    if (std::is_same<TE, float>::value && dy_opt) e = reinterpret_cast<const TE*>(ebuf);
                    else if (dh_opt) e = reinterpret_cast<const TE*>(dh_opt);
                    pdssm_status rr;
                    if (seqc_phaseA_bwd_ok(g, sizeof(TE), {dg, e})) {
                        // beta'_c of every chunk by the chunked single-CTA kernel (Phase A' only)
                        seq::SeqArgs sa{};
                        sa.kstar = kstar; sa.dict_idx = dict_idx; sa.diag = dg; sa.diag_dict = dd; sa.bias = e;
                        sa.cs = cs; sa.betap = betap; sa.mu = mu;
                        sa.H = (int)g.H; sa.L = (int)g.L; sa.N = (int)g.N; sa.K = (int)g.K; sa.flags = g.flags;
                        rr = bwd_seqc_run(g, sa, std::is_same<TE, float>::value && !std::is_same<T, float>::value, st, true);
                    } else {
                        k_bwd_phaseA<T, TE, NC, PD><<<items, thr, (size_t)2 * NC * g.N * 4, st>>>(
                            kstar, dict_idx, dg, dd, e, betap, (int)g.H, (int)g.L, (int)g.N, (int)g.K, g.tau, g.C);
                        rr = cuda_check("bwd_phaseA");
                    }
                    if (rr) return rr;
                    k_bwd_phaseB<NC><<<(unsigned)g.S, thr, (size_t)NC * g.N * 4, st>>>(cs, betap, nullptr, mu,
                                                                                         beta_out, (int)g.N, g.C);
                    return cuda_check("bwd_phaseB");
                };
                if (dy_opt) {
                    pdssm_status rr = prepare_e_run(g, dh_opt, dy_opt, C_opt, ebuf, wbuf, st);
                    if (rr) return rr;
                    return run(float{});
                }
                return run(T{});
            });
        });
    });
}

pdssm_status pdssm_compose_lambda(const void* fwd_summaries, const float* beta_bwd, int32_t rank, int32_t G,
                                  float* lam_out, const pdssm_dims* dims, pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (!fwd_summaries || !beta_bwd || !lam_out) return fail(PDSSM_ERR_NULL, "compose_lambda: null argument");
    if (G < 1 || rank < 0 || rank >= G) return fail(PDSSM_ERR_SHAPE, "compose_lambda: need 0 <= rank < G");
    if (misaligned(fwd_summaries, 16) || misaligned(beta_bwd, 4) || misaligned(lam_out, 4))
        return fail(PDSSM_ERR_ALIGN, "compose_lambda: misaligned");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    SummaryView sv{static_cast<char*>(const_cast<void*>(fwd_summaries)), summary_block_bytes(g), npad8(g.N)};
    return with_nc(g.nc, [&](auto ncv) {
        constexpr int NC = decltype(ncv)::value;
        k_compose_lambda<NC><<<(unsigned)g.S, threads_for(g.N), (size_t)NC * g.N * 4, st>>>(sv, beta_bwd, rank, G,
                                                                                           (int)g.S, lam_out, (int)g.N);
        return cuda_check("compose_lambda");
    });
}

}  // extern "C"
