// C ABI of libpdssm.so (declarations and contracts: include/pdssm.h).
// Validation is synchronous and happens before any CUDA call; every kernel is
// enqueued on the caller's stream; nothing is allocated.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <utility>

#include "pdssm_common.cuh"
#include "k_scan_fwd.cuh"
#include "k_scan_bwd.cuh"
#include "k_select.cuh"
#include "k_sp.cuh"
#include "k_scan_fused.cuh"
#include "k_gemm_tc.cuh"
#include "k_scan_seq.cuh"
#include "k_surrogate.cuh"

#include <mutex>


using namespace pdssm;

namespace {

thread_local std::string g_last_error;

pdssm_status fail(pdssm_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

struct Geo {
    int64_t B, H, L, N, K, S, d_in, P;
    int tau, C, nc, dtype, diag_mode;
    uint32_t flags;
    size_t act;   // bytes per act element
};

constexpr uint32_t kKnownFlags = PDSSM_CHECK_FINITE | PDSSM_DETERMINISTIC | PDSSM_EXPORT_MAPS;

// single-chunk (tau = L) scan kernels: one CTA of N threads per sequence
bool seq_shape_ok(int64_t N, int64_t K, int64_t L, int nc, size_t act) {
    (void)nc; (void)act;
    return N % 32 == 0 && N <= seq::MAXN && (size_t)K * N * 8 <= 64 * 1024 && L <= seq::LMAX;
}
int num_sms_dev() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    return sms;
}
bool env_path_is(const char* v) {
    const char* p = getenv("PDSSM_PATH");
    return p && strcmp(p, v) == 0;
}

// Library default chunk length (reading R20: tuning only).  When the B*H sequences
// alone fill most of the SMs, one chunk per sequence (tau = L) runs the single-pass
// CTA-per-sequence kernels; otherwise tau = 64 (chunked, decoupled look-back).
int default_tau(const pdssm_dims* d) {
    const int64_t S = d->batch * d->heads;
    const bool forced_chunked = env_path_is("fused") || env_path_is("generic");
    if (!forced_chunked && seq_shape_ok(d->state, d->dict, d->len, d->is_complex, d->dtype == PDSSM_BF16 ? 2 : 4) &&
        (env_path_is("seq") || S * 10 >= (int64_t)num_sms_dev() * 6) && d->len <= (int64_t)1 << 30)
        return (int)d->len;
    return 64;
}

pdssm_status geo_of(const pdssm_dims* d, Geo* g) {
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

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

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

size_t plan_bytes(const Geo& g) {
    return align256((size_t)g.H * g.K * (g.N + 1) * 2) + align256((size_t)g.H * g.K * g.N * 2);
}
size_t cs_pi_bytes(const Geo& g) { return align256((size_t)g.S * g.C * g.N * 2); }
size_t cs_f_bytes(const Geo& g) { return align256((size_t)g.S * g.C * g.nc * g.N * 4); }
size_t chunk_state_bytes_g(const Geo& g) { return cs_pi_bytes(g) + 3 * cs_f_bytes(g); }
size_t seq_f_bytes(const Geo& g) { return align256((size_t)g.S * g.L * g.nc * g.N * 4); }
// single-chunk plan: preimage records [H][K][N][8], warp trip counts, overflow flags
size_t seq_rec_bytes(const Geo& g) { return align256((size_t)g.H * g.K * g.N * 8); }
size_t seq_wm_bytes(const Geo& g) { return align256((size_t)g.H * g.K * (g.N / 32 > 0 ? g.N / 32 : 1)); }
size_t seq_ovf_bytes(const Geo& g) { return align256((size_t)g.H * g.K); }
size_t seq_plan_bytes(const Geo& g) { return seq_rec_bytes(g) + seq_wm_bytes(g) + seq_ovf_bytes(g); }
// readout weights staged in act dtype (Cp or CT), H*P*c*N elements
size_t readout_w_bytes(const Geo& g) { return g.P > 0 ? align256((size_t)g.H * g.P * g.nc * g.N * g.act) : 0; }
size_t seq_act_bytes(const Geo& g) { return align256((size_t)g.S * g.L * g.nc * g.N * g.act); }
int npad8(int64_t N) { return (int)((N + 7) & ~7); }
size_t summary_block_bytes(const Geo& g) { return (size_t)npad8(g.N) * 2 + (size_t)2 * g.nc * g.N * 4; }

ChunkStateView cs_view(const Geo& g, void* p) {
    char* b = static_cast<char*>(p);
    ChunkStateView v;
    v.pi = reinterpret_cast<uint16_t*>(b);
    v.d = reinterpret_cast<float*>(b + cs_pi_bytes(g));
    v.beta = reinterpret_cast<float*>(b + cs_pi_bytes(g) + cs_f_bytes(g));
    v.carry = reinterpret_cast<float*>(b + cs_pi_bytes(g) + 2 * cs_f_bytes(g));
    return v;
}

size_t ws_bytes_g(const Geo& g, int op) {
    switch (op) {
        case PDSSM_OP_SELECT:
            return align256((size_t)g.S * g.L * g.K * 4);
        case PDSSM_OP_FWD:
            return plan_bytes(g) + (g.P > 0 ? seq_act_bytes(g) + readout_w_bytes(g) : 0) +
                   fused_plan_bytes(g.H, g.K, g.N) + fused_ctrl_bytes(g.S, g.C, g.H) + seq_plan_bytes(g);
        case PDSSM_OP_BWD:
            return 2 * cs_f_bytes(g) + (g.P > 0 ? seq_f_bytes(g) + readout_w_bytes(g) : 0) +
                   (g.diag_mode == PDSSM_DIAG_PER_DICT ? seq_f_bytes(g) : 0) + fused_ctrl_bytes(g.S, g.C, g.H);
        case PDSSM_OP_READOUT:
            return readout_w_bytes(g);
        case PDSSM_OP_SOFT: {   // s [H][B L][Kp] and Mt [H][N^2][Kp] in the act dtype
            const int64_t kp = (g.K + 7) / 8 * 8;
            return align256((size_t)g.H * g.B * g.L * kp * g.act) + align256((size_t)g.H * g.N * g.N * kp * g.act);
        }
        case PDSSM_OP_LAYER: {
            const size_t sel = align256((size_t)g.S * g.L * g.K * 4), fwd = ws_bytes_g(g, PDSSM_OP_FWD);
            return seq_act_bytes(g) + (sel > fwd ? sel : fwd);
        }
        case PDSSM_OP_SEGMENT: {
            size_t fwd = plan_bytes(g) + chunk_state_bytes_g(g);
            size_t bwd = 2 * cs_f_bytes(g) + (g.P > 0 ? seq_f_bytes(g) + readout_w_bytes(g) : 0);
            return fwd > bwd ? fwd : bwd;
        }
        default:
            return 0;
    }
}

bool misaligned(const void* p, size_t a) { return p && (reinterpret_cast<uintptr_t>(p) % a) != 0; }

pdssm_status cuda_check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return PDSSM_OK;
}

int threads_for(int64_t N) { return (int)((N + 31) / 32 * 32); }

template <typename F>
pdssm_status with_nc(int nc, F&& f) {
    if (nc == 1) return f(std::integral_constant<int, 1>{});
    return f(std::integral_constant<int, 2>{});
}

template <typename F>
pdssm_status with_act(int dtype, F&& f) {
    if (dtype == PDSSM_BF16) return f(__nv_bfloat16{});
    return f(float{});
}

template <typename F>
pdssm_status with_pd(int mode, F&& f) {
    if (mode == PDSSM_DIAG_PER_DICT) return f(std::true_type{});
    return f(std::false_type{});
}

pdssm_status set_smem(const void* fn, size_t bytes) {
    if (bytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    }
    return PDSSM_OK;
}

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

// ------------------------------------------------------------------ fused fast path
// PDSSM_PATH=generic forces the three-phase kernels (used by the tests to cover both).
bool path_generic_forced() {
    const char* p = getenv("PDSSM_PATH");
    return p && strcmp(p, "generic") == 0;
}
// PDSSM_PATH=fused makes the fused path mandatory (tests): a shape it cannot take is an error
bool path_fused_forced() {
    const char* p = getenv("PDSSM_PATH");
    return p && strcmp(p, "fused") == 0;
}

// ---------------------------------------------------------------------------
// tcgen05 GEMMs (a2/a3 select, a5 projection): TMA descriptors and launch
// ---------------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// K-major operand [rows][kdim] (row stride kdim elements): box = one 128-byte K slab x box_rows,
// SWIZZLE_128B (the layout the UMMA descriptors describe); out-of-range boxes read zeros
bool make_kmajor_map(CUtensorMap* m, const void* ptr, size_t esz, int64_t kdim, int64_t rows, int box_rows) {
    EncodeTiledFn f = encode_tiled();
    if (!f) return false;
    cuuint64_t dims[2] = {(cuuint64_t)kdim, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(kdim * esz)};
    cuuint32_t box[2] = {(cuuint32_t)(tc::ROWB / esz), (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return f(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr),
             dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D operand: dims {K, d1, d2} (elements), byte strides of d1 and d2, box {128 B of K, b1, b2}
bool make_map3(CUtensorMap* m, const void* ptr, size_t esz, const int64_t (&dims)[3], const int64_t (&strides)[2],
               int b1, int b2) {
    EncodeTiledFn f = encode_tiled();
    if (!f) return false;
    cuuint64_t d[3] = {(cuuint64_t)dims[0], (cuuint64_t)dims[1], (cuuint64_t)dims[2]};
    cuuint64_t st[2] = {(cuuint64_t)strides[0], (cuuint64_t)strides[1]};
    cuuint32_t box[3] = {(cuuint32_t)(tc::ROWB / esz), (cuuint32_t)b1, (cuuint32_t)b2};
    cuuint32_t es[3] = {1, 1, 1};
    return f(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr),
             d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t gcd64(int64_t a, int64_t b) { return b ? gcd64(b, a % b) : a; }

// operands usable by TMA: 16-byte aligned base and row pitch
bool tc_operands_ok(const Geo& g, std::initializer_list<const void*> ptrs) {
    if (path_generic_forced() || !encode_tiled()) return false;
    if ((g.d_in * (int64_t)g.act) % 16 != 0) return false;
    for (const void* p : ptrs)
        if (misaligned(p, 16)) return false;
    return true;
}

// stages: bf16 4 x 48 KB ring; fp32 (3xTF32, hi + lo slabs) 2 x 96 KB
template <typename T>
constexpr int tc_stages() { return std::is_same<T, float>::value ? 2 : 4; }

template <typename T, class Epi>
pdssm_status launch_tc_maps(const CUtensorMap& mA, const CUtensorMap& mB, int64_t kdim, int bn, tc::TileMap tm,
                            dim3 grid, Epi epi, cudaStream_t st, const char* what) {
    constexpr bool SPLIT = std::is_same<T, float>::value;
    constexpr int STAGES = tc_stages<T>();
    using SM = tc::Smem<T, STAGES, SPLIT>;
    const size_t smem = SM::bytes(256);   // sized for the largest tile: one attribute per instantiation
    auto kern = tc::k_gemm_tc<T, STAGES, SPLIT, Epi>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] { attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
    if (attr_err != cudaSuccess) return fail(PDSSM_ERR_CUDA, "%s: cudaFuncSetAttribute: %s", what, cudaGetErrorString(attr_err));
    const int nk = (int)ceil_div(kdim * (int64_t)sizeof(T), tc::ROWB);
    const tc::TileGrid tg{(int)grid.x, (int)grid.y, (int)grid.z};
    const int ntiles = tg.gx * tg.gy * tg.gz;
    const int nctas = ntiles < num_sms_dev() ? ntiles : num_sms_dev();   // persistent
    kern<<<nctas, tc::THREADS, SM::bytes(bn), st>>>(mA, mB, nk, bn, tm, tg, epi);
    return cuda_check(what);
}

// plain 2-D case: A [rows_a][d_in], B [rows_b][d_in]
template <typename T, class Epi>
pdssm_status launch_tc(const Geo& g, const void* A, int64_t rows_a, const void* Bm, int64_t rows_b, int bn, Epi epi,
                       cudaStream_t st, const char* what) {
    CUtensorMap mA, mB;
    if (!make_kmajor_map(&mA, A, sizeof(T), g.d_in, rows_a, tc::BM) ||
        !make_kmajor_map(&mB, Bm, sizeof(T), g.d_in, rows_b, bn))
        return fail(PDSSM_ERR_CUDA, "%s: cuTensorMapEncodeTiled failed", what);
    dim3 grid((unsigned)ceil_div(rows_a, tc::BM), (unsigned)ceil_div(rows_b, bn));
    return launch_tc_maps<T>(mA, mB, g.d_in, bn, tc::TileMap{0, 1, 1, 0}, grid, epi, st, what);
}

// readout weights, act dtype: Cp[h][p][(c,n)] (y = Cp . h) and CT[h][(c,n)][p] (e = CT . dy),
// both carrying the sign of Re(C h) = C_re h_re - C_im h_im
template <typename T>
__global__ void k_readout_weights(const float* __restrict__ C, T* __restrict__ Cp, T* __restrict__ CT, int H, int nc,
                                  int P, int N) {
    const int64_t total = (int64_t)H * nc * P * N;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int n = (int)(i % N);
        const int p = (int)((i / N) % P);
        const int c = (int)((i / ((int64_t)N * P)) % nc);
        const int h = (int)(i / ((int64_t)N * P * nc));
        const float v = c == 0 ? C[i] : -C[i];
        const int cN = nc * N;
        if (Cp) stact(Cp + ((size_t)h * P + p) * cN + c * N + n, v);
        if (CT) stact(CT + ((size_t)h * cN + c * N + n) * P + p, v);
    }
}

// tensor-core readout applicability: TMA row pitches, 16-column output groups
bool tc_readout_ok(const Geo& g, std::initializer_list<const void*> ptrs) {
    if (path_generic_forced() || !encode_tiled()) return false;
    if ((g.nc * g.N * (int64_t)g.act) % 16 != 0 || g.P % 16 != 0 || (g.nc * g.N) % 16 != 0) return false;
    if ((g.P * (int64_t)g.act) % 16 != 0) return false;
    for (const void* p : ptrs)
        if (misaligned(p, 16)) return false;
    return true;
}

// y[b][t][h][p] = sum_w Cp[h][p][w] h[b][h][t][w]  (A: 3-D (cN, L, S) map, z = sequence)
template <typename T>
pdssm_status readout_tc(const Geo& g, const T* hseq, const T* Cp, T* y, cudaStream_t st) {
    const int64_t cN = g.nc * g.N;
    const int bn = (int)(g.P < 256 ? g.P : 256);
    CUtensorMap mA, mB;
    const int64_t da[3] = {cN, g.L, g.S};
    const int64_t sa[2] = {cN * (int64_t)sizeof(T), g.L * cN * (int64_t)sizeof(T)};
    if (!make_map3(&mA, hseq, sizeof(T), da, sa, tc::BM, 1) || !make_kmajor_map(&mB, Cp, sizeof(T), cN, g.H * g.P, bn))
        return fail(PDSSM_ERR_CUDA, "readout_tc: cuTensorMapEncodeTiled failed");
    const int tiles = (int)ceil_div(g.L, tc::BM);
    dim3 grid((unsigned)(tiles * g.S), (unsigned)ceil_div(g.P, bn));
    return launch_tc_maps<T>(mA, mB, cN, bn, tc::TileMap{1, tiles, (int)g.H, (int)g.P}, grid,
                             tc::EpiReadout<T>{y, (int)g.L, (int)g.H, (int)g.P}, st, "readout_tc");
}

// e[b][h][t][w] = dh + sum_p CT[h][w][p] dy[b][t][h][p]  (A: 3-D (P, H, B*L) map, z = head)
template <typename T>
pdssm_status adjoint_tc(const Geo& g, const T* dy, const T* CT, const T* dh, float* e, cudaStream_t st) {
    const int64_t cN = g.nc * g.N;
    const int bn = (int)(cN < 256 ? cN : 256);
    CUtensorMap mA, mB;
    const int64_t da[3] = {g.P, g.H, g.B * g.L};
    const int64_t sa[2] = {g.P * (int64_t)sizeof(T), g.H * g.P * (int64_t)sizeof(T)};
    if (!make_map3(&mA, dy, sizeof(T), da, sa, 1, tc::BM) || !make_kmajor_map(&mB, CT, sizeof(T), g.P, g.H * cN, bn))
        return fail(PDSSM_ERR_CUDA, "adjoint_tc: cuTensorMapEncodeTiled failed");
    dim3 grid((unsigned)ceil_div(g.B * g.L, tc::BM), (unsigned)ceil_div(cN, bn), (unsigned)g.H);
    return launch_tc_maps<T>(mA, mB, g.P, bn, tc::TileMap{2, 1, 1, (int)cN}, grid,
                             tc::EpiAdjoint<T>{e, dh, g.B * g.L, (int)g.L, (int)g.H, (int)cN}, st, "adjoint_tc");
}

// select tile width: whole heads, a multiple of lcm(K, 16), <= 256 (0: not possible)
int select_bn(const Geo& g) {
    const int64_t l = g.K / gcd64(g.K, 16) * 16;
    if (l > 256) return 0;
    const int64_t full = (256 / l) * l;
    const int64_t need = ceil_div(g.H * g.K, l) * l;
    return (int)(need < full ? need : full);
}

// direct state gradient e = dh + conj(C)^T dy (bwd with a readout): tensor cores when the
// shapes allow it (CT staged in wbuf), else the SIMT kernel
template <typename T, int NC>
pdssm_status prepare_e(const Geo& g, const void* dh, const void* dy, const float* C, float* e, void* wbuf,
                       cudaStream_t st) {
    if (tc_readout_ok(g, {dy, dh, e, wbuf})) {
        T* CT = static_cast<T*>(wbuf);
        k_readout_weights<T><<<(unsigned)ceil_div(g.H * g.nc * g.P * g.N, 256), 256, 0, st>>>(C, nullptr, CT, (int)g.H,
                                                                                              (int)g.nc, (int)g.P, (int)g.N);
        pdssm_status r = cuda_check("readout_weights");
        if (r) return r;
        return adjoint_tc<T>(g, static_cast<const T*>(dy), CT, static_cast<const T*>(dh), e, st);
    }
    k_bwd_prepare_e<T, NC><<<(unsigned)(g.S * g.L), 128, (size_t)g.P * 4, st>>>(
        static_cast<const T*>(dh), static_cast<const T*>(dy), C, e, (int)g.H, (int)g.L, (int)g.N, (int)g.P);
    return cuda_check("bwd_prepare_e");
}

// ---------------------------------------------------------------------------
// single-chunk path: plan, sizing, launches
// ---------------------------------------------------------------------------

constexpr size_t kSeqSmemBudget = 200 * 1024;
constexpr int kSeqG = seq::SEQ_G;     // backward group
constexpr int kSeqGF = seq::SEQ_GF;   // forward group

// ring depth R for this shape (0: the layout does not fit)
// ring depth R for this shape (0: the layout does not fit).  When there are more
// sequences than SMs, the budget is split so that ceil(S / #SMs) CTAs (up to 4) fit per SM.
int seq_ring(const Geo& g, bool bwd, bool agg, size_t esz_e) {
    const int G = bwd ? kSeqG : kSeqGF;
    const int ngroups = (int)ceil_div(g.L, G);
    const int64_t per_sm = std::min<int64_t>(std::max<int64_t>(ceil_div(g.S, num_sms_dev()), 1), 4);
    const size_t budget = std::min<size_t>(kSeqSmemBudget, (size_t)(226 * 1024) / (size_t)per_sm - 1024);
    int best = 0;
    for (int R = 2; R <= 16 && R <= ngroups + 1; ++R) {
        seq::Layout ly((int)g.N, (int)g.K, R, G, g.nc, (int)g.act, (int)esz_e, g.diag_mode == PDSSM_DIAG_PER_DICT, agg, bwd,
                       (int)g.L);
        if (ly.bytes <= budget) best = R;
    }
    if (best == 0 && ngroups <= 1) best = 2;
    return best;
}

bool seq_applicable(const Geo& g, std::initializer_list<const void*> ptrs) {
    if (g.C != 1 || env_path_is("fused") || env_path_is("generic")) return false;
    if (!seq_shape_ok(g.N, g.K, g.L, g.nc, g.act)) return false;
    for (const void* p : ptrs)
        if (misaligned(p, 16)) return false;
    return seq_ring(g, false, true, g.act) >= 2 && seq_ring(g, true, false, 4) >= 2;
}

pdssm_status seq_set_smem(const void* f, size_t bytes) {
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return PDSSM_OK;
}

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

pdssm_status fwd_seq(const Geo& g, seq::SeqArgs& sa, uint8_t* rec, uint8_t* wm, uint8_t* ovf, cudaStream_t st) {
    seq::k_build_seq_plan<<<(unsigned)(g.H * g.K), (unsigned)g.N, (size_t)g.N * 2, st>>>(
        sa.dict_idx, rec, wm, ovf, const_cast<uint16_t*>(sa.pstart), const_cast<uint16_t*>(sa.psrc), (int)g.N, g.flags);
    pdssm_status r = cuda_check("build_seq_plan");
    if (r) return r;
    const bool agg = (g.flags & PDSSM_EXPORT_MAPS) != 0;
    sa.R = seq_ring(g, false, agg, g.act);
    sa.G = kSeqGF;
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
                                   (int)g.L);
                    // compile-time N for the production variants (no maps, no checks)
                    auto kern = seq::k_fwd_seq<T, NC, PD, AGG, CHK, 0>;
                    if constexpr (!AGG && !CHK) {
                        if (g.N == 128) kern = seq::k_fwd_seq<T, NC, PD, false, false, 128>;
                        else if (g.N == 64) kern = seq::k_fwd_seq<T, NC, PD, false, false, 64>;
                    }
                    pdssm_status rr = seq_set_smem((const void*)kern, ly.bytes);
                    if (rr) return rr;
                    // programmatic dependent launch: the prologue overlaps the plan kernel's tail
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3((unsigned)g.S);
                    cfg.blockDim = dim3((unsigned)g.N + 32);   // + producer warp
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
                const bool chk = (g.flags & PDSSM_CHECK_FINITE) != 0;
                if (agg) return chk ? go(std::true_type{}, std::true_type{}) : go(std::true_type{}, std::false_type{});
                return chk ? go(std::false_type{}, std::true_type{}) : go(std::false_type{}, std::false_type{});
            });
        });
    });
}

template <typename TE>
pdssm_status bwd_seq(const Geo& g, seq::SeqArgs& sa, cudaStream_t st) {
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        using TEE = typename std::conditional<std::is_same<TE, void>::value, T, TE>::type;
        sa.R = seq_ring(g, true, false, sizeof(TEE));
        sa.G = kSeqG;
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            return with_pd(g.diag_mode, [&](auto pdv) {
                constexpr bool PD = decltype(pdv)::value;
                seq::Layout ly((int)g.N, (int)g.K, sa.R, sa.G, NC, (int)sizeof(T), (int)sizeof(TEE), PD, false, true,
                               (int)g.L);
                auto kern = g.N == 128 ? seq::k_bwd_seq<T, TEE, NC, PD, 128>
                            : g.N == 64    ? seq::k_bwd_seq<T, TEE, NC, PD, 64>
                                           : seq::k_bwd_seq<T, TEE, NC, PD, 0>;
                pdssm_status rr = seq_set_smem((const void*)kern, ly.bytes);
                if (rr) return rr;
                kern<<<(unsigned)g.S, (unsigned)g.N + 32, ly.bytes, st>>>(sa);   // + producer warp
                return cuda_check("bwd_seq");
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

}  // namespace

// ====================================================================== ABI
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
    e = cudaMemcpyFromSymbol(&w, g_err_word, sizeof(w));
    if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "read error word: %s", cudaGetErrorString(e));
    uint32_t z = 0;
    e = cudaMemcpyToSymbol(g_err_word, &z, sizeof(z));
    if (e != cudaSuccess) return fail(PDSSM_ERR_CUDA, "clear error word: %s", cudaGetErrorString(e));
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

pdssm_status pdssm_select(const void* x, const void* S, const uint16_t* dict_idx, uint8_t* kstar, uint16_t* P_opt,
                          float* logits_opt, const pdssm_dims* dims, void* ws, size_t ws_bytes,
                          pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (g.d_in < 1) return fail(PDSSM_ERR_SHAPE, "select: d_in must be >= 1");
    if (!x || !S || !kstar) return fail(PDSSM_ERR_NULL, "select: x, S, kstar are required");
    if (P_opt && !dict_idx) return fail(PDSSM_ERR_NULL, "select: P_opt needs dict_idx");
    if (misaligned(x, g.act) || misaligned(S, g.act) || misaligned(dict_idx, 2) || misaligned(P_opt, 2) ||
        misaligned(logits_opt, 4))
        return fail(PDSSM_ERR_ALIGN, "select: misaligned pointer");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // tensor-core path (a2 logits in TMEM, a3 argmax + a4 P gather fused in the epilogue)
    const int bn = select_bn(g);
    if (bn > 0 && tc_operands_ok(g, {x, S})) {
        tc::EpiSelect epi{kstar, logits_opt, dict_idx, P_opt, g.B * g.L, (int)g.L, (int)g.H, (int)g.K, (int)g.N, g.flags};
        return with_act(g.dtype, [&](auto tv) {
            using T = decltype(tv);
            return launch_tc<T>(g, x, g.B * g.L, S, g.H * g.K, bn, epi, st, "select_tc");
        });
    }
    float* logits = logits_opt;
    if (!logits) {
        if (!ws || ws_bytes < ws_bytes_g(g, PDSSM_OP_SELECT))
            return fail(PDSSM_ERR_WORKSPACE, "select: workspace too small (need %zu)", ws_bytes_g(g, PDSSM_OP_SELECT));
        logits = static_cast<float*>(ws);
    }
    const int64_t M = g.B * g.L, NN = g.H * g.K;
    dim3 grid((unsigned)ceil_div(M, 64), (unsigned)ceil_div(NN, 64));
    r = with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        k_select_logits_simt<T><<<grid, 256, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(S), logits,
                                                      (int)g.B, (int)g.L, (int)g.H, (int)g.K, (int)g.d_in, g.flags);
        return cuda_check("select_logits");
    });
    if (r) return r;
    const int64_t rows = g.S * g.L;
    k_select_argmax<<<(unsigned)ceil_div(rows, 8), dim3(32, 8), 0, st>>>(logits, dict_idx, kstar, P_opt, rows,
                                                                       (int)g.H, (int)g.L, (int)g.N, (int)g.K);
    return cuda_check("select_argmax");
}

pdssm_status pdssm_project(const void* x, const void* Bw, void* b_out, const pdssm_dims* dims, pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (g.d_in < 1) return fail(PDSSM_ERR_SHAPE, "project: d_in must be >= 1");
    if (!x || !Bw || !b_out) return fail(PDSSM_ERR_NULL, "project: x, Bw, b_out are required");
    if (misaligned(x, g.act) || misaligned(Bw, g.act) || misaligned(b_out, g.act))
        return fail(PDSSM_ERR_ALIGN, "project: misaligned pointer");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t cN = g.nc * g.N, NN = g.H * cN;
    if (cN % 16 == 0 && tc_operands_ok(g, {x, Bw, b_out})) {
        return with_act(g.dtype, [&](auto tv) {
            using T = decltype(tv);
            tc::EpiProject<T> epi{static_cast<T*>(b_out), g.B * g.L, (int)g.L, (int)g.H, (int)cN, NN};
            return launch_tc<T>(g, x, g.B * g.L, Bw, NN, (int)(NN < 256 ? NN : 256), epi, st, "project_tc");
        });
    }
    dim3 grid((unsigned)ceil_div(g.B * g.L, 64), (unsigned)ceil_div(NN, 64));
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        k_project_simt<T><<<grid, 256, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(Bw),
                                                static_cast<T*>(b_out), (int)g.B, (int)g.L, (int)g.H, (int)cN,
                                                (int)g.d_in);
        return cuda_check("project_simt");
    });
}

pdssm_status pdssm_diag_gen(const void* x, const void* Wd, const float* bias_opt, void* D_out, const pdssm_dims* dims,
                            pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (g.d_in < 1) return fail(PDSSM_ERR_SHAPE, "diag_gen: d_in must be >= 1");
    if (!x || !Wd || !D_out) return fail(PDSSM_ERR_NULL, "diag_gen: x, Wd, D_out are required");
    if (misaligned(x, g.act) || misaligned(Wd, g.act) || misaligned(D_out, g.act) || misaligned(bias_opt, 4))
        return fail(PDSSM_ERR_ALIGN, "diag_gen: misaligned pointer");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t cN = g.nc * g.N, NN = g.H * cN;
    if (g.N % 16 == 0 && cN <= 256 && tc_operands_ok(g, {x, Wd, D_out})) {
        return with_act(g.dtype, [&](auto tv) {
            using T = decltype(tv);
            tc::EpiDiag<T> epi{static_cast<T*>(D_out), bias_opt, g.B * g.L, (int)g.L, (int)g.H, (int)g.N, (int)g.nc};
            return launch_tc<T>(g, x, g.B * g.L, Wd, NN, (int)cN, epi, st, "diag_gen_tc");   // one head per tile
        });
    }
    if ((r = pdssm_project(x, Wd, D_out, dims, stream))) return r;
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        const int64_t rows = g.S * g.L;
        sg::k_diag_activate<T><<<(unsigned)std::min<int64_t>(ceil_div(rows * g.N, 256), 65535), 256, 0, st>>>(
            static_cast<T*>(D_out), bias_opt, rows, (int)g.H, (int)g.L, (int)g.N, (int)g.nc);
        return cuda_check("diag_activate");
    });
}

pdssm_status pdssm_soft_select(const float* logits, const float* M, uint16_t* P_out, const pdssm_dims* dims, void* ws,
                               size_t ws_bytes, pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (!logits || !M || !P_out) return fail(PDSSM_ERR_NULL, "soft_select: logits, M, P_out are required");
    if (g.N % 16 != 0 || g.N > 256) return fail(PDSSM_ERR_UNSUPPORTED, "soft_select: N must be a multiple of 16 <= 256");
    if (misaligned(logits, 4) || misaligned(M, 4) || misaligned(P_out, 2) || misaligned(ws, 256))
        return fail(PDSSM_ERR_ALIGN, "soft_select: misaligned pointer");
    const size_t need = ws_bytes_g(g, PDSSM_OP_SOFT);
    if (!ws || ws_bytes < need) return fail(PDSSM_ERR_WORKSPACE, "soft_select: workspace too small (need %zu)", need);
    if (!encode_tiled()) return fail(PDSSM_ERR_UNSUPPORTED, "soft_select: tensor-map encoder unavailable");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t kp = (g.K + 7) / 8 * 8, BL = g.B * g.L;
    Geo gk = g;
    gk.d_in = kp;   // the GEMM's K dimension
    const int bn = (256 / (int)g.N) * (int)g.N;
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        T* sbuf = static_cast<T*>(ws);
        T* Mt = reinterpret_cast<T*>(static_cast<char*>(ws) + align256((size_t)g.H * BL * kp * g.act));
        sg::k_soft_stage_s<T><<<(unsigned)ceil_div(BL * g.H, 8), 256, 0, st>>>(logits, sbuf, BL, (int)g.H, (int)g.L,
                                                                               (int)g.K, (int)kp);
        sg::k_soft_stage_M<T><<<(unsigned)std::min<int64_t>(ceil_div(g.H * g.N * g.N * kp, 256), 65535), 256, 0, st>>>(
            M, Mt, (int)g.H, (int)g.K, (int)g.N, (int)kp);
        pdssm_status rr = cuda_check("soft_stage");
        if (rr) return rr;
        for (int64_t h = 0; h < g.H; ++h) {
            tc::EpiColArgmax epi{P_out, BL, (int)g.L, (int)g.H, (int)g.N, (int)h};
            rr = launch_tc<T>(gk, sbuf + (size_t)h * BL * kp, BL, Mt + (size_t)h * g.N * g.N * kp, g.N * g.N, bn, epi, st,
                              "soft_select_tc");
            if (rr) return rr;
        }
        return PDSSM_OK;
    });
}

pdssm_status pdssm_readout(const void* h, const float* C, void* y, const pdssm_dims* dims, void* ws, size_t ws_bytes,
                           pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (!h || !C || !y) return fail(PDSSM_ERR_NULL, "readout: h, C, y are required");
    if (g.P < 1) return fail(PDSSM_ERR_SHAPE, "readout: p_out must be >= 1");
    if (misaligned(h, g.act) || misaligned(y, g.act) || misaligned(C, 4)) return fail(PDSSM_ERR_ALIGN, "readout: misaligned");
    if (!ws || ws_bytes < readout_w_bytes(g))
        return fail(PDSSM_ERR_WORKSPACE, "readout: workspace too small (need %zu)", readout_w_bytes(g));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        if (tc_readout_ok(g, {h, y, ws})) {
            T* Cp = static_cast<T*>(ws);
            k_readout_weights<T><<<(unsigned)ceil_div(g.H * g.nc * g.P * g.N, 256), 256, 0, st>>>(
                C, Cp, nullptr, (int)g.H, (int)g.nc, (int)g.P, (int)g.N);
            pdssm_status rr = cuda_check("readout_weights");
            if (rr) return rr;
            return readout_tc<T>(g, static_cast<const T*>(h), Cp, static_cast<T*>(y), st);
        }
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            k_readout<T, NC><<<(unsigned)(g.S * g.L), 128, (size_t)NC * g.N * 4, st>>>(
                static_cast<const T*>(h), C, static_cast<T*>(y), (int)g.H, (int)g.L, (int)g.N, (int)g.P);
            return cuda_check("readout");
        });
    });
}

// ---------------------------------------------------------------------------
// layer-level forward: select -> projection -> scan (+ readout)
// ---------------------------------------------------------------------------
pdssm_status pdssm_layer_fwd(const void* x, const void* S, const uint16_t* dict_idx, const void* diag, const void* Bw,
                             const float* C_opt, const float* h0_opt, uint8_t* kstar, void* h_out_opt, void* y_opt,
                             void* chunk_state, const pdssm_dims* dims, void* ws, size_t ws_bytes,
                             pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (!x || !S || !dict_idx || !diag || !Bw || !kstar || !chunk_state)
        return fail(PDSSM_ERR_NULL, "layer_fwd: x, S, dict_idx, diag, Bw, kstar, chunk_state are required");
    if (g.d_in < 1) return fail(PDSSM_ERR_SHAPE, "layer_fwd: d_in must be >= 1");
    const size_t need = ws_bytes_g(g, PDSSM_OP_LAYER);
    if (!ws || ws_bytes < need) return fail(PDSSM_ERR_WORKSPACE, "layer_fwd: workspace too small (need %zu)", need);
    char* b = static_cast<char*>(ws);                 // b_t [B][H][L][c][N] act
    char* rest = b + seq_act_bytes(g);
    const size_t rest_bytes = ws_bytes - seq_act_bytes(g);
    if ((r = pdssm_select(x, S, dict_idx, kstar, nullptr, nullptr, dims, rest, rest_bytes, stream))) return r;
    if ((r = pdssm_project(x, Bw, b, dims, stream))) return r;
    return pdssm_scan_fwd(kstar, dict_idx, diag, b, h0_opt, C_opt, h_out_opt, y_opt, chunk_state, nullptr, dims, rest,
                          rest_bytes, stream);
}

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
    // the single-chunk path builds its records and the CSR plan in one launch (fwd_seq)
    if (!use_seq && (r = launch_plan(g, dict_idx, pstart, psrc, st))) return r;
    if (env_path_is("seq") && !use_seq)
        return fail(PDSSM_ERR_UNSUPPORTED, "scan_fwd: PDSSM_PATH=seq but the single-chunk path does not apply");
    const bool use_fused = !use_seq && fused_applicable(
        g, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, bias, hout, h0_opt, chunk_state, maps});
    if (use_seq) {
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
    if (y_opt) {
        r = with_act(g.dtype, [&](auto tv) {
            using T = decltype(tv);
            if (tc_readout_ok(g, {hout, y_opt, wbuf})) {
                T* Cp = static_cast<T*>(wbuf);
                k_readout_weights<T><<<(unsigned)ceil_div(g.H * g.nc * g.P * g.N, 256), 256, 0, st>>>(
                    C_opt, Cp, nullptr, (int)g.H, (int)g.nc, (int)g.P, (int)g.N);
                pdssm_status rr = cuda_check("readout_weights");
                if (rr) return rr;
                return readout_tc<T>(g, static_cast<const T*>(hout), Cp, static_cast<T*>(y_opt), st);
            }
            return with_nc(g.nc, [&](auto ncv) {
                constexpr int NC = decltype(ncv)::value;
                k_readout<T, NC><<<(unsigned)(g.S * g.L), 128, (size_t)NC * g.N * 4, st>>>(
                    static_cast<const T*>(hout), C_opt, static_cast<T*>(y_opt), (int)g.H, (int)g.L, (int)g.N, (int)g.P);
                return cuda_check("readout");
            });
        });
    }
    return r;
}

pdssm_status pdssm_scan_bwd(const uint8_t* kstar, const uint16_t* dict_idx, const void* diag, const void* h_saved,
                            const float* h0_opt, const void* chunk_state, const void* dh_opt, const void* dy_opt,
                            const float* C_opt, const float* lam_in_opt, void* dbias, void* ddiag, float* gsel,
                            float* dh0_opt, const pdssm_dims* dims, void* ws, size_t ws_bytes,
                            pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if ((r = common_scan_checks(g, kstar, dict_idx, diag))) return r;
    if (!h_saved) return fail(PDSSM_ERR_NULL, "scan_bwd: h_saved is required");
    if (!chunk_state) return fail(PDSSM_ERR_WORKSPACE, "scan_bwd: chunk_state is required");
    if (!dbias || !ddiag) return fail(PDSSM_ERR_NULL, "scan_bwd: dbias and ddiag are required");
    if (dy_opt && (!C_opt || g.P < 1)) return fail(PDSSM_ERR_NULL, "scan_bwd: dy_opt needs C_opt and p_out >= 1");
    if (misaligned(h_saved, g.act) || misaligned(dh_opt, g.act) || misaligned(dy_opt, g.act) || misaligned(dbias, g.act) ||
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
    uint32_t* ctrl = bump.take<uint32_t>(fused_ctrl_bytes(g.S, g.C, g.H));
    ChunkStateView cs = cs_view(g, const_cast<void*>(chunk_state));
    const int thr = threads_for(g.N);
    const unsigned items = (unsigned)(g.S * g.C);
    const bool use_seq = seq_applicable(g, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, h_saved, dh_opt, ebuf});
    if (env_path_is("seq") && !use_seq)
        return fail(PDSSM_ERR_UNSUPPORTED, "scan_bwd: PDSSM_PATH=seq but the single-chunk path does not apply");
    const bool use_fused = !use_seq &&
        fused_applicable(g, {g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr, h_saved, dh_opt, h0_opt, lam_in_opt,
                             dbias, g.diag_mode == PDSSM_DIAG_PER_STEP ? ddiag : nullptr, dh0_opt, chunk_state});
    if (!use_fused && !use_seq && path_fused_forced())
        return fail(PDSSM_ERR_UNSUPPORTED, "scan_bwd: PDSSM_PATH=fused but the fused path does not apply to these dims");
    if (use_seq) {
        if (dy_opt) {
            r = with_act(g.dtype, [&](auto tv) {
                using T = decltype(tv);
                return with_nc(g.nc, [&](auto ncv) {
                    constexpr int NC = decltype(ncv)::value;
                    return prepare_e<T, NC>(g, dh_opt, dy_opt, C_opt, ebuf, wbuf, st);
                });
            });
            if (r) return r;
        }
        seq::SeqArgs sa{};
        sa.kstar = kstar; sa.dict_idx = dict_idx;
        sa.diag = g.diag_mode == PDSSM_DIAG_PER_STEP ? diag : nullptr;
        sa.diag_dict = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<const float*>(diag) : nullptr;
        sa.bias = dy_opt ? static_cast<const void*>(ebuf) : dh_opt;
        sa.hsaved = h_saved; sa.h0 = h0_opt; sa.lam_in = lam_in_opt; sa.cs = cs;
        sa.out0 = dbias; sa.out1 = g.diag_mode == PDSSM_DIAG_PER_DICT ? static_cast<void*>(dDbuf) : ddiag;
        sa.gsel = gsel; sa.dh0 = dh0_opt;
        sa.H = (int)g.H; sa.L = (int)g.L; sa.N = (int)g.N; sa.K = (int)g.K; sa.flags = g.flags;
        r = dy_opt ? bwd_seq<float>(g, sa, st) : bwd_seq<void>(g, sa, st);
        if (r) return r;
        if (g.diag_mode == PDSSM_DIAG_PER_DICT) {
            r = with_nc(g.nc, [&](auto ncv) {
                constexpr int NC = decltype(ncv)::value;
                k_bwd_reduce_dict<NC><<<(unsigned)(g.H * g.K), 256, 0, st>>>(
                    kstar, dDbuf, static_cast<float*>(ddiag), (int)g.B, (int)g.H, (int)g.L, (int)g.N, (int)g.K);
                return cuda_check("bwd_reduce_dict");
            });
        }
        return r;
    }
    if (use_fused) {
        if (dy_opt) {
            r = with_act(g.dtype, [&](auto tv) {
                using T = decltype(tv);
                return with_nc(g.nc, [&](auto ncv) {
                    constexpr int NC = decltype(ncv)::value;
                    return prepare_e<T, NC>(g, dh_opt, dy_opt, C_opt, ebuf, wbuf, st);
                });
            });
            if (r) return r;
        }
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
        r = dy_opt ? bwd_fused<float>(g, fa, st) : bwd_fused<void>(g, fa, st);
        if (r) return r;
        if (g.diag_mode == PDSSM_DIAG_PER_DICT) {
            r = with_nc(g.nc, [&](auto ncv) {
                constexpr int NC = decltype(ncv)::value;
                k_bwd_reduce_dict<NC><<<(unsigned)(g.H * g.K), 256, 0, st>>>(
                    kstar, dDbuf, static_cast<float*>(ddiag), (int)g.B, (int)g.H, (int)g.L, (int)g.N, (int)g.K);
                return cuda_check("bwd_reduce_dict");
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
                    k_bwd_phaseB<NC><<<(unsigned)g.S, thr, (size_t)NC * g.N * 4, st>>>(cs, betap, lam_in_opt, mu,
                                                                                         dh0_opt, (int)g.N, g.C);
                    if ((rr = cuda_check("bwd_phaseB"))) return rr;
                    const int nw = thr / 32;
                    size_t smC = (size_t)2 * NC * g.N * 4 + (size_t)64 * nw * 4;
                    if ((rr = set_smem((const void*)k_bwd_phaseC<T, TE, NC, PD>, smC))) return rr;
                    k_bwd_phaseC<T, TE, NC, PD><<<items, thr, smC, st>>>(
                        kstar, dict_idx, dg, dd, static_cast<const T*>(h_saved), h0_opt, e, mu, static_cast<T*>(dbias),
                        PD ? nullptr : static_cast<T*>(ddiag), dDbuf, gsel, (int)g.H, (int)g.L, (int)g.N, (int)g.K,
                        g.tau, g.C);
                    if ((rr = cuda_check("bwd_phaseC"))) return rr;
                    if (PD) {
                        k_bwd_reduce_dict<NC><<<(unsigned)(g.H * g.K), 256, 0, st>>>(
                            kstar, dDbuf, static_cast<float*>(ddiag), (int)g.B, (int)g.H, (int)g.L, (int)g.N, (int)g.K);
                        if ((rr = cuda_check("bwd_reduce_dict"))) return rr;
                    }
                    return PDSSM_OK;
                };
                if (dy_opt) {
                    pdssm_status rr = prepare_e<T, NC>(g, dh_opt, dy_opt, C_opt, ebuf, wbuf, st);
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
    ChunkStateView cs = cs_view(g, csmem);
    if ((r = launch_plan(g, dict_idx, pstart, psrc, st))) return r;
    if ((r = fwd_three_phase(g, kstar, dict_idx, pstart, psrc, diag, bias, nullptr, cs, nullptr, nullptr, false, st)))
        return r;
    SummaryView sv{static_cast<char*>(summary_out), summary_block_bytes(g), npad8(g.N)};
    return with_nc(g.nc, [&](auto ncv) {
        constexpr int NC = decltype(ncv)::value;
        k_fold_aggregates<NC><<<(unsigned)g.S, threads_for(g.N), (size_t)NC * g.N * 4 + g.N * 2 + 16, st>>>(
            cs, sv, (int)g.N, g.C);
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
                    k_bwd_phaseA<T, TE, NC, PD><<<items, thr, (size_t)2 * NC * g.N * 4, st>>>(
                        kstar, dict_idx, dg, dd, e, betap, (int)g.H, (int)g.L, (int)g.N, (int)g.K, g.tau, g.C);
                    pdssm_status rr = cuda_check("bwd_phaseA");
                    if (rr) return rr;
                    k_bwd_phaseB<NC><<<(unsigned)g.S, thr, (size_t)NC * g.N * 4, st>>>(cs, betap, nullptr, mu,
                                                                                         beta_out, (int)g.N, g.C);
                    return cuda_check("bwd_phaseB");
                };
                if (dy_opt) {
                    pdssm_status rr = prepare_e<T, NC>(g, dh_opt, dy_opt, C_opt, ebuf, wbuf, st);
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
