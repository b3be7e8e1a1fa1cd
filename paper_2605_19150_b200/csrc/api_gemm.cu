// libpdssm.so: tcgen05 GEMMs (select a2-a4, projection a5, readout a8, adjoint, D_t generator, soft generator).
#include "api_internal.cuh"
#include "k_select.cuh"
#include "k_scan_bwd.cuh"
#include "k_gemm_tc.cuh"
#include "k_surrogate.cuh"

using namespace pdssm;
using namespace pdssm::api;

namespace pdssm {
namespace api {

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

template <typename T, class Epi, bool BPRE = false, int BPRE_STAGES = 3, int MT = 1, bool ATM = false>
pdssm_status launch_tc_maps(const CUtensorMap& mA, const CUtensorMap& mB, int64_t kdim, int bn, tc::TileMap tm,
                            dim3 grid, Epi epi, cudaStream_t st, const char* what, const CUtensorMap* mBlo = nullptr) {
    constexpr bool SPLIT = std::is_same<T, float>::value;
    // pre-split weights: three stages of (A hi/lo + B hi/lo) slabs fit at bn <= 128, four at bn <= 64
    constexpr int STAGES = BPRE ? BPRE_STAGES : tc_stages<T>();
    constexpr int BN_MAX = (BPRE || MT > 1) ? (BPRE_STAGES >= 4 && MT == 1 && !ATM ? 64 : 128) : 256;
    using SM = tc::Smem<T, STAGES, SPLIT, MT, ATM>;
    const size_t smem = SM::bytes(BN_MAX);   // sized for the largest tile: one attribute per instantiation
    if (bn > BN_MAX) return fail(PDSSM_ERR_UNSUPPORTED, "%s: tile width %d above %d", what, bn, BN_MAX);
    auto kern = tc::k_gemm_tc<T, STAGES, SPLIT, Epi, BPRE, MT, ATM>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] { attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
    if (attr_err != cudaSuccess) return fail(PDSSM_ERR_CUDA, "%s: cudaFuncSetAttribute: %s", what, cudaGetErrorString(attr_err));
    const int nk = (int)ceil_div(kdim * (int64_t)sizeof(T), tc::ROWB);
    const tc::TileGrid tg{(int)grid.x, (int)grid.y, (int)grid.z};
    const int ntiles = tg.gx * tg.gy * tg.gz;
    const int nctas = ntiles < num_sms_dev() ? ntiles : num_sms_dev();   // persistent
    // programmatic dependent launch: the prologue (barriers, TMEM allocation, tensormap prefetch)
    // overlaps the tail of the previous launch (the readout's weight split triggers it at entry);
    // the TMA producer's griddepcontrol.wait orders every global access of the kernel after it
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nctas);
    cfg.blockDim = dim3(tc::THREADS);
    cfg.dynamicSmemBytes = SM::bytes(bn);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const CUtensorMap mBl = mBlo ? *mBlo : mB;
    cudaError_t le = cudaLaunchKernelEx(&cfg, kern, mA, mB, mBl, (int)nk, bn, tm, tg, epi);
    if (le != cudaSuccess) return fail(PDSSM_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(le));
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
// With Cp_lo (fp32 only) Cp receives the tf32 hi part and Cp_lo the rest (the 3xTF32 split of the
// GEMM, done once here instead of per tile: k_gemm_tc BPRE).
template <typename T>
__global__ void k_readout_weights(const float* __restrict__ C, T* __restrict__ Cp, T* __restrict__ CT, int H, int nc,
                                  int P, int N, float* __restrict__ Cp_lo = nullptr) {
    asm volatile("griddepcontrol.launch_dependents;");   // the GEMM after it may start its prologue
    const int64_t total = (int64_t)H * nc * P * N;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int n = (int)(i % N);
        const int p = (int)((i / N) % P);
        const int c = (int)((i / ((int64_t)N * P)) % nc);
        const int h = (int)(i / ((int64_t)N * P * nc));
        const float v = c == 0 ? C[i] : -C[i];
        const int cN = nc * N;
        if (Cp && Cp_lo) {
            const float vh = __uint_as_float(tc::tf32_rna(v));
            Cp[((size_t)h * P + p) * cN + c * N + n] = vh;
            Cp_lo[((size_t)h * P + p) * cN + c * N + n] = v - vh;
        } else if (Cp) {
            stact(Cp + ((size_t)h * P + p) * cN + c * N + n, v);
        }
        if (CT) stact(CT + ((size_t)h * cN + c * N + n) * P + p, v);
    }
}

// the fp32 pre-split alone (no CT), four consecutive n per thread, 32-bit index arithmetic:
// the per-call cost of the readout's weight split (5.4 -> ~2 us at config 2)
__global__ void k_readout_split4(const float4* __restrict__ C, float4* __restrict__ Cp, float4* __restrict__ Cp_lo,
                                 int H, int nc, int P, int N) {
    asm volatile("griddepcontrol.launch_dependents;");   // the GEMM after it may start its prologue
    const int N4 = N >> 2;
    const int total = H * nc * P * N4;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int n4 = i % N4, row = i / N4;   // row = (h * nc + c) * P + p
    const int p = row % P, hc = row / P;
    const int c = hc % nc, h = hc / nc;
    float4 v = __ldg(C + i);
    if (c == 1) v = make_float4(-v.x, -v.y, -v.z, -v.w);
    const float4 vh = make_float4(__uint_as_float(tc::tf32_rna(v.x)), __uint_as_float(tc::tf32_rna(v.y)),
                                  __uint_as_float(tc::tf32_rna(v.z)), __uint_as_float(tc::tf32_rna(v.w)));
    const int o = ((h * P + p) * nc + c) * N4 + n4;   // Cp[h][p][c * N + n]
    Cp[o] = vh;
    Cp_lo[o] = make_float4(v.x - vh.x, v.y - vh.y, v.z - vh.z, v.w - vh.w);
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
// fp32 with P <= 128: the weights come pre-split (Cp_lo, k_readout_weights) and the GEMM splits
// only the states (k_gemm_tc BPRE, three stages)
template <typename T>
pdssm_status readout_tc(const Geo& g, const T* hseq, const T* Cp, T* y, cudaStream_t st, const float* Cp_lo = nullptr) {
    const int64_t cN = g.nc * g.N;
    const bool pre = std::is_same<T, float>::value && Cp_lo != nullptr && g.P <= 128;
    // pre-split fp32: 64-column tiles with four stages keep more of the states in flight
    const bool narrow = pre && g.P % 64 == 0 && getenv("PDSSM_READOUT_NARROW");
    const int bn = narrow ? 64 : (int)(g.P < 256 ? g.P : 256);
    CUtensorMap mA, mB, mBl;
    const int64_t da[3] = {cN, g.L, g.S};
    const int64_t sa[2] = {cN * (int64_t)sizeof(T), g.L * cN * (int64_t)sizeof(T)};
    if (!make_map3(&mA, hseq, sizeof(T), da, sa, tc::BM, 1) || !make_kmajor_map(&mB, Cp, sizeof(T), cN, g.H * g.P, bn) ||
        (pre && !make_kmajor_map(&mBl, Cp_lo, sizeof(T), cN, g.H * g.P, bn)))
        return fail(PDSSM_ERR_CUDA, "readout_tc: cuTensorMapEncodeTiled failed");
    // fp32 pre-split with bn = P <= 128: 256-row tiles sharing each weight slab (MT = 2)
    // (opt-in: measured 113 vs 107 us at config 2 with the shared-tile stores: the two-stage ring
    // it leaves room for costs more than the halved weight traffic saves)
    const bool mt2 = pre && !narrow && bn <= 128 && getenv("PDSSM_READOUT_MT2");
    const int tiles = (int)ceil_div(g.L, tc::BM * (mt2 ? 2 : 1));
    dim3 grid((unsigned)(tiles * g.S), (unsigned)ceil_div(g.P, bn));
    // fp32 pre-split, bn <= 128: A (the states) from tensor memory (PDSSM_READOUT_ATM=0: from shared memory)
    const char* atm_env = getenv("PDSSM_READOUT_ATM");
    const bool atm = pre && !narrow && !mt2 && bn <= 128 && !(atm_env && atm_env[0] == '0');
    if constexpr (std::is_same<T, float>::value) {
        if (atm)
            return launch_tc_maps<T, tc::EpiReadout<T>, true, 4, 1, true>(mA, mB, cN, bn, tc::TileMap{1, tiles, (int)g.H, (int)g.P},
                                                                          grid, tc::EpiReadout<T>{y, (int)g.L, (int)g.H, (int)g.P},
                                                                          st, "readout_tc", &mBl);
        if (mt2)
            return launch_tc_maps<T, tc::EpiReadout<T>, true, 2, 2>(mA, mB, cN, bn, tc::TileMap{1, tiles, (int)g.H, (int)g.P},
                                                                    grid, tc::EpiReadout<T>{y, (int)g.L, (int)g.H, (int)g.P},
                                                                    st, "readout_tc", &mBl);
        if (pre && narrow)
            return launch_tc_maps<T, tc::EpiReadout<T>, true, 4>(mA, mB, cN, bn, tc::TileMap{1, tiles, (int)g.H, (int)g.P},
                                                                 grid, tc::EpiReadout<T>{y, (int)g.L, (int)g.H, (int)g.P},
                                                                 st, "readout_tc", &mBl);
        if (pre)
            return launch_tc_maps<T, tc::EpiReadout<T>, true>(mA, mB, cN, bn, tc::TileMap{1, tiles, (int)g.H, (int)g.P},
                                                              grid, tc::EpiReadout<T>{y, (int)g.L, (int)g.H, (int)g.P}, st,
                                                              "readout_tc", &mBl);
    }
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

// y = Re(C h) right after the scan: tensor cores when the shapes allow it, else SIMT
pdssm_status readout_run(const Geo& g, const void* hout, const float* C_opt, void* y_opt, void* wbuf, cudaStream_t st) {
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        if (tc_readout_ok(g, {hout, y_opt, wbuf})) {
            T* Cp = static_cast<T*>(wbuf);
            float* Cl = readout_lo_part(g, wbuf);
            const int64_t nw = g.H * g.nc * g.P * g.N;
            if (std::is_same<T, float>::value && Cl && g.N % 4 == 0 && !misaligned(C_opt, 16) && !misaligned(Cp, 16) &&
                !misaligned(Cl, 16) && nw / 4 < (int64_t)1 << 31) {
                k_readout_split4<<<(unsigned)ceil_div(nw / 4, 256), 256, 0, st>>>(
                    reinterpret_cast<const float4*>(C_opt), reinterpret_cast<float4*>(Cp), reinterpret_cast<float4*>(Cl),
                    (int)g.H, (int)g.nc, (int)g.P, (int)g.N);
            } else {
                k_readout_weights<T><<<(unsigned)ceil_div(nw, 256), 256, 0, st>>>(C_opt, Cp, nullptr, (int)g.H, (int)g.nc,
                                                                                   (int)g.P, (int)g.N, Cl);
            }
            pdssm_status rr = cuda_check("readout_weights");
            if (rr) return rr;
            return readout_tc<T>(g, static_cast<const T*>(hout), Cp, static_cast<T*>(y_opt), st, Cl);
        }
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            k_readout<T, NC><<<(unsigned)(g.S * g.L), 128, (size_t)NC * g.N * 4, st>>>(
                static_cast<const T*>(hout), C_opt, static_cast<T*>(y_opt), (int)g.H, (int)g.L, (int)g.N, (int)g.P);
            return cuda_check("readout");
        });
    });
}

pdssm_status prepare_e_run(const Geo& g, const void* dh, const void* dy, const float* C, float* e, void* wbuf,
                           cudaStream_t st) {
    return with_act(g.dtype, [&](auto tv) {
        using T = decltype(tv);
        return with_nc(g.nc, [&](auto ncv) {
            constexpr int NC = decltype(ncv)::value;
            return prepare_e<T, NC>(g, dh, dy, C, e, wbuf, st);
        });
    });
}


// ---------------------------------------------------------------------------
// NEXT-2 fused layer GEMM: selector logits + argmax (a2-a4), projection b = B x
// (a5) and optionally the D_t generator (R30) as ONE tcgen05 launch over the stacked weight rows
// [S | zero pad to n_sel | B | W_d]: every tile of a token block reads the same x slabs (the tiles
// of one block run concurrently on neighbouring SMs and share them through L2), the column range
// picks the epilogue (tc::EpiLayer).  fp32 weights are stacked pre-split (tf32 hi / lo, BPRE).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_stack_layer_weights(const T* __restrict__ S, const T* __restrict__ Bw, const T* __restrict__ Wd,
                                      T* __restrict__ Whi, float* __restrict__ Wlo, int H, int K, int N, int nc,
                                      int64_t d, int n_sel, int n_prj, int ns, int64_t n_tot) {
    const int64_t total = n_tot * d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / d, k = i - r * d;
        float v = 0.f;
        if (r < (int64_t)H * K) {
            v = ldact(S + r * d + k);
        } else if (r >= n_sel && r < n_sel + n_prj) {
            v = ldact(Bw + (r - n_sel) * d + k);
        } else if (r >= n_sel + n_prj) {   // D rows: tile jt holds [mag of ns states | phase of the same states]
            const int64_t q = r - n_sel - n_prj;
            const int64_t jt = q / (nc * ns), c2 = q - jt * (nc * ns);
            const int h = (int)(jt / (N / ns)), s0 = (int)(jt % (N / ns)) * ns;
            const int plane = (int)(c2 / ns), st = s0 + (int)(c2 % ns);
            v = ldact(Wd + (((int64_t)h * nc + plane) * N + st) * d + k);
        }
        if (Wlo) {
            const float vh = __uint_as_float(tc::tf32_rna(v));
            stact(Whi + i, vh);
            Wlo[i] = v - vh;
        } else {
            stact(Whi + i, v);
        }
    }
}

struct LayerTiles {
    int bn, n_sel, n_prj, n_dg, ns;
};

// the common tile width of the three ranges (0: the fused GEMM does not apply to these shapes)
inline LayerTiles layer_tiles(const Geo& g, bool with_dg) {
    LayerTiles lt{0, 0, 0, 0, 0};
    const int64_t K = g.K, cN = g.nc * g.N, l = K / gcd64(K, 16) * 16;
    const int cands_f32[] = {128};
    const int cands_bf16[] = {256, 128};
    const int* cands = g.act == 4 ? cands_f32 : cands_bf16;
    const int nc_ = g.act == 4 ? 1 : 2;
    for (int i = 0; i < nc_; ++i) {
        const int bn = cands[i];
        if (bn % l != 0 || (g.H * cN) % bn != 0 || cN % 16 != 0) continue;
        if (with_dg) {
            if (bn % g.nc != 0) continue;
            const int ns = bn / g.nc;
            if (ns % 16 != 0 || g.N % ns != 0) continue;
            lt.ns = ns;
            lt.n_dg = (int)(g.H * cN);
        }
        lt.bn = bn;
        lt.n_sel = (int)(ceil_div(g.H * K, bn) * bn);
        lt.n_prj = (int)(g.H * cN);
        return lt;
    }
    return lt;
}

pdssm_status layer_gemm(const Geo& g, const void* x, const void* S, const uint16_t* dict_idx, const void* Bw, const void* Wd,
                        const float* bias_mag, uint8_t* kstar, void* b_out, void* D_out, void* wbuf, cudaStream_t st,
                        bool* done) {
    *done = false;
    const LayerTiles lt = layer_tiles(g, Wd != nullptr);
    if (lt.bn == 0 || !tc_operands_ok(g, {x, S, Bw, Wd, b_out, D_out, wbuf}) || (Wd && g.N % 16 != 0)) return PDSSM_OK;
    const int64_t n_tot = (int64_t)lt.n_sel + lt.n_prj + lt.n_dg;
    if (n_tot > layer_w_rows(g)) return PDSSM_OK;
    return with_act(g.dtype, [&](auto tv) -> pdssm_status {
        using T = decltype(tv);
        constexpr bool F32 = std::is_same<T, float>::value;
        T* Whi = static_cast<T*>(wbuf);
        float* Wlo = F32 ? reinterpret_cast<float*>(static_cast<char*>(wbuf) + align256((size_t)layer_w_rows(g) * g.d_in * sizeof(T)))
                         : nullptr;
        const int64_t total = n_tot * g.d_in;
        k_stack_layer_weights<T><<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 4 * 148 * 8), 256, 0, st>>>(
            static_cast<const T*>(S), static_cast<const T*>(Bw), static_cast<const T*>(Wd), Whi, Wlo, (int)g.H, (int)g.K,
            (int)g.N, g.nc, g.d_in, lt.n_sel, lt.n_prj, lt.ns ? lt.ns : 1, n_tot);
        pdssm_status r = cuda_check("stack_layer_weights");
        if (r) return r;
        CUtensorMap mA, mB, mBl;
        if (!make_kmajor_map(&mA, x, sizeof(T), g.d_in, g.B * g.L, tc::BM) ||
            !make_kmajor_map(&mB, Whi, sizeof(T), g.d_in, n_tot, lt.bn) ||
            (F32 && !make_kmajor_map(&mBl, Wlo, sizeof(T), g.d_in, n_tot, lt.bn)))
            return fail(PDSSM_ERR_CUDA, "layer_gemm: cuTensorMapEncodeTiled failed");
        const int64_t M = g.B * g.L, cN = g.nc * g.N;
        tc::EpiLayer<T> epi{tc::EpiSelect{kstar, nullptr, dict_idx, nullptr, M, (int)g.L, (int)g.H, (int)g.K, (int)g.N,
                                          g.flags},
                            tc::EpiProject<T>{static_cast<T*>(b_out), M, (int)g.L, (int)g.H, (int)cN, g.H * cN},
                            tc::EpiDiag<T>{static_cast<T*>(D_out), bias_mag, M, (int)g.L, (int)g.H, (int)g.N, g.nc, lt.ns},
                            lt.n_sel, lt.n_prj};
        dim3 grid((unsigned)ceil_div(M, tc::BM), (unsigned)(n_tot / lt.bn));
        *done = true;
        if constexpr (F32) {
            // A (the token rows) from tensor memory (bn = 128): the MMAs read only the weights from shared
            // memory (PDSSM_LAYER_ATM=0: the shared-memory split)
            const char* e = getenv("PDSSM_LAYER_ATM");
            if (lt.bn <= 128 && !(e && e[0] == '0'))
                return launch_tc_maps<T, tc::EpiLayer<T>, true, 4, 1, true>(mA, mB, g.d_in, lt.bn, tc::TileMap{0, 1, 1, 0}, grid,
                                                                            epi, st, "layer_gemm", &mBl);
            return launch_tc_maps<T, tc::EpiLayer<T>, true>(mA, mB, g.d_in, lt.bn, tc::TileMap{0, 1, 1, 0}, grid, epi, st,
                                                            "layer_gemm", &mBl);
        }
        else
            return launch_tc_maps<T>(mA, mB, g.d_in, lt.bn, tc::TileMap{0, 1, 1, 0}, grid, epi, st, "layer_gemm");
    });
}

}  // namespace api
}  // namespace pdssm

PDSSM_DEFINE_ERRWORD(gemm)

extern "C" {

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
    return readout_run(g, h, C, y, ws, reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------------------
// layer-level forward: (select + projection [+ D_t generator]) -> scan (+ readout)
// ---------------------------------------------------------------------------
static pdssm_status layer_common(const void* x, const void* S, const uint16_t* dict_idx, const void* diag, const void* Wd,
                                 const float* bias_mag, const void* Bw, const float* C_opt, const float* h0_opt,
                                 uint8_t* kstar, void* h_out_opt, void* y_opt, void* chunk_state, const pdssm_dims* dims,
                                 void* ws, size_t ws_bytes, pdssm_stream_t stream) {
    Geo g;
    pdssm_status r = geo_of(dims, &g);
    if (r) return r;
    if (!x || !S || !dict_idx || !(diag || Wd) || !Bw || !kstar || !chunk_state)
        return fail(PDSSM_ERR_NULL, "layer_fwd: x, S, dict_idx, diag (or Wd), Bw, kstar, chunk_state are required");
    if (g.d_in < 1) return fail(PDSSM_ERR_SHAPE, "layer_fwd: d_in must be >= 1");
    if (Wd && g.diag_mode != PDSSM_DIAG_PER_STEP) return fail(PDSSM_ERR_DTYPE, "layer_fwd_gen: generated D_t is PER_STEP");
    const size_t need = ws_bytes_g(g, PDSSM_OP_LAYER);
    if (!ws || ws_bytes < need) return fail(PDSSM_ERR_WORKSPACE, "layer_fwd: workspace too small (need %zu)", need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    char* b = static_cast<char*>(ws);                   // b_t [B][H][L][c][N] act
    char* D = b + seq_act_bytes(g);                      // generated D_t (layer_fwd_gen)
    char* W = D + seq_act_bytes(g);                      // stacked weights of the fused GEMM
    char* rest = W + layer_w_bytes(g);
    const size_t rest_bytes = ws_bytes - (size_t)(rest - static_cast<char*>(ws));
    bool fused = false;
    if ((r = layer_gemm(g, x, S, dict_idx, Bw, Wd, bias_mag, kstar, b, Wd ? D : nullptr, W, st, &fused))) return r;
    if (!fused) {   // shapes the fused GEMM does not take: the separate launches
        if ((r = pdssm_select(x, S, dict_idx, kstar, nullptr, nullptr, dims, rest, rest_bytes, stream))) return r;
        if ((r = pdssm_project(x, Bw, b, dims, stream))) return r;
        if (Wd && (r = pdssm_diag_gen(x, Wd, bias_mag, D, dims, stream))) return r;
    }
    return pdssm_scan_fwd(kstar, dict_idx, Wd ? D : diag, b, h0_opt, C_opt, h_out_opt, y_opt, chunk_state, nullptr, dims,
                          rest, rest_bytes, stream);
}

pdssm_status pdssm_layer_fwd(const void* x, const void* S, const uint16_t* dict_idx, const void* diag, const void* Bw,
                             const float* C_opt, const float* h0_opt, uint8_t* kstar, void* h_out_opt, void* y_opt,
                             void* chunk_state, const pdssm_dims* dims, void* ws, size_t ws_bytes,
                             pdssm_stream_t stream) {
    if (!diag) return fail(PDSSM_ERR_NULL, "layer_fwd: diag is required");
    return layer_common(x, S, dict_idx, diag, nullptr, nullptr, Bw, C_opt, h0_opt, kstar, h_out_opt, y_opt, chunk_state,
                        dims, ws, ws_bytes, stream);
}

pdssm_status pdssm_layer_fwd_gen(const void* x, const void* S, const uint16_t* dict_idx, const void* Wd,
                                 const float* bias_mag_opt, const void* Bw, const float* C_opt, const float* h0_opt,
                                 uint8_t* kstar, void* h_out_opt, void* y_opt, void* chunk_state,
                                 const pdssm_dims* dims, void* ws, size_t ws_bytes, pdssm_stream_t stream) {
    if (!Wd) return fail(PDSSM_ERR_NULL, "layer_fwd_gen: Wd is required");
    return layer_common(x, S, dict_idx, nullptr, Wd, bias_mag_opt, Bw, C_opt, h0_opt, kstar, h_out_opt, y_opt,
                        chunk_state, dims, ws, ws_bytes, stream);
}

}  // extern "C"
