/*
 * pdssm.h -- C ABI of the B200 (sm_100a) Flash PD-SSM hot path.
 *
 * Paper: "Flash PD-SSM" (arXiv 2605.19150), cited as PAPER.md:<line>.
 *
 * The library computes, per batch element b and head h, the input-dependent
 * structured-sparse recurrence (Eq. 1, with A_t = P_t D_t,
 * PAPER.md:926):
 *
 *     h_t = P_t D_t h_{t-1} + b_t,        y_t = Re(C_h h_t)
 *
 * where P_t = dict_idx[h][k*_t] is hard-selected (Eqs. 5-8)
 * and A_t acts as a COLUMN-ONE-HOT scatter:  A_t[P_t[j], j] = D_t[j], i.e.
 * (A_t v)[i] = sum_{j : P_t[j] = i} D_t[j] v[j]   (the
 * gather form of PAPER.md:938 is the transpose -- DESIGN.md reading R1).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All tensor pointers are caller-owned DEVICE memory unless stated; the
 *    library never allocates, never synchronises the host (except
 *    pdssm_check_device), and enqueues all work on the given stream, so every
 *    call is CUDA-graph capturable.  stream = NULL is the legacy default stream.
 *  - Indices are 0-based.  Every argmax breaks ties toward the smallest index
 *    and treats NaN as -inf (readings R6-R8).
 *  - Complex tensors are split re/im planes: a "[c][N]" block holds c = 1 (real)
 *    or c = 2 (re plane, then im plane) rows of N values.
 *  - Floating tensors marked "act" are in dims->dtype (PDSSM_F32 = float32,
 *    PDSSM_BF16 = bfloat16 bits); all accumulation is fp32.  Tensors marked
 *    f32 are always float32.
 *  - Validation is synchronous and happens before any CUDA call; a violation
 *    returns the status code and records a message (pdssm_last_error) without
 *    touching the device.
 *  - Kernels never trap.  Out-of-range k* / dict_idx values are a caller
 *    precondition: they are clamped into range (memory safety) and, when
 *    PDSSM_CHECK_FINITE is set, reported (with NaN/Inf inputs) through a device
 *    error word read by pdssm_check_device.
 *  - Outputs are fully overwritten.  Inputs are read-only.
 *  - Integer outputs (dict_idx, k*, P, maps) are bit-exact and run-to-run
 *    identical; float outputs are run-to-run bitwise identical (the scatter
 *    sums colliding sources in ascending source order; no float atomics).
 *  - Pointer alignment: every tensor pointer must be aligned to its element
 *    size; 16-byte alignment enables the vectorised/bulk-copy paths
 *    (otherwise PDSSM_ERR_ALIGN).
 */
#ifndef PDSSM_H
#define PDSSM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* pdssm_stream_t; /* == cudaStream_t */

typedef enum {
    PDSSM_OK = 0,
    PDSSM_ERR_NULL = 1,        /* a required pointer is NULL                        */
    PDSSM_ERR_SHAPE = 2,       /* a dimension is out of the supported range         */
    PDSSM_ERR_RANGE = 3,       /* device reported an out-of-range index (CHECK_FINITE) */
    PDSSM_ERR_ALIGN = 4,       /* a pointer is misaligned                           */
    PDSSM_ERR_DTYPE = 5,       /* unknown dtype / diag mode / flag combination      */
    PDSSM_ERR_WORKSPACE = 6,   /* workspace or chunk_state too small / NULL         */
    PDSSM_ERR_NONFINITE = 7,   /* device reported NaN/Inf input (CHECK_FINITE)      */
    PDSSM_ERR_CUDA = 8,        /* a CUDA runtime call failed (message in last_error) */
    PDSSM_ERR_UNSUPPORTED = 9  /* valid request this build does not implement       */
} pdssm_status;

typedef enum { PDSSM_F32 = 0, PDSSM_BF16 = 1 } pdssm_dtype;

/* Origin of the transition diagonal D_t (reading R3):
 *  PER_STEP: D_t given per step, diag = act [B][H][L][c][N]
 *  PER_DICT: D_t = D_k[h][k*_t], diag = f32 [H][K][c][N] ("dictionary {P_k, D_k}") */
typedef enum { PDSSM_DIAG_PER_STEP = 0, PDSSM_DIAG_PER_DICT = 1 } pdssm_diag_mode;

enum {
    PDSSM_CHECK_FINITE = 1u,   /* scan inputs for NaN/Inf and out-of-range indices   */
    PDSSM_DETERMINISTIC = 2u,  /* accepted; the library is always deterministic      */
    PDSSM_SAVE_STATES = 4u,    /* pdssm_scan_fwd must write h_out_opt (the caller keeps
                                  the states for the backward); without it h_out_opt may
                                  be NULL and pdssm_scan_bwd(h_saved = NULL, bias_opt)
                                  recomputes them from bias + the chunk carries          */
    PDSSM_EXPORT_MAPS = 8u     /* pdssm_scan_fwd also writes maps_opt                 */
};

enum { PDSSM_OP_SELECT = 0, PDSSM_OP_FWD = 1, PDSSM_OP_BWD = 2, PDSSM_OP_SEGMENT = 3, PDSSM_OP_READOUT = 4,
       PDSSM_OP_LAYER = 5, PDSSM_OP_SOFT = 6 };

/* Problem statement (north_star: x, selector S, dictionary {P_k, D_k}, B, C,
 * L, N, K, batch, heads).  Plain C struct; all fields are read-only inputs. */
typedef struct {
    int64_t batch;       /* B >= 1                                                  */
    int64_t heads;       /* H >= 1                                                  */
    int64_t len;         /* L >= 1 (time steps)                                     */
    int64_t state;       /* N, 1 <= N <= 1024 (index maps stored as uint16)         */
    int64_t dict;        /* K, 1 <= K <= 256 (k* stored as uint8)     */
    int64_t d_in;        /* selector input width (pdssm_select only)                */
    int64_t p_out;       /* readout rows P per head (0 = no readout)                */
    int32_t chunk;       /* tau >= 1, or 0 = library default (pdssm_default_chunk)  */
    int32_t is_complex;  /* c: 1 = real, 2 = complex (split re/im planes)           */
    int32_t dtype;       /* pdssm_dtype of the "act" tensors                        */
    int32_t diag_mode;   /* pdssm_diag_mode                                         */
    uint32_t flags;      /* PDSSM_CHECK_FINITE | PDSSM_EXPORT_MAPS | ...            */
    uint32_t reserved;   /* must be 0                                               */
} pdssm_dims;

/* ---------------------------------------------------------------------------
 * Sizes
 * ------------------------------------------------------------------------- */
/* tau actually used for these dims (dims->chunk, or the tuned default).  The default is
 * tau = L (one chunk per sequence) when B*H >= 0.6 x the device's SM count, N is a
 * multiple of 32 up to 128, K*N <= 8192 and L <= 16384: then the scans run one CTA per
 * (b, h) sequence (a single barrier per step, no aggregate pass); otherwise tau = 64
 * (chunked scan with decoupled look-back).  Reading R20: tau is tuning only. */
int32_t pdssm_default_chunk(const pdssm_dims* dims);

/* Bytes of device workspace `op` (PDSSM_OP_*) needs; 0 on invalid dims.
 * Workspace contents are scratch: nothing is kept between calls. */
size_t pdssm_workspace_bytes(const pdssm_dims* dims, int op);

/* Bytes of the chunk_state buffer written by pdssm_scan_fwd and read by
 * pdssm_scan_bwd.  Layout (sections 256-byte aligned, S = B*H, C = ceil(L/tau)):
 *   section 0: pi_bar  uint16 [S][C][N]     chunk aggregate index maps   (Alg. 1 A_c)
 *   section 1: d_bar   f32    [S][C][c][N]  chunk aggregate diagonals    (Alg. 1 A_c)
 *   section 2: beta_bar f32   [S][C][c][N]  chunk local-replay biases    (Alg. 1 B_c)
 *   section 3: carry   f32    [S][C][c][N]  state entering chunk c, carry_0 = h0
 *                                           (Alg. 1 Carry_c)
 * pdssm_chunk_state_offsets writes the 4 byte offsets.
 * With a single chunk (C = 1, tau >= L) on the one-CTA-per-sequence path, sections 0-2
 * (the whole-sequence aggregate) are written only under PDSSM_EXPORT_MAPS -- no later
 * chunk consumes them -- and section 3 always (carry_0 = h0). */
size_t pdssm_chunk_state_bytes(const pdssm_dims* dims);
pdssm_status pdssm_chunk_state_offsets(const pdssm_dims* dims, size_t offsets[4]);

/* ---------------------------------------------------------------------------
 * a1: dictionary sparsification (Eq. 5; App. E.2.1)
 *   M        f32    [H][K][N][N]   dense dictionary, M[h][k][i][j] (row i, column j)
 *   dict_idx uint16 [H][K][N]      out: dict_idx[h][k][j] = argmax_i M[h][k][i][j]
 * "only done once, e.g. at the beginning of the optimization step".
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_sparsify(const float* M, uint16_t* dict_idx, const pdssm_dims* dims,
                            pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * a2-a4: selection (Eqs. 6-8; App. E.2.1)
 *   x        act    [B][L][d_in]  tokens
 *   S        act    [H][K][d_in]  selector weights
 *   dict_idx uint16 [H][K][N]     sparse dictionary (needed only if P_opt)
 *   kstar    uint8  [B][H][L]     out: k* = argmax_k sum_d S[h][k][d] x[b][t][d]
 *   P_opt    uint16 [B][H][L][N]  out (optional): P_t = dict_idx[h][k*]
 *   logits_opt f32  [B][H][L][K]  out (optional): the selector logits
 * Logits are accumulated in fp32 from the act-dtype products.
 * Path: when x and S are 16-byte aligned, d_in * sizeof(act) % 16 == 0 and
 * lcm(K, 16) <= 256, the logits are a tcgen05 GEMM (bf16: kind::f16; f32:
 * 3xTF32 split, ~2^-21 relative per product) with the argmax and the P gather
 * fused into the TMEM epilogue (no workspace used, ws may be NULL); otherwise a
 * SIMT GEMM writes the logits to ws (pdssm_workspace_bytes(dims, OP_SELECT)) or
 * logits_opt, then the argmax kernel runs.  Under PDSSM_CHECK_FINITE the tensor
 * -core path reports non-finite logits, the SIMT path non-finite x.
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_select(const void* x, const void* S, const uint16_t* dict_idx,
                          uint8_t* kstar, uint16_t* P_opt, float* logits_opt,
                          const pdssm_dims* dims, void* ws, size_t ws_bytes,
                          pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * a5: input projection feeding the scan, b_t = B u_t (Eq. 1; "standard
 * matrix multiplication"), static B (reading R4), written directly in
 * the scan layout:
 *   x      act [B][L][d_in]        tokens (dims.d_in)
 *   Bw     act [H][c][N][d_in]     projection rows; plane c=0 real part, c=1 imaginary
 *   b_out  act [B][H][L][c][N]     out: b[b][h][t][c][n] = sum_d Bw[h][c][n][d] x[b][t][d]
 * Uses dims.batch, heads, len, state, is_complex, d_in, dtype.  fp32 accumulation.
 * Path: tcgen05 GEMM (bf16: kind::f16; f32: 3xTF32) when x, Bw, b_out are 16-byte
 * aligned, d_in * sizeof(act) % 16 == 0 and c*N % 16 == 0; otherwise a SIMT GEMM.
 * Errors: ERR_NULL, ERR_SHAPE (d_in < 1 or bad dims), ERR_ALIGN (element misalignment).
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_project(const void* x, const void* Bw, void* b_out, const pdssm_dims* dims,
                           pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT-2: the input-dependent diagonal D_t = D(u_t) (the form is never
 * given in the paper -- SPEC.md:367 fixes it, reading R30):
 *   D[b][h][t][n] = sigmoid((W_mag x_t)[n] + bias[h][n]) * exp(i (W_phase x_t)[n])
 * (real mode c = 1: the magnitude alone), written in the scan layout as PER_STEP diag.
 *   x        act [B][L][d_in]
 *   Wd       act [H][c][N][d_in]   plane 0 = W_mag rows, plane 1 = W_phase rows
 *   bias_opt f32 [H][N]            magnitude bias (NULL = 0)
 *   D_out    act [B][H][L][c][N]   out
 * Path: tcgen05 GEMM with the sigmoid / sincos epilogue fused (one head's c*N <= 256 columns
 * per tile; N % 16 == 0; 16-byte aligned operands); otherwise pdssm_project + an elementwise
 * kernel.  fp32 accumulation (3xTF32 for f32 operands).
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_diag_gen(const void* x, const void* Wd, const float* bias_opt, void* D_out,
                            const pdssm_dims* dims, pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT-3: the PD-SSM (soft) generator that Flash PD-SSM replaces (Eqs. 2-4):
 *   s = softmax(S u_t) (Eq. 2),  M(u_t) = sum_k s_k M_k (Eq. 3),
 *   P_t[j] = column_hardmax_i(M(u_t)[i][j]) (Eq. 4; smallest i on ties, NaN never wins)
 *   logits  f32    [B][H][L][K]   S u_t (the logits_opt of pdssm_select)
 *   M       f32    [H][K][N][N]   dense dictionary
 *   P_out   uint16 [B][H][L][N]   out
 *   ws  >= pdssm_workspace_bytes(dims, PDSSM_OP_SOFT)   (s and the transposed dictionary)
 * The mixture is a (B L) x N^2 x K GEMM per head on tcgen05 (3xTF32 for f32 dims, kind::f16
 * for bf16 dims) whose epilogue takes the column hardmax: the L N^2 mixture is never stored.
 * A comparison baseline for the hard selection of pdssm_select (the cost the paper removes).
 * Requires N % 16 == 0, N <= 256.
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_soft_select(const float* logits, const float* M, uint16_t* P_out, const pdssm_dims* dims,
                               void* ws, size_t ws_bytes, pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * a8 readout, standalone (the same kernel pdssm_scan_fwd runs for y_opt):
 * y_t = Re(C_h h_t) = C_re h_re - C_im h_im (Eq. 1 y_t = C x_t with psi = Re)
 *   h   act [B][H][L][c][N]   states (e.g. h_out of pdssm_scan_fwd)
 *   C   f32 [H][c][P][N]      readout (P = dims.p_out >= 1)
 *   y   act [B][L][H][P]      out
 *   ws  >= pdssm_workspace_bytes(dims, PDSSM_OP_READOUT): C staged in act dtype
 * Path: tcgen05 GEMM per head (bf16: kind::f16; f32: 3xTF32) when P % 16 == 0, c*N % 16
 * == 0, the row pitches are 16-byte multiples and h, y, ws are 16-byte aligned;
 * otherwise a SIMT kernel.
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_readout(const void* h, const float* C, void* y, const pdssm_dims* dims,
                           void* ws, size_t ws_bytes, pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * a6-a8: forward chunked scan (Alg. 1; Kernels A/B/C
 * PAPER.md:1020-1095) + fused readout (Eq. 1 y_t = Re(C x_t))
 *   kstar      uint8  [B][H][L]
 *   dict_idx   uint16 [H][K][N]
 *   diag       PER_STEP: act [B][H][L][c][N];  PER_DICT: f32 [H][K][c][N]
 *   bias       act    [B][H][L][c][N]   b_t (= B x_t, computed by the caller)
 *   h0_opt     f32    [B][H][c][N]      initial state (NULL = 0; reading R5)
 *   C_opt      f32    [H][c][P][N]      readout (needed iff y_opt)
 *   h_out_opt  act    [B][H][L][c][N]   out: h_t
 *   y_opt      act    [B][L][H][P]      out: y_t = Re(C_h h_t)
 *   chunk_state                          out: see pdssm_chunk_state_bytes (required)
 *   maps_opt   uint16 [B][H][C+1][N]     out (PDSSM_EXPORT_MAPS): exclusive prefix
 *              maps Pi before chunk c (maps[0] = identity) and the final map Pi_{L-1}
 * At least one of h_out_opt / y_opt must be given; PDSSM_SAVE_STATES requires h_out_opt.
 * chunk_state always holds, per (sequence, chunk c): the aggregate (pi_bar_c, d_bar_c,
 * beta_bar_c) and the carry h_{c tau - 1} (carry_0 = h0) -- the O(C N) state from which the
 * backward can recompute the chunk's states (recompute mode, pdssm_scan_bwd).
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_scan_fwd(const uint8_t* kstar, const uint16_t* dict_idx, const void* diag,
                            const void* bias, const float* h0_opt, const float* C_opt,
                            void* h_out_opt, void* y_opt, void* chunk_state, uint16_t* maps_opt,
                            const pdssm_dims* dims, void* ws, size_t ws_bytes,
                            pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * a9: backward (reverse, transposed) scan (App. C; Prop. 2
 * PAPER.md:210-223).  Real-linear split gradients packed re + i*im (reading R13):
 *   lambda_{L-1} = e_{L-1} + lam_in,  lambda_{t-1} = e_{t-1} + A_t^T lambda_t,
 *   (A_t^T mu)[j] = conj(D_t[j]) mu[P_t[j]]           (a pure gather)
 *   dbias_t = lambda_t
 *   ddiag_t[j] = conj(h_{t-1}[j]) lambda_t[P_t[j]]       (h_{-1} = h0)
 *   gsel_t = sum_j Re(conj(lambda_t[P_t[j]]) D_t[j] h_{t-1}[j])   (dl/dP_t . P_t, reading R14)
 *   dh0 = A_0^T lambda_0
 * with the direct gradient e_t = dh_t + conj(C_h)^T dy_t.
 *   kstar, dict_idx, diag, h0_opt : the SAME tensors given to pdssm_scan_fwd
 *   h_saved    act [B][H][L][c][N]  the forward states h_t, or NULL: recompute mode
 *   bias_opt   act [B][H][L][c][N]  b_t, the forward's bias (required iff h_saved is NULL).
 *              Recompute mode (the O(L N)-activation-free backward of PAPER.md:190, :280):
 *              each chunk is replayed forward from its carry in chunk_state (Alg. 1 Phase C,
 *              PAPER.md:905-913) into shared memory and h_{t-1} is read from there -- one CTA per
 *              sequence walking the chunks backwards (N % 32 == 0, N <= 128), else one CTA per
 *              (sequence, chunk); needs chunk * c * N * 4 <= ~200 KB, i.e. the forward and the
 *              backward must be called with the same (small) dims.chunk, else
 *              PDSSM_ERR_UNSUPPORTED.
 *   chunk_state                      the forward's chunk_state (reused Abar_c; carries)
 *   dh_opt     act [B][H][L][c][N]  direct state gradient (NULL = 0)
 *   dy_opt     act [B][L][H][P] with C_opt f32 [H][c][P][N] (NULL = 0)
 *   lam_in_opt f32 [B][H][c][N]     adjoint entering h_{L-1} from a later
 *                                    sequence segment (NULL = 0; sequence parallel)
 *   dbias      act [B][H][L][c][N]  out
 *   ddiag      PER_STEP act [B][H][L][c][N]; PER_DICT f32 [H][K][c][N] (summed over b,t) out
 *   gsel       f32 [B][H][L]        out (optional)
 *   dh0_opt    f32 [B][H][c][N]     out (optional)
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_scan_bwd(const uint8_t* kstar, const uint16_t* dict_idx, const void* diag,
                            const void* h_saved_opt, const void* bias_opt, const float* h0_opt,
                            const void* chunk_state,
                            const void* dh_opt, const void* dy_opt, const float* C_opt,
                            const float* lam_in_opt, void* dbias, void* ddiag, float* gsel,
                            float* dh0_opt, const pdssm_dims* dims, void* ws, size_t ws_bytes,
                            pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * Layer-level forward with the north_star argument list (x, the selector weights, the
 * dictionary {P_k, D_k}, B, C): the hot path end to end on the caller's stream,
 *   a2-a4  k*_t = argmax_k S_{h,k} . x_t        (Eqs. 6-7)  pdssm_select
 *   a5     b_t  = B x_t                         (Eq. 1)  pdssm_project
 *   a6-a8  h_t  = P_t D_t h_{t-1} + b_t,  y_t = Re(C h_t)  (Alg. 1)
 *   x         act  [B][L][d_in]       tokens (dims.d_in >= 1)
 *   S         act  [H][K][d_in]       selector weights
 *   dict_idx  uint16 [H][K][N]        sparsified dictionary maps (pdssm_sparsify)
 *   diag      PER_DICT f32 [H][K][c][N] (the dictionary's D_k) | PER_STEP act [B][H][L][c][N]
 *   Bw        act  [H][c][N][d_in]    input projection
 *   C_opt     f32  [H][c][P][N]       readout (needed iff y_opt; dims.p_out = P)
 *   h0_opt    f32  [B][H][c][N]       (NULL = 0)
 *   kstar     uint8 [B][H][L]         out: the selections (needed by the backward)
 *   h_out_opt act  [B][H][L][c][N]    out: states;   y_opt act [B][L][H][P] out
 *   chunk_state                        out (pdssm_chunk_state_bytes)
 *   ws  >= pdssm_workspace_bytes(dims, PDSSM_OP_LAYER)  (b_t plus the scan's workspace)
 * Paths (NEXT-2): when the shapes allow one common tile width (fp32: 128; bf16: 256 or 128) the
 * selector logits + argmax and the projection run as ONE tcgen05 launch over the stacked weight
 * rows [S | B] (the x slabs of a token block are read once per tile set and shared through L2;
 * fp32 weights are stacked pre-split for 3xTF32); otherwise pdssm_select + pdssm_project.
 * Errors: those of the calls it chains.
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_layer_fwd(const void* x, const void* S, const uint16_t* dict_idx, const void* diag,
                             const void* Bw, const float* C_opt, const float* h0_opt, uint8_t* kstar,
                             void* h_out_opt, void* y_opt, void* chunk_state, const pdssm_dims* dims,
                             void* ws, size_t ws_bytes, pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT-2 layer-level forward with the input-dependent diagonal generated in the same GEMM:
 *   D_t = sigmoid(W_mag x_t + bias_mag) exp(i W_phase x_t)   (reading R30)
 * fused with the selector and the projection as one tcgen05 launch (stacked rows [S | B | W_d],
 * the D range tiled per (head, block of states)), then the scan (PER_STEP) and readout.
 *   Wd        act [H][c][N][d_in]  rows W_mag (c = 0) and W_phase (c = 1)
 *   bias_mag_opt f32 [H][N]        (NULL = 0)
 *   other arguments as pdssm_layer_fwd (dims.diag_mode must be PDSSM_DIAG_PER_STEP);
 *   ws >= pdssm_workspace_bytes(dims, PDSSM_OP_LAYER).
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_layer_fwd_gen(const void* x, const void* S, const uint16_t* dict_idx, const void* Wd,
                                 const float* bias_mag_opt, const void* Bw, const float* C_opt, const float* h0_opt,
                                 uint8_t* kstar, void* h_out_opt, void* y_opt, void* chunk_state,
                                 const pdssm_dims* dims, void* ws, size_t ws_bytes, pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT-1: Prop. 2 surrogate gradients (derivation App. C
 * PAPER.md:814-841).  Slope-annealed straight-through estimation: every hardmax of
 * the forward is a tempered softmax (temperature temp > 0) in the backward
 * (PAPER.md:201-203).  Both calls consume the outputs of pdssm_scan_bwd.
 *
 * pdssm_select_grad -- selector logits gradient:
 *   dlogits[b][h][t][k] = g_t s_{k*} (delta_{k,k*} - s_k) / temp,
 *   s = softmax(logits[b][h][t][:] / temp),  g_t = gsel of pdssm_scan_bwd (reading R14)
 *   logits   f32   [B][H][L][K]   (the logits_opt of pdssm_select)
 *   kstar    uint8 [B][H][L]
 *   gsel     f32   [B][H][L]
 *   dlogits  f32   [B][H][L][K]   out
 * Errors: NULL pointer -> ERR_NULL; temp not finite or <= 0 -> ERR_RANGE.
 * One warp per (b, h, t); fp32 with expf; warp reductions in a fixed order.
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_select_grad(const float* logits, const uint8_t* kstar, const float* gsel, float temp,
                               float* dlogits, const pdssm_dims* dims, pdssm_stream_t stream);

/* pdssm_dict_grad -- dense dictionary gradient:
 *   G[h][k][i][j]  = sum_{b,t: k*[b][h][t] = k} Re(conj(lambda_t[i]) (D_t h_{t-1})[j])   (h_{-1} = h0)
 *   dM[h][k][:][j] = (diag(sigma_j) - sigma_j sigma_j^T) / temp  G[h][k][:][j],
 *   sigma_j = softmax(M[h][k][:][j] / temp)   (column-wise, the column hardmax of Eq. 5)
 *   M        f32   [H][K][N][N]   the dense dictionary given to pdssm_sparsify
 *   kstar    uint8 [B][H][L]
 *   diag     PER_STEP act [B][H][L][c][N] | PER_DICT f32 [H][K][c][N]  (as in the scan)
 *   h_saved  act   [B][H][L][c][N]  forward states;  h0_opt f32 [B][H][c][N] (NULL = 0)
 *   dbias    act   [B][H][L][c][N]  lambda_t = dbias of pdssm_scan_bwd
 *   dM       f32   [H][K][N][N]   out;   G_opt f32 [H][K][N][N] out (optional)
 * Requires N <= 128 (ERR_UNSUPPORTED otherwise).  N = 128: tcgen05 kind::tf32 3xTF32
 * grouped GEMM (one CTA per (h, k), fp32 accumulator in TMEM); other N: SIMT.  Steps are
 * accumulated in ascending (b, t) order: results are run-to-run bitwise identical.
 * ------------------------------------------------------------------------- */
pdssm_status pdssm_dict_grad(const float* M, const uint8_t* kstar, const void* diag, const void* h_saved,
                             const float* h0_opt, const void* dbias, float temp, float* dM, float* G_opt,
                             const pdssm_dims* dims, pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * Sequence parallelism (the chunk algebra lifted to per-rank segments; the
 * associativity of PAPER.md:927-932).  A summary of a segment is, per (b,h):
 *   pi uint16[N] (padded to an even count), d f32[c][N], beta f32[c][N]
 * stored contiguously as pdssm_summary_bytes(dims) bytes per (b,h) in the
 * order [B][H] { pi, d, beta }.
 * ------------------------------------------------------------------------- */
size_t pdssm_summary_bytes(const pdssm_dims* dims);

/* forward summary (pi, d, beta) of the segment described by dims (len = the
 * segment length): its Phase-A aggregate from identity / zero state. */
pdssm_status pdssm_segment_summary(const uint8_t* kstar, const uint16_t* dict_idx,
                                   const void* diag, const void* bias, void* summary_out,
                                   const pdssm_dims* dims, void* ws, size_t ws_bytes,
                                   pdssm_stream_t stream);

/* Compose the first `rank` of G gathered summaries ([G][B][H] blocks, rank
 * order) onto h0: carry_out = S_{rank-1} o ... o S_0 (h0) (f32 [B][H][c][N]);
 * map_out_opt uint16 [B][H][N] = composed index map.  Deterministic order. */
pdssm_status pdssm_compose_carry(const void* summaries, int32_t rank, int32_t G,
                                 const float* h0_opt, float* carry_out, uint16_t* map_out_opt,
                                 const pdssm_dims* dims, pdssm_stream_t stream);

/* Backward summary of a segment: beta'_seg = A_{s}^T lambda_loc_{s} (the adjoint
 * the segment sends to the state before it, from zero incoming adjoint),
 * f32 [B][H][c][N].  Needs the segment's forward chunk_state. */
pdssm_status pdssm_segment_summary_bwd(const uint8_t* kstar, const uint16_t* dict_idx,
                                       const void* diag, const void* chunk_state,
                                       const void* dh_opt, const void* dy_opt, const float* C_opt,
                                       float* beta_out, const pdssm_dims* dims, void* ws,
                                       size_t ws_bytes, pdssm_stream_t stream);

/* Adjoint entering segment `rank` from the segments after it:
 * mu = sum over g > rank of (Abar_{rank+1}^T ... Abar_{g-1}^T) beta'_g, where
 * fwd_summaries are the gathered FORWARD summaries (their (pi, d) = Abar_g)
 * and beta_bwd the gathered backward summaries f32 [G][B][H][c][N]. */
pdssm_status pdssm_compose_lambda(const void* fwd_summaries, const float* beta_bwd, int32_t rank,
                                  int32_t G, float* lam_out, const pdssm_dims* dims,
                                  pdssm_stream_t stream);

/* ---------------------------------------------------------------------------
 * Diagnostics
 * ------------------------------------------------------------------------- */
const char* pdssm_status_string(pdssm_status s);
const char* pdssm_last_error(void);           /* thread-local message of the last failure */
const char* pdssm_version(void);
/* Synchronises `stream`, reads and clears the device error word set under
 * PDSSM_CHECK_FINITE: PDSSM_ERR_RANGE / PDSSM_ERR_NONFINITE / PDSSM_OK. */
pdssm_status pdssm_check_device(pdssm_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* PDSSM_H */
