// Recompute-mode backward, one CTA per (b, h) sequence (pdssm_scan_bwd with h_saved_opt = NULL;
// reading R33): the forward states are not kept between the passes.  Walking the chunks of
// chunk_state from the last to the first, the CTA
//   F: replays chunk c forward from its carry (Alg. 1 Phase C; the column-one-hot
//      scatter as the 8-slot preimage gather of k_fwd_seq) into a shared-memory buffer of tau rows,
//   R: runs the reverse transposed scan over the chunk (App. C; k_bwd_seq's step)
//      reading h_{t-1} from that buffer (h_{s_c - 1} = carry_c, which is h0 at c = 0),
// so lambda flows across chunk boundaries in registers and no O(L N) state is read from HBM.
// A producer warp streams, group by group, the rows each phase consumes through a TMA ring:
// F groups [D_t | b_t], R groups [D_t | e_{t-1}] (D_t of a chunk is read twice; the second read of
// the chunk's 2 x tau rows is normally served by L2).  The g_t terms of the chunk are parked per
// source and summed in source order after its R phase (deterministic, off the lambda chain).
#pragma once
#include "k_scan_seq.cuh"

namespace pdssm {
namespace seq {

constexpr int RC_G = 8;   // steps per TMA group

struct RcLayout {
    size_t ring, bars, xf, xb, kb, rec, wm, prow, dk, hbuf, gp, bytes;
    int slot;
    __host__ __device__ RcLayout(int N, int K, int R, int NC, int esz, int esz_e, bool PD, int L, int tau) {
        const int row = NC * N * esz, erow = NC * N * esz_e;
        const int NW = N / 32;
        const int sv = NC == 2 ? 8 : 4;
        slot = (int)a16((size_t)(PD ? 0 : RC_G * row) + (size_t)RC_G * (row > erow ? row : erow));
        size_t o = 0;
        ring = o; o = a16(o + (size_t)R * slot);
        bars = o; o = a16(o + (size_t)(2 * R + 1) * 8);      // full[R], empty[R], table barrier
        xf = o; o = a16(o + (size_t)2 * (N + 1) * sv);       // forward exchange rows (+ zero slot)
        xb = o; o = a16(o + (size_t)2 * N * sv);             // reverse exchange rows
        kb = o; o = a16(o + (size_t)L + 2 + 15);             // k* row at its address mod 16 (stage_k)
        rec = o; o = a16(o + (size_t)K * N * 8);
        wm = o; o = a16(o + (size_t)K * NW);
        prow = o; o = a16(o + (size_t)K * N * 2);
        dk = o; o = a16(o + (PD ? (size_t)K * NC * N * 4 : 0));
        hbuf = o; o = a16(o + (size_t)tau * NC * N * 4);     // the chunk's recomputed states (f32)
        gp = o; o = a16(o + (size_t)tau * N * 4);            // the chunk's g_t terms [tau][N] (summed after it)
        bytes = o;
    }
};

struct RcArgs {
    const uint8_t* kstar;
    const uint16_t* dict_idx;
    const uint8_t* rec;       // [H][K][N][8] preimage records (k_build_seq_plan)
    const uint8_t* wm;        // [H][K][NW]
    const uint16_t* pstart;   // CSR plan (records that overflow)
    const uint16_t* psrc;
    const void* diag;         // PER_STEP act
    const float* diag_dict;   // PER_DICT f32 [H][K][NC][N]
    const void* bias;         // b_t, act
    const void* e;            // e_t, TE (or null: 0)
    const float* lam_in;
    ChunkStateView cs;        // carries [S][C][NC][N]
    void* dbias;
    void* ddiag;              // act (PER_STEP) or f32 per step (PER_DICT, reduced later)
    float* gsel;
    float* dh0;
    int H, L, N, K, R, tau, C;
    uint32_t flags;
};

template <typename T, typename TE, int NC, bool PD>
__global__ void __launch_bounds__(MAXN + 32, 1) k_bwd_seq_rc(RcArgs a) {
    using SV = typename fused::SVal<NC>::type;
    constexpr int G = RC_G;
    constexpr int SVB = (int)sizeof(SV);
    extern __shared__ __align__(128) uint8_t smem[];
    const int N = a.N, K = a.K, L = a.L, R = a.R, tau = a.tau, C = a.C;
    const int i = threadIdx.x, w = i >> 5, NW = N >> 5;
    const int s = blockIdx.x, h = s % a.H;
    const RcLayout Ly(N, K, R, NC, (int)sizeof(T), (int)sizeof(TE), PD, L, tau);
    uint8_t* ring = smem + Ly.ring;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Ly.bars);
    SV* xf = reinterpret_cast<SV*>(smem + Ly.xf);
    SV* xb = reinterpret_cast<SV*>(smem + Ly.xb);
    uint8_t* kb = smem + Ly.kb;   // (re-pointed by stage_k below)
    uint2* rec = reinterpret_cast<uint2*>(smem + Ly.rec);
    uint8_t* wm = smem + Ly.wm;
    uint16_t* prow = reinterpret_cast<uint16_t*>(smem + Ly.prow);
    float* dk = reinterpret_cast<float*>(smem + Ly.dk);
    float* hbuf = reinterpret_cast<float*>(smem + Ly.hbuf);
    float* gp = reinterpret_cast<float*>(smem + Ly.gp);   // [tau][N]
    const size_t row = (size_t)NC * N;
    const size_t seq0 = (size_t)s * L;
    const uint64_t pol = fused::policy_evict_first();
    const TE* ein = static_cast<const TE*>(a.e);
    kb = stage_k(a.kstar + seq0, K, a.flags, kb, L);   // the sequence's k* (clamped; reported under CHECK_FINITE)
    if (i == 0) {
        for (int q = 0; q < 2 * R + 1; ++q) fused::mbar_init(bars + q, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    stage_rec(a.rec + (size_t)h * K * N * CAP, rec, K * N, bars + 2 * R);
    {
        for (int x = i; x < K * NW; x += blockDim.x) wm[x] = a.wm[(size_t)h * K * NW + x];
        stage_prow(a.dict_idx + (size_t)h * K * N, prow, K * N, N);
        if constexpr (PD) stage_f32(a.diag_dict + (size_t)h * K * NC * N, dk, K * NC * N);
    }
    if (i == 0) {
        xf[N] = fused::mk<NC>(0.f, 0.f);
        xf[(N + 1) + N] = fused::mk<NC>(0.f, 0.f);
    }
    __syncthreads();
    const int ROWB = (int)(row * sizeof(T)), EROWB = (int)(row * sizeof(TE));
    const int OFF2 = PD ? 0 : G * ROWB;   // second stream of a slot: b (F) or e (R)
    // group schedule: for c = C-1 .. 0: F groups ascending over the chunk, then R groups descending.
    // Group (c, phase, q): F q-th group covers [s_c + qG, ...); R q-th group covers (e_c - qG] downwards.
    auto chunk_lo = [&](int c) { return c * tau; };
    auto chunk_hi = [&](int c) { return min((c + 1) * tau, L) - 1; };
    auto ngr = [&](int c) { return (chunk_hi(c) - chunk_lo(c) + 1 + G - 1) / G; };
    if (i >= N) {   // producer warp: one elected lane issues every group in schedule order
        if ((i & 31) == 0) {
            int gi = 0;
            for (int c = C - 1; c >= 0; --c) {
                const int lo = chunk_lo(c), hi = chunk_hi(c), ng = ngr(c);
                for (int ph = 0; ph < 2; ++ph) {
                    for (int q = 0; q < ng; ++q, ++gi) {
                        const int slot = gi % R;
                        if (gi >= R) fused::mbar_wait(bars + R + slot, (uint32_t)((gi / R) - 1) & 1u);
                        uint8_t* dst = ring + (size_t)slot * Ly.slot;
                        int t0, len;
                        if (ph == 0) { t0 = lo + q * G; len = min(G, hi - t0 + 1); }
                        else { const int th = hi - q * G; t0 = max(th - G + 1, lo); len = th - t0 + 1; }
                        uint32_t bytes = PD ? 0 : (uint32_t)(len * ROWB);
                        // F: b_t rows; R: e_{t-1} rows for t in [t0, t0 + len) with t >= 1 (row t - 1 - (t0 - 1))
                        int f_first = 0, f_cnt = 0;
                        if (ph == 0) {
                            bytes += (uint32_t)(len * ROWB);
                        } else if (ein) {
                            f_first = max(t0 - 1, 0);
                            f_cnt = max(0, t0 + len - 1 - f_first);
                            bytes += (uint32_t)(f_cnt * EROWB);
                        }
                        fused::mbar_expect_tx(bars + slot, bytes);
                        if constexpr (!PD)
                            fused::tma_1d_hint(dst, static_cast<const T*>(a.diag) + (seq0 + t0) * row, len * ROWB,
                                               bars + slot, pol);
                        if (ph == 0) {
                            fused::tma_1d_hint(dst + OFF2, static_cast<const T*>(a.bias) + (seq0 + t0) * row, len * ROWB,
                                               bars + slot, pol);
                        } else if (f_cnt > 0) {
                            const int f_off = f_first - (t0 - 1);
                            fused::tma_1d_hint(dst + OFF2 + (size_t)f_off * EROWB, ein + (seq0 + f_first) * row,
                                               f_cnt * EROWB, bars + slot, pol);
                        }
                    }
                }
            }
        }
        return;
    }
    // ---- compute threads: thread i owns state i (forward) / source i (reverse)
    fused::mbar_wait(bars + 2 * R, 0);   // the records (stage_rec)
    float lr = 0.f, li = 0.f;   // lambda_{L-1} = e_{L-1} + lam_in
    if (ein) {
        lr = ldact(ein + (seq0 + L - 1) * row + i);
        if constexpr (NC == 2) li = ldact(ein + (seq0 + L - 1) * row + N + i);
    }
    if (a.lam_in) {
        lr += a.lam_in[(size_t)s * row + i];
        if constexpr (NC == 2) li += a.lam_in[(size_t)s * row + N + i];
    }
    int gi = 0;
    int fx = 0, bx = 0;   // exchange-row parities
    for (int c = C - 1; c >= 0; --c) {
        const int lo = chunk_lo(c), hi = chunk_hi(c), ng = ngr(c);
        const size_t ci = (size_t)s * C + c;
        const float c_r = a.cs.carry[ci * row + i];
        const float c_i = NC == 2 ? a.cs.carry[ci * row + N + i] : 0.f;
        // ---------------- F: forward replay of the chunk into hbuf (the next step's operands are
        // loaded while this step's gather is in flight, within a group)
        float hr = c_r, hi_ = c_i;
        for (int q = 0; q < ng; ++q, ++gi) {
            const int slot = gi % R;
            fused::mbar_wait(bars + slot, (uint32_t)(gi / R) & 1u);
            const uint8_t* sb = ring + (size_t)slot * Ly.slot;
            const int t0 = lo + q * G, len = min(G, hi - t0 + 1);
            int k, m;
            uint2 rc;
            float Dr, Di, Br, Bi;
            auto load_f = [&](int r) {
                k = kb[t0 + r];
                rc = rec[(size_t)k * N + i];
                m = wm[k * NW + w];
                Di = 0.f;
                if constexpr (PD) {
                    Dr = dk[(size_t)k * row + i];
                    if constexpr (NC == 2) Di = dk[(size_t)k * row + N + i];
                } else {
                    const T* Dp = reinterpret_cast<const T*>(sb + r * ROWB);
                    Dr = ldact_s(Dp + i);
                    if constexpr (NC == 2) Di = ldact_s(Dp + N + i);
                }
                const T* Bp = reinterpret_cast<const T*>(sb + OFF2 + r * ROWB);
                Br = ldact_s(Bp + i);
                Bi = NC == 2 ? ldact_s(Bp + N + i) : 0.f;
            };
            load_f(0);
            for (int r = 0; r < len; ++r) {
                const int t = t0 + r;
                SV* vb = xf + fx * (N + 1);
                vb[i] = fused::mk<NC>(Dr * hr - Di * hi_, Dr * hi_ + Di * hr);
                uint32_t ga[CAP];   // shared addresses of the gather, before the barrier
                {
                    uint32_t lo4[4], hi4[4];
                    const uint32_t vb_s = fused::smem_u32(vb);
                    gather_addr4(rc.x, vb_s, SVB, lo4);
                    gather_addr4(rc.y, vb_s, SVB, hi4);
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        ga[x] = lo4[x];
                        ga[4 + x] = hi4[x];
                    }
                }
                const int kc = k, mc = m;
                const float bcr = Br, bci = Bi;
                compute_sync(N);
                if (r == 0 && i == 0 && gi >= 1) mbar_arrive(bars + R + ((gi - 1) % R));   // previous group consumed
                float ar, ai;
                if (mc == WM_OVF) {   // preimage longer than the records: CSR plan (rare, warp-uniform)
                    ar = ai = 0.f;
                    const size_t e = (size_t)h * K + kc;
                    const int st = __ldg(a.pstart + e * (N + 1) + i), en = __ldg(a.pstart + e * (N + 1) + i + 1);
                    for (int x = st; x < en; ++x) {
                        const SV v = vb[__ldg(a.psrc + e * N + x)];
                        ar += fused::re_of<NC>(v);
                        ai += fused::im_of<NC>(v);
                    }
                    if (r + 1 < len) load_f(r + 1);
                } else if (mc <= 4) {   // warp-uniform: the warp's in-degree fits 4 slots
                    float vr[4], vi[4];
#pragma unroll
                    for (int x = 0; x < 4; ++x) lds_sv<NC>(ga[x], vr[x], vi[x]);
                    if (r + 1 < len) load_f(r + 1);
                    ar = (vr[0] + vr[1]) + (vr[2] + vr[3]);
                    ai = (vi[0] + vi[1]) + (vi[2] + vi[3]);
                } else {
                    float vr[CAP], vi[CAP];
#pragma unroll
                    for (int x = 0; x < CAP; ++x) lds_sv<NC>(ga[x], vr[x], vi[x]);   // past the in-degree: zero slot
                    if (r + 1 < len) load_f(r + 1);
                    ar = ((vr[0] + vr[1]) + (vr[2] + vr[3])) + ((vr[4] + vr[5]) + (vr[6] + vr[7]));
                    ai = ((vi[0] + vi[1]) + (vi[2] + vi[3])) + ((vi[4] + vi[5]) + (vi[6] + vi[7]));
                }
                hr = ar + bcr;
                hi_ = NC == 2 ? ai + bci : 0.f;
                float* hrow = hbuf + (size_t)(t - lo) * row;
                hrow[i] = hr;
                if constexpr (NC == 2) hrow[N + i] = hi_;
                fx ^= 1;
            }
        }
        // ---------------- R: reverse scan of the chunk
        for (int q = 0; q < ng; ++q, ++gi) {
            const int slot = gi % R;
            fused::mbar_wait(bars + slot, (uint32_t)(gi / R) & 1u);
            const uint8_t* sb = ring + (size_t)slot * Ly.slot;
            const int th = hi - q * G, t0 = max(th - G + 1, lo), len = th - t0 + 1;
            for (int rr = 0; rr < len; ++rr) {
                const int t = th - rr, ro = t - t0;
                const int k = kb[t];
                const int p = prow[(size_t)k * N + i];
                float Dr, Di = 0.f;
                if constexpr (PD) {
                    Dr = dk[(size_t)k * row + i];
                    if constexpr (NC == 2) Di = dk[(size_t)k * row + N + i];
                } else {
                    const T* Dp = reinterpret_cast<const T*>(sb + ro * ROWB);
                    Dr = ldact_s(Dp + i);
                    if constexpr (NC == 2) Di = ldact_s(Dp + N + i);
                }
                float er = 0.f, ei = 0.f;   // e_{t-1}
                if (t > 0 && ein) {
                    const TE* ep = reinterpret_cast<const TE*>(sb + OFF2 + ro * EROWB);
                    er = ldact_s(ep + i);
                    if constexpr (NC == 2) ei = ldact_s(ep + N + i);
                }
                float hr0, hi0;   // h_{t-1}
                if (t > lo) {
                    const float* hrow = hbuf + (size_t)(t - 1 - lo) * row;
                    hr0 = hrow[i];
                    hi0 = NC == 2 ? hrow[N + i] : 0.f;
                } else {
                    hr0 = c_r;
                    hi0 = c_i;
                }
                const size_t off = (seq0 + t) * row + i;
                stact(static_cast<T*>(a.dbias) + off, lr);                 // db_t = lambda_t
                if constexpr (NC == 2) stact(static_cast<T*>(a.dbias) + off + N, li);
                SV* lb = xb + bx * N;
                lb[i] = fused::mk<NC>(lr, li);
                compute_sync(N);
                if (rr == 0 && i == 0) mbar_arrive(bars + R + ((gi - 1) % R));   // previous group consumed
                const SV lp = lb[p];
                const float pr = fused::re_of<NC>(lp), pm = fused::im_of<NC>(lp);
                // the chain first: lambda_{t-1} = e_{t-1} + conj(D_t) lp (the next step's exchange waits on it)
                const float lr_old = lr, li_old = li;
                if (t > 0) {
                    lr = er + Dr * pr + Di * pm;
                    li = NC == 2 ? ei + Dr * pm - Di * pr : 0.f;
                }
                const float ddr = hr0 * pr + hi0 * pm, ddi = hr0 * pm - hi0 * pr;   // dD_t = conj(h_{t-1}) lp
                if constexpr (PD) {
                    float* dd = static_cast<float*>(a.ddiag) + off;
                    dd[0] = ddr;
                    if constexpr (NC == 2) dd[N] = ddi;
                } else {
                    stact(static_cast<T*>(a.ddiag) + off, ddr);
                    if constexpr (NC == 2) stact(static_cast<T*>(a.ddiag) + off + N, ddi);
                }
                const float qr = Dr * hr0 - Di * hi0, qi = Dr * hi0 + Di * hr0;
                gp[(size_t)(t - lo) * N + i] = pr * qr + pm * qi;            // this source's term of g_t (off the chain)
                (void)lr_old;
                (void)li_old;
                if (t == 0 && a.dh0) {                                       // dh0 = A_0^T lambda_0
                    a.dh0[(size_t)s * row + i] = Dr * pr + Di * pm;
                    if constexpr (NC == 2) a.dh0[(size_t)s * row + N + i] = Dr * pm - Di * pr;
                }
                bx ^= 1;
            }
        }
        compute_sync(N);   // the chunk's g partials are complete (and hbuf is free for the next chunk)
        if (a.gsel) {   // g_t = sum over the N sources, in a fixed order (deterministic)
            for (int t = lo + i; t <= hi; t += N) {
                const float* gr = gp + (size_t)(t - lo) * N;
                float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
                for (int x = 0; x < N; x += 4) {
                    a0 += gr[x];
                    a1 += gr[x + 1];
                    a2 += gr[x + 2];
                    a3 += gr[x + 3];
                }
                a.gsel[seq0 + t] = (a0 + a1) + (a2 + a3);
            }
        }
        compute_sync(N);   // partials read before the next chunk overwrites them
    }
    if (i == 0 && gi >= 1) mbar_arrive(bars + R + ((gi - 1) % R));
}

}  // namespace seq
}  // namespace pdssm
