// K3: fused piecewise attention -- Algorithm 1 of the paper as
// implemented by pisa_streaming_impl (engine.hpp:232-370), in ONE kernel:
//
//   Phase 1  exact online softmax over the selected key blocks S_i
//            (attend_block_row, attention.hpp:66-91)
//   Phase 2  zeroth-order tail: centroid "keys" k_bar_j with value sums v_hat_j
//            over the complement U_i, denominator weight n_j (= B) per centroid,
//            ell_tail += p (engine.hpp:297-329)
//   Phase 3  O = (acc + scale * ell_tail * (q . H_bar)) / ell   (engine.hpp:335-358)
//
// Tiling. One CTA owns 128 query rows = query blocks (2t, 2t+1), because the
// tcgen05 M=128 MMA is the full-rate shape (M=64 runs at half rate). The CTA
// walks the ascending UNION of the two selections; a per-half flag masks the
// block for the half that did not select it (its P rows are zero). Since
// |union| <= 2k this never does more MMA work than two M=64 passes, and with
// correlated neighbours (real DiT activations, clustered data) |union| ~ k.
// Phase 2 is the same loop over ceil(N/64) centroid tiles, with a per-half
// column mask (the selection bitmask) and per-column weight n_j. Phase 3 is one
// more MMA, Q . H_bar, into the S columns of TMEM.
//
// Warp roles (256 threads, two CTAs per SM so one CTA's softmax overlaps the
// other's MMAs):
//   warp 0     TMA producer for Q (once), K / k_bar tiles (2-stage ring), H_bar
//   warp 1     single-thread tcgen05.mma issuer: S_t = Q K_t^T (SS, K-major),
//              O += P_{t-1} V_{t-1} (TS: P from TMEM, V MN-major), Q H_bar
//   warp 2     TMEM allocator (256 columns: O | S0 | S1), then TMA producer for
//              the second 64-column half of every V / v_hat tile
//   warp 3     builds the union list from the two selection bitmasks, then is
//              the TMA producer for the first half of every V / v_hat tile
//              (a TMA issue stream runs at ~32 B/clk, so two streams halve the
//              latency of the V loads on the critical path; tools/tma_bw.cu)
//   warps 4-7  softmax / correction / epilogue, one thread per query row
//              (TMEM lane), exp2 with log2(e)*scale folded into one FFMA, lazy
//              rescale of O (only when the running max grows by > 2^8), P
//              written back to TMEM as bf16 over the S columns it came from.
#include "kernels.h"
#include "sm100.cuh"

#ifndef PISA_TRACE
#define PISA_TRACE 0
#endif

namespace pisa_b200 {
using namespace pisa_sm100;

namespace {

constexpr int kThreads = 256;
constexpr float kRescaleThresh = 8.0f;  // log2 units
// Fraction of softmax exponentials computed by ex2_poly on the FMA pipe (FA4's
// trick for MUFU-bound softmax): 0 = all on MUFU. With two CTAs sharing each
// SMSP the softmax here is issue-bound, not MUFU-bound, so it is off.
constexpr int kPolyEvery = 0;
constexpr uint32_t kColO = 0, kColS = 128;

template <int D>
struct FusedCfg {
    static constexpr int kQ = 128 * D * 2;  // Q tile bytes (2 halves of 128 rows for D=128)
    static constexpr int kKV = 64 * D * 2;  // one K or V stage
    static constexpr int kOffQ = 0;
    static constexpr int kOffK = kQ;
    static constexpr int kOffV = kQ + 2 * kKV;
    static constexpr int kOffBar = kQ + 4 * kKV;
    static constexpr int kBarBytes = 256;
    static constexpr int kOffMask = kOffBar + kBarBytes;
};

struct Bars {
    uint64_t q_full, h_full, qh_full;
    uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
    uint64_t s_full[2], p_full[2];
    uint64_t o_done;
    uint32_t tmem_base;
    uint32_t n_union;
};

#if PISA_TRACE
// Timeline of one CTA: trace[role][t] = clock64 delta from kernel start.
__device__ __forceinline__ void trace_mark(const FusedArgs& a, int role, int t, long long t0) {
    if (a.trace && blockIdx.x == a.trace_tile && blockIdx.y == 0 && t < 1024)
        a.trace[role * 1024 + t] = (unsigned long long)(clock64() - t0);
}
#define TRACE(role, t) trace_mark(a, role, t, tstart)
#else
#define TRACE(role, t) ((void)0)
#endif

// max of 64 values as a 3-level tree (FMNMX3-friendly, short dependency chain)
__device__ __forceinline__ float max64(const float* x) {
    float m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        m[j] = fmaxf(fmaxf(fmaxf(x[8 * j], x[8 * j + 1]), fmaxf(x[8 * j + 2], x[8 * j + 3])),
                     fmaxf(fmaxf(x[8 * j + 4], x[8 * j + 5]), fmaxf(x[8 * j + 6], x[8 * j + 7])));
    return fmaxf(fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3])), fmaxf(fmaxf(m[4], m[5]), fmaxf(m[6], m[7])));
}

// Writes P (bf16 pairs) over the first 32 S columns and releases the S buffer.
__device__ __forceinline__ void publish_p(uint32_t sc, const uint32_t (&pk)[32], uint64_t* bar,
                                          int lane) {
    tmem_st32(sc, pk);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
}

template <int D>
__device__ __forceinline__ void rescale_o(uint32_t tmem_o, float f) {
#pragma unroll 1
    for (int cc = 0; cc < D; cc += 32) {
        uint32_t ro[32];
        tmem_ld32(tmem_o + cc, ro);
        tmem_ld_wait(ro);
#pragma unroll
        for (int i = 0; i < 32; ++i) ro[i] = __float_as_uint(__uint_as_float(ro[i]) * f);
        tmem_st32(tmem_o + cc, ro);
    }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 2)
    fused_attn_kernel(const __grid_constant__ CUtensorMap tmQ,
                      const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmKb,
                      const __grid_constant__ CUtensorMap tmVh,
                      const __grid_constant__ CUtensorMap tmH, FusedArgs a) {
    using Cfg = FusedCfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    Bars& bar = *reinterpret_cast<Bars*>(smem + Cfg::kOffBar);
    uint32_t* maskA = reinterpret_cast<uint32_t*>(smem + Cfg::kOffMask);
    uint32_t* maskB = maskA + a.W;
    uint16_t* ulist = reinterpret_cast<uint16_t*>(maskB + a.W);
#if PISA_TRACE
    const long long tstart = clock64();
#endif

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int tile = blockIdx.x;
    const int bh = blockIdx.y;
    const int b = bh / a.H, h = bh % a.H;
    const int iA = 2 * tile, iB = 2 * tile + 1;
    const bool hasB = iB < a.N;
    const bool tail = a.variant != 0;                       // Zeroth, Hybrid, GlobalCentroid
    const bool first_order = a.variant == 3 || a.variant == 4;
    const int n_last = a.L - (a.N - 1) * 64;

    // ------------------------------------------------------------ setup --
    if (threadIdx.x == 0) {
        mbar_init(&bar.q_full, 1);
        mbar_init(&bar.h_full, 1);
        mbar_init(&bar.qh_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bar.k_full[s], 1);
            mbar_init(&bar.k_empty[s], 1);
            mbar_init(&bar.v_full[s], D / 64);  // one arrive per V producer (one per 64-col half)
            mbar_init(&bar.v_empty[s], 1);
            mbar_init(&bar.s_full[s], 1);
            mbar_init(&bar.p_full[s], 4);
        }
        mbar_init(&bar.o_done, 1);
        fence_mbar_init();
        tma_prefetch(&tmQ);
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
    }
    if (warp == 2) {
        tmem_alloc(&bar.tmem_base, 256);
        tmem_relinquish();
    }
    if (warp == 3) {
        // selection bitmasks of the two query blocks -> ascending union with flags
        const uint32_t* mA = a.mask + (size_t(bh) * a.N + iA) * a.W;
        const uint32_t* mB = a.mask + (size_t(bh) * a.N + iB) * a.W;
        uint32_t base = 0;
        for (int w0 = 0; w0 < a.W; w0 += 32) {
            const int w = w0 + lane;
            const uint32_t wa = w < a.W ? mA[w] : 0u;
            const uint32_t wb = (w < a.W && hasB) ? mB[w] : 0u;
            if (w < a.W) {
                maskA[w] = wa;
                maskB[w] = hasB ? wb : 0xffffffffu;
            }
            uint32_t bits = wa | wb;
            const uint32_t cnt = __popc(bits);
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            uint32_t pos = base + incl - cnt;
            while (bits) {
                const int bit = __ffs(bits) - 1;
                bits &= bits - 1;
                const uint32_t j = uint32_t(w * 32 + bit);
                ulist[pos++] = uint16_t(j | (((wa >> bit) & 1u) << 14) | (((wb >> bit) & 1u) << 15));
            }
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) bar.n_union = base;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar.tmem_base;
    const int U = int(bar.n_union);
    const int T = U + (tail ? a.nchunk2 : 0);  // key tiles: union blocks, then centroid tiles

    if (warp == 0) {
        // ------------------------------------------------ producer: Q, K, H --
        uint8_t* sQ = smem + Cfg::kOffQ;
        if (elect_one()) {
            mbar_expect_tx(&bar.q_full, Cfg::kQ);
#pragma unroll
            for (int half = 0; half < D / 64; ++half)
                tma_load_4d(sQ + half * 16384, &tmQ, &bar.q_full, half * 64, tile * 128, h, b);
        }
        __syncwarp();
        for (int t = 0; t < T; ++t) {
            const int s = t & 1;
            uint8_t* sK = smem + Cfg::kOffK + s * Cfg::kKV;
            mbar_wait(&bar.k_empty[s], ((t >> 1) & 1) ^ 1);
            const bool exact = t < U;
            const int row = exact ? int(ulist[t] & 0x3FFFu) * 64 : (t - U) * 64;
            if (elect_one()) {
                mbar_expect_tx(&bar.k_full[s], Cfg::kKV);
#pragma unroll
                for (int half = 0; half < D / 64; ++half) {
                    if (exact)
                        tma_load_4d(sK + half * 8192, &tmK, &bar.k_full[s], half * 64, row, h, b);
                    else
                        tma_load_3d(sK + half * 8192, &tmKb, &bar.k_full[s], half * 64, row, bh);
                }
                TRACE(0, t);
            }
            __syncwarp();
        }
        if (first_order) {
            // H_bar (D rows) into the K ring: half c lands in K stage c.
            for (int t = T; t < T + 2; ++t) mbar_wait(&bar.k_empty[t & 1], ((t >> 1) & 1) ^ 1);
            if (elect_one()) {
                mbar_expect_tx(&bar.h_full, D * D * 2);
#pragma unroll
                for (int half = 0; half < D / 64; ++half)
                    tma_load_3d(smem + Cfg::kOffK + half * Cfg::kKV, &tmH, &bar.h_full, half * 64, 0, bh);
            }
            __syncwarp();
        }
    } else if (warp == 3 || (warp == 2 && D == 128)) {
        // -------------------------------------------- producers: V halves --
        // Each 64-column half of a V tile has its own issuing warp (two TMA
        // issue streams; V is on the critical path: V_t can only load once
        // PV_{t-2} has retired).
        const int vh = (warp == 3) ? 0 : 1;
        for (int t = 0; t < T; ++t) {
            const int s = t & 1;
            uint8_t* sV = smem + Cfg::kOffV + s * Cfg::kKV + vh * 8192;
            mbar_wait(&bar.v_empty[s], ((t >> 1) & 1) ^ 1);
            const bool exact = t < U;
            const int row = exact ? int(ulist[t] & 0x3FFFu) * 64 : (t - U) * 64;
            if (elect_one()) {
                mbar_expect_tx(&bar.v_full[s], 8192);
                if (exact)
                    tma_load_4d(sV, &tmV, &bar.v_full[s], vh * 64, row, h, b);
                else
                    tma_load_3d(sV, &tmVh, &bar.v_full[s], vh * 64, row, bh);
                if (vh == 0) TRACE(1, t);
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA --
        // Whole-warp loop, one elected lane issues (and commits: a commit
        // tracks the MMAs of the thread that executes it).
        constexpr uint32_t idS = idesc_bf16(128, 64, 0, 0);   // S = Q K^T
        constexpr uint32_t idPV = idesc_bf16(128, D, 0, 1);   // O += P V (V MN-major)
        constexpr uint32_t idQH = idesc_bf16(128, D, 0, 1);   // Q H_bar
        const uint32_t qbase = smem_u32(smem + Cfg::kOffQ);
        auto issue_pv = [&](int u) {
            const int s = u & 1;
            const uint32_t ph = (u >> 1) & 1;
            mbar_wait(&bar.p_full[s], ph);
            mbar_wait(&bar.v_full[s], ph);
            tc_fence_after();
            const uint32_t vb = smem_u32(smem + Cfg::kOffV + s * Cfg::kKV);
            if (elect_one()) {
                TRACE(10, u);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    mma_ts(tmem + kColO, tmem + kColS + s * 64 + ks * 8,
                           sdesc_sw128(vb + ks * 2048, 8192, 1024), idPV, (u | ks) != 0);
                mma_commit(&bar.v_empty[s]);
                mma_commit(&bar.o_done);
                TRACE(3, u);
            }
            __syncwarp();
        };
        mbar_wait(&bar.q_full, 0);
        for (int t = 0; t < T; ++t) {
            const int s = t & 1;
            mbar_wait(&bar.k_full[s], (t >> 1) & 1);
            tc_fence_after();
            const uint32_t kb = smem_u32(smem + Cfg::kOffK + s * Cfg::kKV);
            if (elect_one()) {
                TRACE(8, t);
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t hq = (ks >> 2), kq = (ks & 3) * 32;
                    mma_ss(tmem + kColS + s * 64,
                           sdesc_sw128(qbase + hq * 16384 + kq, 16, 1024),
                           sdesc_sw128(kb + hq * 8192 + kq, 16, 1024), idS, ks != 0);
                }
                mma_commit(&bar.k_empty[s]);
                mma_commit(&bar.s_full[s]);
                TRACE(2, t);
            }
            __syncwarp();
            if (t > 0) issue_pv(t - 1);
        }
        issue_pv(T - 1);
        if (first_order) {
            mbar_wait(&bar.h_full, 0);
            tc_fence_after();
        }
        const uint32_t hb = smem_u32(smem + Cfg::kOffK);
        if (elect_one()) {
            if (first_order) {
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t hq = (ks >> 2), kq = (ks & 3) * 32;
                    mma_ss(tmem + kColS, sdesc_sw128(qbase + hq * 16384 + kq, 16, 1024),
                           sdesc_sw128(hb + ks * 2048, Cfg::kKV, 1024), idQH, ks != 0);
                }
            }
            mma_commit(&bar.qh_full);  // also: every PV done
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ------------------------------------------------ softmax warpgroup --
        const int q4 = warp & 3;            // TMEM lane quadrant
        const int row = q4 * 32 + lane;     // 0..127 within the tile
        const int half = row >> 6;          // 0: block iA, 1: block iB (warp-uniform)
        const int grow = tile * 128 + row;  // query row within the sequence
        const bool active = grow < a.L;
        const bool warp_active = __all_sync(0xffffffffu, active);
        const uint32_t* hmask = half ? maskB : maskA;
        const uint32_t lane_off = uint32_t(q4 * 32) << 16;
        const float sl2 = a.scale * 1.4426950408889634f;

        float m = -INFINITY, l = 0.f, lt = 0.f;
        // Online-softmax step shared by both phases. x: raw scores (masked = -inf).
        // Returns the shift to exponentiate against; rescales O when needed.
        auto update_max = [&](float bm_raw, int t) -> float {
            const float bm = bm_raw * sl2;
            float m_use = m;
            bool resc = false;
            if (bm > -INFINITY) {
                if (m == -INFINITY) {
                    m_use = bm;
                } else if (bm > m + kRescaleThresh) {
                    m_use = bm;
                    resc = true;
                }
            }
            if (__any_sync(0xffffffffu, resc)) {
                const float f = resc ? ex2(m - m_use) : 1.f;
                mbar_wait(&bar.o_done, (t - 1) & 1);  // PV_{t-1} done (t >= 1 whenever resc)
                tc_fence_after();
                rescale_o<D>(tmem + lane_off + kColO, f);
                l *= f;
                lt *= f;
            }
            m = m_use;
            return (m == -INFINITY) ? 0.f : m;  // all-masked row: p = 0, not NaN
        };

        // ---- Phase 1: exact blocks of the union
        for (int t = 0; t < U; ++t) {
            const int s = t & 1;
            const uint32_t sc = tmem + lane_off + kColS + s * 64;
            const uint32_t e = ulist[t];
            const bool use = ((e >> (14 + half)) & 1u) != 0;  // warp-uniform
            const int nvalid = (int(e & 0x3FFFu) == a.N - 1) ? n_last : 64;
            mbar_wait(&bar.s_full[s], (t >> 1) & 1);
            tc_fence_after();
            TRACE(4 + (q4 >> 1), t);
            uint32_t pk[32];
            if (use) {
                uint32_t ra[32], rb[32];
                tmem_ld32(sc, ra);
                tmem_ld32(sc + 32, rb);
                tmem_ld_wait(ra);
                tmem_ld_wait(rb);
                float x[64];
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    x[i] = __uint_as_float(ra[i]);
                    x[i + 32] = __uint_as_float(rb[i]);
                }
                const bool full_tile = warp_active && nvalid == 64;
                if (!full_tile) {  // ragged last key block / rows past L
#pragma unroll
                    for (int i = 0; i < 64; ++i) x[i] = (active && i < nvalid) ? x[i] : -INFINITY;
                }
                const float mm = update_max(max64(x), t);
                float ps[4] = {0.f, 0.f, 0.f, 0.f};
                if (kPolyEvery > 0 && full_tile) {
                    // every kPolyEvery-th exponential on the FMA pipe, the rest on MUFU
#pragma unroll
                    for (int i = 0; i < 64; i += 2) {
                        const float a0 = fmaf(x[i], sl2, -mm), a1 = fmaf(x[i + 1], sl2, -mm);
                        const float p0 = (kPolyEvery > 0 && i % kPolyEvery == kPolyEvery - 1) ? ex2_poly(a0) : ex2(a0);
                        const float p1 = (kPolyEvery > 0 && (i + 1) % kPolyEvery == kPolyEvery - 1) ? ex2_poly(a1) : ex2(a1);
                        ps[(i >> 1) & 3] += p0 + p1;
                        pk[i >> 1] = pack_bf16(p0, p1);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 64; i += 2) {
                        const float p0 = ex2(fmaf(x[i], sl2, -mm));
                        const float p1 = ex2(fmaf(x[i + 1], sl2, -mm));
                        ps[(i >> 1) & 3] += p0 + p1;
                        pk[i >> 1] = pack_bf16(p0, p1);
                    }
                }
                l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) pk[i] = 0u;
            }
            publish_p(sc, pk, &bar.p_full[s], lane);
            TRACE(6 + (q4 >> 1), t);
        }
        // ---- Phase 2: centroid tiles, column mask = own selection, weight n_j
        for (int t = U; t < T; ++t) {
            const int s = t & 1;
            const uint32_t sc = tmem + lane_off + kColS + s * 64;
            const int c = t - U;
            const uint32_t cm_lo = hmask[2 * c];
            const uint32_t cm_hi = (2 * c + 1 < a.W) ? hmask[2 * c + 1] : 0xffffffffu;
            const int nvalid = min(64, a.N - c * 64);
            const bool has_last = (c == a.nchunk2 - 1) && n_last != 64;
            mbar_wait(&bar.s_full[s], (t >> 1) & 1);
            tc_fence_after();
            uint32_t ra[32], rb[32];
            tmem_ld32(sc, ra);
            tmem_ld32(sc + 32, rb);
            tmem_ld_wait(ra);
            tmem_ld_wait(rb);
            float x[64];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const bool ok_lo = active && i < nvalid && !((cm_lo >> i) & 1u);
                const bool ok_hi = active && i + 32 < nvalid && !((cm_hi >> i) & 1u);
                x[i] = ok_lo ? __uint_as_float(ra[i]) : -INFINITY;
                x[i + 32] = ok_hi ? __uint_as_float(rb[i]) : -INFINITY;
            }
            const float mm = update_max(max64(x), t);
            uint32_t pk[32];
            float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
                const float p0 = ex2(fmaf(x[i], sl2, -mm));
                const float p1 = ex2(fmaf(x[i + 1], sl2, -mm));
                ps0 += p0;
                ps1 += p1;
                pk[i >> 1] = pack_bf16(p0, p1);
            }
            const float ps = ps0 + ps1;
            float pw = 64.f * ps;
            if (has_last) {  // the ragged last block weighs n_last, not 64
                const int lc = a.N - 1 - c * 64;
                float plast = 0.f;
#pragma unroll
                for (int i = 0; i < 64; ++i)
                    if (i == lc) plast = ex2(fmaf(x[i], sl2, -mm));
                pw += (float(n_last) - 64.f) * plast;
            }
            l += pw;
            lt += ps;
            publish_p(sc, pk, &bar.p_full[s], lane);
        }

        // ------------------------------------------------------- epilogue --
        mbar_wait(&bar.qh_full, 0);
        tc_fence_after();
        float cw = 0.f;
        float lfin = l;
        if (a.variant == 3) {
            cw = a.scale * lt;
            if (a.literal_phase3) cw *= (1.0f / 64.0f);
        }
        float fo = 1.f;  // extra scale on O and l (GlobalCentroid shift)
        if (a.variant == 4 && active) {
            // slope = |U_i| exp(scale q.k_bar_global - m)   (engine.hpp:202-205)
            const uint8_t* sQ = smem + Cfg::kOffQ;
            const float* kg = a.kbar_global + size_t(bh) * D;
            float dot = 0.f;
            for (int c = 0; c < D; ++c) {
                const uint32_t off = (c >> 6) * 16384 + sw128_off(row, c & 63);
                dot = fmaf(__bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(sQ + off)), kg[c], dot);
            }
            const float gx = dot * sl2;
            const int nU = a.N - a.k;
            if (nU > 0) {
                const float mm = fmaxf(m, gx);
                fo = ex2(m - mm);
                cw = a.scale * float(nU) * ex2(gx - mm);
                if (a.literal_phase3) cw *= (1.0f / 64.0f);
                m = mm;
                lfin = l * fo;
                lt *= fo;
            }
        }
        const float inv_l = 1.0f / lfin;
        bool bad = false;
        char* orow = reinterpret_cast<char*>(a.out) +
                     (size_t(b) * a.os_b + size_t(h) * a.os_h + size_t(grow) * a.os_l) *
                         (a.out_f32 ? 4 : 2);
#pragma unroll 1
        for (int cc = 0; cc < D; cc += 32) {
            uint32_t ro[32], rq[32];
            tmem_ld32(tmem + lane_off + kColO + cc, ro);
            if (first_order) tmem_ld32(tmem + lane_off + kColS + cc, rq);
            tmem_ld_wait(ro);
            if (first_order) tmem_ld_wait(rq);
            float o[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                float acc = __uint_as_float(ro[i]) * fo;
                if (first_order) acc = fmaf(cw, __uint_as_float(rq[i]), acc);
                o[i] = acc * inv_l;
                bad |= active && !isfinite(o[i]);
            }
            if (active) {
                if (a.out_f32) {
                    float4* dst = reinterpret_cast<float4*>(orow) + cc / 4;
#pragma unroll
                    for (int i = 0; i < 32; i += 4) dst[i / 4] = make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]);
                } else {
                    uint4* dst = reinterpret_cast<uint4*>(orow + cc * 2);
#pragma unroll
                    for (int i = 0; i < 32; i += 8)
                        dst[i / 8] = make_uint4(pack_bf16(o[i], o[i + 1]), pack_bf16(o[i + 2], o[i + 3]),
                                                pack_bf16(o[i + 4], o[i + 5]), pack_bf16(o[i + 6], o[i + 7]));
                }
            }
        }
        if (active) {
            const size_t di = size_t(bh) * a.L + grow;
            if (a.diag_m) a.diag_m[di] = m * 0.6931471805599453f;  // log2 units -> natural log
            if (a.diag_l) a.diag_l[di] = lfin;
            if (a.diag_lt) a.diag_lt[di] = lt;
            if (bad && a.nonfinite) atomicExch(a.nonfinite, 1);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, 256);
}

}  // namespace

size_t fused_smem_bytes(int D, int N, int W) {
    const size_t core = (D == 128) ? size_t(FusedCfg<128>::kOffMask) : size_t(FusedCfg<64>::kOffMask);
    return 1024 + core + size_t(2 * W) * 4 + size_t(N) * 2 + 16;
}

cudaError_t launch_fused(int D, const CUtensorMap& tmQ, const CUtensorMap& tmK,
                         const CUtensorMap& tmV, const CUtensorMap& tmKb,
                         const CUtensorMap& tmVh, const CUtensorMap& tmH, const FusedArgs& a,
                         int BH, cudaStream_t s) {
    const size_t smem = fused_smem_bytes(D, a.N, a.W);
    dim3 grid((a.N + 1) / 2, BH);
    if (D == 128) {
        auto k = fused_attn_kernel<128>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k<<<grid, kThreads, smem, s>>>(tmQ, tmK, tmV, tmKb, tmVh, tmH, a);
    } else {
        auto k = fused_attn_kernel<64>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k<<<grid, kThreads, smem, s>>>(tmQ, tmK, tmV, tmKb, tmVh, tmH, a);
    }
    return cudaGetLastError();
}

}  // namespace pisa_b200
