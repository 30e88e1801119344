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
// Tiling. One CTA (one per SM) owns 128 query rows = query blocks (2t, 2t+1):
// the tcgen05 M=128 MMA is the full-rate shape (M=64 runs at half rate). The
// CTA walks the ascending UNION of the two selections, TWO union entries (128
// keys) per tile, so every S = Q K^T MMA is N=128 (M=128, N=64 SS MMAs are
// shared-memory bound at 2/3 rate, tools/mma_rate.cu). A per-half flag zeroes
// P for a 64-key group the half did not select, so executed MMA work is at most
// two M=64 passes and about one pass when neighbouring blocks route alike.
// Phase 2 is the same loop over ceil(N/128) centroid tiles with a per-half
// column mask (the selection bitmask) and per-column weight n_j; Phase 3 is one
// more MMA, Q . H_bar, into freed S columns.
//
// Split-KV softmax. Two softmax warpgroups take alternate tiles, each with its
// own running max / sums and its own O accumulator in TMEM (O0 | O1 | S0 | S1 =
// 512 columns); the epilogue merges them. While warpgroup w handles tile u the
// tensor core runs PV_{u-1} and S_{u+1} for the other warpgroup, and because
// S_u's commit retires every earlier MMA, O_w is quiescent during the softmax
// of tile u: the lazy rescale (only when the max grows by > 2^8) needs no wait.
//
// Warp roles (512 threads, one CTA per SM). TMA throughput scales with the
// number of issuing WARPS (~24 B/clk/SM each, tools/tma_bw.cu), and a tile needs
// 64 KB per ~1000 tensor cycles, so four warps produce: one per (tensor, 64-key
// block of the tile).
//   warp 0      TMA producer K, block a (+ Q once, H_bar at the end)
//   warp 12     TMA producer K, block b
//   warp 3      builds the union list from the two selection bitmasks, then is
//               the TMA producer V, block a
//   warp 13     TMA producer V, block b
//   warp 1      tcgen05.mma issuer for warpgroup 0's tiles (elected lane issues)
//   warp 2      TMEM allocator (512 columns), then the MMA issuer for
//               warpgroup 1's tiles
//   warps 4-7   softmax warpgroup 0 (even tiles), one thread per query row
//   warps 8-11  softmax warpgroup 1 (odd tiles)
//   warps 14-15 idle (the block is 16 warps so the four producers fit)
#include "kernels.h"
#include "sm100.cuh"

#ifndef PISA_TRACE
#define PISA_TRACE 0
#endif

namespace pisa_b200 {
using namespace pisa_sm100;

namespace {

constexpr int kThreads = 512;
constexpr int kKStages = 3;  // K ring (freed early, right after S); V ring has 2
constexpr float kRescaleThresh = 8.0f;  // log2 units
constexpr int kPolyEvery = 4;           // 1 in 4 softmax exponentials via ex2_poly (FMA pipe)
// TMEM columns: O0 | O1 | S0 | S1 (128 each; O uses the first D)
__device__ __forceinline__ constexpr uint32_t colO(int w) { return uint32_t(w) * 128u; }
__device__ __forceinline__ constexpr uint32_t colS(int w) { return 256u + uint32_t(w) * 128u; }

template <int D>
struct FusedCfg {
    static constexpr int NH = D / 64;           // 64-column halves per row
    static constexpr int kQ = 128 * D * 2;      // Q tile bytes
    static constexpr int kStage = 128 * D * 2;  // one 128-key K or V stage
    static constexpr int kOffQ = 0;
    static constexpr int kOffK = kQ;
    static constexpr int kOffV = kQ + kKStages * kStage;
    static constexpr int kOffBar = kOffV + 2 * kStage;
    static constexpr int kBarBytes = 256;
    static constexpr int kOffStat = kOffBar + kBarBytes;  // [2][128][3] fp32 epilogue merge
    static constexpr int kOffMask = kOffStat + 2 * 128 * 3 * 4;
};

struct Bars {
    uint64_t q_full, h_full, qh_full;
    uint64_t k_full[kKStages], k_empty[kKStages], v_full[2], v_empty[2];
    uint64_t s_full[2], p_full[2];
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

__device__ __forceinline__ float max64(const float* x) {
    float m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        m[j] = fmaxf(fmaxf(fmaxf(x[8 * j], x[8 * j + 1]), fmaxf(x[8 * j + 2], x[8 * j + 3])),
                     fmaxf(fmaxf(x[8 * j + 4], x[8 * j + 5]), fmaxf(x[8 * j + 6], x[8 * j + 7])));
    return fmaxf(fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3])), fmaxf(fmaxf(m[4], m[5]), fmaxf(m[6], m[7])));
}

// p = 2^(x*sl2 - mm) for 64 scores, packed bf16 pairs into pk[32]; returns the sum.
// kPoly: every kPolyEvery-th exponential goes through ex2_poly (finite x only).
template <bool kPoly>
__device__ __forceinline__ float exp_pack64(const float* x, float sl2, float mm, uint32_t* pk) {
    float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 64; i += 2) {
        const float a0 = fmaf(x[i], sl2, -mm), a1 = fmaf(x[i + 1], sl2, -mm);
        const float p0 = (kPoly && (i % kPolyEvery == kPolyEvery - 1)) ? ex2_poly(a0) : ex2(a0);
        const float p1 = (kPoly && ((i + 1) % kPolyEvery == kPolyEvery - 1)) ? ex2_poly(a1) : ex2(a1);
        ps[(i >> 1) & 3] += p0 + p1;
        pk[i >> 1] = pack_bf16(p0, p1);
    }
    return (ps[0] + ps[1]) + (ps[2] + ps[3]);
}

// 32-score variant: p for 32 columns packed into pk[16]; returns the sum.
template <bool kPoly>
__device__ __forceinline__ float exp_pack32(const float* x, float sl2, float mm, uint32_t* pk) {
    float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
        const float a0 = fmaf(x[i], sl2, -mm), a1 = fmaf(x[i + 1], sl2, -mm);
        const float p0 = (kPoly && (i % kPolyEvery == kPolyEvery - 1)) ? ex2_poly(a0) : ex2(a0);
        const float p1 = (kPoly && ((i + 1) % kPolyEvery == kPolyEvery - 1)) ? ex2_poly(a1) : ex2(a1);
        ps[(i >> 1) & 3] += p0 + p1;
        pk[i >> 1] = pack_bf16(p0, p1);
    }
    return (ps[0] + ps[1]) + (ps[2] + ps[3]);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    fused_attn_kernel(const __grid_constant__ CUtensorMap tmQ,
                      const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmKb,
                      const __grid_constant__ CUtensorMap tmVh,
                      const __grid_constant__ CUtensorMap tmH, FusedArgs a) {
    using Cfg = FusedCfg<D>;
    constexpr int NH = Cfg::NH;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    Bars& bar = *reinterpret_cast<Bars*>(smem + Cfg::kOffBar);
    float* stat = reinterpret_cast<float*>(smem + Cfg::kOffStat);
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
    const bool tail = a.variant != 0;  // Zeroth, Hybrid, GlobalCentroid
    const bool first_order = a.variant == 3 || a.variant == 4;
    const int n_last = a.L - (a.N - 1) * 64;

    // ------------------------------------------------------------ setup --
    if (threadIdx.x == 0) {
        mbar_init(&bar.q_full, 1);
        mbar_init(&bar.h_full, 1);
        mbar_init(&bar.qh_full, 2);  // one commit per MMA warp
        for (int s = 0; s < kKStages; ++s) {
            mbar_init(&bar.k_full[s], 2);  // one expect_tx arrive per producer warp
            mbar_init(&bar.k_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bar.v_full[s], 2);
            mbar_init(&bar.v_empty[s], 1);
            mbar_init(&bar.s_full[s], 1);
            mbar_init(&bar.p_full[s], 4);
        }
        fence_mbar_init();
        tma_prefetch(&tmQ);
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
    }
    if (warp == 2) {
        tmem_alloc(&bar.tmem_base, 512);
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
    // Producer / MMA warpgroups (warps 0-3, 12-15) hand registers to the two
    // softmax warpgroups (warps 4-11): 2*128*64 + 2*128*184 <= 64K. Every role
    // branch starts with its warpgroup's setmaxnreg.
    const uint32_t tmem = bar.tmem_base;
    const int U = int(bar.n_union);
    const int T1 = (U + 1) >> 1;                        // exact tiles (2 union entries each)
    const int T = T1 + (tail ? (a.N + 127) / 128 : 0);  // + centroid tiles (128 centroids each)

    if (warp == 0 || warp == 3 || warp == 12 || warp == 13) {
        // ------------------------- producers: K (warps 0, 12), V (warps 3, 13) --
        regs_dec<64>();
        const bool isK = (warp == 0 || warp == 12);
        const int blk = (warp >= 12) ? 1 : 0;  // which 64-key block of the tile
        const CUtensorMap* tmx = isK ? &tmK : &tmV;
        const CUtensorMap* tmc = isK ? &tmKb : &tmVh;
        const int nst = isK ? kKStages : 2;
        uint64_t* full = isK ? bar.k_full : bar.v_full;
        uint64_t* empty = isK ? bar.k_empty : bar.v_empty;
        uint8_t* ring = smem + (isK ? Cfg::kOffK : Cfg::kOffV);
        if (warp == 0 && elect_one()) {
            mbar_expect_tx(&bar.q_full, Cfg::kQ);
#pragma unroll
            for (int half = 0; half < NH; ++half)
                tma_load_4d(smem + Cfg::kOffQ + half * 16384, &tmQ, &bar.q_full, half * 64,
                            tile * 128, h, b);
        }
        __syncwarp();
        // Stage layout (K-major B of S and MN-major B of PV alike): column half hh
        // is [128 keys][128 B] at +hh*16 KB; block blk fills keys [64 blk, 64 blk + 64).
        int s = 0, ph = 0;
        for (int u = 0; u < T; ++u) {
            mbar_wait(&empty[s], ph ^ 1);
            if (lane == 0 && blk == 0) TRACE(isK ? 11 : 12, u);
            int row;
            if (u < T1) {
                const int e = 2 * u + blk;
                row = int(ulist[e < U ? e : 2 * u] & 0x3FFFu) * 64;  // odd tail: repeat (masked)
            } else {
                row = (u - T1) * 128 + blk * 64;
            }
            if (elect_one()) {
                mbar_expect_tx(&full[s], Cfg::kStage / 2);
#pragma unroll
                for (int hh = 0; hh < NH; ++hh) {
                    uint8_t* dst = ring + s * Cfg::kStage + hh * 16384 + blk * 8192;
                    if (u < T1)
                        tma_load_4d(dst, tmx, &full[s], hh * 64, row, h, b);
                    else
                        tma_load_3d(dst, tmc, &full[s], hh * 64, row, bh);
                }
                if (blk == 0) TRACE(isK ? 0 : 1, u);
            }
            __syncwarp();
            if (++s == nst) {
                s = 0;
                ph ^= 1;
            }
        }
        if (warp == 0 && first_order) {
            // H_bar (D rows x D cols, MN-major B operand of Q.H_bar) into K stage 0,
            // once every K stage has been released.
            for (int i = 0; i < kKStages; ++i) {
                mbar_wait(&empty[s], ph ^ 1);
                if (++s == kKStages) {
                    s = 0;
                    ph ^= 1;
                }
            }
            if (elect_one()) {
                mbar_expect_tx(&bar.h_full, D * D * 2);
#pragma unroll
                for (int hh = 0; hh < NH; ++hh)
                    tma_load_3d(smem + Cfg::kOffK + hh * 16384, &tmH, &bar.h_full, hh * 64, 0, bh);
            }
            __syncwarp();
        }
    } else if (warp == 1 || warp == 2) {
        // ------------------------------------------------------------ MMA --
        // One issuing warp per softmax warpgroup (warp 1: even tiles -> S0/O0,
        // warp 2: odd tiles -> S1/O1), so one warpgroup's PV never waits behind
        // the other's S. Whole-warp loops; one elected lane issues and commits (a
        // commit tracks the MMAs of the thread that executes it).
        regs_dec<64>();
        const int w = warp - 1;
        constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);  // S = Q K^T over 128 keys
        constexpr uint32_t idPV = idesc_bf16(128, D, 0, 1);   // O += P V (V MN-major)
        const uint32_t qbase = smem_u32(smem + Cfg::kOffQ);
        mbar_wait(&bar.q_full, 0);
        for (int u = w; u < T; u += 2) {
            const int ks_ = u % kKStages;
            mbar_wait(&bar.k_full[ks_], (u / kKStages) & 1);
            tc_fence_after();
            const uint32_t kb = smem_u32(smem + Cfg::kOffK + ks_ * Cfg::kStage);
            if (elect_one()) {
                TRACE(8, u);
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t hq = (ks >> 2), kq = (ks & 3) * 32;
                    mma_ss(tmem + colS(w), sdesc_sw128(qbase + hq * 16384 + kq, 16, 1024),
                           sdesc_sw128(kb + hq * 16384 + kq, 16, 1024), idS, ks != 0);
                }
                mma_commit(&bar.k_empty[ks_]);
                mma_commit(&bar.s_full[w]);
                TRACE(2, u);
            }
            __syncwarp();
            // PV_u once this warpgroup has published P_u (S_{u+2} reuses the buffer)
            mbar_wait(&bar.p_full[w], (u >> 1) & 1);
            if (lane == 0) TRACE(9, u);
            mbar_wait(&bar.v_full[w], (u >> 1) & 1);
            if (lane == 0) TRACE(10, u);
            tc_fence_after();
            const uint32_t vb = smem_u32(smem + Cfg::kOffV + w * Cfg::kStage);
            if (elect_one()) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    mma_ts(tmem + colO(w), tmem + colS(w) + ks * 8,
                           sdesc_sw128(vb + ks * 2048, 16384, 1024), idPV,
                           (u >= 2 || ks > 0) ? 1u : 0u);
                mma_commit(&bar.v_empty[w]);
                TRACE(3, u);
            }
            __syncwarp();
        }
        if (w == 0 && first_order) {
            mbar_wait(&bar.h_full, 0);
            tc_fence_after();
        }
        const uint32_t hb = smem_u32(smem + Cfg::kOffK);
        if (elect_one()) {
            if (w == 0 && first_order) {
                // Q.H_bar into S0, after warpgroup 0's last PV has read P from it
                constexpr uint32_t idQH = idesc_bf16(128, D, 0, 1);
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t hq = (ks >> 2), kq = (ks & 3) * 32;
                    mma_ss(tmem + colS(0), sdesc_sw128(qbase + hq * 16384 + kq, 16, 1024),
                           sdesc_sw128(hb + ks * 2048, 16384, 1024), idQH, ks != 0);
                }
            }
            mma_commit(&bar.qh_full);  // both MMA warps: all their PVs (and QH) done
        }
        __syncwarp();
    } else if (warp >= 4 && warp < 12) {
        // ------------------------------------------------ softmax warpgroups --
        regs_inc<184>();
        const int wg = (warp - 4) >> 2;     // 0: even tiles, 1: odd tiles
        const int q4 = warp & 3;            // TMEM lane quadrant
        const int row = q4 * 32 + lane;     // 0..127 within the tile
        const int half = row >> 6;          // 0: block iA, 1: block iB (warp-uniform)
        const int grow = tile * 128 + row;  // query row within the sequence
        const bool active = grow < a.L;
        const bool warp_active = __all_sync(0xffffffffu, active);
        const uint32_t* hmask = half ? maskB : maskA;
        const uint32_t lane_off = uint32_t(q4 * 32) << 16;
        const uint32_t tO = tmem + lane_off + colO(wg);
        const uint32_t tS = tmem + lane_off + colS(wg);
        const float sl2 = a.scale * 1.4426950408889634f;

        float m = -INFINITY, l = 0.f, lt = 0.f;
        // Exponent shift for this tile; rescales O_wg only if the max grew by more
        // than 2^8. O_wg is quiescent here: S_u's commit retired PV_{u-2}.
        auto update_max = [&](float bm_raw) -> float {
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
                rescale_o<D>(tO, f);
                l *= f;
                lt *= f;
            }
            m = m_use;
            return (m == -INFINITY) ? 0.f : m;  // all-masked row: p = 0, not NaN
        };

        // 64 S columns [c0, c0 + 64) of this row -> x
        auto load64 = [&](uint32_t c0, float* x) {
            uint32_t r0[32], r1[32];
            tmem_ld32(tS + c0, r0);
            tmem_ld32(tS + c0 + 32, r1);
            tmem_ld_wait(r0);
            tmem_ld_wait(r1);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                x[i] = __uint_as_float(r0[i]);
                x[i + 32] = __uint_as_float(r1[i]);
            }
        };

        for (int u = wg; u < T; u += 2) {
            mbar_wait(&bar.s_full[wg], (u >> 1) & 1);
            tc_fence_after();
            if (q4 == 0) TRACE(4 + wg, u);
            uint32_t pk[32];
            float x[64];
            if (u < T1) {
                // ---- Phase 1: two exact 64-key blocks (groups g = 0, 1)
                const uint32_t ea = ulist[2 * u];
                const bool hasb = 2 * u + 1 < U;
                const uint32_t eb = hasb ? ulist[2 * u + 1] : 0u;
                const bool use[2] = {((ea >> (14 + half)) & 1u) != 0,
                                     hasb && ((eb >> (14 + half)) & 1u) != 0};  // warp-uniform
                const int nv[2] = {(int(ea & 0x3FFFu) == a.N - 1) ? n_last : 64,
                                   (int(eb & 0x3FFFu) == a.N - 1) ? n_last : 64};
                bool fast[2];
                float bm = -INFINITY;
#pragma unroll
                for (int g = 0; g < 2; ++g) {  // pass 1: masked max
                    fast[g] = warp_active && nv[g] == 64;
                    if (!use[g]) continue;
                    load64(g * 64, x);
                    if (!fast[g]) {  // ragged last key block / rows past L
#pragma unroll
                        for (int i = 0; i < 64; ++i) x[i] = (active && i < nv[g]) ? x[i] : -INFINITY;
                    }
                    bm = fmaxf(bm, max64(x));
                }
                if (use[0] || use[1]) {
                    const float mm = update_max(bm);
                    float ps = 0.f;
#pragma unroll
                    for (int g = 0; g < 2; ++g) {  // pass 2: exponentials, P over S columns
                        if (use[g]) {
                            load64(g * 64, x);
                            if (fast[g]) {
                                ps += exp_pack64<true>(x, sl2, mm, pk);
                            } else {
#pragma unroll
                                for (int i = 0; i < 64; ++i) x[i] = (active && i < nv[g]) ? x[i] : -INFINITY;
                                ps += exp_pack64<false>(x, sl2, mm, pk);
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < 32; ++i) pk[i] = 0u;
                        }
                        tmem_st32(tS + g * 32, pk);
                    }
                    l += ps;
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) pk[i] = 0u;
                    tmem_st32(tS, pk);
                    tmem_st32(tS + 32, pk);
                }
            } else {
                // ---- Phase 2: 128 centroids; column mask = own selection; weight n_j
                const int j0 = (u - T1) * 128;
                const int nvalid = min(128, a.N - j0);
                auto mask64 = [&](int g, float* xx) {
#pragma unroll
                    for (int wq = 0; wq < 2; ++wq) {
                        const int w = (j0 >> 5) + 2 * g + wq;
                        const uint32_t cm = w < a.W ? hmask[w] : 0xffffffffu;
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const int col = g * 64 + wq * 32 + i;
                            const bool ok = active && col < nvalid && !((cm >> i) & 1u);
                            xx[wq * 32 + i] = ok ? xx[wq * 32 + i] : -INFINITY;
                        }
                    }
                };
                float bm = -INFINITY;
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    load64(g * 64, x);
                    mask64(g, x);
                    bm = fmaxf(bm, max64(x));
                }
                const float mm = update_max(bm);
                const int lc = a.N - 1 - j0;  // column of the ragged last block, if in this tile
                float ps = 0.f, plast = 0.f;
#pragma unroll
                for (int c = 0; c < 4; ++c) {  // 32-column chunks
                    uint32_t r[32];
                    tmem_ld32(tS + c * 32, r);
                    tmem_ld_wait(r);
                    const int w = (j0 >> 5) + c;
                    const uint32_t cm = w < a.W ? hmask[w] : 0xffffffffu;
                    float xc[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const bool ok = active && (c * 32 + i) < nvalid && !((cm >> i) & 1u);
                        xc[i] = ok ? __uint_as_float(r[i]) : -INFINITY;
                    }
                    uint32_t pk16[16];
                    ps += exp_pack32<false>(xc, sl2, mm, pk16);
                    tmem_st16(tS + c * 16, pk16);
                    if (n_last != 64 && lc >= c * 32 && lc < c * 32 + 32) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (c * 32 + i == lc) plast = ex2(fmaf(xc[i], sl2, -mm));
                    }
                }
                l += 64.f * ps + (float(n_last) - 64.f) * plast;
                lt += ps;
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar.p_full[wg]);
            if (q4 == 0) TRACE(6 + wg, u);
        }

        // ------------------------------------------------------- epilogue --
        // Merge the two warpgroups' (m, l, lt); WG0 writes columns [0, D/2),
        // WG1 columns [D/2, D).
        stat[(wg * 128 + row) * 3 + 0] = m;
        stat[(wg * 128 + row) * 3 + 1] = l;
        stat[(wg * 128 + row) * 3 + 2] = lt;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const int o = 1 - wg;
        const float m0 = wg == 0 ? m : stat[(o * 128 + row) * 3 + 0];
        const float m1 = wg == 1 ? m : stat[(o * 128 + row) * 3 + 0];
        const float l0 = wg == 0 ? l : stat[(o * 128 + row) * 3 + 1];
        const float l1 = wg == 1 ? l : stat[(o * 128 + row) * 3 + 1];
        const float lt0 = wg == 0 ? lt : stat[(o * 128 + row) * 3 + 2];
        const float lt1 = wg == 1 ? lt : stat[(o * 128 + row) * 3 + 2];
        float M = fmaxf(m0, m1);
        float fa = (m0 == -INFINITY) ? 0.f : ex2(m0 - M);  // scale of O0
        float fb = (m1 == -INFINITY) ? 0.f : ex2(m1 - M);  // scale of O1
        float lfin = l0 * fa + l1 * fb;
        float ltfin = lt0 * fa + lt1 * fb;
        mbar_wait(&bar.qh_full, 0);
        tc_fence_after();
        float cw = 0.f;
        if (a.variant == 3) {
            cw = a.scale * ltfin;
            if (a.literal_phase3) cw *= (1.0f / 64.0f);
        }
        if (a.variant == 4 && active) {
            // slope = |U_i| exp(scale q.k_bar_global - m)   (engine.hpp:202-205)
            const uint8_t* sQ = smem + Cfg::kOffQ;
            const float* kg = a.kbar_global + size_t(bh) * D;
            float dot = 0.f;
            for (int cc = 0; cc < D; ++cc) {
                const uint32_t off = (cc >> 6) * 16384 + sw128_off(row, cc & 63);
                dot = fmaf(__bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(sQ + off)), kg[cc], dot);
            }
            const float gx = dot * sl2;
            const int nU = a.N - a.k;
            if (nU > 0) {
                const float M2 = fmaxf(M, gx);
                const float g = ex2(M - M2);
                fa *= g;
                fb *= g;
                lfin *= g;
                ltfin *= g;
                cw = a.scale * float(nU) * ex2(gx - M2);
                if (a.literal_phase3) cw *= (1.0f / 64.0f);
                M = M2;
            }
        }
        const float inv_l = 1.0f / lfin;
        bool bad = false;
        const uint32_t tb = tmem + lane_off;
        char* orow = reinterpret_cast<char*>(a.out) +
                     (size_t(b) * a.os_b + size_t(h) * a.os_h + size_t(grow) * a.os_l) *
                         (a.out_f32 ? 4 : 2);
#pragma unroll 1
        for (int cc = wg * (D / 2); cc < (wg + 1) * (D / 2); cc += 32) {
            uint32_t r0[32], r1[32], rq[32];
            tmem_ld32(tb + colO(0) + cc, r0);
            tmem_ld32(tb + colO(1) + cc, r1);
            if (first_order) tmem_ld32(tb + colS(0) + cc, rq);
            tmem_ld_wait(r0);
            tmem_ld_wait(r1);
            if (first_order) tmem_ld_wait(rq);
            float ov[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                // a warpgroup that saw no tile has f = 0 and an uninitialised O: select, not multiply
                float acc = (fa != 0.f ? __uint_as_float(r0[i]) * fa : 0.f) +
                            (fb != 0.f ? __uint_as_float(r1[i]) * fb : 0.f);
                if (first_order) acc = fmaf(cw, __uint_as_float(rq[i]), acc);
                ov[i] = acc * inv_l;
                bad |= active && !isfinite(ov[i]);
            }
            if (active) {
                if (a.out_f32) {
                    float4* dst = reinterpret_cast<float4*>(orow) + cc / 4;
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        dst[i / 4] = make_float4(ov[i], ov[i + 1], ov[i + 2], ov[i + 3]);
                } else {
                    uint4* dst = reinterpret_cast<uint4*>(orow + cc * 2);
#pragma unroll
                    for (int i = 0; i < 32; i += 8)
                        dst[i / 8] = make_uint4(pack_bf16(ov[i], ov[i + 1]), pack_bf16(ov[i + 2], ov[i + 3]),
                                                pack_bf16(ov[i + 4], ov[i + 5]), pack_bf16(ov[i + 6], ov[i + 7]));
                }
            }
        }
        if (active) {
            if (wg == 0) {
                const size_t di = size_t(bh) * a.L + grow;
                if (a.diag_m) a.diag_m[di] = M * 0.6931471805599453f;  // log2 units -> natural log
                if (a.diag_l) a.diag_l[di] = lfin;
                if (a.diag_lt) a.diag_lt[di] = ltfin;
            }
            if (bad && a.nonfinite) atomicExch(a.nonfinite, 1);
        }
    } else {
        regs_dec<64>();  // warps 14, 15: no role after setup
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, 512);
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
