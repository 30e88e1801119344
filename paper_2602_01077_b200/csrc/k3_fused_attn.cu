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
// tcgen05 M=128 MMA is the full-rate shape (M=64 costs the same time). The CTA
// walks the ascending UNION of the two selections; a per-block flag masks the
// key block for the query block that did not select it (its P rows are zero),
// so executed MMA work <= two M=64 passes. Phase 2 is the same loop over
// ceil(N/64) centroid tiles with a per-block column mask (the selection bitmask)
// and per-column weight n_j. Phase 3 is one more MMA, Q . H_bar.
//
// Why this shape (tools/l2_bw.cu, tools/st_mix.cu, profiles/): the kernel
// streams a random 32 KB K tile and a 32 KB V tile from L2 per super-tile
// (~220 GB per Wan2.1-14B step, 9-10 TB/s), and a tile takes 1500-3000 cycles
// under that load, so the design spends shared memory on K/V stages:
//   * ONE CTA per SM: Q (32 KB) + 2 K + 3 V stages of two key blocks each
//     (192 KB at d = 128) in shared memory, plus the two selection bitmasks and
//     the union list; a third K stage measured no faster and no longer fits
//     beside the list;
//   * key blocks go through the pipeline in pairs ("super-tiles" of 128 keys):
//     S = Q [K_a; K_b]^T is one set of N=128 MMAs, and each barrier round trip,
//     commit and softmax hand-off covers two blocks -- a single issuing thread
//     is otherwise latency-bound on ~100 instructions per 64-key block;
//   * TMEM (512 columns): O [0, 128) | three S/P buffers of 128 columns (P_g is
//     written over the S_g columns it came from), so the chain
//     S_g -> softmax_g -> PV_g -> S_{g+3} spans three super-tiles and the
//     tensor pipe stays fed while one super-tile is in the softmax.
//     (Designs with two S buffers -- Q in TMEM, or O split per warpgroup --
//     measured 10-20 % slower: tools/k3_variants/README.md. Issuing TMA boxes
//     one per lane, which moves the first S MMA ~1.5K cycles earlier, measured
//     neutral: profiles/r02_k3_variants.log batch ay.)
//
// Warp roles (384 threads):
//   warp 0     TMA producer: Q (once), K / k_bar tiles (3-stage ring of pairs),
//              H_bar at the end
//   warp 1     single-thread tcgen05.mma issuer: S_g = Q K_g^T (SS, K-major),
//              O += P_g V_g (TS: P from TMEM, V MN-major), Q H_bar (SS)
//   warp 2     TMEM allocator, then TMA producer for V columns [0, 64)
//   warp 3     TMA producer for V columns [64, 128) (two issue streams for V)
//   warps 0-3  first (prologue): copy the two selection bitmasks and build the
//              union list together
//   warps 4-7  softmax / correction / epilogue of query block 2t   (warpgroup A)
//   warps 8-11 softmax / correction / epilogue of query block 2t+1 (warpgroup B)
// TMEM lane layout: lane q4*32 + hh*16 + r16 holds row q4*16 + r16 of query
// block 2t + hh. Warp q4 of warpgroup hh owns those 16 lanes (16x32bx2 view:
// thread t holds row t & 15, columns [32*(t >> 4), +32) of each 64-key half), so
// each block's exponentials use all four SM sub-partitions (all four MUFU
// units), and the two blocks' online softmaxes run in parallel. exp2 with
// log2(e)*scale folded into one FFMA, single pass against the running max (see
// Phase 1); lazy rescale of O (only when the running max grows by > 2^8); P
// written back to TMEM as bf16 over its S columns.
#include "kernels.h"
#include "sm100.cuh"

#ifndef PISA_TRACE
#define PISA_TRACE 0
#endif

namespace pisa_b200 {
using namespace pisa_sm100;

namespace {

constexpr int kThreads = 384;
// K stages: 2 measured as fast as 3 with the previous softmax and 1-1.5 %
// faster with the single-pass one (profiles/r02_k3_variants.log, batches l, s)
#ifndef PISA_KSTAGES
#define PISA_KSTAGES 2
#endif
#ifndef PISA_VSTAGES
#define PISA_VSTAGES 3
#endif
constexpr int kSK = PISA_KSTAGES;  // K ring stages (two key blocks each)
constexpr int kSV = PISA_VSTAGES;  // V ring stages (two key blocks each)
constexpr int kSB = 3;  // S/P TMEM buffers (128 columns each)
constexpr float kRescaleThresh = 8.0f;  // log2 units
constexpr uint32_t kColO = 0, kColS = 128;  // O | three S/P buffers (P_g over the S_g columns)
// Exponentials of the softmax: element i of each pair-unrolled 32-column row
// chunk goes to ex2_poly (FMA pipe) when bit (i % 8) of kPolyMask is set, else
// to MUFU.EX2 (FA4's split of exp2 across pipes; measured slower here: the
// softmax is issue-bound, not MUFU-bound, so the default is all-MUFU).
#ifndef PISA_POLY_MASK
#define PISA_POLY_MASK 0x00
#endif
constexpr uint32_t kPolyMask = PISA_POLY_MASK;
// Sub-tiles that BOTH query blocks of the tile selected (every Phase-1 entry
// on clustered routing, every Phase-2 centroid chunk) are exponentiated by
// both warpgroups, which share the four MUFU units (2 x 8192 ex2 per 128-key
// super-tile = 1024 MUFU cycles = the tensor time). Elements whose index bit
// is set in kPolyBoth go to the FMA pipe (ex2_poly) on those sub-tiles only.
// Measured (Wan2.1-14B, same box, 2 x interleaved, profiles/r02_ab_poly.log):
// 0x00 19.02-19.13 ms clustered / 25.31-25.39 gaussian, 0x11 19.18-19.30 /
// 25.47-25.58, 0x55 20.18-20.22 / 25.89-26.02: the softmax is not MUFU-bound
// even when both blocks use every sub-tile, so the default is off.
#ifndef PISA_POLY_BOTH
#define PISA_POLY_BOTH 0x00
#endif
constexpr uint32_t kPolyBoth = PISA_POLY_BOTH;
// The softmax warps' wait for S: spin (poll) or suspend in hardware between
// polls. Polling steals issue slots from the other warpgroup's warps on the
// same sub-partitions while one warpgroup runs ahead.
// 2: poll with a PISA_SOFTMAX_NS nanosleep between polls.
#ifndef PISA_SOFTMAX_SPIN
#define PISA_SOFTMAX_SPIN 1
#endif
#ifndef PISA_SOFTMAX_NS
#define PISA_SOFTMAX_NS 32
#endif
constexpr bool kSoftmaxSpin = PISA_SOFTMAX_SPIN != 0;
#ifndef PISA_REGS_PRODUCER
#define PISA_REGS_PRODUCER 0  // 0: no setmaxnreg
#endif
#ifndef PISA_REGS_SOFTMAX
#define PISA_REGS_SOFTMAX 208
#endif
__device__ __forceinline__ void softmax_wait(uint64_t* bar, uint32_t parity) {
#if PISA_SOFTMAX_SPIN == 2
    mbar_wait_backoff<PISA_SOFTMAX_NS>(bar, parity);
#else
    mbar_wait<kSoftmaxSpin>(bar, parity);
#endif
}
// PISA_MMA_WAIT 1: the MMA warp polls its barriers with a short nanosleep
// (instead of a pure spin that takes issue slots from the two softmax warps on
// its sub-partition). PISA_PSPLIT 1: P is published per 64-key sub-tile and
// the MMA warp issues PV of the first sub-tile while the softmax computes the
// second.
#ifndef PISA_MMA_WAIT
#define PISA_MMA_WAIT 0
#endif
#ifndef PISA_MMA_NS
#define PISA_MMA_NS 20
#endif
#ifndef PISA_PSPLIT
#define PISA_PSPLIT 0
#endif
__device__ __forceinline__ void mma_wait(uint64_t* bar, uint32_t parity) {
#if PISA_MMA_WAIT == 2
    mbar_wait<false>(bar, parity);  // hardware-suspended try_wait (time-limit hint)
#elif PISA_MMA_WAIT
    mbar_wait_backoff<PISA_MMA_NS>(bar, parity);
#else
    mbar_wait<true>(bar, parity);
#endif
}

// The MMA warp (PISA_MMA_WARP 1 or 3) and the second V producer (the other of
// the two) -- the MMA warp shares its SM sub-partition with softmax warps q4 =
// PISA_MMA_WARP of both warpgroups.
#ifndef PISA_MMA_WARP
#define PISA_MMA_WARP 1
#endif
constexpr int kMmaWarp = PISA_MMA_WARP;
constexpr int kVWarp1 = PISA_MMA_WARP == 1 ? 3 : 1;
static_assert(PISA_MMA_WARP == 1 || PISA_MMA_WARP == 3, "MMA warp");
// (An S prefetch -- the next super-tile's TMEM loads issued before P_g is
// published -- measured slower: 24.0 vs 22.9 ms gaussian, batch ag; and 16
// softmax warps, two per row set with 16 columns per thread, measured slower
// too: 23.2-23.6 vs 22.2 ms gaussian, 17.6 vs 16.2 ms clustered, batch bb.)
// PISA_SPEC_MAX 1: single-pass softmax (see Phase 1)
#ifndef PISA_SPEC_MAX
#define PISA_SPEC_MAX 1
#endif
// Phase-1 block order: the ascending union. (A balanced order -- A&B pairs,
// then (A-only, B-only) pairs -- and a grouped one measured slower: 26.5 / 25.4
// vs 24.7-25.1 ms gaussian, round 1; the per-super-tile fixed softmax cost
// penalises balancing, and scrambling the order costs the L2 reuse between
// neighbouring CTAs walking similar selections in step.)
template <uint32_t Mask>
__device__ __forceinline__ float ex2_mix(float x, int i) {
    return ((Mask >> (i & 7)) & 1u) ? ex2_poly(x) : ex2(x);
}

template <int D>
struct FusedCfg {
    static constexpr int kQ = 128 * D * 2;  // Q tile: [64-col half][128 rows], rows interleaved
    // one K or V stage: two 64-key blocks, laid out [64-col half][128 rows] with
    // 128-byte rows (SW128), so a stage is one N=128 (K) / K=128 (V) operand
    static constexpr int kKV = 2 * 64 * D * 2;
    static constexpr int kOffQ = 0;
    static constexpr int kOffK = kQ;
    static constexpr int kOffV = kQ + kSK * kKV;
    static constexpr int kOffBar = kQ + (kSK + kSV) * kKV;
    static constexpr int kBarBytes = 512;
    static constexpr int kOffMask = kOffBar + kBarBytes;
};

struct Bars {
    uint64_t q_full, h_full, qh_full;
    uint64_t k_full[kSK], v_full[kSV], v_empty[kSV];
    uint64_t s_full[kSB], p_full[kSB], p_half[kSB];
    uint32_t tmem_base;
    uint32_t n_u;     // |A u B|
    uint32_t n_w[4];  // union entries per 32-word quarter (list build)
};
static_assert(sizeof(Bars) <= 512, "barrier block");

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

// max of 32 values as a tree
__device__ __forceinline__ float max32(const float* x) {
    float m[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        m[j] = fmaxf(fmaxf(fmaxf(x[8 * j], x[8 * j + 1]), fmaxf(x[8 * j + 2], x[8 * j + 3])),
                     fmaxf(fmaxf(x[8 * j + 4], x[8 * j + 5]), fmaxf(x[8 * j + 6], x[8 * j + 7])));
    return fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
}

// Rescales this thread's half of the O columns of its row: 16x32bx2 view, the
// half-warp split is D/2 columns (thread t < 16: [0, D/2), t >= 16: [D/2, D)).
template <int D>
__device__ __forceinline__ void rescale_o(uint32_t tmem_o, float f) {
#pragma unroll 1
    for (int cc = 0; cc < D / 2; cc += 32) {
        uint32_t ro[32];
        tmem_ld16x2_32<D / 2>(tmem_o + cc, ro);
        tmem_ld_wait(ro);
#pragma unroll
        for (int i = 0; i < 32; ++i) ro[i] = __float_as_uint(__uint_as_float(ro[i]) * f);
        tmem_st16x2_32<D / 2>(tmem_o + cc, ro);
    }
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
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1 KB alignment for the SW128 stages, by offset (keeps the pointer's
    // shared-space provenance: loads of the masks compile to LDS).
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    Bars& bar = *reinterpret_cast<Bars*>(smem + Cfg::kOffBar);
    uint32_t* maskA = reinterpret_cast<uint32_t*>(smem + Cfg::kOffMask);
    uint32_t* maskB = maskA + a.W;
    uint16_t* ulist = reinterpret_cast<uint16_t*>(maskB + a.W);  // [2 * ceil(|A u B| / 2)]
#if PISA_TRACE
    const long long tstart = clock64();
#endif

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int tile = blockIdx.x;
    const int bh = blockIdx.y;
    const int b = bh / a.H, h = bh % a.H;
    // query blocks of this tile (within the range [qb0, qb1)): the pairing
    // kernel's choice, or consecutive blocks
    int iA = a.qb0 + 2 * tile, iB = iA + 1;
    if (a.pairs) {
        const int2 pr = a.pairs[size_t(bh) * ((a.N + 1) / 2) + tile];
        iA = pr.x;
        iB = pr.y;
    }
    const bool hasB = iB >= 0 && iB < a.qb1;
    const bool tail = a.variant != 0;                       // Zeroth, Hybrid, GlobalCentroid
    const bool first_order = a.variant == 3 || a.variant == 4;
    const int n_last = a.L - (a.N - 1) * 64;

    // the two selection bitmasks (K2's output, L2-resident): warps 0-3 load one
    // word per lane first, so the round trip overlaps the setup below
    const int wl = warp * 32 + lane;
    uint32_t ra = 0u, rb = 0u;
    if (warp < 4 && wl < a.W) {
        ra = __ldcg(a.mask + (size_t(bh) * a.N + iA) * a.W + wl);
        if (hasB) rb = __ldcg(a.mask + (size_t(bh) * a.N + iB) * a.W + wl);
    }
    // ------------------------------------------------------------ setup --
    if (threadIdx.x == 0) {
        mbar_init(&bar.q_full, 1);
        mbar_init(&bar.h_full, 1);
        mbar_init(&bar.qh_full, 1);
        for (int s = 0; s < kSK; ++s) mbar_init(&bar.k_full[s], 1);
        for (int s = 0; s < kSV; ++s) {
            mbar_init(&bar.v_full[s], D / 64);  // one arrive per V producer (one per 64-col half)
            mbar_init(&bar.v_empty[s], 1);
        }
        for (int s = 0; s < kSB; ++s) {
            mbar_init(&bar.s_full[s], 1);
            mbar_init(&bar.p_full[s], 8);  // one arrive per softmax warp
            mbar_init(&bar.p_half[s], 8);  // (PISA_PSPLIT) first sub-tile of P
        }
        fence_mbar_init();
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
        // Q first: it needs nothing but its barrier, so its 16 TMA boxes go out
        // before the CTA barrier (they used to sit on the prologue's critical
        // path). Interleaved row order: the 16-row chunk (quadrant q4, block hh)
        // of the tile lands at shared-memory / TMEM rows q4*32 + hh*16.
        mbar_expect_tx(&bar.q_full, Cfg::kQ);
#pragma unroll
        for (int half = 0; half < D / 64; ++half)
#pragma unroll
            for (int c = 0; c < 8; ++c)
                tma_load_4d(smem + Cfg::kOffQ + half * 16384 + c * 2048, &tmQ, &bar.q_full, half * 64,
                            ((c & 1) && hasB ? iB : iA) * 64 + (c >> 1) * 16, h, b);
    }
    if (warp == 2) {
        tmem_alloc(&bar.tmem_base, 512);
        tmem_relinquish();
        TRACE(12, 0);  // (trace builds) prologue: TMEM allocated
    }
    if (warp < 4) {
        // Selection bitmasks of the two query blocks into shared memory, and the
        // ascending union as a list of 16-bit entries: block index | (selected by
        // A) << 14 | (by B) << 15, padded to an even length with a copy of the
        // last entry whose use flags are 0 (fully masked: P = 0, finite V rows).
        // Every role reads super-tile g's two entries with one shared load.
        // Warps 0-3 build it together, one word per lane (W <= 128), after their
        // own prologue tasks (a serial build in one warp cost ~2.5K cycles per
        // CTA: 11 % of a FLUX-sized CTA).
        __syncwarp();
        const int w = wl;
        if (w < a.W) {
            maskA[w] = ra;
            maskB[w] = rb;
        }
        const uint32_t u = ra | rb;
        const uint32_t c = __popc(u);
        uint32_t x = c;  // inclusive prefix over the warp's 32 words
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) bar.n_w[warp] = x;
        asm volatile("bar.sync 1, 128;" ::: "memory");  // warps 0-3
        uint32_t base = 0, total = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t n = bar.n_w[q];
            base += q < warp ? n : 0u;
            total += n;
        }
        uint32_t pos = base + x - c;
        uint16_t last = 0;
        for (uint32_t bits = u; bits; bits &= bits - 1) {
            const int bt = __ffs(bits) - 1;
            last = uint16_t((w * 32 + bt) | (((ra >> bt) & 1u) << 14) | (((rb >> bt) & 1u) << 15));
            ulist[pos++] = last;
        }
        if (c != 0 && pos == total && (total & 1u)) ulist[total] = uint16_t(last & 0x3FFFu);
        if (warp == 3 && lane == 0) bar.n_u = total;
        if (warp == 3) TRACE(13, 0);  // masks copied, union listed
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) TRACE(14, 0);  // CTA barrier passed
    const uint32_t tmem = bar.tmem_base;
    const int nU = int(bar.n_u);
    // Key tiles are processed in pairs ("super-tiles" of 128 keys): one K / V
    // stage, one S buffer, one barrier round trip and N=128 S MMAs per pair.
    // Phase 1 walks the union list; Phase 2 pairs consecutive centroid chunks.
    const int G1 = (nU + 1) >> 1;
    const int G = G1 + (tail ? (a.nchunk2 + 1) >> 1 : 0);
    auto pair_of = [&](int g, uint32_t& e0, uint32_t& e1) {
        const uint32_t v = reinterpret_cast<const uint32_t*>(ulist)[g];
        e0 = v & 0xFFFFu;
        e1 = v >> 16;
    };
    auto tile_rows = [&](int g, int& r0, int& r1) {
        if (g < G1) {
            uint32_t e0, e1;
            pair_of(g, e0, e1);
            r0 = int(e0 & 0x3FFFu) * 64;
            r1 = int(e1 & 0x3FFFu) * 64;
        } else {
            const int c = 2 * (g - G1);
            r0 = c * 64;
            r1 = (c + 1 < a.nchunk2 ? c + 1 : c) * 64;
        }
    };

    if (warp == 0) {
        // ------------------------------------------------ producer: Q, K, H --
#if PISA_REGS_PRODUCER
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PISA_REGS_PRODUCER));
#endif
        // K stage of S_g is free once S_{g-kSK} is done: s_full of that S
        // (no separate "empty" commit; S_{g-kSK+3} cannot complete before K_g is
        // loaded, so the parity is unambiguous)
        auto wait_s_done = [&](int j) {
            if (j >= 0) mbar_wait(&bar.s_full[j % kSB], uint32_t((j / kSB) & 1));
        };
        int s = 0;
        for (int g = 0; g < G; ++g) {
            uint8_t* sK = smem + Cfg::kOffK + s * Cfg::kKV;
            wait_s_done(g - kSK);
            const bool exact = g < G1;
            int r0, r1;
            if (g == 0) TRACE(12, 1);
            tile_rows(g, r0, r1);
            if (g == 0) TRACE(13, 1);
            if (elect_one()) {
                mbar_expect_tx(&bar.k_full[s], Cfg::kKV);
                if (g == 0) TRACE(14, 1);
#pragma unroll
                for (int half = 0; half < D / 64; ++half) {
                    if (exact) {
                        tma_load_4d(sK + half * 16384, &tmK, &bar.k_full[s], half * 64, r0, h, b);
                        tma_load_4d(sK + half * 16384 + 8192, &tmK, &bar.k_full[s], half * 64, r1, h, b);
                    } else {
                        tma_load_3d(sK + half * 16384, &tmKb, &bar.k_full[s], half * 64, r0, bh);
                        tma_load_3d(sK + half * 16384 + 8192, &tmKb, &bar.k_full[s], half * 64, r1, bh);
                    }
                }
                TRACE(0, g);
            }
            __syncwarp();
            if (++s == kSK) s = 0;
        }
        if (first_order) {
            // H_bar (D x D = one stage) into K stage 0 once every S MMA is done
            for (int j = G - kSK; j < G; ++j) wait_s_done(j);
            if (elect_one()) {
                mbar_expect_tx(&bar.h_full, D * D * 2);
#pragma unroll
                for (int half = 0; half < D / 64; ++half)
                    tma_load_3d(smem + Cfg::kOffK + half * 16384, &tmH, &bar.h_full, half * 64, 0, bh);
            }
            __syncwarp();
        }
    } else if (warp == 2 || (warp == kVWarp1 && D == 128)) {
#if PISA_REGS_PRODUCER
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PISA_REGS_PRODUCER));
#endif
        // -------------------------------------------- producers: V halves --
        const int vh = warp == 2 ? 0 : 1;
        int s = 0;
        uint32_t ph = 0;
        for (int g = 0; g < G; ++g) {
            uint8_t* sV = smem + Cfg::kOffV + s * Cfg::kKV + vh * 16384;
            mbar_wait(&bar.v_empty[s], ph ^ 1);
            const bool exact = g < G1;
            int r0, r1;
            tile_rows(g, r0, r1);
            if (elect_one()) {
                mbar_expect_tx(&bar.v_full[s], 16384);
                if (exact) {
                    tma_load_4d(sV, &tmV, &bar.v_full[s], vh * 64, r0, h, b);
                    tma_load_4d(sV + 8192, &tmV, &bar.v_full[s], vh * 64, r1, h, b);
                } else {
                    tma_load_3d(sV, &tmVh, &bar.v_full[s], vh * 64, r0, bh);
                    tma_load_3d(sV + 8192, &tmVh, &bar.v_full[s], vh * 64, r1, bh);
                }
                if (vh == 0) TRACE(1, g);
            }
            __syncwarp();
            if (++s == kSV) { s = 0; ph ^= 1u; }
        }
    } else if (warp == kVWarp1) {
        // (D = 64: one V producer; warp 3 only joins its warpgroup's setmaxnreg)
#if PISA_REGS_PRODUCER
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PISA_REGS_PRODUCER));
#endif
    } else if (warp == kMmaWarp) {
#if PISA_REGS_PRODUCER
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PISA_REGS_PRODUCER));
#endif
        // ------------------------------------------------------------- MMA --
        // Lean issue loop: shared-memory descriptors are built once and
        // advanced by adding (byte offset >> 4) to their address field; ring
        // positions advance incrementally (no div/mod). One elected lane issues
        // (and commits: a commit tracks the MMAs of the thread that runs it).
        constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);  // S = Q K^T, 128 keys
        constexpr uint32_t idPV = idesc_bf16(128, D, 0, 1);   // O += P V (P from TMEM, V MN-major)
        constexpr uint32_t idQH = idesc_bf16(128, D, 0, 1);   // Q H_bar
        const uint64_t qdesc0 = sdesc_sw128(smem_u32(smem + Cfg::kOffQ), 16, 1024);
        const uint64_t kdesc0 = sdesc_sw128(smem_u32(smem + Cfg::kOffK), 16, 1024);
        const uint64_t vdesc0 = sdesc_sw128(smem_u32(smem + Cfg::kOffV), 16384, 1024);
        const uint64_t hdesc0 = sdesc_sw128(smem_u32(smem + Cfg::kOffK), 16384, 1024);
        const uint32_t tS = tmem + kColS, tO = tmem + kColO;
        int sk = 0, sbk = 0;            // K stage and S buffer of the next S
        uint32_t phk = 0;               // its k_full parity
        int sv = 0, sbv = 0;            // V stage and S/P buffer of the next PV
        uint32_t phv = 0, php = 0;      // v_full / p_full parities
        // MMAs of S_g into S buffer g % 3 (SS: Q and K from shared memory);
        // commit: s_full (the softmax's "S ready" and the K producer's "stage free")
        auto mma_s = [&](int g) {
            TRACE(8, g);
            const uint64_t kd = kdesc0 + uint64_t(sk * (Cfg::kKV >> 4));
            const uint32_t d = tS + uint32_t(sbk) * 128;
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
                const uint64_t off = uint64_t(((ks >> 2) * 16384 + (ks & 3) * 32) >> 4);
                mma_ss(d, qdesc0 + off, kd + off, idS, ks != 0);
            }
            mma_commit(&bar.s_full[sbk]);
            TRACE(2, g);
        };
        auto advance_s = [&]() {
            if (++sk == kSK) { sk = 0; phk ^= 1u; }
            if (++sbk == kSB) sbk = 0;
        };
        // MMAs of O += P_g V_g, P_g over the S_g columns; commit: v_empty (the V
        // producer's "stage free" and the softmax's "PV_g done")
        // PV of sub-tiles [k0, k1) of super-tile g (4 MMAs of 16 keys each);
        // the last one commits the V stage
        auto mma_pv = [&](int g, int k0, int k1) {
            TRACE(10, g);
            const uint64_t vd = vdesc0 + uint64_t(sv * (Cfg::kKV >> 4));
            const uint32_t pa = tS + uint32_t(sbv) * 128;
#pragma unroll
            for (int ks = 4 * k0; ks < 4 * k1; ++ks)
                mma_ts(tO, pa + (ks >> 2) * 64 + (ks & 3) * 8, vd + uint64_t((ks * 2048) >> 4), idPV,
                       (g == 0 && ks == 0) ? 0u : 1u);
            if (k1 == 2) mma_commit(&bar.v_empty[sv]);
            TRACE(3, g);
        };
        auto advance_pv = [&]() {
            if (++sv == kSV) { sv = 0; phv ^= 1u; }
            if (++sbv == kSB) { sbv = 0; php ^= 1u; }
        };
        if (a.tile_count && lane == 0) atomicAdd(a.tile_count, (unsigned long long)(2 * G));
        mma_wait(&bar.q_full, 0);
        TRACE(15, 0);  // Q landed
        tc_fence_after();
        for (int g = 0; g < kSB && g < G; ++g) {
            mma_wait(&bar.k_full[sk], phk);
            tc_fence_after();
            if (elect_one()) mma_s(g);
            __syncwarp();
            advance_s();
        }
        for (int g = 0; g < G; ++g) {
            // PV_g as soon as P_g and V_g are in, then S_{g+3} once K_{g+3} is
            // (in-order tensor pipe: S_{g+3} overwrites P_g after PV_g read it).
            // A late K_{g+3} holds back PV_{g+1}; an event loop issuing whichever
            // is ready first measured slower (26.1 vs 23.5 ms at Wan2.1-14B,
            // profiles/r02_k3_variants.log batch ae): S early feeds the softmax,
            // the kernel's bottleneck, and PV_{g+1} before S_{g+3} delays it.
#if PISA_PSPLIT
            mma_wait(&bar.p_half[sbv], php);
            mma_wait(&bar.v_full[sv], phv);
            tc_fence_after();
            if (elect_one()) mma_pv(g, 0, 1);
            __syncwarp();
            mma_wait(&bar.p_full[sbv], php);
            TRACE(9, g);
            tc_fence_after();
            if (elect_one()) mma_pv(g, 1, 2);
            __syncwarp();
#else
            mma_wait(&bar.p_full[sbv], php);
            TRACE(9, g);
            mma_wait(&bar.v_full[sv], phv);
            tc_fence_after();
            if (elect_one()) mma_pv(g, 0, 2);
            __syncwarp();
#endif
            advance_pv();
            if (g + kSB < G) {
                mma_wait(&bar.k_full[sk], phk);
                tc_fence_after();
                if (elect_one()) mma_s(g + kSB);
                __syncwarp();
                advance_s();
            }
        }
        if (first_order) {
            mma_wait(&bar.h_full, 0);
            tc_fence_after();
        }
        if (elect_one()) {
            if (first_order) {
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks)
                    mma_ss(tS, qdesc0 + uint64_t(((ks >> 2) * 16384 + (ks & 3) * 32) >> 4),
                           hdesc0 + uint64_t((ks * 2048) >> 4), idQH, ks != 0);
            }
            mma_commit(&bar.qh_full);  // also: every PV done
            TRACE(12, 2);  // (trace builds) tail: QH issued
        }
        __syncwarp();
    } else if (warp >= 4) {
#if PISA_REGS_PRODUCER
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(PISA_REGS_SOFTMAX));
#endif
        // ------------------------------------------------ softmax warpgroups --
        const int hh = (warp - 4) >> 2;  // query block 2*tile + hh
        const int q4 = warp & 3;         // TMEM lane quadrant
        const int r16 = lane & 15;
        const int ch = lane >> 4;        // column half of a 64-key sub-tile
        const float sl2 = a.scale * 1.4426950408889634f;
        const uint32_t lbase = tmem + (uint32_t(q4 * 32 + hh * 16) << 16);
        // no partner (a lone last block, or iB outside a query-block range):
        // warpgroup B is idle and writes nothing
        const int qblk = hh ? (hasB ? iB : -1) : iA;
        const int grow = qblk * 64 + q4 * 16 + r16;
        const bool active = qblk >= 0 && grow < a.L;
        const bool wact = __all_sync(0xffffffffu, active);
        const uint32_t* hmask = hh ? maskB : maskA;
        const __nv_bfloat16* qrow = a.q + size_t(b) * a.qs_b + size_t(h) * a.qs_h + size_t(grow) * a.qs_l;

        float m = -INFINITY, l = 0.f, lt = 0.f;  // l, lt: this thread's partial sums

        // Online-softmax step over one 128-key super-tile: bm_loc = max of this
        // thread's live scores (masked = -inf). Returns the shift to
        // exponentiate against (log2 units); rescales O lazily when the max
        // grows by > 2^8 (after PV_{g-1}: O must be quiescent).
        // S/P buffer ring: super-tile g uses buffer sb = g % 3, phase parity phs
        int sb = 0;
        uint32_t phs = 0;
        auto wait_pv_prev = [&](int g) {  // PV_{g-1} done = its V stage released
            if (g > 0) {
                // PV_{g-1-kSV} is known done (S_g was issued after PV_{g-3}), so
                // the parity names PV_{g-1} unambiguously
                const int j = g - 1;
                mbar_wait<true>(&bar.v_empty[j % kSV], uint32_t((j / kSV) & 1));
                tc_fence_after();
            }
        };
        auto advance = [&]() {
            if (++sb == kSB) { sb = 0; phs ^= 1u; }
        };
        auto update_max = [&](float bm_loc, int g) -> float {
            const float bm = fmaxf(bm_loc, __shfl_xor_sync(0xffffffffu, bm_loc, 16)) * sl2;
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
                wait_pv_prev(g);
                TRACE(24 + hh * 4 + q4, g);  // (trace builds) rescale of this warp's rows
                rescale_o<D>(lbase + kColO, f);
                l *= f;
                lt *= f;
            }
            m = m_use;
            return (m_use == -INFINITY) ? 0.f : m_use;  // all-masked row: p = 0, not NaN
        };
        auto publish_half = [&]() {  // first sub-tile of P stored (PISA_PSPLIT)
#if PISA_PSPLIT
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar.p_half[sb]);
#endif
        };
        auto publish_p = [&](int g_cur) {
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar.p_full[sb]);
            TRACE(16 + hh * 4 + q4, g_cur);  // (trace builds) every warp's P publish
        };
        const uint32_t kZero16[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};

        // ---- Phase 1: exact blocks of the union, two per super-tile
        uint32_t r0[32], r1[32];  // scores of the used sub-tiles (raw bits)
        for (int g = 0; g < G1; ++g) {
            uint32_t e0, e1;
            pair_of(g, e0, e1);  // pad: use flags 0
            const bool use0 = (e0 >> (14 + hh)) & 1u, use1 = (e1 >> (14 + hh)) & 1u;  // warp-uniform
            const int nv0 = (int(e0 & 0x3FFFu) == a.N - 1) ? n_last : 64;
            const int nv1 = (int(e1 & 0x3FFFu) == a.N - 1) ? n_last : 64;
            const uint32_t sc = lbase + kColS + sb * 128;
            softmax_wait(&bar.s_full[sb], phs);
            tc_fence_after();
            if (use0) tmem_ld16x2_32<32>(sc, r0);
            if (use1) tmem_ld16x2_32<32>(sc + 64, r1);
            if (q4 == 0) TRACE(4 + hh, g);
            if (use0 || use1) {
                // scores as raw bits, masked in place (only the ragged last key
                // block / rows past L need masks); loads only of the selected
                // sub-tiles
                tmem_ld_wait(r0);
                tmem_ld_wait(r1);
                if (!(wact && nv0 == 64 && nv1 == 64)) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int col = ch * 32 + i;
                        if (!(active && col < nv0)) r0[i] = 0xff800000u;  // -inf
                        if (!(active && col < nv1)) r1[i] = 0xff800000u;
                    }
                }
                // exponentials only for the selected sub-tiles (warp-uniform);
                // sub-tiles both blocks selected split exp2 across MUFU and FMA
                float lsum = 0.f;
                auto expo_store = [&](const uint32_t (&r)[32], uint32_t addr, bool both, float mm) {
                    uint32_t pk[16];
                    float ps[4] = {0.f, 0.f, 0.f, 0.f};
                    if (kPolyBoth != kPolyMask && both) {  // (one code path when the splits agree)
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            const float p0 = ex2_mix<kPolyBoth>(fmaf(__uint_as_float(r[i]), sl2, -mm), i);
                            const float p1 = ex2_mix<kPolyBoth>(fmaf(__uint_as_float(r[i + 1]), sl2, -mm), i + 1);
                            ps[(i >> 1) & 3] += p0 + p1;
                            pk[i >> 1] = pack_bf16(p0, p1);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            const float p0 = ex2_mix<kPolyMask>(fmaf(__uint_as_float(r[i]), sl2, -mm), i);
                            const float p1 = ex2_mix<kPolyMask>(fmaf(__uint_as_float(r[i + 1]), sl2, -mm), i + 1);
                            ps[(i >> 1) & 3] += p0 + p1;
                            pk[i >> 1] = pack_bf16(p0, p1);
                        }
                    }
                    lsum += (ps[0] + ps[1]) + (ps[2] + ps[3]);
                    tmem_st16x2_16<16>(addr, pk);  // P (bf16 pairs)
                };
                const bool both0 = ((e0 >> 14) & 3u) == 3u, both1 = ((e1 >> 14) & 3u) == 3u;
                auto exact_max = [&]() -> float {  // lazy update of m from the super-tile's row max
                    float bm_loc = -INFINITY;
                    if (use0) bm_loc = max32(reinterpret_cast<const float*>(r0));
                    if (use1) bm_loc = fmaxf(bm_loc, max32(reinterpret_cast<const float*>(r1)));
                    return update_max(bm_loc, g);
                };
#if PISA_SPEC_MAX
                // single pass: exponentiate against the running max without this
                // super-tile's max; it is only needed (the exact lazy update, then
                // P again) when the row has no max yet or the p sum exceeds 2^16,
                // which keeps p bounded as the 2^8 rescale threshold did
                // (warp-uniform: the P stores are warp-collective tcgen05.st)
                const bool fresh = __any_sync(0xffffffffu, m == -INFINITY && active);
                if (!fresh) {
                    const float mm = m == -INFINITY ? 0.f : m;
                    if (use0) expo_store(r0, sc, both0, mm);
                    if (use1) expo_store(r1, sc + 64, both1, mm);
                }
                if (__any_sync(0xffffffffu, fresh || !(lsum <= 65536.f))) {
                    const float mm = exact_max();
                    lsum = 0.f;
                    if (use0) expo_store(r0, sc, both0, mm);
                    if (use1) expo_store(r1, sc + 64, both1, mm);
                }
                if (!use0) tmem_st16x2_16<16>(sc, kZero16);
                if (!use1) tmem_st16x2_16<16>(sc + 64, kZero16);
#else
                const float mm = exact_max();
                if (use0) expo_store(r0, sc, both0, mm); else tmem_st16x2_16<16>(sc, kZero16);
                publish_half();
                if (use1) expo_store(r1, sc + 64, both1, mm); else tmem_st16x2_16<16>(sc + 64, kZero16);
#endif
                l += lsum;
            } else {
                tmem_st16x2_16<16>(sc, kZero16);
                publish_half();
                tmem_st16x2_16<16>(sc + 64, kZero16);
            }
            publish_p(g);
            advance();
            if (q4 == 0) TRACE(6 + hh, g);
        }
        // ---- Phase 2: centroid chunks, two per super-tile; column mask = own
        // selection, weight n_j (the ragged last block weighs n_last)
        for (int g = G1; g < G; ++g) {
            const int c0 = 2 * (g - G1);
            const uint32_t sc = lbase + kColS + sb * 128;
            // this thread's 32 columns of chunk c: blocks c*64 + ch*32 + i
            auto colmask = [&](int c) -> uint32_t {
                const int w = 2 * c + ch;
                return (c < a.nchunk2 && w < a.W) ? hmask[w] : 0xffffffffu;
            };
            const uint32_t cm0 = colmask(c0), cm1 = colmask(c0 + 1);
            const int nv0 = min(64, a.N - c0 * 64), nv1 = min(64, a.N - (c0 + 1) * 64);
            softmax_wait(&bar.s_full[sb], phs);
            tc_fence_after();
            uint32_t r0[32], r1[32];
            tmem_ld16x2_32<32>(sc, r0);
            tmem_ld16x2_32<32>(sc + 64, r1);
            tmem_ld_wait(r0);
            tmem_ld_wait(r1);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int col = ch * 32 + i;
                if (!(active && col < nv0 && !((cm0 >> i) & 1u))) r0[i] = 0xff800000u;
                if (!(active && col < nv1 && !((cm1 >> i) & 1u))) r1[i] = 0xff800000u;
            }
            // column (within this thread's 32) of the ragged last block, if here
            const int lb = a.N - 1 - c0 * 64 - ch * 32;  // 0..31 -> sub-tile 0, 64..95 -> sub-tile 1
            const bool ragged = n_last != 64;
            float ps = 0.f, plast = 0.f;
            auto expo_store = [&](const uint32_t (&r)[32], uint32_t addr, int lbo, float mm) {
                uint32_t pk[16];
                float q0 = 0.f, q1 = 0.f;
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                    const float p0 = ex2_mix<kPolyBoth>(fmaf(__uint_as_float(r[i]), sl2, -mm), i);
                    const float p1 = ex2_mix<kPolyBoth>(fmaf(__uint_as_float(r[i + 1]), sl2, -mm), i + 1);
                    q0 += p0;
                    q1 += p1;
                    pk[i >> 1] = pack_bf16(p0, p1);
                }
                ps += q0 + q1;
                tmem_st16x2_16<16>(addr, pk);
                // the ragged last block's p (weight n_last, not 64): only in the
                // super-tile and thread half that hold it, picked by a static
                // select chain (a dynamic index would put r in local memory)
                if (ragged && lbo >= 0 && lbo < 32) {
                    uint32_t sb_ = 0xff800000u;
#pragma unroll
                    for (int i = 0; i < 32; ++i) sb_ = (i == lbo) ? r[i] : sb_;
                    plast += ex2_mix<kPolyBoth>(fmaf(__uint_as_float(sb_), sl2, -mm), lbo);
                }
            };
            auto run = [&](float mm) {
                ps = plast = 0.f;
                expo_store(r0, sc, lb, mm);
                expo_store(r1, sc + 64, lb - 64, mm);
            };
            auto exact_max = [&]() -> float {
                return update_max(fmaxf(max32(reinterpret_cast<const float*>(r0)),
                                        max32(reinterpret_cast<const float*>(r1))), g);
            };
#if PISA_SPEC_MAX
            const bool fresh = __any_sync(0xffffffffu, m == -INFINITY && active);
            if (!fresh) run(m == -INFINITY ? 0.f : m);
            if (__any_sync(0xffffffffu, fresh || !(ps <= 65536.f))) run(exact_max());
#else
            run(exact_max());
#endif
            l += 64.f * ps + (float(n_last) - 64.f) * plast;
            lt += ps;
            publish_p(g);
            advance();
        }

        // ------------------------------------------------------- epilogue --
        mbar_wait(&bar.qh_full, 0);
        tc_fence_after();
        if (warp == 4) TRACE(13, 2);  // tail: O and QH complete
        float mrow = m;
        float lfin = l + __shfl_xor_sync(0xffffffffu, l, 16);
        float ltot = lt + __shfl_xor_sync(0xffffffffu, lt, 16);
        float cw = 0.f;
        if (a.variant == 3) {
            cw = a.scale * ltot;
            if (a.literal_phase3) cw *= (1.0f / 64.0f);
        }
        float fo = 1.f;  // extra scale on O and l (GlobalCentroid shift)
        if (a.variant == 4) {
            // slope = |U_i| exp(scale q.k_bar_global - m)   (engine.hpp:202-205)
            const float* kg = a.kbar_global + size_t(bh) * D;
            float dot = 0.f;
            if (active) {
                for (int c = ch * (D / 2); c < (ch + 1) * (D / 2); ++c)
                    dot = fmaf(__bfloat162float(qrow[c]), kg[c], dot);
            }
            dot += __shfl_xor_sync(0xffffffffu, dot, 16);
            const float gx = dot * sl2;
            const int nU = a.N - a.k;
            if (active && nU > 0) {
                const float mm = fmaxf(mrow, gx);
                fo = ex2(mrow - mm);
                cw = a.scale * float(nU) * ex2(gx - mm);  // pisa_reference: no literal_phase3
                mrow = mm;
                lfin *= fo;
                ltot *= fo;
            }
        }
        const float inv_l = 1.0f / lfin;
        bool bad = false;
        char* orow = reinterpret_cast<char*>(a.out) +
                     (size_t(b) * a.os_b + size_t(h) * a.os_h + size_t(grow) * a.os_l) *
                         (a.out_f32 ? 4 : 2);
#pragma unroll 1
        for (int cc = 0; cc < D / 2; cc += 32) {
            uint32_t ro[32], rq[32];
            tmem_ld16x2_32<D / 2>(lbase + kColO + cc, ro);
            if (first_order) tmem_ld16x2_32<D / 2>(lbase + kColS + cc, rq);
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
            const int col = ch * (D / 2) + cc;
            if (active) {
                if (a.out_f32) {
                    float4* dst = reinterpret_cast<float4*>(orow) + col / 4;
#pragma unroll
                    for (int i = 0; i < 32; i += 4) dst[i / 4] = make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]);
                } else {
                    uint4* dst = reinterpret_cast<uint4*>(orow + col * 2);
#pragma unroll
                    for (int i = 0; i < 32; i += 8)
                        dst[i / 8] = make_uint4(pack_bf16(o[i], o[i + 1]), pack_bf16(o[i + 2], o[i + 3]),
                                                pack_bf16(o[i + 4], o[i + 5]), pack_bf16(o[i + 6], o[i + 7]));
                }
            }
        }
        if (active) {
            const size_t di = size_t(bh) * a.L + grow;
            if (ch == 0) {
                if (a.diag_m) a.diag_m[di] = mrow * 0.6931471805599453f;  // log2 units -> natural log
                if (a.diag_l) a.diag_l[di] = lfin;
                if (a.diag_lt) a.diag_lt[di] = ltot;
            }
            if (bad && a.nonfinite) atomicExch(a.nonfinite, 1);
        }
        if (warp == 4) TRACE(14, 2);  // tail: this warp's rows stored
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace

size_t fused_smem_bytes(int D, int N, int W) {
    const size_t core = (D == 128) ? size_t(FusedCfg<128>::kOffMask) : size_t(FusedCfg<64>::kOffMask);
    // masks (2 W words) + the union list (<= N entries + 1 pad, 16-bit)
    return 1024 + core + size_t(2 * W) * 4 + size_t(N + 2) * 2 + 16;
}

cudaError_t launch_fused(int D, const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                         const CUtensorMap& tmKb, const CUtensorMap& tmVh, const CUtensorMap& tmH,
                         const FusedArgs& a, int BH, cudaStream_t s) {
    const size_t smem = fused_smem_bytes(D, a.N, a.W);
    dim3 grid((a.qb1 - a.qb0 + 1) / 2, BH);
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
