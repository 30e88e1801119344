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
// Tiling. One CTA owns 128 query rows = query blocks A, B (a pair chosen by the
// pairing kernel, or (2t, 2t+1)), because the tcgen05 M=128 MMA is the
// full-rate shape (M=64 costs the same time). The CTA walks the ascending UNION
// of the two selections in "super-tiles" of two key blocks (128 keys); a per-
// block flag zeroes P for the block that did not select a key block, so
// executed MMA work <= two M=64 passes. Phase 2 is the same loop over
// ceil(N/64) centroid tiles with a per-block column mask (the selection
// bitmask) and per-column weight n_j. Phase 3 is one more MMA, Q . H_bar.
//
// Why this shape (tools/l2_bw.cu, tools/st_mix.cu, profiles/): a super-tile is
// 1024 tensor cycles (8 SS MMAs S = Q [K_a; K_b]^T at N=128, 8 TS MMAs
// O += P V), and it streams a random 32 KB K and 32 KB V tile from L2, which
// takes 1300-2000 cycles per tile under load, so ~100+ KB must be in flight
// per SM: ONE CTA per SM with Q (32 KB) + 3 K + 3 V stages of 32 KB (224 KB at
// d = 128). The 64 KB of K/V copies per super-tile do not slow the MMAs
// (st_mix mode 4). A transposed S^T = K Q^T tile per query block (no union
// waste) is shared-memory-port bound at 430 cycles per useful pair against 455
// for this tile (st_mix mode 6) and was not built.
//
// Softmax: thread per row, two warpgroups ALTERNATING super-tiles (the
// FlashAttention-4 shape). TMEM (512 columns): O_0 | O_1 (D columns each) |
// S_0 | S_1 (128 columns each, P_g written over S_g as bf16). Super-tile g
// goes to S buffer g & 1, is exponentiated by warpgroup g & 1 and accumulated
// into O_{g & 1}; each warpgroup keeps its own running max / sums, and the
// epilogue merges the two partial softmaxes (max, rescale, add). Each thread
// owns one row and all 128 columns of a super-tile: no shuffles for the row
// max, and the fixed per-super-tile cost (barrier wait, TMEM ld/st latency,
// publish) is paid once per 128 elements, while the other warpgroup works on
// the next super-tile. The previous layout (two threads per row, both
// warpgroups on the same super-tile in lockstep, three S buffers) reached
// ~6 exponentials / clock / SM on clustered routing against the 13-14 the
// instruction sequence reaches alone (tools/mufu_rate.cu).
//
// Row layout: TMEM lanes / Q rows [0, 64) = query block A, [64, 128) = B.
// Warp q4 of a warpgroup owns lanes [32 q4, +32), so warps q4 = 0, 1 hold
// block A and q4 = 2, 3 block B: the use flags of a super-tile are
// warp-uniform and a block's unselected key block costs its warps nothing.
//
// Warp roles (384 threads):
//   warp 0     TMA producer: Q (once), K / k_bar tiles (3-stage ring of pairs),
//              H_bar at the end
//   warp 1     single-thread tcgen05.mma issuer: S_g = Q K_g^T (SS, K-major),
//              O_{g&1} += P_g V_g (TS: P from TMEM, V MN-major), Q H_bar (SS)
//   warp 2     TMEM allocator, then TMA producer for V columns [0, 64)
//   warp 3     builds the union sizes from the two selection bitmasks, then TMA
//              producer for V columns [64, 128) (two issue streams for V)
//   warps 4-7  softmax of the even super-tiles (warpgroup 0), epilogue columns [0, D/2)
//   warps 8-11 softmax of the odd super-tiles (warpgroup 1), epilogue columns [D/2, D)
// exp2 with log2(e)*scale folded into one FFMA; lazy rescale of O_x (only
// when the running max grows by > 2^8).
#include "kernels.h"
#include "sm100.cuh"

#ifndef PISA_TRACE
#define PISA_TRACE 0
#endif

namespace pisa_b200 {
using namespace pisa_sm100;

namespace {

constexpr int kThreads = 384;
constexpr int kSK = 3;  // K ring stages (two key blocks each)
constexpr int kSV = 3;  // V ring stages (two key blocks each)
constexpr float kRescaleThresh = 8.0f;  // log2 units
constexpr uint32_t kColS = 256;         // S_0 | S_1 at [256, 384) | [384, 512); O_x at x * D
#ifndef PISA_MUFU_PINGPONG
#define PISA_MUFU_PINGPONG 1
#endif
#ifndef PISA_REGS_PRODUCER
#define PISA_REGS_PRODUCER 0
#endif
#ifndef PISA_REGS_SOFTMAX
#define PISA_REGS_SOFTMAX 224
#endif
static_assert(4 * PISA_REGS_PRODUCER + 8 * PISA_REGS_SOFTMAX <= 2048, "register file (per 32 threads)");

template <int D>
struct FusedCfg {
    static constexpr int kQ = 128 * D * 2;  // Q tile: [64-col half][128 rows] (A rows 0-63, B rows 64-127)
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
    uint64_t k_full[kSK], k_empty[kSK], v_full[kSV], v_empty[kSV];
    uint64_t s_full[2], p_full[2];
    uint32_t tmem_base;
    uint32_t n_u;
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

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
// max of 32 values (3-input FMNMX tree, 16 instructions)
__device__ __forceinline__ float max32(const uint32_t (&r)[32], float m) {
    float a[11];
#pragma unroll
    for (int j = 0; j < 10; ++j)
        a[j] = fmax3(__uint_as_float(r[3 * j]), __uint_as_float(r[3 * j + 1]), __uint_as_float(r[3 * j + 2]));
    a[10] = fmaxf(__uint_as_float(r[30]), __uint_as_float(r[31]));
    return fmax3(fmax3(fmax3(a[0], a[1], a[2]), fmax3(a[3], a[4], a[5]), fmax3(a[6], a[7], a[8])),
                 fmax3(a[9], a[10], m), m);
}

// Rescales this thread's row of O_x (D columns at tmem_o).
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

// entry = block index | (selected by query block A) << 14 | (by B) << 15,
// ascending over the union of the two selection bitmasks
struct UnionCursor {
    const uint32_t* ma;
    const uint32_t* mb;
    int w;
    uint32_t bits;
    __device__ __forceinline__ UnionCursor(const uint32_t* a, const uint32_t* b) : ma(a), mb(b), w(-1), bits(0u) {}
    __device__ __forceinline__ uint32_t next() {
        while (bits == 0) {
            ++w;
            bits = ma[w] | mb[w];
        }
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        return uint32_t(w * 32 + b) | (((ma[w] >> b) & 1u) << 14) | (((mb[w] >> b) & 1u) << 15);
    }
    // the two entries of super-tile g (called for g = 0, 1, ... in order); an
    // odd tail is padded with a copy of the last entry whose use flags are 0
    // (fully masked: P = 0, finite V rows)
    __device__ __forceinline__ void pair(int g, int nU, uint32_t& e0, uint32_t& e1) {
        e0 = next();
        e1 = (2 * g + 1 < nU) ? next() : (e0 & 0x3FFFu);
    }
};

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

    // ------------------------------------------------------------ setup --
    if (threadIdx.x == 0) {
        mbar_init(&bar.q_full, 1);
        mbar_init(&bar.h_full, 1);
        mbar_init(&bar.qh_full, 1);
        for (int s = 0; s < kSK; ++s) {
            mbar_init(&bar.k_full[s], 1);
            mbar_init(&bar.k_empty[s], 1);
        }
        for (int s = 0; s < kSV; ++s) {
            mbar_init(&bar.v_full[s], D / 64);  // one arrive per V producer (one per 64-col half)
            mbar_init(&bar.v_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bar.s_full[s], 1);
            mbar_init(&bar.p_full[s], 4);  // one arrive per warp of the owning warpgroup
        }
        fence_mbar_init();
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
        // Q first: it needs nothing but its barrier, so its TMA boxes go out
        // before the CTA barrier. Rows [0, 64) = block A, [64, 128) = block B
        // (16-row boxes; a missing B reloads A: finite, never stored).
        mbar_expect_tx(&bar.q_full, Cfg::kQ);
#pragma unroll
        for (int half = 0; half < D / 64; ++half)
#pragma unroll
            for (int c = 0; c < 8; ++c)
                tma_load_4d(smem + Cfg::kOffQ + half * 16384 + c * 2048, &tmQ, &bar.q_full, half * 64,
                            ((c >> 2) && hasB ? iB : iA) * 64 + (c & 3) * 16, h, b);
    }
    if (warp == 2) {
        tmem_alloc(&bar.tmem_base, 512);
        tmem_relinquish();
        TRACE(12, 0);  // (trace builds) prologue: TMEM allocated
    }
    if (warp == 3) {
        // selection bitmasks of the two query blocks into shared memory, and the
        // size of their union (every role walks it itself with a UnionCursor)
        const uint32_t* mA = a.mask + (size_t(bh) * a.N + iA) * a.W;
        const uint32_t* mB = a.mask + (size_t(bh) * a.N + iB) * a.W;
        uint32_t nu = 0;
        // all loads in flight at once (one L2 round trip; W <= 128 for N <= 4096)
        uint32_t ra[4], rb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int w = lane + 32 * i;
            ra[i] = w < a.W ? __ldcg(mA + w) : 0u;
            rb[i] = (w < a.W && hasB) ? __ldcg(mB + w) : 0u;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int w = lane + 32 * i;
            if (w < a.W) {
                maskA[w] = ra[i];
                maskB[w] = rb[i];
            }
            nu += __popc(ra[i] | rb[i]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nu += __shfl_xor_sync(0xffffffffu, nu, o);
        if (lane == 0) bar.n_u = nu;
        TRACE(13, 0);  // masks copied, union sized
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) TRACE(14, 0);  // CTA barrier passed
    const uint32_t tmem = bar.tmem_base;
    const int nU = int(bar.n_u);
    // Phase 1: ceil(|A u B| / 2) super-tiles; Phase 2: consecutive centroid chunks in pairs
    const int G1 = (nU + 1) >> 1;
    const int G = G1 + (tail ? (a.nchunk2 + 1) >> 1 : 0);
    auto tile_rows = [&](UnionCursor& cur, int g, int& r0, int& r1) {
        if (g < G1) {
            uint32_t e0, e1;
            cur.pair(g, nU, e0, e1);
            r0 = int(e0 & 0x3FFFu) * 64;
            r1 = int(e1 & 0x3FFFu) * 64;
        } else {
            const int c = 2 * (g - G1);
            r0 = c * 64;
            r1 = (c + 1 < a.nchunk2 ? c + 1 : c) * 64;
        }
    };

    if (warp < 4) {
#if PISA_REGS_PRODUCER
        regs_dec<PISA_REGS_PRODUCER>();
#endif
    } else {
#if PISA_REGS_PRODUCER
        regs_inc<PISA_REGS_SOFTMAX>();
#endif
    }

    if (warp == 0) {
        // ------------------------------------------------ producer: Q, K, H --
        // K stage s is free once the S MMA that read it is done (k_empty,
        // committed after every S; S_g cannot complete before K_g is loaded,
        // so the parity names S_{g-kSK} unambiguously)
        int s = 0;
        uint32_t ph = 0;
        UnionCursor cur(maskA, maskB);
        for (int g = 0; g < G; ++g) {
            uint8_t* sK = smem + Cfg::kOffK + s * Cfg::kKV;
            mbar_wait(&bar.k_empty[s], ph ^ 1);
            const bool exact = g < G1;
            int r0, r1;
            tile_rows(cur, g, r0, r1);
            if (elect_one()) {
                mbar_expect_tx(&bar.k_full[s], Cfg::kKV);
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
            if (++s == kSK) { s = 0; ph ^= 1u; }
        }
        if (first_order) {
            // H_bar (D x D = one stage) into K stage 0 once the last S that read
            // it (S_j, j the largest multiple of kSK below G) is done
            const int j = ((G - 1) / kSK) * kSK;
            mbar_wait(&bar.k_empty[0], uint32_t((j / kSK) & 1));
            if (elect_one()) {
                mbar_expect_tx(&bar.h_full, D * D * 2);
#pragma unroll
                for (int half = 0; half < D / 64; ++half)
                    tma_load_3d(smem + Cfg::kOffK + half * 16384, &tmH, &bar.h_full, half * 64, 0, bh);
            }
            __syncwarp();
        }
    } else if (warp == 2 || (warp == 3 && D == 128)) {
        // -------------------------------------------- producers: V halves --
        const int vh = warp - 2;
        int s = 0;
        uint32_t ph = 0;
        UnionCursor cur(maskA, maskB);
        for (int g = 0; g < G; ++g) {
            uint8_t* sV = smem + Cfg::kOffV + s * Cfg::kKV + vh * 16384;
            mbar_wait(&bar.v_empty[s], ph ^ 1);
            const bool exact = g < G1;
            int r0, r1;
            tile_rows(cur, g, r0, r1);
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
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA --
        // Shared-memory descriptors are built once and advanced by adding (byte
        // offset >> 4) to their address field; ring positions advance
        // incrementally. One elected lane issues (and commits: a commit tracks
        // the MMAs of the thread that runs it).
        constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);  // S = Q K^T, 128 keys
        constexpr uint32_t idPV = idesc_bf16(128, D, 0, 1);   // O += P V (P from TMEM, V MN-major)
        constexpr uint32_t idQH = idesc_bf16(128, D, 0, 1);   // Q H_bar
        const uint64_t qdesc0 = sdesc_sw128(smem_u32(smem + Cfg::kOffQ), 16, 1024);
        const uint64_t kdesc0 = sdesc_sw128(smem_u32(smem + Cfg::kOffK), 16, 1024);
        const uint64_t vdesc0 = sdesc_sw128(smem_u32(smem + Cfg::kOffV), 16384, 1024);
        const uint64_t hdesc0 = sdesc_sw128(smem_u32(smem + Cfg::kOffK), 16384, 1024);
        const uint32_t tS = tmem + kColS;
        int sk = 0;        // K stage of the next S
        uint32_t phk = 0;  // its k_full parity
        int sv = 0;        // V stage of the next PV
        uint32_t phv = 0;  // its v_full parity
        // S_g into buffer g & 1 (SS: Q and K from shared memory); commit:
        // s_full (the softmax's "S ready" and the K producer's "stage free")
        auto mma_s = [&](int g) {
            TRACE(8, g);
            mbar_wait<true>(&bar.k_full[sk], phk);
            tc_fence_after();
            if (elect_one()) {
                const uint64_t kd = kdesc0 + uint64_t(sk * (Cfg::kKV >> 4));
                const uint32_t d = tS + uint32_t(g & 1) * 128;
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint64_t off = uint64_t(((ks >> 2) * 16384 + (ks & 3) * 32) >> 4);
                    mma_ss(d, qdesc0 + off, kd + off, idS, ks != 0);
                }
                mma_commit(&bar.s_full[g & 1]);
                mma_commit(&bar.k_empty[sk]);
            }
            __syncwarp();
            if (++sk == kSK) { sk = 0; phk ^= 1u; }
            TRACE(2, g);
        };
        if (a.tile_count && lane == 0) atomicAdd(a.tile_count, (unsigned long long)(2 * G));
        mbar_wait<true>(&bar.q_full, 0);
        TRACE(15, 0);  // Q landed
        tc_fence_after();
        for (int g = 0; g < 2 && g < G; ++g) mma_s(g);
        for (int g = 0; g < G; ++g) {
            // PV_g as soon as P_g and V_g are in, then S_{g+2} into the same
            // buffer (in-order tensor pipe: S_{g+2} overwrites P_g after PV_g
            // read it)
            mbar_wait<true>(&bar.p_full[g & 1], uint32_t((g >> 1) & 1));
            TRACE(9, g);
            mbar_wait<true>(&bar.v_full[sv], phv);
            tc_fence_after();
            if (elect_one()) {
                TRACE(10, g);
                const uint64_t vd = vdesc0 + uint64_t(sv * (Cfg::kKV >> 4));
                const uint32_t pa = tS + uint32_t(g & 1) * 128;
                const uint32_t tO = tmem + uint32_t(g & 1) * D;
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    mma_ts(tO, pa + (ks >> 2) * 64 + (ks & 3) * 8, vd + uint64_t((ks * 2048) >> 4), idPV,
                           (g >= 2 || ks != 0) ? 1u : 0u);
                mma_commit(&bar.v_empty[sv]);
                TRACE(3, g);
            }
            __syncwarp();
            if (++sv == kSV) { sv = 0; phv ^= 1u; }
            if (g + 2 < G) mma_s(g + 2);
        }
        if (first_order) {
            mbar_wait<true>(&bar.h_full, 0);
            tc_fence_after();
        }
        if (elect_one()) {
            if (first_order) {
                // Q H_bar into S buffer 0 (every PV that read it is done: in order)
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
        // ------------------------------------------------ softmax warpgroups --
        const int x = (warp - 4) >> 2;   // warpgroup: super-tiles g with g & 1 == x
        const int q4 = warp & 3;         // TMEM lane quadrant
        const int blk = q4 >> 1;         // 0: query block A, 1: B
        const int row = q4 * 32 + lane;  // tile row = TMEM lane
        const float sl2 = a.scale * 1.4426950408889634f;
        const uint32_t lbase = tmem + (uint32_t(q4 * 32) << 16);
        const uint32_t tOx = lbase + uint32_t(x) * D;
        const uint32_t sc = lbase + kColS + uint32_t(x) * 128;
        // no partner (a lone last block, or iB outside a query-block range):
        // block B's warps are idle and write nothing
        const int qblk = blk ? (hasB ? iB : -1) : iA;
        const int grow = qblk * 64 + (row & 63);
        const bool active = qblk >= 0 && grow < a.L;
        const bool wact = __all_sync(0xffffffffu, active);
        const uint32_t* hmask = blk ? maskB : maskA;
        const __nv_bfloat16* qrow = a.q + size_t(b) * a.qs_b + size_t(h) * a.qs_h + size_t(grow) * a.qs_l;

        float m = -INFINITY, l = 0.f, lt = 0.f;  // this warpgroup's partial softmax of the row

        // Exponentials of one 64-key sub-tile (scores r0 | r1 as raw bits, masked
        // = -inf) against the running max mm, packed as bf16 pairs into pk;
        // returns their sum (and the p of column lbo, the ragged last key block
        // in Phase 2, in plast).
        auto expo = [&](const uint32_t (&r0)[32], const uint32_t (&r1)[32], float mm, uint32_t (&pk)[32],
                        int lbo, float& plast) -> float {
            float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
                const uint32_t s0 = i < 32 ? r0[i] : r1[i - 32], s1 = i < 32 ? r0[i + 1] : r1[i - 31];
                const float p0 = ex2(fmaf(__uint_as_float(s0), sl2, -mm));
                const float p1 = ex2(fmaf(__uint_as_float(s1), sl2, -mm));
                ps[(i >> 1) & 3] += p0 + p1;
                if (lbo >= 0) plast += (lbo == i ? p0 : 0.f) + (lbo == i + 1 ? p1 : 0.f);
                pk[i >> 1] = pack_bf16(p0, p1);
            }
            return (ps[0] + ps[1]) + (ps[2] + ps[3]);
        };
        // One sub-tile of the online softmax, single pass: exponentiate against
        // the running max m without computing this sub-tile's max first. The
        // max only has to keep p bounded (P is bf16, O / l are fp32 sums), so
        // m is raised -- exactly, from the scores still in registers -- only
        // when the sub-tile's sum exceeds 2^16 (or the row has no max yet).
        // Raising rescales O_x (quiescent: its last PV, g - 2, precedes S_g),
        // the sums, and P of the super-tile's first sub-tile if it is already
        // in TMEM (pdone). Returns the sum; P goes to TMEM at paddr.
        auto subtile = [&](const uint32_t (&r0)[32], const uint32_t (&r1)[32], uint32_t paddr, uint32_t pdone,
                           int lbo, float& plast) -> float {
            uint32_t pk[32];
            float pl = 0.f;
            float sum = (m == -INFINITY && active) ? INFINITY
                                                   : expo(r0, r1, m == -INFINITY ? 0.f : m, pk, lbo, pl);
            if (__any_sync(0xffffffffu, !(sum <= 65536.f))) {
                // exact max of the row's live scores (3-input FMNMX tree)
                const float bm = max32(r1, max32(r0, -INFINITY)) * sl2;
                const float mn = fmaxf(m, bm);
                const float f = (m == -INFINITY || mn == -INFINITY) ? 1.f : ex2(m - mn);
                if (__any_sync(0xffffffffu, f != 1.f)) {
                    rescale_o<D>(tOx, f);
                    l *= f;
                    lt *= f;
                    if (pdone) {  // P of the first sub-tile, stored against the old max
                        uint32_t rp[32];
                        tmem_st_wait();
                        tmem_ld32(pdone, rp);
                        tmem_ld_wait(rp);
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&rp[i]);
                            rp[i] = pack_bf16(__low2float(v) * f, __high2float(v) * f);
                        }
                        tmem_st32(pdone, rp);
                    }
                }
                m = mn;
                pl = 0.f;
                sum = expo(r0, r1, m == -INFINITY ? 0.f : m, pk, lbo, pl);
            }
            plast += pl;
            tmem_st32(paddr, pk);
            return sum;
        };
        auto zero_store = [&](uint32_t addr) {
            uint32_t z[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) z[i] = 0u;
            tmem_st32(addr, z);
        };
        auto publish_p = [&](int g) {
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar.p_full[x]);
            if (q4 == 0) TRACE(16 + x, g);
        };
        float unused_plast = 0.f;
        // MUFU ping-pong: the two softmax warps of an SM sub-partition (warp q4
        // of each warpgroup) take turns on its exponential unit, so each
        // super-tile's softmax finishes in its own MUFU time instead of both
        // running at half rate (the chain softmax_g -> PV_g -> S_{g+2} ->
        // softmax_{g+2} is on the critical path). Named barriers 2 + 2 q4 + x,
        // 64 threads: this warp syncs on its own, the partner arrives.
        const int tok_mine = 2 + 2 * q4 + x, tok_other = 2 + 2 * q4 + (1 - x);
        auto mufu_acquire = [&]() {
#if PISA_MUFU_PINGPONG
            asm volatile("bar.sync %0, 64;" ::"r"(tok_mine) : "memory");
#endif
        };
        auto mufu_release = [&](int g) {  // hand the unit over if the partner has a super-tile left
#if PISA_MUFU_PINGPONG
            if (g + 1 < G) asm volatile("bar.arrive %0, 64;" ::"r"(tok_other) : "memory");
#endif
        };
#if PISA_MUFU_PINGPONG
        if (x == 1) asm volatile("bar.arrive %0, 64;" ::"r"(tok_other) : "memory");  // warpgroup 0 goes first
#endif

        // ---- Phase 1: exact blocks of the union, two per super-tile
        UnionCursor cur(maskA, maskB);
        int g = 0;
        for (; g < G1; ++g) {
            uint32_t e0, e1;
            cur.pair(g, nU, e0, e1);  // pad: use flags 0
            if ((g & 1) != x) continue;
            const bool use0 = (e0 >> (14 + blk)) & 1u, use1 = (e1 >> (14 + blk)) & 1u;  // warp-uniform
            const int nv0 = (int(e0 & 0x3FFFu) == a.N - 1) ? n_last : 64;
            const int nv1 = (int(e1 & 0x3FFFu) == a.N - 1) ? n_last : 64;
            mbar_wait<true>(&bar.s_full[x], uint32_t((g >> 1) & 1));
            tc_fence_after();
            if (q4 == 0) TRACE(4 + x, g);
            mufu_acquire();
            // a sub-tile's scores as raw bits, masked in place (only the ragged
            // last key block / rows past L need masks)
            auto load = [&](uint32_t addr, int nv, uint32_t (&r0)[32], uint32_t (&r1)[32]) {
                tmem_ld32(addr, r0);
                tmem_ld32(addr + 32, r1);
                tmem_ld_wait(r0);
                tmem_ld_wait(r1);
                if (!(wact && nv == 64)) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        if (!(active && i < nv)) r0[i] = 0xff800000u;  // -inf
                        if (!(active && i + 32 < nv)) r1[i] = 0xff800000u;
                    }
                }
            };
            if (use0) {
                uint32_t r0[32], r1[32];
                load(sc, nv0, r0, r1);
                l += subtile(r0, r1, sc, 0u, -1, unused_plast);
            } else {
                zero_store(sc);
            }
            if (use1) {
                uint32_t r0[32], r1[32];
                load(sc + 64, nv1, r0, r1);
                l += subtile(r0, r1, sc + 64, use0 ? sc : 0u, -1, unused_plast);
            } else {
                zero_store(sc + 64);
            }
            mufu_release(g);
            publish_p(g);
        }
        // ---- Phase 2: centroid chunks, two per super-tile; column mask = own
        // selection, weight n_j (the ragged last block weighs n_last)
        for (g = G1 + ((G1 & 1) != x ? 1 : 0); g < G; g += 2) {
            const int c0 = 2 * (g - G1);
            mbar_wait<true>(&bar.s_full[x], uint32_t((g >> 1) & 1));
            tc_fence_after();
            // column of the ragged last block within this super-tile (0..127), if here
            const int lb = n_last != 64 ? a.N - 1 - c0 * 64 : -1;
            mufu_acquire();
#pragma unroll 1
            for (int st = 0; st < 2; ++st) {
                const int c = c0 + st;
                // the 64 columns of chunk c: blocks c*64 + i, masked when selected or >= N
                const uint32_t cm0 = (c < a.nchunk2 && 2 * c < a.W) ? hmask[2 * c] : 0xffffffffu;
                const uint32_t cm1 = (c < a.nchunk2 && 2 * c + 1 < a.W) ? hmask[2 * c + 1] : 0xffffffffu;
                const int nv = min(64, a.N - c * 64);
                uint32_t r0[32], r1[32];
                tmem_ld32(sc + 64 * st, r0);
                tmem_ld32(sc + 64 * st + 32, r1);
                tmem_ld_wait(r0);
                tmem_ld_wait(r1);
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if (!(active && i < nv && !((cm0 >> i) & 1u))) r0[i] = 0xff800000u;
                    if (!(active && i + 32 < nv && !((cm1 >> i) & 1u))) r1[i] = 0xff800000u;
                }
                const int lbo = (lb >= 64 * st && lb < 64 * st + 64) ? lb - 64 * st : -1;
                float plast = 0.f;
                const float ps = subtile(r0, r1, sc + 64 * st, st ? sc : 0u, lbo, plast);
                // (sums enter l / lt per sub-tile: a raise in the second one rescales them)
                l += 64.f * ps + (float(n_last) - 64.f) * plast;
                lt += ps;
            }
            mufu_release(g);
            publish_p(g);
        }

        // ------------------------------------------------------- epilogue --
        mbar_wait(&bar.qh_full, 0);
        tc_fence_after();
        if (warp == 4) TRACE(13, 2);  // tail: O and QH complete
        // merge the two warpgroups' partial softmaxes of the row (exchange
        // through the now idle V stages)
        float* xch = reinterpret_cast<float*>(smem + Cfg::kOffV);
        xch[(x * 3 + 0) * 128 + row] = m;
        xch[(x * 3 + 1) * 128 + row] = l;
        xch[(x * 3 + 2) * 128 + row] = lt;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const float m0 = xch[0 * 128 + row], l0 = xch[1 * 128 + row], lt0 = xch[2 * 128 + row];
        const float m1 = xch[3 * 128 + row], l1 = xch[4 * 128 + row], lt1 = xch[5 * 128 + row];
        float mrow = fmaxf(m0, m1);
        const bool hasO1 = G >= 2;  // O_1 written (else its TMEM columns are undefined)
        const float f0 = (m0 == -INFINITY) ? 0.f : ex2(m0 - mrow);
        const float f1 = (m1 == -INFINITY || !hasO1) ? 0.f : ex2(m1 - mrow);
        float lfin = l0 * f0 + l1 * f1;
        float ltot = lt0 * f0 + lt1 * f1;
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
                for (int c = 0; c < D; ++c) dot = fmaf(__bfloat162float(qrow[c]), kg[c], dot);
            }
            const float gx = dot * sl2;
            const int nUc = a.N - a.k;
            if (active && nUc > 0) {
                const float mm = fmaxf(mrow, gx);
                fo = ex2(mrow - mm);
                cw = a.scale * float(nUc) * ex2(gx - mm);  // pisa_reference: no literal_phase3
                mrow = mm;
                lfin *= fo;
                ltot *= fo;
            }
        }
        const float inv_l = 1.0f / lfin;
        const float w0 = f0 * fo * inv_l, w1 = f1 * fo * inv_l, wq = cw * inv_l;
        bool bad = false;
        char* orow = reinterpret_cast<char*>(a.out) +
                     (size_t(b) * a.os_b + size_t(h) * a.os_h + size_t(grow) * a.os_l) * (a.out_f32 ? 4 : 2);
        // this warpgroup's D/2 columns of the row
#pragma unroll 1
        for (int cc = x * (D / 2); cc < (x + 1) * (D / 2); cc += 32) {
            uint32_t r0[32], r1[32], rq[32];
            tmem_ld32(lbase + cc, r0);
            if (hasO1) tmem_ld32(lbase + D + cc, r1);
            if (first_order) tmem_ld32(lbase + kColS + cc, rq);
            tmem_ld_wait(r0);
            tmem_ld_wait(r1);
            tmem_ld_wait(rq);
            float o[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                float acc = __uint_as_float(r0[i]) * w0;
                if (hasO1) acc = fmaf(__uint_as_float(r1[i]), w1, acc);
                if (first_order) acc = fmaf(wq, __uint_as_float(rq[i]), acc);
                o[i] = acc;
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
            if (x == 0) {
                const size_t di = size_t(bh) * a.L + grow;
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
    (void)N;
    return 1024 + core + size_t(2 * W) * 4 + 16;
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
