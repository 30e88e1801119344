// K2: block scoring + top-k routing (the "select" step, engine.hpp:443-457).
//
// Replaces select_topk_plain (router.hpp:126-151) with topk_ascending (:96-108)
// and force_block (:111-121), in two launches:
//   K2a score_kernel : s_ij = scale * <q_bar_i, k_bar_j> on tcgen05 from an exact
//                      3-way bf16 split (fp32-accurate, deterministic; SURVEY.md
//                      §0: fp32 scoring keeps the index sets bit-exact against
//                      the fp64 reference on the Wan shapes, plain bf16 / TF32
//                      does not), stored as order-preserving uint32 keys; from
//                      N >= 512 the pipelined select_fused_kernel<D, true>
//   K2b topk_kernel  : one warp per query block: radix select of the k-th largest
//                      key, ties to the LOWER index, ballot compaction to the
//                      ascending index list plus the bitmask row.
#include "kernels.h"
#include "sm100.cuh"

namespace pisa_b200 {
using namespace pisa_sm100;

namespace {


__device__ __forceinline__ uint32_t order_key(float f) {
    if (f == 0.0f) f = 0.0f;  // -0 == +0 as in the fp64 comparison
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// K2a: score tile on the tensor cores. keys[bh][i][j] = order_key(scale *
// <q_bar_i, k_bar_j> [+ rect_j]) for a 128 x 128 tile of (query block, key
// block) pairs. q_bar / k_bar (fp32) are split exactly (to 2^-27 relative) into
// bf16 hi + mid + lo parts; the six cross products above 2^-26 run as tcgen05
// MMAs (bf16 products are exact, fp32 accumulation), so the scores carry fp32
// accuracy (at least that of the reference-order fp32 dot product) and are
// deterministic. 256 threads: all split, warp 0 issues, all eight read TMEM
// (warp w: lane quadrant w % 4, columns (w / 4) * 64 ..).
constexpr int kTile = 128;
constexpr int kScoreThreads = 256;

template <int D>
struct ScoreCfg {
    static constexpr int kPart = kTile * D * 2;  // one bf16 operand part (K-major, SW128 halves of 64)
    static constexpr int kOffB = 3 * kPart;      // A: hi | mid | lo, then B: hi | mid | lo
    static constexpr int kSmem = 1024 + 6 * kPart + 64;
};

// x = hi + mid + lo, each a bf16 pair (exact to 2^-27 relative)
__device__ __forceinline__ void split3(float x0, float x1, uint32_t& h, uint32_t& m, uint32_t& l) {
    const __nv_bfloat162 h2 = __floats2bfloat162_rn(x0, x1);
    const float2 hf = __bfloat1622float2(h2);
    const float y0 = x0 - hf.x, y1 = x1 - hf.y;  // exact
    const __nv_bfloat162 m2 = __floats2bfloat162_rn(y0, y1);
    const float2 mf = __bfloat1622float2(m2);
    const __nv_bfloat162 l2 = __floats2bfloat162_rn(y0 - mf.x, y1 - mf.y);
    h = *reinterpret_cast<const uint32_t*>(&h2);
    m = *reinterpret_cast<const uint32_t*>(&m2);
    l = *reinterpret_cast<const uint32_t*>(&l2);
}

// rect (covariance router, router.hpp:176-183): per key block log(M_j + eps),
// added after the scaled dot product; null for the plain router.
template <int D>
__global__ void __launch_bounds__(kScoreThreads, 1) score_kernel(const float* __restrict__ qbar,
                                                                 const float* __restrict__ kbar,
                                                                 const float* __restrict__ rect,
                                                                 uint32_t* __restrict__ keys, int N,
                                                                 float scale) {
    using Cfg = ScoreCfg<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* done = reinterpret_cast<uint64_t*>(smem + 6 * Cfg::kPart);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    const int bh = blockIdx.z;
    const int i0 = blockIdx.y * kTile, j0 = blockIdx.x * kTile;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tslot, 128);
        tmem_relinquish();
    }
    // split q_bar rows i0.. (A) and k_bar rows j0.. (B), 4 fp32 per step, into
    // the 128B-swizzled K-major bf16 parts
    constexpr int kQ4 = D / 4;  // float4 per row
    const float* qb = qbar + size_t(bh) * N * D;
    const float* kb = kbar + size_t(bh) * N * D;
    // 16 independent 16-byte loads in flight per thread (one CTA per SM: the
    // load phase is latency-bound otherwise)
    constexpr int kPer = 2 * kTile * kQ4 / kScoreThreads;  // float4 per thread (32 / 16)
    constexpr int kBatch = 16;
#pragma unroll
    for (int b0 = 0; b0 < kPer; b0 += kBatch) {
        float4 x[kBatch];
#pragma unroll
        for (int t = 0; t < kBatch; ++t) {
            const int e = tid + (b0 + t) * kScoreThreads;
            const int op = e / (kTile * kQ4), r = (e / kQ4) % kTile, c = (e % kQ4) * 4;
            const int row = (op ? j0 : i0) + r;
            x[t] = row < N ? __ldg(reinterpret_cast<const float4*>((op ? kb : qb) + size_t(row) * D + c))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int t = 0; t < kBatch; ++t) {
            const int e = tid + (b0 + t) * kScoreThreads;
            const int op = e / (kTile * kQ4), r = (e / kQ4) % kTile, c = (e % kQ4) * 4;
            uint2 h, m, l;
            split3(x[t].x, x[t].y, h.x, m.x, l.x);
            split3(x[t].z, x[t].w, h.y, m.y, l.y);
            const uint32_t off = uint32_t(op * Cfg::kOffB + (c >> 6) * (kTile * 128)) + sw128_off(r, c & 63);
            *reinterpret_cast<uint2*>(smem + off) = h;
            *reinterpret_cast<uint2*>(smem + off + Cfg::kPart) = m;
            *reinterpret_cast<uint2*>(smem + off + 2 * Cfg::kPart) = l;
        }
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (warp == 0) {
        if (elect_one()) {
            constexpr uint32_t idesc = idesc_bf16(128, 128, 0, 0);
            const uint32_t base = smem_u32(smem);
            // (lo,hi) (hi,lo) (mid,mid) (mid,hi) (hi,mid) (hi,hi): small terms first
            constexpr int kA[6] = {2, 0, 1, 1, 0, 0}, kB[6] = {0, 2, 1, 0, 1, 0};
#pragma unroll
            for (int p = 0; p < 6; ++p)
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t off = uint32_t((ks >> 2) * (kTile * 128) + (ks & 3) * 32);
                    mma_ss(tmem, sdesc_sw128(base + kA[p] * Cfg::kPart + off, 16, 1024),
                           sdesc_sw128(base + Cfg::kOffB + kB[p] * Cfg::kPart + off, 16, 1024), idesc,
                           p != 0 || ks != 0);
                }
            mma_commit(done);
        }
        __syncwarp();
    }
    mbar_wait(done, 0);
    tc_fence_after();
    // epilogue: keys of row i (TMEM lane), 64 columns per warp, staged through
    // shared memory (the operand parts are dead) so that each row leaves as
    // coalesced 128-byte warp stores (rows of `keys` are N * 4 bytes apart,
    // generally not 16-byte aligned)
    constexpr int kTS = kTile + 1;  // padded row: conflict-free row writes and column reads
    uint32_t* T = reinterpret_cast<uint32_t*>(smem);
    const int q = warp & 3, ch = warp >> 2;
    const int rl = q * 32 + lane;  // local row
    const float* rc = rect ? rect + size_t(bh) * N + j0 : nullptr;
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
        uint32_t r[32];
        tmem_ld32(tmem + (uint32_t(q * 32) << 16) + ch * 64 + cc * 32, r);
        tmem_ld_wait(r);
        const int cb = ch * 64 + cc * 32;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            float v = scale * __uint_as_float(r[t]);
            if (rc && j0 + cb + t < N) v += rc[cb + t];
            T[rl * kTS + cb + t] = order_key(v);
        }
    }
    tc_fence_before();
    __syncthreads();
    for (int rr = warp; rr < kTile; rr += kScoreThreads / 32) {
        const int i = i0 + rr;
        if (i >= N) break;
        uint32_t* krow = keys + (size_t(bh) * N + i) * N + j0;
#pragma unroll
        for (int m = 0; m < kTile / 32; ++m) {
            const int c = m * 32 + lane;
            if (j0 + c < N) krow[c] = T[rr * kTS + c];
        }
    }
    if (warp == 0) tmem_dealloc(tmem, 128);
}

// K2b: per query block, radix-select the k-th largest key (8-bit digits from the
// top), then a ballot compaction in ascending index order takes every key above
// it plus the lowest-index ties: topk_ascending semantics (router.hpp:96-108).
constexpr int kRowsPerCta = 4;
#ifndef PISA_TOPK_EARLY
#define PISA_TOPK_EARLY 1  // stop the radix once the k-th key's bin is taken whole
#endif

// One query block's top-k from its N order keys in shared memory (kr), one
// warp: radix-select the k-th largest key (8-bit digits from the top, hw = 256
// shared counters), then a ballot compaction in ascending index order takes
// every key above it plus the lowest-index ties (topk_ascending,
// router.hpp:96-108), with optional diagonal forcing (force_block, :111-121)
// for query block i. Writes the ascending list (sel, may be null) and the
// bitmask row (mrow).
__device__ __forceinline__ void select_row(const uint32_t* kr, uint32_t* hw, int N, int kk, int i,
                                           bool force_diagonal, int32_t* sel, uint32_t* mrow, int lane) {
    uint32_t prefix = 0, pmask = 0;
    int rem = kk;  // rank (1-based) of the wanted element among prefix matches
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = lane; b < 256; b += 32) hw[b] = 0;
        __syncwarp();
        for (int j = lane; j < N; j += 32) {
            const uint32_t key = kr[j];
            if ((key & pmask) == prefix) atomicAdd(&hw[(key >> shift) & 255u], 1u);
        }
        __syncwarp();
        // lane l owns digits [255 - 8l - 7, 255 - 8l], scanned from the top
        int cnt[8], tot = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            cnt[t] = int(hw[255 - lane * 8 - t]);
            tot += cnt[t];
        }
        int incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int excl = incl - tot;
        int digit = -1, above = 0, dcnt = 0;
        if (rem > excl && rem <= incl) {
            int run = excl;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                if (digit < 0 && rem <= run + cnt[t]) {
                    digit = 255 - lane * 8 - t;
                    above = run;
                    dcnt = cnt[t];
                }
                run += cnt[t];
            }
        }
        const uint32_t owner = __ballot_sync(0xffffffffu, digit >= 0);
        const int src_lane = __ffs(owner) - 1;
        digit = __shfl_sync(0xffffffffu, digit, src_lane);
        above = __shfl_sync(0xffffffffu, above, src_lane);
        dcnt = __shfl_sync(0xffffffffu, dcnt, src_lane);
        rem -= above;
        prefix |= uint32_t(digit) << shift;
        pmask |= 255u << shift;
        __syncwarp();  // every read of hw precedes the next pass's clear
#if PISA_TOPK_EARLY
        // the bin holds exactly the keys still wanted: all of it is taken (see
        // select_row_reg); T = its minimum, every tie of T kept
        if (PISA_TOPK_EARLY && dcnt == rem && shift > 0) {
            uint32_t mn = 0xffffffffu;
            for (int j = lane; j < N; j += 32) {
                const uint32_t key = kr[j];
                if ((key & pmask) == prefix) mn = min(mn, key);
            }
            prefix = __reduce_min_sync(0xffffffffu, mn);
            int ties = 0;
            for (int j = lane; j < N; j += 32) ties += kr[j] == prefix;
            rem = __reduce_add_sync(0xffffffffu, ties);
            break;
        }
#endif
    }
    const uint32_t T = prefix;  // key of the k-th largest; take `rem` ties, lowest indices first

    const uint32_t lt_mask = (1u << lane) - 1u;
    int swap_out = -1;  // force_diagonal: the kept tie to drop (worst kept, highest index)
    bool swap_in = false;
    if (force_diagonal && i < N) {
        int ties = 0, last_tie = -1;
        bool diag_sel = false;
        for (int j0 = 0; j0 < N; j0 += 32) {
            const int j = j0 + lane;
            const uint32_t key = j < N ? kr[j] : 0u;
            const bool eq = j < N && key == T;
            const uint32_t eqb = __ballot_sync(0xffffffffu, eq);
            const int rank = ties + __popc(eqb & lt_mask);
            const bool take = j < N && (key > T || (eq && rank < rem));
            if (j == i) diag_sel = take;
            const uint32_t tb = __ballot_sync(0xffffffffu, eq && rank < rem);
            if (tb) last_tie = j0 + 31 - __clz(tb);
            ties += __popc(eqb);
        }
        diag_sel = __shfl_sync(0xffffffffu, diag_sel, i & 31);
        if (!diag_sel) {
            swap_out = last_tie;
            swap_in = true;
        }
    }
    int ties = 0, out = 0;
    for (int j0 = 0; j0 < N; j0 += 32) {
        const int j = j0 + lane;
        const uint32_t key = j < N ? kr[j] : 0u;
        const bool eq = j < N && key == T;
        const uint32_t eqb = __ballot_sync(0xffffffffu, eq);
        const int rank = ties + __popc(eqb & lt_mask);
        bool take = j < N && (key > T || (eq && rank < rem));
        if (swap_in) {
            if (j == swap_out) take = false;
            if (j == i) take = true;
        }
        const uint32_t tb = __ballot_sync(0xffffffffu, take);
        if (take && sel) sel[out + __popc(tb & lt_mask)] = j;
        if (lane == 0) mrow[j0 >> 5] = tb;
        out += __popc(tb);
        ties += __popc(eqb);
    }
}

// select_row with the row's keys in registers (key j = t * 32 + lane in
// kr[t], kPer >= ceil(N / 32)): no shared-memory round trip per element and
// pass, and the radix stops early once the bin holding the k-th largest key
// holds exactly the keys still wanted -- then every key of that bin is taken,
// T is its minimum and all of T's ties are kept, which is the same index set
// the full radix yields (topk_kernel was instruction-issue bound: 3.9K warp
// instructions per row, profiles/r02i_topk_ncu.md).
template <int kPer>
__device__ __forceinline__ void select_row_reg(const uint32_t (&kr)[kPer], uint32_t* hw, int N, int kk, int i,
                                               bool force_diagonal, int32_t* sel, uint32_t* mrow, int lane) {
    uint32_t prefix = 0, pmask = 0;
    int rem = kk;
    bool whole = false;  // early exit: every key matching prefix / pmask is taken
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = lane; b < 256; b += 32) hw[b] = 0;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
            const int j = t * 32 + lane;
            if (j < N && (kr[t] & pmask) == prefix) atomicAdd(&hw[(kr[t] >> shift) & 255u], 1u);
        }
        __syncwarp();
        int cnt[8], tot = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            cnt[u] = int(hw[255 - lane * 8 - u]);
            tot += cnt[u];
        }
        int incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int excl = incl - tot;
        int digit = -1, above = 0, dcnt = 0;
        if (rem > excl && rem <= incl) {
            int run = excl;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (digit < 0 && rem <= run + cnt[u]) {
                    digit = 255 - lane * 8 - u;
                    above = run;
                    dcnt = cnt[u];
                }
                run += cnt[u];
            }
        }
        const uint32_t owner = __ballot_sync(0xffffffffu, digit >= 0);
        const int src_lane = __ffs(owner) - 1;
        digit = __shfl_sync(0xffffffffu, digit, src_lane);
        above = __shfl_sync(0xffffffffu, above, src_lane);
        dcnt = __shfl_sync(0xffffffffu, dcnt, src_lane);
        rem -= above;
        prefix |= uint32_t(digit) << shift;
        pmask |= 255u << shift;
        __syncwarp();
        if (dcnt == rem) {
            whole = shift > 0;
            break;
        }
    }
    uint32_t T = prefix;  // the k-th largest key (full radix), or the bin's minimum (early exit)
    if (whole) {
        uint32_t mn = 0xffffffffu;
#pragma unroll
        for (int t = 0; t < kPer; ++t)
            if (t * 32 + lane < N && (kr[t] & pmask) == prefix) mn = min(mn, kr[t]);
        T = __reduce_min_sync(0xffffffffu, mn);
        int ties = 0;
#pragma unroll
        for (int t = 0; t < kPer; ++t) ties += __popc(__ballot_sync(0xffffffffu, t * 32 + lane < N && kr[t] == T));
        rem = ties;  // every tie of T is kept
    }

    const uint32_t lt_mask = (1u << lane) - 1u;
    int swap_out = -1;
    bool swap_in = false;
    if (force_diagonal && i < N) {
        int ties = 0, last_tie = -1;
        bool diag_sel = false;
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
            const int j = t * 32 + lane;
            const uint32_t key = j < N ? kr[t] : 0u;
            const bool eq = j < N && key == T;
            const uint32_t eqb = __ballot_sync(0xffffffffu, eq);
            const int rank = ties + __popc(eqb & lt_mask);
            const bool take = j < N && (key > T || (eq && rank < rem));
            if (j == i) diag_sel = take;
            const uint32_t tb = __ballot_sync(0xffffffffu, eq && rank < rem);
            if (tb) last_tie = t * 32 + 31 - __clz(tb);
            ties += __popc(eqb);
        }
        diag_sel = __shfl_sync(0xffffffffu, diag_sel, i & 31);
        if (!diag_sel) {
            swap_out = last_tie;
            swap_in = true;
        }
    }
    int ties = 0, out = 0;
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
        if (t * 32 >= N) break;
        const int j = t * 32 + lane;
        const uint32_t key = j < N ? kr[t] : 0u;
        const bool eq = j < N && key == T;
        const uint32_t eqb = __ballot_sync(0xffffffffu, eq);
        const int rank = ties + __popc(eqb & lt_mask);
        bool take = j < N && (key > T || (eq && rank < rem));
        if (swap_in) {
            if (j == swap_out) take = false;
            if (j == i) take = true;
        }
        const uint32_t tb = __ballot_sync(0xffffffffu, take);
        if (take && sel) sel[out + __popc(tb & lt_mask)] = j;
        if (lane == 0) mrow[t] = tb;
        out += __popc(tb);
        ties += __popc(eqb);
    }
}

template <int kPer>
__global__ void __launch_bounds__(kRowsPerCta * 32) topk_reg_kernel(const uint32_t* __restrict__ keys,
                                                                    SelectArgs a) {
    __shared__ uint32_t hist[kRowsPerCta][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bh = blockIdx.y;
    const int i = blockIdx.x * kRowsPerCta + warp;
    const int N = a.N;
    if (i >= N) return;
    const uint32_t* src = keys + (size_t(bh) * N + i) * N;
    uint32_t kr[kPer];
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
        const int j = t * 32 + lane;
        kr[t] = j < N ? __ldcs(src + j) : 0u;
    }
    select_row_reg<kPer>(kr, hist[warp], N, a.k, i, a.force_diagonal != 0,
                         a.selected ? a.selected + (size_t(bh) * N + i) * a.k : nullptr,
                         a.mask + (size_t(bh) * N + i) * a.W, lane);
}

__global__ void __launch_bounds__(kRowsPerCta * 32) topk_kernel(const uint32_t* __restrict__ keys,
                                                                SelectArgs a) {
    extern __shared__ uint32_t smk[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bh = blockIdx.y;
    const int i = blockIdx.x * kRowsPerCta + warp;
    const int N = a.N;
    uint32_t* kr = smk + warp * (N + 256);
    uint32_t* hw = kr + N;
    if (i >= N) return;
    const uint32_t* src = keys + (size_t(bh) * N + i) * N;
    for (int j = lane; j < N; j += 32) kr[j] = src[j];
    __syncwarp();
    select_row(kr, hw, N, a.k, i, a.force_diagonal != 0,
               a.selected ? a.selected + (size_t(bh) * N + i) * a.k : nullptr,
               a.mask + (size_t(bh) * N + i) * a.W, lane);
}

// ------------------------------------------------------------------ K2 fused --
// One CTA per (128 query blocks i0.., b*h), 256 threads, one CTA per SM:
//   all warps  : q_bar rows -> exact bf16 hi / mid / lo split -> TMEM (the A
//                operand of every score MMA, 3 x D/2 columns)
//   warp 0     : TMA of the k_bar split tiles (128 key blocks x D, 3 parts),
//                double-buffered
//   warp 1     : 6 cross products x D/16 TS MMAs per key tile into one of two
//                TMEM accumulators (the same products, in the same order, as
//                score_kernel: fp32-accurate, deterministic)
//   warps 4-7  : order keys of the tile (scale * s [+ rect]) -> this SM's
//                scratch, column-major ([key][row]: 128-byte warp stores)
// then all 8 warps select the top-k of the CTA's rows, RB rows at a time
// staged through the (now free) tile buffers. The scratch is indexed by the
// SM, so successive CTAs on an SM overwrite the same lines: the keys live in
// L2 and never make the HBM round trip of the two-kernel path.
constexpr int kFThreads = 256;

template <int D>
struct FusedSelCfg {
    static constexpr int kPart = 128 * D * 2;    // one split part of a 128-key tile
    static constexpr int kStage = 3 * kPart;     // hi | mid | lo
    static constexpr int kSmem = 1024 + 2 * kStage + 256;
    static constexpr int kAcol = D / 2;          // TMEM columns per A part
    static constexpr int kOffT = 2 * kStage + 256;               // score-only: 4 x [32][33] u32 transposes
    static constexpr int kSmemScore = 1024 + kOffT + 4 * 32 * 33 * 4;
};

__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

// kScoreOnly: the same pipelined scoring, but the keys go to the row-major
// [BH][N][N] array of the two-kernel path (each epilogue warp transposes its
// 32 x 32 block in shared memory so every row leaves as 128-byte warp stores)
// and topk_kernel selects afterwards at full occupancy: score_kernel's
// operands without its one-CTA-per-tile load -> MMA -> store serialisation.
template <int D, bool kScoreOnly = false>
__global__ void __launch_bounds__(kFThreads, 1)
    select_fused_kernel(const __grid_constant__ CUtensorMap tmKs, SelectArgs a, uint32_t* __restrict__ scratch,
                        int BH) {
    using Cfg = FusedSelCfg<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * Cfg::kStage);
    uint64_t* bfull = bars;       // [2]
    uint64_t* bempty = bars + 2;  // [2]
    uint64_t* afull = bars + 4;   // [2]
    uint64_t* aempty = bars + 6;  // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = a.N;
    const int i0 = blockIdx.x * 128;
    const int bh = blockIdx.y;
    const int nt = (N + 127) / 128;
    const uint32_t sm = kScoreOnly ? 0u : smid();
    if (sm >= uint32_t(kScratchSlots)) __trap();  // the scratch has one slot per SM id
    uint32_t* ks = scratch + size_t(sm) * 128 * N;  // [key][row], this SM's slot

    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bfull[s], 1);
            mbar_init(&bempty[s], 1);
            mbar_init(&afull[s], 1);
            mbar_init(&aempty[s], 4);
        }
        fence_mbar_init();
        tma_prefetch(&tmKs);
    }
    if (warp == 1) {
        tmem_alloc(tslot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    // A operand: row i0 + r of q_bar, split exactly into three bf16 parts,
    // packed pairs in TMEM columns [part * D/2, +D/2) of lane r. Warps w and
    // w + 4 share lane quadrant w % 4 and take the two column halves.
    {
        const int q4 = warp & 3, r = q4 * 32 + lane, i = i0 + r;
        const int c0 = (warp >> 2) * (D / 2);
        const float* src = a.qbar + (size_t(bh) * N + i) * D + c0;
        constexpr int kP = D / 4;  // packed pairs per warp half: 32 (D = 128) or 16 (D = 64)
        uint32_t h[kP], m[kP], l[kP];
#pragma unroll
        for (int e = 0; e < kP; ++e) {
            const float2 x = i < N ? *reinterpret_cast<const float2*>(src + 2 * e) : make_float2(0.f, 0.f);
            split3(x.x, x.y, h[e], m[e], l[e]);
        }
        const uint32_t lb = tmem + (uint32_t(q4 * 32) << 16) + uint32_t(c0 / 2);
        if constexpr (D == 128) {
            tmem_st32(lb, h);
            tmem_st32(lb + Cfg::kAcol, m);
            tmem_st32(lb + 2 * Cfg::kAcol, l);
        } else {
            tmem_st16(lb, h);
            tmem_st16(lb + Cfg::kAcol, m);
            tmem_st16(lb + 2 * Cfg::kAcol, l);
        }
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    constexpr uint32_t kAcc = 256;  // two accumulators of 128 columns at 256 / 384
    if (warp == 0) {
        for (int t = 0; t < nt; ++t) {
            const int s = t & 1;
            if (t >= 2) mbar_wait(&bempty[s], ((t >> 1) - 1) & 1);
            if (elect_one()) {
                mbar_expect_tx(&bfull[s], Cfg::kStage);
                uint8_t* st = smem + s * Cfg::kStage;
#pragma unroll
                for (int p = 0; p < 3; ++p)
#pragma unroll
                    for (int half = 0; half < D / 64; ++half)
                        tma_load_3d(st + p * Cfg::kPart + half * 16384, &tmKs, &bfull[s], half * 64, t * 128,
                                    p * BH + bh);
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_bf16(128, 128, 0, 0);
        // (lo,hi) (hi,lo) (mid,mid) (mid,hi) (hi,mid) (hi,hi): small terms first
        constexpr int kA[6] = {2, 0, 1, 1, 0, 0}, kB[6] = {0, 2, 1, 0, 1, 0};
        for (int t = 0; t < nt; ++t) {
            const int s = t & 1;
            mbar_wait(&bfull[s], (t >> 1) & 1);
            if (t >= 2) mbar_wait(&aempty[s], ((t >> 1) - 1) & 1);
            tc_fence_after();
            const uint32_t b = smem_u32(smem + s * Cfg::kStage);
            const uint32_t acc = tmem + kAcc + uint32_t(s) * 128;
            if (elect_one()) {
#pragma unroll
                for (int p = 0; p < 6; ++p)
#pragma unroll
                    for (int kq = 0; kq < D / 16; ++kq)
                        mma_ts(acc, tmem + uint32_t(kA[p] * Cfg::kAcol + kq * 8),
                               sdesc_sw128(b + kB[p] * Cfg::kPart + (kq >> 2) * 16384 + (kq & 3) * 32, 16, 1024),
                               idesc, (p | kq) != 0);
                mma_commit(&bempty[s]);
                mma_commit(&afull[s]);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        const int q4 = warp & 3, r = q4 * 32 + lane;
        const float* rc = a.rect ? a.rect + size_t(bh) * N : nullptr;
        for (int t = 0; t < nt; ++t) {
            const int s = t & 1;
            mbar_wait(&afull[s], (t >> 1) & 1);
            tc_fence_after();
            const uint32_t acc = tmem + kAcc + uint32_t(s) * 128 + (uint32_t(q4 * 32) << 16);
#pragma unroll 1
            for (int cc = 0; cc < 128; cc += 32) {
                uint32_t v[32];
                tmem_ld32(acc + cc, v);
                tmem_ld_wait(v);
                const int j0 = t * 128 + cc;
                if constexpr (kScoreOnly) {
                    uint32_t* T = reinterpret_cast<uint32_t*>(smem + Cfg::kOffT) + q4 * 32 * 33;
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        float x = a.scale * __uint_as_float(v[e]);
                        if (rc && j0 + e < N) x += rc[j0 + e];
                        T[lane * 33 + e] = order_key(x);
                    }
                    __syncwarp();
                    const int rb = i0 + q4 * 32, nr = min(32, N - rb);
                    if (j0 + lane < N) {
                        uint32_t* dst = scratch + (size_t(bh) * N + rb) * N + j0 + lane;
#pragma unroll 4
                        for (int rr = 0; rr < nr; ++rr) dst[size_t(rr) * N] = T[rr * 33 + lane];
                    }
                    __syncwarp();
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const int j = j0 + e;
                        if (j < N) {
                            float x = a.scale * __uint_as_float(v[e]);
                            if (rc) x += rc[j];
                            ks[size_t(j) * 128 + r] = order_key(x);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&aempty[s]);
        }
    }
    tc_fence_before();
    __syncthreads();  // every key of the CTA's rows is in the scratch (block-scope ordering)
    tc_fence_after();
    if constexpr (kScoreOnly) {
        if (warp == 1) tmem_dealloc(tmem, 512);
        return;
    }
    // top-k of rows [i0, i0 + nrows): RB rows per round, transposed into smem
    // (coalesced 128-byte reads of the [key][row] scratch), one warp per row
    const int nrows = min(128, N - i0);
    const int RB = max(1, min(32, (2 * Cfg::kStage - 8 * 256 * 4) / ((N + 1) * 4)));
    uint32_t* kr_all = reinterpret_cast<uint32_t*>(smem);
    uint32_t* hist = kr_all + RB * (N + 1);
    for (int r0 = 0; r0 < nrows; r0 += RB) {
        const int nr = min(RB, nrows - r0);
        for (int idx = threadIdx.x; idx < RB * N; idx += kFThreads) {
            const int j = idx / RB, rr = idx % RB;
            if (rr < nr) kr_all[rr * (N + 1) + j] = ks[size_t(j) * 128 + r0 + rr];
        }
        __syncthreads();
        for (int rr = warp; rr < nr; rr += kFThreads / 32) {
            const int i = i0 + r0 + rr;
            select_row(kr_all + rr * (N + 1), hist + warp * 256, N, a.k, i, a.force_diagonal != 0,
                       a.selected ? a.selected + (size_t(bh) * N + i) * a.k : nullptr,
                       a.mask + (size_t(bh) * N + i) * a.W, lane);
        }
        __syncthreads();
    }
    if (warp == 1) tmem_dealloc(tmem, 512);
}

__global__ void plan_to_mask_kernel(const int32_t* __restrict__ selected, int N, int k, int W,
                                    uint32_t* __restrict__ mask, int* bad) {
    const int bh = blockIdx.y;
    const int i = blockIdx.x;
    uint32_t* mrow = mask + (size_t(bh) * N + i) * W;
    const int32_t* srow = selected + (size_t(bh) * N + i) * k;
    for (int w = threadIdx.x; w < W; w += blockDim.x) mrow[w] = 0u;
    __syncthreads();
    for (int p = threadIdx.x; p < k; p += blockDim.x) {
        const int j = srow[p];
        if (j < 0 || j >= N || (p > 0 && j <= srow[p - 1])) {
            atomicExch(bad, 1);
            continue;
        }
        atomicOr(&mrow[j >> 5], 1u << (j & 31));
    }
}

// K2b: the register-resident top-k up to N = 2048 key blocks, keys per lane
// rounded up to a few buckets (Wan2.1-14B's N = 1182: 40); PISA_TOPK_REG=0:
// always the shared-memory form
#ifndef PISA_TOPK_REG
#define PISA_TOPK_REG 8  // largest keys-per-lane bucket of the register form (0: never)
#endif
cudaError_t launch_topk(const SelectArgs& a, int BH, const uint32_t* keys, cudaStream_t s) {
    const dim3 grid((a.N + kRowsPerCta - 1) / kRowsPerCta, BH), block(kRowsPerCta * 32);
    const int per = (a.N + 31) / 32;
#define PISA_TOPK_BUCKET(P)                                      \
    if (P <= PISA_TOPK_REG && per <= P) {                             \
        topk_reg_kernel<P><<<grid, block, 0, s>>>(keys, a);      \
        return cudaGetLastError();                               \
    }
    PISA_TOPK_BUCKET(4)
    PISA_TOPK_BUCKET(8)
    PISA_TOPK_BUCKET(16)
    PISA_TOPK_BUCKET(24)
    PISA_TOPK_BUCKET(32)
    PISA_TOPK_BUCKET(40)
    PISA_TOPK_BUCKET(48)
    PISA_TOPK_BUCKET(64)
#undef PISA_TOPK_BUCKET
    const size_t smem = sizeof(uint32_t) * size_t(kRowsPerCta) * (a.N + 256);
    cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    topk_kernel<<<grid, block, smem, s>>>(keys, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_select(int D, const SelectArgs& a, int BH, uint32_t* keys, cudaStream_t s) {
    const int nt = (a.N + kTile - 1) / kTile;
    dim3 g1(nt, nt, BH);
    if (D == 128) {
        cudaFuncSetAttribute(score_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, ScoreCfg<128>::kSmem);
        score_kernel<128><<<g1, kScoreThreads, ScoreCfg<128>::kSmem, s>>>(a.qbar, a.kbar, a.rect, keys, a.N, a.scale);
    } else {
        cudaFuncSetAttribute(score_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, ScoreCfg<64>::kSmem);
        score_kernel<64><<<g1, kScoreThreads, ScoreCfg<64>::kSmem, s>>>(a.qbar, a.kbar, a.rect, keys, a.N, a.scale);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_topk(a, BH, keys, s);
}

cudaError_t launch_select_stream(int D, const CUtensorMap& tmKs, const SelectArgs& a, int BH, uint32_t* keys,
                                 cudaStream_t s) {
    dim3 grid((a.N + 127) / 128, BH);
    if (D == 128) {
        auto k = select_fused_kernel<128, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FusedSelCfg<128>::kSmemScore);
        k<<<grid, kFThreads, FusedSelCfg<128>::kSmemScore, s>>>(tmKs, a, keys, BH);
    } else {
        auto k = select_fused_kernel<64, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FusedSelCfg<64>::kSmemScore);
        k<<<grid, kFThreads, FusedSelCfg<64>::kSmemScore, s>>>(tmKs, a, keys, BH);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_topk(a, BH, keys, s);
}

cudaError_t launch_select_fused(int D, const CUtensorMap& tmKs, const SelectArgs& a, int BH, uint32_t* keys,
                                cudaStream_t s) {
    dim3 grid((a.N + 127) / 128, BH);
    if (D == 128) {
        auto k = select_fused_kernel<128>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FusedSelCfg<128>::kSmem);
        k<<<grid, kFThreads, FusedSelCfg<128>::kSmem, s>>>(tmKs, a, keys, BH);
    } else {
        auto k = select_fused_kernel<64>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FusedSelCfg<64>::kSmem);
        k<<<grid, kFThreads, FusedSelCfg<64>::kSmem, s>>>(tmKs, a, keys, BH);
    }
    return cudaGetLastError();
}

cudaError_t launch_plan_to_mask(const int32_t* selected, int N, int k, int W, uint32_t* mask,
                                int* bad, int BH, cudaStream_t s) {
    plan_to_mask_kernel<<<dim3(N, BH), 128, 0, s>>>(selected, N, k, W, mask, bad);
    return cudaGetLastError();
}

namespace {
__global__ void rectifier_kernel(const float* __restrict__ m, double eps, float* __restrict__ rect, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) rect[i] = float(log(double(m[i]) + eps));
}
}  // namespace

cudaError_t launch_rectifier(const float* m, double eps, float* rect, int n, cudaStream_t s) {
    rectifier_kernel<<<(n + 255) / 256, 256, 0, s>>>(m, eps, rect, n);
    return cudaGetLastError();
}

}  // namespace pisa_b200
