// K1: block statistics (the "prepare" step of pisa_multihead, engine.hpp:437-441).
//
// Replaces compute_block_stats (block_stats.hpp:155-202), the H_bar part of
// compute_global_stats (:207-226) and query_block_means (:259-278). One CTA
// streams kStatsG consecutive 64-row blocks of one (batch, head):
//   * warp 0     : TMA producer, 3-stage ring of {K, V, Q} 64-row tiles (128B swizzle)
//   * warp 1     : tcgen05 MMA issuer: TMEM[a][c] += sum_rows K[r][a] V[r][c]
//                  (both operands MN-major straight from the TMA image)
//   * warps 2..5 : one thread per column: fp32 column sums -> k_bar, v_hat, q_bar;
//                  epilogue: partial H = K^T V - sum_j k_bar_j (x) v_hat_j
// The first-order moment uses the identity
//   sum_n (k_n - k_bar)^T v_n = sum_n k_n^T v_n - k_bar^T v_hat      (per block)
// so the tensor core sees exact bf16 inputs and accumulates in fp32; only the
// rank-one correction runs on CUDA cores. HBM-bound: every input byte is read
// once. Ragged last block: TMA zero-fills rows >= L, means divide by n_j.
#include <algorithm>

#include "kernels.h"
#include "sm100.cuh"

namespace pisa_b200 {
using namespace pisa_sm100;

namespace {

// k_bar = hi + mid + lo, each bf16, exact to 2^-27 relative (the fused K2's
// operand split, identical to split3 in k2_select.cu)
__device__ __forceinline__ void store_split3(const StatsArgs& a, int bh, int j, int c, int D, float x) {
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const float y = x - __bfloat162float(h);
    const __nv_bfloat16 m = __float2bfloat16_rn(y);
    const __nv_bfloat16 l = __float2bfloat16_rn(y - __bfloat162float(m));
    const size_t part = size_t(a.BH) * a.N * D, o = (size_t(bh) * a.N + j) * D + c;
    a.kbar_split[o] = h;
    a.kbar_split[part + o] = m;
    a.kbar_split[2 * part + o] = l;
}

constexpr int kStages = 3;
constexpr int kCtasPerSm = 1;
constexpr int kThreads = 192;

template <int D>
struct StatsCfg {
    static constexpr int kTile = 64 * D * 2;        // one 64-row tile of K, V or Q (bytes)
    static constexpr int kStage = 3 * kTile;        // K | V | Q
    static constexpr int kRing = kStages * kStage;
    static constexpr int kKbS = kStatsG * D * 4;    // k_bar of the chunk (fp32)
    static constexpr int kRed = 2 * 4 * 3 * D * 4;  // column-sum partials, double-buffered
    static constexpr int kSmem = 1024 + kRing + 2 * kKbS + kRed + 256;
};

template <int D>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    block_stats_kernel(const __grid_constant__ CUtensorMap tmQ,
                       const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, StatsArgs a) {
    using Cfg = StatsCfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* ring = smem;
    float* kb_s = reinterpret_cast<float*>(smem + Cfg::kRing);
    float* vh_s = kb_s + kStatsG * D;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kRing + 2 * Cfg::kKbS + Cfg::kRed);
    uint64_t* full = bars;               // [kStages]
    uint64_t* empty = bars + kStages;    // [kStages]
    uint64_t* done = bars + 2 * kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int chunk = blockIdx.x;
    const int bh = blockIdx.y;
    const int b = bh / a.H, h = bh % a.H;
    const int j0 = chunk * a.G;
    const int nb = min(a.G, a.N - j0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1 + 4);  // MMA commit + 4 column warps
        }
        mbar_init(done, 1);
        fence_mbar_init();
        tma_prefetch(&tmQ);
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, 128);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        for (int jl = 0; jl < nb; ++jl) {
            const int s = jl % kStages;
            mbar_wait(&empty[s], ((jl / kStages) & 1) ^ 1);
            uint8_t* st = ring + s * Cfg::kStage;
            const int row = (j0 + jl) * 64;
            if (elect_one()) {
                mbar_expect_tx(&full[s], Cfg::kStage);
#pragma unroll
                for (int half = 0; half < D / 64; ++half) {
                    tma_load_4d(st + half * 8192, &tmK, &full[s], half * 64, row, h, b);
                    tma_load_4d(st + Cfg::kTile + half * 8192, &tmV, &full[s], half * 64, row, h, b);
                    tma_load_4d(st + 2 * Cfg::kTile + half * 8192, &tmQ, &full[s], half * 64, row, h, b);
                }
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // M = 128: for D = 128 the two MN chunks are K's column halves; for D = 64
        // the second chunk is the V tile right behind K (rows 64..127 of the
        // product are V^T V and are ignored). N = D.
        constexpr uint32_t idesc = idesc_bf16(128, D, 1, 1);
        for (int jl = 0; jl < nb; ++jl) {
            const int s = jl % kStages;
            mbar_wait(&full[s], (jl / kStages) & 1);
            tc_fence_after();
            const uint32_t kbase = smem_u32(ring + s * Cfg::kStage);
            const uint32_t vbase = kbase + Cfg::kTile;
            if (elect_one()) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint64_t ad = sdesc_sw128(kbase + ks * 2048, 8192, 1024);
                    const uint64_t bd = sdesc_sw128(vbase + ks * 2048, 8192, 1024);
                    mma_ss(tmem, ad, bd, idesc, (jl | ks) != 0);
                }
                mma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(done);
        __syncwarp();
    } else {
        // Column warps. Sums over the 64 rows: thread (row group rg, 16-byte
        // column chunk cg) adds D/16 rows of 8 columns of K, V and Q (24
        // independent fp32 accumulators, 16-byte loads), the row groups are
        // combined by shuffles and through shared memory (double-buffered by
        // block parity), then thread c owns column c. Rows past L are TMA
        // zero-fill, so they add nothing.
        const int q = warp & 3;
        const int c = q * 32 + lane;
        const bool has_col = c < D;
        const int t = threadIdx.x - 64;           // 0..127 over the four column warps
        constexpr int kCh = D / 8;                // 16-byte chunks per row
        constexpr int kRows = 64 * kCh / 128;     // rows per row group (8 / 4)
        const int cg = t % kCh, rg = t / kCh;
        float* red = vh_s + kStatsG * D;          // [2][4 warps][3][D]
        for (int jl = 0; jl < nb; ++jl) {
            const int s = jl % kStages;
            mbar_wait(&full[s], (jl / kStages) & 1);
            const int j = j0 + jl;
            const int nrow = min(64, a.L - j * 64);
            const uint8_t* st = ring + s * Cfg::kStage;
            float acc[3][8];
#pragma unroll
            for (int m = 0; m < 3; ++m)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[m][e] = 0.f;
#pragma unroll
            for (int rr = 0; rr < kRows; ++rr) {
                const int r = rg * kRows + rr;
                const uint32_t off = uint32_t((cg >> 3) * 8192 + r * 128 + (((cg & 7) ^ (r & 7)) << 4));
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    const uint4 w = *reinterpret_cast<const uint4*>(st + m * Cfg::kTile + off);
                    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = __bfloat1622float2(b2[e]);
                        acc[m][2 * e] += f.x;
                        acc[m][2 * e + 1] += f.y;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // the tile is read
            // row groups inside the warp: lanes kCh apart
#pragma unroll
            for (int o = kCh; o < 32; o <<= 1)
#pragma unroll
                for (int m = 0; m < 3; ++m)
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc[m][e] += __shfl_xor_sync(0xffffffffu, acc[m][e], o);
            float* rb = red + (jl & 1) * (4 * 3 * D) + q * (3 * D);
            if (lane < kCh) {
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    *reinterpret_cast<float4*>(rb + m * D + cg * 8) =
                        make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
                    *reinterpret_cast<float4*>(rb + m * D + cg * 8 + 4) =
                        make_float4(acc[m][4], acc[m][5], acc[m][6], acc[m][7]);
                }
            }
            asm volatile("bar.sync 2, 128;" ::: "memory");
            if (has_col) {
                const float* rb0 = red + (jl & 1) * (4 * 3 * D);
                float sk = 0.f, sv = 0.f, sq = 0.f;
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    sk += rb0[w * 3 * D + c];
                    sv += rb0[w * 3 * D + D + c];
                    sq += rb0[w * 3 * D + 2 * D + c];
                }
                const float inv = 1.0f / float(nrow);
                const float kbv = sk * inv;
                const size_t o = (size_t(bh) * a.N + j) * D + c;
                a.kbar[o] = kbv;
                a.vhat[o] = sv;
                a.qbar[o] = sq * inv;
                const size_t ob = (size_t(bh) * a.Npad + j) * D + c;
                a.kbar_bf[ob] = __float2bfloat16_rn(kbv);
                a.vhat_bf[ob] = __float2bfloat16_rn(sv);
                if (a.kbar_split) store_split3(a, bh, j, c, D, kbv);
                kb_s[jl * D + c] = kbv;
                vh_s[jl * D + c] = sv;
            }
        }
        // Zero the bf16 padding rows [N, Npad) once per (b, h).
        if (has_col && j0 + nb == a.N) {
            for (int j = a.N; j < a.Npad; ++j) {
                const size_t ob = (size_t(bh) * a.Npad + j) * D + c;
                a.kbar_bf[ob] = __float2bfloat16_rn(0.f);
                a.vhat_bf[ob] = __float2bfloat16_rn(0.f);
            }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // kb_s / vh_s complete
        mbar_wait(done, 0);
        tc_fence_after();
        // Epilogue: row a == c of the D x D partial.
        if (q < D / 32) {
            const int arow = c;
            float* dst = a.hpart + ((size_t(bh) * a.nchunk + chunk) * D + arow) * D;
#pragma unroll 1
            for (int cc = 0; cc < D; cc += 32) {
                uint32_t r[32];
                tmem_ld32(tmem + (uint32_t(q * 32) << 16) + cc, r);
                tmem_ld_wait(r);
                float acc[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) acc[i] = __uint_as_float(r[i]);
                for (int jl = 0; jl < nb; ++jl) {
                    const float ka = kb_s[jl * D + arow];
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[i] = fmaf(-ka, vh_s[jl * D + cc + i], acc[i]);
                }
#pragma unroll
                for (int i = 0; i < 32; i += 4)
                    *reinterpret_cast<float4*>(dst + cc + i) =
                        make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 128);
}

// Persistent form of the same computation (the default): one CTA per SM walks
// the flattened (b*h, chunk) list with stride gridDim.x, so the TMA ring never
// drains between chunks. The TMEM accumulator and the chunk's k_bar / v_hat
// are double-buffered, and a dedicated epilogue warpgroup turns chunk i into
// its H partial while the producer, the MMA warp and the column warps already
// stream chunk i + 1. Every chunk is computed exactly as in the one-chunk-per-
// CTA kernel above (same block order, same reductions), so the outputs are
// bit-identical; only which CTA computes a chunk changes.
#ifndef PISA_K1_DIAG
#define PISA_K1_DIAG 0
#endif
#ifndef PISA_K1_STG256
#define PISA_K1_STG256 1  // H partial written with 32-byte stores (0: 16-byte)
#endif
constexpr int kPThreads = 320;  // warp 0 TMA, 1 MMA, 2-5 columns, 6-9 epilogue

template <int D>
struct PStatsCfg {
    static constexpr int kTile = 64 * D * 2;
    static constexpr int kStage = 3 * kTile;
    static constexpr int kRing = 3 * kStage;        // 3 stages
    static constexpr int kKbS = kStatsG * D * 4;    // one chunk's k_bar (fp32)
    static constexpr int kRed = 2 * 4 * 3 * D * 4;
    static constexpr int kSmem = 1024 + kRing + 4 * kKbS + kRed + 512;
};

template <int D>
__global__ void __launch_bounds__(kPThreads, 1)
    block_stats_persistent_kernel(const __grid_constant__ CUtensorMap tmQ,
                                  const __grid_constant__ CUtensorMap tmK,
                                  const __grid_constant__ CUtensorMap tmV, StatsArgs a, int BH) {
    using Cfg = PStatsCfg<D>;
    constexpr int kS = 3;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* ring = smem;
    float* kb_s = reinterpret_cast<float*>(smem + Cfg::kRing);  // [2][G][D]
    float* vh_s = kb_s + 2 * kStatsG * D;                        // [2][G][D]
    float* red = vh_s + 2 * kStatsG * D;                         // [2][4][3][D]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kRing + 4 * Cfg::kKbS + Cfg::kRed);
    uint64_t* full = bars;             // [3] stage loaded
    uint64_t* empty = bars + 3;        // [3] stage consumed (MMA + 4 column warps)
    uint64_t* acc_full = bars + 6;     // [2] chunk's K^T V complete (MMA commit)
    uint64_t* stats_full = bars + 8;   // [2] chunk's k_bar / v_hat in smem (4 column warps)
    uint64_t* acc_empty = bars + 10;   // [2] epilogue done with the buffer (4 epilogue warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int total = BH * a.nchunk;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1 + 4);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&acc_full[s], 1);
            // every thread arrives (its own shared-memory stores / loads are
            // ordered by its own release), 4 warps each side
            mbar_init(&stats_full[s], 128);
            mbar_init(&acc_empty[s], 128);
        }
        fence_mbar_init();
        tma_prefetch(&tmQ);
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, 256);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // blocks of chunk t: (bh, j0, nb)
    auto chunk_of = [&](int t, int& bh, int& chunk, int& j0, int& nb) {
        bh = t / a.nchunk;
        chunk = t % a.nchunk;
        j0 = chunk * a.G;
        nb = min(a.G, a.N - j0);
    };

    if (warp == 0) {
        int it = 0;  // ring position over all blocks of all chunks
        for (int t = blockIdx.x; t < total; t += gridDim.x) {
            int bh, chunk, j0, nb;
            chunk_of(t, bh, chunk, j0, nb);
            const int b = bh / a.H, h = bh % a.H;
            for (int jl = 0; jl < nb; ++jl, ++it) {
                const int s = it % kS;
                mbar_wait(&empty[s], ((it / kS) & 1) ^ 1);
                uint8_t* st = ring + s * Cfg::kStage;
                const int row = (j0 + jl) * 64;
                if (elect_one()) {
                    mbar_expect_tx(&full[s], Cfg::kStage);
#pragma unroll
                    for (int half = 0; half < D / 64; ++half) {
                        tma_load_4d(st + half * 8192, &tmK, &full[s], half * 64, row, h, b);
                        tma_load_4d(st + Cfg::kTile + half * 8192, &tmV, &full[s], half * 64, row, h, b);
                        tma_load_4d(st + 2 * Cfg::kTile + half * 8192, &tmQ, &full[s], half * 64, row, h, b);
                    }
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_bf16(128, D, 1, 1);
        int it = 0, ci = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++ci) {
            int bh, chunk, j0, nb;
            chunk_of(t, bh, chunk, j0, nb);
            const int buf = ci & 1;
            if (ci >= 2) mbar_wait(&acc_empty[buf], ((ci >> 1) - 1) & 1);
            tc_fence_after();
            const uint32_t acc = tmem + uint32_t(buf) * 128;
            for (int jl = 0; jl < nb; ++jl, ++it) {
                const int s = it % kS;
                mbar_wait(&full[s], (it / kS) & 1);
                tc_fence_after();
                const uint32_t kbase = smem_u32(ring + s * Cfg::kStage);
                const uint32_t vbase = kbase + Cfg::kTile;
                if (elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        const uint64_t ad = sdesc_sw128(kbase + ks * 2048, 8192, 1024);
                        const uint64_t bd = sdesc_sw128(vbase + ks * 2048, 8192, 1024);
                        mma_ss(acc, ad, bd, idesc, (jl | ks) != 0);
                    }
                    mma_commit(&empty[s]);
                    if (jl == nb - 1) mma_commit(&acc_full[buf]);
                }
                __syncwarp();
            }
        }
    } else if (warp < 6) {
        // Column warps (as in block_stats_kernel): per-block column sums ->
        // k_bar / v_hat / q_bar, and the chunk's k_bar / v_hat into kb_s[buf]
        const int q = warp & 3;
        const int c = q * 32 + lane;
        const bool has_col = c < D;
        const int tt = threadIdx.x - 64;
        constexpr int kCh = D / 8;
        constexpr int kRows = 64 * kCh / 128;
        const int cg = tt % kCh, rg = tt / kCh;
        int it = 0, ci = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++ci) {
            int bh, chunk, j0, nb;
            chunk_of(t, bh, chunk, j0, nb);
            const int buf = ci & 1;
            float* kbs = kb_s + buf * kStatsG * D;
            float* vhs = vh_s + buf * kStatsG * D;
            // kb_s[buf] is free once the epilogue of chunk ci - 2 is done
            if (ci >= 2) mbar_wait(&acc_empty[buf], ((ci >> 1) - 1) & 1);
            for (int jl = 0; jl < nb; ++jl, ++it) {
                const int s = it % kS;
                mbar_wait(&full[s], (it / kS) & 1);
#if PISA_K1_DIAG == 1  // diagnostic only (wrong statistics): the column warps release the stage at once
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                continue;
#endif
                const int j = j0 + jl;
                const int nrow = min(64, a.L - j * 64);
                const uint8_t* st = ring + s * Cfg::kStage;
                float acc[3][8];
#pragma unroll
                for (int m = 0; m < 3; ++m)
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc[m][e] = 0.f;
#pragma unroll
                for (int rr = 0; rr < kRows; ++rr) {
                    const int r = rg * kRows + rr;
                    const uint32_t off = uint32_t((cg >> 3) * 8192 + r * 128 + (((cg & 7) ^ (r & 7)) << 4));
#pragma unroll
                    for (int m = 0; m < 3; ++m) {
                        const uint4 w = *reinterpret_cast<const uint4*>(st + m * Cfg::kTile + off);
                        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 f = __bfloat1622float2(b2[e]);
                            acc[m][2 * e] += f.x;
                            acc[m][2 * e + 1] += f.y;
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
                for (int o = kCh; o < 32; o <<= 1)
#pragma unroll
                    for (int m = 0; m < 3; ++m)
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc[m][e] += __shfl_xor_sync(0xffffffffu, acc[m][e], o);
                float* rb = red + (it & 1) * (4 * 3 * D) + q * (3 * D);
                if (lane < kCh) {
#pragma unroll
                    for (int m = 0; m < 3; ++m) {
                        *reinterpret_cast<float4*>(rb + m * D + cg * 8) =
                            make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
                        *reinterpret_cast<float4*>(rb + m * D + cg * 8 + 4) =
                            make_float4(acc[m][4], acc[m][5], acc[m][6], acc[m][7]);
                    }
                }
                asm volatile("bar.sync 2, 128;" ::: "memory");
                if (has_col) {
                    const float* rb0 = red + (it & 1) * (4 * 3 * D);
                    float sk = 0.f, sv = 0.f, sq = 0.f;
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        sk += rb0[w * 3 * D + c];
                        sv += rb0[w * 3 * D + D + c];
                        sq += rb0[w * 3 * D + 2 * D + c];
                    }
                    const float inv = 1.0f / float(nrow);
                    const float kbv = sk * inv;
                    const size_t o = (size_t(bh) * a.N + j) * D + c;
                    a.kbar[o] = kbv;
                    a.vhat[o] = sv;
                    a.qbar[o] = sq * inv;
                    const size_t ob = (size_t(bh) * a.Npad + j) * D + c;
                    a.kbar_bf[ob] = __float2bfloat16_rn(kbv);
                    a.vhat_bf[ob] = __float2bfloat16_rn(sv);
                    if (a.kbar_split) store_split3(a, bh, j, c, D, kbv);
                    kbs[jl * D + c] = kbv;
                    vhs[jl * D + c] = sv;
                }
            }
            if (has_col && j0 + nb == a.N) {
                for (int j = a.N; j < a.Npad; ++j) {
                    const size_t ob = (size_t(bh) * a.Npad + j) * D + c;
                    a.kbar_bf[ob] = __float2bfloat16_rn(0.f);
                    a.vhat_bf[ob] = __float2bfloat16_rn(0.f);
                }
            }
            mbar_arrive(&stats_full[buf]);  // release: orders this thread's k_bar / v_hat stores
        }
    } else {
        // Epilogue warps 6..9: H partial of chunk ci from TMEM buffer ci & 1,
        // lanes (warp % 4) * 32 .. +31 (= rows a of the D x D partial)
        const int q = warp & 3;  // TMEM lane quadrant this warp may access
        const int arow = q * 32 + lane;
        int ci = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++ci) {
            int bh, chunk, j0, nb;
            chunk_of(t, bh, chunk, j0, nb);
            const int buf = ci & 1;
            mbar_wait(&acc_full[buf], (ci >> 1) & 1);
            mbar_wait(&stats_full[buf], (ci >> 1) & 1);
            tc_fence_after();
            const float* kbs = kb_s + buf * kStatsG * D;
            const float* vhs = vh_s + buf * kStatsG * D;
            if (q < D / 32 && PISA_K1_DIAG != 2) {  // (2: diagnostic, no H partial written)
                float* dst = a.hpart + ((size_t(bh) * a.nchunk + chunk) * D + arow) * D;
#pragma unroll 1
                for (int cc = 0; cc < D; cc += 32) {
                    uint32_t r[32];
                    tmem_ld32(tmem + uint32_t(buf) * 128 + (uint32_t(q * 32) << 16) + cc, r);
                    tmem_ld_wait(r);
                    float acc[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[i] = __uint_as_float(r[i]);
                    for (int jl = 0; jl < nb; ++jl) {
                        const float ka = kbs[jl * D + arow];
#pragma unroll
                        for (int i = 0; i < 32; ++i) acc[i] = fmaf(-ka, vhs[jl * D + cc + i], acc[i]);
                    }
#if PISA_K1_STG256
                    // 32-byte stores: every lane writes a whole sector of its row
                    // (the row-per-thread TMEM layout scatters a warp's store over
                    // 32 lines; 16-byte stores half-filled 32 sectors per instruction)
#pragma unroll
                    for (int i = 0; i < 32; i += 8)
                        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + cc + i),
                                     "f"(acc[i]), "f"(acc[i + 1]), "f"(acc[i + 2]), "f"(acc[i + 3]), "f"(acc[i + 4]),
                                     "f"(acc[i + 5]), "f"(acc[i + 6]), "f"(acc[i + 7])
                                     : "memory");
#else
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        *reinterpret_cast<float4*>(dst + cc + i) =
                            make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
#endif
                }
            }
            tc_fence_before();
            mbar_arrive(&acc_empty[buf]);  // release: this thread's reads of the chunk are done
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 256);
}

template <int D>
__global__ void hbar_reduce_kernel(const float* __restrict__ hpart, int nchunk, int N,
                                   const float* __restrict__ kbar, float* __restrict__ hbar,
                                   __nv_bfloat16* __restrict__ hbar_bf,
                                   float* __restrict__ kbar_global) {
    const int bh = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < D * D) {
        const float* p = hpart + size_t(bh) * nchunk * D * D + e;
        float s = 0.f;
        for (int c = 0; c < nchunk; ++c) s += p[size_t(c) * D * D];
        s /= float(N);
        hbar[size_t(bh) * D * D + e] = s;
        hbar_bf[size_t(bh) * D * D + e] = __float2bfloat16_rn(s);
    }
    if (kbar_global != nullptr && blockIdx.x == 0 && threadIdx.x < D) {
        const float* kb = kbar + size_t(bh) * N * D + threadIdx.x;
        float s = 0.f;
        for (int j = 0; j < N; ++j) s += kb[size_t(j) * D];
        kbar_global[size_t(bh) * D + threadIdx.x] = s / float(N);
    }
}

template <int D>
__global__ void stats_to_bf16_kernel(const float* __restrict__ kbar,
                                     const float* __restrict__ vhat,
                                     const float* __restrict__ hbar, int N, int Npad,
                                     __nv_bfloat16* __restrict__ kbar_bf,
                                     __nv_bfloat16* __restrict__ vhat_bf,
                                     __nv_bfloat16* __restrict__ hbar_bf,
                                     float* __restrict__ kbar_global) {
    const int bh = blockIdx.y;
    const int total = Npad * D;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int j = e / D;
        const float kv = j < N ? kbar[size_t(bh) * N * D + e] : 0.f;
        const float vv = j < N ? vhat[size_t(bh) * N * D + e] : 0.f;
        kbar_bf[size_t(bh) * Npad * D + e] = __float2bfloat16_rn(kv);
        vhat_bf[size_t(bh) * Npad * D + e] = __float2bfloat16_rn(vv);
    }
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < D * D; e += gridDim.x * blockDim.x)
        hbar_bf[size_t(bh) * D * D + e] = __float2bfloat16_rn(hbar[size_t(bh) * D * D + e]);
    if (kbar_global != nullptr && blockIdx.x == 0 && threadIdx.x < D) {
        const float* kb = kbar + size_t(bh) * N * D + threadIdx.x;
        float s = 0.f;
        for (int j = 0; j < N; ++j) s += kb[size_t(j) * D];
        kbar_global[size_t(bh) * D + threadIdx.x] = s / float(N);
    }
}

}  // namespace

#ifndef PISA_K1_PERSISTENT
#define PISA_K1_PERSISTENT 1
#endif

cudaError_t launch_block_stats(int D, const CUtensorMap& tmQ, const CUtensorMap& tmK,
                               const CUtensorMap& tmV, const StatsArgs& a, int BH,
                               cudaStream_t s) {
    if (PISA_K1_PERSISTENT) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int grid = std::min(sms, BH * a.nchunk);
        if (D == 128) {
            auto k = block_stats_persistent_kernel<128>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PStatsCfg<128>::kSmem);
            k<<<grid, kPThreads, PStatsCfg<128>::kSmem, s>>>(tmQ, tmK, tmV, a, BH);
        } else {
            auto k = block_stats_persistent_kernel<64>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PStatsCfg<64>::kSmem);
            k<<<grid, kPThreads, PStatsCfg<64>::kSmem, s>>>(tmQ, tmK, tmV, a, BH);
        }
        return cudaGetLastError();
    }
    dim3 grid(a.nchunk, BH);
    if (D == 128) {
        auto k = block_stats_kernel<128>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, StatsCfg<128>::kSmem);
        k<<<grid, kThreads, StatsCfg<128>::kSmem, s>>>(tmQ, tmK, tmV, a);
    } else {
        auto k = block_stats_kernel<64>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, StatsCfg<64>::kSmem);
        k<<<grid, kThreads, StatsCfg<64>::kSmem, s>>>(tmQ, tmK, tmV, a);
    }
    return cudaGetLastError();
}

cudaError_t launch_hbar_reduce(int D, const float* hpart, int nchunk, int N, const float* kbar,
                               float* hbar, __nv_bfloat16* hbar_bf, float* kbar_global, int BH,
                               cudaStream_t s) {
    dim3 grid((D * D + 255) / 256, BH);
    if (D == 128)
        hbar_reduce_kernel<128><<<grid, 256, 0, s>>>(hpart, nchunk, N, kbar, hbar, hbar_bf, kbar_global);
    else
        hbar_reduce_kernel<64><<<grid, 256, 0, s>>>(hpart, nchunk, N, kbar, hbar, hbar_bf, kbar_global);
    return cudaGetLastError();
}

cudaError_t launch_stats_to_bf16(int D, const float* kbar, const float* vhat, const float* hbar,
                                 int N, int Npad, __nv_bfloat16* kbar_bf, __nv_bfloat16* vhat_bf,
                                 __nv_bfloat16* hbar_bf, float* kbar_global, int BH,
                                 cudaStream_t s) {
    dim3 grid(32, BH);
    if (D == 128)
        stats_to_bf16_kernel<128><<<grid, 256, 0, s>>>(kbar, vhat, hbar, N, Npad, kbar_bf, vhat_bf,
                                                       hbar_bf, kbar_global);
    else
        stats_to_bf16_kernel<64><<<grid, 256, 0, s>>>(kbar, vhat, hbar, N, Npad, kbar_bf, vhat_bf,
                                                      hbar_bf, kbar_global);
    return cudaGetLastError();
}

}  // namespace pisa_b200
