// K1c: spectral deviation norms M_j = ||H_j - H_bar||_2 per key block, the
// covariance-aware router's rectifier (compute_global_stats with compute_norms,
// block_stats.hpp:207-241; select_topk_covariance, router.hpp:157-193).
//
// sigma_max(D)^2 = lambda_max(D^T D), D = H_j - H_bar, by kLanczos steps of
// Lanczos from the normalised all-ones start (the reference's power-iteration
// start, block_stats.hpp:98); the extreme Ritz value of the tridiagonal is found
// by a warp-parallel multisection on its Sturm sequence. The reference uses the
// exact Jacobi eigen-solve in fp64 (block_stats.hpp:42-94); the extreme
// eigenvalue of D^T D is well separated after a few dozen Lanczos steps, so M_j
// agrees to fp32 rounding (~1e-6 relative, measured in the tests).
// Outputs m[bh][j] (fp32) and rect[bh][j] = log(M_j + eps) (computed in fp64).
//
// Two kernels:
//   * block_norms_tc_kernel (D = 128, the hot configuration): H_j and
//     G = D^T D on the tensor cores, Lanczos on G from registers;
//   * block_norms_kernel<64>: CUDA-core H_j and Lanczos on D^T D as two
//     matvecs per step (D = 64 is 8x less work per block).
#include <type_traits>

#include "kernels.h"
#include "sm100.cuh"

namespace pisa_b200 {
using namespace pisa_sm100;

namespace {

constexpr int kNormThreads = 256;
#ifndef PISA_K1C_PAIR_D64
#define PISA_K1C_PAIR_D64 1  // d = 64: the paired tensor-core kernel (0: CUDA-core kernel)
#endif
constexpr bool kK1cPairD64 = PISA_K1C_PAIR_D64 != 0;
#ifndef PISA_LANCZOS_STEPS
#define PISA_LANCZOS_STEPS 24
#endif
#ifndef PISA_K1C_HBAR_STAGE
#define PISA_K1C_HBAR_STAGE 1  // H_bar pre-load through shared memory (0: per-thread row loads)
#endif
#ifndef PISA_K1C_CLOCKS
#define PISA_K1C_CLOCKS 0  // diagnostic: n = 1..7 stores a phase's cycles in place of M_j
// (1 Lanczos loop, 2 tridiagonal store, 3 start -> G in registers, 4 whole CTA,
// 5 start -> K/V landed, 6 start -> CTA barrier, 7 start -> -H_bar in TMEM);
// the ritz kernel is not launched in these builds
#endif
constexpr int kLanczos = PISA_LANCZOS_STEPS;  // fp32-converged on every Wan2.1-14B block (20 steps: 0.8% off)

// Largest eigenvalue of the m x m Lanczos tridiagonal (alpha = ab[0..m),
// beta = ab[kLanczos..]) by a 32-way multisection on its Sturm count (the
// number of eigenvalues below x, from the LDL^T pivots); each round shrinks the
// bracket 33x (fp32 is the precision M_j is delivered in). One warp; lane 0
// stores M_j = sqrt(lambda_max) and the rectifier log(M_j + eps) (fp64).
__device__ __forceinline__ void ritz_max_and_store(const float* ab, int m, int lane, const NormArgs& a, size_t o) {
    float hi = 0.f;
    for (int i = 0; i < m; ++i) {
        const float r = fabsf(ab[i]) + (i > 0 ? fabsf(ab[kLanczos + i - 1]) : 0.f) +
                        (i + 1 < m ? fabsf(ab[kLanczos + i]) : 0.f);
        hi = fmaxf(hi, r);  // Gershgorin bound
    }
    float lo = 0.f;  // D^T D is positive semi-definite
    for (int round = 0; round < 7 && hi > lo; ++round) {
        const float x = lo + (hi - lo) * float(lane + 1) * (1.0f / 33.0f);
        int c = 0;
        float q = 1.f;
        for (int i = 0; i < m; ++i) {
            const float bb = i > 0 ? ab[kLanczos + i - 1] : 0.f;
            q = (ab[i] - x) - (i > 0 ? bb * bb / q : 0.f);
            if (q == 0.f) q = -1e-30f;
            c += q < 0.f;
        }
        const unsigned all_below = __ballot_sync(0xffffffffu, c >= m);  // lambda_max < x
        const int f = all_below ? __ffs(all_below) - 1 : 32;
        const float xf = __shfl_sync(0xffffffffu, x, f < 32 ? f : 31);
        const float xp = __shfl_sync(0xffffffffu, x, f > 0 ? f - 1 : 0);
        const float nlo = f > 0 ? xp : lo, nhi = f < 32 ? xf : hi;
        lo = nlo;
        hi = nhi;
    }
    if (lane == 0) {
        const double sigma = sqrt(fmax(0.0, double(0.5f * (lo + hi))));
        a.m[o] = float(sigma);
        if (a.rect) a.rect[o] = float(log(sigma + a.eps));
    }
}

// The extreme Ritz value off the K1c CTA: the tensor-core kernel stores each
// block's tridiagonal (alpha, beta, step count) and exits, and this kernel runs
// the multisection with one warp per key block at full occupancy, where the
// dependent Sturm chains of many blocks overlap. Inside K1c the single-warp
// multisection held the CTA's 64 KB of registers and 67 KB of shared memory for
// ~22K cycles, 28% of the CTA's lifetime (PISA_K1C_CLOCKS=2 before the split).
constexpr int kRitzWarps = 8;
static_assert(2 * kLanczos <= kTriStride, "tridiagonal row does not fit");
__global__ void __launch_bounds__(32 * kRitzWarps) ritz_kernel(NormArgs a, int nblk) {
    const int w = blockIdx.x * kRitzWarps + int(threadIdx.x >> 5);
    if (w >= nblk) return;
    const float* ab = a.tri + size_t(w) * kTriStride;
    ritz_max_and_store(ab, __float_as_int(ab[2 * kLanczos - 1]), threadIdx.x & 31, a, size_t(w));
}

// ---------------------------------------------------------------------------
// D = 64: one CTA (256 threads) per (key block j, batch*head):
//   1. centred keys kc = K_j - k_bar_j and V_j into shared memory (fp32; the
//      ragged last block has n < 64 rows, the rest are zero),
//   2. H_j = kc^T V_j (each thread an 8 x 8 tile, fp32, fixed order over rows),
//      D = H_j - H_bar (H_bar from K1b),
//   3. Lanczos on D^T D, two matvecs per step, two threads per row / column.
template <int D>
__global__ void __launch_bounds__(kNormThreads, 4) block_norms_kernel(const __nv_bfloat16* __restrict__ k,
                                                                   const __nv_bfloat16* __restrict__ v,
                                                                   NormArgs a) {
    extern __shared__ __align__(16) float sm[];
    float* kc = sm;                 // [64][D]  centred keys, later D (= H_j - H_bar) [D][D]
    float* vv = sm + 64 * D;        // [64][D]
    float* Dm = sm;                 // [D][D + 1] (padded: conflict-free row and column walks)
    float* vc = sm + D * (D + 1);   // Lanczos vector v_m [D]
    float* vp = vc + D;             // v_{m-1} [D]
    float* w = vp + D;              // D v_m [D]
    float* red = w + D;             // [2][8] reduction scratch (double-buffered)
    float* ab = red + 16;           // alpha [kLanczos], beta [kLanczos]
    const int j = blockIdx.x, bh = blockIdx.y;
    const int b = bh / a.H, h = bh % a.H;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = min(64, a.L - j * 64);
    const float* kb = a.kbar + (size_t(bh) * a.N + j) * D;

    // ---- 1. centred keys and values (fp32), 8 bf16 per 16-byte load
    for (int e = tid; e < 64 * D / 8; e += kNormThreads) {
        const int r = e / (D / 8), c = (e % (D / 8)) * 8;
        float kx[8], vx[8];
        if (r < n) {
            const size_t row = size_t(j) * 64 + r;
            const uint4 kw = *reinterpret_cast<const uint4*>(k + size_t(b) * a.ks_b + size_t(h) * a.ks_h + row * a.ks_l + c);
            const uint4 vw = *reinterpret_cast<const uint4*>(v + size_t(b) * a.vs_b + size_t(h) * a.vs_h + row * a.vs_l + c);
            const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kw);
            const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vw);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float2 kf = __bfloat1622float2(k2[t]), vf = __bfloat1622float2(v2[t]);
                kx[2 * t] = kf.x - kb[c + 2 * t];
                kx[2 * t + 1] = kf.y - kb[c + 2 * t + 1];
                vx[2 * t] = vf.x;
                vx[2 * t + 1] = vf.y;
            }
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t) kx[t] = vx[t] = 0.f;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            kc[r * D + c + t] = kx[t];
            vv[r * D + c + t] = vx[t];
        }
    }
    __syncthreads();
    // ---- 2. H_j = kc^T V (thread tile: rows ta*TS.., cols tb*TS..), minus
    // H_bar. TS = 4 for D = 64: every thread owns a tile and the accumulators
    // stay small enough for four CTAs per SM (the Lanczos below is latency-bound)
    constexpr int TS = D == 64 ? 4 : 8;
    constexpr int T = D / TS;  // tiles per side
    float acc[TS][TS];
    const bool owns = tid < T * T;
    const int ta = tid / T, tb = tid % T;
    if (owns) {
#pragma unroll
        for (int x = 0; x < TS; ++x)
#pragma unroll
            for (int y = 0; y < TS; ++y) acc[x][y] = 0.f;
        for (int r = 0; r < n; ++r) {
            float ka[TS], vb[TS];
#pragma unroll
            for (int x = 0; x < TS; ++x) ka[x] = kc[r * D + ta * TS + x];
#pragma unroll
            for (int y = 0; y < TS; ++y) vb[y] = vv[r * D + tb * TS + y];
#pragma unroll
            for (int x = 0; x < TS; ++x)
#pragma unroll
                for (int y = 0; y < TS; ++y) acc[x][y] = fmaf(ka[x], vb[y], acc[x][y]);
        }
        const float* hb = a.hbar + size_t(bh) * D * D;
#pragma unroll
        for (int x = 0; x < TS; ++x)
#pragma unroll
            for (int y = 0; y < TS; ++y) acc[x][y] -= hb[(ta * TS + x) * D + tb * TS + y];
    }
    __syncthreads();  // kc / vv are dead: D overwrites them
    if (owns) {
#pragma unroll
        for (int x = 0; x < TS; ++x)
#pragma unroll
            for (int y = 0; y < TS; ++y) Dm[(ta * TS + x) * (D + 1) + tb * TS + y] = acc[x][y];
    }
    // ---- 3. Lanczos on G = D^T D (three-term recurrence; without
    // re-orthogonalisation fp32 round-off only adds ghost copies of converged
    // eigenvalues, the extreme Ritz value still converges: 24 steps reach
    // <5e-8 relative on gaussian / clustered blocks)
    // Two threads per row / column: hf = tid & 1 takes half of the D terms, with
    // the walk staggered by 16 so the two halves never share a bank.
    const int rc = tid >> 1, hf = tid & 1;
    const bool live = rc < D;
    int par = 0;  // reduction scratch parity
    auto block_sum = [&](float x) -> float {  // sum over threads with hf == 0 of x
        x = hf == 0 ? x : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) red[par * 8 + warp] = x;
        __syncthreads();
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < kNormThreads / 32; ++i) s += red[par * 8 + i];
        par ^= 1;
        return s;
    };
    if (tid < D) {
        vc[tid] = rsqrtf(float(D));
        vp[tid] = 0.f;
    }
    __syncthreads();
    int m = 0;
    float beta_prev = 0.f;
    for (; m < kLanczos; ++m) {
        // w = D v_m: row rc, columns hf*D/2 + (t + 16 hf) mod D/2
        float y = 0.f;
        if (live) {
            float u0 = 0.f, u1 = 0.f, u2 = 0.f, u3 = 0.f;
            const float* row = Dm + rc * (D + 1) + hf * (D / 2);
            const float* vv2 = vc + hf * (D / 2);
#pragma unroll 4
            for (int t = 0; t < D / 2; t += 4) {
                const int c0 = (t + 16 * hf) & (D / 2 - 1);
                u0 = fmaf(row[c0], vv2[c0], u0);
                u1 = fmaf(row[c0 + 1], vv2[c0 + 1], u1);
                u2 = fmaf(row[c0 + 2], vv2[c0 + 2], u2);
                u3 = fmaf(row[c0 + 3], vv2[c0 + 3], u3);
            }
            float u = (u0 + u1) + (u2 + u3);
            u += __shfl_xor_sync(0xffffffffu, u, 1);
            if (hf == 0) w[rc] = u;
        }
        __syncthreads();
        // y = D^T w: column rc, rows hf*D/2 + (t + 16 hf) mod D/2
        if (live) {
            float y0 = 0.f, y1 = 0.f, y2 = 0.f, y3 = 0.f;
            const float* col = Dm + hf * (D / 2) * (D + 1) + rc;
            const float* ww = w + hf * (D / 2);
#pragma unroll 4
            for (int t = 0; t < D / 2; t += 4) {
                const int i0 = (t + 16 * hf) & (D / 2 - 1);
                y0 = fmaf(col[i0 * (D + 1)], ww[i0], y0);
                y1 = fmaf(col[(i0 + 1) * (D + 1)], ww[i0 + 1], y1);
                y2 = fmaf(col[(i0 + 2) * (D + 1)], ww[i0 + 2], y2);
                y3 = fmaf(col[(i0 + 3) * (D + 1)], ww[i0 + 3], y3);
            }
            y = (y0 + y1) + (y2 + y3);
            y += __shfl_xor_sync(0xffffffffu, y, 1);
        }
        const float vcur = live ? vc[rc] : 0.f;
        const float alpha = block_sum(vcur * y);
        if (live) y -= alpha * vcur + beta_prev * vp[rc];
        const float beta = sqrtf(block_sum(y * y));
        if (tid == 0) {
            ab[m] = alpha;
            ab[kLanczos + m] = beta;
        }
        if (!(beta > 1e-30f * fmaxf(1.f, fabsf(alpha)))) {  // invariant subspace (or D == 0)
            ++m;
            break;
        }
        __syncthreads();  // every thread has read vc / vp for this step
        if (live && hf == 0) {
            vp[rc] = vcur;
            vc[rc] = y / beta;
        }
        beta_prev = beta;
        __syncthreads();
    }
    __syncthreads();
    if (warp == 0) ritz_max_and_store(ab, m, lane, a, size_t(bh) * a.N + j);
}

// ---------------------------------------------------------------------------
// D = 128 (the hot configuration): everything GEMM-shaped on the tensor cores.
// One CTA (4 warps) per (key block j, batch*head), three CTAs per SM:
//   1. TMA: K_j and V_j (bf16, 128B-swizzled 64-row tiles, rows >= L zero-filled),
//   2. centring kc = K_j - k_bar_j in fp32 and an exact-to-fp32 split
//      kc = hi + mid + lo into three bf16 tiles (in place of K and behind it),
//   3. tcgen05: TMEM[a][c] = sum_rows (lo + mid + hi)[r][a] V[r][c] (12 MMAs,
//      M = N = 128, both operands MN-major; bf16 products are exact, fp32
//      accumulation) -- H_j to fp32 accuracy without the cancellation of the
//      uncentred identity,
//   4. thread a reads row a of H_j and subtracts H_bar: row a of D,
//   5. G = D^T D on the tensor cores from the same kind of split of D
//      (hi/mid/lo, the six products above 2^-26 relative), written to shared
//      memory 64 rows at a time (two passes, 24 MMAs each; the buffer of the
//      K split is reused and G overwrites H_j in TMEM),
//   6. thread a holds row a of G in registers; Lanczos on G needs one matvec
//      per step against the broadcast Lanczos vector (packed FFMA2).
// Measured (Wan2.1-14B shape, 40 heads): 5.35 ms, from 13.6 ms for the CUDA-core
// H_j + two-matvec Lanczos. The bound is now the latency of the 24 dependent
// Lanczos steps (two block reductions each) with only three blocks resident per
// SM (each block's G is 64 KB of registers); a register-blocked G (4 rows x 32
// columns per thread, 4x less vector traffic) measured the same.
constexpr int kTcThreads = 128;
struct TcCfg {
    static constexpr int kTile = 64 * 128 * 2;            // one 64-row bf16 tile (two 64-column SW128 halves)
    static constexpr int kOffV = 3 * kTile;               // hi | mid | lo | V
    static constexpr int kOffVec = 4 * kTile;             // Lanczos vector [128]
    static constexpr int kOffKb = kOffVec + 128 * 4;      // k_bar_j [128]
    static constexpr int kOffRed = kOffKb + 128 * 4;      // [2][4][2] reduction scratch, alpha / beta
    static constexpr int kOffBar = (kOffRed + (16 + 4 * kLanczos) * 4 + 7) & ~7;  // alpha / beta x 2 halves
    static constexpr int kSmem = 1024 + kOffBar + 48;
};

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(r)
        : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
          "l"(*reinterpret_cast<uint64_t*>(&c)));
    return *reinterpret_cast<float2*>(&r);
}

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

// TMEM row (lane) of the issuing warp's quadrant, 128 fp32 columns
__device__ __forceinline__ void tmem_row128(uint32_t taddr, float (&x)[128]) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        uint32_t r[32];
        tmem_ld32(taddr + cc * 32, r);
        tmem_ld_wait(r);
#pragma unroll
        for (int i = 0; i < 32; ++i) x[cc * 32 + i] = __uint_as_float(r[i]);
    }
}

// kPair (head dim 64): two key blocks per CTA in the same 128-wide shapes.
// Block j0 fills TMA half 0 (d columns 0-63 of the MN-major operands), block
// j1 = j0 + 1 half 1, so one M = N = 128 MMA yields H_j0 and H_j1 on its
// diagonal quadrants (the cross quadrants pair one block's keys with the
// other's values and are dropped). D is then block-diagonal, so G = D^T D is
// blockdiag(G_j0, G_j1), and threads 0-63 / 64-127 run two independent
// Lanczos processes on their quadrants.
template <bool kPair>
__global__ void __launch_bounds__(kTcThreads, 3)
    block_norms_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                          NormArgs a) {
    using Cfg = TcCfg;
    constexpr int D = 128;   // MMA / register width
    constexpr int DR = kPair ? 64 : 128;  // head dim
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    float* vs = reinterpret_cast<float*>(smem + Cfg::kOffVec);
    float* kb = reinterpret_cast<float*>(smem + Cfg::kOffKb);
    float* red = reinterpret_cast<float*>(smem + Cfg::kOffRed);
    float* ab = red + 16;
    // [0] tiles landed, [1] H_j MMAs done, [2] / [3] G passes done
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::kOffBar);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
    const int j = kPair ? 2 * blockIdx.x : blockIdx.x, bh = blockIdx.y;
    const int b = bh / a.H, h = bh % a.H;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int hq = tid >> 6;  // kPair: this thread's block (quadrant)
    const int n = min(64, a.L - j * 64);
    const int n1 = kPair ? min(64, a.L - (j + 1) * 64) : n;  // rows of block j + 1 (<= 0: absent)
#if PISA_K1C_CLOCKS  // diagnostic build: M_j is replaced by a phase's cycle count
    const long long t0 = clock64();
    long long t1 = 0, t4 = 0, t5 = 0, ta = 0, tb = 0;
#endif

    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
        // K_j / V_j first: their latency overlaps the TMEM allocation and the
        // CTA barrier below
        mbar_expect_tx(&bar[0], 2 * Cfg::kTile);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            // kPair: half = block j + half, all 64 columns; else: column half of block j
            const int c0 = kPair ? 0 : half * 64, r0 = (kPair ? j + half : j) * 64;
            tma_load_4d(smem + half * 8192, &tmK, &bar[0], c0, r0, h, b);
            tma_load_4d(smem + Cfg::kOffV + half * 8192, &tmV, &bar[0], c0, r0, h, b);
        }
    }
    if (warp == 0) {
        tmem_alloc(tslot, 128);
        tmem_relinquish();
    }
    if constexpr (kPair)
        kb[tid] = (j + hq < a.N) ? a.kbar[(size_t(bh) * a.N + j + hq) * DR + (tid & 63)] : 0.f;
    else
        kb[tid] = a.kbar[(size_t(bh) * a.N + j) * D + tid];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
#if PISA_K1C_CLOCKS
    ta = clock64();
#endif
    const uint32_t tmem = *tslot;
    const uint32_t trow = tmem + (uint32_t(warp * 32) << 16);  // this thread's TMEM lane = tid
    // -H_bar into this thread's TMEM row, the accumulator the H_j MMAs add to
    // (so they produce D = H_j - H_bar directly): the H_bar load latency
    // overlaps the K / V TMA and the split instead of following the MMAs
#if PISA_K1C_HBAR_STAGE
    // Coalesced: rows of H_bar read 256 B per 16 threads into the mid / lo tiles
    // (free until the split), 16-byte chunks XOR-swizzled by row, then each
    // thread reads its own row back. Loading row tid straight from global made
    // every warp load touch 32 lines (one 16-byte chunk each): ~4K L1 wavefronts
    // and ~5K cycles per CTA (PISA_K1C_CLOCKS=7), a tenth of its lifetime.
    {
        float4* stage = reinterpret_cast<float4*>(smem + Cfg::kTile);  // [rows][16 chunks of 4 floats]
        constexpr int kRows = kPair ? 64 : 128;  // kPair: one 64 x 64 H_bar for both blocks
        constexpr int kHalves = kPair ? 1 : 2;   // 64-column halves of H_bar
        const float4* hb = reinterpret_cast<const float4*>(a.hbar + size_t(bh) * DR * DR);
#pragma unroll
        for (int half = 0; half < kHalves; ++half) {
#pragma unroll
            for (int i = 0; i < kRows * 16 / kTcThreads; ++i) {
                const int ci = tid + kTcThreads * i, r = ci >> 4, c = ci & 15;
                stage[r * 16 + (c ^ (r & 15))] = __ldg(hb + r * (DR / 4) + half * 16 + c);
            }
            __syncthreads();
            const int row = kPair ? (tid & 63) : tid;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {  // 32 TMEM columns per store
                uint32_t r[32];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int c = cc * 8 + i;
                    const float4 h4 = stage[row * 16 + (c ^ (row & 15))];
                    r[4 * i] = __float_as_uint(-h4.x);
                    r[4 * i + 1] = __float_as_uint(-h4.y);
                    r[4 * i + 2] = __float_as_uint(-h4.z);
                    r[4 * i + 3] = __float_as_uint(-h4.w);
                }
                // kPair: block hq's row goes to its own 64-column quadrant
                tmem_st32(trow + ((kPair ? hq : half) * 2 + cc) * 32, r);
            }
            __syncthreads();  // every row is read before the next half (or the split) overwrites the stage
        }
        if constexpr (kPair) {  // the cross quadrant starts at 0
            uint32_t z[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) z[i] = 0u;
            tmem_st32(trow + ((1 - hq) * 2) * 32, z);
            tmem_st32(trow + ((1 - hq) * 2 + 1) * 32, z);
        }
        tmem_st_wait();
    }
#else
    {
        // kPair: row a of block hq gets -H_bar[a % 64] in its own quadrant, 0 in the other
        const float4* hb = reinterpret_cast<const float4*>(a.hbar + (size_t(bh) * DR + (kPair ? (tid & 63) : tid)) * DR);
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) {
            uint32_t r[32];
            const bool own = !kPair || (cc >> 1) == hq;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float4 h4 = own ? __ldg(hb + (kPair ? (cc & 1) : cc) * 8 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
                r[4 * i] = __float_as_uint(-h4.x);
                r[4 * i + 1] = __float_as_uint(-h4.y);
                r[4 * i + 2] = __float_as_uint(-h4.z);
                r[4 * i + 3] = __float_as_uint(-h4.w);
            }
            tmem_st32(trow + cc * 32, r);
        }
        tmem_st_wait();
    }
#endif
#if PISA_K1C_CLOCKS
    tb = clock64();
#endif
    mbar_wait(&bar[0], 0);
#if PISA_K1C_CLOCKS
    t1 = clock64();
#endif

    // ---- 2. centre and split, one 16-byte chunk (8 keys of one row) at a time
#pragma unroll 2
    for (int i = 0; i < 8; ++i) {
        const int ci = tid + kTcThreads * i;
        const int r = (ci >> 3) & 63;
        const int d0 = (ci >> 9) * 64 + (((ci & 7) ^ (r & 7)) << 3);  // undo the 128B swizzle
        uint4 w = *reinterpret_cast<const uint4*>(smem + ci * 16);
        const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&w);
        uint4 hw, mw, lw;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float2 kf = __bfloat1622float2(k2[t]);
            const int nr = (kPair && (ci >> 9)) ? n1 : n;  // rows of this half's block
            const float x0 = r < nr ? kf.x - kb[d0 + 2 * t] : 0.f;
            const float x1 = r < nr ? kf.y - kb[d0 + 2 * t + 1] : 0.f;
            split3(x0, x1, (&hw.x)[t], (&mw.x)[t], (&lw.x)[t]);
        }
        *reinterpret_cast<uint4*>(smem + ci * 16) = hw;
        *reinterpret_cast<uint4*>(smem + Cfg::kTile + ci * 16) = mw;
        *reinterpret_cast<uint4*>(smem + 2 * Cfg::kTile + ci * 16) = lw;
    }
    fence_proxy_async();  // generic-proxy tile writes -> tcgen05 operand reads
    tc_fence_before();    // the -H_bar TMEM stores precede the MMAs
    __syncthreads();

    constexpr uint32_t idesc = idesc_bf16(128, 128, 1, 1);
    const uint32_t base = smem_u32(smem);
    auto desc = [&](int tile, int ks) { return sdesc_sw128(base + tile * Cfg::kTile + ks * 2048, 8192, 1024); };
    // ---- 3. H_j = kc^T V: small parts first
    if (warp == 0) {
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
            for (int part = 2; part >= 0; --part)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) mma_ss(tmem, desc(part, ks), desc(3, ks), idesc, 1u);
            mma_commit(&bar[1]);
        }
        __syncwarp();
    }
    mbar_wait(&bar[1], 0);
    tc_fence_after();

    // ---- 4. row a = tid of D = H_j - H_bar (the accumulator started at -H_bar)
    float x[D];
    tmem_row128(trow, x);
    if constexpr (kPair) {  // drop the cross quadrant: D = blockdiag(D_j0, D_j1)
#pragma unroll
        for (int c = 0; c < D; ++c)
            if ((c >> 6) != hq) x[c] = 0.f;
    }
    // ---- 5. G = D^T D, rows of D 64 at a time through the split tiles
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
        if ((tid >> 6) == pass) {
            const int r = tid & 63;
#pragma unroll
            for (int c8 = 0; c8 < D / 8; ++c8) {  // 16-byte chunk of row r, swizzled
                const uint32_t off = uint32_t((c8 >> 3) * 8192 + r * 128 + (((c8 & 7) ^ (r & 7)) << 4));
                uint4 hw, mw, lw;
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    split3(x[c8 * 8 + 2 * t], x[c8 * 8 + 2 * t + 1], (&hw.x)[t], (&mw.x)[t], (&lw.x)[t]);
                *reinterpret_cast<uint4*>(smem + off) = hw;
                *reinterpret_cast<uint4*>(smem + Cfg::kTile + off) = mw;
                *reinterpret_cast<uint4*>(smem + 2 * Cfg::kTile + off) = lw;
            }
        }
        fence_proxy_async();
        tc_fence_before();  // pass 0: every H_j row is read out of TMEM before G overwrites it
        __syncthreads();
        if (warp == 0) {
            tc_fence_after();
            if (elect_one()) {
                // (lo,hi) (hi,lo) (mid,mid) (mid,hi) (hi,mid) (hi,hi); tiles 0 = hi, 1 = mid, 2 = lo
                constexpr int kA[6] = {2, 0, 1, 1, 0, 0}, kB[6] = {0, 2, 1, 0, 1, 0};
#pragma unroll
                for (int p = 0; p < 6; ++p)
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        mma_ss(tmem, desc(kA[p], ks), desc(kB[p], ks), idesc, pass != 0 || p != 0 || ks != 0);
                mma_commit(&bar[2 + pass]);
            }
            __syncwarp();
        }
        mbar_wait(&bar[2 + pass], 0);  // the tiles are rewritten by the next pass
        tc_fence_after();
    }
    // ---- 6. row a of G into registers; Lanczos on G with delayed
    // normalisation: the matvec runs on the unnormalised w_m = beta_{m-1} v_m,
    // and ONE reduction of (|w_m|^2, w_m . G w_m) gives beta_{m-1} and alpha_m
    // exactly (no cancellation formula) -- one reduction and two barriers per
    // step instead of two and three; the steps are latency-bound
    tmem_row128(trow, x);
#if PISA_K1C_CLOCKS
    t4 = clock64();
#endif
    float wown = rsqrtf(float(DR)), vprev = 0.f, alpha_prev = 0.f;  // w_0 = v_0, |v_0| = 1
    vs[tid] = wown;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 128);

    int par = 0;
    auto block_sum2 = [&](float p, float q) -> float2 {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            p += __shfl_xor_sync(0xffffffffu, p, o);
            q += __shfl_xor_sync(0xffffffffu, q, o);
        }
#if PISA_K1C_DIAG_WARPSUM  // diagnostic only (wrong numerics): warp-local sums, no CTA barrier
        par ^= 1;
        return make_float2(4.f * p, 4.f * q);
#endif
        if (lane == 0) {
            red[par * 8 + warp * 2] = p;
            red[par * 8 + warp * 2 + 1] = q;
        }
        __syncthreads();
        const float* r = red + par * 8;
        par ^= 1;
        if constexpr (kPair)  // the two warps of this thread's block
            return make_float2(r[4 * hq] + r[4 * hq + 2], r[4 * hq + 1] + r[4 * hq + 3]);
        return make_float2((r[0] + r[2]) + (r[4] + r[6]), (r[1] + r[3]) + (r[5] + r[7]));
    };
    float* abq = ab + (kPair ? hq * 2 * kLanczos : 0);  // this block's alpha / beta
    const bool lead = (tid & (kPair ? 63 : 127)) == 0;
    bool done = false;  // kPair: a block's Lanczos may stop earlier than the other's
    int mq = kLanczos;
    for (int m = 0; m < kLanczos; ++m) {
        if (m > 0) {
            vs[tid] = wown;  // every read of vs in step m-1 preceded its reduction barrier
            __syncthreads();
        }
        // y_a = G[a] . w (w broadcast from shared memory; kPair: own quadrant)
        float2 y0 = make_float2(0.f, 0.f), y1 = y0, y2 = y0, y3 = y0;
        auto matvec = [&](auto c_begin) {
            constexpr int cb = decltype(c_begin)::value;
#if PISA_K1C_DIAG_NOLDS  // diagnostic only (wrong numerics): one vector load per step, not 32
            const float4 v4c = *reinterpret_cast<const float4*>(vs + cb);
            const float4 w4c = *reinterpret_cast<const float4*>(vs + cb + 4);
#endif
#pragma unroll
            for (int c = cb; c < cb + (kPair ? 64 : D); c += 8) {
#if PISA_K1C_DIAG_NOLDS
                const float4 v4 = v4c, w4 = w4c;
#else
                const float4 v4 = *reinterpret_cast<const float4*>(vs + c);
                const float4 w4 = *reinterpret_cast<const float4*>(vs + c + 4);
#endif
                y0 = ffma2(make_float2(x[c], x[c + 1]), make_float2(v4.x, v4.y), y0);
                y1 = ffma2(make_float2(x[c + 2], x[c + 3]), make_float2(v4.z, v4.w), y1);
                y2 = ffma2(make_float2(x[c + 4], x[c + 5]), make_float2(w4.x, w4.y), y2);
                y3 = ffma2(make_float2(x[c + 6], x[c + 7]), make_float2(w4.z, w4.w), y3);
            }
        };
        if (!kPair || hq == 0)
            matvec(std::integral_constant<int, 0>{});
        else
            matvec(std::integral_constant<int, 64>{});
        const float y = ((y0.x + y0.y) + (y1.x + y1.y)) + ((y2.x + y2.y) + (y3.x + y3.y));
        const float2 r = block_sum2(wown * wown, wown * y);
        if (done) continue;  // (kPair) keep joining the barriers
        const float b = m == 0 ? 1.f : sqrtf(r.x);  // beta_{m-1} = |w_m|
        if (m > 0) {
            if (lead) abq[kLanczos + m - 1] = b;
            if (!(b > 1e-30f * fmaxf(1.f, fabsf(alpha_prev)))) {  // invariant subspace (or D == 0)
                done = true;
                mq = m;
                if constexpr (!kPair) break;
                continue;
            }
        }
        const float inv = 1.f / b;
        const float vm = wown * inv;             // v_m
        const float alpha = r.y * inv * inv;     // v_m . G v_m
        if (lead) abq[m] = alpha;
        wown = y * inv - alpha * vm - b * vprev;  // w_{m+1} = G v_m - alpha_m v_m - beta_{m-1} v_{m-1}
        vprev = vm;
        alpha_prev = alpha;
    }
    __syncthreads();
#if PISA_K1C_CLOCKS
    t5 = clock64();
#endif
    {  // this block's tridiagonal (kPair: each half its own block) -> ritz_kernel
        const int t = kPair ? (tid & 63) : tid;
        const int jb = j + (kPair ? hq : 0);
        if (t < 2 * kLanczos && jb < a.N)
            a.tri[(size_t(bh) * a.N + jb) * kTriStride + t] = t == 2 * kLanczos - 1 ? __int_as_float(mq) : abq[t];
    }
#if PISA_K1C_CLOCKS  // (the ritz kernel overwrites M_j: read the clocks with it disabled)
    if (tid == 0) {
        const long long t6 = clock64();
        const long long c[7] = {t5 - t4, t6 - t5, t4 - t0, t6 - t0, t1 - t0, ta - t0, tb - t0};
        a.m[size_t(bh) * a.N + j] = float(c[PISA_K1C_CLOCKS - 1]);
    }
#endif
}

}  // namespace

int block_norms_launches(int D) { return (D == 128 || kK1cPairD64) ? 2 : 1; }

size_t block_norms_smem_bytes(int D) {
    if (D == 128) return TcCfg::kSmem;
    // phase 1 (centred K and V, 2 x 64 x D floats) and phases 2-3 (D, Lanczos
    // basis, scratch) share the buffer
    const size_t p1 = size_t(2) * 64 * D * 4;
    const size_t p3 = (size_t(D) * (D + 1) + 3 * size_t(D) + 16 + 2 * kLanczos) * 4 + 64;
    return p1 > p3 ? p1 : p3;
}

cudaError_t launch_block_norms(int D, const CUtensorMap& tmK, const CUtensorMap& tmV, const __nv_bfloat16* k,
                               const __nv_bfloat16* v, const NormArgs& a, int BH, cudaStream_t s) {
    const size_t smem = block_norms_smem_bytes(D);
    dim3 grid(a.N, BH);
    const int nblk = a.N * BH;
    if (D == 128 || kK1cPairD64) {
        if (D == 128) {
            cudaFuncSetAttribute(block_norms_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            block_norms_tc_kernel<false><<<grid, kTcThreads, smem, s>>>(tmK, tmV, a);
        } else {  // two key blocks per CTA on the tensor cores
            const size_t smem2 = TcCfg::kSmem;
            cudaFuncSetAttribute(block_norms_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2));
            block_norms_tc_kernel<true><<<dim3((a.N + 1) / 2, BH), kTcThreads, smem2, s>>>(tmK, tmV, a);
        }
#if !PISA_K1C_CLOCKS
        ritz_kernel<<<(nblk + kRitzWarps - 1) / kRitzWarps, 32 * kRitzWarps, 0, s>>>(a, nblk);
#endif
    } else {
        auto kern = block_norms_kernel<64>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        kern<<<grid, kNormThreads, smem, s>>>(k, v, a);
    }
    return cudaGetLastError();
}

}  // namespace pisa_b200
