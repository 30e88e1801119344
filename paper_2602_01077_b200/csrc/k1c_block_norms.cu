// K1c: spectral deviation norms M_j = ||H_j - H_bar||_2 per key block, the
// covariance-aware router's rectifier (compute_global_stats with compute_norms,
// block_stats.hpp:207-241; select_topk_covariance, router.hpp:157-193).
//
// One CTA (256 threads) per (key block j, batch*head):
//   1. centred keys kc = K_j - k_bar_j and V_j into shared memory (fp32; the
//      ragged last block has n < 64 rows, the rest are zero),
//   2. H_j = kc^T V_j (each thread an 8 x 8 tile, fp32, fixed order over rows),
//      D = H_j - H_bar (H_bar from K1b),
//   3. sigma_max(D)^2 = lambda_max(D^T D) by kLanczos steps of Lanczos on D^T D
//      from the normalised all-ones start (the reference's power-iteration
//      start, block_stats.hpp:98);
//      the extreme Ritz value of the kLanczos-step tridiagonal is found by a
//      warp-parallel multisection on its Sturm sequence.
// The reference uses the exact Jacobi eigen-solve in fp64 (block_stats.hpp:42-94);
// the extreme eigenvalue of D^T D is well separated after a few dozen Lanczos
// steps, so M_j agrees to fp32 rounding (~1e-6 relative, measured in the tests).
// Outputs m[bh][j] (fp32) and rect[bh][j] = log(M_j + eps) (computed in fp64).
#include "kernels.h"
#include "sm100.cuh"

namespace pisa_b200 {
namespace {

constexpr int kNormThreads = 256;
constexpr int kLanczos = 24;  // fp32-converged (<5e-8 rel.) on gaussian / clustered blocks

template <int D>
__global__ void __launch_bounds__(kNormThreads) block_norms_kernel(const __nv_bfloat16* __restrict__ k,
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
    // ---- 2. H_j = kc^T V (thread tile: rows ta*8.., cols tb*8..), minus H_bar
    constexpr int T = D / 8;  // tiles per side (16 for D = 128, 8 for D = 64)
    float acc[8][8];
    const bool owns = tid < T * T;
    const int ta = tid / T, tb = tid % T;
    if (owns) {
#pragma unroll
        for (int x = 0; x < 8; ++x)
#pragma unroll
            for (int y = 0; y < 8; ++y) acc[x][y] = 0.f;
        for (int r = 0; r < n; ++r) {
            float ka[8], vb[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) ka[x] = kc[r * D + ta * 8 + x];
#pragma unroll
            for (int y = 0; y < 8; ++y) vb[y] = vv[r * D + tb * 8 + y];
#pragma unroll
            for (int x = 0; x < 8; ++x)
#pragma unroll
                for (int y = 0; y < 8; ++y) acc[x][y] = fmaf(ka[x], vb[y], acc[x][y]);
        }
        const float* hb = a.hbar + size_t(bh) * D * D;
#pragma unroll
        for (int x = 0; x < 8; ++x)
#pragma unroll
            for (int y = 0; y < 8; ++y) acc[x][y] -= hb[(ta * 8 + x) * D + tb * 8 + y];
    }
    __syncthreads();  // kc / vv are dead: D overwrites them
    if (owns) {
#pragma unroll
        for (int x = 0; x < 8; ++x)
#pragma unroll
            for (int y = 0; y < 8; ++y) Dm[(ta * 8 + x) * (D + 1) + tb * 8 + y] = acc[x][y];
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
    if (warp == 0) {
        // largest eigenvalue of the m x m tridiagonal (alpha, beta): 32-way
        // multisection on the Sturm count (number of eigenvalues below x from
        // the LDL^T pivots), each round shrinks the bracket 33x (fp32 is the
        // precision M_j is delivered in)
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
            a.m[size_t(bh) * a.N + j] = float(sigma);
            if (a.rect) a.rect[size_t(bh) * a.N + j] = float(log(sigma + a.eps));
        }
    }
}

}  // namespace

size_t block_norms_smem_bytes(int D) {
    // phase 1 (centred K and V, 2 x 64 x D floats) and phases 2-3 (D, Lanczos
    // basis, scratch) share the buffer
    const size_t p1 = size_t(2) * 64 * D * 4;
    const size_t p3 = (size_t(D) * (D + 1) + 3 * size_t(D) + 16 + 2 * kLanczos) * 4 + 64;
    return p1 > p3 ? p1 : p3;
}

cudaError_t launch_block_norms(int D, const __nv_bfloat16* k, const __nv_bfloat16* v, const NormArgs& a,
                               int BH, cudaStream_t s) {
    const size_t smem = block_norms_smem_bytes(D);
    dim3 grid(a.N, BH);
    if (D == 128) {
        auto kern = block_norms_kernel<128>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        kern<<<grid, kNormThreads, smem, s>>>(k, v, a);
    } else {
        auto kern = block_norms_kernel<64>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        kern<<<grid, kNormThreads, smem, s>>>(k, v, a);
    }
    return cudaGetLastError();
}

}  // namespace pisa_b200
