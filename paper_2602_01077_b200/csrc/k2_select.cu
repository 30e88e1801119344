// K2: block scoring + top-k routing (the "select" step, engine.hpp:443-457).
//
// Replaces select_topk_plain (router.hpp:126-151) with topk_ascending (:96-108)
// and force_block (:111-121), in two launches:
//   K2a score_kernel : s_ij = scale * <q_bar_i, k_bar_j>, a register-tiled fp32
//                      FMA GEMM per (batch, head), fixed summation order over d
//                      (fp32 scoring keeps the index sets bit-exact
//                      against the fp64 reference on the Wan shapes; bf16 / TF32
//                      scoring does not), stored as order-preserving uint32 keys
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

// K2a: score tile. keys[bh][i][j] = order_key(scale * <q_bar_i, k_bar_j>) for a
// 64 x 64 tile of (query block, key block) pairs; 256 threads, 4 x 4 outputs
// each. Every output accumulates a = 0 .. D-1 in order with fp32 FMA (the
// same order as the reference's dot_d loop), so results are reproducible.
constexpr int kTile = 64, kAK = 32;

// rect (covariance router, router.hpp:176-183): per key block log(M_j + eps),
// added after the scaled dot product; null for the plain router.
template <int D>
__global__ void __launch_bounds__(256) score_kernel(const float* __restrict__ qbar,
                                                    const float* __restrict__ kbar,
                                                    const float* __restrict__ rect,
                                                    uint32_t* __restrict__ keys, int N,
                                                    float scale) {
    __shared__ float As[kAK][kTile + 4];
    __shared__ float Bs[kAK][kTile + 4];
    const int bh = blockIdx.z;
    const int i0 = blockIdx.y * kTile, j0 = blockIdx.x * kTile;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const float* qb = qbar + size_t(bh) * N * D;
    const float* kb = kbar + size_t(bh) * N * D;
    float acc[4][4] = {};
    for (int a0 = 0; a0 < D; a0 += kAK) {
        __syncthreads();
        for (int e = threadIdx.x; e < kTile * kAK; e += 256) {
            const int r = e / kAK, c = e % kAK;
            As[c][r] = (i0 + r < N) ? qb[size_t(i0 + r) * D + a0 + c] : 0.f;
            Bs[c][r] = (j0 + r < N) ? kb[size_t(j0 + r) * D + a0 + c] : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int c = 0; c < kAK; ++c) {
            const float4 av = *reinterpret_cast<const float4*>(&As[c][ty * 4]);
            const float4 bv = *reinterpret_cast<const float4*>(&Bs[c][tx * 4]);
            const float ar[4] = {av.x, av.y, av.z, av.w};
            const float br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int w = 0; w < 4; ++w) acc[u][w] = fmaf(ar[u], br[w], acc[u][w]);
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int i = i0 + ty * 4 + u;
        if (i >= N) continue;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int j = j0 + tx * 4 + w;
            if (j < N) {
                float sc = scale * acc[u][w];
                if (rect) sc += rect[size_t(bh) * N + j];
                keys[(size_t(bh) * N + i) * N + j] = order_key(sc);
            }
        }
    }
}

// K2b: per query block, radix-select the k-th largest key (8-bit digits from the
// top), then a ballot compaction in ascending index order takes every key above
// it plus the lowest-index ties: topk_ascending semantics (router.hpp:96-108).
constexpr int kRowsPerCta = 4;

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

    uint32_t prefix = 0, pmask = 0;
    int rem = a.k;  // rank (1-based) of the wanted element among prefix matches
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
        int digit = -1, above = 0;
        if (rem > excl && rem <= incl) {
            int run = excl;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                if (digit < 0 && rem <= run + cnt[t]) {
                    digit = 255 - lane * 8 - t;
                    above = run;
                }
                run += cnt[t];
            }
        }
        const uint32_t owner = __ballot_sync(0xffffffffu, digit >= 0);
        const int src_lane = __ffs(owner) - 1;
        digit = __shfl_sync(0xffffffffu, digit, src_lane);
        above = __shfl_sync(0xffffffffu, above, src_lane);
        rem -= above;
        prefix |= uint32_t(digit) << shift;
        pmask |= 255u << shift;
        __syncwarp();
    }
    const uint32_t T = prefix;  // key of the k-th largest; take `rem` ties, lowest indices first

    const uint32_t lt_mask = (1u << lane) - 1u;
    int swap_out = -1;  // force_diagonal: the kept tie to drop (worst kept, highest index)
    bool swap_in = false;
    if (a.force_diagonal && i < N) {
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
    int32_t* sel = a.selected ? a.selected + (size_t(bh) * N + i) * a.k : nullptr;
    uint32_t* mrow = a.mask + (size_t(bh) * N + i) * a.W;
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

}  // namespace

cudaError_t launch_select(int D, const SelectArgs& a, int BH, uint32_t* keys, cudaStream_t s) {
    const int nt = (a.N + kTile - 1) / kTile;
    dim3 g1(nt, nt, BH);
    if (D == 128)
        score_kernel<128><<<g1, 256, 0, s>>>(a.qbar, a.kbar, a.rect, keys, a.N, a.scale);
    else
        score_kernel<64><<<g1, 256, 0, s>>>(a.qbar, a.kbar, a.rect, keys, a.N, a.scale);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(uint32_t) * size_t(kRowsPerCta) * (a.N + 256);
    cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    topk_kernel<<<dim3((a.N + kRowsPerCta - 1) / kRowsPerCta, BH), kRowsPerCta * 32, smem, s>>>(keys, a);
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
