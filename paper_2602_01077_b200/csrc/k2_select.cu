// K2: block scoring + top-k routing (the "select" step, engine.hpp:443-457).
//
// Replaces sparsity_to_k's consumer select_topk_plain (router.hpp:126-151) with
// topk_ascending (:96-108) and force_block (:111-121). One CTA scores kQB query
// blocks of one (batch, head) against every key centroid:
//   s_ij = scale * <q_bar_i, k_bar_j>     fp32 FMA, fixed summation order over d
// (fp32 scoring keeps the index sets bit-exact against the fp64
// reference on the Wan shapes; bf16 / TF32 scoring does not). Each row's k-th
// largest score is found by an 8-bit-digit radix select on the order-preserving
// uint32 image of the float, ties resolve to the LOWER index, and a ballot
// compaction emits the ascending index list plus a bitmask row in one pass.
#include "kernels.h"
#include "sm100.cuh"

namespace pisa_b200 {
using namespace pisa_sm100;

namespace {

constexpr int kQB = 4;        // query blocks per CTA
constexpr int kKeyTile = 64;  // centroids staged per step
constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t order_key(float f) {
    if (f == 0.0f) f = 0.0f;  // -0 == +0 as in the fp64 comparison
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <int D>
__global__ void __launch_bounds__(kThreads) select_kernel(SelectArgs a) {
    extern __shared__ float sm[];
    float* q_s = sm;                              // [kQB][D]
    float* kt_s = q_s + kQB * D;                  // [kKeyTile][D + 1]
    uint32_t* keys = reinterpret_cast<uint32_t*>(kt_s + kKeyTile * (D + 1));  // [kQB][N]
    uint32_t* hist = keys + kQB * a.N;            // [kQB][256]

    const int bh = blockIdx.y;
    const int i0 = blockIdx.x * kQB;
    const int tid = threadIdx.x;
    const float* qb = a.qbar + size_t(bh) * a.N * D;
    const float* kb = a.kbar + size_t(bh) * a.N * D;

    for (int e = tid; e < kQB * D; e += kThreads) {
        const int r = e / D, i = i0 + r;
        q_s[e] = i < a.N ? qb[size_t(i) * D + (e % D)] : 0.f;
    }
    // ---- scores
    const int r = tid / kKeyTile;   // query row of this thread (warp-uniform)
    const int jj = tid % kKeyTile;  // centroid within the tile
    for (int j0 = 0; j0 < a.N; j0 += kKeyTile) {
        __syncthreads();
        for (int e = tid; e < kKeyTile * D; e += kThreads) {
            const int row = e / D, col = e % D;
            kt_s[row * (D + 1) + col] = (j0 + row < a.N) ? kb[size_t(j0 + row) * D + col] : 0.f;
        }
        __syncthreads();
        const float* qr = q_s + r * D;
        const float* kr = kt_s + jj * (D + 1);
        float acc = 0.f;
#pragma unroll 16
        for (int c = 0; c < D; ++c) acc = fmaf(qr[c], kr[c], acc);
        if (j0 + jj < a.N) keys[r * a.N + j0 + jj] = order_key(a.scale * acc);
    }
    __syncthreads();

    // ---- per-row radix select + ballot compaction: warp w < kQB owns row w
    const int warp = tid >> 5, lane = tid & 31;
    if (warp >= kQB) return;
    const int i = i0 + warp;
    if (i >= a.N) return;
    const uint32_t* kr = keys + warp * a.N;
    uint32_t* hw = hist + warp * 256;
    const int N = a.N;

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
        const int src = __ffs(owner) - 1;
        digit = __shfl_sync(0xffffffffu, digit, src);
        above = __shfl_sync(0xffffffffu, above, src);
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
        diag_sel = __shfl_sync(0xffffffffu, diag_sel, i & 31) ;
        // diag_sel was set by the lane whose j == i in the chunk holding i
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

cudaError_t launch_select(int D, const SelectArgs& a, int BH, cudaStream_t s) {
    const size_t smem = sizeof(float) * (kQB * D + kKeyTile * (D + 1)) +
                        sizeof(uint32_t) * (size_t(kQB) * a.N + kQB * 256);
    dim3 grid((a.N + kQB - 1) / kQB, BH);
    if (D == 128) {
        cudaFuncSetAttribute(select_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        select_kernel<128><<<grid, kThreads, smem, s>>>(a);
    } else {
        cudaFuncSetAttribute(select_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        select_kernel<64><<<grid, kThreads, smem, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_plan_to_mask(const int32_t* selected, int N, int k, int W, uint32_t* mask,
                                int* bad, int BH, cudaStream_t s) {
    plan_to_mask_kernel<<<dim3(N, BH), 128, 0, s>>>(selected, N, k, W, mask, bad);
    return cudaGetLastError();
}

}  // namespace pisa_b200
