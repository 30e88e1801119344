// K2c / K2d: query-block pairing for the fused kernel (no reference
// counterpart: it only regroups work; every query block computes the same math,
// equal to rounding -- the grouping of its key blocks into super-tiles moves
// the online softmax's lazy-rescale points).
//
// K3 runs two query blocks per CTA over the UNION of their selections, so its
// executed work is proportional to sum over pairs |S_a U S_b|. Pairing
// consecutive blocks (2t, 2t+1) is what a spatially coherent DiT sequence wants,
// but not in general: on independent (gaussian) routing the union of two
// neighbours is 1.87 k, and on multi-cluster data blocks that route alike can
// be far apart. Here:
//   K2c pair_candidates_kernel: warp per query block i, overlap
//       o(i, j) = popcount(mask_i & mask_j) for j within +-kWindow of i, keeps
//       the best kCand partners (overlap desc, index asc; 16: measured on
//       clustered routing union/k 1.113 -> 1.059 vs 8, -1.8 % step time;
//       gaussian +0.2 %; a +-96 window was worse on both);
//   K2d pair_match_kernel: one CTA per (batch, head), locally-dominant matching
//       on the candidate graph (the parallel form of greedy max-weight
//       matching, a 1/2-approximation): every unmatched block proposes its best
//       unmatched candidate, mutual proposals match, repeat; the blocks left
//       over are paired in index order. Deterministic (ties -> lower index).
// Output pairs[bh][t] = (a, b), a < b, b = -1 for a lone last block; the fused
// kernel's tile t processes query blocks a and b. Only query blocks in
// [qb0, qb1) take part (a rank's share of a head under (head x query-block
// range) sharding); t counts from 0.
#include "kernels.h"

namespace pisa_b200 {
namespace {

constexpr int kCand = kPairCand;
// Candidate partners of block i are the blocks within +-kWindow of it: full
// O(N^2 W) search costs ~2.5 ms at Wan2.1-14B for a further ~2 % fewer union
// tiles (simulated: gaussian union/k 1.871 -> 1.77 windowed vs 1.735 full;
// multi-cluster 1.856 -> 1.06 vs 1.02).
#ifndef PISA_PAIR_WINDOW
#define PISA_PAIR_WINDOW 48
#endif
constexpr int kWindow = PISA_PAIR_WINDOW;

// candidate (overlap, index) ordering: higher overlap first, then lower index
__device__ __forceinline__ bool better(int ov, int j, int ov2, int j2) {
    return ov > ov2 || (ov == ov2 && j < j2);
}

__global__ void __launch_bounds__(256) pair_candidates_kernel(const uint32_t* __restrict__ mask, int N,
                                                             int W, int qb0, int qb1, int* __restrict__ cand) {
    // The CTA's 8 query blocks share one window: its rows [wb, we) are staged
    // in shared memory with coalesced loads (a W-word row stride with W odd is
    // conflict-free across lanes reading 32 consecutive rows; even W costs a
    // 2-way conflict at most for the W <= 128 this path sees).
    extern __shared__ uint32_t mrow[];  // [we - wb][W]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bh = blockIdx.y;
    const int ib = qb0 + blockIdx.x * 8;
    const int i = ib + warp;
    const int wb = max(qb0, ib - kWindow), we = min(qb1, ib + 8 + kWindow);
    const uint32_t* M = mask + size_t(bh) * N * W;
    for (int e = threadIdx.x; e < (we - wb) * W; e += blockDim.x) mrow[e] = __ldg(M + size_t(wb) * W + e);
    __syncthreads();
    if (i >= qb1) return;
    const uint32_t* mi = mrow + (i - wb) * W;
    // each lane scores its <= kPerLane candidates j = j0 + lane + 32 t (kept in
    // registers, statically indexed), then the warp pops the kCand best in
    // order (a per-lane sorted list of kCand with dynamic indexing lived in
    // local memory: 0.19 ms of latency stalls at Wan2.1-14B)
    constexpr int kPerLane = (2 * kWindow + 1 + 31) / 32;  // the window is i +- kWindow inclusive
    const int j0 = max(qb0, i - kWindow), j1 = min(qb1, i + kWindow + 1);
    int co[kPerLane], cj[kPerLane];
#pragma unroll
    for (int t = 0; t < kPerLane; ++t) {
        const int j = j0 + lane + 32 * t;
        co[t] = -1;
        cj[t] = 0x7fffffff;
        if (j < j1 && j != i) {
            const uint32_t* mj = mrow + (j - wb) * W;
            int ov = 0;
            for (int w = 0; w < W; ++w) ov += __popc(mi[w] & mj[w]);
            co[t] = ov;
            cj[t] = j;
        }
    }
    for (int c = 0; c < kCand; ++c) {
        // this lane's best remaining candidate
        int myo = co[0], myj = cj[0];
#pragma unroll
        for (int t = 1; t < kPerLane; ++t)
            if (better(co[t], cj[t], myo, myj)) {
                myo = co[t];
                myj = cj[t];
            }
        int o = myo, jj = myj;
#pragma unroll
        for (int sft = 16; sft > 0; sft >>= 1) {
            const int o2 = __shfl_xor_sync(0xffffffffu, o, sft), j2 = __shfl_xor_sync(0xffffffffu, jj, sft);
            if (better(o2, j2, o, jj)) {
                o = o2;
                jj = j2;
            }
        }
        // the winner retires it (candidate indices are unique across lanes)
#pragma unroll
        for (int t = 0; t < kPerLane; ++t)
            if (cj[t] == jj && o >= 0) {
                co[t] = -1;
                cj[t] = 0x7fffffff;
            }
        if (lane == 0) cand[(size_t(bh) * N + i) * kCand + c] = (o >= 0 && jj < N) ? jj : -1;
    }
}

// kSmemC: the candidate lists staged in shared memory as 16-bit indices (one
// coalesced pass over global memory instead of a dependent L2 load per
// candidate and round), and each block's scan resumes where the previous
// round's stopped (a matched block stays matched, so candidates passed over
// never become available again): the same proposals, round by round, as the
// plain form.
constexpr int kMatchThreads = 1024;
constexpr int kMatchPer = 4;  // blocks per thread in the staged form (N <= 4096)

template <bool kSmemC>
__global__ void __launch_bounds__(kMatchThreads) pair_match_kernel(const int* __restrict__ cand, int N, int qb0,
                                                                   int qb1, int2* __restrict__ pairs) {
    extern __shared__ int partner[];  // [N], then prop [N], then (kSmemC) cs [N][kCand] int16
    int* prop = partner + N;
    int16_t* cs = reinterpret_cast<int16_t*>(prop + N);
    __shared__ int progress;
    const int bh = blockIdx.x;
    const int* C = cand + size_t(bh) * N * kCand;
    for (int i = qb0 + threadIdx.x; i < qb1; i += blockDim.x) partner[i] = -1;
    if constexpr (kSmemC) {
        for (int e = qb0 * kCand + threadIdx.x; e < qb1 * kCand; e += blockDim.x) cs[e] = int16_t(__ldg(C + e));
    }
    __syncthreads();
    int cur[kMatchPer];  // kSmemC: first candidate of block i still worth looking at
#pragma unroll
    for (int u = 0; u < kMatchPer; ++u) cur[u] = 0;
    for (int round = 0; round < 64; ++round) {
        // every unmatched block proposes its best unmatched candidate
        if constexpr (kSmemC) {
#pragma unroll
            for (int u = 0; u < kMatchPer; ++u) {
                const int i = qb0 + threadIdx.x + u * kMatchThreads;
                if (i >= qb1) break;
                int p = -1;
                if (partner[i] < 0) {
                    int c = cur[u];
                    for (; c < kCand; ++c) {
                        const int j = cs[i * kCand + c];
                        if (j >= 0 && partner[j] < 0) {
                            p = j;
                            break;
                        }
                    }
                    cur[u] = c;
                }
                prop[i] = p;
            }
        } else {
            for (int i = qb0 + threadIdx.x; i < qb1; i += blockDim.x) {
                int p = -1;
                if (partner[i] < 0) {
                    for (int c = 0; c < kCand; ++c) {
                        const int j = C[size_t(i) * kCand + c];
                        if (j >= 0 && partner[j] < 0) {
                            p = j;
                            break;
                        }
                    }
                }
                prop[i] = p;
            }
        }
        if (threadIdx.x == 0) progress = 0;
        __syncthreads();
        for (int i = qb0 + threadIdx.x; i < qb1; i += blockDim.x) {
            const int j = prop[i];
            if (j >= 0 && prop[j] == i) {  // mutual: both sides record it
                partner[i] = j;
                progress = 1;
            }
        }
        __syncthreads();
        if (!progress) break;
        __syncthreads();
    }
    // emit pairs in order of the lower index; leftovers paired in index order
    if constexpr (kSmemC) {
        // in parallel: tile t of a matched block i < partner is ML(< i) +
        // floor(U(< i) / 2) (ML: matched leads, U: unmatched blocks before i);
        // the u-th unmatched block (u odd) closes the tile (unm[u - 1], i)
        __shared__ int wsum[2][kMatchThreads / 32];
        const int n = qb1 - qb0;
        const int seg = (n + kMatchThreads - 1) / kMatchThreads;  // <= kMatchPer
        const int b0 = qb0 + threadIdx.x * seg, b1 = min(qb1, b0 + seg);
        int ml = 0, un = 0;
        for (int i = b0; i < b1; ++i) {
            const int j = partner[i];
            ml += j > i;
            un += j < 0;
        }
        const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
        int sml = ml, sun = un;  // inclusive warp scans
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int a = __shfl_up_sync(0xffffffffu, sml, o), b = __shfl_up_sync(0xffffffffu, sun, o);
            if (lane >= o) {
                sml += a;
                sun += b;
            }
        }
        if (lane == 31) {
            wsum[0][wp] = sml;
            wsum[1][wp] = sun;
        }
        __syncthreads();
        if (wp == 0) {
            int a = wsum[0][lane], b = wsum[1][lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int x = __shfl_up_sync(0xffffffffu, a, o), y = __shfl_up_sync(0xffffffffu, b, o);
                if (lane >= o) {
                    a += x;
                    b += y;
                }
            }
            wsum[0][lane] = a;  // inclusive over warps
            wsum[1][lane] = b;
        }
        __syncthreads();
        int ML = sml - ml + (wp > 0 ? wsum[0][wp - 1] : 0);  // exclusive prefixes of this segment
        int U = sun - un + (wp > 0 ? wsum[1][wp - 1] : 0);
        const int Utot = wsum[1][kMatchThreads / 32 - 1], MLtot = wsum[0][kMatchThreads / 32 - 1];
        int* unm = prop;  // unmatched blocks in index order
        {
            int u = U;
            for (int i = b0; i < b1; ++i)
                if (partner[i] < 0) unm[u++] = i;
        }
        __syncthreads();
        int2* P = pairs + size_t(bh) * ((N + 1) / 2);
        for (int i = b0; i < b1; ++i) {
            const int j = partner[i];
            if (j > i) {
                P[ML + U / 2] = make_int2(i, j);
                ++ML;
            } else if (j < 0) {
                if (U & 1) P[ML + U / 2] = make_int2(unm[U - 1], i);
                ++U;
            }
        }
        if (threadIdx.x == 0 && (Utot & 1)) P[MLtot + Utot / 2] = make_int2(unm[Utot - 1], -1);
    } else if (threadIdx.x == 0) {
        int t = 0, pending = -1;
        for (int i = qb0; i < qb1; ++i) {
            const int j = partner[i];
            if (j > i) {
                pairs[size_t(bh) * ((N + 1) / 2) + t++] = make_int2(i, j);
            } else if (j < 0) {
                if (pending < 0) {
                    pending = i;
                } else {
                    pairs[size_t(bh) * ((N + 1) / 2) + t++] = make_int2(pending, i);
                    pending = -1;
                }
            }
        }
        if (pending >= 0) pairs[size_t(bh) * ((N + 1) / 2) + t++] = make_int2(pending, -1);
    }
}

#ifndef PISA_MATCH_SMEM
#define PISA_MATCH_SMEM 1
#endif

}  // namespace

cudaError_t launch_pairing(const uint32_t* mask, int N, int W, int qb0, int qb1, int BH, int* cand,
                           int2* pairs, cudaStream_t s, uint16_t* ov) {
    cudaError_t e;
    if (ov && pairing_full_supported(qb0, qb1, W)) {
        e = launch_pairing_full_candidates(mask, N, W, qb0, qb1, BH, ov, cand, s);
    } else {
        const size_t sm1 = size_t(8 + 2 * kWindow) * W * 4;
        cudaFuncSetAttribute(pair_candidates_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm1));
        pair_candidates_kernel<<<dim3((qb1 - qb0 + 7) / 8, BH), 256, sm1, s>>>(mask, N, W, qb0, qb1, cand);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) return e;
    const size_t sm2 = size_t(2) * N * 4;
    const size_t sm2c = sm2 + size_t(N) * kCand * 2;
    if (PISA_MATCH_SMEM && N <= kMatchPer * kMatchThreads && N < 32768 && sm2c <= 200 * 1024) {
        cudaFuncSetAttribute(pair_match_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm2c));
        pair_match_kernel<true><<<BH, kMatchThreads, sm2c, s>>>(cand, N, qb0, qb1, pairs);
    } else {
        cudaFuncSetAttribute(pair_match_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm2));
        pair_match_kernel<false><<<BH, kMatchThreads, sm2, s>>>(cand, N, qb0, qb1, pairs);
    }
    return cudaGetLastError();
}

}  // namespace pisa_b200
