// Microbenchmark: chip-wide TMA delivery of random 64-row x 128-col bf16 blocks
// (16 KB, the fused kernel's K/V tiles) from an L2-resident buffer, one CTA per
// SM, 8 x 16 KB stages per round.
//   mode 0: unicast, every CTA its own random blocks
//   mode 1: unicast, the C CTAs of a cluster load the SAME blocks (L2 dedup?)
//   mode 2: multicast: CTA r of the cluster loads stage s if s % C == r and
//           multicasts it to all C CTAs (each CTA still receives every block)
// Reports delivered bytes/s (into shared memory, all SMs) and L2-read bytes/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_01077_b200/csrc l2_bw.cu -o l2_bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "sm100.cuh"

using namespace pisa_sm100;

constexpr int kStages = 8;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                               int c1, int c2, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
        : "memory");
}

__global__ void __launch_bounds__(32, 1) bw(const __grid_constant__ CUtensorMap tm, int nblocks, int rounds,
                                            int mode, int C) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * 16384);
    const uint32_t rank = C > 1 ? cluster_rank() : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (C > 1) cluster_sync();
    const uint32_t seed = (mode == 0) ? blockIdx.x : blockIdx.x / C;
    uint32_t h = seed * 2654435761u + 12345u;
    for (int r = 0; r < rounds; ++r) {
        if (elect_one()) {
            for (int s = 0; s < kStages; ++s) {
                h = h * 1664525u + 1013904223u;
                const int blk = int((h >> 8) % uint32_t(nblocks));
                mbar_expect_tx(&full[s], 16384);
                if (mode == 2) {
                    if (s % C == int(rank)) {
                        tma_load_3d_mc(smem + s * 16384, &tm, &full[s], 0, blk * 64, 0, uint16_t((1u << C) - 1));
                        tma_load_3d_mc(smem + s * 16384 + 8192, &tm, &full[s], 64, blk * 64, 0,
                                       uint16_t((1u << C) - 1));
                    }
                } else {
                    tma_load_3d(smem + s * 16384, &tm, &full[s], 0, blk * 64, 0);
                    tma_load_3d(smem + s * 16384 + 8192, &tm, &full[s], 64, blk * 64, 0);
                }
            }
        }
        __syncwarp();
        for (int s = 0; s < kStages; ++s) mbar_wait(&full[s], r & 1);
        if (C > 1) cluster_sync();
    }
}

// Continuous ring: S stages always in flight (wait oldest, re-issue it).
__global__ void __launch_bounds__(128, 1) ring(const __grid_constant__ CUtensorMap tm, int nblocks, int iters,
                                              int S, unsigned long long* lat) {
    extern __shared__ uint8_t raw[];
    const int w = threadIdx.x >> 5;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023)) +
                    w * (S * 16384 + 1024);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * 16384);
    if ((threadIdx.x & 31) == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t h = (blockIdx.x * 4 + w) * 2654435761u + 12345u;
    long long t_issue[16];
    long long tsum = 0;
    for (int i = 0; i < iters + S; ++i) {
        const int s = i % S;
        if (i >= S) {
            mbar_wait(&full[s], ((i / S) - 1) & 1);
            tsum += clock64() - t_issue[s];
        }
        if (i >= iters) continue;
        h = h * 1664525u + 1013904223u;
        const int blk = int((h >> 8) % uint32_t(nblocks));
        t_issue[s] = clock64();
        if (elect_one()) {
            mbar_expect_tx(&full[s], 16384);
            tma_load_3d(smem + s * 16384, &tm, &full[s], 0, blk * 64, 0);
            tma_load_3d(smem + s * 16384 + 8192, &tm, &full[s], 64, blk * 64, 0);
        }
        __syncwarp();
    }
    if (lat && (threadIdx.x & 31) == 0) atomicAdd(lat, (unsigned long long)(tsum / iters));
}

// One ring of S 16 KB stages per CTA; each stage = 4 boxes of 64 cols x 32 rows.
// how 0: lane 0 of warp 0 issues all 4 boxes; 1: lanes 0..3 of warp 0 one box
// each; 2: warps 0..3 one box each (elected lane).
__global__ void __launch_bounds__(128, 1) split(const __grid_constant__ CUtensorMap tm32, int nblocks, int iters,
                                               int S, int how, unsigned long long* lat) {
    extern __shared__ uint8_t raw[];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * 16384);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], how >= 1 ? 4 : 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (how < 2 && w != 0) return;
    uint32_t h = blockIdx.x * 2654435761u + 12345u;
    long long t_issue[16];
    long long tsum = 0;
    for (int i = 0; i < iters + S; ++i) {
        const int s = i % S;
        if (i >= S) {
            mbar_wait(&full[s], ((i / S) - 1) & 1);
            tsum += clock64() - t_issue[s];
        }
        if (i >= iters) continue;
        h = h * 1664525u + 1013904223u;
        const int blk = int((h >> 8) % uint32_t(nblocks));
        t_issue[s] = clock64();
        if (how == 0) {
            if (elect_one()) {
                mbar_expect_tx(&full[s], 16384);
                for (int b = 0; b < 4; ++b)
                    tma_load_3d(smem + s * 16384 + b * 4096, &tm32, &full[s], (b & 1) * 64, blk * 64 + (b >> 1) * 32, 0);
            }
        } else if (how == 1) {
            if (l < 4) {
                mbar_expect_tx(&full[s], 4096);
                tma_load_3d(smem + s * 16384 + l * 4096, &tm32, &full[s], (l & 1) * 64, blk * 64 + (l >> 1) * 32, 0);
            }
        } else if (how == 2) {
            if (elect_one()) {
                mbar_expect_tx(&full[s], 4096);
                tma_load_3d(smem + s * 16384 + w * 4096, &tm32, &full[s], (w & 1) * 64, blk * 64 + (w >> 1) * 32, 0);
            }
        } else if (how == 3) {  // 4 warps, each its quarter from a DIFFERENT random block
            const int b2 = int(((h ^ (uint32_t(w) * 0x9E3779B9u)) >> 8) % uint32_t(nblocks));
            if (elect_one()) {
                mbar_expect_tx(&full[s], 4096);
                tma_load_3d(smem + s * 16384 + w * 4096, &tm32, &full[s], (w & 1) * 64, b2 * 64 + (w >> 1) * 32, 0);
            }
        } else {  // how 4: 4 warps, 64-col x 32-row quarter of the same block but via 1 lane per warp, no elect
            if (l == 0) {
                mbar_expect_tx(&full[s], 4096);
                tma_load_3d(smem + s * 16384 + w * 4096, &tm32, &full[s], (w & 1) * 64, blk * 64 + (w >> 1) * 32, 0);
            }
        }
        __syncwarp();
    }
    if (lat && threadIdx.x == 0) atomicAdd(lat, (unsigned long long)(tsum / iters));
}

// Generic ring: W warps, S stages per warp, stage s of warp w at
// w*wstride + s*sstride; shared=1: warp w uses barrier set 0 (count W) and
// loads quarter w of the stage (4 KB) instead of its own 16 KB.
__global__ void __launch_bounds__(128, 1) gring(const __grid_constant__ CUtensorMap tm, int nblocks, int iters,
                                               int S, int sstride, int wstride, unsigned long long* lat) {
    extern __shared__ uint8_t raw[];
    const int w = threadIdx.x >> 5;
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(base);  // [4][16]
    uint8_t* smem = base + 1024 + w * wstride;
    uint64_t* full = bars + w * 16;
    if ((threadIdx.x & 31) == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t h = (blockIdx.x * 4 + w) * 2654435761u + 12345u;
    long long t_issue[16];
    long long tsum = 0;
    for (int i = 0; i < iters + S; ++i) {
        const int s = i % S;
        if (i >= S) {
            mbar_wait(&full[s], ((i / S) - 1) & 1);
            tsum += clock64() - t_issue[s];
        }
        if (i >= iters) continue;
        h = h * 1664525u + 1013904223u;
        const int blk = int((h >> 8) % uint32_t(nblocks));
        t_issue[s] = clock64();
        if (elect_one()) {
            mbar_expect_tx(&full[s], 16384);
            tma_load_3d(smem + s * sstride, &tm, &full[s], 0, blk * 64, 0);
            tma_load_3d(smem + s * sstride + 8192, &tm, &full[s], 64, blk * 64, 0);
        }
        __syncwarp();
    }
    if (lat && (threadIdx.x & 31) == 0) atomicAdd(lat, (unsigned long long)(tsum / iters));
}

// Pair test: per iteration, issue 2 x 16 KB loads (A, B) and wait for both.
// mode 0: one warp, A->barA, B->barB (record both completion times)
// mode 1: one warp, A and B -> one barrier (32 KB)
// mode 2: warp 0 issues A->barA, warp 1 issues B->barB
__global__ void __launch_bounds__(64, 1) pair(const __grid_constant__ CUtensorMap tm, int nblocks, int iters, int mode,
                                             unsigned long long* lat) {
    extern __shared__ uint8_t raw[];
    const int w = threadIdx.x >> 5;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (mode != 2 && w == 1) return;
    uint32_t h = blockIdx.x * 2654435761u + 12345u;
    long long ta = 0, tb = 0;
    for (int i = 0; i < iters; ++i) {
        h = h * 1664525u + 1013904223u;
        const int b1 = int((h >> 8) % uint32_t(nblocks));
        const int b2 = int((h >> 3) % uint32_t(nblocks));
        const long long t0 = clock64();
        if (elect_one()) {
            if (mode == 0) {
                mbar_expect_tx(&bar[0], 16384);
                tma_load_3d(smem, &tm, &bar[0], 0, b1 * 64, 0);
                tma_load_3d(smem + 8192, &tm, &bar[0], 64, b1 * 64, 0);
                mbar_expect_tx(&bar[1], 16384);
                tma_load_3d(smem + 16384, &tm, &bar[1], 0, b2 * 64, 0);
                tma_load_3d(smem + 24576, &tm, &bar[1], 64, b2 * 64, 0);
            } else if (mode >= 3) {
                mbar_expect_tx(&bar[0], 16384);
                tma_load_3d(smem, &tm, &bar[0], 0, b1 * 64, 0);
                tma_load_3d(smem + 8192, &tm, &bar[0], 64, b1 * 64, 0);
                const long long t1 = clock64();
                while (clock64() - t1 < (mode == 3 ? 300 : 600)) {
                }
                mbar_expect_tx(&bar[1], 16384);
                tma_load_3d(smem + 16384, &tm, &bar[1], 0, b2 * 64, 0);
                tma_load_3d(smem + 24576, &tm, &bar[1], 64, b2 * 64, 0);
            } else if (mode == 1) {
                mbar_expect_tx(&bar[0], 32768);
                tma_load_3d(smem, &tm, &bar[0], 0, b1 * 64, 0);
                tma_load_3d(smem + 8192, &tm, &bar[0], 64, b1 * 64, 0);
                tma_load_3d(smem + 16384, &tm, &bar[0], 0, b2 * 64, 0);
                tma_load_3d(smem + 24576, &tm, &bar[0], 64, b2 * 64, 0);
            } else {
                mbar_expect_tx(&bar[w], 16384);
                tma_load_3d(smem + w * 16384, &tm, &bar[w], 0, (w ? b2 : b1) * 64, 0);
                tma_load_3d(smem + w * 16384 + 8192, &tm, &bar[w], 64, (w ? b2 : b1) * 64, 0);
            }
        }
        __syncwarp();
        if (mode == 0 || mode >= 3) {
            mbar_wait(&bar[0], i & 1);
            ta += clock64() - t0;
            mbar_wait(&bar[1], i & 1);
            tb += clock64() - t0;
        } else if (mode == 1) {
            mbar_wait(&bar[0], i & 1);
            ta += clock64() - t0;
            tb = ta;
        } else {
            mbar_wait(&bar[w], i & 1);
            ta += clock64() - t0;
        }
        if (mode == 2) asm volatile("bar.sync 1, 64;");
    }
    if (lat && (threadIdx.x & 31) == 0 && w == 0) {
        atomicAdd(lat, (unsigned long long)(ta / iters));
        atomicAdd(lat + 1, (unsigned long long)(tb / iters));
    }
}

int main(int argc, char** argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int rows = 64 * 2048;  // 2048 blocks of 16 KB = 32 MB (L2 resident)
    void* buf;
    cudaMalloc(&buf, size_t(rows) * 128 * 2);
    cudaMemset(buf, 0, size_t(rows) * 128 * 2);
    CUtensorMap tm;
    cuuint64_t gd[3] = {128, cuuint64_t(rows), 1};
    cuuint64_t gs[2] = {256, cuuint64_t(rows) * 256};
    cuuint32_t bx[3] = {64, 64, 1}, es[3] = {1, 1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, gd, gs, bx, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
        printf("encode failed %d\n", int(cr));
        return 1;
    }
    const int smem = kStages * 16384 + 1024 + 256;
    cudaFuncSetAttribute(bw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bw, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int rounds = 400;
    struct Cfg {
        int mode, C;
    } cfgs[] = {{0, 1}};
    for (auto c : cfgs) {
        const int grid = (nsm / c.C) * c.C;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(32);
        lc.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c.C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&lc, bw, tm, 2048, rounds, c.mode, c.C);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&lc, bw, tm, 2048, rounds, c.mode, c.C);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double delivered = double(grid) * rounds * kStages * 16384;
        const double l2read = (c.mode == 0) ? delivered : delivered / c.C;
        printf("mode %d C %d grid %d: %.3f ms  delivered %.2f TB/s  per-SM %.1f B/ns  L2-read %.2f TB/s  %s\n",
               c.mode, c.C, grid, ms, delivered / ms / 1e9, delivered / ms / 1e6 / grid, l2read / ms / 1e9,
               cudaGetErrorString(e));
    }
    unsigned long long* dlat;  // per-warp rings below
    CUtensorMap tm32;
    {
        cuuint32_t bx32[3] = {64, 32, 1};
        cuTensorMapEncodeTiled(&tm32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, gd, gs, bx32, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    cudaMalloc(&dlat, 8);
    {
        unsigned long long* pl;
        cudaMalloc(&pl, 16);
        cudaFuncSetAttribute(pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
        for (int per_sm = 1; per_sm <= 2; ++per_sm)
            for (int mode = 0; mode < 5; ++mode) {
                cudaMemset(pl, 0, 16);
                pair<<<nsm * per_sm, 64, 40000>>>(tm, 2048, 500, mode, pl);
                unsigned long long hl[2];
                cudaError_t e = cudaMemcpy(hl, pl, 16, cudaMemcpyDeviceToHost);
                printf("pair %d CTA/SM mode %d (%s): A done %llu cyc, B done %llu cyc  %s\n", per_sm, mode,
                       mode == 0 ? "1 warp, 2 barriers" : mode == 1 ? "1 warp, 1 barrier 32K" : mode == 2 ? "2 warps" : mode == 3 ? "B 300 cyc after A" : "B 600 cyc after A",
                       hl[0] / (nsm * per_sm), hl[1] / (nsm * per_sm), cudaGetErrorString(e));
            }
    }
    struct G { int W, S, ss, ws; const char* what; } gs_[] = {
        {1, 2, 16384, 0, "W1 S2 stride16K"},
        {1, 2, 17408, 0, "W1 S2 stride17K"},
        {1, 2, 65536, 0, "W1 S2 stride64K"},
        {2, 1, 16384, 16384, "W2 S1 adjacent"},
        {2, 1, 16384, 17408, "W2 S1 +1K"},
        {2, 2, 16384, 32768, "W2 S2 adjacent"},
        {4, 1, 16384, 16384, "W4 S1 adjacent"},
    };
    for (auto g : gs_) {
        const int sm = 2048 + (g.W - 1) * g.ws + (g.S - 1) * g.ss + 16384;
        cudaFuncSetAttribute(gring, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        const int grid = nsm, iters = 1000;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        gring<<<grid, 32 * g.W, sm>>>(tm, 2048, iters, g.S, g.ss, g.ws, nullptr);
        cudaMemset(dlat, 0, 8);
        cudaEventRecord(e0);
        gring<<<grid, 32 * g.W, sm>>>(tm, 2048, iters, g.S, g.ss, g.ws, dlat);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long hl = 0;
        cudaMemcpy(&hl, dlat, 8, cudaMemcpyDeviceToHost);
        const double bytes = double(grid) * g.W * iters * 16384;
        printf("gring %-18s: %.2f TB/s (%.1f B/ns/SM), latency %llu cyc  %s\n", g.what, bytes / ms / 1e9,
               bytes / ms / 1e6 / nsm, hl / (grid * g.W), cudaGetErrorString(e));
    }
    for (int how = 2; how < 3; ++how)
        for (int S : {1, 2, 4}) {
            const int sm = S * 16384 + 2048;
            cudaFuncSetAttribute(split, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            const int grid = nsm, iters = 1000;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            split<<<grid, 128, sm>>>(tm32, 2048, iters, S, how, nullptr);
            cudaMemset(dlat, 0, 8);
            cudaEventRecord(e0);
            split<<<grid, 128, sm>>>(tm32, 2048, iters, S, how, dlat);
            cudaEventRecord(e1);
            cudaError_t e = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long hl = 0;
            cudaMemcpy(&hl, dlat, 8, cudaMemcpyDeviceToHost);
            const double bytes = double(grid) * iters * 16384;
            printf("split how=%d (%s) S=%d: %.2f TB/s (%.1f B/ns/SM), latency %llu cyc  %s\n", how,
                   how == 0 ? "1 lane, 4 boxes" : how == 1 ? "4 lanes of 1 warp" : how == 2 ? "4 warps" : how == 3 ? "4 warps, distinct blocks" : "4 warps lane0", S,
                   bytes / ms / 1e9, bytes / ms / 1e6 / nsm, hl / grid, cudaGetErrorString(e));
        }
    cudaMalloc(&dlat, 8);
    for (int per_sm = 1; per_sm <= 2; ++per_sm) {
      for (int W : {1, 2, 4}) {
        for (int S : {1, 2, 3, 4, 6}) {
            const int sm = W * (S * 16384 + 1024) + 1024;
            if (sm * per_sm > 227 * 1024) continue;
            cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            const int grid = nsm * per_sm, iters = 1000;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            ring<<<grid, 32 * W, sm>>>(tm, 2048, iters, S, nullptr);
            cudaMemset(dlat, 0, 8);
            cudaEventRecord(e0);
            ring<<<grid, 32 * W, sm>>>(tm, 2048, iters, S, dlat);
            cudaEventRecord(e1);
            cudaError_t e = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long hl = 0;
            cudaMemcpy(&hl, dlat, 8, cudaMemcpyDeviceToHost);
            const double bytes = double(grid) * W * iters * 16384;
            printf("ring: %d CTA/SM x %d warps, %d stages (%3d KB in flight/SM): %.2f TB/s (%.1f B/ns/SM), latency %llu cyc  %s\n",
                   per_sm, W, S, S * 16 * per_sm * W, bytes / ms / 1e9, bytes / ms / 1e6 / nsm, hl / (grid * W),
                   cudaGetErrorString(e));
        }
      }
    }
    return 0;
}
