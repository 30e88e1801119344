// Microbenchmark for the "transposed" Phase-1 tile the r01 verdict asked to
// evaluate (S^T = K_pair Q_i^T with M = 128 keys of two key blocks of ONE
// query block, N = 64 queries; O^T += V^T P^T), against the current union tile
// (S = Q_pair [K_a;K_b]^T, N = 128, SS; O += P V, TS with P from TMEM).
//
// Per loop iteration, all operands resident in shared memory / TMEM:
//   mode 0  current tile : 8 x SS M128 N128 (S) + 8 x TS M128 N128 (PV)   = 4 (q-block, k-block) slots
//   mode 1  transposed   : 8 x SS M128 N64  (S^T) + 8 x SS M128 N64 (PV^T, A = V^T MN-major,
//                          B = P^T MN-major)                               = 2 slots, all useful
//   mode 2  transposed + the 16 KB of P^T stores per iteration (8 warps of st.shared.v4,
//                          the softmax's output) on the same shared-memory port
//   mode 3  transposed + P^T stores + a free-running cp.async.bulk copy stream
//                          (global->shared, like the K/V tiles)
//   mode 4  current tile + exactly 64 KB of bulk copies per iteration (the K
//                          and V tiles of one super-tile): is the fused kernel's
//                          tile bound by the shared-memory port?
//   mode 5  current tile with Q in TMEM (S as TS, A from TMEM) + 64 KB copies
//                          per iteration: the shared-memory traffic of S halves
//   mode 7  current tile + the softmax's TMEM traffic, paced: per MMA iteration
//                          8 warps each load 64 fp32 columns of their 16-lane
//                          half (64 KB, the S of a super-tile) and store 32
//                          (32 KB, its P) with tcgen05.ld/st 16x32bx2
//   mode 8  as 7, free-running TMEM traffic (an upper bound on contention)
//   mode 6  transposed + 16 KB P^T stores + 64 KB bulk copies per iteration,
//                          both paced (the full shared-memory load of a
//                          transposed tile: K and V of 128 keys, P^T)
// Prints cycles per iteration and per USEFUL (query block, key block) pair at
// gaussian routing (union/k = 1.78 -> 4 slots hold 2.25 useful pairs).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_01077_b200/csrc st_mix.cu -o st_mix -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "sm100.cuh"

using namespace pisa_sm100;

__global__ void __launch_bounds__(384, 1) st_mix(int mode, int iters, unsigned long long* out, const uint8_t* gsrc) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    // [0,64K): operand A/B tiles, [64K,80K): P^T, [96K, 192K): copy ring (3 x 32 KB), 200K: barriers
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 204800);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 16);
    volatile uint32_t* stop = reinterpret_cast<volatile uint32_t*>(bar + 17);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    volatile uint32_t* ctr = reinterpret_cast<volatile uint32_t*>(bar + 18);  // MMA iterations issued
    if (threadIdx.x == 0) {
        *stop = 0;
        *ctr = 0;
        for (int i = 0; i < 8; ++i) mbar_init(bar + i, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        tmem_alloc(slot, 512);
        tmem_relinquish();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    const bool ptx = mode == 2 || mode == 3 || mode == 6;  // transposed modes with P^T stores
    if (warp >= 4 && (mode == 7 || mode == 8)) {
        // softmax-like TMEM traffic on columns [384, 512) (the MMAs use [0, 384))
        const uint32_t base = tmem + (uint32_t((warp & 3) * 32 + ((warp - 4) >> 2) * 16) << 16) + 384;
        for (uint32_t r = 0; __shfl_sync(0xffffffffu, *stop, 0) == 0; ++r) {
            if (mode == 7)
                while (__shfl_sync(0xffffffffu, (*stop == 0 && r >= (*ctr) + 2u) ? 1u : 0u, 0)) {
                }
            uint32_t a0[32], a1[32];
            tmem_ld16x2_32<32>(base, a0);
            tmem_ld16x2_32<32>(base + 64, a1);
            tmem_ld_wait(a0);
            tmem_ld_wait(a1);
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = a0[2 * i] ^ a1[2 * i + 1];
            tmem_st16x2_16<16>(base, pk);
            tmem_st16x2_16<16>(base + 64, pk);
            tmem_st_wait();
        }
    }
    if (warp >= 4 && ptx) {
        // P^T producer traffic: each of 8 warps stores 2 KB (16 B per lane x 4) per round
        uint4* pt = reinterpret_cast<uint4*>(smem + 65536) + (warp - 4) * 128;
        uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
        for (uint32_t r = 0; __shfl_sync(0xffffffffu, *stop, 0) == 0; ++r) {
            if (mode == 6)  // paced: one 16 KB P^T per MMA iteration
                while (__shfl_sync(0xffffffffu, (*stop == 0 && r >= (*ctr) + 2u) ? 1u : 0u, 0)) {
                }
#pragma unroll
            for (int j = 0; j < 4; ++j) pt[j * 32 + lane_id()] = v;
            v.x += 1;
            __syncwarp();
        }
    }
    if (warp == 2 && mode >= 3) {
        // 32 KB per round through cp.async.bulk (the K / V tile stream); modes
        // 4 / 5 pace it at two rounds (64 KB) per MMA iteration
        uint8_t* ring = smem + 98304;
        int i = 0;
        for (; __shfl_sync(0xffffffffu, *stop, 0) == 0; ++i) {
            if (mode >= 4)
                while (__shfl_sync(0xffffffffu, (*stop == 0 && uint32_t(i) >= 2u * (*ctr) + 3u) ? 1u : 0u, 0)) {
                }
            const int s = i % 3;
            if (i >= 3) mbar_wait(bar + 4 + s, ((i / 3) - 1) & 1);
            if (elect_one()) {
                mbar_expect_tx(bar + 4 + s, 32768);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                        smem_u32(ring + s * 32768)),
                    "l"(gsrc + size_t((i * 7919) & 4095) * 32768), "r"(32768), "r"(smem_u32(bar + 4 + s))
                    : "memory");
            }
            __syncwarp();
        }
        for (int j = i - 3; j < i; ++j)
            if (j >= 0) mbar_wait(bar + 4 + (j % 3), (j / 3) & 1);
    }
    if (warp == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768), p = smem_u32(smem + 65536);
        const uint32_t dS = tmem + 256, dO = tmem;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (elect_one()) {
                if (mode == 0 || mode == 4 || mode == 5 || mode == 7 || mode == 8) {
                    if (mode == 5) {
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks)  // S = Q K^T with Q in TMEM (columns 448..511)
                            mma_ts(dS, tmem + 448 + ks * 8, sdesc_sw128(b + (ks & 3) * 32, 16, 1024),
                                   idesc_bf16(128, 128, 0, 0), 1);
                    } else {
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks)
                            mma_ss(dS, sdesc_sw128(a + (ks & 3) * 32, 16, 1024),
                                   sdesc_sw128(b + (ks & 3) * 32, 16, 1024), idesc_bf16(128, 128, 0, 0), 1);
                    }
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks)
                        mma_ts(dO, dS + ks * 8, sdesc_sw128(b + (ks & 3) * 2048, 8192, 1024), idesc_bf16(128, 128, 0, 1),
                               1);
                } else {
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks)  // S^T: A = K (K-major), B = Q (K-major)
                        mma_ss(dS, sdesc_sw128(a + (ks & 3) * 32, 16, 1024), sdesc_sw128(b + (ks & 3) * 32, 16, 1024),
                               idesc_bf16(128, 64, 0, 0), 1);
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks)  // PV^T: A = V^T (MN-major), B = P^T (MN-major)
                        mma_ss(dO, sdesc_sw128(a + (ks & 3) * 2048, 8192, 1024),
                               sdesc_sw128(p + (ks & 3) * 2048, 8192, 1024), idesc_bf16(128, 64, 1, 1), 1);
                }
            }
            __syncwarp();
            if (lane_id() == 0) *ctr = uint32_t(it + 1);
        }
        if (elect_one()) mma_commit(bar);
        __syncwarp();
        mbar_wait(bar, 0);
        const long long t1 = clock64();
        if (lane_id() == 0) {
            atomicAdd(out, (unsigned long long)(t1 - t0));
            *stop = 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

int main(int argc, char** argv) {
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    unsigned long long* d;
    cudaMalloc(&d, 8);
    uint8_t* g;
    cudaMalloc(&g, size_t(4096) * 32768);
    cudaMemset(g, 0, size_t(4096) * 32768);
    const int smem = 229376 - 1024;
    cudaFuncSetAttribute(st_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[] = {"current union tile (8 SS N128 + 8 TS N128)", "transposed (8 SS N64 S^T + 8 SS N64 PV^T)",
                           "transposed + 16 KB P^T st.shared / iter", "transposed + P^T stores + bulk copies",
                           "current tile + 64 KB bulk copies / iter", "current, Q in TMEM + 64 KB copies / iter",
                           "transposed + P^T + 64 KB copies / iter (paced)",
                           "current tile + softmax TMEM ld/st (paced)", "current tile + softmax TMEM ld/st (free)"};
    const double useful[] = {2.25, 2.0, 2.0, 2.0, 2.25, 2.25, 2.0, 2.25, 2.25};  // useful (q-block, k-block) pairs / iter (gaussian)
    for (int mode = 0; mode < 9; ++mode) {
        if (only >= 0 && mode != only) continue;
        st_mix<<<148, 384, smem>>>(mode, 16, d, g);
        cudaMemset(d, 0, 8);
        const int iters = 4096;
        st_mix<<<148, 384, smem>>>(mode, iters, d, g);
        unsigned long long h = 0;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        const double cyc = double(h) / 148 / iters;
        printf("%-48s %7.1f cyc/iter  %6.1f cyc per useful pair  (%s)\n", names[mode], cyc, cyc / useful[mode],
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
