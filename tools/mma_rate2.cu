// Microbenchmark: tcgen05.mma (kind::f16, M=128, K=16) throughput per shape with a
// warp-uniform issue loop (whole warp, elect.sync issues), 1 CTA per SM:
// cycles per instruction and MAC/clk/SM for SS / TS operands and N = 64/128/256,
// plus the fused kernel's per-tile mixes (S over one or two key tiles + PV).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_01077_b200/csrc mma_rate2.cu -o mma_rate2
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace pisa_sm100;

// mode: 0 SS N64, 1 SS N128, 2 SS N256, 3 TS N64, 4 TS N128, 5 TS N256 (A from TMEM, B MN-major),
//       6 tile mix A: 8x TS N64 (S) + 4x TS N128 (PV)   [current kernel, per 64-key tile]
//       7 tile mix B: 8x TS N128 (S for 2 tiles) + 8x TS N128 (PV for 2 tiles)   [per 2 tiles]
//       8 tile mix C: 8x TS N256 (S for 4 tiles) + 16x TS N128 (PV for 4 tiles)  [per 4 tiles]
__global__ void __launch_bounds__(384, 1) rate(int mode_in, int iters, unsigned long long* out,
                                                const __grid_constant__ CUtensorMap tm) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    volatile uint32_t* stop = reinterpret_cast<volatile uint32_t*>(bar + 3);
    if (threadIdx.x == 0) *stop = 0;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        for (int i = 4; i < 8; ++i) mbar_init(bar + i, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(slot, 512);
        tmem_relinquish();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    int mode = mode_in;
    const int base_mode0 = 0; (void)base_mode0;
    const bool commits = mode >= 36;
    if (commits) mode -= 36;
    const bool tmem_noise = (mode >= 9 && mode < 18) || mode >= 27, tma_noise = mode >= 18 && mode < 36;
    const int base_mode = (mode >= 45) ? mode - 36 : mode % 9;
    if (warp >= 4 && tmem_noise) {
        // softmax-like TMEM traffic: 16x32bx2 loads of 32 columns + stores of 16, lanes of this warp
        const uint32_t lb = tmem + (uint32_t(((warp & 3) * 32) + ((warp >> 2) & 1) * 16) << 16) + 384;
        uint32_t r[32];
        while (*stop == 0) {
            tmem_ld16x2_32<32>(lb, r);
            tmem_ld_wait(r);
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = r[2 * i] ^ r[2 * i + 1];
            tmem_st16x2_16<16>(lb, pk);
            tmem_st_wait();
        }
    }
    if (warp == 2 && tma_noise) {
        // TMA ring into smem [128 KB, 224 KB): random 16 KB blocks, 6 stages
        uint8_t* ring = smem + 131072;
        uint64_t* fb = bar + 8;
        if (lane_id() == 0) {
            for (int s2 = 0; s2 < 5; ++s2) mbar_init(&fb[s2], 1);
            fence_mbar_init();
        }
        __syncwarp();
        uint32_t hsh = blockIdx.x * 2654435761u + 7u;
        int i = 0;
        for (; *stop == 0; ++i) {
            const int s2 = i % 5;
            if (i >= 5) mbar_wait(&fb[s2], ((i / 5) - 1) & 1);
            hsh = hsh * 1664525u + 1013904223u;
            const int blk = int((hsh >> 8) % 2048u);
            if (elect_one()) {
                mbar_expect_tx(&fb[s2], 16384);
                tma_load_3d(ring + s2 * 16384, &tm, &fb[s2], 0, blk * 64, 0);
                tma_load_3d(ring + s2 * 16384 + 8192, &tm, &fb[s2], 64, blk * 64, 0);
            }
            __syncwarp();
        }
        for (int j = i - 5; j < i; ++j)  // drain the last (up to) 5 loads
            if (j >= 0) mbar_wait(&fb[j % 5], (j / 5) & 1);
    }
    if (warp == 0) {
        const int mode = base_mode;
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        const uint32_t dS = tmem + 256, dO = tmem, aT = tmem + 128;
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (elect_one()) {
                switch (mode) {
                    case 0:
                    case 1:
                    case 2: {
                        const uint32_t idn = idesc_bf16(128, 64 << mode, 0, 0);
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks)
                            mma_ss(dS, sdesc_sw128(a + (ks & 3) * 32, 16, 1024), sdesc_sw128(b + (ks & 3) * 32, 16, 1024),
                                   idn, 1);
                        break;
                    }
                    case 3:
                    case 4:
                    case 5: {
                        const uint32_t idn = idesc_bf16(128, 64 << (mode - 3), 0, 0);
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks)
                            mma_ts(dS, aT + ks * 8, sdesc_sw128(b + (ks & 3) * 32, 16, 1024), idn, 1);
                        break;
                    }
                    case 9:
                    case 10:
                    case 11: {  // M=64 SS, N = 64/128/256
                        const uint32_t idn = idesc_bf16(64, 64 << (mode - 9), 0, 0);
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks)
                            mma_ss(dS, sdesc_sw128(a + (ks & 3) * 32, 16, 1024), sdesc_sw128(b + (ks & 3) * 32, 16, 1024),
                                   idn, 1);
                        break;
                    }
                    case 12: {  // M=64 TS N=128
                        const uint32_t idn = idesc_bf16(64, 128, 0, 0);
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks)
                            mma_ts(dS, aT + ks * 8, sdesc_sw128(b + (ks & 3) * 32, 16, 1024), idn, 1);
                        break;
                    }
                    case 6: {
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks)
                            mma_ts(dS, aT + ks * 8, sdesc_sw128(b + (ks & 3) * 32, 16, 1024), idesc_bf16(128, 64, 0, 0), 1);
                        if (commits) { mma_commit(bar + 4); mma_commit(bar + 5); }
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            mma_ts(dO, dS + ks * 8, sdesc_sw128(b + ks * 2048, 8192, 1024), idesc_bf16(128, 128, 0, 1), 1);
                        if (commits) { mma_commit(bar + 6); mma_commit(bar + 7); }
                        break;
                    }
                    case 7: {
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks)
                            mma_ts(dS, aT + ks * 8, sdesc_sw128(b + (ks & 3) * 32, 16, 1024), idesc_bf16(128, 128, 0, 0), 1);
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks)
                            mma_ts(dO, dS + ks * 8, sdesc_sw128(b + (ks & 3) * 2048, 8192, 1024), idesc_bf16(128, 128, 0, 1), 1);
                        break;
                    }
                    case 8: {
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks)
                            mma_ts(dS, aT + ks * 8, sdesc_sw128(b + (ks & 3) * 32, 16, 1024), idesc_bf16(128, 256, 0, 0), 1);
#pragma unroll
                        for (int ks = 0; ks < 16; ++ks)
                            mma_ts(dO, dS + ks * 8, sdesc_sw128(b + (ks & 3) * 2048, 8192, 1024), idesc_bf16(128, 128, 0, 1), 1);
                        break;
                    }
                }
            }
            __syncwarp();
        }
        const long long t1 = clock64();
        if (elect_one()) mma_commit(bar);
        __syncwarp();
        mbar_wait(bar, 0);
        const long long t2 = clock64();
        if (lane_id() == 0) {
            atomicAdd(out + 0, (unsigned long long)(t1 - t0));
            atomicAdd(out + 1, (unsigned long long)(t2 - t0));
            *stop = 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    const char* names[] = {"SS N64 x8", "SS N128 x8", "SS N256 x8", "TS N64 x8", "TS N128 x8", "TS N256 x8",
                           "mix A: 1 tile (8 S N64 + 4 PV)", "mix B: 2 tiles (8 S N128 + 8 PV)",
                           "mix C: 4 tiles (8 S N256 + 16 PV)"};
    // MACs per loop iteration
    const double macs[] = {8.0 * 128 * 64 * 16,  8.0 * 128 * 128 * 16, 8.0 * 128 * 256 * 16,
                           8.0 * 128 * 64 * 16,  8.0 * 128 * 128 * 16, 8.0 * 128 * 256 * 16,
                           8.0 * 128 * 64 * 16 + 4.0 * 128 * 128 * 16, 8.0 * 128 * 128 * 16 + 8.0 * 128 * 128 * 16,
                           8.0 * 128 * 256 * 16 + 16.0 * 128 * 128 * 16};
    const double tiles[] = {0, 0, 0, 0, 0, 0, 1, 2, 4};
    const int smem = 229376 - 2048;
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    void* buf;
    const int rows = 64 * 2048;
    cudaMalloc(&buf, size_t(rows) * 256);
    cudaMemset(buf, 0, size_t(rows) * 256);
    CUtensorMap tm;
    {
        cuuint64_t gd[3] = {128, cuuint64_t(rows), 1};
        cuuint64_t gs[2] = {256, cuuint64_t(rows) * 256};
        cuuint32_t bx[3] = {64, 64, 1}, es[3] = {1, 1, 1};
        cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    for (int mode : {6, 6 + 9, 6 + 18, 6 + 27, 7, 7 + 18}) {
        const int iters = 2048;
        rate<<<148, 384, smem>>>(mode, 16, d, tm);
        cudaMemset(d, 0, 16);
        rate<<<148, 384, smem>>>(mode, iters, d, tm);
        unsigned long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        const double total = double(h[1]) / 148 / iters;
        const int bm = mode >= 45 ? 0 : mode % 9;
        if (mode >= 45) {
            const double total = double(h[1]) / 148 / iters;
            const int n = mode == 48 ? 128 : (64 << (mode - 45));
            const double mac = 8.0 * 64 * n * 16;
            printf("M64 %s N%d x8: %.1f cyc/iter -> %.0f MAC/clk/SM\n", mode == 48 ? "TS" : "SS", n, total, mac / total);
            continue;
        }
        printf("%s", mode >= 36 ? "[4 commits/tile] " : "");
        printf("%-36s %-22s %.1f cyc/iter -> %.0f MAC/clk/SM (%.0f%% of 4096)  %s\n", names[bm],
               mode >= 27 ? "+TMEM +TMA" : mode >= 18 ? "+TMA ring" : mode >= 9 ? "+TMEM ld/st (8 warps)" : "",
               total, macs[bm] / total, 100.0 * macs[bm] / total / 4096.0, cudaGetErrorString(cudaGetLastError()));
        if (tiles[bm] > 0) printf("   -> %.1f cycles per 64-key tile (tensor floor 512)\n", total / tiles[bm]);
    }
    return 0;
}
