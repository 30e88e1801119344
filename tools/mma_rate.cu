// Microbenchmark: tcgen05.mma issue/throughput per instruction shape and operand
// source, the shapes the fused kernel issues (cycles per instruction, 1 or 2 CTAs/SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_01077_b200/csrc mma_rate.cu -o mma_rate
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace pisa_sm100;

// mode 0: SS M128 N64 (S = Q K^T); 1: SS M128 N128; 2: TS M128 N128 (P V, V MN-major);
// 3: SS M128 N256; 4: TS M128 N64
__global__ void __launch_bounds__(128, 1) rate(int mode, int iters, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(slot, 256);
        tmem_relinquish();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (mode == 8 || mode == 9) {
        // 8: whole warp 0 runs the loop (uniform values), elect.sync issues;
        // 9: same in warps 0 AND 1, each into its own accumulator
        if (warp == 0 || (mode == 9 && warp == 1)) {
            const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
            const uint32_t d = tmem + uint32_t(warp) * 64;
            const long long t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                const uint32_t ks = i & 3;
                uint32_t pred;
                asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(pred));
                if (pred)
                    mma_ss(d, sdesc_sw128(a + ks * 32, 16, 1024), sdesc_sw128(b + ks * 32, 16, 1024),
                           idesc_bf16(128, 64, 0, 0), 1);
                __syncwarp();
            }
            const long long t1 = clock64();
            if (threadIdx.x % 32 == 0) {
                mma_commit(bar + warp);
            }
            __syncwarp();
            mbar_wait(bar + warp, 0);
            const long long t2 = clock64();
            if (threadIdx.x % 32 == 0) {
                atomicAdd(out + 0, (unsigned long long)(t1 - t0));
                atomicAdd(out + 1, (unsigned long long)(t2 - t0));
            }
        }
    } else if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t ks = i & 3;
            const uint32_t acc = (mode >= 5) ? uint32_t((i % (mode - 3)) * 64) : 0u;  // 5: 2 chains, 6: 3, 7: 4
            if (mode >= 5) {
                mma_ss(tmem + acc, sdesc_sw128(a + ks * 32, 16, 1024), sdesc_sw128(b + ks * 32, 16, 1024),
                       idesc_bf16(128, 64, 0, 0), 1);
                continue;
            }
            switch (mode) {
                case 0:
                    mma_ss(tmem + 128, sdesc_sw128(a + ks * 32, 16, 1024), sdesc_sw128(b + ks * 32, 16, 1024),
                           idesc_bf16(128, 64, 0, 0), 1);
                    break;
                case 1:
                    mma_ss(tmem + 128, sdesc_sw128(a + ks * 32, 16, 1024), sdesc_sw128(b + ks * 32, 16, 1024),
                           idesc_bf16(128, 128, 0, 0), 1);
                    break;
                case 2:
                    mma_ts(tmem, tmem + 128 + ks * 8, sdesc_sw128(b + ks * 2048, 8192, 1024),
                           idesc_bf16(128, 128, 0, 1), 1);
                    break;
                case 3:
                    mma_ss(tmem, sdesc_sw128(a + ks * 32, 16, 1024), sdesc_sw128(b + ks * 32, 16, 1024),
                           idesc_bf16(128, 256, 0, 0), 1);
                    break;
                case 4:
                    mma_ts(tmem + 128, tmem + 192 + ks * 8, sdesc_sw128(b + ks * 2048, 8192, 1024),
                           idesc_bf16(128, 64, 0, 1), 1);
                    break;
            }
        }
        const long long t1 = clock64();
        mma_commit(bar);
        mbar_wait(bar, 0);
        const long long t2 = clock64();
        atomicAdd(out + 0, (unsigned long long)(t1 - t0));
        atomicAdd(out + 1, (unsigned long long)(t2 - t0));
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    const char* names[] = {"SS M128 N64  (S=QK^T)", "SS M128 N128", "TS M128 N128 (PV)", "SS M128 N256",
                           "TS M128 N64", "SS N64 2 acc chains", "SS N64 3 acc chains", "SS N64 4 acc chains",
                           "SS N64 warp-uniform", "SS N64 2 issuing warps"};
    const double macs[] = {128 * 64 * 16, 128 * 128 * 16, 128 * 128 * 16, 128 * 256 * 16, 128 * 64 * 16,
                           128 * 64 * 16, 128 * 64 * 16, 128 * 64 * 16, 128 * 64 * 16, 128 * 64 * 16};
    const int smem = 65536 + 2048;
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int cps : {1, 2}) {
        for (int mode = 0; mode < 10; ++mode) {
            const int iters = 4096;
            rate<<<148 * cps, 128, smem>>>(mode, 64, d);
            cudaMemset(d, 0, 16);
            rate<<<148 * cps, 128, smem>>>(mode, iters, d);
            unsigned long long h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            const int issuers = mode == 9 ? 2 : 1;
            const double issue = double(h[0]) / (148 * cps * issuers) / iters, total = double(h[1]) / (148 * cps * issuers) / iters;
            printf("CTAs/SM %d %-22s issue %.1f cyc/inst, complete %.1f cyc/inst -> %.0f MAC/clk/SM (%s)\n", cps,
                   names[mode], issue, total, macs[mode] * cps * issuers / total, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
