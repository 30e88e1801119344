// Microbenchmark: the fused kernel's MMA-warp issue loop in isolation. Per
// iteration: wait on three (already completed) mbarriers, fence, one elected
// block issuing 8 TS PV MMAs (M128 N128) + commit and 8 SS S MMAs (M128 N128)
// + commit -- 1024 tensor cycles of work. Modes: 0 alone; 1 with 8 extra warps
// running an FFMA/MUFU loop (the softmax's instruction mix) on all four SM
// sub-partitions; 2 same but the extra warps only on sub-partitions != the MMA
// warp's.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_01077_b200/csrc issue_loop.cu -o issue_loop
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace pisa_sm100;

__global__ void __launch_bounds__(384, 1) loop(int mode, int iters, unsigned long long* out, float* sink) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 98304);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 8);
    volatile int* stop = reinterpret_cast<volatile int*>(bar + 9);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 6; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
        *stop = 0;
    }
    if (warp == 2) {
        tmem_alloc(slot, 512);
        tmem_relinquish();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (warp == 1) {
        // complete barriers 3..5 once (phase 0 done): the waits below return at once
        if (elect_one()) {
            mma_commit(&bar[3]);
            mma_commit(&bar[4]);
            mma_commit(&bar[5]);
        }
        __syncwarp();
        mbar_wait(&bar[3], 0);
        const uint64_t qd = sdesc_sw128(smem_u32(smem), 16, 1024);
        const uint64_t kd = sdesc_sw128(smem_u32(smem + 32768), 16, 1024);
        const uint64_t vd = sdesc_sw128(smem_u32(smem + 65536), 16384, 1024);
        const uint32_t idS = idesc_bf16(128, 128, 0, 0), idPV = idesc_bf16(128, 128, 0, 1);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            mbar_wait<true>(&bar[3], 0);
            mbar_wait<true>(&bar[4], 0);
            mbar_wait<true>(&bar[5], 0);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    mma_ts(tmem, tmem + 256 + (ks >> 2) * 64 + (ks & 3) * 8, vd + uint64_t((ks * 2048) >> 4), idPV,
                           1u);
                mma_commit(&bar[0]);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t off = uint64_t(((ks >> 2) * 16384 + (ks & 3) * 32) >> 4);
                    mma_ss(tmem + 128 + 128 * (it % 3), qd + off, kd + off, idS, ks != 0);
                }
                mma_commit(&bar[1]);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(&bar[2]);
        __syncwarp();
        mbar_wait(&bar[2], 0);
        const long long t1 = clock64();
        if (lane_id() == 0) {
            atomicAdd(out, (unsigned long long)(t1 - t0));
            *stop = 1;
        }
    } else if (warp >= 4 && mode > 0) {
        if (mode == 2 && (warp & 3) == 1) return;  // keep the MMA warp's sub-partition free
        float a = threadIdx.x * 1e-3f, b = 0.f;
        while (!*stop) {
#pragma unroll 16
            for (int i = 0; i < 64; ++i) {
                a = fmaf(a, 0.999f, 0.001f);
                b += ex2(a);
            }
        }
        if (b == 12345.f) sink[threadIdx.x] = b;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 8);
    cudaMalloc(&sink, 4096);
    const int smem = 98304 + 2048;
    cudaFuncSetAttribute(loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 3; ++mode) {
        const int iters = 1000;
        loop<<<148, 384, smem>>>(mode, 16, d, sink);
        cudaMemset(d, 0, 8);
        loop<<<148, 384, smem>>>(mode, iters, d, sink);
        unsigned long long h = 0;
        cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %d (%s): %.1f cycles per iteration (1024 = tensor-bound)  %s\n", mode,
               mode == 0 ? "MMA warp alone" : mode == 1 ? "+8 FFMA/MUFU warps on all SMSPs" : "+6 warps, MMA SMSP free",
               double(h) / 148 / iters, cudaGetErrorString(e));
    }
    return 0;
}
