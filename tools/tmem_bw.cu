// TMEM load / store bandwidth per SM on B200: is the fused kernel's softmax
// (S read as fp32 from TMEM, P written back as bf16) bound by TMEM traffic?
//
//   mode 0  tcgen05.ld 32x32b.x32   (one warp: 32 lanes x 32 columns x 4 B = 4 KB)
//   mode 1  tcgen05.ld 16x32bx2.x32 (the fused kernel's shape: 16 lanes x 2 halves)
//   mode 2  tcgen05.st 32x32b.x32
//   mode 3  ld 32x32b.x32 with 2 loads in flight before the wait
// Prints bytes per clock per SM for 4, 8, 12, 16 warps per SM (one CTA per SM).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_01077_b200/csrc tmem_bw.cu -o tmem_bw
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "sm100.cuh"

using namespace pisa_sm100;

__global__ void tmem_bw(int mode, int iters, unsigned long long* cyc, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        tmem_alloc(&slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    // warp w: lane quadrant w % 4, columns (w / 4) * 64 .. (a 64-column slice each)
    const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) & 7) * 64;
    uint32_t acc = 0;
    uint32_t r[32], r2[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = threadIdx.x + i;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 0) {
            tmem_ld32(base + (it & 1) * 32, r);
            tmem_ld_wait(r);
            acc ^= r[0] ^ r[17] ^ r[31];
        } else if (mode == 1) {
            tmem_ld16x2_32<32>(base + (it & 1) * 16, r);
            tmem_ld_wait(r);
            acc ^= r[0] ^ r[17] ^ r[31];
        } else if (mode == 2) {
            r[0] = it;
            tmem_st32(base + (it & 1) * 32, r);
            tmem_st_wait();
        } else {
            tmem_ld32(base, r);
            tmem_ld32(base + 32, r2);
            tmem_ld_wait(r);
            tmem_ld_wait(r2);
            acc ^= r[0] ^ r[31] ^ r2[5] ^ r2[30];
        }
    }
    const long long t1 = clock64();
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;
    if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* d;
    uint32_t* sink;
    cudaMalloc(&d, 8);
    cudaMalloc(&sink, 4096 * 4);
    const char* names[] = {"ld 32x32b.x32", "ld 16x32bx2.x32", "st 32x32b.x32", "ld 32x32b.x32, 2 in flight"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int warps : {4, 8, 12, 16}) {
            const int iters = 4096;
            tmem_bw<<<148, warps * 32>>>(mode, 16, d, sink);
            cudaMemset(d, 0, 8);
            tmem_bw<<<148, warps * 32>>>(mode, iters, d, sink);
            unsigned long long h = 0;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            const double c = double(h) / 148;  // cycles per SM
            const double bytes = double(iters) * warps * 4096.0 * (mode == 3 ? 2 : 1);
            printf("%-30s warps/SM %2d : %7.1f B/clk/SM  (%s)\n", names[mode], warps, bytes / c,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
