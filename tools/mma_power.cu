// Microbenchmark: power and clocks of sustained tcgen05 MMAs at M=128 vs M=64
// (same N, K and instruction count; M=64 does half the MACs). One CTA per SM,
// one elected thread issuing SS MMAs (kind::f16, N=128, K=16) in batches of 8
// with two batches in flight, random bf16 operands (zeros would understate
// power). Run with nvidia-smi sampling power.draw / clocks.sm alongside; the
// host prints wall-clock phase boundaries.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_01077_b200/csrc mma_power.cu -o mma_power
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>

#include "sm100.cuh"

using namespace pisa_sm100;

__global__ void __launch_bounds__(128, 1) pw(int M, long long iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5;
    // random bf16 in (-1, 1): hash of the element index
    for (int i = threadIdx.x; i < 65536 / 2; i += blockDim.x) {
        uint32_t h = uint32_t(i) * 2654435761u ^ (blockIdx.x * 97u);
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        h ^= h >> 15;
        const float f = (float(h & 0xffffu) / 32768.f) - 1.f;
        reinterpret_cast<__nv_bfloat16*>(smem)[i] = __float2bfloat16_rn(f);
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
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
    if (warp == 0) {
        const uint32_t idesc = idesc_bf16(M, 128, 0, 0);
        const uint64_t ad = sdesc_sw128(smem_u32(smem), 16, 1024);
        const uint64_t bd = sdesc_sw128(smem_u32(smem + 32768), 16, 1024);
        const long long t0 = clock64();
        for (long long it = 0; it < iters; ++it) {
            if (it >= 2) mbar_wait(&bar[it & 1], uint32_t(((it - 2) >> 1) & 1));
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t off = uint64_t(((ks >> 2) * 16384 + (ks & 3) * 32) >> 4);
                    mma_ss(tmem + (it & 1) * 128, ad + off, bd + off, idesc, ks != 0);
                }
                mma_commit(&bar[it & 1]);
            }
            __syncwarp();
        }
        for (long long it = iters; it < iters + 2; ++it) mbar_wait(&bar[it & 1], uint32_t(((it - 2) >> 1) & 1));
        if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int smem = 65536 + 2048;
    cudaFuncSetAttribute(pw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    pw<<<148, 128, smem>>>(128, 1000, d);  // warm-up
    cudaDeviceSynchronize();
    const long long iters = 600000;  // ~3 s at M=128 (512 cycles per batch)
    for (int M : {128, 64, 128, 64}) {
        const auto t0 = std::chrono::system_clock::now();
        pw<<<148, 128, smem>>>(M, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        const auto t1 = std::chrono::system_clock::now();
        unsigned long long cyc[148];
        cudaMemcpy(cyc, d, sizeof(cyc), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += double(cyc[i]) / 148;
        const double secs = std::chrono::duration<double>(t1 - t0).count();
        const double macs = 148.0 * iters * 8 * double(M) * 128 * 16;
        printf("M=%d: wall %.3f s (%.3f .. %.3f s since epoch mod 1000), %.1f cycles/batch, SM clock %.0f MHz, "
               "%.0f dense TFLOP/s  %s\n",
               M, secs, std::fmod(std::chrono::duration<double>(t0.time_since_epoch()).count(), 1000.0),
               std::fmod(std::chrono::duration<double>(t1.time_since_epoch()).count(), 1000.0), avg / iters,
               avg / secs / 1e6, 2 * macs / secs / 1e12, cudaGetErrorString(e));
        fflush(stdout);
    }
    return 0;
}
