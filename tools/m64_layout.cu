// Checks the TMEM layout of tcgen05.mma M=64 (cta_group::1, kind::f16) with A
// from TMEM: D row r (0..63) is expected at lane (r/16)*32 + off + r%16 where
// `off` is the lane offset in the D / A addresses (0 or 16), i.e. the layout the
// fused kernel uses for query block 2t (+0) and 2t+1 (+16). Also times M=64 TS
// MMAs (N = 64 / 128) with a warp-uniform issue loop.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_01077_b200/csrc m64_layout.cu -o m64_layout
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace pisa_sm100;

// A: [64][128] bf16 row-major (global), B: [N][128] bf16 (K-major, global)
// out: [64][N] fp32
template <int N>
__global__ void __launch_bounds__(128, 1) m64(const __nv_bfloat16* A, const __nv_bfloat16* B, float* out, int off) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // B into smem, SW128 K-major: half h (cols 64h..), row n at h*N*128 + n*128, 16B chunk swizzled
    for (int i = threadIdx.x; i < N * 16; i += 128) {
        const int n = i / 16, c16 = i % 16;  // 16 chunks of 8 bf16 per row
        const int h = c16 / 8, c = c16 % 8;
        const uint4 v = reinterpret_cast<const uint4*>(B + size_t(n) * 128)[c16];
        *reinterpret_cast<uint4*>(smem + h * N * 128 + n * 128 + ((c ^ (n & 7)) << 4)) = v;
    }
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
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
    // A rows into TMEM cols [128, 192) at lanes (r/16)*32 + off + r%16 (warp q4 = r/16)
    {
        const int q4 = warp, r16 = lane & 15, ch = lane >> 4, r = q4 * 16 + r16;
        uint32_t qr[32];
        const uint4* src = reinterpret_cast<const uint4*>(A + size_t(r) * 128) + ch * 8;
        for (int i = 0; i < 8; ++i) {
            const uint4 v = src[i];
            qr[4 * i] = v.x, qr[4 * i + 1] = v.y, qr[4 * i + 2] = v.z, qr[4 * i + 3] = v.w;
        }
        tmem_st16x2_32<32>(tmem + (uint32_t(q4 * 32 + off) << 16) + 128, qr);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        const uint32_t id = idesc_bf16(64, N, 0, 0);
        const uint32_t lo = uint32_t(off) << 16;
        if (elect_one()) {
            for (int ks = 0; ks < 8; ++ks)
                mma_ts(tmem + lo, tmem + lo + 128 + ks * 8,
                       sdesc_sw128(smem_u32(smem) + (ks >> 2) * N * 128 + (ks & 3) * 32, 16, 1024), id, ks != 0);
            mma_commit(bar);
        }
        __syncwarp();
    }
    mbar_wait(bar, 0);
    tc_fence_after();
    {
        const int q4 = warp, r16 = lane & 15, ch = lane >> 4, r = q4 * 16 + r16;
        for (int c0 = 0; c0 < N; c0 += 64) {
            uint32_t v[32];
            tmem_ld16x2_32<32>(tmem + (uint32_t(q4 * 32 + off) << 16) + c0, v);
            tmem_ld_wait(v);
            for (int i = 0; i < 32; ++i) out[r * N + c0 + ch * 32 + i] = __uint_as_float(v[i]);
        }
    }
    // timing: issue 2048 x 8 MMAs
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        const uint32_t id = idesc_bf16(64, N, 0, 0);
        const uint32_t lo = uint32_t(off) << 16;
        const long long t0 = clock64();
        for (int it = 0; it < 2048; ++it) {
            if (elect_one()) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    mma_ts(tmem + lo, tmem + lo + 128 + ks * 8,
                           sdesc_sw128(smem_u32(smem) + (ks >> 2) * N * 128 + (ks & 3) * 32, 16, 1024), id, 1);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(bar);
        __syncwarp();
        mbar_wait(bar, 1);
        const long long t1 = clock64();
        if (lane == 0 && blockIdx.x == 0) printf("M64 TS N%d lane-offset %d: %.1f cyc/instr\n", N, off, double(t1 - t0) / (2048 * 8));
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

template <int N>
void run(int off) {
    std::vector<__nv_bfloat16> a(64 * 128), b(N * 128);
    std::vector<float> af(64 * 128), bf(N * 128);
    srand(1 + off + N);
    for (int i = 0; i < 64 * 128; ++i) {
        a[i] = __float2bfloat16(float(rand() % 17 - 8) / 8.f);
        af[i] = __bfloat162float(a[i]);
    }
    for (int i = 0; i < N * 128; ++i) {
        b[i] = __float2bfloat16(float(rand() % 17 - 8) / 8.f);
        bf[i] = __bfloat162float(b[i]);
    }
    __nv_bfloat16 *da, *db;
    float* dout;
    cudaMalloc(&da, a.size() * 2);
    cudaMalloc(&db, b.size() * 2);
    cudaMalloc(&dout, 64 * N * 4);
    cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(m64<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
    m64<N><<<148, 128, 65536 + 2048>>>(da, db, dout, off);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> out(64 * N);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int r = 0; r < 64; ++r)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < 128; ++k) s += double(af[r * 128 + k]) * bf[n * 128 + k];
            maxerr = fmax(maxerr, fabs(s - out[r * N + n]));
        }
    printf("M64 N%d lane-offset %d: max |err| = %g (%s)\n", N, off, maxerr, cudaGetErrorString(e));
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    run<64>(0);
    run<64>(16);
    run<128>(0);
    run<128>(16);
    return 0;
}
