// Tensor-core self test: the exact operand modes the fused kernel and K1 use,
// on one 128x128 tile, so descriptor / layout mistakes show up as a clean
// numeric mismatch on the host instead of a wrong attention output.
//   out[0][m][n<64] = sum_c A[m][c] B[n][c]        S = Q K^T  (SS, both K-major)
//   out[1][a][c]    = sum_{r<64} A[r][a] B[r][c]   K^T V      (SS, both MN-major)
//   out[2][m][c]    = sum_{k<64} A[m][k] B[k][c]   P V        (TS: A from TMEM)
//   out[3][m][c]    = sum_{a<128} A[m][a] B[a][c]  Q H_bar    (SS, K-major A, MN-major B)
#include "kernels.h"
#include "sm100.cuh"

namespace pisa_b200 {
using namespace pisa_sm100;

namespace {

__global__ void __launch_bounds__(128, 1)
    selftest_kernel(const __grid_constant__ CUtensorMap tmA,
                    const __grid_constant__ CUtensorMap tmB128,
                    const __grid_constant__ CUtensorMap tmB64, const __nv_bfloat16* A,
                    float* out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* sQA = smem;              // A as a 128-row K-major tile, 2 halves x 16 KB
    uint8_t* sKB = smem + 32768;      // B rows 0..63, 2 halves x 8 KB
    uint8_t* sHB = smem + 49152;      // B rows 0..127, 2 halves x 16 KB
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 81920);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;

    if (threadIdx.x == 0) {
        mbar_expect_tx(&bars[0], 32768 + 16384 + 32768);
        for (int h = 0; h < 2; ++h) {
            tma_load_3d(sQA + h * 16384, &tmA, &bars[0], h * 64, 0, 0);
            tma_load_3d(sKB + h * 8192, &tmB64, &bars[0], h * 64, 0, 0);
            tma_load_3d(sHB + h * 16384, &tmB128, &bars[0], h * 64, 0, 0);
        }
    }
    // P = A[:, 0:64] as packed bf16 into TMEM columns 448..479
    {
        const int m = threadIdx.x;
        uint32_t pk[32];
        for (int i = 0; i < 32; ++i) {
            const float lo = __bfloat162float(A[m * 128 + 2 * i]);
            const float hi = __bfloat162float(A[m * 128 + 2 * i + 1]);
            pk[i] = pack_bf16(lo, hi);
        }
        tmem_st32(tmem + (uint32_t(warp * 32) << 16) + 448, pk);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    mbar_wait(&bars[0], 0);
    if (threadIdx.x == 0) {
        tc_fence_after();
        const uint32_t qa = smem_u32(sQA), kb = smem_u32(sKB), hb = smem_u32(sHB);
        // 1) S = A B[0:64]^T
        for (int ks = 0; ks < 8; ++ks) {
            const uint32_t hq = ks >> 2, kq = (ks & 3) * 32;
            mma_ss(tmem + 0, sdesc_sw128(qa + hq * 16384 + kq, 16, 1024),
                   sdesc_sw128(kb + hq * 8192 + kq, 16, 1024), idesc_bf16(128, 64, 0, 0), ks != 0);
        }
        // 2) A[0:64]^T B[0:64]  (A MN-major: its two 64-col chunks are the 16 KB halves)
        for (int ks = 0; ks < 4; ++ks)
            mma_ss(tmem + 64, sdesc_sw128(qa + ks * 2048, 16384, 1024),
                   sdesc_sw128(kb + ks * 2048, 8192, 1024), idesc_bf16(128, 128, 1, 1), ks != 0);
        // 3) P B[0:64]
        for (int ks = 0; ks < 4; ++ks)
            mma_ts(tmem + 192, tmem + 448 + ks * 8, sdesc_sw128(kb + ks * 2048, 8192, 1024),
                   idesc_bf16(128, 128, 0, 1), ks != 0);
        // 4) A B  (B MN-major with 128 K rows)
        for (int ks = 0; ks < 8; ++ks) {
            const uint32_t hq = ks >> 2, kq = (ks & 3) * 32;
            mma_ss(tmem + 320, sdesc_sw128(qa + hq * 16384 + kq, 16, 1024),
                   sdesc_sw128(hb + ks * 2048, 16384, 1024), idesc_bf16(128, 128, 0, 1), ks != 0);
        }
        mma_commit(&bars[1]);
    }
    __syncwarp();
    mbar_wait(&bars[1], 0);
    tc_fence_after();
    const int m = threadIdx.x;
    const int base_col[4] = {0, 64, 192, 320};
    const int ncols[4] = {64, 128, 128, 128};
    for (int tst = 0; tst < 4; ++tst) {
        for (int cc = 0; cc < ncols[tst]; cc += 32) {
            uint32_t r[32];
            tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + base_col[tst] + cc, r);
            tmem_ld_wait(r);
            for (int i = 0; i < 32; ++i) out[(tst * 128 + m) * 128 + cc + i] = __uint_as_float(r[i]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace

cudaError_t launch_selftest_mma(const CUtensorMap& tmA, const CUtensorMap& tmB128,
                                const CUtensorMap& tmB64, const __nv_bfloat16* a, float* out,
                                cudaStream_t s) {
    const int smem = 1024 + 81920 + 64;
    cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    selftest_kernel<<<1, 128, smem, s>>>(tmA, tmB128, tmB64, a, out);
    return cudaGetLastError();
}

}  // namespace pisa_b200
