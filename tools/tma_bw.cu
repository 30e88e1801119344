// Microbenchmark: TMA gather bandwidth/latency of random 64-row x 128-col bf16
// blocks (the fused kernel's K/V access) from an L2-resident buffer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_01077_b200/csrc tma_bw.cu -o tma_bw
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "sm100.cuh"

using namespace pisa_sm100;

__global__ void __launch_bounds__(128) gather(const __grid_constant__ CUtensorMap tm, int nblocks,
                                             int stages, int iters, unsigned long long* lat) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int w = threadIdx.x >> 5;  // one issuing thread per warp, its own ring
    uint8_t* smem = smem0 + w * (stages * 16384 + 1024);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * 16384);
    if ((threadIdx.x & 31) == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    // whole-warp loop, elected lane issues (warp-uniform values)
    uint32_t h = (blockIdx.x * 4 + w) * 2654435761u + 12345u;
    long long tsum = 0;
    long long t_issue[16];
    for (int i = 0; i < iters; ++i) {
        const int s = i % stages;
        if (i >= stages) {
            mbar_wait(&full[s], ((i / stages) - 1) & 1);
            tsum += clock64() - t_issue[s];
        }
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
    for (int i = iters; i < iters + stages; ++i) {
        const int s = i % stages;
        if (i >= stages) mbar_wait(&full[s], ((i / stages) - 1) & 1);
    }
    if (lat && (threadIdx.x & 31) == 0) atomicAdd(lat, (unsigned long long)(tsum / (iters - stages)));
}

// one warp, lanes 0..nl-1 each drive their own ring (divergent lanes issue TMA)
__global__ void __launch_bounds__(32) gather_lanes(const __grid_constant__ CUtensorMap tm, int nblocks,
                                                   int stages, int iters, int nl) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int l = threadIdx.x;
    if (l >= nl) return;
    uint8_t* smem = smem0 + l * (stages * 16384 + 1024);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * 16384);
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    uint32_t h = (blockIdx.x * 32 + l) * 2654435761u + 12345u;
    for (int i = 0; i < iters + stages; ++i) {
        const int s = i % stages;
        if (i >= stages) mbar_wait(&full[s], ((i / stages) - 1) & 1);
        if (i >= iters) continue;
        h = h * 1664525u + 1013904223u;
        const int blk = int((h >> 8) % uint32_t(nblocks));
        mbar_expect_tx(&full[s], 16384);
        tma_load_3d(smem + s * 16384, &tm, &full[s], 0, blk * 64, 0);
        tma_load_3d(smem + s * 16384 + 8192, &tm, &full[s], 64, blk * 64, 0);
    }
}

__global__ void __launch_bounds__(512) gather_sweep(const __grid_constant__ CUtensorMap tm, int nblocks,
                                                   int stages, int iters, int nl, unsigned long long* lat) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l >= nl) return;
    const int id = w * nl + l;
    uint8_t* smem = smem0 + id * (stages * 16384);
    __shared__ uint64_t fulls[64 * 4];
    uint64_t* full = fulls + id * 4;
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    uint32_t h = (blockIdx.x * 64 + id) * 2654435761u + 12345u;
    long long tsum = 0, t_issue[4] = {0, 0, 0, 0};
    for (int i = 0; i < iters + stages; ++i) {
        const int s = i % stages;
        if (i >= stages) {
            mbar_wait(&full[s], ((i / stages) - 1) & 1);
            tsum += clock64() - t_issue[s];
        }
        if (i >= iters) continue;
        h = h * 1664525u + 1013904223u;
        const int blk = int((h >> 8) % uint32_t(nblocks));
        mbar_expect_tx(&full[s], 16384);
        t_issue[s] = clock64();
        tma_load_3d(smem + s * 16384, &tm, &full[s], 0, blk * 64, 0);
        tma_load_3d(smem + s * 16384 + 8192, &tm, &full[s], 64, blk * 64, 0);
    }
    if (lat) atomicAdd(lat, (unsigned long long)(tsum / iters));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const size_t mb = argc > 1 ? atoi(argv[1]) : 40;  // buffer MB (L2-resident if < ~100)
    const size_t rows = mb * 1024 * 1024 / 256;
    void* buf;
    cudaMalloc(&buf, rows * 256);
    cudaMemset(buf, 0, rows * 256);
    void* p;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)p;
    CUtensorMap tm;
    cuuint64_t dims[3] = {128, rows, 1}, strides[2] = {256, rows * 256};
    cuuint32_t box[3] = {64, 64, 1}, es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    unsigned long long* lat;
    cudaMalloc(&lat, 8);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("buffer %zu MB\n", mb);
    if (argc > 2 && atoi(argv[2]) == 0) {  // sweep: warps x lanes x stages, 1 CTA/SM
        for (int nw : {1, 2, 4, 8}) for (int nl : {1, 2}) for (int stages : {2, 3, 4}) {
            const int streams = nw * nl;
            const int smem = streams * stages * 16384 + 1024;
            if (smem > 200 * 1024) continue;
            const int iters = 1000;
            cudaFuncSetAttribute(gather_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            gather_sweep<<<148, 32 * nw, smem>>>(tm, int(rows / 64), stages, 100, nl, nullptr);
            cudaMemset(lat, 0, 8);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            gather_sweep<<<148, 32 * nw, smem>>>(tm, int(rows / 64), stages, iters, nl, lat);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            unsigned long long lt;
            cudaMemcpy(&lt, lat, 8, cudaMemcpyDeviceToHost);
            printf("warps %d lanes %d stages %d (in flight %3d KB/SM): %.2f TB/s, latency %llu (%s)\n", nw, nl,
                   stages, streams * stages * 16, double(148) * streams * iters * 16384 / (ms * 1e-3) / 1e12,
                   lt / (148 * streams), cudaGetErrorString(cudaGetLastError()));
        }
        return 0;
    }
    // lanes-per-warp mode: argv[2] = number of issuing lanes in the one warp (each its own ring)
    if (argc > 2) {
        const int nl = atoi(argv[2]);
        for (int stages : {1, 2}) {
            const int iters = 2000;
            const int smem = nl * (stages * 16384 + 1024) + 1024;
            cudaFuncSetAttribute(gather_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            gather_lanes<<<148, 32, smem>>>(tm, int(rows / 64), stages, 200, nl);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            gather_lanes<<<148, 32, smem>>>(tm, int(rows / 64), stages, iters, nl);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("1 warp, %d issuing lanes, stages %d: %.2f TB/s (%s)\n", nl, stages,
                   double(148) * nl * iters * 16384 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        }
        return 0;
    }
    for (int wpc : {1, 2, 4}) for (int cps : {1, 2}) {
        for (int stages : {1, 2, 3}) {
            const int iters = 2000;
            const int smem = wpc * (stages * 16384 + 1024) + 1024;
            if (smem * cps > 220 * 1024) continue;
            cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            const int grid = 148 * cps;
            gather<<<grid, 32 * wpc, smem>>>(tm, int(rows / 64), stages, 200, nullptr);
            cudaMemset(lat, 0, 8);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            gather<<<grid, 32 * wpc, smem>>>(tm, int(rows / 64), stages, iters, lat);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            unsigned long long l;
            cudaMemcpy(&l, lat, 8, cudaMemcpyDeviceToHost);
            const double bytes = double(grid) * wpc * iters * 16384;
            printf("issuers/CTA %d ctas/SM %d stages %d: %.2f TB/s, latency %llu cycles (%s)\n", wpc, cps,
                   stages, bytes / (ms * 1e-3) / 1e12, l / (grid * wpc), cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
