// MUFU.EX2 throughput on B200 (and what the fused kernel's softmax sequence
// reaches per SM): is the Phase-1 softmax at a hardware bound?
//
//   mode 0  ex2.approx.ftz.f32 only, 32 independent chains per thread
//   mode 1  the softmax element sequence: FFMA (scale, -max) -> MUFU.EX2 ->
//           FADD (row sum) -> F2FP pack (every second element)
//   mode 2  mode 1 with the row max (FMNMX tree) of the 32 inputs first
//   mode 3  ex2.approx.ftz.bf16x2 (two exponentials per MUFU op)
//   mode 4  mode 1 with a 3-input max (fmax3) tree
// Prints exponentials per clock per SM for warps = 4, 8, 12, 16 per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_01077_b200/csrc mufu_rate.cu -o mufu_rate
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t ex2bf2(uint32_t x) {
    uint32_t y;
    asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

__global__ void mufu(int mode, int iters, float sl, unsigned long long* cyc, float* sink) {
    float s[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) s[i] = -0.01f * float((threadIdx.x + i) & 63);
    float l = 0.f, m = 0.f;
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) s[i] = ex2f(s[i]) - 1.0f;
        } else if (mode == 3) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                uint32_t x = pack(s[i], s[i + 1]);
                x = ex2bf2(x);
                acc ^= x;
                s[i] = __uint_as_float(x & 0xffff0000u) - 1.0f;
                s[i + 1] = __uint_as_float(x << 16) - 1.0f;
            }
        } else {
            float mm = m;
            if (mode == 2) {
                float a[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    a[j] = fmaxf(fmaxf(s[4 * j], s[4 * j + 1]), fmaxf(s[4 * j + 2], s[4 * j + 3]));
                mm = fmaxf(mm, fmaxf(fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3])), fmaxf(fmaxf(a[4], a[5]), fmaxf(a[6], a[7]))));
            } else if (mode == 4) {
                float a[11];
#pragma unroll
                for (int j = 0; j < 10; ++j) a[j] = fmax3(s[3 * j], s[3 * j + 1], s[3 * j + 2]);
                a[10] = fmaxf(s[30], s[31]);
                const float b0 = fmax3(a[0], a[1], a[2]), b1 = fmax3(a[3], a[4], a[5]), b2 = fmax3(a[6], a[7], a[8]);
                mm = fmax3(fmax3(b0, b1, b2), fmax3(a[9], a[10], mm), mm);
            }
            float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const float p0 = ex2f(fmaf(s[i], sl, -mm));
                const float p1 = ex2f(fmaf(s[i + 1], sl, -mm));
                ps[(i >> 1) & 3] += p0 + p1;
                acc ^= pack(p0, p1);
                s[i] = p0 - 0.5f;
                s[i + 1] = p1 - 0.5f;
            }
            l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
            m = mm * 0.5f;
        }
    }
    const long long t1 = clock64();
    float tot = l + float(acc & 1u);
#pragma unroll
    for (int i = 0; i < 32; ++i) tot += s[i];
    if (tot == 12345.f) sink[threadIdx.x] = tot;
    if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
}

int main(int argc, char** argv) {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 8);
    cudaMalloc(&sink, 4096 * 4);
    const char* names[] = {"ex2.f32 only", "softmax seq (ffma,ex2,fadd,pack)", "softmax seq + fmax tree",
                           "ex2.bf16x2 (2 exp / op)", "softmax seq + fmax3 tree"};
    for (int mode = 0; mode < 5; ++mode) {
        for (int warps : {4, 8, 12, 16}) {
            const int iters = 2000;
            mufu<<<148, warps * 32>>>(mode, 10, 1.4427f, d, sink);
            cudaMemset(d, 0, 8);
            mufu<<<148, warps * 32>>>(mode, iters, 1.4427f, d, sink);
            unsigned long long h = 0;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            const double cyc = double(h) / 148;  // cycles per SM (one timing thread per CTA)
            const double exps = double(iters) * 32 * warps * 32;
            printf("%-36s warps/SM %2d : %6.2f exp/clk/SM  (%s)\n", names[mode], warps, exps / cyc,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
