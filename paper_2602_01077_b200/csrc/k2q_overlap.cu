// K2c (full search): candidate partners of every query block among ALL query
// blocks of its range, for the pairing of K2d (k2p_pairing.cu).
//
// The windowed K2c scores the +-48 blocks around i; a search over the whole
// range finds better partners on independent routing (tools/sim_pairing.py on
// a real Wan2.1-14B plan: union/k 1.776 -> 1.737, profiles/r02n_pairing_sim.log)
// provided candidates of equal overlap are taken nearest-first (index-order
// ties crowd every block onto the same popular partners on clustered routing).
// Its cost is the N x N overlap matrix o(i, j) = |S_i & S_j| per head, a 0/1
// matrix product -- here on the tensor cores with int8 mma.sync (m16n8k32):
//   overlap_kernel: one CTA per upper-triangular 128 x 128 tile of (i, j)
//     block pairs; the tile's 2 x 128 bitmask rows are staged in shared memory;
//     each warp expands 32-bit mask words into 0/1 bytes in its fragments
//     ((nibble * 0x00204081) & 0x01010101) and accumulates a 64 x 64 block in
//     s32 registers; the block and its mirror are stored as u16.
//   overlap_tc_kernel (default; PISA_OVERLAP_TC=0: overlap_kernel, int8
//     mma.sync): the same tiles on tcgen05 kind::i8, bit-identical results;
//   cand_full_kernel: warp per query block i; key(j) = o(i, j) << 14 |
//     (4095 - |i - j|) << 1 | (j < i), unique per j; every lane keeps its four
//     largest keys and the kCand largest of the warp are popped in order (the
//     same contract as the windowed kernel's lists: best first, -1 padded).
// Default up to 2048 blocks per range (PISA_B200_PAIR_FULL=0: the window):
// 0.29 ms at Wan2.1-14B (overlap 123 us, candidates 92 us, matching 30 us)
// against the window's 0.25 ms, for 2.2 % fewer union tiles on gaussian
// routing: -0.3 ms a step (pisa_b200.cu:pair_full_on).
#include "kernels.h"
#include "sm100.cuh"

namespace pisa_b200 {
using namespace pisa_sm100;
namespace {

constexpr int kCand = kPairCand;
#ifndef PISA_OVERLAP_TC
#define PISA_OVERLAP_TC 1  // overlap matrix on tcgen05 kind::i8 (0: int8 mma.sync)
#endif
constexpr int kOvTile = 128;
constexpr int kOvThreads = 128;  // 4 warps, 2 x 2 blocks of 64 x 64

__device__ __forceinline__ uint32_t expand_nibble(uint32_t word, int shift) {
    return (((word >> shift) & 0xFu) * 0x00204081u) & 0x01010101u;
}

__device__ __forceinline__ void imma_16832(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// tile (ti, tj), tj >= ti, of the range [qb0, qb1); ov: u16 [BH][N][N]
__global__ void __launch_bounds__(kOvThreads) overlap_kernel(const uint32_t* __restrict__ mask, int N, int W,
                                                             int qb0, int qb1, uint16_t* __restrict__ ov) {
    extern __shared__ uint32_t sm[];  // A rows [128][W + 1], B rows [128][W + 1]
    const int nt = (qb1 - qb0 + kOvTile - 1) / kOvTile;
    // blockIdx.x enumerates the upper triangle row by row
    int t = blockIdx.x, ti = 0;
    while (t >= nt - ti) {
        t -= nt - ti;
        ++ti;
    }
    const int tj = ti + t;
    const int bh = blockIdx.y;
    const int i0 = qb0 + ti * kOvTile, j0 = qb0 + tj * kOvTile;
    const int WS = W + 1;  // padded row stride: conflict-free column reads
    uint32_t* As = sm;
    uint32_t* Bs = sm + kOvTile * WS;
    const uint32_t* M = mask + size_t(bh) * N * W;
    for (int e = threadIdx.x; e < kOvTile * W; e += kOvThreads) {
        const int r = e / W, w = e % W;
        As[r * WS + w] = i0 + r < qb1 ? __ldg(M + size_t(i0 + r) * W + w) : 0u;
        Bs[r * WS + w] = j0 + r < qb1 ? __ldg(M + size_t(j0 + r) * W + w) : 0u;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tq = lane & 3;
    const int wi = (warp >> 1) * 64, wj = (warp & 1) * 64;  // this warp's 64 x 64 block
    int acc[4][8][4];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 8; ++n)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[m][n][c] = 0;
    for (int w = 0; w < W; ++w) {
        // K = the 32 key blocks of mask word w; A rows wi + 16m + g (+8),
        // columns tq*4.. (regs 0/1) and 16 + tq*4.. (regs 2/3)
        uint32_t a[4][4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const uint32_t lo = As[(wi + 16 * m + g) * WS + w], hi = As[(wi + 16 * m + g + 8) * WS + w];
            a[m][0] = expand_nibble(lo, tq * 4);
            a[m][1] = expand_nibble(hi, tq * 4);
            a[m][2] = expand_nibble(lo, 16 + tq * 4);
            a[m][3] = expand_nibble(hi, 16 + tq * 4);
        }
#pragma unroll
        for (int n = 0; n < 8; ++n) {
            const uint32_t bw = Bs[(wj + 8 * n + g) * WS + w];
            const uint32_t b0 = expand_nibble(bw, tq * 4), b1 = expand_nibble(bw, 16 + tq * 4);
#pragma unroll
            for (int m = 0; m < 4; ++m) imma_16832(acc[m][n], a[m], b0, b1);
        }
    }
    // C fragment: c0 / c1 row g, columns 2tq / 2tq + 1; c2 / c3 row g + 8
    uint16_t* O = ov + size_t(bh) * N * N;
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 8; ++n)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int i = i0 + wi + 16 * m + g + (c >> 1) * 8, j = j0 + wj + 8 * n + 2 * tq + (c & 1);
                if (i < qb1 && j < qb1) {
                    O[size_t(i) * N + j] = uint16_t(acc[m][n][c]);
                    if (ti != tj) O[size_t(j) * N + i] = uint16_t(acc[m][n][c]);
                }
            }
}

// The same tiles on tcgen05 (kind::i8, u8 x u8 -> s32 in TMEM): per chunk of
// 4 mask words (128 key blocks) every thread expands its row of A and of B
// into 128 0/1 bytes, 128B-swizzled K-major like the TMA image, double
// buffered against the 4 MMAs (K = 32 each) of the previous chunk; the
// accumulator row (thread = row i) leaves as 16-byte stores, its mirror as
// 64-byte column runs (lanes = consecutive i).
__host__ __device__ constexpr uint32_t idesc_u8(int M, int N) {
    return (2u << 4)                   // D format s32
           | (0u << 7) | (0u << 10)    // A, B unsigned 8-bit, K-major
           | (uint32_t(N >> 3) << 17)  // N / 8
           | (uint32_t(M >> 4) << 24);  // M / 16
}

__device__ __forceinline__ void mma_u8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum));
}

constexpr int kOvChunk = 128 * 128;  // one operand chunk: 128 rows x 128 K-bytes
constexpr int kOvTcThreads = 256;    // thread t expands row t % 128 of A (t < 128) or B

__global__ void __launch_bounds__(kOvTcThreads, 3) overlap_tc_kernel(const uint32_t* __restrict__ mask, int N, int W,
                                                                  int qb0, int qb1, uint16_t* __restrict__ ov) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    // [2 buffers][A | B] chunks, then the barriers
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 4 * kOvChunk);  // [2] chunk consumed by its MMAs
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
    const int nt = (qb1 - qb0 + kOvTile - 1) / kOvTile;
    int t = blockIdx.x, ti = 0;
    while (t >= nt - ti) {
        t -= nt - ti;
        ++ti;
    }
    const int tj = ti + t;
    const int bh = blockIdx.y;
    const int i0 = qb0 + ti * kOvTile, j0 = qb0 + tj * kOvTile;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int op = tid >> 7, r = tid & 127;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tslot, 128);
        tmem_relinquish();
    }
    // this thread's mask row (straight from L2: the mask is a few MB)
    const int row = (op ? j0 : i0) + r;
    const uint32_t* src = row < qb1 ? mask + (size_t(bh) * N + row) * W : nullptr;
    const int nchunk = (W + 3) / 4;
    uint32_t wd[4], nx[4];  // this chunk's and the next chunk's words; two more chunks in flight
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        wd[q] = (src && q < W) ? __ldg(src + q) : 0u;
        nx[q] = (src && 4 + q < W) ? __ldg(src + 4 + q) : 0u;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    constexpr uint32_t idesc = idesc_u8(128, 128);
    for (int c = 0; c < nchunk; ++c) {
        const int buf = c & 1;
        uint32_t nn[4];  // chunk c + 2's words
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int w = (c + 2) * 4 + q;
            nn[q] = (src && w < W) ? __ldg(src + w) : 0u;
        }
        if (c >= 2) mbar_wait(&bar[buf], ((c >> 1) - 1) & 1);  // the MMAs of chunk c - 2 are done with it
        uint8_t* dst = smem + buf * 2 * kOvChunk + op * kOvChunk + r * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // 16-byte chunk 2q + h: bits 16h .. 16h + 15 of word q
                uint4 v;
                v.x = expand_nibble(wd[q], 16 * h);
                v.y = expand_nibble(wd[q], 16 * h + 4);
                v.z = expand_nibble(wd[q], 16 * h + 8);
                v.w = expand_nibble(wd[q], 16 * h + 12);
                *reinterpret_cast<uint4*>(dst + (((2 * q + h) ^ (r & 7)) << 4)) = v;
            }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            wd[q] = nx[q];
            nx[q] = nn[q];
        }
        fence_proxy_async();
        tc_fence_before();
        __syncthreads();
        if (warp == 0) {
            tc_fence_after();
            if (elect_one()) {
                const uint32_t a = smem_u32(smem + buf * 2 * kOvChunk), b = a + kOvChunk;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    mma_u8_ss(tmem, sdesc_sw128(a + ks * 32, 16, 1024), sdesc_sw128(b + ks * 32, 16, 1024), idesc,
                              (c | ks) != 0);
                mma_commit(&bar[buf]);
            }
            __syncwarp();
        }
    }
    const int cl = nchunk - 1;
    mbar_wait(&bar[cl & 1], (cl >> 1) & 1);
    tc_fence_after();
    // warps w and w + 4 share TMEM lane quadrant w % 4 and take column halves.
    // O[j][i] (the mirror) leaves straight from the registers: lanes hold
    // consecutive i, so each store is a 64-byte run. O[i][j] is transposed
    // through shared memory (the chunk buffers are free now) so that a warp
    // writes a whole 256-byte row segment at a time; the row-per-thread TMEM
    // layout would scatter every store over 32 rows.
    uint16_t* O = ov + size_t(bh) * N * N;
    constexpr int kSt = 136;  // staging row stride in u16 (16-byte aligned, 4-bank skew per row)
    uint16_t* stage = reinterpret_cast<uint16_t*>(smem);
    const int il = (warp & 3) * 32 + (tid & 31);
    const int i = i0 + il;
#pragma unroll 1
    for (int cc = (warp >> 2) * 64; cc < (warp >> 2) * 64 + 64; cc += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + (uint32_t((warp & 3) * 32) << 16) + cc, v);
        tmem_ld_wait(v);
        const int jb = j0 + cc;
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
            uint4 p4;
            p4.x = v[e] | (v[e + 1] << 16);
            p4.y = v[e + 2] | (v[e + 3] << 16);
            p4.z = v[e + 4] | (v[e + 5] << 16);
            p4.w = v[e + 6] | (v[e + 7] << 16);
            *reinterpret_cast<uint4*>(stage + il * kSt + cc + e) = p4;
        }
        if (ti != tj && i < qb1) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
                if (jb + e < qb1) O[size_t(jb + e) * N + i] = uint16_t(v[e]);
        }
    }
    __syncthreads();
    // O[i][j]: warp w writes rows w, w + 8, ...; lane l columns 4l .. 4l + 3
    {
        const int lane = tid & 31;
        const int jc = j0 + 4 * lane;
        for (int rl = warp; rl < kOvTile; rl += kOvTcThreads / 32) {
            const int ir = i0 + rl;
            if (ir >= qb1) break;
            const uint2 q2 = *reinterpret_cast<const uint2*>(stage + rl * kSt + 4 * lane);
            uint16_t* dst = O + size_t(ir) * N + jc;
            if (jc + 4 <= qb1 && ((reinterpret_cast<uintptr_t>(dst) & 3u) == 0)) {  // 4-byte aligned pairs
                // (an odd N, or an odd first block qb0 of a query range, shifts the pairs)
                reinterpret_cast<uint32_t*>(dst)[0] = q2.x;
                reinterpret_cast<uint32_t*>(dst)[1] = q2.y;
            } else {
                const uint16_t e4[4] = {uint16_t(q2.x), uint16_t(q2.x >> 16), uint16_t(q2.y), uint16_t(q2.y >> 16)};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (jc + e < qb1) dst[e] = e4[e];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 128);
}

// warp per query block i of [qb0, qb1): the kCand best partners
template <int kPer>
__global__ void __launch_bounds__(256) cand_full_kernel(const uint16_t* __restrict__ ov, int N, int qb0, int qb1,
                                                        int* __restrict__ cand) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bh = blockIdx.y;
    const int i = qb0 + blockIdx.x * 8 + warp;
    if (i >= qb1) return;
    const uint16_t* row = ov + (size_t(bh) * N + i) * N;
    auto make_key = [&](int j, uint32_t o) -> uint32_t {
        if (j >= qb1 || j == i) return 0u;
        const int dist = j > i ? j - i : i - j;
        return (o << 14) | (uint32_t(4095 - dist) << 1) | uint32_t(j < i) | 0x40000000u;
    };
    uint32_t key[kPer];
    if (((reinterpret_cast<uintptr_t>(row + qb0)) & 3u) == 0) {
        // pairs of overlaps per 4-byte load (lane l: j = qb0 + 64 t + 2 l, + 1);
        // which lane holds which key does not change the kCand largest
        const uint32_t* row2 = reinterpret_cast<const uint32_t*>(row + qb0);
#pragma unroll
        for (int t = 0; t < kPer / 2; ++t) {
            const int j = qb0 + 64 * t + 2 * lane;
            const uint32_t w = j < qb1 ? row2[32 * t + lane] : 0u;  // (j + 1 < N: the row holds it)
            key[2 * t] = make_key(j, w & 0xffffu);
            key[2 * t + 1] = make_key(j + 1, w >> 16);
        }
    } else {
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
            const int j = qb0 + t * 32 + lane;
            key[t] = j < qb1 ? make_key(j, row[j]) : 0u;
        }
    }
    // this lane's four largest keys, descending (a min / max insertion network)
    uint32_t c0 = 0u, c1 = 0u, c2 = 0u, c3 = 0u;
    auto insert = [&](uint32_t x) {
        uint32_t y = max(c0, x);
        x = min(c0, x);
        c0 = y;
        y = max(c1, x);
        x = min(c1, x);
        c1 = y;
        y = max(c2, x);
        x = min(c2, x);
        c2 = y;
        c3 = max(c3, x);
    };
#pragma unroll
    for (int t = 0; t < kPer; ++t) insert(key[t]);
    int taken = 0;  // keys this lane gave up from its list
    for (int c = 0; c < kCand; ++c) {
        const uint32_t top = __reduce_max_sync(0xffffffffu, c0);
        int jj = -1;
        if (top != 0u) {
            // recover j from (distance, side): unique per key
            const int dist = 4095 - int((top >> 1) & 4095u);
            jj = (top & 1u) ? i - dist : i + dist;
            if (c0 == top) {  // the one lane holding it
                c0 = c1;
                c1 = c2;
                c2 = c3;
                c3 = 0u;
                if (++taken == 4) {  // list used up: the next four below the last one taken
                    taken = 0;
#pragma unroll
                    for (int t = 0; t < kPer; ++t) insert(key[t] < top ? key[t] : 0u);
                }
            }
        }
        if (lane == 0) cand[(size_t(bh) * N + i) * kCand + c] = jj;
    }
}

}  // namespace

bool pairing_full_supported(int qb0, int qb1, int W) { return qb1 - qb0 <= 2048 && W <= 64; }

cudaError_t launch_pairing_full_candidates(const uint32_t* mask, int N, int W, int qb0, int qb1, int BH,
                                           uint16_t* ov, int* cand, cudaStream_t s) {
    const int nt = (qb1 - qb0 + kOvTile - 1) / kOvTile;
    if (PISA_OVERLAP_TC) {
        const size_t sm = 1024 + size_t(4) * kOvChunk + 64;
        cudaFuncSetAttribute(overlap_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        overlap_tc_kernel<<<dim3(nt * (nt + 1) / 2, BH), kOvTcThreads, sm, s>>>(mask, N, W, qb0, qb1, ov);
    } else {
        const size_t sm = size_t(2) * kOvTile * (W + 1) * 4;
        cudaFuncSetAttribute(overlap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        overlap_kernel<<<dim3(nt * (nt + 1) / 2, BH), kOvThreads, sm, s>>>(mask, N, W, qb0, qb1, ov);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const dim3 grid((qb1 - qb0 + 7) / 8, BH);
    const int per = (qb1 - qb0 + 31) / 32;
    if (per <= 16)
        cand_full_kernel<16><<<grid, 256, 0, s>>>(ov, N, qb0, qb1, cand);
    else if (per <= 40)
        cand_full_kernel<40><<<grid, 256, 0, s>>>(ov, N, qb0, qb1, cand);
    else
        cand_full_kernel<64><<<grid, 256, 0, s>>>(ov, N, qb0, qb1, cand);
    return cudaGetLastError();
}

}  // namespace pisa_b200
