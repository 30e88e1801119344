// kernels.h -- launch interfaces of the four sm_100a kernels (host side).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pisa_b200 {

// K1: block statistics. One CTA per (chunk of kStatsG key blocks, batch*head).
//   k_bar / v_hat / q_bar fp32 [BH][N][D]   (compute_block_stats / query_block_means)
//   kbar_bf / vhat_bf bf16  [BH][Npad][D]   (operands of the fused kernel's Phase 2)
//   hpart fp32 [BH][nchunk][D][D]            (per-chunk sum_j H_j, reduced by K1b)
constexpr int kStatsG = 32;
struct StatsArgs {
    float* kbar;
    float* vhat;
    float* qbar;
    __nv_bfloat16* kbar_bf;
    __nv_bfloat16* vhat_bf;
    float* hpart;
    __nv_bfloat16* kbar_split;  // [3][BH][N][D] exact bf16 hi / mid / lo split of k_bar (fused K2's
                                // B operand), or null
    int BH;
    int L, N, Npad, H, nchunk;
    int G;  // key blocks per CTA (<= kStatsG)
};
cudaError_t launch_block_stats(int D, const CUtensorMap& tmQ, const CUtensorMap& tmK,
                               const CUtensorMap& tmV, const StatsArgs& a, int BH,
                               cudaStream_t s);

// K1b: H_bar = (1/N) sum_chunks hpart (fixed order), fp32 + bf16 copies, plus
// k_bar_global = mean_j k_bar_j.
cudaError_t launch_hbar_reduce(int D, const float* hpart, int nchunk, int N, const float* kbar,
                               float* hbar, __nv_bfloat16* hbar_bf, float* kbar_global, int BH,
                               cudaStream_t s);

// Conversion of externally supplied fp32 statistics into the fused kernel's
// bf16 operands (pisa_b200_attention path).
cudaError_t launch_stats_to_bf16(int D, const float* kbar, const float* vhat, const float* hbar,
                                 int N, int Npad, __nv_bfloat16* kbar_bf, __nv_bfloat16* vhat_bf,
                                 __nv_bfloat16* hbar_bf, float* kbar_global, int BH,
                                 cudaStream_t s);

// K1c: spectral deviation norms M_j = ||H_j - H_bar||_2 (covariance router).
struct NormArgs {
    const float* kbar;  // [BH][N][D]
    const float* hbar;  // [BH][D][D]
    float* m;           // [BH][N]
    float* rect;        // [BH][N] log(M_j + eps), or null
    double eps;
    int L, N, H;
    int64_t ks_b, ks_h, ks_l, vs_b, vs_h, vs_l;  // element strides of k / v
    float* tri;  // [BH][N][kTriStride] Lanczos tridiagonal per block (tensor-core kernel -> ritz kernel)
};
constexpr int kTriStride = 64;  // alpha [kLanczos] | beta [kLanczos - 1] | step count
// D = 128 reads K / V through the tensor maps (64-row boxes), D = 64 through k / v
cudaError_t launch_block_norms(int D, const CUtensorMap& tmK, const CUtensorMap& tmV, const __nv_bfloat16* k,
                               const __nv_bfloat16* v, const NormArgs& a, int BH, cudaStream_t s);
size_t block_norms_smem_bytes(int D);
int block_norms_launches(int D);  // kernels launch_block_norms launches (tensor-core path: K1c + ritz)

// K2: fp32 block scoring + top-k (score desc, index asc) per query block.
struct SelectArgs {
    const float* qbar;  // [BH][N][D]
    const float* kbar;  // [BH][N][D]
    const float* rect;  // [BH][N] covariance rectifier log(M_j + eps) added to scores, or null
    int32_t* selected;  // [BH][N][k]  (may be null)
    uint32_t* mask;     // [BH][N][W]
    int N, W, k, force_diagonal;
    float scale;
};
// rect[i] = log(m[i] + eps) (covariance rectifier from caller-supplied norms)
cudaError_t launch_rectifier(const float* m, double eps, float* rect, int n, cudaStream_t s);
// keys: scratch uint32 [BH][N][N]
cudaError_t launch_select(int D, const SelectArgs& a, int BH, uint32_t* keys, cudaStream_t s);

// K2 fused (N >= kSelectFusedMinN): one CTA per (128 query blocks, b*h) scores
// its rows against every key tile on tcgen05 (q_bar split into TMEM, k_bar
// splits from K1 by TMA), writes the order keys of its rows to an L2-resident
// scratch and selects each row's top-k right away. keys: scratch uint32
// [BH][N][N] (rows of the CTA only are touched); tmKs: 3-D map over
// kbar_split (D, N, 3*BH), 64 x 128 boxes, SW128.
constexpr int kSelectFusedMinN = 512;
constexpr int kScratchSlots = 256;  // scratch rows: kScratchSlots x 128 x N uint32 (one slot per SM id)
cudaError_t launch_select_fused(int D, const CUtensorMap& tmKs, const SelectArgs& a, int BH, uint32_t* keys,
                                cudaStream_t s);
// K2 streamed (N >= kSelectFusedMinN): the fused kernel's pipelined scoring
// writing the [BH][N][N] keys, then topk_kernel. keys: scratch uint32 [BH][N][N].
cudaError_t launch_select_stream(int D, const CUtensorMap& tmKs, const SelectArgs& a, int BH, uint32_t* keys,
                                 cudaStream_t s);

// K2c/K2d: overlap-aware pairing of query blocks for the fused kernel.
// cand: scratch int [BH][N][kPairCand]; pairs: int2 [BH][ceil(N/2)].
#ifndef PISA_PAIR_CAND
#define PISA_PAIR_CAND 16
#endif
constexpr int kPairCand = PISA_PAIR_CAND;  // candidate partners kept per query block
// ov: scratch u16 [BH][N][N] for the full-range candidate search (K2c over
// every block of the range, k2q_overlap.cu), or null: the +-kWindow search.
cudaError_t launch_pairing(const uint32_t* mask, int N, int W, int qb0, int qb1, int BH, int* cand, int2* pairs,
                           cudaStream_t s, uint16_t* ov = nullptr);
bool pairing_full_supported(int qb0, int qb1, int W);
cudaError_t launch_pairing_full_candidates(const uint32_t* mask, int N, int W, int qb0, int qb1, int BH,
                                           uint16_t* ov, int* cand, cudaStream_t s);

// Plan (ascending lists) -> bitmask, with SelectionPlan::validate semantics
// (router.hpp:50-70): sets *bad = 1 on out-of-range / non-ascending entries.
cudaError_t launch_plan_to_mask(const int32_t* selected, int N, int k, int W, uint32_t* mask,
                                int* bad, int BH, cudaStream_t s);

// K3: fused piecewise attention (Phase 1 exact over S_i, Phase 2 centroid tail,
// Phase 3 global first-order correction), one CTA (one SM) per pair of query blocks.
struct FusedArgs {
    const int2* pairs;         // [BH][ceil(N/2)] query blocks per tile (K2d), or null: (2t, 2t+1)
    const __nv_bfloat16* q;    // queries (GlobalCentroid slope reads rows directly)
    int64_t qs_b, qs_h, qs_l;  // element strides of q
    const uint32_t* mask;      // [BH][N][W]
    const float* kbar_global;  // [BH][D] (GlobalCentroid) or null
    void* out;
    int64_t os_b, os_h, os_l;
    float* diag_m;   // [BH][L] or null
    float* diag_l;
    float* diag_lt;
    int* nonfinite;  // device flag or null
    int L, N, H, W, nchunk2, variant, literal_phase3, out_f32, k;
    int qb0, qb1;  // query blocks [qb0, qb1) are computed (the rest of O is untouched)
    float scale;
    unsigned long long* trace;  // PISA_TRACE builds only: [8][1024] clock deltas
    unsigned long long* tile_count;  // instrumentation: += 64-key tiles processed (incl. padding), or null
    int trace_tile;
};
cudaError_t launch_fused(int D, const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                         const CUtensorMap& tmKb, const CUtensorMap& tmVh, const CUtensorMap& tmH,
                         const FusedArgs& a, int BH, cudaStream_t s);
size_t fused_smem_bytes(int D, int N, int W);

// Tensor-core self test (pisa_b200_selftest_mma).
cudaError_t launch_selftest_mma(const CUtensorMap& tmA, const CUtensorMap& tmB128,
                                const CUtensorMap& tmB64, const __nv_bfloat16* a, float* out,
                                cudaStream_t s);

}  // namespace pisa_b200
