/* pisa_b200.h -- C ABI of the B200-native PISA (Piecewise Sparse Attention) forward.
 *
 * The drop-in boundary for the reference's hot path (BASELINE.json north_star):
 *   pisa::pisa_multihead(bundle, r, RouterOptions{Plain}, PisaVariant::Hybrid, cfg,
 *                        use_streaming=true)          /root/reference/proj/include/pisa/engine.hpp:408-470
 * and its three steps (prepare / select / attention):
 *   compute_block_stats + compute_global_stats + query_block_means   block_stats.hpp:155-278
 *   sparsity_to_k + select_topk_plain                                router.hpp:80-151
 *   pisa_streaming (Algorithm 1) / pisa_reference (other variants)   engine.hpp:103-383
 *
 * Plain C types only: pointers, sizes, a POD descriptor. No exceptions cross this
 * boundary; every entry point returns a pisa_status whose values map 1:1 onto the
 * reference's typed errors (errors.hpp:22-94). The header-only C++ shim
 * include/pisa_b200.hpp rethrows them as the matching pisa:: classes.
 *
 * Device pointers are raw CUDA device addresses; `stream` is a cudaStream_t passed
 * as void* (NULL = legacy default stream). All launches are stream-ordered and
 * asynchronous unless a function says otherwise.
 */
#ifndef PISA_B200_H
#define PISA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PISA_B200_ABI_VERSION 3

/* Status codes. Reference class in brackets (errors.hpp line). */
typedef enum pisa_status {
    PISA_OK = 0,
    PISA_ERR_INVALID_DIMENSION = 1,  /* InvalidDimension   errors.hpp:22-28 */
    PISA_ERR_BLOCK_DIVISIBILITY = 2, /* BlockDivisibility  errors.hpp:36-39 (only when ragged=0) */
    PISA_ERR_INVALID_SPARSITY = 3,   /* InvalidSparsity    errors.hpp:41-44 */
    PISA_ERR_INVALID_EPSILON = 4,    /* InvalidEpsilon     errors.hpp:46-49 */
    PISA_ERR_EMPTY_SELECTION = 5,    /* EmptySelection     errors.hpp:51-54 */
    PISA_ERR_NUMERICAL_OVERFLOW = 6, /* NumericalOverflow  errors.hpp:91-94 (device non-finite flag) */
    PISA_ERR_DEGENERATE_SCALE = 7,   /* DegenerateScale    errors.hpp:31-34 */
    PISA_ERR_UNSUPPORTED = 8,        /* no reference class: variant / dtype / shape outside the GPU path */
    PISA_ERR_CUDA = 9                /* no reference class: CUDA runtime / driver failure */
} pisa_status;

/* Approximation order, numbered as pisa::PisaVariant (engine.hpp:30). */
typedef enum pisa_variant {
    PISA_SPARSE_ONLY = 0,
    PISA_ZEROTH = 1,
    PISA_BLOCK_FIRST = 2, /* not on the GPU path: PISA_ERR_UNSUPPORTED */
    PISA_HYBRID = 3,
    PISA_GLOBAL_CENTROID = 4
} pisa_variant;

/* Router strategy, numbered as pisa::RouterStrategy (router.hpp:16). */
typedef enum pisa_router { PISA_ROUTER_PLAIN = 0, PISA_ROUTER_COVARIANCE = 1 } pisa_router;

/* Element type of Q/K/V/O. The reference's T in {float, double} (bundle.hpp:15)
 * becomes bf16 on the GPU; O may also be written as fp32 (parity mode). */
typedef enum pisa_dtype {
    PISA_DTYPE_BF16 = 0,
    PISA_DTYPE_F32 = 1,
    PISA_DTYPE_F64 = 2 /* the generators' output only (TensorBundle<double>) */
} pisa_dtype;

/* Problem descriptor: the reference's TensorBundle shape (bundle.hpp:28-51) plus
 * AttentionConfig (attention.hpp:19-49) plus RouterOptions (engine.hpp:385-390)
 * plus the sparsity argument r of pisa_multihead (engine.hpp:409).
 *
 * Layout: element (b, h, s, c) of X lives at X + b*x_strides[0] + h*x_strides[1]
 * + s*x_strides[2] + c (strides in ELEMENTS, last dim contiguous). The reference
 * [H][L][d] bundle is strides {H*L*d, L*d, d}; DiT [B][L][H][d] is {L*H*d, d, H*d}.
 * Strides of q/k/v must be multiples of 8 elements (16-byte TMA rows). */
typedef struct pisa_attn_desc {
    int64_t batch;     /* B  (>= 1) */
    int64_t heads;     /* H  (>= 1) */
    int64_t seq_len;   /* L  (>= 1) */
    int64_t head_dim;  /* d  (64 or 128 on the GPU path) */
    int64_t q_strides[3], k_strides[3], v_strides[3], o_strides[3];
    int32_t block_size;     /* B_blk: 64 (the paper's tile); else UNSUPPORTED */
    int32_t group_size;     /* C: math-neutral Phase-2 group width, >= 1 (attention.hpp:21) */
    double scale;           /* 0 => 1/sqrt(d) (attention.hpp:34-37) */
    double sparsity;        /* r in [0,1): fraction of key blocks approximated (router.hpp:80) */
    int64_t topk;           /* > 0 overrides r with an explicit k in [1, N] */
    int32_t variant;        /* pisa_variant */
    int32_t router;         /* pisa_router (RouterOptions::strategy, engine.hpp:386) */
    int32_t force_diagonal; /* RouterOptions::force_diagonal (router.hpp:146-148) */
    int32_t literal_phase3; /* AttentionConfig::literal_phase3 (engine.hpp:345-346): Phase-3
                               weight / B. Honoured for HYBRID only (the streaming path's
                               diagnostic; pisa_reference ignores it, so callers mirroring
                               pisa_reference / use_streaming=false clear it) */
    int32_t ragged;         /* 1: allow L % 64 != 0 (documented extension); 0: BLOCK_DIVISIBILITY */
    int32_t out_dtype;      /* pisa_dtype of O */
    int32_t check_finite;   /* 1: report NUMERICAL_OVERFLOW on a non-finite output
                               (check_output_finite, engine.hpp:83-93): pisa_b200_fwd /
                               _qrange / _attention synchronize the stream to read the
                               device flag; pisa_b200_fwd_host reads it after its final
                               synchronisation (no extra sync) */
    int32_t row_level;      /* RouterOptions::row_level (engine.hpp:389): not on the GPU path
                               (UNSUPPORTED); must be 0 */
    double epsilon;         /* RouterOptions::epsilon (engine.hpp:387), default 1e-6; the
                               covariance router requires > 0 (INVALID_EPSILON) */
} pisa_attn_desc;

/* Optional per-row diagnostics (PisaOutput, engine.hpp:43-57), fp32, [batch][heads][seq_len].
 * The reference's denom = ell * exp(row_max), tail_mass = B * ell_tail * exp(row_max),
 * ell_tail(ref) = ell_tail * exp(row_max). Any pointer may be NULL. `selected`
 * receives the routing plan, int32 [batch][heads][N][k] ascending (SelectionPlan,
 * router.hpp:24-71). */
typedef struct pisa_diag {
    float* row_max;   /* natural-log shift actually used per row */
    float* ell;       /* denominator / exp(row_max) */
    float* ell_tail;  /* tail exponential sum / exp(row_max) */
    int32_t* selected;
} pisa_diag;

/* A context owns the device workspace. It may be used from several streams
 * (each stream gets its own workspace, so forwards enqueued on different streams
 * never share scratch), but not from several host threads concurrently.
 * Workspaces grow with the problem size and are only freed by
 * pisa_b200_destroy, so a CUDA graph captured from a call stays valid for the
 * lifetime of the context. */
typedef struct pisa_ctx pisa_ctx;

/* ---- lifetime ------------------------------------------------------------ */
pisa_status pisa_b200_create(pisa_ctx** ctx, int device);
void pisa_b200_destroy(pisa_ctx* ctx);
/* Human-readable message of the last failing call on this ctx ("ClassName: ..."). */
const char* pisa_b200_last_error(const pisa_ctx* ctx);
int pisa_b200_abi_version(void);

/* ---- helpers ------------------------------------------------------------- */
/* sparsity_to_k (router.hpp:80-90). */
pisa_status pisa_b200_sparsity_to_k(double r, int64_t num_blocks, int64_t* k, double* realized);
/* Resolved (N, k, scale) for a descriptor; validates it like pisa_multihead's
 * cfg.check + sparsity_to_k (engine.hpp:418-421). */
pisa_status pisa_b200_resolve(const pisa_attn_desc* desc, int64_t* num_blocks, int64_t* k,
                              double* scale);

/* ---- the hot path -------------------------------------------------------- */
/* Full forward: K1 block statistics [-> K1c spectral norms, covariance router]
 * -> K2 fp32 scoring + top-k -> K3 fused
 * piecewise attention, stream-ordered, no host synchronisation (unless
 * desc->check_finite). Replaces pisa_multihead(..., use_streaming=true). */
pisa_status pisa_b200_fwd(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* q,
                          const void* k, const void* v, void* o, const pisa_diag* diag,
                          void* stream);
/* Query-block pairing for the fused kernel (which query blocks share a CTA):
 * 0 = consecutive blocks, 1 = auto
 * (overlap-aware pairing when >= 768 query blocks are computed, the default),
 * 2 = always overlap-aware. Env PISA_B200_PAIRING sets the initial mode. The
 * plan does not depend on it; outputs agree to rounding (the grouping of a
 * block's key blocks into super-tiles moves its lazy-rescale points). */
pisa_status pisa_b200_set_pairing(pisa_ctx* ctx, int mode);

/* The forward restricted to query blocks [qb_begin, qb_end) of every (b, h):
 * the unit of (head x query-block range) sharding when heads do
 * not divide evenly over ranks. Statistics and routing use the full K / V
 * (pisa_multihead's per-head prepare, engine.hpp:437-441); output rows (and
 * diag rows) outside the range are not written. Every query block's result
 * equals the full call's to rounding (query blocks may be paired differently,
 * which moves the online softmax's lazy-rescale points; the plan is identical).
 * qb_end = -1 means N. A range outside
 * [0, N) -> PISA_ERR_INVALID_DIMENSION. */
pisa_status pisa_b200_fwd_qrange(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* q,
                                 const void* k, const void* v, void* o, int64_t qb_begin,
                                 int64_t qb_end, const pisa_diag* diag, void* stream);

/* Same, with Q/K/V/O in (ideally pinned) HOST memory: the ctx stages heads through
 * device buffers on its own streams, overlapping H2D copy, compute and D2H copy.
 * Host layout must be dense [batch][heads][seq_len][d] (the reference bundle).
 * `diag` (optional) holds HOST pointers with the pisa_diag layout.
 * Synchronous: returns when O (and diag) are in host memory. */
pisa_status pisa_b200_fwd_host(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* q,
                               const void* k, const void* v, void* o, const pisa_diag* diag);

/* ---- the three steps, for parity against the reference's step functions ---- */
/* Prepare (compute_block_stats + compute_global_stats(norms off) + query_block_means).
 * Outputs fp32, per (b,h): k_bar [N][d], v_hat [N][d], q_bar [N][d], h_bar [d][d].
 * Any output pointer may be NULL. */
pisa_status pisa_b200_block_stats(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* q,
                                  const void* k, const void* v, float* k_bar, float* v_hat,
                                  float* q_bar, float* h_bar, void* stream);

/* Select (select_topk_plain): fp32 scores scale*<q_bar_i, k_bar_j>, top-k by
 * (score desc, index asc), ascending output. Inputs fp32 [B*H][N][d];
 * selected int32 [B*H][N][k]; mask (optional) uint32 [B*H][N][ceil(N/32)].
 * desc->router must be PLAIN. */
pisa_status pisa_b200_select(pisa_ctx* ctx, const pisa_attn_desc* desc, const float* q_bar,
                             const float* k_bar, int32_t* selected, uint32_t* mask, void* stream);
/* Spectral deviation norms M_j = ||H_j - H_bar||_2 per key block
 * (compute_global_stats(.., compute_norms=true), block_stats.hpp:207-241), fp32
 * [B*H][N], computed from Q/K/V like pisa_b200_block_stats (Lanczos on
 * (H_j - H_bar)^T (H_j - H_bar); the reference uses an exact Jacobi solve). */
pisa_status pisa_b200_block_norms(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* q,
                                  const void* k, const void* v, float* m, void* stream);
/* Covariance-aware select (select_topk_covariance, router.hpp:157-193): scores
 * scale*<q_bar_i, k_bar_j> + log(M_j + desc->epsilon); m fp32 [B*H][N]. */
pisa_status pisa_b200_select_cov(pisa_ctx* ctx, const pisa_attn_desc* desc, const float* q_bar,
                                 const float* k_bar, const float* m, int32_t* selected,
                                 uint32_t* mask, void* stream);

/* Attention (pisa_streaming / pisa_reference) for a GIVEN plan and prepare
 * products (device, as produced above): selected int32 [B*H][N][k] ascending,
 * k_bar / v_hat fp32 [B*H][N][d], h_bar fp32 [B*H][d][d]. */
pisa_status pisa_b200_attention(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* q,
                                const void* k, const void* v, const int32_t* selected,
                                const float* k_bar, const float* v_hat, const float* h_bar,
                                void* o, const pisa_diag* diag, void* stream);

/* ---- the steps with HOST buffers (synchronous) ---------------------------- */
/* Same as the device entries above, for callers that keep tensors in host memory
 * like the reference (the C++ shim's compute_block_stats, query_block_means,
 * compute_global_stats(.., compute_norms), select_topk_plain / _covariance,
 * pisa_streaming, pisa_reference). Inputs bf16, dense [batch][heads][seq_len][d]
 * (desc strides are ignored); statistics fp32 as in the device entries. The ctx
 * stages through temporary device buffers and returns when the outputs are in
 * host memory. */
/* q may be NULL (then q_bar must be NULL): k_bar / v_hat / h_bar only. */
pisa_status pisa_b200_block_stats_host(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* q,
                                       const void* k, const void* v, float* k_bar, float* v_hat,
                                       float* q_bar, float* h_bar);
pisa_status pisa_b200_block_norms_host(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* k,
                                       const void* v, float* m);
/* m == NULL: select_topk_plain; else select_topk_covariance with desc->epsilon. */
pisa_status pisa_b200_select_host(pisa_ctx* ctx, const pisa_attn_desc* desc, const float* q_bar,
                                  const float* k_bar, const float* m, int32_t* selected);
/* diag: HOST pointers (row_max / ell / ell_tail; `selected` is ignored). */
pisa_status pisa_b200_attention_host(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* q,
                                     const void* k, const void* v, const int32_t* selected,
                                     const float* k_bar, const float* v_hat, const float* h_bar,
                                     void* o, const pisa_diag* diag);

/* ---- synthetic inputs: the reference's generators, bit-identical ---------- */
/* gen_gaussian (generate.hpp:29-49) and gen_clustered (generate.hpp:57-116) on
 * the reference RNG (xoshiro256++ seeded by splitmix64, Box-Muller pairs,
 * rng.hpp:10-72): q, k, v HOST arrays [heads][L][d] of dtype PISA_DTYPE_F32
 * (the reference's T = float), PISA_DTYPE_F64 (T = double) or PISA_DTYPE_BF16
 * (RNE rounding of the T = float value).
 * The single reference stream is split over `threads` host threads (<= 0: all)
 * by exact GF(2) jumps of the generator state, so the values do not depend on
 * the thread count. Errors: INVALID_DIMENSION / DEGENERATE_SCALE as the
 * reference throws them. */
pisa_status pisa_b200_gen_gaussian(uint64_t seed, int64_t heads, int64_t L, int64_t d, double std_dev,
                                   int32_t dtype, void* q, void* k, void* v, int threads);
pisa_status pisa_b200_gen_clustered(uint64_t seed, int64_t heads, int64_t L, int64_t d,
                                    int64_t n_clusters, double concentration, double noise_std,
                                    int32_t dtype, void* q, void* k, void* v, int threads);

/* ---- instrumentation ----------------------------------------------------- */
/* Number of kernel launches the last pisa_b200_fwd / _attention / _block_stats /
 * _select call issued (bench.py's gpu_launches). */
int64_t pisa_b200_last_launch_count(const pisa_ctx* ctx);
/* Name of kernel i of the fused forward (for profiles). NULL past the end. */
const char* pisa_b200_kernel_name(int i);
/* Per-kernel CUDA-event timing: while enabled, every launch is bracketed by a pair
 * of events recorded on the launching stream. read_profile synchronises on the
 * recorded events, writes the summed milliseconds and launch counts per kernel id
 * (ids as pisa_b200_kernel_name; arrays of length 8), and clears the record. */
pisa_status pisa_b200_set_profiling(pisa_ctx* ctx, int enable);
/* Debug timeline of one fused-kernel CTA (tile index `tile`, head 0): only
 * libraries built with -DPISA_TRACE=1 write it. dev_buf: 16*1024 u64 (device). */
pisa_status pisa_b200_debug_trace(pisa_ctx* ctx, unsigned long long* dev_buf, int tile);
pisa_status pisa_b200_read_profile(pisa_ctx* ctx, double* ms, int64_t* launches);
/* 64-key tiles (union blocks + centroid chunks, including pair padding) the
 * fused kernel processed while profiling was enabled, summed over launches;
 * synchronises and resets the counter. bench.py derives executed MMA FLOPs from it. */
pisa_status pisa_b200_fused_tiles(pisa_ctx* ctx, int64_t* tiles);

/* Standalone tensor-core self test: runs the tcgen05 operand modes the fused
 * kernel and K1 use (K-major SS, MN-major SS, TMEM-A TS, K-major A with MN-major
 * B) on small
 * tiles and writes the fp32 results for host comparison. a,b bf16 [128][128];
 * out fp32 [4][128][128]. */
pisa_status pisa_b200_selftest_mma(pisa_ctx* ctx, const void* a, const void* b, float* out,
                                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PISA_B200_H */
