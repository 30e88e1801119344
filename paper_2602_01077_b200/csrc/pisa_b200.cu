// pisa_b200.cu -- the C ABI (include/pisa_b200.h): validation with the
// reference's error semantics, workspace management, TMA descriptor creation,
// and the stream-ordered K1 -> K1b -> K2 -> K3 launch sequence.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/pisa_b200.h"
#include "kernels.h"

using namespace pisa_b200;

struct pisa_ctx {
    int device = 0;
    int sms = 148;  // multiprocessor count (K1 chunk sizing)
    std::string last_error;
    // Device workspace, one grow-only arena per stream that has called into
    // this ctx, so forwards enqueued on different streams never share scratch.
    // A superseded arena is retired, not freed, until pisa_b200_destroy: a CUDA
    // graph captured from an earlier call keeps pointing at it.
    struct Arena {
        cudaStream_t stream = nullptr;
        void* base = nullptr;
        size_t bytes = 0;
        int* flags = nullptr;  // [0] non-finite output, [1] invalid plan (never reallocated)
    };
    std::vector<Arena> arenas;
    std::vector<void*> retired;
    int* flag_host = nullptr;  // pinned mirror of a device flag
    int64_t launches = 0;
    // host-staged path
    cudaStream_t st_h2d = nullptr, st_comp = nullptr, st_d2h = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {};
    void* stage = nullptr;
    size_t stage_bytes = 0;
    // per-kernel event timing
    bool prof = false;
    struct Rec {
        int id;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    unsigned long long* trace = nullptr;  // debug timeline (PISA_TRACE builds)
    int trace_tile = 0;
    // overlap-aware query-block pairing: 0 off, 1 auto (only when the range has
    // >= kPairMinBlocks query blocks: below that its fixed cost exceeds the union
    // it saves -- measured: FLUX N=72 +25 us for -2 us, Wan2.1-1.3B N=512 +66 us
    // for -50 us, Wan2.1-14B N=1182 +0.32 ms for -0.84 ms), 2 always.
    // env PISA_B200_PAIRING, API pisa_b200_set_pairing
    int pairing = 1;
    int host_chunks = 16;  // head chunks of the host path's copy/compute pipeline (env PISA_B200_HOST_CHUNKS)
    // K1b (H_bar reduce) runs on a side stream beside the select: ev_k1 forks
    // it after K1, ev_k1b joins it back before K1c / K3
    cudaStream_t side = nullptr;
    cudaEvent_t ev_k1 = nullptr, ev_k1b = nullptr;
    unsigned long long* tiles_dev = nullptr;  // fused-kernel tile counter (profiling only)
};

namespace {

const char* kKernelNames[] = {"block_stats_kernel", "hbar_reduce_kernel", "select_kernels",
                              "fused_attn_kernel",  "plan_to_mask_kernel", "stats_to_bf16_kernel",
                              "block_norms_kernel", "pairing_kernels",    nullptr};
enum KernelId { kK1 = 0, kK1b = 1, kK2 = 2, kK3 = 3, kPlan = 4, kToBf16 = 5, kK1c = 6, kPair = 7 };

cudaEvent_t pooled_event(pisa_ctx* c) {
    if (!c->pool.empty()) {
        cudaEvent_t e = c->pool.back();
        c->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Brackets one launch with events on its stream when profiling is on.
struct ProfScope {
    pisa_ctx* c;
    int id;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    ProfScope(pisa_ctx* c_, int id_, cudaStream_t s_) : c(c_), id(id_), s(s_) {
        if (c->prof) {
            a = pooled_event(c);
            cudaEventRecord(a, s);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEvent_t b = pooled_event(c);
            cudaEventRecord(b, s);
            c->recs.push_back({id, a, b});
        }
    }
};

pisa_status fail(pisa_ctx* ctx, pisa_status st, const std::string& msg) {
    if (ctx) {
        static const char* cls[] = {"Ok",           "InvalidDimension", "BlockDivisibility",
                                    "InvalidSparsity", "InvalidEpsilon", "EmptySelection",
                                    "NumericalOverflow", "DegenerateScale", "Unsupported",
                                    "CudaError"};
        ctx->last_error = std::string(cls[int(st)]) + ": " + msg;
    }
    return st;
}

pisa_status cuda_fail(pisa_ctx* ctx, cudaError_t e, const char* where) {
    return fail(ctx, PISA_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------ TMA maps --
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// bf16 tensor, 128B swizzle, zero OOB fill. dims/strides innermost first;
// strides_bytes has rank-1 entries.
bool make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
              const uint64_t* strides_bytes, const uint32_t* box) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t gd[5], gs[4];
    cuuint32_t bx[5], es[5];
    for (int i = 0; i < rank; ++i) {
        gd[i] = dims[i];
        bx[i] = box[i];
        es[i] = 1;
    }
    for (int i = 0; i < rank - 1; ++i) gs[i] = strides_bytes[i];
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, cuuint32_t(rank),
                          const_cast<void*>(base), gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// [B][L][H][d]-general strided input viewed as (d, L, H, B) with a box of `rows` rows.
bool make_qkv_map(CUtensorMap* m, const void* base, const pisa_attn_desc& d,
                  const int64_t* st, uint32_t rows) {
    const uint64_t dims[4] = {uint64_t(d.head_dim), uint64_t(d.seq_len), uint64_t(d.heads),
                              uint64_t(d.batch)};
    uint64_t sb = uint64_t(st[0]) * 2;
    if (d.batch == 1) sb = std::max<uint64_t>(16, (uint64_t(st[1]) * d.heads) * 2);
    uint64_t sh = uint64_t(st[1]) * 2;
    if (d.heads == 1) sh = std::max<uint64_t>(16, uint64_t(st[2]) * d.seq_len * 2);
    const uint64_t strides[3] = {uint64_t(st[2]) * 2, sh, sb};
    const uint32_t box[4] = {64, rows, 1, 1};
    return make_map(m, base, 4, dims, strides, box);
}

bool make_3d_map(CUtensorMap* m, const void* base, uint64_t D, uint64_t rows, uint64_t BH,
                 uint32_t box_rows) {
    const uint64_t dims[3] = {D, rows, BH};
    const uint64_t strides[2] = {D * 2, rows * D * 2};
    const uint32_t box[3] = {64, box_rows, 1};
    return make_map(m, base, 3, dims, strides, box);
}

// Select path when K1 emitted the k_bar splits (N >= kSelectFusedMinN), env
// PISA_B200_FUSED_SELECT (read per call, so a test can switch it):
//   unset / other  streamed scoring (select_fused_kernel<D, true>: q_bar split
//                  in TMEM, k_bar splits by TMA, double-buffered accumulators,
//                  row-major keys) + topk_kernel;
//   1              the one-launch select (top-k in the scoring CTA): 1.32 ms
//                  against 0.56 ms at Wan2.1-14B (profiles/r02c_ab_select.log):
//                  its 400 CTAs select 128 rows each with 8 warps, where
//                  topk_kernel spreads one row per warp over the whole chip;
//   0              score_kernel (one CTA per 128 x 128 tile) + topk_kernel.
enum SelectMode { kSelectTiles = 0, kSelectOneLaunch = 1, kSelectStream = 2 };
SelectMode select_mode() {
    const char* e = std::getenv("PISA_B200_FUSED_SELECT");
    if (e && e[0] == '1') return kSelectOneLaunch;
    if (e && e[0] == '0') return kSelectTiles;
    return kSelectStream;
}

// K2c candidate search over the whole query-block range (k2q_overlap.cu; env
// PISA_B200_PAIR_FULL=0: the +-48 window), read per call. It cuts the union
// tiles of independent routing by 2.2 % (Wan2.1-14B gaussian: union/k 1.781 ->
// 1.741) for 0.37 ms of search against the window's 0.25 ms: -0.3 ms a step at
// Wan2.1-14B, neutral to -0.5 ms on clustered routing and HunyuanVideo
// (profiles/r02qrtu_ab_pair_full.log, batch v).
bool pair_full_on() {
    const char* e = std::getenv("PISA_B200_PAIR_FULL");
    return !(e && e[0] == '0');
}

// heads per two-kernel select chunk (env PISA_B200_SELECT_CHUNK_MB: key
// matrices of at most that many MB, so they stay L2-resident between the two
// kernels). Default 0 = all heads in one pair of launches: at Wan2.1-14B the
// chunked form measured 0.60 / 0.66 / 0.83 ms for 80 / 40 / 20 MB chunks
// against 0.56 ms (profiles/r02p_ab_select_chunks.log) -- smaller launches
// cost more than the HBM round trip of the keys saves.
int64_t select_chunk_heads(int64_t N, int64_t BH) {
    static const int64_t mb = [] {
        const char* e = std::getenv("PISA_B200_SELECT_CHUNK_MB");
        return e ? int64_t(std::atoll(e)) : int64_t(0);
    }();
    if (mb <= 0) return BH;
    const int64_t per_head = N * N * 4;
    return std::max<int64_t>(1, std::min<int64_t>(BH, (mb << 20) / per_head));
}

// ------------------------------------------------------------ resolve --
struct Plan {
    int64_t BH, L, D, N, Npad, W, k, nchunk1, nchunk2;
    int64_t statsG;  // key blocks per K1 CTA
    double scale;
    int64_t qb0 = 0, qb1 = 0;  // query-block range of the fused step ([0, N) unless restricted)
};

pisa_status resolve(pisa_ctx* ctx, const pisa_attn_desc* d, Plan* p) {
    if (!d) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null descriptor");
    if (d->batch < 1 || d->heads < 1 || d->seq_len < 1 || d->head_dim < 1)
        return fail(ctx, PISA_ERR_INVALID_DIMENSION,
                    "batch, heads, seq_len and head_dim must all be >= 1");
    if (d->block_size < 1 || d->group_size < 1)  // attention.hpp:40-42
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "block_size and group_size must be >= 1");
    if (!d->ragged && d->seq_len % d->block_size != 0)  // attention.hpp:43-47
        return fail(ctx, PISA_ERR_BLOCK_DIVISIBILITY,
                    "seq_len " + std::to_string(d->seq_len) + " not divisible by block size " +
                        std::to_string(d->block_size));
    if (d->block_size != 64)
        return fail(ctx, PISA_ERR_UNSUPPORTED, "the GPU path tiles 64-row blocks only");
    if (d->head_dim != 64 && d->head_dim != 128)
        return fail(ctx, PISA_ERR_UNSUPPORTED, "head_dim must be 64 or 128 on the GPU path");
    if (d->variant < 0 || d->variant > 4)
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "unknown variant");
    if (d->variant == PISA_BLOCK_FIRST)
        return fail(ctx, PISA_ERR_UNSUPPORTED, "BlockFirst is not on the GPU path");
    if (d->router != PISA_ROUTER_PLAIN && d->router != PISA_ROUTER_COVARIANCE)
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "unknown router");
    if (d->router == PISA_ROUTER_COVARIANCE && !(d->epsilon > 0.0))  // router.hpp:164-166
        return fail(ctx, PISA_ERR_INVALID_EPSILON,
                    "epsilon must be > 0, got " + std::to_string(d->epsilon));
    if (d->row_level)
        return fail(ctx, PISA_ERR_UNSUPPORTED, "row-level routing is not on the GPU path");
    const int64_t N = (d->seq_len + 63) / 64;
    if (N > 4096)  // the fused kernel keeps the union list and masks in shared memory
        return fail(ctx, PISA_ERR_UNSUPPORTED, "more than 4096 key blocks (seq_len > 262144)");
    int64_t k = d->topk;
    if (k <= 0) {
        if (k < 0) return fail(ctx, PISA_ERR_INVALID_SPARSITY, "k must lie in [1, N]");
        const double r = d->sparsity;
        if (!(r >= 0.0) || r >= 1.0)  // router.hpp:81-84
            return fail(ctx, PISA_ERR_INVALID_SPARSITY,
                        "sparsity must lie in [0, 1), got " + std::to_string(r));
        k = std::llround((1.0 - r) * double(N));
        k = std::max<int64_t>(1, std::min<int64_t>(k, N));
    } else if (k > N) {
        return fail(ctx, PISA_ERR_INVALID_SPARSITY,
                    "k must lie in [1, N], got " + std::to_string(k) + " for N = " + std::to_string(N));
    }
    const int64_t D = d->head_dim;
    // strides of extents > 1 must keep 16-byte rows: TMA (q/k/v) and the fused
    // epilogue's 16-byte stores (o: 8 bf16 or 4 fp32 elements)
    auto st_ok = [&](const int64_t* s, int64_t m) {
        return s[2] >= D && s[2] % m == 0 && (d->heads == 1 || (s[1] >= 0 && s[1] % m == 0)) &&
               (d->batch == 1 || (s[0] >= 0 && s[0] % m == 0));
    };
    if (!st_ok(d->q_strides, 8) || !st_ok(d->k_strides, 8) || !st_ok(d->v_strides, 8))
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "q/k/v strides must be multiples of 8 elements");

    p->BH = d->batch * d->heads;
    p->L = d->seq_len;
    p->D = D;
    p->N = N;
    p->Npad = (N + 127) / 128 * 128;  // K3 reads 128-centroid tiles
    p->W = (N + 31) / 32;
    p->k = k;
    // K1: up to kStatsG key blocks per chunk (work unit; every chunk writes a
    // D x D fp32 H partial). Short (image) heads: 6 chunks per head, so that
    // their 24 heads make about one wave of work units on 148 SMs (FLUX's
    // N = 72: 6 chunks of 12 -- 144 units -- 0.141 ms a step against 0.143 for
    // 18 chunks of 4, profiles/r02m_ab_k1.log); longer heads: 24 chunks per
    // head (Wan2.1-1.3B, N = 512 with 12 heads: 16 chunks of 32 measured 0.097
    // ms against 0.076 for 24 chunks of 22, profiles/r02n_*). A function of N
    // only: a head's H_bar partial sums -- and with them its output bits -- do
    // not depend on how many other heads share the launch, so head-sharded
    // ranks reproduce the single-GPU result exactly.
    p->statsG = std::max<int64_t>(4, std::min<int64_t>(kStatsG, N < 256 ? (N + 5) / 6 : (N + 23) / 24));
    if (const char* e = std::getenv("PISA_B200_STATS_G"))  // (A/B of K1's chunk size)
        p->statsG = std::max<int64_t>(1, std::min<int64_t>(kStatsG, std::atoll(e)));
    p->nchunk1 = (N + p->statsG - 1) / p->statsG;
    p->nchunk2 = (N + 63) / 64;
    p->scale = d->scale > 0.0 ? d->scale : 1.0 / std::sqrt(double(D));  // attention.hpp:34-37
    return PISA_OK;
}

// ------------------------------------------------------------ workspace --
struct Work {
    float *kbar, *vhat, *qbar, *hpart, *hbar, *kglob, *norms, *rect, *tri;
    int* cand;
    int2* pairs;
    __nv_bfloat16 *kbar_bf, *vhat_bf, *hbar_bf;
    __nv_bfloat16* ksplit;  // k_bar hi / mid / lo [3][BH][N][D] (fused K2 only, else null)
    int32_t* selected;
    uint32_t* mask;
    uint32_t* keys;
    int* flag;
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// cudaMalloc is a "potentially unsafe" call while a stream of this thread is
// being captured in global mode (torch.cuda.graph's default); allocating a
// workspace for a new stream / shape inside a capture is still correct (the
// memory outlives the graph), so allocate in relaxed mode, as torch's own
// caching allocator does.
struct RelaxedCapture {
    cudaStreamCaptureMode prev = cudaStreamCaptureModeRelaxed;
    RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&prev); }
    ~RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&prev); }
};

pisa_ctx::Arena* arena_of(pisa_ctx* ctx, cudaStream_t s) {
    for (auto& a : ctx->arenas)
        if (a.stream == s) return &a;
    pisa_ctx::Arena a;
    a.stream = s;
    // flags are reset with cudaMemsetAsync on the stream before every use
    RelaxedCapture rc;
    if (cudaMalloc(&a.flags, 16 * sizeof(int)) != cudaSuccess) return nullptr;
    ctx->arenas.push_back(a);
    return &ctx->arenas.back();
}

pisa_status workspace(pisa_ctx* ctx, const Plan& p, Work* w, cudaStream_t s) {
    const size_t BH = size_t(p.BH), N = size_t(p.N), D = size_t(p.D);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes);
        return o;
    };
    const size_t o_kbar = take(BH * N * D * 4), o_vhat = take(BH * N * D * 4),
                 o_qbar = take(BH * N * D * 4), o_hpart = take(BH * p.nchunk1 * D * D * 4),
                 o_hbar = take(BH * D * D * 4), o_kglob = take(BH * D * 4),
                 o_kbf = take(BH * p.Npad * D * 2), o_vbf = take(BH * p.Npad * D * 2),
                 o_hbf = take(BH * D * D * 2), o_sel = take(BH * N * p.k * 4),
                 o_mask = take(BH * N * p.W * 4),
                 o_keys = take(std::max({size_t(select_chunk_heads(p.N, p.BH)) * N * N,
                                         p.N >= kSelectFusedMinN ? size_t(kScratchSlots) * 128 * N : size_t(0),
                                         (BH * N * N + 1) / 2}) * 4),  // (+ K2c's u16 overlap matrix)
                 o_ksplit = take(p.N >= kSelectFusedMinN ? 3 * BH * N * D * 2 : 0),
                 o_norms = take(BH * N * 4), o_rect = take(BH * N * 4), o_tri = take(BH * N * kTriStride * 4),
                 o_cand = take(BH * N * kPairCand * 4), o_pairs = take(BH * ((N + 1) / 2) * 8);
    pisa_ctx::Arena* ar = arena_of(ctx, s);
    if (!ar) return fail(ctx, PISA_ERR_CUDA, "workspace flag allocation failed");
    if (off > ar->bytes) {
        // grow geometrically (few retired arenas under slowly growing shapes)
        const size_t want = std::max(off, ar->bytes + ar->bytes / 2);
        void* nb = nullptr;
        RelaxedCapture rc;
        const cudaError_t e = cudaMalloc(&nb, want);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "workspace cudaMalloc");
        if (ar->base) ctx->retired.push_back(ar->base);
        ar->base = nb;
        ar->bytes = want;
    }
    char* b = static_cast<char*>(ar->base);
    w->kbar = reinterpret_cast<float*>(b + o_kbar);
    w->vhat = reinterpret_cast<float*>(b + o_vhat);
    w->qbar = reinterpret_cast<float*>(b + o_qbar);
    w->hpart = reinterpret_cast<float*>(b + o_hpart);
    w->hbar = reinterpret_cast<float*>(b + o_hbar);
    w->kglob = reinterpret_cast<float*>(b + o_kglob);
    w->norms = reinterpret_cast<float*>(b + o_norms);
    w->rect = reinterpret_cast<float*>(b + o_rect);
    w->tri = reinterpret_cast<float*>(b + o_tri);
    w->cand = reinterpret_cast<int*>(b + o_cand);
    w->pairs = reinterpret_cast<int2*>(b + o_pairs);
    w->kbar_bf = reinterpret_cast<__nv_bfloat16*>(b + o_kbf);
    w->vhat_bf = reinterpret_cast<__nv_bfloat16*>(b + o_vbf);
    w->hbar_bf = reinterpret_cast<__nv_bfloat16*>(b + o_hbf);
    w->selected = reinterpret_cast<int32_t*>(b + o_sel);
    w->mask = reinterpret_cast<uint32_t*>(b + o_mask);
    w->keys = reinterpret_cast<uint32_t*>(b + o_keys);
    w->ksplit = p.N >= kSelectFusedMinN ? reinterpret_cast<__nv_bfloat16*>(b + o_ksplit) : nullptr;
    w->flag = ar->flags;
    return PISA_OK;
}

// fork: K1b goes to ctx->side after K1 (the caller joins with join_hbar
// before anything that reads H_bar / k_bar_global: K1c, K3); the select only
// needs K1's k_bar / q_bar, so at image sizes the reduce hides under it.
pisa_status run_stats(pisa_ctx* ctx, const pisa_attn_desc& d, const Plan& p, const Work& w,
                      const void* q, const void* k, const void* v, cudaStream_t s, bool fork = false) {
    CUtensorMap tq, tk, tv;
    if (!make_qkv_map(&tq, q, d, d.q_strides, 64) || !make_qkv_map(&tk, k, d, d.k_strides, 64) ||
        !make_qkv_map(&tv, v, d, d.v_strides, 64))
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "TMA descriptor rejected the q/k/v layout");
    StatsArgs sa{w.kbar,  w.vhat,      w.qbar,       w.kbar_bf,        w.vhat_bf,
                 w.hpart, w.ksplit,    int(p.BH),    int(p.L),         int(p.N),
                 int(p.Npad), int(d.heads), int(p.nchunk1), int(p.statsG)};
    cudaError_t e;
    {
        ProfScope ps(ctx, kK1, s);
        e = launch_block_stats(int(p.D), tq, tk, tv, sa, int(p.BH), s);
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "block_stats launch");
    cudaStream_t sr = s;
    if (fork) {
        if (!ctx->side) {
            e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_k1, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_k1b, cudaEventDisableTiming);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "side stream setup");
        }
        if ((e = cudaEventRecord(ctx->ev_k1, s)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(ctx->side, ctx->ev_k1, 0)) != cudaSuccess)
            return cuda_fail(ctx, e, "K1b fork");
        sr = ctx->side;
    }
    {
        ProfScope ps(ctx, kK1b, sr);
        e = launch_hbar_reduce(int(p.D), w.hpart, int(p.nchunk1), int(p.N), w.kbar, w.hbar, w.hbar_bf,
                               d.variant == PISA_GLOBAL_CENTROID ? w.kglob : nullptr, int(p.BH), sr);
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "hbar_reduce launch");
    if (fork && (e = cudaEventRecord(ctx->ev_k1b, sr)) != cudaSuccess) return cuda_fail(ctx, e, "K1b event");
    ctx->launches += 2;
    return PISA_OK;
}

// s waits for the forked K1b (run_stats(fork = true))
pisa_status join_hbar(pisa_ctx* ctx, cudaStream_t s) {
    const cudaError_t e = cudaStreamWaitEvent(s, ctx->ev_k1b, 0);
    return e == cudaSuccess ? PISA_OK : cuda_fail(ctx, e, "K1b join");
}

// K1c: M_j = ||H_j - H_bar||_2 and the rectifier log(M_j + eps) (covariance router),
// after run_stats (needs k_bar and H_bar in the workspace).
pisa_status run_norms(pisa_ctx* ctx, const pisa_attn_desc& d, const Plan& p, const Work& w,
                      const void* k, const void* v, cudaStream_t s) {
    NormArgs a{w.kbar,      w.hbar,        w.norms,       w.rect,        d.epsilon,
               int(p.L),    int(p.N),      int(d.heads),  d.k_strides[0], d.k_strides[1],
               d.k_strides[2], d.v_strides[0], d.v_strides[1], d.v_strides[2], w.tri};
    CUtensorMap tk, tv;
    if (!make_qkv_map(&tk, k, d, d.k_strides, 64) || !make_qkv_map(&tv, v, d, d.v_strides, 64))
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "TMA descriptor rejected the k/v layout");
    ProfScope ps(ctx, kK1c, s);
    const cudaError_t e = launch_block_norms(int(p.D), tk, tv, static_cast<const __nv_bfloat16*>(k),
                                             static_cast<const __nv_bfloat16*>(v), a, int(p.BH), s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "block_norms launch");
    ctx->launches += block_norms_launches(int(p.D));
    return PISA_OK;
}

// ksplit: K1's hi / mid / lo split of k_bar (the forward's own statistics):
// the fused one-launch select; null (caller-supplied statistics, short
// heads): score_kernel + topk_kernel
pisa_status run_select(pisa_ctx* ctx, const pisa_attn_desc& d, const Plan& p, const float* qbar,
                       const float* kbar, const float* rect, int32_t* selected, uint32_t* mask,
                       uint32_t* keys, cudaStream_t s, const __nv_bfloat16* ksplit = nullptr) {
    SelectArgs a{qbar, kbar, rect, selected, mask, int(p.N), int(p.W), int(p.k), d.force_diagonal,
                 float(p.scale)};
    const SelectMode mode = select_mode();
    if (ksplit && mode != kSelectTiles && (mode == kSelectOneLaunch || select_chunk_heads(p.N, p.BH) >= p.BH)) {
        CUtensorMap tks;
        if (!make_3d_map(&tks, ksplit, p.D, p.N, 3 * p.BH, 128))
            return fail(ctx, PISA_ERR_CUDA, "TMA descriptor creation failed (k_bar split)");
        ProfScope ps(ctx, kK2, s);
        const cudaError_t e = mode == kSelectOneLaunch ? launch_select_fused(int(p.D), tks, a, int(p.BH), keys, s)
                                                       : launch_select_stream(int(p.D), tks, a, int(p.BH), keys, s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "select launch");
        ctx->launches += mode == kSelectOneLaunch ? 1 : 2;
        return PISA_OK;
    }
    // (optionally) heads in chunks whose N x N key matrix (u32) stays
    // L2-resident between score_kernel and topk_kernel: the scratch is reused
    // chunk after chunk (select_chunk_heads)
    const int64_t hc = select_chunk_heads(p.N, p.BH);
    ProfScope ps(ctx, kK2, s);
    for (int64_t h0 = 0; h0 < p.BH; h0 += hc) {
        const int64_t nh = std::min(hc, p.BH - h0);
        SelectArgs c = a;
        c.qbar = qbar + h0 * p.N * p.D;
        c.kbar = kbar + h0 * p.N * p.D;
        c.rect = rect ? rect + h0 * p.N : nullptr;
        c.selected = selected ? selected + h0 * p.N * p.k : nullptr;
        c.mask = mask + h0 * p.N * p.W;
        const cudaError_t e = launch_select(int(p.D), c, int(nh), keys, s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "select launch");
        ctx->launches += 2;
    }
    return PISA_OK;
}

// Non-finite output check (check_output_finite, engine.hpp:83-93):
//   kFiniteOff   no check;
//   kFiniteArm   the fused kernel ORs into the stream's device flag, nobody
//                resets or reads it (the host path resets it once and reads it
//                after its final synchronisation);
//   kFiniteSync  reset, arm, synchronise and report NUMERICAL_OVERFLOW.
enum FiniteMode { kFiniteOff = 0, kFiniteArm = 1, kFiniteSync = 2 };

pisa_status run_fused(pisa_ctx* ctx, const pisa_attn_desc& d, const Plan& p, const Work& w,
                      const void* q, const void* k, const void* v, void* o, const pisa_diag* diag,
                      cudaStream_t s, FiniteMode fm) {
    CUtensorMap tq, tk, tv, tkb, tvh, th;
    if (!make_qkv_map(&tq, q, d, d.q_strides, 16) || !make_qkv_map(&tk, k, d, d.k_strides, 64) ||
        !make_qkv_map(&tv, v, d, d.v_strides, 64))
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "TMA descriptor rejected the q/k/v layout");
    if (!make_3d_map(&tkb, w.kbar_bf, p.D, p.Npad, p.BH, 64) ||
        !make_3d_map(&tvh, w.vhat_bf, p.D, p.Npad, p.BH, 64) ||
        !make_3d_map(&th, w.hbar_bf, p.D, p.D, p.BH, uint32_t(p.D)))
        return fail(ctx, PISA_ERR_CUDA, "TMA descriptor creation failed");
    // overlap-aware pairing of query blocks (K2c/K2d); PISA_B200_PAIRING=0 keeps (2t, 2t+1)
    const int qb0 = int(p.qb0), qb1 = int(p.qb1 > 0 ? p.qb1 : p.N);
    constexpr int kPairMinBlocks = 768;
    const bool pairing = qb1 - qb0 > 2 && (ctx->pairing == 2 || (ctx->pairing == 1 && qb1 - qb0 >= kPairMinBlocks));
    if (pairing) {
        ProfScope ps(ctx, kPair, s);
        // full-range candidate search (overlap matrix on the tensor cores, in the
        // keys scratch: the select is done with it) up to 2048 blocks a range
        const bool full = pair_full_on() && pairing_full_supported(qb0, qb1, int(p.W));
        const cudaError_t e = launch_pairing(w.mask, int(p.N), int(p.W), qb0, qb1, int(p.BH), w.cand, w.pairs, s,
                                             full ? reinterpret_cast<uint16_t*>(w.keys) : nullptr);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "pairing launch");
        ctx->launches += full ? 3 : 2;
    }
    FusedArgs a{};
    a.pairs = pairing ? w.pairs : nullptr;
    a.q = static_cast<const __nv_bfloat16*>(q);
    a.qs_b = d.q_strides[0];
    a.qs_h = d.q_strides[1];
    a.qs_l = d.q_strides[2];
    a.mask = w.mask;
    a.kbar_global = w.kglob;
    a.out = o;
    a.os_b = d.o_strides[0];
    a.os_h = d.o_strides[1];
    a.os_l = d.o_strides[2];
    a.diag_m = diag ? diag->row_max : nullptr;
    a.diag_l = diag ? diag->ell : nullptr;
    a.diag_lt = diag ? diag->ell_tail : nullptr;
    a.nonfinite = fm != kFiniteOff ? w.flag : nullptr;
    a.L = int(p.L);
    a.N = int(p.N);
    a.H = int(d.heads);
    a.W = int(p.W);
    a.nchunk2 = int(p.nchunk2);
    a.variant = d.variant;
    a.literal_phase3 = d.literal_phase3;
    a.out_f32 = d.out_dtype == PISA_DTYPE_F32;
    a.k = int(p.k);
    a.qb0 = qb0;
    a.qb1 = qb1;
    a.scale = float(p.scale);
    a.trace = ctx->trace;
    a.tile_count = ctx->prof ? ctx->tiles_dev : nullptr;
    a.trace_tile = ctx->trace_tile;
    if (fm == kFiniteSync) {
        const cudaError_t e = cudaMemsetAsync(w.flag, 0, sizeof(int), s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "flag reset");
    }
    cudaError_t e;
    {
        ProfScope ps(ctx, kK3, s);
        e = launch_fused(int(p.D), tq, tk, tv, tkb, tvh, th, a, int(p.BH), s);
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "fused launch");
    ctx->launches += 1;
    if (fm == kFiniteSync) {
        cudaError_t e2 = cudaMemcpyAsync(ctx->flag_host, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s);
        if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(s);
        if (e2 != cudaSuccess) return cuda_fail(ctx, e2, "non-finite check");
        if (*ctx->flag_host)  // engine.hpp:83-93
            return fail(ctx, PISA_ERR_NUMERICAL_OVERFLOW, "non-finite output");
    }
    return PISA_OK;
}

// The streams (and events) of the host-buffer entries, created on first use.
pisa_status host_streams(pisa_ctx* ctx) {
    if (ctx->st_h2d) return PISA_OK;
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->st_h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->st_comp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->st_d2h, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&ctx->ev_h2d[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_comp[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_d2h[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "stream setup");
    return PISA_OK;
}

// Device copies of host arrays for the synchronous host-buffer step entries
// (not a hot path: plain cudaMalloc / cudaMemcpy, freed on scope exit).
struct DevBufs {
    std::vector<void*> ptrs;
    cudaError_t err = cudaSuccess;
    void* alloc(size_t bytes) {
        void* p = nullptr;
        if (err == cudaSuccess) err = cudaMalloc(&p, std::max<size_t>(bytes, 16));
        if (err == cudaSuccess) ptrs.push_back(p);
        return err == cudaSuccess ? p : nullptr;
    }
    void* upload(const void* h, size_t bytes) {
        void* p = h ? alloc(bytes) : nullptr;
        if (p && err == cudaSuccess) err = cudaMemcpy(p, h, bytes, cudaMemcpyHostToDevice);
        return p;
    }
    ~DevBufs() {
        for (void* p : ptrs) cudaFree(p);
    }
};

// dense [B][H][L][d] strides (the host entries' layout)
void dense_strides(pisa_attn_desc& d) {
    const int64_t ld = d.seq_len * d.head_dim;
    for (int64_t* s : {d.q_strides, d.k_strides, d.v_strides, d.o_strides}) {
        s[0] = d.heads * ld;
        s[1] = ld;
        s[2] = d.head_dim;
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Output checks of the calls that write O: dtype, and strides of extents > 1
// keeping 16-byte rows for the fused epilogue's 16-byte stores.
pisa_status check_out(pisa_ctx* ctx, const pisa_attn_desc* d, const void* o) {
    if (d->out_dtype != PISA_DTYPE_BF16 && d->out_dtype != PISA_DTYPE_F32)
        return fail(ctx, PISA_ERR_UNSUPPORTED, "output dtype must be bf16 or fp32");
    const int64_t m = d->out_dtype == PISA_DTYPE_F32 ? 4 : 8;
    const int64_t* s = d->o_strides;
    const bool ok = s[2] >= d->head_dim && s[2] % m == 0 && (d->heads == 1 || (s[1] >= 0 && s[1] % m == 0)) &&
                    (d->batch == 1 || (s[0] >= 0 && s[0] % m == 0));
    if (!ok)
        return fail(ctx, PISA_ERR_INVALID_DIMENSION,
                    "o strides must be >= head_dim and multiples of 16 bytes (8 bf16 / 4 fp32 elements)");
    if (o && !aligned16(o)) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "o must be 16-byte aligned");
    return PISA_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace

extern "C" {

int pisa_b200_abi_version(void) { return PISA_B200_ABI_VERSION; }

pisa_status pisa_b200_create(pisa_ctx** out, int device) {
    if (!out) return PISA_ERR_INVALID_DIMENSION;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return PISA_ERR_CUDA;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return PISA_ERR_CUDA;
    if (prop.major != 10) return PISA_ERR_UNSUPPORTED;  // sm_100a kernels only
    pisa_ctx* c = new pisa_ctx;
    c->device = device;
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    if (const char* ev = std::getenv("PISA_B200_PAIRING")) c->pairing = std::max(0, std::min(2, std::atoi(ev)));
    if (const char* ev = std::getenv("PISA_B200_HOST_CHUNKS")) c->host_chunks = std::max(1, std::atoi(ev));
    DeviceGuard g(device);
    if (cudaMallocHost(&c->flag_host, sizeof(int)) != cudaSuccess) {
        delete c;
        return PISA_ERR_CUDA;
    }
    *out = c;
    return PISA_OK;
}

void pisa_b200_destroy(pisa_ctx* c) {
    if (c && c->tiles_dev) cudaFree(c->tiles_dev);
    if (!c) return;
    DeviceGuard g(c->device);
    cudaDeviceSynchronize();
    for (auto& a : c->arenas) {
        if (a.base) cudaFree(a.base);
        if (a.flags) cudaFree(a.flags);
    }
    for (void* r : c->retired) cudaFree(r);
    if (c->stage) cudaFree(c->stage);
    if (c->flag_host) cudaFreeHost(c->flag_host);
    for (auto& r : c->recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : c->pool) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
        if (c->ev_h2d[i]) cudaEventDestroy(c->ev_h2d[i]);
        if (c->ev_comp[i]) cudaEventDestroy(c->ev_comp[i]);
        if (c->ev_d2h[i]) cudaEventDestroy(c->ev_d2h[i]);
    }
    if (c->st_h2d) cudaStreamDestroy(c->st_h2d);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->ev_k1) cudaEventDestroy(c->ev_k1);
    if (c->ev_k1b) cudaEventDestroy(c->ev_k1b);
    if (c->st_comp) cudaStreamDestroy(c->st_comp);
    if (c->st_d2h) cudaStreamDestroy(c->st_d2h);
    delete c;
}

const char* pisa_b200_last_error(const pisa_ctx* c) { return c ? c->last_error.c_str() : ""; }

int64_t pisa_b200_last_launch_count(const pisa_ctx* c) { return c ? c->launches : 0; }

const char* pisa_b200_kernel_name(int i) {
    if (i < 0 || i >= 8) return nullptr;
    return kKernelNames[i];
}

pisa_status pisa_b200_fused_tiles(pisa_ctx* c, int64_t* tiles) {
    if (!c || !tiles) return PISA_ERR_INVALID_DIMENSION;
    DeviceGuard g(c->device);
    unsigned long long h = 0;
    cudaError_t e = cudaSuccess;
    if (c->tiles_dev) {
        e = cudaMemcpy(&h, c->tiles_dev, sizeof(h), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemset(c->tiles_dev, 0, sizeof(h));
    }
    if (e != cudaSuccess) return cuda_fail(c, e, "fused_tiles");
    *tiles = int64_t(h);
    return PISA_OK;
}

pisa_status pisa_b200_debug_trace(pisa_ctx* c, unsigned long long* dev_buf, int tile) {
    if (!c) return PISA_ERR_INVALID_DIMENSION;
    c->trace = dev_buf;
    c->trace_tile = tile;
    return PISA_OK;
}

pisa_status pisa_b200_set_profiling(pisa_ctx* c, int enable) {
    if (!c) return PISA_ERR_INVALID_DIMENSION;
    c->prof = enable != 0;
    if (c->prof && !c->tiles_dev) {
        DeviceGuard g(c->device);
        cudaError_t e = cudaMalloc(&c->tiles_dev, sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaMemset(c->tiles_dev, 0, sizeof(unsigned long long));
        if (e != cudaSuccess) return cuda_fail(c, e, "profiling counter");
    }
    return PISA_OK;
}

pisa_status pisa_b200_read_profile(pisa_ctx* c, double* ms, int64_t* launches) {
    if (!c) return PISA_ERR_INVALID_DIMENSION;
    DeviceGuard g(c->device);
    for (int i = 0; i < 8; ++i) {
        if (ms) ms[i] = 0.0;
        if (launches) launches[i] = 0;
    }
    for (auto& r : c->recs) {
        cudaError_t e = cudaEventSynchronize(r.b);
        float t = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
        if (e != cudaSuccess) return cuda_fail(c, e, "read_profile");
        if (ms) ms[r.id] += t;
        if (launches) launches[r.id] += 1;
        c->pool.push_back(r.a);
        c->pool.push_back(r.b);
    }
    c->recs.clear();
    return PISA_OK;
}

pisa_status pisa_b200_sparsity_to_k(double r, int64_t n, int64_t* k, double* realized) {
    if (!(r >= 0.0) || r >= 1.0) return PISA_ERR_INVALID_SPARSITY;
    if (n <= 0) return PISA_ERR_INVALID_DIMENSION;
    int64_t kk = std::llround((1.0 - r) * double(n));
    kk = std::max<int64_t>(1, std::min<int64_t>(kk, n));
    if (k) *k = kk;
    if (realized) *realized = double(n - kk) / double(n);
    return PISA_OK;
}

pisa_status pisa_b200_resolve(const pisa_attn_desc* d, int64_t* num_blocks, int64_t* k,
                              double* scale) {
    Plan p;
    const pisa_status st = resolve(nullptr, d, &p);
    if (st != PISA_OK) return st;
    if (num_blocks) *num_blocks = p.N;
    if (k) *k = p.k;
    if (scale) *scale = p.scale;
    return PISA_OK;
}

namespace {
pisa_status fwd_range(pisa_ctx* ctx, const pisa_attn_desc* d, const void* q, const void* k, const void* v,
                      void* o, int64_t qb_begin, int64_t qb_end, const pisa_diag* diag, void* stream,
                      FiniteMode fm) {
    if (!ctx) return PISA_ERR_INVALID_DIMENSION;
    ctx->launches = 0;
    Plan p;
    pisa_status st = resolve(ctx, d, &p);
    if (st != PISA_OK) return st;
    if (qb_end < 0) qb_end = p.N;
    if (qb_begin < 0 || qb_begin >= qb_end || qb_end > p.N)
        return fail(ctx, PISA_ERR_INVALID_DIMENSION,
                    "query-block range [" + std::to_string(qb_begin) + ", " + std::to_string(qb_end) +
                        ") outside [0, " + std::to_string(p.N) + ")");
    p.qb0 = qb_begin;
    p.qb1 = qb_end;
    if (!q || !k || !v || !o) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null tensor pointer");
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "q/k/v/o must be 16-byte aligned");
    if ((st = check_out(ctx, d, o)) != PISA_OK) return st;
    DeviceGuard g(ctx->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    Work w;
    if ((st = workspace(ctx, p, &w, s)) != PISA_OK) return st;
    // (not under stream capture: a replayed graph with the fork/join measured
    // slower than the serial one, 0.163 vs 0.149 ms at FLUX, while eager
    // launches gain, 0.150 vs 0.158 ms; profiles/r02aq_ab_fork.log)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    const bool fork = cudaStreamIsCapturing(s, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone;
    if ((st = run_stats(ctx, *d, p, w, q, k, v, s, fork)) != PISA_OK) return st;
    const bool cov = d->router == PISA_ROUTER_COVARIANCE;
    if (cov && ((fork && (st = join_hbar(ctx, s)) != PISA_OK) || (st = run_norms(ctx, *d, p, w, k, v, s)) != PISA_OK))
        return st;
    int32_t* sel = (diag && diag->selected) ? diag->selected : nullptr;
    if ((st = run_select(ctx, *d, p, w.qbar, w.kbar, cov ? w.rect : nullptr, sel, w.mask, w.keys, s, w.ksplit)) !=
        PISA_OK)
        return st;
    if (fork && !cov && (st = join_hbar(ctx, s)) != PISA_OK) return st;
    return run_fused(ctx, *d, p, w, q, k, v, o, diag, s, fm);
}
}  // namespace

pisa_status pisa_b200_set_pairing(pisa_ctx* ctx, int mode) {
    if (!ctx) return PISA_ERR_INVALID_DIMENSION;
    if (mode < 0 || mode > 2) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "pairing mode must be 0, 1 or 2");
    ctx->pairing = mode;
    return PISA_OK;
}

pisa_status pisa_b200_fwd(pisa_ctx* ctx, const pisa_attn_desc* d, const void* q, const void* k,
                          const void* v, void* o, const pisa_diag* diag, void* stream) {
    if (!d) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null descriptor");
    return fwd_range(ctx, d, q, k, v, o, 0, -1, diag, stream, d->check_finite ? kFiniteSync : kFiniteOff);
}

pisa_status pisa_b200_fwd_qrange(pisa_ctx* ctx, const pisa_attn_desc* d, const void* q, const void* k,
                                 const void* v, void* o, int64_t qb_begin, int64_t qb_end,
                                 const pisa_diag* diag, void* stream) {
    if (!d) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null descriptor");
    return fwd_range(ctx, d, q, k, v, o, qb_begin, qb_end, diag, stream,
                     d->check_finite ? kFiniteSync : kFiniteOff);
}

pisa_status pisa_b200_block_stats(pisa_ctx* ctx, const pisa_attn_desc* d, const void* q,
                                  const void* k, const void* v, float* k_bar, float* v_hat,
                                  float* q_bar, float* h_bar, void* stream) {
    if (!ctx) return PISA_ERR_INVALID_DIMENSION;
    ctx->launches = 0;
    Plan p;
    pisa_status st = resolve(ctx, d, &p);
    if (st != PISA_OK) return st;
    if (!q || !k || !v) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null tensor pointer");
    if (!aligned16(q) || !aligned16(k) || !aligned16(v))
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "q/k/v must be 16-byte aligned");
    DeviceGuard g(ctx->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    Work w;
    if ((st = workspace(ctx, p, &w, s)) != PISA_OK) return st;
    if ((st = run_stats(ctx, *d, p, w, q, k, v, s)) != PISA_OK) return st;
    const size_t nd = size_t(p.BH) * p.N * p.D * 4, dd = size_t(p.BH) * p.D * p.D * 4;
    cudaError_t e = cudaSuccess;
    if (k_bar && e == cudaSuccess) e = cudaMemcpyAsync(k_bar, w.kbar, nd, cudaMemcpyDeviceToDevice, s);
    if (v_hat && e == cudaSuccess) e = cudaMemcpyAsync(v_hat, w.vhat, nd, cudaMemcpyDeviceToDevice, s);
    if (q_bar && e == cudaSuccess) e = cudaMemcpyAsync(q_bar, w.qbar, nd, cudaMemcpyDeviceToDevice, s);
    if (h_bar && e == cudaSuccess) e = cudaMemcpyAsync(h_bar, w.hbar, dd, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "block_stats copy-out");
    return PISA_OK;
}

pisa_status pisa_b200_select(pisa_ctx* ctx, const pisa_attn_desc* d, const float* q_bar,
                             const float* k_bar, int32_t* selected, uint32_t* mask, void* stream) {
    if (!ctx) return PISA_ERR_INVALID_DIMENSION;
    ctx->launches = 0;
    Plan p;
    pisa_status st = resolve(ctx, d, &p);
    if (st != PISA_OK) return st;
    if (!q_bar || !k_bar || (!selected && !mask))
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null pointer");
    DeviceGuard g(ctx->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    Work w;
    if ((st = workspace(ctx, p, &w, s)) != PISA_OK) return st;
    if (d->router != PISA_ROUTER_PLAIN)
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "covariance routing: use pisa_b200_select_cov");
    return run_select(ctx, *d, p, q_bar, k_bar, nullptr, selected, mask ? mask : w.mask, w.keys, s);
}

pisa_status pisa_b200_block_norms(pisa_ctx* ctx, const pisa_attn_desc* d, const void* q,
                                  const void* k, const void* v, float* m, void* stream) {
    if (!ctx) return PISA_ERR_INVALID_DIMENSION;
    ctx->launches = 0;
    Plan p;
    pisa_status st = resolve(ctx, d, &p);
    if (st != PISA_OK) return st;
    if (!q || !k || !v || !m) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null pointer");
    DeviceGuard g(ctx->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    Work w;
    if ((st = workspace(ctx, p, &w, s)) != PISA_OK) return st;
    if ((st = run_stats(ctx, *d, p, w, q, k, v, s)) != PISA_OK) return st;
    pisa_attn_desc dd = *d;
    if (!(dd.epsilon > 0.0)) dd.epsilon = 1e-6;  // M_j itself does not depend on eps
    if ((st = run_norms(ctx, dd, p, w, k, v, s)) != PISA_OK) return st;
    const cudaError_t e =
        cudaMemcpyAsync(m, w.norms, size_t(p.BH) * p.N * 4, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "block_norms copy-out");
    return PISA_OK;
}

pisa_status pisa_b200_select_cov(pisa_ctx* ctx, const pisa_attn_desc* d, const float* q_bar,
                                 const float* k_bar, const float* m, int32_t* selected,
                                 uint32_t* mask, void* stream) {
    if (!ctx) return PISA_ERR_INVALID_DIMENSION;
    ctx->launches = 0;
    Plan p;
    pisa_status st = resolve(ctx, d, &p);
    if (st != PISA_OK) return st;
    if (!(d->epsilon > 0.0))  // router.hpp:164-166
        return fail(ctx, PISA_ERR_INVALID_EPSILON, "epsilon must be > 0, got " + std::to_string(d->epsilon));
    if (!q_bar || !k_bar || !m || (!selected && !mask))
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null pointer");
    DeviceGuard g(ctx->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    Work w;
    if ((st = workspace(ctx, p, &w, s)) != PISA_OK) return st;
    cudaError_t e = launch_rectifier(m, d->epsilon, w.rect, int(p.BH) * int(p.N), s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "rectifier launch");
    ctx->launches += 1;
    return run_select(ctx, *d, p, q_bar, k_bar, w.rect, selected, mask ? mask : w.mask, w.keys, s);
}

pisa_status pisa_b200_attention(pisa_ctx* ctx, const pisa_attn_desc* d, const void* q,
                                const void* k, const void* v, const int32_t* selected,
                                const float* k_bar, const float* v_hat, const float* h_bar,
                                void* o, const pisa_diag* diag, void* stream) {
    if (!ctx) return PISA_ERR_INVALID_DIMENSION;
    ctx->launches = 0;
    Plan p;
    pisa_status st = resolve(ctx, d, &p);
    if (st != PISA_OK) return st;
    if (!q || !k || !v || !o || !selected || !k_bar || !v_hat || !h_bar)
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null pointer");
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "q/k/v/o must be 16-byte aligned");
    if ((st = check_out(ctx, d, o)) != PISA_OK) return st;
    DeviceGuard g(ctx->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    Work w;
    if ((st = workspace(ctx, p, &w, s)) != PISA_OK) return st;
    // plan -> mask, with SelectionPlan::validate (router.hpp:50-70)
    cudaError_t e = cudaMemsetAsync(w.flag + 1, 0, sizeof(int), s);
    if (e == cudaSuccess) {
        ProfScope ps(ctx, kPlan, s);
        e = launch_plan_to_mask(selected, int(p.N), int(p.k), int(p.W), w.mask, w.flag + 1, int(p.BH), s);
    }
    if (e == cudaSuccess) {
        ProfScope ps(ctx, kToBf16, s);
        e = launch_stats_to_bf16(int(p.D), k_bar, v_hat, h_bar, int(p.N), int(p.Npad), w.kbar_bf,
                                 w.vhat_bf, w.hbar_bf,
                                 d->variant == PISA_GLOBAL_CENTROID ? w.kglob : nullptr, int(p.BH), s);
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(ctx->flag_host, w.flag + 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "plan upload");
    ctx->launches += 2;
    if (*ctx->flag_host)
        return fail(ctx, PISA_ERR_INVALID_SPARSITY, "plan has out-of-range or non-ascending indices");
    return run_fused(ctx, *d, p, w, q, k, v, o, diag, s, d->check_finite ? kFiniteSync : kFiniteOff);
}

pisa_status pisa_b200_fwd_host(pisa_ctx* ctx, const pisa_attn_desc* d, const void* q,
                               const void* k, const void* v, void* o, const pisa_diag* hdiag) {
    if (!ctx) return PISA_ERR_INVALID_DIMENSION;
    Plan p;
    pisa_status st = resolve(ctx, d, &p);
    if (st != PISA_OK) return st;
    if (!q || !k || !v || !o) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null tensor pointer");
    if (d->out_dtype != PISA_DTYPE_BF16 && d->out_dtype != PISA_DTYPE_F32)
        return fail(ctx, PISA_ERR_UNSUPPORTED, "output dtype must be bf16 or fp32");
    DeviceGuard g(ctx->device);
    // host layout: dense [B][H][L][d]; stage a few (b,h) slices at a time
    const int64_t BH = p.BH, L = p.L, D = p.D;
    const size_t in_bytes = size_t(L) * D * 2;
    const size_t out_bytes = size_t(L) * D * (d->out_dtype == PISA_DTYPE_F32 ? 4 : 2);
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(BH, (BH + ctx->host_chunks - 1) / ctx->host_chunks));
    const bool want_diag = hdiag && (hdiag->row_max || hdiag->ell || hdiag->ell_tail || hdiag->selected);
    const size_t diag_bytes = want_diag ? size_t(L) * 4 * 3 + size_t(p.N) * p.k * 4 : 0;
    const size_t set_bytes = size_t(chunk) * (3 * in_bytes + out_bytes + diag_bytes);
    cudaError_t e = cudaSuccess;
    if ((st = host_streams(ctx)) != PISA_OK) return st;
    if (2 * set_bytes > ctx->stage_bytes) {
        if (ctx->stage) cudaFree(ctx->stage);
        ctx->stage = nullptr;
        ctx->stage_bytes = 0;
        e = cudaMalloc(&ctx->stage, 2 * set_bytes);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "staging cudaMalloc");
        ctx->stage_bytes = 2 * set_bytes;
    }
    int64_t launches = 0;
    // non-finite check over all chunks: reset the compute stream's flag once,
    // every chunk's fused kernel ORs into it, read after the final sync
    int* flag = nullptr;
    if (d->check_finite) {
        pisa_ctx::Arena* ar = arena_of(ctx, ctx->st_comp);
        if (!ar) return fail(ctx, PISA_ERR_CUDA, "workspace flag allocation failed");
        flag = ar->flags;
        e = cudaMemsetAsync(flag, 0, sizeof(int), ctx->st_comp);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "flag reset");
    }
    // chunk sizes: a remainder first, then `chunk`-sized ones, then a shrinking
    // tail (2, 1) so that each chunk's compute hides behind the next chunk's
    // H2D (compute is ~0.6x the H2D time per head) and the exposed tail --
    // compute + D2H of the last chunk -- is one head
    std::vector<int64_t> sizes;
    {
        const bool shrink = chunk >= 3 && BH >= chunk + 3;
        const int64_t rest = shrink ? BH - 3 : BH;
        if (rest % chunk) sizes.push_back(rest % chunk);
        for (int64_t i = 0; i < rest / chunk; ++i) sizes.push_back(chunk);
        if (shrink) {
            sizes.push_back(2);
            sizes.push_back(1);
        }
    }
    const int64_t nchunks = int64_t(sizes.size());
    int64_t h0 = 0;
    for (int64_t c = 0; c < nchunks; h0 += sizes[size_t(c)], ++c) {
        const int sidx = int(c & 1);
        const int64_t hc = sizes[size_t(c)];
        char* set = static_cast<char*>(ctx->stage) + sidx * set_bytes;
        char* dq = set;
        char* dk = dq + chunk * in_bytes;
        char* dv = dk + chunk * in_bytes;
        char* dout = dv + chunk * in_bytes;
        char* ddiag = dout + chunk * out_bytes;
        pisa_diag dd{};
        if (want_diag) {
            dd.row_max = reinterpret_cast<float*>(ddiag);
            dd.ell = dd.row_max + chunk * L;
            dd.ell_tail = dd.ell + chunk * L;
            dd.selected = reinterpret_cast<int32_t*>(dd.ell_tail + chunk * L);
        }
        if (c >= 2) cudaStreamWaitEvent(ctx->st_h2d, ctx->ev_comp[sidx], 0);
        e = cudaMemcpyAsync(dq, static_cast<const char*>(q) + h0 * in_bytes, hc * in_bytes, cudaMemcpyHostToDevice, ctx->st_h2d);
        if (e == cudaSuccess) e = cudaMemcpyAsync(dk, static_cast<const char*>(k) + h0 * in_bytes, hc * in_bytes, cudaMemcpyHostToDevice, ctx->st_h2d);
        if (e == cudaSuccess) e = cudaMemcpyAsync(dv, static_cast<const char*>(v) + h0 * in_bytes, hc * in_bytes, cudaMemcpyHostToDevice, ctx->st_h2d);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_h2d[sidx], ctx->st_h2d);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D");
        cudaStreamWaitEvent(ctx->st_comp, ctx->ev_h2d[sidx], 0);
        if (c >= 2) cudaStreamWaitEvent(ctx->st_comp, ctx->ev_d2h[sidx], 0);
        pisa_attn_desc dc = *d;
        dc.batch = 1;
        dc.heads = hc;
        const int64_t ld = L * D;
        for (int t = 0; t < 3; ++t) {
            int64_t* s3 = t == 0 ? dc.q_strides : t == 1 ? dc.k_strides : dc.v_strides;
            s3[0] = hc * ld;
            s3[1] = ld;
            s3[2] = D;
        }
        dc.o_strides[0] = hc * ld;
        dc.o_strides[1] = ld;
        dc.o_strides[2] = D;
        st = fwd_range(ctx, &dc, dq, dk, dv, dout, 0, -1, want_diag ? &dd : nullptr, ctx->st_comp,
                       flag ? kFiniteArm : kFiniteOff);
        if (st != PISA_OK) return st;
        launches += ctx->launches;
        cudaEventRecord(ctx->ev_comp[sidx], ctx->st_comp);
        cudaStreamWaitEvent(ctx->st_d2h, ctx->ev_comp[sidx], 0);
        e = cudaMemcpyAsync(static_cast<char*>(o) + h0 * out_bytes, dout, hc * out_bytes, cudaMemcpyDeviceToHost, ctx->st_d2h);
        if (want_diag && e == cudaSuccess) {
            const size_t rb = size_t(hc) * L * 4;
            if (hdiag->row_max && e == cudaSuccess)
                e = cudaMemcpyAsync(hdiag->row_max + h0 * L, dd.row_max, rb, cudaMemcpyDeviceToHost, ctx->st_d2h);
            if (hdiag->ell && e == cudaSuccess)
                e = cudaMemcpyAsync(hdiag->ell + h0 * L, dd.ell, rb, cudaMemcpyDeviceToHost, ctx->st_d2h);
            if (hdiag->ell_tail && e == cudaSuccess)
                e = cudaMemcpyAsync(hdiag->ell_tail + h0 * L, dd.ell_tail, rb, cudaMemcpyDeviceToHost, ctx->st_d2h);
            if (hdiag->selected && e == cudaSuccess)
                e = cudaMemcpyAsync(hdiag->selected + h0 * p.N * p.k, dd.selected,
                                    size_t(hc) * p.N * p.k * 4, cudaMemcpyDeviceToHost, ctx->st_d2h);
        }
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_d2h[sidx], ctx->st_d2h);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H");
    }
    e = cudaStreamSynchronize(ctx->st_d2h);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st_comp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "host-path sync");
    ctx->launches = launches;
    if (flag) {
        e = cudaMemcpy(ctx->flag_host, flag, sizeof(int), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "non-finite check");
        if (*ctx->flag_host)  // engine.hpp:83-93, :368
            return fail(ctx, PISA_ERR_NUMERICAL_OVERFLOW, "non-finite output");
    }
    return PISA_OK;
}

// ---- the step entries with HOST buffers (synchronous; the C++ shim's
// compute_block_stats / query_block_means / select_topk_* / pisa_streaming /
// pisa_reference). Inputs bf16 dense [B][H][L][d]; desc strides are ignored.
namespace {
struct HostCall {
    pisa_ctx* ctx;
    pisa_attn_desc d;
    Plan p;
    size_t in_bytes = 0, nd = 0, dd = 0;
    pisa_status st = PISA_OK;
    HostCall(pisa_ctx* c, const pisa_attn_desc* desc) : ctx(c) {
        if (!c) {
            st = PISA_ERR_INVALID_DIMENSION;
            return;
        }
        if (!desc) {
            st = fail(c, PISA_ERR_INVALID_DIMENSION, "null descriptor");
            return;
        }
        d = *desc;
        dense_strides(d);
        if ((st = resolve(c, &d, &p)) != PISA_OK) return;
        st = host_streams(c);
        in_bytes = size_t(p.BH) * p.L * p.D * 2;
        nd = size_t(p.BH) * p.N * p.D * 4;
        dd = size_t(p.BH) * p.D * p.D * 4;
    }
    pisa_status finish(DevBufs& b, const char* where) {
        if (b.err != cudaSuccess) return cuda_fail(ctx, b.err, where);
        const cudaError_t e = cudaStreamSynchronize(ctx->st_comp);
        return e == cudaSuccess ? PISA_OK : cuda_fail(ctx, e, where);
    }
};

cudaError_t download(void* h, const void* dptr, size_t bytes, cudaError_t e) {
    if (e == cudaSuccess && h && dptr) e = cudaMemcpy(h, dptr, bytes, cudaMemcpyDeviceToHost);
    return e;
}
}  // namespace

pisa_status pisa_b200_block_stats_host(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* q,
                                       const void* k, const void* v, float* k_bar, float* v_hat,
                                       float* q_bar, float* h_bar) {
    HostCall c(ctx, desc);
    if (c.st != PISA_OK) return c.st;
    if (!k || !v || (!q && q_bar)) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null tensor pointer");
    DeviceGuard g(ctx->device);
    DevBufs b;
    void* dk = b.upload(k, c.in_bytes);
    void* dv = b.upload(v, c.in_bytes);
    void* dq = q ? b.upload(q, c.in_bytes) : dk;
    float* o[4] = {nullptr, nullptr, nullptr, nullptr};
    float* h[4] = {k_bar, v_hat, q_bar, h_bar};
    const size_t sz[4] = {c.nd, c.nd, c.nd, c.dd};
    for (int i = 0; i < 4; ++i)
        if (h[i]) o[i] = static_cast<float*>(b.alloc(sz[i]));
    if (b.err != cudaSuccess) return cuda_fail(ctx, b.err, "block_stats_host staging");
    pisa_status st = pisa_b200_block_stats(ctx, &c.d, dq, dk, dv, o[0], o[1], o[2], o[3], ctx->st_comp);
    if (st != PISA_OK) return st;
    if ((st = c.finish(b, "block_stats_host")) != PISA_OK) return st;
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 4; ++i) e = download(h[i], o[i], sz[i], e);
    return e == cudaSuccess ? PISA_OK : cuda_fail(ctx, e, "block_stats_host copy-out");
}

pisa_status pisa_b200_block_norms_host(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* k,
                                       const void* v, float* m) {
    HostCall c(ctx, desc);
    if (c.st != PISA_OK) return c.st;
    if (!k || !v || !m) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null pointer");
    DeviceGuard g(ctx->device);
    DevBufs b;
    void* dk = b.upload(k, c.in_bytes);
    void* dv = b.upload(v, c.in_bytes);
    float* dm = static_cast<float*>(b.alloc(size_t(c.p.BH) * c.p.N * 4));
    if (b.err != cudaSuccess) return cuda_fail(ctx, b.err, "block_norms_host staging");
    pisa_status st = pisa_b200_block_norms(ctx, &c.d, dk, dk, dv, dm, ctx->st_comp);
    if (st != PISA_OK) return st;
    if ((st = c.finish(b, "block_norms_host")) != PISA_OK) return st;
    const cudaError_t e = download(m, dm, size_t(c.p.BH) * c.p.N * 4, cudaSuccess);
    return e == cudaSuccess ? PISA_OK : cuda_fail(ctx, e, "block_norms_host copy-out");
}

pisa_status pisa_b200_select_host(pisa_ctx* ctx, const pisa_attn_desc* desc, const float* q_bar,
                                  const float* k_bar, const float* m, int32_t* selected) {
    HostCall c(ctx, desc);
    if (c.st != PISA_OK) return c.st;
    if (!q_bar || !k_bar || !selected) return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null pointer");
    DeviceGuard g(ctx->device);
    DevBufs b;
    const float* dq = static_cast<const float*>(b.upload(q_bar, c.nd));
    const float* dk = static_cast<const float*>(b.upload(k_bar, c.nd));
    const float* dm = m ? static_cast<const float*>(b.upload(m, size_t(c.p.BH) * c.p.N * 4)) : nullptr;
    const size_t sb = size_t(c.p.BH) * c.p.N * c.p.k * 4;
    int32_t* ds = static_cast<int32_t*>(b.alloc(sb));
    if (b.err != cudaSuccess) return cuda_fail(ctx, b.err, "select_host staging");
    pisa_status st = m ? pisa_b200_select_cov(ctx, &c.d, dq, dk, dm, ds, nullptr, ctx->st_comp)
                       : pisa_b200_select(ctx, &c.d, dq, dk, ds, nullptr, ctx->st_comp);
    if (st != PISA_OK) return st;
    if ((st = c.finish(b, "select_host")) != PISA_OK) return st;
    const cudaError_t e = download(selected, ds, sb, cudaSuccess);
    return e == cudaSuccess ? PISA_OK : cuda_fail(ctx, e, "select_host copy-out");
}

pisa_status pisa_b200_attention_host(pisa_ctx* ctx, const pisa_attn_desc* desc, const void* q,
                                     const void* k, const void* v, const int32_t* selected,
                                     const float* k_bar, const float* v_hat, const float* h_bar,
                                     void* o, const pisa_diag* hdiag) {
    HostCall c(ctx, desc);
    if (c.st != PISA_OK) return c.st;
    if (!q || !k || !v || !o || !selected || !k_bar || !v_hat || !h_bar)
        return fail(ctx, PISA_ERR_INVALID_DIMENSION, "null pointer");
    DeviceGuard g(ctx->device);
    DevBufs b;
    const Plan& p = c.p;
    void* dq = b.upload(q, c.in_bytes);
    void* dk = b.upload(k, c.in_bytes);
    void* dv = b.upload(v, c.in_bytes);
    const size_t sb = size_t(p.BH) * p.N * p.k * 4;
    const int32_t* ds = static_cast<const int32_t*>(b.upload(selected, sb));
    const float* dkb = static_cast<const float*>(b.upload(k_bar, c.nd));
    const float* dvh = static_cast<const float*>(b.upload(v_hat, c.nd));
    const float* dhb = static_cast<const float*>(b.upload(h_bar, c.dd));
    const size_t ob = size_t(p.BH) * p.L * p.D * (c.d.out_dtype == PISA_DTYPE_F32 ? 4 : 2);
    void* dout = b.alloc(ob);
    pisa_diag dd{};
    const size_t rb = size_t(p.BH) * p.L * 4;
    if (hdiag) {
        if (hdiag->row_max) dd.row_max = static_cast<float*>(b.alloc(rb));
        if (hdiag->ell) dd.ell = static_cast<float*>(b.alloc(rb));
        if (hdiag->ell_tail) dd.ell_tail = static_cast<float*>(b.alloc(rb));
    }
    if (b.err != cudaSuccess) return cuda_fail(ctx, b.err, "attention_host staging");
    pisa_status st = pisa_b200_attention(ctx, &c.d, dq, dk, dv, ds, dkb, dvh, dhb, dout, hdiag ? &dd : nullptr,
                                         ctx->st_comp);
    if (st != PISA_OK) return st;
    if ((st = c.finish(b, "attention_host")) != PISA_OK) return st;
    cudaError_t e = download(o, dout, ob, cudaSuccess);
    if (hdiag) {
        e = download(hdiag->row_max, dd.row_max, rb, e);
        e = download(hdiag->ell, dd.ell, rb, e);
        e = download(hdiag->ell_tail, dd.ell_tail, rb, e);
    }
    return e == cudaSuccess ? PISA_OK : cuda_fail(ctx, e, "attention_host copy-out");
}

pisa_status pisa_b200_selftest_mma(pisa_ctx* ctx, const void* a, const void* b, float* out,
                                   void* stream) {
    if (!ctx || !a || !b || !out) return PISA_ERR_INVALID_DIMENSION;
    DeviceGuard g(ctx->device);
    CUtensorMap ta, tb128, tb64;
    if (!make_3d_map(&ta, a, 128, 128, 1, 128) || !make_3d_map(&tb128, b, 128, 128, 1, 128) ||
        !make_3d_map(&tb64, b, 128, 128, 1, 64))
        return fail(ctx, PISA_ERR_CUDA, "TMA descriptor creation failed");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(out, 0, 4 * 128 * 128 * sizeof(float), s);
    if (e == cudaSuccess)
        e = launch_selftest_mma(ta, tb128, tb64, static_cast<const __nv_bfloat16*>(a), out, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "selftest launch");
    return PISA_OK;
}

}  // extern "C"
