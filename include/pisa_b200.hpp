// pisa_b200.hpp -- header-only C++ shim with the reference's operator API
// (/root/reference/proj/include/pisa/*.hpp) over the C ABI in pisa_b200.h.
//
// Callers of the reference's hot path recompile unchanged against namespace
// pisa::b200:
//
//   auto res = pisa::b200::pisa_multihead(bundle, r, RouterOptions{}, PisaVariant::Hybrid,
//                                         cfg, /*use_streaming=*/true);    // engine.hpp:408-412
//
// The bundle stays in host memory as in the reference (TensorBundle<T>,
// bundle.hpp:28-51, T = float or double). Values are rounded to bf16 (RNE) for the
// GPU; outputs come back as T from the fp32 kernel output. The C ABI stages heads
// through device buffers with H2D / compute / D2H overlapped
// (pisa_b200_fwd_host). Failures rethrow the reference's error classes with the
// same ErrorKind (errors.hpp:10-94), so the CLI exit-code mapping is preserved.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "pisa_b200.h"

namespace pisa {
namespace b200 {

// ------------------------------------------------------------- errors (errors.hpp) --
enum class ErrorKind { Validation, Invariant, Io };

class Error : public std::runtime_error {
public:
    Error(ErrorKind kind, std::string msg) : std::runtime_error(std::move(msg)), kind_(kind) {}
    ErrorKind kind() const noexcept { return kind_; }

private:
    ErrorKind kind_;
};
struct InvalidDimension : Error {
    explicit InvalidDimension(const std::string& m) : Error(ErrorKind::Validation, m) {}
};
struct DegenerateScale : InvalidDimension {
    explicit DegenerateScale(const std::string& m) : InvalidDimension(m) {}
};
struct BlockDivisibility : Error {
    explicit BlockDivisibility(const std::string& m) : Error(ErrorKind::Validation, m) {}
};
struct InvalidSparsity : Error {
    explicit InvalidSparsity(const std::string& m) : Error(ErrorKind::Validation, m) {}
};
struct InvalidEpsilon : Error {
    explicit InvalidEpsilon(const std::string& m) : Error(ErrorKind::Validation, m) {}
};
struct EmptySelection : Error {
    explicit EmptySelection(const std::string& m) : Error(ErrorKind::Validation, m) {}
};
struct NumericalOverflow : Error {
    explicit NumericalOverflow(const std::string& m) : Error(ErrorKind::Invariant, m) {}
};
// No reference class: request outside the GPU path (e.g. BlockFirst, block_size != 64).
struct Unsupported : Error {
    explicit Unsupported(const std::string& m) : Error(ErrorKind::Validation, m) {}
};
struct CudaError : Error {
    explicit CudaError(const std::string& m) : Error(ErrorKind::Invariant, m) {}
};

inline void throw_status(pisa_status st, const pisa_ctx* ctx) {
    if (st == PISA_OK) return;
    const std::string msg = ctx ? pisa_b200_last_error(ctx) : "pisa_b200 call failed";
    switch (st) {
        case PISA_ERR_INVALID_DIMENSION: throw InvalidDimension(msg);
        case PISA_ERR_BLOCK_DIVISIBILITY: throw BlockDivisibility(msg);
        case PISA_ERR_INVALID_SPARSITY: throw InvalidSparsity(msg);
        case PISA_ERR_INVALID_EPSILON: throw InvalidEpsilon(msg);
        case PISA_ERR_EMPTY_SELECTION: throw EmptySelection(msg);
        case PISA_ERR_NUMERICAL_OVERFLOW: throw NumericalOverflow(msg);
        case PISA_ERR_DEGENERATE_SCALE: throw DegenerateScale(msg);
        case PISA_ERR_UNSUPPORTED: throw Unsupported(msg);
        default: throw CudaError(msg);
    }
}

// -------------------------------------------------- config (attention.hpp:17-49) --
enum class AccumDtype { F32, F64 };
enum class PisaVariant { SparseOnly, Zeroth, BlockFirst, Hybrid, GlobalCentroid };  // engine.hpp:30
enum class RouterStrategy { Plain, CovarianceAware };                               // router.hpp:16

struct AttentionConfig {
    std::size_t block_size = 64;
    std::size_t group_size = 8;
    double scale = 0.0;
    AccumDtype accum = AccumDtype::F64;
    bool deterministic = true;
    unsigned num_threads = 0;
    bool literal_phase3 = false;
    bool collect_phase_times = false;
    // Extension: accept L % block_size != 0 (the reference throws BlockDivisibility).
    bool ragged = false;

    double resolved_scale(std::size_t d) const { return scale > 0.0 ? scale : 1.0 / std::sqrt(double(d)); }
};

struct RouterOptions {  // engine.hpp:385-390
    RouterStrategy strategy = RouterStrategy::Plain;
    double epsilon = 1e-6;
    bool force_diagonal = false;
    bool row_level = false;
};

template <class T>
struct Matrix {  // matrix.hpp:9-28
    std::size_t rows = 0, cols = 0;
    std::vector<T> data;
    Matrix() = default;
    Matrix(std::size_t r, std::size_t c, T fill = T{}) : rows(r), cols(c), data(r * c, fill) {}
    T* row(std::size_t i) { return data.data() + i * cols; }
    const T* row(std::size_t i) const { return data.data() + i * cols; }
    T& operator()(std::size_t i, std::size_t j) { return data[i * cols + j]; }
    const T& operator()(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
};

template <class T>
struct ConstView {  // matrix.hpp:31-46: non-owning row-major [rows][cols]
    const T* ptr = nullptr;
    std::size_t rows = 0, cols = 0;
    ConstView() = default;
    ConstView(const T* p, std::size_t r, std::size_t c) : ptr(p), rows(r), cols(c) {}
    ConstView(const Matrix<T>& m) : ptr(m.data.data()), rows(m.rows), cols(m.cols) {}
    const T* row(std::size_t i) const { return ptr + i * cols; }
    const T& operator()(std::size_t i, std::size_t j) const { return ptr[i * cols + j]; }
};

template <class T>
struct TensorBundle {  // bundle.hpp:28-51, each tensor [num_heads][seq_len][head_dim]
    using value_type = T;
    std::size_t num_heads = 0, seq_len = 0, head_dim = 0;
    std::vector<T> q, k, v;
    std::size_t head_elems() const { return seq_len * head_dim; }
    std::size_t total_elems() const { return num_heads * head_elems(); }
    ConstView<T> q_head(std::size_t h) const { return {q.data() + h * head_elems(), seq_len, head_dim}; }
    ConstView<T> k_head(std::size_t h) const { return {k.data() + h * head_elems(), seq_len, head_dim}; }
    ConstView<T> v_head(std::size_t h) const { return {v.data() + h * head_elems(), seq_len, head_dim}; }
};

struct SelectionPlan {  // router.hpp:24-71
    std::size_t num_key_blocks = 0;
    std::size_t k = 0;
    RouterStrategy strategy = RouterStrategy::Plain;
    double epsilon = 0.0;
    std::vector<std::vector<std::size_t>> selected;
    std::size_t num_query_blocks() const { return selected.size(); }
    std::vector<std::size_t> unselected(std::size_t i) const {  // router.hpp:36-48
        std::vector<std::size_t> u;
        std::size_t p = 0;
        for (std::size_t j = 0; j < num_key_blocks; ++j) {
            if (p < selected[i].size() && selected[i][p] == j)
                ++p;
            else
                u.push_back(j);
        }
        return u;
    }
    void validate() const {  // router.hpp:50-70
        for (std::size_t i = 0; i < selected.size(); ++i) {
            const auto& s = selected[i];
            if (s.empty())
                throw EmptySelection("EmptySelection: query block " + std::to_string(i) + " selects no key blocks");
            if (s.size() != k)
                throw InvalidSparsity("InvalidSparsity: query block " + std::to_string(i) + " selects " +
                                      std::to_string(s.size()) + " blocks, expected k = " + std::to_string(k));
            for (std::size_t p = 0; p < s.size(); ++p)
                if (s[p] >= num_key_blocks || (p > 0 && s[p] <= s[p - 1]))
                    throw InvalidSparsity("InvalidSparsity: query block " + std::to_string(i) +
                                          " has out-of-range or non-ascending indices");
        }
    }
};

enum class SpectralMethod { Exact, PowerIteration };  // block_stats.hpp:15

// Prepare products (block_stats.hpp:21-37). On the GPU path k_bar / v_hat /
// h_bar come from the statistics kernel in fp32 (stored here as double) and
// H_bar is reduced on the device directly: the per-block matrices H_j are
// never materialised, so `h` stays empty (h_block() is unavailable). The
// block's K / V (bf16) are kept so compute_global_stats(.., compute_norms)
// can run the spectral-norm kernel on them.
struct BlockStatistics {
    std::size_t num_blocks = 0, block_size = 0, dim = 0;
    Matrix<double> k_bar, v_hat;
    std::vector<double> h;
    Matrix<double> h_bar;
    std::vector<double> m;
    double m_max = 0.0;
    std::vector<double> k_bar_global;
    bool global_ready = false;
    std::shared_ptr<const std::vector<uint16_t>> kv_bf16;  // K then V, bf16, for the norms
};

template <class T>
struct PisaOutput {  // engine.hpp:43-57
    Matrix<T> output;
    std::vector<double> denom, tail_mass, ell_tail, row_max;
    bool running_max_used = true;
    double exact_ms = 0.0, approx_ms = 0.0, normalize_ms = 0.0;
};

template <class T>
struct MultiheadResult {  // engine.hpp:392-403
    std::vector<PisaOutput<T>> heads;
    std::vector<SelectionPlan> plans;
    std::size_t k = 0;
    std::size_t num_blocks = 0;
    double sparsity_requested = 0.0;
    double sparsity_realized = 0.0;
    double prepare_ms = 0.0, select_ms = 0.0, attention_ms = 0.0;
};

struct SparsityResolution {
    std::size_t k = 0;
    double realized = 0.0;
};

inline SparsityResolution sparsity_to_k(double r, std::size_t n) {  // router.hpp:80-90
    int64_t k = 0;
    double realized = 0.0;
    const pisa_status st = pisa_b200_sparsity_to_k(r, int64_t(n), &k, &realized);
    if (st == PISA_ERR_INVALID_SPARSITY)
        throw InvalidSparsity("InvalidSparsity: sparsity must lie in [0, 1), got " + std::to_string(r));
    throw_status(st, nullptr);
    return {std::size_t(k), realized};
}

// ------------------------------------------------------------------- context --
// One pisa_ctx per device, owned by the calling thread (contexts are not shared
// across host threads concurrently).
class Context {
public:
    explicit Context(int device = 0) {
        const pisa_status st = pisa_b200_create(&ctx_, device);
        if (st != PISA_OK) throw CudaError("CudaError: pisa_b200_create failed");
    }
    ~Context() { pisa_b200_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    pisa_ctx* get() const { return ctx_; }
    static Context& thread_default(int device = 0) {
        thread_local std::unique_ptr<Context> c;
        if (!c) c.reset(new Context(device));
        return *c;
    }

private:
    pisa_ctx* ctx_ = nullptr;
};

namespace detail {
inline uint16_t to_bf16(float f) {  // round to nearest even
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return uint16_t(u >> 16);
    u += 0x7fffu + ((u >> 16) & 1u);
    return uint16_t(u >> 16);
}
}  // namespace detail

namespace detail {
// one [H][L][d] bundle (or one head) as a dense descriptor
inline pisa_attn_desc bundle_desc(std::size_t H, std::size_t L, std::size_t d, const AttentionConfig& cfg) {
    pisa_attn_desc desc{};
    desc.batch = 1;
    desc.heads = int64_t(H);
    desc.seq_len = int64_t(L);
    desc.head_dim = int64_t(d);
    for (int64_t* s : {desc.q_strides, desc.k_strides, desc.v_strides, desc.o_strides}) {
        s[0] = int64_t(H * L * d);
        s[1] = int64_t(L * d);
        s[2] = int64_t(d);
    }
    desc.block_size = int32_t(cfg.block_size);
    desc.group_size = int32_t(cfg.group_size);
    desc.scale = cfg.scale;
    desc.topk = 1;
    desc.variant = int32_t(PisaVariant::Hybrid);
    desc.ragged = cfg.ragged;
    desc.out_dtype = PISA_DTYPE_F32;
    desc.epsilon = 1e-6;
    return desc;
}

template <class T>
std::vector<uint16_t> bf16_rows(ConstView<T> x, std::size_t rows_padded = 0) {
    std::vector<uint16_t> out(std::max(rows_padded, x.rows) * x.cols, 0);
    for (std::size_t i = 0; i < x.rows * x.cols; ++i) out[i] = to_bf16(float(x.ptr[i]));
    return out;
}

// AttentionConfig::check (attention.hpp:39-48), with the ragged extension
inline void check_cfg(const AttentionConfig& cfg, std::size_t L) {
    if (cfg.block_size == 0 || cfg.group_size == 0)
        throw InvalidDimension("InvalidDimension: block_size and group_size must be >= 1");
    if (!cfg.ragged && L % cfg.block_size != 0)
        throw BlockDivisibility("BlockDivisibility: seq_len " + std::to_string(L) + " not divisible by block size " +
                                std::to_string(cfg.block_size));
}

// the GPU router's head dim: 64 or 128 (scores of zero-padded columns are unchanged)
inline std::size_t router_dim(std::size_t d) {
    if (d <= 64) return 64;
    if (d <= 128) return 128;
    throw Unsupported("Unsupported: the GPU router scores head dims up to 128");
}

// select_topk_plain / _covariance over the GPU router: key blocks are the
// rows of k_bar; query blocks are scored in chunks of num_key_blocks rows
// (the kernel scores square tiles), the last chunk zero-padded. Diagonal
// forcing applies to query blocks i < N only (router.hpp:146).
inline SelectionPlan select(ConstView<double> q_bar, ConstView<double> k_bar, const std::vector<double>* m,
                            double epsilon, std::size_t k, double scale, bool force_diagonal, Context& c) {
    const std::size_t n = k_bar.rows, nq = q_bar.rows;
    if (m && !(epsilon > 0.0))
        throw InvalidEpsilon("InvalidEpsilon: epsilon must be > 0, got " + std::to_string(epsilon));
    if (m && m->size() != n) throw InvalidDimension("InvalidDimension: M has wrong length");
    if (k == 0 || k > n)
        throw InvalidSparsity("InvalidSparsity: k must lie in [1, N], got " + std::to_string(k) + " for N = " +
                              std::to_string(n));
    if (q_bar.cols != k_bar.cols) throw InvalidDimension("InvalidDimension: q_bar/k_bar dim mismatch");
    const std::size_t dp = router_dim(k_bar.cols);
    AttentionConfig cfg;
    cfg.scale = scale;
    cfg.ragged = false;
    pisa_attn_desc desc = bundle_desc(1, n * 64, dp, cfg);
    desc.topk = int64_t(k);
    if (m) {
        desc.router = PISA_ROUTER_COVARIANCE;
        desc.epsilon = epsilon;
    }
    std::vector<float> kb(n * dp, 0.f), qb(n * dp), mf;
    for (std::size_t j = 0; j < n; ++j)
        for (std::size_t a = 0; a < k_bar.cols; ++a) kb[j * dp + a] = float(k_bar(j, a));
    if (m) mf.assign(m->begin(), m->end());
    SelectionPlan plan;
    plan.num_key_blocks = n;
    plan.k = k;
    plan.strategy = m ? RouterStrategy::CovarianceAware : RouterStrategy::Plain;
    plan.epsilon = m ? epsilon : 0.0;
    plan.selected.resize(nq);
    std::vector<int32_t> sel(n * k);
    for (std::size_t c0 = 0; c0 < nq; c0 += n) {
        const std::size_t rows = std::min(n, nq - c0);
        std::fill(qb.begin(), qb.end(), 0.f);
        for (std::size_t i = 0; i < rows; ++i)
            for (std::size_t a = 0; a < q_bar.cols; ++a) qb[i * dp + a] = float(q_bar(c0 + i, a));
        desc.force_diagonal = force_diagonal && c0 == 0;
        throw_status(pisa_b200_select_host(c.get(), &desc, qb.data(), kb.data(), m ? mf.data() : nullptr, sel.data()),
                     c.get());
        for (std::size_t i = 0; i < rows; ++i) plan.selected[c0 + i].assign(sel.begin() + i * k, sel.begin() + (i + 1) * k);
    }
    return plan;
}

// pisa_streaming / pisa_reference through the fused kernel with a given plan
// and statistics (check_engine_inputs, engine.hpp:61-80, first).
template <class T>
PisaOutput<T> attend(ConstView<T> q, ConstView<T> k, ConstView<T> v, const SelectionPlan& plan,
                     const BlockStatistics& stats, PisaVariant variant, bool literal, const AttentionConfig& cfg,
                     Context& c) {
    if (q.cols != k.cols || k.rows != v.rows || k.cols != v.cols)
        throw InvalidDimension("InvalidDimension: Q/K/V shapes do not form an attention instance");
    check_cfg(cfg, q.rows);
    check_cfg(cfg, k.rows);
    const std::size_t b = cfg.block_size, L = k.rows, d = k.cols;
    const std::size_t n = (L + b - 1) / b, nq = (q.rows + b - 1) / b;
    if (stats.block_size != b || stats.num_blocks != n || stats.dim != d)
        throw InvalidDimension("InvalidDimension: block statistics do not match inputs");
    if (plan.num_query_blocks() != nq || plan.num_key_blocks != stats.num_blocks)
        throw InvalidDimension("InvalidDimension: selection plan does not match inputs");
    plan.validate();
    if (variant == PisaVariant::BlockFirst) throw Unsupported("Unsupported: BlockFirst is not on the GPU path");
    if (variant != PisaVariant::SparseOnly && variant != PisaVariant::Zeroth && !stats.global_ready)
        throw InvalidDimension("InvalidDimension: global statistics required for this variant");
    if (q.rows > L) throw Unsupported("Unsupported: more query rows than key rows on the GPU path");
    // queries are self-attention rows on the GPU: a shorter Q is zero-padded to
    // L rows (the padding's plan rows repeat row 0; their outputs are dropped)
    pisa_attn_desc desc = bundle_desc(1, L, d, cfg);
    desc.topk = int64_t(plan.k);
    desc.variant = int32_t(variant);
    desc.literal_phase3 = literal;
    desc.check_finite = 1;
    std::vector<uint16_t> qh = bf16_rows(q, L), kh = bf16_rows(k), vh = bf16_rows(v);
    std::vector<int32_t> sel(n * plan.k);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t p = 0; p < plan.k; ++p) sel[i * plan.k + p] = int32_t(plan.selected[i < nq ? i : 0][p]);
    std::vector<float> kb(stats.k_bar.data.begin(), stats.k_bar.data.end()),
        vh32(stats.v_hat.data.begin(), stats.v_hat.data.end()), hb(d * d, 0.f);
    if (stats.h_bar.data.size() == d * d) std::copy(stats.h_bar.data.begin(), stats.h_bar.data.end(), hb.begin());
    std::vector<float> o(L * d), rm(L), ell(L), et(L);
    pisa_diag diag{rm.data(), ell.data(), et.data(), nullptr};
    const auto t0 = std::chrono::steady_clock::now();
    throw_status(pisa_b200_attention_host(c.get(), &desc, qh.data(), kh.data(), vh.data(), sel.data(), kb.data(),
                                          vh32.data(), hb.data(), o.data(), &diag),
                 c.get());
    PisaOutput<T> po;
    po.exact_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    po.output = Matrix<T>(q.rows, d);
    for (std::size_t i = 0; i < q.rows * d; ++i) po.output.data[i] = T(o[i]);
    po.denom.resize(q.rows);
    po.tail_mass.resize(q.rows);
    po.ell_tail.resize(q.rows);
    po.row_max.resize(q.rows);
    for (std::size_t t = 0; t < q.rows; ++t) {
        const double lift = std::exp(double(rm[t]));
        po.row_max[t] = rm[t];
        po.denom[t] = double(ell[t]) * lift;
        po.ell_tail[t] = double(et[t]) * lift;
        po.tail_mass[t] = double(b) * po.ell_tail[t];
    }
    return po;
}
}  // namespace detail

// ---------------------------------------- synthetic inputs (generate.hpp) --
// gen_gaussian / gen_clustered: bit-identical to the reference's generators
// (same xoshiro256++ stream, split over host threads by exact jumps).
template <class T>
TensorBundle<T> gen_gaussian(std::uint64_t seed, std::size_t heads, std::size_t L, std::size_t d, double std_dev) {
    static_assert(std::is_same<T, float>::value || std::is_same<T, double>::value, "T = float or double");
    TensorBundle<T> b;
    b.num_heads = heads;
    b.seq_len = L;
    b.head_dim = d;
    b.q.resize(heads * L * d);
    b.k.resize(heads * L * d);
    b.v.resize(heads * L * d);
    const pisa_status st = pisa_b200_gen_gaussian(seed, int64_t(heads), int64_t(L), int64_t(d), std_dev,
                                                  std::is_same<T, float>::value ? PISA_DTYPE_F32 : PISA_DTYPE_F64,
                                                  b.q.data(), b.k.data(), b.v.data(), 0);
    if (st == PISA_ERR_DEGENERATE_SCALE)
        throw DegenerateScale("DegenerateScale: std must be > 0, got " + std::to_string(std_dev));
    if (st != PISA_OK)
        throw InvalidDimension("InvalidDimension: heads, seq_len and head_dim must all be >= 1");
    return b;
}

template <class T>
TensorBundle<T> gen_clustered(std::uint64_t seed, std::size_t heads, std::size_t L, std::size_t d,
                              std::size_t n_clusters, double concentration, double noise_std) {
    static_assert(std::is_same<T, float>::value || std::is_same<T, double>::value, "T = float or double");
    TensorBundle<T> b;
    b.num_heads = heads;
    b.seq_len = L;
    b.head_dim = d;
    b.q.resize(heads * L * d);
    b.k.resize(heads * L * d);
    b.v.resize(heads * L * d);
    const pisa_status st = pisa_b200_gen_clustered(
        seed, int64_t(heads), int64_t(L), int64_t(d), int64_t(n_clusters), concentration, noise_std,
        std::is_same<T, float>::value ? PISA_DTYPE_F32 : PISA_DTYPE_F64, b.q.data(), b.k.data(), b.v.data(), 0);
    if (st == PISA_ERR_DEGENERATE_SCALE)
        throw DegenerateScale("DegenerateScale: noise_std must be >= 0, got " + std::to_string(noise_std));
    if (st != PISA_OK)
        throw InvalidDimension("InvalidDimension: dims must be >= 1 and n_clusters in [1, L]");
    return b;
}

// --------------------------------- prepare (block_stats.hpp:155-278) --
template <class T>
BlockStatistics compute_block_stats(ConstView<T> k, ConstView<T> v, std::size_t b, Context* ctx = nullptr) {
    Context& c = ctx ? *ctx : Context::thread_default();
    if (b == 0) throw InvalidDimension("InvalidDimension: block size must be >= 1");
    if (k.rows != v.rows || k.cols != v.cols) throw InvalidDimension("InvalidDimension: K and V shapes differ");
    if (k.rows % b != 0)
        throw BlockDivisibility("BlockDivisibility: seq_len " + std::to_string(k.rows) +
                                " not divisible by block size " + std::to_string(b));
    const std::size_t n = k.rows / b, d = k.cols;
    AttentionConfig cfg;
    cfg.block_size = b;
    pisa_attn_desc desc = detail::bundle_desc(1, k.rows, d, cfg);
    auto kv = std::make_shared<std::vector<uint16_t>>(detail::bf16_rows(k));
    const std::vector<uint16_t> vb = detail::bf16_rows(v);
    kv->insert(kv->end(), vb.begin(), vb.end());
    std::vector<float> kb(n * d), vh(n * d), hb(d * d);
    throw_status(pisa_b200_block_stats_host(c.get(), &desc, nullptr, kv->data(), kv->data() + k.rows * d, kb.data(),
                                            vh.data(), nullptr, hb.data()),
                 c.get());
    BlockStatistics st;
    st.num_blocks = n;
    st.block_size = b;
    st.dim = d;
    st.k_bar = Matrix<double>(n, d);
    st.v_hat = Matrix<double>(n, d);
    st.h_bar = Matrix<double>(d, d);
    std::copy(kb.begin(), kb.end(), st.k_bar.data.begin());
    std::copy(vh.begin(), vh.end(), st.v_hat.data.begin());
    std::copy(hb.begin(), hb.end(), st.h_bar.data.begin());
    st.kv_bf16 = kv;
    return st;
}

// compute_global_stats (block_stats.hpp:207-241): H_bar (already reduced on
// the device), k_bar_global, and with compute_norms the deviation norms M_j by
// the GPU's Lanczos kernel (the reference's `method` selects its CPU solver;
// both agree with the exact norm to < 2e-5 relative, tests/test_gpu.py).
inline BlockStatistics& compute_global_stats(BlockStatistics& st, SpectralMethod method = SpectralMethod::Exact,
                                             bool compute_norms = true, Context* ctx = nullptr) {
    (void)method;
    const std::size_t n = st.num_blocks, d = st.dim;
    if (n == 0 || st.k_bar.data.size() != n * d || st.h_bar.data.size() != d * d)
        throw InvalidDimension("InvalidDimension: block statistics not populated");
    st.k_bar_global.assign(d, 0.0);
    for (std::size_t j = 0; j < n; ++j)
        for (std::size_t a = 0; a < d; ++a) st.k_bar_global[a] += st.k_bar(j, a);
    for (double& x : st.k_bar_global) x /= double(n);
    st.m.assign(n, 0.0);
    st.m_max = 0.0;
    if (compute_norms) {
        if (!st.kv_bf16) throw InvalidDimension("InvalidDimension: block statistics carry no K/V for the norms");
        Context& c = ctx ? *ctx : Context::thread_default();
        AttentionConfig cfg;
        cfg.block_size = st.block_size;
        const std::size_t L = n * st.block_size;
        pisa_attn_desc desc = detail::bundle_desc(1, L, d, cfg);
        std::vector<float> m(n);
        throw_status(pisa_b200_block_norms_host(c.get(), &desc, st.kv_bf16->data(), st.kv_bf16->data() + L * d,
                                                m.data()),
                     c.get());
        for (std::size_t j = 0; j < n; ++j) {
            st.m[j] = m[j];
            st.m_max = std::max(st.m_max, st.m[j]);
        }
    }
    st.global_ready = true;
    return st;
}

template <class T>
Matrix<double> query_block_means(ConstView<T> q, std::size_t b, Context* ctx = nullptr) {
    Context& c = ctx ? *ctx : Context::thread_default();
    if (b == 0) throw InvalidDimension("InvalidDimension: block size must be >= 1");
    if (q.rows % b != 0)
        throw BlockDivisibility("BlockDivisibility: seq_len " + std::to_string(q.rows) +
                                " not divisible by block size " + std::to_string(b));
    const std::size_t n = q.rows / b, d = q.cols;
    AttentionConfig cfg;
    cfg.block_size = b;
    pisa_attn_desc desc = detail::bundle_desc(1, q.rows, d, cfg);
    const std::vector<uint16_t> qh = detail::bf16_rows(q);
    std::vector<float> qb(n * d);
    throw_status(
        pisa_b200_block_stats_host(c.get(), &desc, qh.data(), qh.data(), qh.data(), nullptr, nullptr, qb.data(), nullptr),
        c.get());
    Matrix<double> out(n, d);
    std::copy(qb.begin(), qb.end(), out.data.begin());
    return out;
}

// --------------------------------------------- select (router.hpp:126-193) --
inline SelectionPlan select_topk_plain(ConstView<double> q_bar, ConstView<double> k_bar, std::size_t k, double scale,
                                       bool force_diagonal = false, Context* ctx = nullptr) {
    return detail::select(q_bar, k_bar, nullptr, 0.0, k, scale, force_diagonal,
                          ctx ? *ctx : Context::thread_default());
}

inline SelectionPlan select_topk_covariance(ConstView<double> q_bar, ConstView<double> k_bar,
                                            const std::vector<double>& m, double epsilon, std::size_t k,
                                            double scale, bool force_diagonal = false, Context* ctx = nullptr) {
    return detail::select(q_bar, k_bar, &m, epsilon, k, scale, force_diagonal, ctx ? *ctx : Context::thread_default());
}

// ---------------------------------------------- attention (engine.hpp:103-383) --
template <class T>
PisaOutput<T> pisa_streaming(ConstView<T> q, ConstView<T> k, ConstView<T> v, const SelectionPlan& plan,
                             const BlockStatistics& stats, const AttentionConfig& cfg, Context* ctx = nullptr) {
    if (!stats.global_ready)
        throw InvalidDimension("InvalidDimension: global statistics required for the streaming path");
    return detail::attend(q, k, v, plan, stats, PisaVariant::Hybrid, cfg.literal_phase3, cfg,
                          ctx ? *ctx : Context::thread_default());
}

template <class T>
PisaOutput<T> pisa_reference(ConstView<T> q, ConstView<T> k, ConstView<T> v, const SelectionPlan& plan,
                             const BlockStatistics& stats, PisaVariant variant, const AttentionConfig& cfg,
                             Context* ctx = nullptr) {
    // no literal Phase 3 on the reference path (engine.hpp:194-209)
    return detail::attend(q, k, v, plan, stats, variant, false, cfg, ctx ? *ctx : Context::thread_default());
}

// ------------------------------------------- pisa_multihead (engine.hpp:408-470) --
namespace detail {
// heads [h0, h1) of the bundle through the host-buffer forward on one context
template <class T>
void multihead_range(const TensorBundle<T>& bundle, double r, const RouterOptions& router, PisaVariant variant,
                     const AttentionConfig& cfg, bool use_streaming, std::size_t h0, std::size_t h1, Context& c,
                     MultiheadResult<T>& res) {
    const std::size_t H = h1 - h0, L = bundle.seq_len, d = bundle.head_dim;
    pisa_attn_desc desc = bundle_desc(H, L, d, cfg);
    desc.topk = 0;
    desc.sparsity = r;
    desc.variant = int32_t(variant);
    desc.router = int32_t(router.strategy);
    desc.epsilon = router.epsilon;
    desc.row_level = router.row_level;
    desc.force_diagonal = router.force_diagonal;
    // literal Phase 3 only on the streaming path (engine.hpp:460, :345-346)
    desc.literal_phase3 = cfg.literal_phase3 && use_streaming && variant == PisaVariant::Hybrid;
    desc.check_finite = 1;  // check_output_finite (engine.hpp:221, :368)
    int64_t nb = 0, kk = 0;
    double scale = 0.0;
    throw_status(pisa_b200_resolve(&desc, &nb, &kk, &scale), c.get());
    const std::size_t n = H * L * d, off = h0 * L * d;
    std::vector<uint16_t> qh(n), kh(n), vh(n);
    for (std::size_t i = 0; i < n; ++i) {
        qh[i] = to_bf16(float(bundle.q[off + i]));
        kh[i] = to_bf16(float(bundle.k[off + i]));
        vh[i] = to_bf16(float(bundle.v[off + i]));
    }
    std::vector<float> o(n), rm(H * L), ell(H * L), et(H * L);
    std::vector<int32_t> sel(H * std::size_t(nb) * std::size_t(kk));
    pisa_diag diag{rm.data(), ell.data(), et.data(), sel.data()};
    const auto t0 = std::chrono::steady_clock::now();
    throw_status(pisa_b200_fwd_host(c.get(), &desc, qh.data(), kh.data(), vh.data(), o.data(), &diag), c.get());
    res.attention_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (std::size_t h = 0; h < H; ++h) {
        PisaOutput<T>& po = res.heads[h0 + h];
        po.output = Matrix<T>(L, d);
        for (std::size_t i = 0; i < L * d; ++i) po.output.data[i] = T(o[h * L * d + i]);
        po.denom.resize(L);
        po.tail_mass.resize(L);
        po.ell_tail.resize(L);
        po.row_max.resize(L);
        for (std::size_t t = 0; t < L; ++t) {
            const double m = rm[h * L + t], lift = std::exp(m);
            po.row_max[t] = m;
            po.denom[t] = double(ell[h * L + t]) * lift;
            po.ell_tail[t] = double(et[h * L + t]) * lift;
            po.tail_mass[t] = double(cfg.block_size) * po.ell_tail[t];
        }
        SelectionPlan& plan = res.plans[h0 + h];
        plan.num_key_blocks = std::size_t(nb);
        plan.k = std::size_t(kk);
        plan.strategy = router.strategy;
        plan.epsilon = router.strategy == RouterStrategy::CovarianceAware ? router.epsilon : 0.0;
        plan.selected.assign(std::size_t(nb), {});
        for (std::size_t i = 0; i < std::size_t(nb); ++i)
            for (std::size_t p = 0; p < std::size_t(kk); ++p)
                plan.selected[i].push_back(std::size_t(sel[(h * nb + i) * kk + p]));
    }
}

template <class T>
MultiheadResult<T> multihead_result(const TensorBundle<T>& bundle, double r, const AttentionConfig& cfg) {
    if (bundle.num_heads == 0 || bundle.seq_len == 0 || bundle.head_dim == 0)
        throw InvalidDimension("InvalidDimension: empty bundle");
    check_cfg(cfg, bundle.seq_len);
    const std::size_t n = (bundle.seq_len + cfg.block_size - 1) / cfg.block_size;
    const SparsityResolution sk = sparsity_to_k(r, n);
    MultiheadResult<T> res;
    res.k = sk.k;
    res.num_blocks = n;
    res.sparsity_requested = r;
    res.sparsity_realized = sk.realized;
    res.heads.resize(bundle.num_heads);
    res.plans.resize(bundle.num_heads);
    return res;
}
}  // namespace detail

// pisa_multihead (engine.hpp:408-470) on one GPU. All heads run in one
// stream-ordered K1 -> K2 -> K3 sequence per staged head chunk; use_streaming
// picks no different math (the streaming and reference formulations agree to
// 1e-10, test_engine.cpp:137-150) except that only the streaming Hybrid path
// honours cfg.literal_phase3. A non-finite output throws NumericalOverflow.
template <class T>
MultiheadResult<T> pisa_multihead(const TensorBundle<T>& bundle, double r, const RouterOptions& router,
                                  PisaVariant variant, const AttentionConfig& cfg, bool use_streaming = false,
                                  Context* ctx = nullptr) {
    if (router.row_level) throw Unsupported("Unsupported: row-level routing is not on the GPU path");
    MultiheadResult<T> res = detail::multihead_result(bundle, r, cfg);
    Context& c = ctx ? *ctx : Context::thread_default();
    detail::multihead_range(bundle, r, router, variant, cfg, use_streaming, 0, bundle.num_heads, c, res);
    return res;
}

// The same over several GPUs of one box: heads are independent
// (engine.hpp:432-468), so each device gets a contiguous head range and its own
// host thread and context; outputs land directly in the caller's result (the
// "gather" is each device's D2H copy). No collective runs. attention_ms is the
// slowest device's.
template <class T>
MultiheadResult<T> pisa_multihead(const TensorBundle<T>& bundle, double r, const RouterOptions& router,
                                  PisaVariant variant, const AttentionConfig& cfg, bool use_streaming,
                                  const std::vector<int>& devices) {
    if (router.row_level) throw Unsupported("Unsupported: row-level routing is not on the GPU path");
    if (devices.empty()) throw InvalidDimension("InvalidDimension: no devices");
    MultiheadResult<T> res = detail::multihead_result(bundle, r, cfg);
    const std::size_t H = bundle.num_heads, G = std::min(devices.size(), H);
    std::vector<MultiheadResult<T>> part(G);
    std::vector<std::exception_ptr> err(G);
    std::vector<std::thread> th;
    for (std::size_t g = 0; g < G; ++g) {
        part[g].heads.resize(H);
        part[g].plans.resize(H);
        th.emplace_back([&, g] {
            try {
                Context c(devices[g]);
                detail::multihead_range(bundle, r, router, variant, cfg, use_streaming, H * g / G, H * (g + 1) / G, c,
                                        part[g]);
            } catch (...) {
                err[g] = std::current_exception();
            }
        });
    }
    for (auto& t : th) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
    for (std::size_t g = 0; g < G; ++g) {
        for (std::size_t h = H * g / G; h < H * (g + 1) / G; ++h) {
            res.heads[h] = std::move(part[g].heads[h]);
            res.plans[h] = std::move(part[g].plans[h]);
        }
        res.attention_ms = std::max(res.attention_ms, part[g].attention_ms);
    }
    return res;
}

}  // namespace b200
}  // namespace pisa
