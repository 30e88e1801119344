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

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
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
struct TensorBundle {  // bundle.hpp:28-51, each tensor [num_heads][seq_len][head_dim]
    using value_type = T;
    std::size_t num_heads = 0, seq_len = 0, head_dim = 0;
    std::vector<T> q, k, v;
};

struct SelectionPlan {  // router.hpp:24-71
    std::size_t num_key_blocks = 0;
    std::size_t k = 0;
    RouterStrategy strategy = RouterStrategy::Plain;
    double epsilon = 0.0;
    std::vector<std::vector<std::size_t>> selected;
    std::size_t num_query_blocks() const { return selected.size(); }
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

// pisa_multihead (engine.hpp:408-470) on the GPU. All heads run in one
// stream-ordered K1 -> K2 -> K3 sequence; use_streaming picks no different math
// (the streaming and reference formulations agree to 1e-10, test_engine.cpp:137-150).
template <class T>
MultiheadResult<T> pisa_multihead(const TensorBundle<T>& bundle, double r,
                                  const RouterOptions& router, PisaVariant variant,
                                  const AttentionConfig& cfg, bool use_streaming = false,
                                  Context* ctx = nullptr) {
    (void)use_streaming;
    using clock = std::chrono::steady_clock;
    Context& c = ctx ? *ctx : Context::thread_default();
    const std::size_t H = bundle.num_heads, L = bundle.seq_len, d = bundle.head_dim;
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
    desc.sparsity = r;
    desc.variant = int32_t(variant);
    desc.router = int32_t(router.strategy);
    desc.epsilon = router.epsilon;
    desc.row_level = router.row_level;
    desc.force_diagonal = router.force_diagonal;
    desc.literal_phase3 = cfg.literal_phase3;
    desc.ragged = cfg.ragged;
    desc.out_dtype = PISA_DTYPE_F32;
    desc.check_finite = 1;
    if (router.row_level) throw Unsupported("Unsupported: row-level routing is not on the GPU path");
    int64_t nb = 0, kk = 0;
    double scale = 0.0;
    throw_status(pisa_b200_resolve(&desc, &nb, &kk, &scale), c.get());

    const std::size_t n = H * L * d;
    std::vector<uint16_t> qh(n), kh(n), vh(n);
    for (std::size_t i = 0; i < n; ++i) {
        qh[i] = detail::to_bf16(float(bundle.q[i]));
        kh[i] = detail::to_bf16(float(bundle.k[i]));
        vh[i] = detail::to_bf16(float(bundle.v[i]));
    }
    std::vector<float> o(n), rm(H * L), ell(H * L), et(H * L);
    std::vector<int32_t> sel(H * std::size_t(nb) * std::size_t(kk));
    pisa_diag diag{rm.data(), ell.data(), et.data(), sel.data()};
    const auto t0 = clock::now();
    throw_status(pisa_b200_fwd_host(c.get(), &desc, qh.data(), kh.data(), vh.data(), o.data(), &diag),
                 c.get());
    const double ms = std::chrono::duration<double, std::milli>(clock::now() - t0).count();

    MultiheadResult<T> res;
    res.k = std::size_t(kk);
    res.num_blocks = std::size_t(nb);
    res.sparsity_requested = r;
    res.sparsity_realized = double(nb - kk) / double(nb);
    res.attention_ms = ms;
    for (std::size_t h = 0; h < H; ++h) {
        PisaOutput<T> po;
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
        res.heads.push_back(std::move(po));
        SelectionPlan plan;
        plan.num_key_blocks = std::size_t(nb);
        plan.k = std::size_t(kk);
        plan.selected.resize(std::size_t(nb));
        for (std::size_t i = 0; i < std::size_t(nb); ++i)
            for (std::size_t p = 0; p < std::size_t(kk); ++p)
                plan.selected[i].push_back(std::size_t(sel[(h * nb + i) * kk + p]));
        res.plans.push_back(std::move(plan));
    }
    return res;
}

}  // namespace b200
}  // namespace pisa
