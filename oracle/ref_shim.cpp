// C-ABI shim over the UNMODIFIED reference library (header-only C++20), so tests
// and bench.py can call the reference itself through ctypes.
//
// TEST INFRASTRUCTURE ONLY: built by oracle/Makefile from the headers where they
// lie (/root/reference/proj/include, never copied) into oracle/_ref/. Used as the
// oracle's pin and as the timed CPU baseline (`bench.py --impl reference`).
//
// Every entry point calls the reference's public API: pisa::gen_gaussian,
// pisa::gen_clustered, pisa::compute_block_stats, pisa::compute_global_stats,
// pisa::query_block_means, pisa::select_topk_plain, pisa::pisa_streaming,
// pisa::pisa_reference, pisa::pisa_multihead, pisa::dense_online.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <variant>

#include "pisa/pisa.hpp"

namespace {

// Same numbering as include/pisa_b200.h.
int status_of(const std::exception& e) {
    if (dynamic_cast<const pisa::BlockDivisibility*>(&e)) return 2;
    if (dynamic_cast<const pisa::InvalidSparsity*>(&e)) return 3;
    if (dynamic_cast<const pisa::InvalidEpsilon*>(&e)) return 4;
    if (dynamic_cast<const pisa::EmptySelection*>(&e)) return 5;
    if (dynamic_cast<const pisa::NumericalOverflow*>(&e)) return 6;
    if (dynamic_cast<const pisa::DegenerateScale*>(&e)) return 7;
    if (dynamic_cast<const pisa::InvalidDimension*>(&e)) return 1;
    return 99;
}

pisa::AttentionConfig make_cfg(int64_t block, int64_t group, double scale, int accum_f64,
                               int literal_phase3, unsigned threads) {
    pisa::AttentionConfig cfg;
    cfg.block_size = std::size_t(block);
    cfg.group_size = std::size_t(group);
    cfg.scale = scale;
    cfg.accum = accum_f64 ? pisa::AccumDtype::F64 : pisa::AccumDtype::F32;
    cfg.literal_phase3 = literal_phase3 != 0;
    cfg.num_threads = threads;
    return cfg;
}

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

}  // namespace

extern "C" {

int ref_rng_u64(uint64_t seed, uint64_t* out, int64_t n) {
    pisa::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
    return 0;
}

int ref_rng_gaussian(uint64_t seed, double* out, int64_t n) {
    pisa::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.gaussian();
    return 0;
}

int ref_gen(int clustered, uint64_t seed, int64_t heads, int64_t L, int64_t d, double std_dev,
            int64_t n_clusters, double concentration, double noise_std, float* q, float* k,
            float* v) {
    return guarded([&] {
        pisa::TensorBundle<float> b =
            clustered ? pisa::gen_clustered<float>(seed, std::size_t(heads), std::size_t(L),
                                                   std::size_t(d), std::size_t(n_clusters),
                                                   concentration, noise_std)
                      : pisa::gen_gaussian<float>(seed, std::size_t(heads), std::size_t(L),
                                                  std::size_t(d), std_dev);
        std::memcpy(q, b.q.data(), b.q.size() * sizeof(float));
        std::memcpy(k, b.k.data(), b.k.size() * sizeof(float));
        std::memcpy(v, b.v.data(), b.v.size() * sizeof(float));
    });
}

int ref_sparsity_to_k(double r, int64_t n, int64_t* k, double* realized) {
    return guarded([&] {
        const auto res = pisa::sparsity_to_k(r, std::size_t(n));
        *k = int64_t(res.k);
        *realized = res.realized;
    });
}

// One head: prepare products (block_stats.hpp:155-278). Norms off, as in the
// Plain-router pisa_multihead path (engine.hpp:431,439).
int ref_block_stats(const float* q, const float* k, const float* v, int64_t L, int64_t d,
                    int64_t B, double* kbar, double* vhat, double* hbar, double* qbar,
                    double* kbar_global) {
    return guarded([&] {
        pisa::ConstView<float> kv(k, std::size_t(L), std::size_t(d));
        pisa::ConstView<float> vv(v, std::size_t(L), std::size_t(d));
        pisa::ConstView<float> qv(q, std::size_t(L), std::size_t(d));
        auto st = pisa::compute_block_stats(kv, vv, std::size_t(B));
        pisa::compute_global_stats(st, pisa::SpectralMethod::Exact, false);
        const auto qb = pisa::query_block_means(qv, std::size_t(B));
        std::memcpy(kbar, st.k_bar.data.data(), st.k_bar.data.size() * sizeof(double));
        std::memcpy(vhat, st.v_hat.data.data(), st.v_hat.data.size() * sizeof(double));
        std::memcpy(hbar, st.h_bar.data.data(), st.h_bar.data.size() * sizeof(double));
        std::memcpy(qbar, qb.data.data(), qb.data.size() * sizeof(double));
        if (kbar_global)
            std::memcpy(kbar_global, st.k_bar_global.data(), st.k_bar_global.size() * sizeof(double));
    });
}

int ref_select_plain(const double* qbar, const double* kbar, int64_t nq, int64_t n, int64_t d,
                     int64_t k, double scale, int force_diagonal, int32_t* selected) {
    return guarded([&] {
        pisa::ConstView<double> qb(qbar, std::size_t(nq), std::size_t(d));
        pisa::ConstView<double> kb(kbar, std::size_t(n), std::size_t(d));
        const auto plan = pisa::select_topk_plain(qb, kb, std::size_t(k), scale, force_diagonal != 0);
        for (int64_t i = 0; i < nq; ++i)
            for (int64_t p = 0; p < k; ++p) selected[i * k + p] = int32_t(plan.selected[i][p]);
    });
}

// Spectral deviation norms M_j = ||H_j - H_bar||_2 (compute_global_stats with
// compute_norms = true, block_stats.hpp:207-241, SpectralMethod::Exact as
// pisa_multihead uses it, engine.hpp:439). m: [N].
int ref_block_norms(const float* k, const float* v, int64_t L, int64_t d, int64_t B, double* m,
                    double* m_max) {
    return guarded([&] {
        pisa::ConstView<float> kv(k, std::size_t(L), std::size_t(d));
        pisa::ConstView<float> vv(v, std::size_t(L), std::size_t(d));
        auto st = pisa::compute_block_stats(kv, vv, std::size_t(B));
        pisa::compute_global_stats(st, pisa::SpectralMethod::Exact, true);
        std::memcpy(m, st.m.data(), st.m.size() * sizeof(double));
        if (m_max) *m_max = st.m_max;
    });
}

// select_topk_covariance (router.hpp:157-193).
int ref_select_cov(const double* qbar, const double* kbar, const double* m, int64_t nq, int64_t n,
                   int64_t d, int64_t k, double scale, double eps, int force_diagonal,
                   int32_t* selected) {
    return guarded([&] {
        pisa::ConstView<double> qb(qbar, std::size_t(nq), std::size_t(d));
        pisa::ConstView<double> kb(kbar, std::size_t(n), std::size_t(d));
        const std::vector<double> mv(m, m + n);
        const auto plan = pisa::select_topk_covariance(qb, kb, mv, eps, std::size_t(k), scale,
                                                       force_diagonal != 0);
        for (int64_t i = 0; i < nq; ++i)
            for (int64_t p = 0; p < k; ++p) selected[i * k + p] = int32_t(plan.selected[i][p]);
    });
}

// select_topk_rowmax (router.hpp:198-233) on float queries [L][d]; m may be NULL.
int ref_select_rowmax(const float* q, const double* kbar, const double* m, int64_t L, int64_t n,
                      int64_t d, int64_t B, int64_t k, double scale, double eps, int32_t* selected) {
    return guarded([&] {
        pisa::ConstView<float> qv(q, std::size_t(L), std::size_t(d));
        pisa::ConstView<double> kb(kbar, std::size_t(n), std::size_t(d));
        std::vector<double> mv;
        if (m) mv.assign(m, m + n);
        const auto plan = pisa::select_topk_rowmax<float>(qv, kb, std::size_t(B), std::size_t(k), scale,
                                                         m ? &mv : nullptr, eps);
        const int64_t nq = L / B;
        for (int64_t i = 0; i < nq; ++i)
            for (int64_t p = 0; p < k; ++p) selected[i * k + p] = int32_t(plan.selected[i][p]);
    });
}

// PQKV (io.hpp): write a bundle through the reference writer (dtype 1 = f32,
// 2 = f64; values given as doubles), and read one back: header fields and the
// payload converted to double. read status != 0 carries the reference's Io
// error class (status_of maps ErrorKind::Io to 3).
int ref_pqkv_write(const char* path, int dtype, const double* q, const double* k, const double* v,
                   int64_t H, int64_t L, int64_t d, int64_t* bytes) {
    return guarded([&] {
        const std::size_t n = std::size_t(H * L * d);
        auto fill = [&](auto& b) {
            b.num_heads = std::size_t(H);
            b.seq_len = std::size_t(L);
            b.head_dim = std::size_t(d);
            b.q.assign(q, q + n);
            b.k.assign(k, k + n);
            b.v.assign(v, v + n);
        };
        if (dtype == 1) {
            pisa::TensorBundle<float> b;
            fill(b);
            *bytes = int64_t(pisa::write_bundle_file(pisa::AnyBundle(b), path));
        } else {
            pisa::TensorBundle<double> b;
            fill(b);
            *bytes = int64_t(pisa::write_bundle_file(pisa::AnyBundle(b), path));
        }
    });
}

int ref_pqkv_read(const char* path, int64_t* shape_dtype, double* qkv, int64_t cap,
                  char* err, int64_t err_cap) {
    try {
        const auto any = pisa::read_bundle_file(path);
        std::visit([&](const auto& b) {
            shape_dtype[0] = int64_t(b.num_heads);
            shape_dtype[1] = int64_t(b.seq_len);
            shape_dtype[2] = int64_t(b.head_dim);
            shape_dtype[3] = int64_t(pisa::dtype_of<typename std::decay_t<decltype(b)>::value_type>());
            const std::size_t n = b.total_elems();
            if (int64_t(3 * n) <= cap)
                for (std::size_t i = 0; i < n; ++i) {
                    qkv[i] = double(b.q[i]);
                    qkv[n + i] = double(b.k[i]);
                    qkv[2 * n + i] = double(b.v[i]);
                }
        }, any);
        return 0;
    } catch (const std::exception& e) {
        if (err && err_cap > 0) {
            std::strncpy(err, e.what(), std::size_t(err_cap - 1));
            err[err_cap - 1] = 0;
        }
        return status_of(e);
    }
}

// flop_model (analysis.hpp:309-355): out = dense, sparse, pisa, sparse_ratio,
// pisa_ratio, overhead_ratio.
int ref_flop_model(int64_t L, int64_t d, int64_t b, int64_t k, int variant, double* out) {
    return guarded([&] {
        const auto r = pisa::flop_model(std::size_t(L), std::size_t(d), std::size_t(b), std::size_t(k),
                                        pisa::PisaVariant(variant));
        out[0] = r.dense_flops;
        out[1] = r.sparse_flops;
        out[2] = r.pisa_flops;
        out[3] = r.sparse_ratio;
        out[4] = r.pisa_ratio;
        out[5] = r.overhead_ratio;
    });
}

// theorem1_check + jensen_check (analysis.hpp:86-223) for one head with the
// Plain router at k selected blocks: plan out [N][k]; rows[5][L] = actual_err,
// bound, rho, alpha_sum, jensen_rhs; scal[6] = c_q, m_max, violations,
// jensen_violations, max_slack_ratio, jensen_check violations.
int ref_theorem1(const float* q, const float* k, const float* v, int64_t L, int64_t d, int64_t B,
                 int64_t ksel, int32_t* plan_out, double* rows, double* scal) {
    return guarded([&] {
        pisa::ConstView<float> qv(q, std::size_t(L), std::size_t(d));
        pisa::ConstView<float> kv(k, std::size_t(L), std::size_t(d));
        pisa::ConstView<float> vv(v, std::size_t(L), std::size_t(d));
        auto st = pisa::compute_block_stats(kv, vv, std::size_t(B));
        pisa::compute_global_stats(st, pisa::SpectralMethod::Exact, true);
        const auto qb = pisa::query_block_means(qv, std::size_t(B));
        pisa::AttentionConfig cfg;
        cfg.block_size = std::size_t(B);
        const double scale = cfg.resolved_scale(std::size_t(d));
        const auto plan = pisa::select_topk_plain(pisa::ConstView<double>(qb.data.data(), qb.rows, qb.cols),
                                                  pisa::ConstView<double>(st.k_bar.data.data(), st.k_bar.rows,
                                                                          st.k_bar.cols),
                                                  std::size_t(ksel), scale, false);
        const int64_t N = L / B;
        for (int64_t i = 0; i < N; ++i)
            for (int64_t p = 0; p < ksel; ++p) plan_out[i * ksel + p] = int32_t(plan.selected[i][p]);
        const auto rep = pisa::theorem1_check(qv, kv, vv, plan, st, cfg);
        for (int64_t t = 0; t < L; ++t) {
            rows[t] = rep.rows[t].actual_err;
            rows[L + t] = rep.rows[t].bound;
            rows[2 * L + t] = rep.rows[t].rho;
            rows[3 * L + t] = rep.rows[t].alpha_sum;
            rows[4 * L + t] = rep.rows[t].jensen_rhs;
        }
        scal[0] = rep.c_q;
        scal[1] = rep.m_max;
        scal[2] = double(rep.violations);
        scal[3] = double(rep.jensen_violations);
        scal[4] = rep.max_slack_ratio;
        scal[5] = double(pisa::jensen_check(qv, kv, plan, std::size_t(B), scale));
    });
}

// pisa_multihead (engine.hpp:408-470) on a [H][L][d] float bundle, Plain router.
// out: [H][L][d] float; selected: [H][N][k]; diagnostics [H][L] doubles
// (optional); times_ms[3] = prepare, select, attention (optional).
int ref_multihead(const float* q, const float* k, const float* v, int64_t H, int64_t L,
                  int64_t d, double r, int variant, int force_diagonal, int64_t block,
                  int64_t group, double scale, int accum_f64, int streaming, int literal_phase3,
                  unsigned threads, float* out, int32_t* selected, double* denom,
                  double* tail_mass, double* ell_tail, double* row_max, double* times_ms,
                  int64_t* k_out) {
    return guarded([&] {
        pisa::TensorBundle<float> b;
        b.num_heads = std::size_t(H);
        b.seq_len = std::size_t(L);
        b.head_dim = std::size_t(d);
        const std::size_t n = std::size_t(H * L * d);
        b.q.assign(q, q + n);
        b.k.assign(k, k + n);
        b.v.assign(v, v + n);
        const auto cfg = make_cfg(block, group, scale, accum_f64, literal_phase3, threads);
        // force_diagonal carries RouterOptions flags: bit 0 force_diagonal,
        // bit 1 CovarianceAware strategy, bit 2 row_level (epsilon stays 1e-6)
        pisa::RouterOptions router;
        router.force_diagonal = (force_diagonal & 1) != 0;
        if (force_diagonal & 2) router.strategy = pisa::RouterStrategy::CovarianceAware;
        router.row_level = (force_diagonal & 4) != 0;
        const auto res = pisa::pisa_multihead(b, r, router, pisa::PisaVariant(variant), cfg,
                                              streaming != 0);
        const std::size_t nb = res.num_blocks, kk = res.k;
        if (k_out) *k_out = int64_t(kk);
        for (std::size_t h = 0; h < std::size_t(H); ++h) {
            const auto& ho = res.heads[h];
            std::memcpy(out + h * L * d, ho.output.data.data(), std::size_t(L * d) * sizeof(float));
            if (selected)
                for (std::size_t i = 0; i < nb; ++i)
                    for (std::size_t p = 0; p < kk; ++p)
                        selected[(h * nb + i) * kk + p] = int32_t(res.plans[h].selected[i][p]);
            for (std::size_t t = 0; t < std::size_t(L); ++t) {
                if (denom) denom[h * L + t] = ho.denom[t];
                if (tail_mass) tail_mass[h * L + t] = ho.tail_mass[t];
                if (ell_tail) ell_tail[h * L + t] = ho.ell_tail[t];
                if (row_max) row_max[h * L + t] = ho.row_max[t];
            }
        }
        if (times_ms) {
            times_ms[0] = res.prepare_ms;
            times_ms[1] = res.select_ms;
            times_ms[2] = res.attention_ms;
        }
    });
}

// The cmd_bench hot path (pisa_cli.cpp:728-729) restricted to a contiguous range
// of query blocks [qb0, qb1) of one head, through the reference's public step
// functions: prepare over the full K/V, route the sampled query blocks, then
// pisa_streaming with accum F32. Used by bench.py --impl reference to time a
// bounded sample. ms[0] = prepare over the full head (compute_block_stats +
// compute_global_stats), ms[1] = query means + routing of the sampled blocks,
// ms[2] = pisa_streaming over the sampled blocks.
int ref_bench_sample(const float* q, const float* k, const float* v, int64_t L, int64_t d,
                     double r, int64_t qb0, int64_t qb1, unsigned threads, float* out,
                     double* ms) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        const auto since = [](clk::time_point t) {
            return std::chrono::duration<double, std::milli>(clk::now() - t).count();
        };
        auto t0 = clk::now();
        const auto cfg = make_cfg(64, 8, 0.0, 0, 0, threads);
        pisa::ConstView<float> kv(k, std::size_t(L), std::size_t(d));
        pisa::ConstView<float> vv(v, std::size_t(L), std::size_t(d));
        const std::size_t rows = std::size_t((qb1 - qb0) * 64);
        pisa::ConstView<float> qv(q + qb0 * 64 * d, rows, std::size_t(d));
        auto st = pisa::compute_block_stats(kv, vv, 64);
        pisa::compute_global_stats(st, pisa::SpectralMethod::Exact, false);
        ms[0] = since(t0);
        t0 = clk::now();
        const auto qb = pisa::query_block_means(qv, 64);
        const auto res = pisa::sparsity_to_k(r, st.num_blocks);
        const auto plan = pisa::select_topk_plain(qb, st.k_bar, res.k, cfg.resolved_scale(std::size_t(d)));
        ms[1] = since(t0);
        t0 = clk::now();
        const auto o = pisa::pisa_streaming(qv, kv, vv, plan, st, cfg);
        ms[2] = since(t0);
        std::memcpy(out, o.output.data.data(), o.output.data.size() * sizeof(float));
    });
}

// Parity of one head against the reference's own pipeline (engine.hpp:437-461):
// compute_block_stats + compute_global_stats(norms off) + query_block_means +
// select_topk_plain over the whole head -> the full plan (selected [N][k]) and
// the fp64 prepare products (q_bar / k_bar [N][d], for near-tie scoring); then
// pisa_streaming (accum F32 or F64) over `nsample` query blocks `blocks`
// (gathered into one query view with the matching sub-plan: query blocks are
// independent, engine.hpp:272) -> out [nsample*B][d] float.
// sub_plan (optional, [nsample][k]) replaces the reference's own plan rows of
// the sampled blocks, e.g. with the GPU's plan, so that the attention step is
// compared on identical selections (isolates attention error from
// near-tie selection swaps); SelectionPlan::validate still runs on it.
int ref_head_parity(const float* q, const float* k, const float* v, int64_t L, int64_t d, double r,
                    int force_diagonal, int64_t nsample, const int64_t* blocks, const int32_t* sub_plan,
                    int accum_f64, unsigned threads, int32_t* selected, double* qbar, double* kbar,
                    float* out) {
    return guarded([&] {
        const std::size_t B = 64;
        const auto cfg = make_cfg(int64_t(B), 8, 0.0, accum_f64, 0, threads);
        pisa::ConstView<float> qv(q, std::size_t(L), std::size_t(d));
        pisa::ConstView<float> kv(k, std::size_t(L), std::size_t(d));
        pisa::ConstView<float> vv(v, std::size_t(L), std::size_t(d));
        cfg.check(std::size_t(L));
        auto st = pisa::compute_block_stats(kv, vv, B);
        pisa::compute_global_stats(st, pisa::SpectralMethod::Exact, false);
        const auto qb = pisa::query_block_means(qv, B);
        const auto res = pisa::sparsity_to_k(r, st.num_blocks);
        const auto plan = pisa::select_topk_plain(qb, st.k_bar, res.k, cfg.resolved_scale(std::size_t(d)),
                                                  force_diagonal != 0);
        const std::size_t n = st.num_blocks, kk = res.k;
        for (std::size_t i = 0; i < n; ++i)
            for (std::size_t p = 0; p < kk; ++p) selected[i * kk + p] = int32_t(plan.selected[i][p]);
        if (qbar) std::memcpy(qbar, qb.data.data(), qb.data.size() * sizeof(double));
        if (kbar) std::memcpy(kbar, st.k_bar.data.data(), st.k_bar.data.size() * sizeof(double));
        if (nsample <= 0) return;
        std::vector<float> qs(std::size_t(nsample) * B * std::size_t(d));
        pisa::SelectionPlan sub;
        sub.num_key_blocks = n;
        sub.k = kk;
        for (int64_t s = 0; s < nsample; ++s) {
            const std::size_t i = std::size_t(blocks[s]);
            std::memcpy(qs.data() + std::size_t(s) * B * std::size_t(d), q + i * B * std::size_t(d),
                        B * std::size_t(d) * sizeof(float));
            if (sub_plan) {
                std::vector<std::size_t> row(kk);
                for (std::size_t p = 0; p < kk; ++p) row[p] = std::size_t(sub_plan[std::size_t(s) * kk + p]);
                sub.selected.push_back(std::move(row));
            } else {
                sub.selected.push_back(plan.selected[i]);
            }
        }
        pisa::ConstView<float> qsv(qs.data(), std::size_t(nsample) * B, std::size_t(d));
        const auto o = pisa::pisa_streaming(qsv, kv, vv, sub, st, cfg);
        std::memcpy(out, o.output.data.data(), o.output.data.size() * sizeof(float));
    });
}

int ref_dense_online(const float* q, const float* k, const float* v, int64_t L, int64_t d,
                     int accum_f64, unsigned threads, float* out) {
    return guarded([&] {
        const auto cfg = make_cfg(64, 8, 0.0, accum_f64, 0, threads);
        pisa::ConstView<float> qv(q, std::size_t(L), std::size_t(d));
        pisa::ConstView<float> kv(k, std::size_t(L), std::size_t(d));
        pisa::ConstView<float> vv(v, std::size_t(L), std::size_t(d));
        const auto o = pisa::dense_online(qv, kv, vv, cfg);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
    });
}

}  // extern "C"
