// Reference-style caller compiled against the C++ shim (include/pisa_b200.hpp):
// the bodies are the reference's own call sequences (pisa_cli.cpp:157-158,
// test_engine.cpp:224, engine.hpp:437-464), only the namespace changes.
//
//   shim_demo in.bin out_dir H L d r
//
// in.bin: float32 [H][L][d] q, k, v. Writes to out_dir:
//   multihead_out.bin / multihead_plan.bin  pisa_multihead (float32 / int32)
//   steps_out.bin / steps_plan.bin           head 0, floored to L - L % 64 rows,
//                                            through the step functions
//   steps_stats.bin                          k_bar | v_hat | q_bar | h_bar (float64)
//   gen.bin                                  gen_gaussian<float>(42, 2, 64, 8, 1.0) q|k|v
// and prints "k num_blocks realized" on the first line, then one "<check> ok"
// line per passed check. Exit codes follow pisa_cli.cpp:844-851.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>

#include "pisa_b200.hpp"

using namespace pisa::b200;

template <class C>
void dump(const std::string& path, const C& c) {
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(c.data()), std::streamsize(c.size() * sizeof(c[0])));
}

int main(int argc, char** argv) {
    if (argc < 7) {
        std::cerr << "usage: shim_demo in.bin out_dir H L d r\n";
        return 2;
    }
    const std::string dir = argv[2];
    TensorBundle<float> b;
    b.num_heads = std::strtoul(argv[3], nullptr, 10);
    b.seq_len = std::strtoul(argv[4], nullptr, 10);
    b.head_dim = std::strtoul(argv[5], nullptr, 10);
    const double r = std::atof(argv[6]);
    const std::size_t n = b.total_elems(), d = b.head_dim;
    b.q.resize(n);
    b.k.resize(n);
    b.v.resize(n);
    std::ifstream in(argv[1], std::ios::binary);
    in.read(reinterpret_cast<char*>(b.q.data()), std::streamsize(n * 4));
    in.read(reinterpret_cast<char*>(b.k.data()), std::streamsize(n * 4));
    in.read(reinterpret_cast<char*>(b.v.data()), std::streamsize(n * 4));
    AttentionConfig cfg;
    cfg.block_size = 64;
    cfg.ragged = true;
    try {
        // ---- pisa_multihead (engine.hpp:408-470)
        const auto res = pisa_multihead(b, r, RouterOptions{}, PisaVariant::Hybrid, cfg, true);
        std::vector<float> out;
        std::vector<int32_t> plan;
        for (const auto& h : res.heads) out.insert(out.end(), h.output.data.begin(), h.output.data.end());
        for (const auto& p : res.plans)
            for (const auto& row : p.selected)
                for (std::size_t j : row) plan.push_back(int32_t(j));
        dump(dir + "/multihead_out.bin", out);
        dump(dir + "/multihead_plan.bin", plan);
        std::cout << res.k << " " << res.num_blocks << " " << res.sparsity_realized << "\n";

        // ---- the same forward split over "devices" (both on GPU 0 here): identical
        const auto res2 = pisa_multihead(b, r, RouterOptions{}, PisaVariant::Hybrid, cfg, true, std::vector<int>{0, 0});
        for (std::size_t h = 0; h < b.num_heads; ++h)
            if (res2.heads[h].output.data != res.heads[h].output.data || res2.plans[h].selected != res.plans[h].selected) {
                std::cerr << "multi-device result differs at head " << h << "\n";
                return 1;
            }
        std::cout << "multidevice ok\n";

        // ---- error mapping: a non-divisible length without the ragged extension
        {
            TensorBundle<float> bad = b;
            bad.seq_len = b.seq_len - 1;
            AttentionConfig strict = cfg;
            strict.ragged = false;
            try {
                pisa_multihead(bad, r, RouterOptions{}, PisaVariant::Hybrid, strict, true);
                std::cerr << "expected BlockDivisibility\n";
                return 1;
            } catch (const BlockDivisibility& e) {
                std::cout << "BlockDivisibility ok: " << e.what() << "\n";
            }
        }

        // ---- the step functions on head 0, floored to whole blocks
        // (engine.hpp:437-461: prepare -> global stats -> query means -> route -> stream)
        const std::size_t Lf = b.seq_len - b.seq_len % 64;
        const ConstView<float> qv(b.q.data(), Lf, d), kv(b.k.data(), Lf, d), vv(b.v.data(), Lf, d);
        BlockStatistics st = compute_block_stats(kv, vv, 64);
        compute_global_stats(st, SpectralMethod::Exact, false);
        const Matrix<double> qb = query_block_means(qv, 64);
        const auto sk = sparsity_to_k(r, st.num_blocks);
        const SelectionPlan sp = select_topk_plain(qb, st.k_bar, sk.k, cfg.resolved_scale(d));
        AttentionConfig strict = cfg;
        strict.ragged = false;
        const PisaOutput<float> po = pisa_streaming(qv, kv, vv, sp, st, strict);
        std::vector<int32_t> splan;
        for (const auto& row : sp.selected)
            for (std::size_t j : row) splan.push_back(int32_t(j));
        dump(dir + "/steps_out.bin", po.output.data);
        dump(dir + "/steps_plan.bin", splan);
        std::vector<double> stats;
        const Matrix<double>* parts[] = {&st.k_bar, &st.v_hat, &qb, &st.h_bar};
        for (const Matrix<double>* m : parts) stats.insert(stats.end(), m->data.begin(), m->data.end());
        dump(dir + "/steps_stats.bin", stats);
        // pisa_reference(Zeroth) on the same plan differs from Hybrid by the
        // first-order term only; diagnostics contract (test_engine.cpp:118-135)
        const PisaOutput<float> pz = pisa_reference(qv, kv, vv, sp, st, PisaVariant::Zeroth, strict);
        for (std::size_t t = 0; t < Lf; ++t)
            if (!(po.denom[t] > 0.0 && po.ell_tail[t] > 0.0 &&
                  std::abs(po.tail_mass[t] - 64.0 * po.ell_tail[t]) <= 1e-9 * po.tail_mass[t]) ||
                !(pz.denom[t] > 0.0)) {
                std::cerr << "diagnostics contract violated at row " << t << "\n";
                return 1;
            }
        std::cout << "steps ok\n";
        // covariance norms through compute_global_stats(.., compute_norms = true)
        compute_global_stats(st, SpectralMethod::Exact, true);
        if (!(st.m_max > 0.0)) {
            std::cerr << "norms missing\n";
            return 1;
        }
        const SelectionPlan cp = select_topk_covariance(qb, st.k_bar, st.m, 1e-6, sk.k, cfg.resolved_scale(d));
        cp.validate();
        std::cout << "covariance ok\n";
        // a plan that does not match the inputs (check_engine_inputs, engine.hpp:75-78)
        try {
            SelectionPlan wrong = sp;
            wrong.selected.pop_back();
            pisa_streaming(qv, kv, vv, wrong, st, strict);
            std::cerr << "expected InvalidDimension\n";
            return 1;
        } catch (const InvalidDimension&) {
            std::cout << "InvalidDimension ok\n";
        }

        // ---- NumericalOverflow (test_engine.cpp:296-308): V = 3e38 overflows
        {
            TensorBundle<float> big = b;
            for (auto& x : big.v) x = 3.0e38f;
            try {
                pisa_multihead(big, r, RouterOptions{}, PisaVariant::Hybrid, cfg, true);
                std::cerr << "expected NumericalOverflow from pisa_multihead\n";
                return 1;
            } catch (const NumericalOverflow& e) {
                if (e.kind() != ErrorKind::Invariant) return 1;
            }
            const ConstView<float> bigv(big.v.data(), Lf, d);
            try {
                pisa_streaming(qv, kv, bigv, sp, st, strict);
                std::cerr << "expected NumericalOverflow from pisa_streaming\n";
                return 1;
            } catch (const NumericalOverflow&) {
            }
            std::cout << "NumericalOverflow ok\n";
        }

        // ---- the reference's generators, bit-identical (test_generate.cpp:13-24)
        const auto g = gen_gaussian<float>(42, 2, 64, 8, 1.0);
        std::vector<float> gq(g.q);
        gq.insert(gq.end(), g.k.begin(), g.k.end());
        gq.insert(gq.end(), g.v.begin(), g.v.end());
        dump(dir + "/gen.bin", gq);
        try {
            gen_gaussian<float>(1, 1, 1, 1, 0.0);
            return 1;
        } catch (const DegenerateScale&) {
            std::cout << "gen ok\n";
        }
    } catch (const Error& e) {
        std::cerr << e.what() << "\n";
        return e.kind() == ErrorKind::Invariant ? 1 : 2;  // pisa_cli.cpp:844-851
    }
    return 0;
}
