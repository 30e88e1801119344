// Reference-style caller compiled against the C++ shim (include/pisa_b200.hpp):
// the body is the reference's pisa_multihead call (pisa_cli.cpp:157-158 /
// test_engine.cpp:224), only the namespace changes. Reads a raw bundle
// (float32 [H][L][d] q, k, v) from argv[1], writes float32 outputs to argv[2]
// and the plan (int32) to argv[3]; prints "k num_blocks realized".
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>

#include "pisa_b200.hpp"

using namespace pisa::b200;

int main(int argc, char** argv) {
    if (argc < 7) {
        std::cerr << "usage: shim_demo in.bin out.bin plan.bin H L d [r]\n";
        return 2;
    }
    TensorBundle<float> b;
    b.num_heads = std::strtoul(argv[4], nullptr, 10);
    b.seq_len = std::strtoul(argv[5], nullptr, 10);
    b.head_dim = std::strtoul(argv[6], nullptr, 10);
    const double r = argc > 7 ? std::atof(argv[7]) : 0.875;
    const std::size_t n = b.num_heads * b.seq_len * b.head_dim;
    b.q.resize(n);
    b.k.resize(n);
    b.v.resize(n);
    std::ifstream in(argv[1], std::ios::binary);
    in.read(reinterpret_cast<char*>(b.q.data()), n * 4);
    in.read(reinterpret_cast<char*>(b.k.data()), n * 4);
    in.read(reinterpret_cast<char*>(b.v.data()), n * 4);
    AttentionConfig cfg;
    cfg.block_size = 64;
    cfg.ragged = true;
    try {
        const auto res = pisa_multihead(b, r, RouterOptions{}, PisaVariant::Hybrid, cfg, true);
        std::ofstream out(argv[2], std::ios::binary), plan(argv[3], std::ios::binary);
        for (const auto& h : res.heads)
            out.write(reinterpret_cast<const char*>(h.output.data.data()), h.output.data.size() * 4);
        for (const auto& p : res.plans)
            for (const auto& row : p.selected)
                for (std::size_t j : row) {
                    const int32_t x = int32_t(j);
                    plan.write(reinterpret_cast<const char*>(&x), 4);
                }
        std::cout << res.k << " " << res.num_blocks << " " << res.sparsity_realized << "\n";
        // error mapping: a non-divisible length without the ragged extension
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
    } catch (const Error& e) {
        std::cerr << e.what() << "\n";
        return e.kind() == ErrorKind::Invariant ? 1 : 2;  // pisa_cli.cpp:844-851
    }
    return 0;
}
