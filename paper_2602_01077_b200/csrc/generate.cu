// Synthetic Q/K/V exactly as the reference generates them (generate.hpp:29-116,
// rng.hpp:10-72): the measurement fixtures bench.py and the parity harness
// feed both the GPU path and the reference, so the two arms time and compare
// identical inputs. Host code (the generators are sequential by definition).
//
// The reference draws everything from ONE xoshiro256++ stream. The stream is
// split over host threads without changing a single draw: the xoshiro state
// transition is linear over GF(2), so a thread's start state is the seed state
// advanced by an exact jump (a product of precomputed T^(2^i) matrices), and
// each thread then runs the reference recurrence (Box-Muller in fp64 with the
// C library's log / sqrt / sin / cos) on its own range. Chunk boundaries are
// placed where the reference holds no spare Gaussian, so every value is
// bit-identical to a single-threaded run (tests/test_generate.py pins it to
// the reference library).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pisa_b200.h"

namespace {

// splitmix64 (rng.hpp:10-16)
uint64_t splitmix64_next(uint64_t& x) {
    x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

struct State {
    uint64_t s[4];
};

// xoshiro256++ with Box-Muller pairs (rng.hpp:24-72)
struct Rng {
    State st;
    bool have_spare = false;
    double spare = 0.0;
    explicit Rng(uint64_t seed) {
        uint64_t x = seed;
        for (auto& w : st.s) w = splitmix64_next(x);
    }
    explicit Rng(const State& s) : st(s) {}
    uint64_t next_u64() {
        uint64_t* s = st.s;
        const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return result;
    }
    double uniform01() { return double(next_u64() >> 11) * 0x1.0p-53; }
    uint64_t below(uint64_t n) { return next_u64() % n; }
    double gaussian() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        const double u1 = 1.0 - uniform01();
        const double u2 = uniform01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;  // std::numbers::pi
        spare = r * std::sin(theta);
        have_spare = true;
        return r * std::cos(theta);
    }
};

// ---- GF(2) jump: Jump[i] = T^(2^i) as 256 columns (the image of each state bit)
struct Mat {
    State col[256];
};

State apply(const Mat& m, const State& x) {
    State r{{0, 0, 0, 0}};
    for (int w = 0; w < 4; ++w) {
        uint64_t bits = x.s[w];
        while (bits) {
            const int b = __builtin_ctzll(bits);
            bits &= bits - 1;
            const State& c = m.col[w * 64 + b];
            for (int i = 0; i < 4; ++i) r.s[i] ^= c.s[i];
        }
    }
    return r;
}

const std::vector<Mat>& jump_table() {
    static std::vector<Mat> tab;
    static std::once_flag once;
    std::call_once(once, [] {
        tab.resize(64);
        for (int b = 0; b < 256; ++b) {  // T applied to each basis state
            Rng r(State{{0, 0, 0, 0}});
            r.st.s[b / 64] = 1ull << (b % 64);
            r.next_u64();
            tab[0].col[b] = r.st;
        }
        for (int i = 1; i < 64; ++i)
            for (int b = 0; b < 256; ++b) tab[size_t(i)].col[b] = apply(tab[size_t(i - 1)], tab[size_t(i - 1)].col[b]);
    });
    return tab;
}

// the state after `steps` next_u64 calls
State jump(State s, uint64_t steps) {
    const auto& tab = jump_table();
    for (int i = 0; i < 64 && steps; ++i, steps >>= 1)
        if (steps & 1) s = apply(tab[size_t(i)], s);
    return s;
}

uint16_t bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return uint16_t((u >> 16) | ((u & 0xffffu) ? 0x40u : 0u));
    u += 0x7fffu + ((u >> 16) & 1u);
    return uint16_t(u >> 16);
}

// writes T(x): T = double, T = float, or the RNE bf16 of the T = float value
struct Sink {
    void* p;
    int32_t dtype;
    void put(size_t i, double x) const {
        if (dtype == PISA_DTYPE_F64) {
            static_cast<double*>(p)[i] = x;
            return;
        }
        const float f = float(x);
        if (dtype == PISA_DTYPE_BF16)
            static_cast<uint16_t*>(p)[i] = bf16_rne(f);
        else
            static_cast<float*>(p)[i] = f;
    }
};

bool dtype_ok(int32_t t) { return t == PISA_DTYPE_BF16 || t == PISA_DTYPE_F32 || t == PISA_DTYPE_F64; }

int resolve_threads(int threads) {
    if (threads > 0) return threads;
    const unsigned hw = std::thread::hardware_concurrency();
    return int(std::max(1u, hw));
}

template <class Fn>
void run_threads(int n, Fn&& fn) {
    if (n <= 1) {
        fn(0);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(size_t(n));
    for (int t = 0; t < n; ++t) th.emplace_back([&, t] { fn(t); });
    for (auto& t : th) t.join();
}

}  // namespace

extern "C" {

pisa_status pisa_b200_gen_gaussian(uint64_t seed, int64_t heads, int64_t L, int64_t d, double std_dev,
                                   int32_t dtype, void* q, void* k, void* v, int threads) {
    if (heads < 1 || L < 1 || d < 1) return PISA_ERR_INVALID_DIMENSION;  // generate.hpp:18-24
    if (!(std_dev > 0.0)) return PISA_ERR_DEGENERATE_SCALE;               // generate.hpp:33-35
    if (!q || !k || !v || !dtype_ok(dtype)) return PISA_ERR_INVALID_DIMENSION;
    const size_t n = size_t(heads) * size_t(L) * size_t(d);
    const Sink sinks[3] = {{q, dtype}, {k, dtype}, {v, dtype}};
    // sample s of the concatenated Q|K|V sequence is half of Box-Muller pair
    // s / 2; pair p consumes draws 2p, 2p+1. Threads own whole pairs.
    const uint64_t samples = 3ull * n, pairs = (samples + 1) / 2;
    const Rng seeded(seed);
    const int nt = int(std::min<uint64_t>(uint64_t(resolve_threads(threads)), std::max<uint64_t>(1, pairs / 4096)));
    run_threads(nt, [&](int t) {
        const uint64_t p0 = pairs * uint64_t(t) / uint64_t(nt), p1 = pairs * uint64_t(t + 1) / uint64_t(nt);
        Rng r(jump(seeded.st, 2 * p0));
        for (uint64_t s = 2 * p0; s < std::min(2 * p1, samples); ++s) {
            const double g = std_dev * r.gaussian();  // generate.hpp:45-47
            sinks[s / n].put(size_t(s % n), g);
        }
    });
    return PISA_OK;
}

pisa_status pisa_b200_gen_clustered(uint64_t seed, int64_t heads, int64_t L, int64_t d, int64_t n_clusters,
                                    double concentration, double noise_std, int32_t dtype, void* q, void* k,
                                    void* v, int threads) {
    if (heads < 1 || L < 1 || d < 1) return PISA_ERR_INVALID_DIMENSION;  // generate.hpp:18-24
    if (n_clusters < 1 || n_clusters > L) return PISA_ERR_INVALID_DIMENSION;  // :65-70
    if (noise_std < 0.0) return PISA_ERR_DEGENERATE_SCALE;                     // :71-74
    if (!q || !k || !v || !dtype_ok(dtype)) return PISA_ERR_INVALID_DIMENSION;
    const Sink sq{q, dtype}, sk{k, dtype}, sv{v, dtype};
    const size_t nc = size_t(n_clusters), Ls = size_t(L), ds = size_t(d);
    const size_t run_len = (Ls + nc - 1) / nc;
    const size_t subset = std::max<size_t>(1, nc / 4);
    const size_t he = Ls * ds;
    // one head of generate.hpp:83-114 from the generator state `r`
    auto head = [&](Rng& r, size_t h) {
        std::vector<double> centers(nc * ds);
        for (double& c : centers) c = r.gaussian();
        std::vector<size_t> perm(nc);
        for (size_t i = 0; i < nc; ++i) perm[i] = i;
        for (size_t i = 0; i < subset; ++i) {
            const size_t j = i + size_t(r.below(nc - i));
            std::swap(perm[i], perm[j]);
        }
        for (size_t row = 0; row < Ls; ++row) {
            const size_t z = std::min(row / run_len, nc - 1);
            const double* c = centers.data() + z * ds;
            for (size_t a = 0; a < ds; ++a) sk.put(h * he + row * ds + a, c[a] + noise_std * r.gaussian());
        }
        for (size_t row = 0; row < Ls; ++row) {
            const size_t u = perm[size_t(r.below(subset))];
            const double* c = centers.data() + u * ds;
            for (size_t a = 0; a < ds; ++a) sq.put(h * he + row * ds + a, concentration * c[a] + r.gaussian());
        }
        for (size_t i = 0; i < he; ++i) sv.put(h * he + i, r.gaussian());
    };
    // With d even every head consumes a fixed number of draws and ends without a
    // spare Gaussian (each row's d Gaussians are whole pairs; below() draws one
    // u64 and leaves the spare alone), so head h starts at draw h * per_head.
    const bool even = ds % 2 == 0;
    const uint64_t per_head = uint64_t(nc * ds) + subset + uint64_t(he) + uint64_t(Ls) * (1 + ds) + uint64_t(he);
    const int nt = even ? int(std::min<int64_t>(resolve_threads(threads), heads)) : 1;
    const Rng seeded(seed);
    run_threads(nt, [&](int t) {
        const size_t h0 = size_t(heads) * size_t(t) / size_t(nt), h1 = size_t(heads) * size_t(t + 1) / size_t(nt);
        Rng r = nt == 1 ? seeded : Rng(jump(seeded.st, per_head * h0));
        for (size_t h = h0; h < h1; ++h) head(r, h);
    });
    return PISA_OK;
}

}  // extern "C"
