// Seeded synthetic inputs for the BASELINE configs.  Host
// code; generated once per run outside every timed region.
//
// Generator: xoshiro256++ seeded through splitmix64, 53-bit uniforms and a
// Box-Muller normal that consumes two draws per value -- the same generator
// family as the reference (P/include/dsattn/rng.hpp:14-78), written here from
// the published algorithms.  Each (b,h) pair draws from its own substream so
// any subset of pairs can be regenerated independently (rng.hpp:62-66).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "dsa_b200.h"
#include "dsa_internal.h"

namespace dsa {
namespace {

class Xoshiro {
  public:
    explicit Xoshiro(uint64_t seed) {
        uint64_t x = seed;
        for (int i = 0; i < 4; ++i) s_[i] = mix(x);
    }
    uint64_t next() {
        const uint64_t out = rotl(s_[0] + s_[3], 23) + s_[0];
        const uint64_t t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rotl(s_[3], 45);
        return out;
    }
    double unit() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
    uint64_t below(uint64_t n) {  // unbiased, bitmask rejection
        if (n <= 1) return 0;
        const uint64_t m = ~uint64_t{0} >> __builtin_clzll(n - 1);
        uint64_t v;
        do v = next() & m;
        while (v >= n);
        return v;
    }
    double gauss() {
        double a;
        do a = unit();
        while (a <= 0.0);
        const double b = unit();
        return std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b);
    }

  private:
    static uint64_t mix(uint64_t& x) {
        uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    static uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
    uint64_t s_[4];
};

// Substream `stream` of `seed`, independent of the order streams are made in.
Xoshiro substream(uint64_t seed, uint64_t stream) {
    Xoshiro root(seed);
    return Xoshiro(root.next() ^ (0x9e3779b97f4a7c15ULL * (stream + 1)));
}

uint16_t to_bf16(double x) {  // round-to-nearest-even through float
    float f = static_cast<float>(x);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

void store(void* base, int32_t dtype, size_t idx, double x) {
    if (dtype == DSA_BF16) static_cast<uint16_t*>(base)[idx] = to_bf16(x);
    else static_cast<float*>(base)[idx] = static_cast<float>(x);
}

std::vector<double> unit_vector(Xoshiro& g, int64_t d) {
    std::vector<double> u(d);
    double n2 = 0.0;
    for (auto& x : u) {
        x = g.gauss();
        n2 += x * x;
    }
    const double inv = 1.0 / std::sqrt(n2);
    for (auto& x : u) x *= inv;
    return u;
}

void gen_pair(const dsa_config& c, uint64_t seed, int32_t planted_pm, int32_t band_w,
              int64_t pair, const std::vector<double>& u, size_t out_off, void* q, void* k,
              void* v) {
    const int64_t L = c.L, d = c.d;
    Xoshiro g = substream(seed, 1000 + static_cast<uint64_t>(pair));
    std::vector<double> Q(L * d), K(L * d), V(L * d);
    for (auto& x : Q) x = g.gauss();
    for (auto& x : K) x = g.gauss();
    for (auto& x : V) x = g.gauss();
    // planted global keys: partial Fisher-Yates over [0, L)
    const int64_t npl = (static_cast<int64_t>(planted_pm) * L + 500) / 1000;
    std::vector<int64_t> pool(L);
    for (int64_t j = 0; j < L; ++j) pool[j] = j;
    for (int64_t t = 0; t < npl; ++t) {
        const int64_t r = t + static_cast<int64_t>(g.below(static_cast<uint64_t>(L - t)));
        std::swap(pool[t], pool[r]);
        for (int64_t c2 = 0; c2 < d; ++c2) K[pool[t] * d + c2] += 3.0 * u[c2];
    }
    for (int64_t i = 0; i < L; ++i)
        for (int64_t c2 = 0; c2 < d; ++c2) Q[i * d + c2] += 0.5 * u[c2];
    // local band: rows in the same band_w window share a random unit vector
    // added to both q and k, a +1.0 score bias inside the window.
    if (band_w > 0) {
        const int64_t nw = (L + band_w - 1) / band_w;
        for (int64_t w = 0; w < nw; ++w) {
            std::vector<double> e = unit_vector(g, d);
            for (int64_t i = w * band_w; i < std::min<int64_t>(L, (w + 1) * band_w); ++i)
                for (int64_t c2 = 0; c2 < d; ++c2) {
                    Q[i * d + c2] += e[c2];
                    K[i * d + c2] += e[c2];
                }
        }
    }
    for (int64_t i = 0; i < L * d; ++i) {
        store(q, c.dtype, out_off + i, Q[i]);
        store(k, c.dtype, out_off + i, K[i]);
        store(v, c.dtype, out_off + i, V[i]);
    }
}

}  // namespace
}  // namespace dsa

extern "C" dsa_status dsa_generate(const dsa_config* cfg, uint64_t seed, int32_t planted_per_mille,
                                   int32_t band_width, int64_t pair0, int64_t npairs, void* q,
                                   void* k, void* v, float* p, int32_t threads) {
    using namespace dsa;
    return guard([&] {
        if (!cfg) throw Error(DSA_ERR_PARAM, "dsa_generate: null config");
        if (cfg->L < 1 || cfg->d < 1 || cfg->k < 1) throw Error(DSA_ERR_SHAPE, "dsa_generate: bad shape");
        if (planted_per_mille < 0 || planted_per_mille > 1000)
            throw Error(DSA_ERR_PARAM, "dsa_generate: planted_per_mille out of [0,1000]");
        Xoshiro shared = substream(seed, 0);
        const std::vector<double> u = unit_vector(shared, cfg->d);
        if (p) {
            Xoshiro gp = substream(seed, 1);
            const double sd = 1.0 / std::sqrt(static_cast<double>(cfg->k));
            for (int64_t i = 0; i < cfg->d * cfg->k; ++i) p[i] = static_cast<float>(sd * gp.gauss());
        }
        if (npairs <= 0) return;
        if (!q || !k || !v) throw Error(DSA_ERR_PARAM, "dsa_generate: null output");
        const int T = std::max<int>(1, std::min<int64_t>(threads > 0 ? threads : 1, npairs));
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                for (int64_t i = t; i < npairs; i += T)
                    gen_pair(*cfg, seed, planted_per_mille, band_width, pair0 + i, u,
                             static_cast<size_t>(i) * cfg->L * cfg->d, q, k, v);
            });
        for (auto& th : pool) th.join();
    });
}
