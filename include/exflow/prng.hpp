// exflow/prng.hpp -- the reproducible random stream the reference's seeded
// algorithms are defined over (xoshiro256** state, splitmix64 seeding;
// reference contract: proj/include/exflow/rng.hpp:17-98). Same seeds produce
// the same draws, which keeps synthetic traces (proj/src/synth.cpp:40-51),
// random placements (proj/src/placement.cpp:504-526) and annealing restarts
// (:319-356) bit-identical to the reference. Pinned by
// tests/golden/rng_ref.json (generated from the reference header itself).
#pragma once

#include <cstdint>
#include <span>
#include <utility>
#include <vector>

namespace exflow {

namespace detail {
inline std::uint64_t mix64(std::uint64_t& counter) {
    counter += 0x9E3779B97F4A7C15ULL;
    std::uint64_t v = counter;
    v = (v ^ (v >> 30)) * 0xBF58476D1CE4E5B9ULL;
    v = (v ^ (v >> 27)) * 0x94D049BB133111EBULL;
    return v ^ (v >> 31);
}
constexpr std::uint64_t rol(std::uint64_t v, unsigned k) { return (v << k) | (v >> (64u - k)); }
}  // namespace detail

class Rng {
  public:
    explicit Rng(std::uint64_t seed) {
        std::uint64_t c = seed;
        a_ = detail::mix64(c);
        b_ = detail::mix64(c);
        c_ = detail::mix64(c);
        d_ = detail::mix64(c);
    }

    std::uint64_t next() {
        const std::uint64_t out = detail::rol(b_ * 5u, 7) * 9u;
        const std::uint64_t shifted = b_ << 17;
        c_ ^= a_;
        d_ ^= b_;
        b_ ^= c_;
        a_ ^= d_;
        c_ ^= shifted;
        d_ = detail::rol(d_, 45);
        return out;
    }

    // unbiased draw in [0, bound) by rejection below (2^64 mod bound)
    std::uint64_t below(std::uint64_t bound) {
        const std::uint64_t reject_under = (~bound + 1u) % bound;
        std::uint64_t v = next();
        while (v < reject_under) v = next();
        return v % bound;
    }
    int below_int(int bound) { return static_cast<int>(below(static_cast<std::uint64_t>(bound))); }

    // 53 random mantissa bits in [0, 1)
    double uniform01() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }

    static std::uint64_t splitmix64(std::uint64_t& state) { return detail::mix64(state); }

  private:
    std::uint64_t a_, b_, c_, d_;
};

inline std::uint64_t seed_stream(std::uint64_t seed, std::uint64_t stream) {
    std::uint64_t c = seed ^ ((stream + 1u) * 0xA0761D6478BD642FULL);
    return detail::mix64(c);
}

// Fisher-Yates from the back, one below(i) draw per position.
template <class T>
void shuffle(std::span<T> v, Rng& rng) {
    for (std::size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[rng.below(i)]);
}

inline std::vector<int> sample_without_replacement(int n, int k, Rng& rng) {
    std::vector<int> pool(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) pool[i] = i;
    std::vector<int> out;
    out.reserve(static_cast<std::size_t>(k));
    for (int i = 0; i < k; ++i) {
        std::swap(pool[i], pool[i + rng.below_int(n - i)]);
        out.push_back(pool[i]);
    }
    return out;
}

}  // namespace exflow
