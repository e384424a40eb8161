// Driver that compiles the REFERENCE's own header-only PRNG
// (/root/reference/proj/include/exflow/rng.hpp, included in place, not copied)
// and prints golden draws as JSON. Built into oracle/_ref/ by
// tests/golden/make_rng_golden.py; the JSON it prints is committed as
// tests/golden/rng_ref.json. rng.hpp is the only reference file on the hot
// path that builds without Eigen.
#include "exflow/rng.hpp"

#include <cstdio>
#include <numeric>
#include <vector>

using exflow::Rng;

int main() {
    std::printf("{\n");
    {
        Rng r(42);
        std::printf("  \"rng42_next\": [");
        for (int i = 0; i < 8; ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)r.next());
        std::printf("],\n");
    }
    {
        Rng r(0);
        std::printf("  \"rng0_next\": [");
        for (int i = 0; i < 4; ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)r.next());
        std::printf("],\n");
    }
    std::printf("  \"seed_stream\": [");
    for (int s = 0; s < 6; ++s)
        std::printf("%s\"%llu\"", s ? ", " : "", (unsigned long long)exflow::seed_stream(7 * s, s));
    std::printf("],\n");
    {
        Rng r(123);
        std::printf("  \"rng123_below\": [");
        const unsigned long long bounds[] = {1, 2, 3, 7, 8, 64, 1000, 1ull << 40, 3000000019ull};
        for (int i = 0; i < 9; ++i) std::printf("%s%llu", i ? ", " : "", (unsigned long long)r.below(bounds[i]));
        std::printf("],\n");
    }
    {
        Rng r(9);
        std::printf("  \"rng9_uniform01\": [");
        for (int i = 0; i < 6; ++i) std::printf("%s%.17g", i ? ", " : "", r.uniform01());
        std::printf("],\n");
    }
    {
        Rng r(4242);
        std::vector<int> perm(32);
        std::iota(perm.begin(), perm.end(), 0);
        exflow::shuffle(std::span<int>(perm), r);
        std::printf("  \"shuffle32_seed4242\": [");
        for (int i = 0; i < 32; ++i) std::printf("%s%d", i ? ", " : "", perm[i]);
        std::printf("],\n");
    }
    {
        Rng r(5);
        auto picked = exflow::sample_without_replacement(30, 7, r);
        std::printf("  \"sample30_7_seed5\": [");
        for (int i = 0; i < 7; ++i) std::printf("%s%d", i ? ", " : "", picked[i]);
        std::printf("]\n");
    }
    std::printf("}\n");
    return 0;
}
