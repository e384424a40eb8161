// test_mirror.cpp -- the reference's own known-answer tests run through the
// C++ mirror (include/exflow/exflow.hpp) linked against libexflow_b200.so,
// the way a reference caller (proj/tools/exflow.cpp, proj/tests/*.cpp) would
// use this library after switching over. doctest is not available here, so
// a tiny CHECK harness counts failures.
//
//   test_mirror host   -- no device work: trace/placement I/O, token_hops,
//                         placement table, solver, error types and messages
//   test_mirror gpu    -- count_transitions and simulate (GPU kernels)
//
// KAT sources: proj/tests/test_trace.cpp:46-119, proj/tests/test_sim.cpp:
// 44-117, proj/tests/test_placement.cpp:56-112 and the proj/data fixtures
// (copied to tests/golden/).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "exflow/exflow.hpp"

using namespace exflow;

static int g_checks = 0, g_fails = 0;

#define CHECK(cond)                                                                  \
    do {                                                                             \
        ++g_checks;                                                                  \
        if (!(cond)) {                                                               \
            ++g_fails;                                                               \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);              \
        }                                                                            \
    } while (0)

// expects `fn` to throw exactly type E whose message contains `part`
template <class E>
static void check_throws(const char* what, const std::function<void()>& fn, const std::string& part) {
    ++g_checks;
    try {
        fn();
    } catch (const E& e) {
        if (std::string(e.what()).find(part) != std::string::npos) return;
        ++g_fails;
        std::printf("FAIL %s: message '%s' lacks '%s'\n", what, e.what(), part.c_str());
        return;
    } catch (const std::exception& e) {
        ++g_fails;
        std::printf("FAIL %s: wrong exception type (%s)\n", what, e.what());
        return;
    }
    ++g_fails;
    std::printf("FAIL %s: no exception\n", what);
}

static RoutingTrace trace_from_paths(int E, const std::vector<std::vector<int>>& paths) {
    RoutingTrace t;
    t.num_experts = E;
    t.num_layers = static_cast<int>(paths.front().size());
    t.paths.resize(static_cast<int>(paths.size()), t.num_layers);
    for (size_t i = 0; i < paths.size(); ++i)
        for (size_t j = 0; j < paths[i].size(); ++j) t.paths(i, j) = paths[i][j];
    return t;
}

static Topology one_node(int gpus) {
    Topology t;
    t.num_nodes = 1;
    t.gpus_per_node = gpus;
    return t;
}

static int total_hops(const std::vector<LayerHop>& h) {
    int s = 0;
    for (const auto& x : h) s += x.hops;
    return s;
}

static TransitionCounts counts_of(const std::vector<CountMatrix>& ms) {
    TransitionCounts c;
    c.num_experts = static_cast<int>(ms[0].rows());
    c.num_layers = static_cast<int>(ms.size()) + 1;
    c.gap = 1;
    for (const auto& m : ms) {
        c.matrices.push_back(m);
        c.row_totals.push_back(m.rowwise_sum());
    }
    return c;
}

static CountMatrix m2(long a, long b, long c, long d) {
    CountMatrix m(2, 2);
    m(0, 0) = a;
    m(0, 1) = b;
    m(1, 0) = c;
    m(1, 1) = d;
    return m;
}

static void host_tests(const std::string& golden) {
    // ---- parse_trace (proj/tests/test_trace.cpp:46-85)
    {
        const RoutingTrace t = parse_trace(std::string("EXFLOW-TRACE v1\nE 2 L 2\n0 0\n1 1\n"));
        CHECK(t.num_experts == 2 && t.num_layers == 2 && t.num_tokens() == 2);
        CHECK(t.paths(0, 0) == 0 && t.paths(1, 1) == 1);
    }
    check_throws<ParseError>("out-of-range id", [] { parse_trace(std::string("EXFLOW-TRACE v1\nE 2 L 2\n0 0\n0 2\n")); },
                             "expert id 2 out of range [0,2) at line 4");
    check_throws<ParseError>("short path", [] { parse_trace(std::string("EXFLOW-TRACE v1\nE 2 L 2\n0\n")); },
                             "path length 1 != L=2");
    {
        const RoutingTrace t =
            parse_trace(std::string("# preamble\nEXFLOW-TRACE v1\n# dims\nE 3 L 2\n\n0 2\n# done\n1 1\n"));
        CHECK(t.num_tokens() == 2 && t.paths(0, 1) == 2);
    }
    check_throws<ParseError>("bad header", [] { parse_trace(std::string("bogus\n")); }, "");
    check_throws<ParseError>("E 0", [] { parse_trace(std::string("EXFLOW-TRACE v1\nE 0 L 2\n")); }, "E must be >= 1");
    check_throws<ParseError>("L 1", [] { parse_trace(std::string("EXFLOW-TRACE v1\nE 2 L 1\n0\n")); }, "L must be >= 2");
    check_throws<ParseError>("no paths", [] { parse_trace(std::string("EXFLOW-TRACE v1\nE 2 L 2\n")); },
                             "no token paths");
    check_throws<ParseError>("bad token", [] { parse_trace(std::string("EXFLOW-TRACE v1\nE 2 L 2\n0 x\n")); },
                             "invalid token 'x' at line 3");
    {  // serialize then parse (proj/tests/test_trace.cpp:87-94)
        Rng rng(7);
        RoutingTrace t;
        t.num_experts = 5;
        t.num_layers = 3;
        t.paths.resize(40, 3);
        for (int i = 0; i < 40; ++i)
            for (int j = 0; j < 3; ++j) t.paths(i, j) = rng.below_int(5);
        const RoutingTrace p = parse_trace(serialize_trace(t));
        CHECK(p.num_experts == 5 && p.num_layers == 3 && p.paths == t.paths);
    }
    {  // count_transitions gap checks happen before any device work
        const RoutingTrace t = trace_from_paths(2, {{0, 1}});
        check_throws<std::invalid_argument>("gap 2", [&] { count_transitions(t, 2); }, "gap 2 out of range [1,1]");
        check_throws<std::invalid_argument>("gap 0", [&] { count_transitions(t, 0); }, "out of range");
    }
    {  // conditional probabilities / most_affiliated on hand counts (test_trace.cpp:121-145)
        const TransitionCounts c = counts_of({m2(2, 1, 0, 1)});
        const AffinityMatrix a = conditional_probabilities(c);
        CHECK(std::fabs(a.matrices[0](0, 0) - 2.0 / 3.0) < 1e-15);
        CHECK(std::fabs(a.matrices[0](0, 1) - 1.0 / 3.0) < 1e-15);
        CHECK(a.matrices[0](1, 1) == 1.0);
        CHECK(most_affiliated(a, 0, 0) == 0 && most_affiliated(a, 0, 1) == 1);
        CHECK(export_heatmap_csv(a, 0).find("0.666667,0.333333") != std::string::npos);
    }
    // ---- fixtures (proj/data/two_token_demo.*)
    const RoutingTrace demo = load_trace(golden + "/two_token_demo.trace");
    CHECK(demo.num_experts == 8 && demo.num_layers == 3 && demo.num_tokens() == 2);
    CHECK(demo.paths(0, 1) == 4 && demo.paths(1, 2) == 4);
    const Placement demo_pl = load_placement(golden + "/two_token_demo_placement.json");
    CHECK(demo_pl.num_experts == 8 && demo_pl.gpus_per_node == 4 && demo_pl.assign(2, 5) == 2);
    CHECK(placement_from_json(placement_to_json(demo_pl)).assign == demo_pl.assign);
    // ---- token_hops (proj/tests/test_sim.cpp:44-73)
    const Topology t4 = one_node(4);
    const Placement cont = contiguous_placement(8, 3, t4);
    CHECK(cont.assign == demo_pl.assign);
    for (int e = 0; e < 8; ++e) CHECK(cont.assign(1, e) == e / 2);
    const std::vector<std::int32_t> first{0, 4, 2}, second{5, 5, 4}, home_path{2, 3, 2};
    CHECK(total_hops(token_hops(first, 1, cont, SimMode::vanilla, t4)) == 4);
    CHECK(total_hops(token_hops(first, 1, cont, SimMode::coherent, t4)) == 3);
    CHECK(total_hops(token_hops(second, 3, cont, SimMode::vanilla, t4)) == 6);
    CHECK(total_hops(token_hops(second, 3, cont, SimMode::coherent, t4)) == 1);
    CHECK(total_hops(token_hops(home_path, 1, cont, SimMode::vanilla, t4)) == 0);
    CHECK(total_hops(token_hops(home_path, 1, cont, SimMode::coherent, t4)) == 0);
    {
        const auto h = token_hops(first, 1, cont, SimMode::coherent, t4);
        CHECK(h[0].crossed && h[0].tier == Tier::intra_node && h[2].crossed);
    }
    const std::vector<std::int32_t> short_path{0, 4};
    check_throws<std::invalid_argument>("short path hops",
                                        [&] { token_hops(short_path, 1, cont, SimMode::vanilla, t4); }, "");
    check_throws<std::invalid_argument>("home 4", [&] { token_hops(first, 4, cont, SimMode::vanilla, t4); },
                                        "home gpu out of range");
    // ---- placement table validation messages (proj/src/placement.cpp:434-470)
    {
        Placement bad = cont;
        bad.assign(1, 3) = 9;
        check_throws<std::invalid_argument>("gpu id", [&] { bad.validate(); }, "gpu id 9 out of range [0,4) at layer 1");
        bad.assign(1, 3) = 0;
        check_throws<std::invalid_argument>("balance", [&] { bad.validate(); },
                                            "layer 1 places 3 experts on gpu 0, expected 2");
    }
    // ---- solver (proj/tests/test_placement.cpp:56-112)
    {
        auto [p, r] = solve_exact_dp(counts_of({m2(10, 0, 0, 10)}), 2);
        CHECK(r.objective == 0.0 && r.solver == "exact-dp");
        CHECK(p.assign(0, 0) == p.assign(1, 0) && p.assign(0, 1) == p.assign(1, 1));
    }
    {
        auto [p, r] = solve_exact_dp(counts_of({m2(0, 10, 10, 0)}), 2);
        CHECK(r.objective == 0.0);
        CHECK(p.assign(0, 0) == p.assign(1, 1) && p.assign(0, 1) == p.assign(1, 0));
    }
    {
        std::vector<CountMatrix> ones(2, CountMatrix(4, 4, 1));
        auto [p, r] = solve_exact_dp(counts_of(ones), 2);
        CHECK(r.objective == 16.0);
    }
    CHECK(balanced_assignment_count(8, 2, kDefaultStateCap) == 70);
    CHECK(balanced_assignment_count(16, 2, kDefaultStateCap) == kDefaultStateCap + 1);
    CHECK(balanced_assignment_count(4, 4, kDefaultStateCap) == 24);
    CHECK(balanced_assignment_count(4, 1, kDefaultStateCap) == 1);
    {
        std::vector<CountMatrix> big(1, CountMatrix(16, 16, 3));
        check_throws<std::invalid_argument>("state cap", [&] { solve_exact_dp(counts_of(big), 2); },
                                            "local-search");
        std::vector<CountMatrix> three(1, CountMatrix(3, 3, 1));
        check_throws<std::invalid_argument>("not divisible", [&] { solve_exact_dp(counts_of(three), 2); },
                                            "not divisible by partitions 2");
    }
    {  // planted chain: staged solve on one node recovers zero crossings
        SynthConfig c;
        c.num_experts = 8;
        c.num_layers = 4;
        c.num_tokens = 2000;
        c.affinity_strength = 1.0;
        c.planted_groups = 4;
        c.seed = 5;
        const RoutingTrace tr = generate_markov_trace(c);
        // hand count on the host: the GPU is not used in this group
        std::vector<CountMatrix> ms(3, CountMatrix(8, 8));
        for (int t = 0; t < tr.num_tokens(); ++t)
            for (int j = 0; j < 3; ++j) ms[j](tr.paths(t, j), tr.paths(t, j + 1))++;
        AnnealParams prm;
        prm.seed = 7;
        auto [p, r] = solve_staged(counts_of(ms), t4, prm);
        CHECK(r.objective == 0.0 && r.solver == "staged");
        CHECK(objective_crossings(counts_of(ms), p, Level::gpu) == 0.0);
        CHECK(std::fabs(expected_planted_locality(c) - 1.0) < 1e-15);
    }
    AnnealParams badp;
    badp.cooling = 0.0;
    check_throws<std::invalid_argument>("cooling", [&] { badp.validate(); }, "cooling must be in (0,1]");
}

static void gpu_tests(const std::string& golden) {
    // ---- count_transitions (proj/tests/test_trace.cpp:95-113)
    {
        const TransitionCounts c = count_transitions(trace_from_paths(2, {{0, 0}, {0, 0}, {0, 1}, {1, 1}}), 1);
        CHECK(c.num_layer_pairs() == 1);
        CHECK(c.matrices[0](0, 0) == 2 && c.matrices[0](0, 1) == 1);
        CHECK(c.matrices[0](1, 0) == 0 && c.matrices[0](1, 1) == 1);
        CHECK(c.row_totals[0][0] == 3 && c.row_totals[0][1] == 1);
    }
    {
        const TransitionCounts c = count_transitions(trace_from_paths(2, {{0, 1, 0}}), 2);
        CHECK(c.num_layer_pairs() == 1 && c.matrices[0](0, 0) == 1 && c.matrices[0].sum() == 1);
    }
    {  // a random trace against a plain host loop (proj/src/trace.cpp:205-209)
        Rng rng(99);
        RoutingTrace t;
        t.num_experts = 16;
        t.num_layers = 6;
        t.paths.resize(5000, 6);
        for (int i = 0; i < 5000; ++i)
            for (int j = 0; j < 6; ++j) t.paths(i, j) = rng.below_int(16);
        const TransitionCounts c = count_transitions(t, 2);
        bool same = c.num_layer_pairs() == 4;
        for (int j = 0; same && j < 4; ++j) {
            CountMatrix want(16, 16);
            for (int i = 0; i < 5000; ++i) want(t.paths(i, j), t.paths(i, j + 2))++;
            same = want == c.matrices[j];
        }
        CHECK(same);
    }
    // ---- simulate on the demo (proj/tests/test_sim.cpp:75-117)
    const RoutingTrace demo = load_trace(golden + "/two_token_demo.trace");
    const Topology t4 = one_node(4);
    const Placement cont = contiguous_placement(8, 3, t4);
    SimConfig cfg;
    cfg.topology = t4;
    cfg.homes = std::vector<int>{1, 3};
    cfg.mode = SimMode::vanilla;
    const SimReport v = simulate(demo, cont, cfg);
    CHECK(v.total_crossings() == 10 && v.hops_inter_node == 0);
    CHECK(std::fabs(v.p - 5.0 / 6.0) < 1e-12);
    cfg.mode = SimMode::coherent;
    const SimReport c = simulate(demo, cont, cfg);
    CHECK(c.total_crossings() == 4 && std::fabs(c.p_star - 4.0 / 6.0) < 1e-12);
    for (std::uint64_t seed = 0; seed < 3; ++seed) {
        const Placement p = random_placement(8, 3, t4, seed);
        SimConfig k;
        k.topology = t4;
        k.mode = SimMode::vanilla;
        const SimReport rv = simulate(demo, p, k);
        CHECK(rv.alltoall_count == 6 && rv.allgather_count == 0 && rv.setup_allgather_count == 0);
        k.mode = SimMode::coherent;
        const SimReport rc = simulate(demo, p, k);
        CHECK(rc.alltoall_count == 3 && rc.allgather_count == 1 && rc.setup_allgather_count == 1);
        // per-token replay == token_hops summed (proj/src/sim.cpp:110-145 vs :34-76)
        long hops = 0;
        for (int t = 0; t < 2; ++t) {
            const std::vector<std::int32_t> path{demo.paths(t, 0), demo.paths(t, 1), demo.paths(t, 2)};
            hops += total_hops(token_hops(path, t % 4, p, SimMode::coherent, t4));
        }
        CHECK(hops == rc.total_crossings());
    }
    SimConfig bad;
    bad.topology = one_node(2);
    check_throws<std::invalid_argument>("grid mismatch", [&] { simulate(demo, cont, bad); },
                                        "topology grid does not match placement grid");
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "host";
    const std::string golden = argc > 2 ? argv[2] : "tests/golden";
    try {
        if (mode == "host") host_tests(golden);
        else if (mode == "gpu") gpu_tests(golden);
        else {
            std::printf("usage: test_mirror host|gpu [golden_dir]\n");
            return 2;
        }
    } catch (const std::exception& e) {
        std::printf("FAIL uncaught exception: %s\n", e.what());
        return 1;
    }
    std::printf("%s: %d checks, %d failures\n", mode.c_str(), g_checks, g_fails);
    return g_fails == 0 ? 0 : 1;
}
