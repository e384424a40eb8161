// capi_host.cpp -- C-ABI wrappers of the host placement/solver/synth code:
// flat row-major arrays in, reference C++ types inside, exceptions mapped to
// exf_status (std::invalid_argument -> EXF_INVALID, others -> EXF_RUNTIME).
#include <cstring>
#include <string>

#include "exflow/exflow.hpp"
#include "exflow_c.h"

namespace exf {
void set_error(const std::string& msg);
}

namespace {

template <class F>
exf_status guarded(F&& f) {
    try {
        f();
        return EXF_OK;
    } catch (const std::invalid_argument& e) {
        exf::set_error(e.what());
        return EXF_INVALID;
    } catch (const std::exception& e) {
        exf::set_error(e.what());
        return EXF_RUNTIME;
    }
}

exflow::Topology topo(int32_t nodes, int32_t gpn, double intra = 1.0, double inter = 4.0) {
    exflow::Topology t;
    t.num_nodes = nodes;
    t.gpus_per_node = gpn;
    t.intra_node_hop_cost = intra;
    t.inter_node_hop_cost = inter;
    return t;
}

void store(const exflow::Placement& p, int32_t* out) {
    for (int j = 0; j < p.num_layers; ++j)
        for (int e = 0; e < p.num_experts; ++e) out[j * p.num_experts + e] = p.assign(j, e);
}

exflow::Placement load(const int32_t* a, int32_t L, int32_t E, int32_t nodes, int32_t gpn) {
    exflow::Placement p;
    p.num_experts = E;
    p.num_layers = L;
    p.num_nodes = nodes;
    p.gpus_per_node = gpn;
    p.assign.resize(L, E);
    for (int j = 0; j < L; ++j)
        for (int e = 0; e < E; ++e) p.assign(j, e) = a[j * E + e];
    return p;
}

exflow::TransitionCounts counts_in(const int64_t* c, int32_t L, int32_t E, int32_t gap) {
    if (E < 1 || L < 2 || gap < 1 || gap > L - 1) throw std::invalid_argument("bad counts shape");
    exflow::TransitionCounts t;
    t.num_experts = E;
    t.num_layers = L;
    t.gap = gap;
    for (int j = 0; j < L - gap; ++j) {
        exflow::CountMatrix m(E, E);
        std::memcpy(m.data(), c + (int64_t)j * E * E, sizeof(int64_t) * E * E);
        t.row_totals.push_back(m.rowwise_sum());
        t.matrices.push_back(std::move(m));
    }
    return t;
}

exflow::AnnealParams params_in(const exf_anneal_params* p) {
    exflow::AnnealParams a;
    if (p) {
        a.restarts = p->restarts;
        a.max_iters = p->max_iters;
        a.initial_temperature = p->initial_temperature;
        a.cooling = p->cooling;
        a.seed = p->seed;
    }
    return a;
}

void report_out(const exflow::SolveReport& r, exf_solve_report* out) {
    if (!out) return;
    std::memset(out, 0, sizeof(*out));
    std::strncpy(out->solver, r.solver.c_str(), sizeof(out->solver) - 1);
    out->objective = r.objective;
    out->seed = r.seed;
    out->iterations = r.iterations;
    out->restarts = r.restarts;
    out->has_optimality_gap = r.optimality_gap.has_value();
    out->optimality_gap = r.optimality_gap.value_or(0.0);
    out->has_tiers = r.inter_node_crossings.has_value();
    out->inter_node_crossings = r.inter_node_crossings.value_or(0.0);
    out->intra_node_crossings = r.intra_node_crossings.value_or(0.0);
    out->weighted_cost = r.weighted_cost.value_or(0.0);
}

}  // namespace

extern "C" {

exf_status exf_contiguous_placement(int32_t E, int32_t L, int32_t nodes, int32_t gpn,
                                    int32_t* h_assign) {
    return guarded([&] { store(exflow::contiguous_placement(E, L, topo(nodes, gpn)), h_assign); });
}

exf_status exf_random_placement(int32_t E, int32_t L, int32_t nodes, int32_t gpn, uint64_t seed,
                                int32_t* h_assign) {
    return guarded(
        [&] { store(exflow::random_placement(E, L, topo(nodes, gpn), seed), h_assign); });
}

exf_status exf_validate_placement(const int32_t* h_assign, int32_t L, int32_t E, int32_t nodes,
                                  int32_t gpn) {
    return guarded([&] { load(h_assign, L, E, nodes, gpn).validate(); });
}

exf_status exf_objective_crossings(const int64_t* h_counts, int32_t L, int32_t E, int32_t gap,
                                   const int32_t* h_assign, int32_t nodes, int32_t gpn,
                                   int32_t level, double* out) {
    return guarded([&] {
        *out = exflow::objective_crossings(counts_in(h_counts, L, E, gap),
                                           load(h_assign, L, E, nodes, gpn),
                                           level == 0 ? exflow::Level::node : exflow::Level::gpu);
    });
}

int64_t exf_balanced_assignment_count(int32_t items, int32_t parts, int64_t cap) {
    try {
        return exflow::balanced_assignment_count(items, parts, cap);
    } catch (const std::exception& e) {
        exf::set_error(e.what());
        return -1;
    }
}

exf_status exf_solve_exact_dp(const int64_t* h_counts, int32_t L, int32_t E, int32_t partitions,
                              int64_t state_cap, int32_t* h_assign, exf_solve_report* report) {
    return guarded([&] {
        auto [p, r] = exflow::solve_exact_dp(counts_in(h_counts, L, E, 1), partitions, state_cap);
        store(p, h_assign);
        report_out(r, report);
    });
}

exf_status exf_solve_local_search(const int64_t* h_counts, int32_t L, int32_t E,
                                  int32_t partitions, const exf_anneal_params* params,
                                  int32_t* h_assign, exf_solve_report* report) {
    return guarded([&] {
        auto [p, r] = exflow::solve_local_search(counts_in(h_counts, L, E, 1), partitions,
                                                 params_in(params));
        store(p, h_assign);
        report_out(r, report);
    });
}

exf_status exf_solve_staged(const int64_t* h_counts, int32_t L, int32_t E, int32_t nodes,
                            int32_t gpn, double intra, double inter,
                            const exf_anneal_params* params, int64_t state_cap, int32_t* h_assign,
                            exf_solve_report* report) {
    return guarded([&] {
        auto [p, r] = exflow::solve_staged(counts_in(h_counts, L, E, 1),
                                           topo(nodes, gpn, intra, inter), params_in(params),
                                           state_cap);
        store(p, h_assign);
        report_out(r, report);
    });
}

exf_status exf_token_hops(const int32_t* h_path, int32_t L, int32_t home, const int32_t* h_assign,
                          int32_t E, int32_t nodes, int32_t gpn, int32_t mode, int32_t* h_crossed,
                          int32_t* h_tier, int32_t* h_hops) {
    return guarded([&] {
        if (!h_path || !h_assign || L < 1) throw std::invalid_argument("null argument");
        if (mode != 0 && mode != 1) throw std::invalid_argument("mode must be 0 (vanilla) or 1 (coherent)");
        const auto hops = exflow::token_hops(std::span<const int32_t>(h_path, static_cast<size_t>(L)), home,
                                             load(h_assign, L, E, nodes, gpn),
                                             mode == 0 ? exflow::SimMode::vanilla : exflow::SimMode::coherent,
                                             topo(nodes, gpn));
        for (int32_t j = 0; j < L; ++j) {
            if (h_crossed) h_crossed[j] = hops[j].crossed ? 1 : 0;
            if (h_tier) h_tier[j] = static_cast<int32_t>(hops[j].tier);
            if (h_hops) h_hops[j] = hops[j].hops;
        }
    });
}

exf_status exf_generate_markov_trace(int32_t E, int32_t L, int64_t T, double alpha,
                                     int32_t groups, uint64_t seed, int32_t* h_paths) {
    return guarded([&] {
        if (T > 0x7fffffffLL) throw std::invalid_argument("num_tokens too large");
        exflow::SynthConfig c;
        c.num_experts = E;
        c.num_layers = L;
        c.num_tokens = static_cast<int>(T);
        c.affinity_strength = alpha;
        c.planted_groups = groups;
        c.seed = seed;
        const exflow::RoutingTrace t = exflow::generate_markov_trace(c);
        std::memcpy(h_paths, t.paths.data(), sizeof(int32_t) * T * L);
    });
}

}  // extern "C"
