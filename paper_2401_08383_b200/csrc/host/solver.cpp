// solver.cpp -- the host-side placement solver that consumes the GPU affinity
// histogram (stays on the CPU per BASELINE.json north_star).
//
// Problem (contract of proj/src/placement.cpp:528-821, paper Eq. 8-12): for
// every layer choose a balanced partition of the experts into groups (GPUs or
// nodes) minimising the number of token transitions between consecutive
// layers whose two experts sit in different groups.
//
// Design (not a transcription of the reference's loops):
//  * ChainGraph keeps each layer pair's weights twice, forward rows and
//    backward columns, so both neighbours of a layer are contiguous reads.
//  * SwapLedger carries, for the current labelling, the per-(layer, item,
//    group) affinity of every item towards each group of the layer above and
//    below. The crossing change of a within-layer swap is then O(1) (four
//    table reads per side) instead of an O(n) rescan, and an accepted swap
//    updates the two neighbouring tables in O(n).
//  * Annealing restarts are independent (restart r owns the stream
//    seed_stream(seed, r), proj/src/placement.cpp:319-320) and run on a pool
//    of host threads; the best restart is then chosen in restart order with
//    the reference's strict 1e-12 improvement rule, so the result does not
//    depend on the thread count or timing.
//  * The exact solver is a dynamic program over all balanced labellings of a
//    layer whose backward sweep is split over host threads by state.
// Weights are integer transition counts: every objective, delta and table
// entry is an exact integer in fp64, so the order in which this code sums
// them cannot change a comparison, and the accept/reject decisions, the
// random-draw order (one layer draw, two item draws, rejection redraws of the
// second item, one uniform per uphill move) and hence the placements equal
// the reference's for the same seed.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <limits>
#include <string>
#include <thread>

#include "exflow/exflow.hpp"

namespace exflow {
namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr double kTieEps = 1e-12;  // strict-improvement margin of the contract

using Labels = std::vector<std::vector<int>>;  // [layer][item] -> group

int host_threads(int work_items) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    return std::max(1, std::min<int>(static_cast<int>(hw), work_items));
}

// Runs body(k) for k in [0, count) on up to host_threads(count) threads.
template <class F>
void parallel_for(int count, F&& body) {
    const int nt = host_threads(count);
    if (nt <= 1) {
        for (int k = 0; k < count; ++k) body(k);
        return;
    }
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    pool.reserve(nt);
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&] {
            for (int k = next.fetch_add(1); k < count; k = next.fetch_add(1)) body(k);
        });
    for (auto& th : pool) th.join();
}

// ------------------------------------------------------------------ graph
struct ChainGraph {
    int n = 0;       // items per layer
    int parts = 1;   // groups per layer (each holds n / parts items)
    int layers = 0;  // layer count (layers - 1 weight matrices)
    std::vector<double> fwd;  // [j][a][b] = w_j(a, b), a in layer j, b in layer j+1
    std::vector<double> bwd;  // [j][b][a] = w_j(a, b)
    std::vector<double> mass;  // [j] sum of w_j

    int cap() const { return n / parts; }
    const double* out_row(int j, int a) const { return fwd.data() + (static_cast<size_t>(j) * n + a) * n; }
    const double* in_col(int j, int b) const { return bwd.data() + (static_cast<size_t>(j) * n + b) * n; }

    void allocate(int items, int groups, int layer_count) {
        n = items;
        parts = groups;
        layers = layer_count;
        const size_t edges = static_cast<size_t>(std::max(layers - 1, 0)) * n * n;
        fwd.assign(edges, 0.0);
        bwd.assign(edges, 0.0);
        mass.assign(std::max(layers - 1, 0), 0.0);
    }
    void set(int j, int a, int b, double w) {
        fwd[(static_cast<size_t>(j) * n + a) * n + b] = w;
        bwd[(static_cast<size_t>(j) * n + b) * n + a] = w;
        mass[j] += w;
    }
};

// The chain over every expert of `counts`, partitioned into `parts` groups
// (make_chain's preconditions and messages, proj/src/placement.cpp:369-385).
ChainGraph full_graph(const TransitionCounts& counts, int parts) {
    if (counts.gap != 1) throw std::invalid_argument("placement solving requires gap-1 transition counts");
    if (parts < 1 || counts.num_experts % parts != 0)
        throw std::invalid_argument("num_experts " + std::to_string(counts.num_experts) +
                                    " not divisible by partitions " + std::to_string(parts));
    ChainGraph g;
    g.allocate(counts.num_experts, parts, counts.num_layers);
    for (int j = 0; j + 1 < g.layers; ++j) {
        const CountMatrix& m = counts.matrices[j];
        for (int a = 0; a < g.n; ++a) {
            const std::int64_t* row = m.row_ptr(a);
            for (int b = 0; b < g.n; ++b)
                if (row[b] != 0) g.set(j, a, b, static_cast<double>(row[b]));
        }
    }
    return g;
}

// The chain restricted to one node's experts (members[j] = expert ids of the
// node at layer j, in increasing order), split over its GPUs.
ChainGraph node_graph(const TransitionCounts& counts, const std::vector<std::vector<int>>& members,
                      int parts) {
    ChainGraph g;
    g.allocate(static_cast<int>(members[0].size()), parts, counts.num_layers);
    for (int j = 0; j + 1 < g.layers; ++j) {
        const CountMatrix& m = counts.matrices[j];
        for (int a = 0; a < g.n; ++a)
            for (int b = 0; b < g.n; ++b) {
                const std::int64_t w = m(members[j][a], members[j + 1][b]);
                if (w != 0) g.set(j, a, b, static_cast<double>(w));
            }
    }
    return g;
}

std::vector<int> blocks(int items, int parts) {
    std::vector<int> v(items);
    const int cap = items / parts;
    for (int i = 0; i < items; ++i) v[i] = i / cap;
    return v;
}

// ------------------------------------------------------------------ ledger
class SwapLedger {
  public:
    SwapLedger(const ChainGraph& g, Labels labels) : g_(&g), lab_(std::move(labels)) {
        const size_t per = static_cast<size_t>(g.n) * g.parts;
        up_.assign(static_cast<size_t>(g.layers) * per, 0.0);
        down_.assign(static_cast<size_t>(g.layers) * per, 0.0);
        for (int j = 1; j < g.layers; ++j) rebuild_up(j);
        for (int j = 0; j + 1 < g.layers; ++j) rebuild_down(j);
    }

    const Labels& labels() const { return lab_; }
    int label(int j, int i) const { return lab_[j][i]; }

    // crossings change if items a and b of layer j exchange groups
    double delta(int j, int a, int b) const {
        const int ga = lab_[j][a], gb = lab_[j][b];
        double d = 0.0;
        if (j > 0) {
            const double* ta = up(j, a);
            const double* tb = up(j, b);
            d += (ta[ga] - ta[gb]) + (tb[gb] - tb[ga]);
        }
        if (j + 1 < g_->layers) {
            const double* ta = down(j, a);
            const double* tb = down(j, b);
            d += (ta[ga] - ta[gb]) + (tb[gb] - tb[ga]);
        }
        return d;
    }

    void swap(int j, int a, int b) {
        const int ga = lab_[j][a], gb = lab_[j][b];
        std::swap(lab_[j][a], lab_[j][b]);
        const int n = g_->n, P = g_->parts;
        if (j + 1 < g_->layers) {  // layer j+1 sees a move from ga to gb (item a) and back (b)
            const double* wa = g_->out_row(j, a);
            const double* wb = g_->out_row(j, b);
            double* t = up_.data() + static_cast<size_t>(j + 1) * n * P;
            for (int y = 0; y < n; ++y) {
                const double shift = wa[y] - wb[y];
                if (shift != 0.0) {
                    t[y * P + ga] -= shift;
                    t[y * P + gb] += shift;
                }
            }
        }
        if (j > 0) {  // layer j-1 sees the same exchange from below
            const double* wa = g_->in_col(j - 1, a);
            const double* wb = g_->in_col(j - 1, b);
            double* t = down_.data() + static_cast<size_t>(j - 1) * n * P;
            for (int x = 0; x < n; ++x) {
                const double shift = wa[x] - wb[x];
                if (shift != 0.0) {
                    t[x * P + ga] -= shift;
                    t[x * P + gb] += shift;
                }
            }
        }
    }

    // total crossings of the current labelling: per layer pair, the pair's
    // mass minus the weight that stays inside a group
    double cost() const {
        double c = 0.0;
        for (int j = 0; j + 1 < g_->layers; ++j) {
            double stay = 0.0;
            for (int a = 0; a < g_->n; ++a) stay += down(j, a)[lab_[j][a]];
            c += g_->mass[j] - stay;
        }
        return c;
    }

  private:
    const double* up(int j, int i) const {
        return up_.data() + (static_cast<size_t>(j) * g_->n + i) * g_->parts;
    }
    const double* down(int j, int i) const {
        return down_.data() + (static_cast<size_t>(j) * g_->n + i) * g_->parts;
    }
    void rebuild_up(int j) {  // up(j, i)[p] = sum over x in group p of layer j-1 of w_{j-1}(x, i)
        const int n = g_->n, P = g_->parts;
        double* t = up_.data() + static_cast<size_t>(j) * n * P;
        std::fill(t, t + static_cast<size_t>(n) * P, 0.0);
        for (int i = 0; i < n; ++i) {
            const double* col = g_->in_col(j - 1, i);
            for (int x = 0; x < n; ++x) t[i * P + lab_[j - 1][x]] += col[x];
        }
    }
    void rebuild_down(int j) {  // down(j, i)[p] = sum over y in group p of layer j+1 of w_j(i, y)
        const int n = g_->n, P = g_->parts;
        double* t = down_.data() + static_cast<size_t>(j) * n * P;
        std::fill(t, t + static_cast<size_t>(n) * P, 0.0);
        for (int i = 0; i < n; ++i) {
            const double* row = g_->out_row(j, i);
            for (int y = 0; y < n; ++y) t[i * P + lab_[j + 1][y]] += row[y];
        }
    }

    const ChainGraph* g_;
    Labels lab_;
    std::vector<double> up_, down_;
};

// Restart 0's start (greedy chain following, the contract of
// proj/src/placement.cpp:231-268): layer 0 in blocks; each later layer is
// filled one (item, group) pair at a time, always the unassigned item / open
// group with the largest weight arriving from the previous layer's groups
// (first such pair in item-major, group-minor order on ties).
Labels greedy_start(const ChainGraph& g) {
    const int n = g.n, P = g.parts, cap = g.cap();
    Labels lab(g.layers);
    lab[0] = blocks(n, P);
    std::vector<double> pull(static_cast<size_t>(n) * P);
    for (int j = 1; j < g.layers; ++j) {
        std::fill(pull.begin(), pull.end(), 0.0);
        for (int b = 0; b < n; ++b) {
            const double* col = g.in_col(j - 1, b);
            for (int a = 0; a < n; ++a) pull[b * P + lab[j - 1][a]] += col[a];
        }
        std::vector<int> cur(n, -1), fill(P, 0);
        for (int placed = 0; placed < n; ++placed) {
            int pick = -1;
            double top = -kInf;
            for (int k = 0; k < n * P; ++k) {
                const int b = k / P, p = k - b * P;
                if (cur[b] < 0 && fill[p] < cap && pull[k] > top) {
                    top = pull[k];
                    pick = k;
                }
            }
            cur[pick / P] = pick % P;
            fill[pick % P]++;
        }
        lab[j] = std::move(cur);
    }
    return lab;
}

// First-improvement descent (contract of proj/src/placement.cpp:270-290):
// sweep layers, then item pairs a < b in order, taking every swap that lowers
// the crossings by more than the tie margin, until a sweep changes nothing
// (at most 200 sweeps).
void descend(SwapLedger& led, const ChainGraph& g) {
    for (int sweep = 0; sweep < 200; ++sweep) {
        bool changed = false;
        for (int j = 0; j < g.layers; ++j)
            for (int a = 0; a < g.n; ++a)
                for (int b = a + 1; b < g.n; ++b)
                    if (led.label(j, a) != led.label(j, b) && led.delta(j, a, b) < -kTieEps) {
                        led.swap(j, a, b);
                        changed = true;
                    }
        if (!changed) return;
    }
}

struct RestartOutcome {
    Labels labels;
    double cost = kInf;
};

RestartOutcome run_restart(const ChainGraph& g, const AnnealParams& prm, int r, long iters,
                           double t0) {
    const int L = g.layers, n = g.n;
    Rng rng(seed_stream(prm.seed, static_cast<std::uint64_t>(r)));
    Labels start;
    if (r == 0) {
        start = greedy_start(g);
    } else {
        start.resize(L);
        for (auto& layer : start) {
            layer = blocks(n, g.parts);
            shuffle(std::span<int>(layer), rng);
        }
    }
    SwapLedger led(g, std::move(start));
    double cost = led.cost();
    Labels best = led.labels();
    double best_cost = cost;
    double temp = t0;
    for (long it = 0; it < iters; ++it, temp *= prm.cooling) {
        const int j = static_cast<int>(rng.below(static_cast<std::uint64_t>(L)));
        const int a = rng.below_int(n);
        int b = rng.below_int(n);
        while (led.label(j, b) == led.label(j, a)) b = rng.below_int(n);
        const double d = led.delta(j, a, b);
        if (d > 0.0 && !(rng.uniform01() < std::exp(-d / std::max(temp, 1e-300)))) continue;
        led.swap(j, a, b);
        cost += d;
        if (cost < best_cost - kTieEps) {
            best_cost = cost;
            best = led.labels();
        }
    }
    SwapLedger fin(g, std::move(best));
    descend(fin, g);
    return {fin.labels(), fin.cost()};
}

Labels anneal(const ChainGraph& g, const AnnealParams& prm, double* objective, long* iterations) {
    if (g.parts == 1) {  // a single group: nothing to swap
        *objective = 0.0;
        *iterations = 0;
        return Labels(g.layers, std::vector<int>(g.n, 0));
    }
    const long iters = prm.max_iters > 0 ? prm.max_iters : 20000L * g.layers;
    double t0 = prm.initial_temperature;
    if (!(t0 > 0.0)) {  // mean positive weight (proj/src/placement.cpp:292-300)
        double s = 0.0;
        long pos = 0;
        for (double w : g.fwd) {
            s += w;
            pos += w > 0.0;
        }
        t0 = pos > 0 ? s / static_cast<double>(pos) : 1.0;
    }
    std::vector<RestartOutcome> out(prm.restarts);
    parallel_for(prm.restarts, [&](int r) { out[r] = run_restart(g, prm, r, iters, t0); });
    int pick = -1;
    double best = kInf;
    for (int r = 0; r < prm.restarts; ++r)  // restart order: thread-count independent
        if (out[r].cost < best - kTieEps) {
            best = out[r].cost;
            pick = r;
        }
    *objective = best;
    *iterations = static_cast<long>(prm.restarts) * iters;
    return pick >= 0 ? std::move(out[pick].labels) : Labels(g.layers, blocks(g.n, g.parts));
}

// ------------------------------------------------------------------ exact DP
// Every balanced labelling of one layer, in lexicographic order (a state's
// index is its rank; ties in the DP resolve to the lowest index).
std::vector<std::vector<int8_t>> balanced_states(int items, int parts) {
    std::vector<std::vector<int8_t>> out;
    std::vector<int8_t> cur(items, 0);
    std::vector<int> fill(parts, 0);
    const int cap = items / parts;
    std::vector<int> next_label(items + 1, 0);
    int pos = 0;
    while (pos >= 0) {
        if (pos == items) {
            out.push_back(cur);
            --pos;
            if (pos >= 0) fill[cur[pos]]--;
            continue;
        }
        int p = next_label[pos];
        while (p < parts && fill[p] >= cap) ++p;
        if (p == parts) {
            next_label[pos] = 0;
            --pos;
            if (pos >= 0) fill[cur[pos]]--;
            continue;
        }
        cur[pos] = static_cast<int8_t>(p);
        fill[p]++;
        next_label[pos] = p + 1;
        ++pos;
        if (pos < items) next_label[pos] = 0;
    }
    return out;
}

// tail[j][s] = cheapest crossings of layers j..L-1 given state s at layer j.
// For a state s at layer j, inflow[b][p] = weight from s's group p into item
// b of layer j+1; a successor t keeps sum_b inflow[b][t(b)] inside groups.
Labels exact_dp(const ChainGraph& g, double* objective) {
    const auto states = balanced_states(g.n, g.parts);
    const int S = static_cast<int>(states.size());
    const int n = g.n, P = g.parts, L = g.layers;
    std::vector<std::vector<double>> tail(L, std::vector<double>(S, 0.0));
    auto inflow_of = [&](int j, int s, std::vector<double>& inflow) {
        std::fill(inflow.begin(), inflow.end(), 0.0);
        for (int a = 0; a < n; ++a) {
            const double* row = g.out_row(j, a);
            const int p = states[s][a];
            for (int b = 0; b < n; ++b) inflow[b * P + p] += row[b];
        }
    };
    auto best_next = [&](int j, const std::vector<double>& inflow, int* arg) {
        const std::vector<double>& nxt = tail[j + 1];
        double best = kInf;
        for (int t = 0; t < S; ++t) {
            const int8_t* lt = states[t].data();
            double stay = 0.0;
            for (int b = 0; b < n; ++b) stay += inflow[b * P + lt[b]];
            const double v = g.mass[j] - stay + nxt[t];
            if (v < best) {
                best = v;
                if (arg) *arg = t;
            }
        }
        return best;
    };
    for (int j = L - 2; j >= 0; --j) {
        const int chunks = std::min(S, 4 * host_threads(S));
        parallel_for(chunks, [&](int c) {
            std::vector<double> inflow(static_cast<size_t>(n) * P);
            for (int s = c; s < S; s += chunks) {
                inflow_of(j, s, inflow);
                tail[j][s] = best_next(j, inflow, nullptr);
            }
        });
    }
    int state = 0;
    for (int s = 1; s < S; ++s)
        if (tail[0][s] < tail[0][state]) state = s;
    if (objective) *objective = tail[0][state];
    Labels out(L);
    out[0].assign(states[state].begin(), states[state].end());
    std::vector<double> inflow(static_cast<size_t>(n) * P);
    for (int j = 0; j + 1 < L; ++j) {
        inflow_of(j, state, inflow);
        int t = -1;
        best_next(j, inflow, &t);
        state = t;
        out[j + 1].assign(states[state].begin(), states[state].end());
    }
    return out;
}

Placement labels_to_placement(const Labels& lab, int experts, int groups) {
    Placement p;
    p.num_experts = experts;
    p.num_layers = static_cast<int>(lab.size());
    p.num_nodes = 1;
    p.gpus_per_node = groups;
    p.assign.resize(p.num_layers, experts);
    for (int j = 0; j < p.num_layers; ++j) std::copy(lab[j].begin(), lab[j].end(), p.assign.row_ptr(j));
    return p;
}

}  // namespace

// ------------------------------------------------------------------ public API
void AnnealParams::validate() const {
    if (restarts < 1) throw std::invalid_argument("restarts must be >= 1");
    if (max_iters < 0) throw std::invalid_argument("max_iters must be >= 0 (0 selects the default)");
    if (cooling <= 0.0 || cooling > 1.0) throw std::invalid_argument("cooling must be in (0,1]");
    if (initial_temperature < 0.0)
        throw std::invalid_argument("initial_temperature must be >= 0 (0 selects the default)");
}

std::pair<Placement, SolveReport> solve_exact_dp(const TransitionCounts& counts, int partitions,
                                                 long state_cap) {
    const ChainGraph g = full_graph(counts, partitions);
    const long states = balanced_assignment_count(g.n, g.parts, state_cap);
    if (states > state_cap)
        throw std::invalid_argument("balanced state space exceeds cap " + std::to_string(state_cap) +
                                    " for " + std::to_string(g.n) + " experts in " +
                                    std::to_string(g.parts) +
                                    " partitions; use the local-search solver (anneal)");
    SolveReport r;
    Placement p = labels_to_placement(exact_dp(g, &r.objective), counts.num_experts, partitions);
    p.validate();
    r.solver = "exact-dp";
    r.iterations = states;
    r.restarts = 0;
    r.optimality_gap = 0.0;
    return {std::move(p), std::move(r)};
}

std::pair<Placement, SolveReport> solve_local_search(const TransitionCounts& counts, int partitions,
                                                     const AnnealParams& params) {
    params.validate();
    const ChainGraph g = full_graph(counts, partitions);
    SolveReport r;
    Placement p = labels_to_placement(anneal(g, params, &r.objective, &r.iterations),
                                      counts.num_experts, partitions);
    p.validate();
    r.solver = "local-search";
    r.seed = params.seed;
    r.restarts = params.restarts;
    return {std::move(p), std::move(r)};
}

std::pair<Placement, SolveReport> solve_staged(const TransitionCounts& counts,
                                               const Topology& topology, const AnnealParams& params,
                                               long state_cap) {
    params.validate();
    topology.validate();
    if (counts.gap != 1) throw std::invalid_argument("placement solving requires gap-1 transition counts");
    if (counts.num_experts % topology.num_nodes != 0 || counts.num_experts % topology.total_gpus() != 0)
        throw std::invalid_argument("num_experts must be divisible by node and GPU counts");
    const int E = counts.num_experts, L = counts.num_layers;
    long iterations = 0;
    // exact when the per-layer state space fits the cap, annealing otherwise
    auto solve_chain = [&](const ChainGraph& g, std::uint64_t seed) {
        const long states = balanced_assignment_count(g.n, g.parts, state_cap);
        double obj = 0.0;
        if (states <= state_cap) {
            iterations += states;
            return exact_dp(g, &obj);
        }
        AnnealParams p = params;
        p.seed = seed;
        long it = 0;
        Labels lab = anneal(g, p, &obj, &it);
        iterations += it;
        return lab;
    };
    Placement placement;
    if (topology.num_nodes == 1) {  // one node: the GPU-level chain alone
        const Labels lab = solve_chain(full_graph(counts, topology.total_gpus()), params.seed);
        placement = regrid(labels_to_placement(lab, E, topology.total_gpus()), 1, topology.gpus_per_node);
    } else {
        // stage 1 splits the experts over nodes; stage 2 splits each node's
        // experts over its GPUs, seeing only the transitions inside the node
        const Labels node_of = solve_chain(full_graph(counts, topology.num_nodes), params.seed);
        placement.num_experts = E;
        placement.num_layers = L;
        placement.num_nodes = topology.num_nodes;
        placement.gpus_per_node = topology.gpus_per_node;
        placement.assign.resize(L, E);
        for (int node = 0; node < topology.num_nodes; ++node) {
            std::vector<std::vector<int>> members(L);
            for (int j = 0; j < L; ++j)
                for (int e = 0; e < E; ++e)
                    if (node_of[j][e] == node) members[j].push_back(e);
            const Labels gpu = solve_chain(node_graph(counts, members, topology.gpus_per_node),
                                           seed_stream(params.seed, 1 + static_cast<std::uint64_t>(node)));
            for (int j = 0; j < L; ++j)
                for (size_t k = 0; k < members[j].size(); ++k)
                    placement.assign(j, members[j][k]) = node * topology.gpus_per_node + gpu[j][k];
        }
        placement.validate();
    }
    const double inter = objective_crossings(counts, placement, Level::node);
    const double total = objective_crossings(counts, placement, Level::gpu);
    SolveReport r;
    r.solver = "staged";
    r.objective = total;
    r.seed = params.seed;
    r.iterations = iterations;
    r.restarts = params.restarts;
    r.inter_node_crossings = inter;
    r.intra_node_crossings = total - inter;
    r.weighted_cost = inter * topology.inter_node_hop_cost + (total - inter) * topology.intra_node_hop_cost;
    return {std::move(placement), std::move(r)};
}

}  // namespace exflow
