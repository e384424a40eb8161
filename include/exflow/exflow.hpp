// exflow/exflow.hpp -- C++ API of the B200-native ExFlow hot path.
//
// Restores the reference's namespace exflow signatures on top
// of the C-ABI (include/exflow_c.h) so the reference's callers (the cmd_*
// functions of proj/tools/exflow.cpp and its tests) can switch over:
//   count_transitions      proj/include/exflow/trace.hpp:71   -> GPU kernel (5)
//   simulate               proj/include/exflow/sim.hpp:65     -> GPU routing replay
//   solve_staged & friends proj/include/exflow/placement.hpp:132-154 (host, CPU)
//   generate_markov_trace  proj/include/exflow/synth.hpp:33   (host)
// Types keep the reference field names; matrices are exflow::Matrix
// (row-major) instead of Eigen. Errors throw the reference's exception types
// with its messages (std::invalid_argument, ParseError, std::runtime_error).
#pragma once

#include <cstdint>
#include <filesystem>
#include <iosfwd>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "exflow/matrix.hpp"
#include "exflow/prng.hpp"

namespace exflow {

using CountMatrix = Matrix<std::int64_t>;
using ProbMatrix = Matrix<double>;
using CountVector = std::vector<std::int64_t>;
using SeenMask = std::vector<bool>;
using PathMatrix = Matrix<std::int32_t>;  // [T][L], row-major like the reference

// ---------------------------------------------------------------- traces
struct RoutingTrace {
    int num_experts = 0;
    int num_layers = 0;
    PathMatrix paths;
    int num_tokens() const { return static_cast<int>(paths.rows()); }
    void validate() const;  // proj/src/trace.cpp:53-70
};

class ParseError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

RoutingTrace parse_trace(std::istream& in);          // EXFLOW-TRACE v1
RoutingTrace parse_trace(const std::string& text);
RoutingTrace load_trace(const std::filesystem::path& path);
void write_trace(std::ostream& out, const RoutingTrace& trace);
std::string serialize_trace(const RoutingTrace& trace);
void save_trace(const std::filesystem::path& path, const RoutingTrace& trace);

struct TransitionCounts {
    int num_experts = 0;
    int num_layers = 0;
    int gap = 1;
    std::vector<CountMatrix> matrices;
    std::vector<CountVector> row_totals;
    int num_layer_pairs() const { return static_cast<int>(matrices.size()); }
};

// GPU kernel (5); bit-exact with the reference loop.
TransitionCounts count_transitions(const RoutingTrace& trace, int gap = 1);

struct AffinityMatrix {
    int num_experts = 0;
    int num_layers = 0;
    int gap = 1;
    std::vector<ProbMatrix> matrices;
    std::vector<SeenMask> seen;
    int num_layer_pairs() const { return static_cast<int>(matrices.size()); }
};

AffinityMatrix conditional_probabilities(const TransitionCounts& counts);
int most_affiliated(const AffinityMatrix& affinity, int source_layer, int expert);
std::string export_heatmap_csv(const AffinityMatrix& affinity, int source_layer);

// ---------------------------------------------------------------- synth
struct SynthConfig {
    int num_experts = 8;
    int num_layers = 2;
    int num_tokens = 1;
    double affinity_strength = 0.5;
    int planted_groups = 1;
    std::uint64_t seed = 0;
    int group_size() const { return num_experts / planted_groups; }
    void validate() const;
};
RoutingTrace generate_markov_trace(const SynthConfig& config);
double expected_planted_locality(const SynthConfig& config);

// ---------------------------------------------------------------- placement
struct Topology {
    int num_nodes = 1;
    int gpus_per_node = 1;
    double intra_node_hop_cost = 1.0;
    double inter_node_hop_cost = 4.0;
    int total_gpus() const { return num_nodes * gpus_per_node; }
    int node_of(int gpu) const { return gpu / gpus_per_node; }
    void validate() const;
};

enum class Level { node, gpu };

struct Placement {
    int num_experts = 0;
    int num_layers = 0;
    int num_nodes = 1;
    int gpus_per_node = 1;
    Matrix<int> assign;  // [L][E] GPU ids
    int total_gpus() const { return num_nodes * gpus_per_node; }
    int node_of(int gpu) const { return gpu / gpus_per_node; }
    int gpu_of(int layer, int expert) const { return assign(layer, expert); }
    void validate() const;  // proj/src/placement.cpp:434-470
};

Placement regrid(Placement placement, int num_nodes, int gpus_per_node);
Placement contiguous_placement(int num_experts, int num_layers, const Topology& topology);
Placement random_placement(int num_experts, int num_layers, const Topology& topology,
                           std::uint64_t seed);
double objective_crossings(const TransitionCounts& counts, const Placement& placement,
                           Level level);
long balanced_assignment_count(int items, int parts, long cap);

inline constexpr long kDefaultStateCap = 10000;

struct AnnealParams {
    int restarts = 8;
    long max_iters = 0;               // 0 -> 20000 * L
    double initial_temperature = 0.0;  // 0 -> mean positive weight
    double cooling = 0.999;
    std::uint64_t seed = 0;
    void validate() const;
};

struct SolveReport {
    std::string solver;
    double objective = 0.0;
    std::uint64_t seed = 0;
    long iterations = 0;
    int restarts = 0;
    std::optional<double> optimality_gap;
    std::optional<double> inter_node_crossings;
    std::optional<double> intra_node_crossings;
    std::optional<double> weighted_cost;
};

std::pair<Placement, SolveReport> solve_exact_dp(const TransitionCounts& counts, int partitions,
                                                 long state_cap = kDefaultStateCap);
std::pair<Placement, SolveReport> solve_local_search(const TransitionCounts& counts, int partitions,
                                                     const AnnealParams& params);
std::pair<Placement, SolveReport> solve_staged(const TransitionCounts& counts,
                                               const Topology& topology, const AnnealParams& params,
                                               long state_cap = kDefaultStateCap);

// Placement JSON: {"experts","layers","nodes","gpus_per_node","assign"}
Placement load_placement(const std::filesystem::path& path);
Placement placement_from_json(const std::string& text);
std::string placement_to_json(const Placement& placement);

// ---------------------------------------------------------------- simulator
enum class SimMode { vanilla, coherent };
enum class Tier { intra_gpu, intra_node, inter_node };

struct LayerHop {
    bool crossed = false;
    Tier tier = Tier::intra_gpu;
    int hops = 0;
};

std::vector<LayerHop> token_hops(std::span<const std::int32_t> path, int home_gpu,
                                 const Placement& placement, SimMode mode,
                                 const Topology& topology);

struct SimConfig {
    SimMode mode = SimMode::vanilla;
    Topology topology;
    int tokens_per_gpu = 1;
    int iterations = 1;
    std::optional<std::vector<int>> homes;
    void validate() const;
};

struct SimReport {
    long hops_intra_node = 0;
    long hops_inter_node = 0;
    double locality_gpu = 0.0;
    double locality_node = 0.0;
    double p = 0.0;
    double p_star = 0.0;
    long alltoall_count = 0;
    long allgather_count = 0;
    long setup_allgather_count = 0;
    double volume_units = 0.0;
    double estimated_latency = 0.0;
    long total_crossings() const { return hops_intra_node + hops_inter_node; }
};

// GPU routing replay (exf_route_replay) + host report derivation.
SimReport simulate(const RoutingTrace& trace, const Placement& placement, const SimConfig& config);

enum class Gating { top1, top2 };
enum class VolumeMethod { deepspeed, fastermoe, tamoe, exflow };
double volume_table1(int gpus, int tokens_per_gpu, int layers, double ratio, Gating gating,
                     VolumeMethod method);

const char* to_string(SimMode mode);
const char* to_string(Tier tier);

}  // namespace exflow
