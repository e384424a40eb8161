// placement_table.cpp -- the expert-placement table (which GPU holds expert e
// of layer j) and its baselines. The fused layer kernel reads the same table
// as its routing table (model.cu uploads gpu_of / slot_of per layer).
//
// Contracts (messages and error precedence are part of them):
//   Topology::validate           proj/src/placement.cpp:425-432
//   Placement::validate          proj/src/placement.cpp:434-470
//   regrid                       proj/src/placement.cpp:472-480
//   contiguous_placement         proj/src/placement.cpp:482-502 (vanilla EP)
//   random_placement             proj/src/placement.cpp:504-526
//   objective_crossings          proj/src/placement.cpp:618-643
//   balanced_assignment_count    proj/src/placement.cpp:645-667
#include <string>

#include "exflow/exflow.hpp"

namespace exflow {
namespace {

void require(bool ok, const std::string& msg) {
    if (!ok) throw std::invalid_argument(msg);
}

// A placement of `topology`'s grid with every layer's labels produced by
// `layer_labels(j, labels)`; validated before it is returned.
template <class F>
Placement build_grid_placement(int num_experts, int num_layers, const Topology& topology, F&& layer_labels) {
    topology.validate();
    require(num_experts % topology.total_gpus() == 0, "num_experts not divisible by total GPUs");
    Placement p;
    p.num_experts = num_experts;
    p.num_layers = num_layers;
    p.num_nodes = topology.num_nodes;
    p.gpus_per_node = topology.gpus_per_node;
    p.assign.resize(num_layers, num_experts);
    std::vector<int> labels(num_experts);
    for (int j = 0; j < num_layers; ++j) {
        layer_labels(j, labels);
        std::copy(labels.begin(), labels.end(), p.assign.row_ptr(j));
    }
    p.validate();
    return p;
}

// group g holds experts [g*cap, (g+1)*cap)
void fill_blocks(std::vector<int>& labels, int groups) {
    const int cap = static_cast<int>(labels.size()) / groups;
    for (size_t i = 0; i < labels.size(); ++i) labels[i] = static_cast<int>(i) / cap;
}

}  // namespace

void Topology::validate() const {
    require(num_nodes >= 1 && gpus_per_node >= 1,
            "topology must have at least one node and one GPU per node");
    require(intra_node_hop_cost >= 0.0 && inter_node_hop_cost >= intra_node_hop_cost,
            "hop costs must satisfy inter >= intra >= 0");
}

void Placement::validate() const {
    require(num_experts >= 1 && num_layers >= 1, "placement must cover at least one expert and layer");
    require(num_nodes >= 1 && gpus_per_node >= 1, "placement grid must be at least 1x1");
    require(assign.rows() == num_layers && assign.cols() == num_experts, "placement table shape mismatch");
    const int gpus = total_gpus();
    require(num_experts % gpus == 0, "num_experts " + std::to_string(num_experts) +
                                         " not divisible by total GPUs " + std::to_string(gpus));
    const int want = num_experts / gpus;
    // per layer: ids first (first bad id in expert order), then balance
    // (first unbalanced GPU in id order)
    std::vector<int> load(gpus);
    for (int j = 0; j < num_layers; ++j) {
        load.assign(gpus, 0);
        const int* row = assign.row_ptr(j);
        for (int e = 0; e < num_experts; ++e) {
            require(row[e] >= 0 && row[e] < gpus, "gpu id " + std::to_string(row[e]) + " out of range [0," +
                                                      std::to_string(gpus) + ") at layer " + std::to_string(j));
            ++load[row[e]];
        }
        for (int g = 0; g < gpus; ++g)
            require(load[g] == want, "layer " + std::to_string(j) + " places " + std::to_string(load[g]) +
                                         " experts on gpu " + std::to_string(g) + ", expected " +
                                         std::to_string(want));
    }
}

Placement regrid(Placement placement, int num_nodes, int gpus_per_node) {
    require(num_nodes * gpus_per_node == placement.total_gpus(), "regrid must preserve the total GPU count");
    placement.num_nodes = num_nodes;
    placement.gpus_per_node = gpus_per_node;
    placement.validate();
    return placement;
}

Placement contiguous_placement(int num_experts, int num_layers, const Topology& topology) {
    const int gpus = topology.total_gpus();
    return build_grid_placement(num_experts, num_layers, topology,
                                [&](int, std::vector<int>& labels) { fill_blocks(labels, gpus); });
}

Placement random_placement(int num_experts, int num_layers, const Topology& topology,
                           std::uint64_t seed) {
    const int gpus = topology.total_gpus();
    Rng rng(seed);  // one stream over all layers, one shuffle per layer
    return build_grid_placement(num_experts, num_layers, topology, [&](int, std::vector<int>& labels) {
        fill_blocks(labels, gpus);
        shuffle(std::span<int>(labels), rng);
    });
}

double objective_crossings(const TransitionCounts& counts, const Placement& placement, Level level) {
    require(counts.num_experts == placement.num_experts && counts.num_layers == placement.num_layers,
            "counts and placement shapes disagree");
    const int E = counts.num_experts;
    // group of every expert at both ends of the pair, at the requested level
    std::vector<int> src(E), dst(E);
    auto group = [&](int g) { return level == Level::node ? placement.node_of(g) : g; };
    double total = 0.0;
    for (int j = 0; j < counts.num_layer_pairs(); ++j) {
        for (int e = 0; e < E; ++e) {
            src[e] = group(placement.assign(j, e));
            dst[e] = group(placement.assign(j + counts.gap, e));
        }
        const CountMatrix& m = counts.matrices[j];
        for (int a = 0; a < E; ++a) {
            const std::int64_t* row = m.row_ptr(a);
            for (int b = 0; b < E; ++b)
                if (row[b] != 0 && src[a] != dst[b]) total += static_cast<double>(row[b]);
        }
    }
    return total;
}

long balanced_assignment_count(int items, int parts, long cap) {
    require(parts >= 1 && items >= 1 && items % parts == 0, "items must be divisible by parts");
    // items! / (k!)^parts = prod_{m=1..parts} C(m*k, k), saturating at cap+1:
    // every partial binomial is <= the final count, so the walk stops as soon
    // as any partial value passes the cap
    const int k = items / parts;
    const unsigned __int128 limit = static_cast<unsigned __int128>(cap);
    unsigned __int128 count = 1;
    for (int m = 1; m <= parts; ++m) {
        unsigned __int128 binom = 1;  // C((m-1)k + i, i) for i = 1..k
        for (int i = 1; i <= k; ++i) {
            binom = binom * static_cast<unsigned>((m - 1) * k + i) / static_cast<unsigned>(i);
            if (binom > limit) return cap + 1;
        }
        count *= binom;
        if (count > limit) return cap + 1;
    }
    return static_cast<long>(count);
}

}  // namespace exflow
