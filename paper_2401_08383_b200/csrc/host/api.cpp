// api.cpp -- the exflow:: C++ surface that is not the solver: trace I/O
// (EXFLOW-TRACE v1), synthetic routes, affinity post-processing,
// the routing-replay report, placement JSON; count_transitions and simulate
// dispatch to the sm_100a kernels through the C-ABI.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <istream>
#include <ostream>
#include <sstream>

#include "exflow/exflow.hpp"
#include "exflow_c.h"

namespace exflow {

namespace {

void raise_status(exf_status st) {
    if (st == EXF_OK) return;
    const std::string msg = exf_last_error();
    if (st == EXF_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

std::vector<std::string> fields_of(const std::string& line) {
    std::vector<std::string> out;
    std::istringstream is(line);
    std::string f;
    while (is >> f) out.push_back(f);
    return out;
}

long to_long(const std::string& s, int line_no) {
    long v = 0;
    auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
    if (ec != std::errc{} || p != s.data() + s.size())
        throw ParseError("invalid token '" + s + "' at line " + std::to_string(line_no));
    return v;
}

}  // namespace

// ---------------------------------------------------------------- traces
void RoutingTrace::validate() const {
    if (num_experts < 1) throw std::invalid_argument("num_experts must be >= 1, got " + std::to_string(num_experts));
    if (num_layers < 2) throw std::invalid_argument("num_layers must be >= 2, got " + std::to_string(num_layers));
    if (paths.rows() < 1) throw std::invalid_argument("trace contains no token paths");
    if (paths.cols() != num_layers)
        throw std::invalid_argument("path length " + std::to_string(paths.cols()) + " != L=" +
                                    std::to_string(num_layers));
    for (std::int64_t i = 0; i < paths.size(); ++i)
        if (paths.data()[i] < 0 || paths.data()[i] >= num_experts)
            throw std::invalid_argument("expert id out of range [0," + std::to_string(num_experts) + ")");
}

RoutingTrace parse_trace(std::istream& in) {
    RoutingTrace t;
    std::vector<std::int32_t> ids;
    std::string line;
    int line_no = 0;
    bool magic = false, dims = false;
    long rows = 0;
    while (std::getline(in, line)) {
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        const bool blank = std::all_of(line.begin(), line.end(),
                                       [](unsigned char c) { return std::isspace(c); });
        if (blank || line[0] == '#') continue;
        if (!magic) {
            if (line != "EXFLOW-TRACE v1")
                throw ParseError("missing or unsupported EXFLOW-TRACE header at line " +
                                 std::to_string(line_no));
            magic = true;
            continue;
        }
        const auto f = fields_of(line);
        if (!dims) {
            if (f.size() != 4 || f[0] != "E" || f[2] != "L")
                throw ParseError("expected 'E <experts> L <layers>' at line " + std::to_string(line_no));
            const long e = to_long(f[1], line_no), l = to_long(f[3], line_no);
            if (e < 1) throw ParseError("E must be >= 1, got " + std::to_string(e) + " at line " + std::to_string(line_no));
            if (l < 2) throw ParseError("L must be >= 2, got " + std::to_string(l) + " at line " + std::to_string(line_no));
            t.num_experts = static_cast<int>(e);
            t.num_layers = static_cast<int>(l);
            dims = true;
            continue;
        }
        if (static_cast<int>(f.size()) != t.num_layers)
            throw ParseError("path length " + std::to_string(f.size()) + " != L=" +
                             std::to_string(t.num_layers) + " at line " + std::to_string(line_no));
        for (const auto& s : f) {
            const long id = to_long(s, line_no);
            if (id < 0 || id >= t.num_experts)
                throw ParseError("expert id " + std::to_string(id) + " out of range [0," +
                                 std::to_string(t.num_experts) + ") at line " + std::to_string(line_no));
            ids.push_back(static_cast<std::int32_t>(id));
        }
        ++rows;
    }
    if (!magic) throw ParseError("missing or unsupported EXFLOW-TRACE header at line 1");
    if (!dims) throw ParseError("missing 'E <experts> L <layers>' line");
    if (rows == 0) throw ParseError("trace contains no token paths");
    t.paths.resize(rows, t.num_layers);
    std::copy(ids.begin(), ids.end(), t.paths.data());
    return t;
}

RoutingTrace parse_trace(const std::string& text) {
    std::istringstream in(text);
    return parse_trace(in);
}

RoutingTrace load_trace(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open trace file: " + path.string());
    return parse_trace(in);
}

void write_trace(std::ostream& out, const RoutingTrace& t) {
    t.validate();
    out << "EXFLOW-TRACE v1\nE " << t.num_experts << " L " << t.num_layers << "\n";
    for (std::int64_t r = 0; r < t.paths.rows(); ++r) {
        for (std::int64_t j = 0; j < t.paths.cols(); ++j) out << (j ? " " : "") << t.paths(r, j);
        out << '\n';
    }
}

std::string serialize_trace(const RoutingTrace& t) {
    std::ostringstream os;
    write_trace(os, t);
    return os.str();
}

void save_trace(const std::filesystem::path& path, const RoutingTrace& t) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write trace file: " + path.string());
    write_trace(out, t);
}

TransitionCounts count_transitions(const RoutingTrace& trace, int gap) {
    trace.validate();
    if (gap < 1 || gap > trace.num_layers - 1)
        throw std::invalid_argument("gap " + std::to_string(gap) + " out of range [1," +
                                    std::to_string(trace.num_layers - 1) + "]");
    const int E = trace.num_experts, pairs = trace.num_layers - gap;
    std::vector<std::int64_t> flat(static_cast<std::size_t>(pairs) * E * E);
    std::vector<std::int64_t> totals(static_cast<std::size_t>(pairs) * E);
    raise_status(exf_count_transitions_host(trace.paths.data(), trace.paths.rows(), trace.num_layers,
                                            E, gap, flat.data(), totals.data()));
    TransitionCounts c;
    c.num_experts = E;
    c.num_layers = trace.num_layers;
    c.gap = gap;
    for (int j = 0; j < pairs; ++j) {
        CountMatrix m(E, E);
        std::copy_n(flat.data() + static_cast<std::size_t>(j) * E * E, E * E, m.data());
        c.matrices.push_back(std::move(m));
        c.row_totals.emplace_back(totals.begin() + j * E, totals.begin() + (j + 1) * E);
    }
    return c;
}

AffinityMatrix conditional_probabilities(const TransitionCounts& counts) {
    AffinityMatrix a;
    a.num_experts = counts.num_experts;
    a.num_layers = counts.num_layers;
    a.gap = counts.gap;
    for (std::size_t j = 0; j < counts.matrices.size(); ++j) {
        const CountMatrix& m = counts.matrices[j];
        ProbMatrix p(m.rows(), m.cols(), 0.0);
        SeenMask seen(static_cast<std::size_t>(m.rows()), false);
        for (std::int64_t r = 0; r < m.rows(); ++r) {
            const std::int64_t tot = counts.row_totals[j][r];
            if (tot <= 0) continue;
            seen[r] = true;
            for (std::int64_t b = 0; b < m.cols(); ++b)
                p(r, b) = static_cast<double>(m(r, b)) / static_cast<double>(tot);
        }
        a.matrices.push_back(std::move(p));
        a.seen.push_back(std::move(seen));
    }
    return a;
}

int most_affiliated(const AffinityMatrix& a, int source_layer, int expert) {
    if (source_layer < 0 || source_layer >= a.num_layer_pairs())
        throw std::invalid_argument("source layer " + std::to_string(source_layer) + " out of range [0," +
                                    std::to_string(a.num_layer_pairs()) + ")");
    if (expert < 0 || expert >= a.num_experts)
        throw std::invalid_argument("expert " + std::to_string(expert) + " out of range");
    if (!a.seen[source_layer][expert])
        throw std::invalid_argument("no observations for expert " + std::to_string(expert) +
                                    " at layer " + std::to_string(source_layer));
    const ProbMatrix& m = a.matrices[source_layer];
    int best = 0;
    for (int b = 1; b < m.cols(); ++b)
        if (m(expert, b) > m(expert, best)) best = b;  // first maximum wins
    return best;
}

std::string export_heatmap_csv(const AffinityMatrix& a, int source_layer) {
    if (source_layer < 0 || source_layer >= a.num_layer_pairs())
        throw std::invalid_argument("source layer " + std::to_string(source_layer) + " out of range [0," +
                                    std::to_string(a.num_layer_pairs()) + ")");
    const ProbMatrix& m = a.matrices[source_layer];
    std::string out;
    char buf[32];
    for (std::int64_t r = 0; r < m.rows(); ++r) {
        for (std::int64_t b = 0; b < m.cols(); ++b) {
            std::snprintf(buf, sizeof(buf), "%.6f", m(r, b));
            if (b) out += ',';
            out += buf;
        }
        out += '\n';
    }
    return out;
}

// ---------------------------------------------------------------- synth
void SynthConfig::validate() const {
    if (num_experts < 1) throw std::invalid_argument("num_experts must be >= 1");
    if (num_layers < 2) throw std::invalid_argument("num_layers must be >= 2");
    if (num_tokens < 1) throw std::invalid_argument("num_tokens must be >= 1");
    if (affinity_strength < 0.0 || affinity_strength > 1.0)
        throw std::invalid_argument("affinity_strength must be in [0,1]");
    if (planted_groups < 1 || num_experts % planted_groups != 0)
        throw std::invalid_argument("planted_groups " + std::to_string(planted_groups) +
                                    " must divide num_experts " + std::to_string(num_experts));
}

RoutingTrace generate_markov_trace(const SynthConfig& c) {
    c.validate();
    RoutingTrace t;
    t.num_experts = c.num_experts;
    t.num_layers = c.num_layers;
    t.paths.resize(c.num_tokens, c.num_layers);
    const int block = c.group_size();
    Rng rng(c.seed);
    // draw order of the reference generator (proj/src/synth.cpp:40-51)
    for (int r = 0; r < c.num_tokens; ++r) {
        std::int32_t* row = t.paths.row_ptr(r);
        int e = rng.below_int(c.num_experts);
        row[0] = e;
        for (int j = 1; j < c.num_layers; ++j) {
            const bool stay = rng.uniform01() < c.affinity_strength;
            e = stay ? (e / block) * block + rng.below_int(block) : rng.below_int(c.num_experts);
            row[j] = e;
        }
    }
    return t;
}

double expected_planted_locality(const SynthConfig& c) {
    c.validate();
    return c.affinity_strength + (1.0 - c.affinity_strength) / c.planted_groups;
}

// ---------------------------------------------------------------- simulator
void SimConfig::validate() const {
    topology.validate();
    if (tokens_per_gpu < 1) throw std::invalid_argument("tokens_per_gpu must be >= 1");
    if (iterations < 1) throw std::invalid_argument("iterations must be >= 1");
}

std::vector<LayerHop> token_hops(std::span<const std::int32_t> path, int home, const Placement& p,
                                 SimMode mode, const Topology& topo) {
    topo.validate();
    p.validate();
    if (static_cast<int>(path.size()) != p.num_layers)
        throw std::invalid_argument("path length does not match placement layers");
    if (topo.num_nodes != p.num_nodes || topo.gpus_per_node != p.gpus_per_node)
        throw std::invalid_argument("topology grid does not match placement grid");
    if (home < 0 || home >= topo.total_gpus()) throw std::invalid_argument("home gpu out of range");
    auto tier = [&](int a, int b) {
        return a == b ? Tier::intra_gpu
                      : (topo.node_of(a) == topo.node_of(b) ? Tier::intra_node : Tier::inter_node);
    };
    std::vector<LayerHop> out;
    int at = home;
    for (int j = 0; j < static_cast<int>(path.size()); ++j) {
        if (path[j] < 0 || path[j] >= p.num_experts)
            throw std::invalid_argument("expert id out of range in path");
        const int g = p.gpu_of(j, path[j]);
        LayerHop h;
        if (mode == SimMode::vanilla) {  // dispatch + return home (sim.cpp:60-64)
            h.crossed = g != home;
            h.tier = tier(home, g);
            h.hops = h.crossed ? 2 : 0;
        } else {  // coherent: move once, stay (sim.cpp:65-71)
            h.crossed = g != at;
            h.tier = tier(at, g);
            h.hops = h.crossed ? 1 : 0;
            at = g;
        }
        out.push_back(h);
    }
    return out;
}

SimReport simulate(const RoutingTrace& trace, const Placement& placement, const SimConfig& config) {
    trace.validate();
    placement.validate();
    config.validate();
    if (trace.num_experts != placement.num_experts || trace.num_layers != placement.num_layers)
        throw std::invalid_argument("trace and placement shapes disagree");
    if (config.topology.num_nodes != placement.num_nodes ||
        config.topology.gpus_per_node != placement.gpus_per_node)
        throw std::invalid_argument("topology grid does not match placement grid");
    const int T = trace.num_tokens();
    if (config.homes && static_cast<int>(config.homes->size()) != T)
        throw std::invalid_argument("homes must list one GPU per token");
    exf_sim_report r{};
    raise_status(exf_simulate_host(trace.paths.data(), T, trace.num_layers, trace.num_experts,
                                   placement.assign.data(), config.topology.num_nodes,
                                   config.topology.gpus_per_node, config.topology.intra_node_hop_cost,
                                   config.topology.inter_node_hop_cost, config.tokens_per_gpu,
                                   config.mode == SimMode::vanilla ? 0 : 1,
                                   config.homes ? config.homes->data() : nullptr, &r));
    SimReport s;
    s.hops_intra_node = r.hops_intra_node;
    s.hops_inter_node = r.hops_inter_node;
    s.locality_gpu = r.locality_gpu;
    s.locality_node = r.locality_node;
    s.p = r.p;
    s.p_star = r.p_star;
    s.alltoall_count = r.alltoall_count;
    s.allgather_count = r.allgather_count;
    s.setup_allgather_count = r.setup_allgather_count;
    s.volume_units = r.volume_units;
    s.estimated_latency = r.estimated_latency;
    return s;
}

double volume_table1(int gpus, int n, int layers, double ratio, Gating gating, VolumeMethod m) {
    if (gpus < 1 || n < 1 || layers < 1)
        throw std::invalid_argument("gpus, tokens_per_gpu and layers must be positive");
    if (!(ratio >= 0.0 && ratio <= 1.0)) throw std::invalid_argument("ratio must be in [0,1]");
    const double g = gpus, t = n, l = layers;
    if (m == VolumeMethod::exflow)
        return gating == Gating::top1 ? g * t * (l * ratio + g) : g * t * (2.0 * l * ratio + g);
    return (gating == Gating::top1 ? 2.0 : 4.0) * g * t * l * ratio;
}

const char* to_string(SimMode m) { return m == SimMode::vanilla ? "vanilla" : "coherent"; }
const char* to_string(Tier t) {
    return t == Tier::intra_gpu ? "intra_gpu" : (t == Tier::intra_node ? "intra_node" : "inter_node");
}

// ---------------------------------------------------------------- placement JSON
namespace {

struct JsonCursor {
    const std::string& s;
    std::size_t i = 0;
    void ws() {
        while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
    }
    void expect(char c) {
        ws();
        if (i >= s.size() || s[i] != c)
            throw std::runtime_error(std::string("placement JSON: expected '") + c + "'");
        ++i;
    }
    bool peek(char c) {
        ws();
        return i < s.size() && s[i] == c;
    }
    std::string key() {
        expect('"');
        const std::size_t b = i;
        while (i < s.size() && s[i] != '"') ++i;
        std::string k = s.substr(b, i - b);
        ++i;
        return k;
    }
    long number() {
        ws();
        const std::size_t b = i;
        if (i < s.size() && (s[i] == '-' || s[i] == '+')) ++i;
        while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) ++i;
        if (b == i) throw std::runtime_error("placement JSON: expected an integer");
        return std::stol(s.substr(b, i - b));
    }
};

}  // namespace

Placement placement_from_json(const std::string& text) {
    JsonCursor c{text};
    Placement p;
    std::vector<std::vector<int>> rows;
    bool have[5] = {false, false, false, false, false};
    c.expect('{');
    while (!c.peek('}')) {
        const std::string k = c.key();
        c.expect(':');
        if (k == "assign") {
            c.expect('[');
            while (!c.peek(']')) {
                std::vector<int> row;
                c.expect('[');
                while (!c.peek(']')) {
                    row.push_back(static_cast<int>(c.number()));
                    if (c.peek(',')) c.expect(',');
                }
                c.expect(']');
                rows.push_back(std::move(row));
                if (c.peek(',')) c.expect(',');
            }
            c.expect(']');
            have[4] = true;
        } else {
            const int v = static_cast<int>(c.number());
            if (k == "experts") p.num_experts = v, have[0] = true;
            else if (k == "layers") p.num_layers = v, have[1] = true;
            else if (k == "nodes") p.num_nodes = v, have[2] = true;
            else if (k == "gpus_per_node") p.gpus_per_node = v, have[3] = true;
        }
        if (c.peek(',')) c.expect(',');
    }
    c.expect('}');
    for (bool h : have)
        if (!h) throw std::runtime_error("placement JSON: missing key");
    if (static_cast<int>(rows.size()) != p.num_layers)
        throw std::invalid_argument("placement assign table has wrong layer count");
    p.assign.resize(p.num_layers, p.num_experts);
    for (int j = 0; j < p.num_layers; ++j) {
        if (static_cast<int>(rows[j].size()) != p.num_experts)
            throw std::invalid_argument("placement assign row has wrong expert count");
        for (int e = 0; e < p.num_experts; ++e) p.assign(j, e) = rows[j][e];
    }
    p.validate();
    return p;
}

Placement load_placement(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open placement file: " + path.string());
    std::stringstream ss;
    ss << in.rdbuf();
    return placement_from_json(ss.str());
}

std::string placement_to_json(const Placement& p) {
    std::ostringstream os;
    os << "{\"experts\":" << p.num_experts << ",\"layers\":" << p.num_layers
       << ",\"nodes\":" << p.num_nodes << ",\"gpus_per_node\":" << p.gpus_per_node << ",\"assign\":[";
    for (int j = 0; j < p.num_layers; ++j) {
        os << (j ? ",[" : "[");
        for (int e = 0; e < p.num_experts; ++e) os << (e ? "," : "") << p.assign(j, e);
        os << "]";
    }
    os << "]}";
    return os.str();
}

}  // namespace exflow
