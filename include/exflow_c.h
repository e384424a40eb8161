/*
 * exflow_c.h -- C-ABI drop-in boundary of the B200-native ExFlow hot path.
 *
 * The reference has no FFI: its boundary is the in-process C++ API of
 * namespace exflow. Each entry point below replaces one
 * reference function (file:line under /root/reference/proj) or adds the model
 * surface the reference leaves out (gate/FFN/collectives: SPEC.md:8, :108,
 * :343). The headers in include/exflow/ restore the reference C++ signatures on top of
 * this header; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - plain pointers and sizes; no torch or Eigen types.
 *  - d_* arguments are DEVICE pointers (caller-owned); h_* are host pointers.
 *  - exf_stream_t is a cudaStream_t passed as void* (NULL = legacy stream).
 *  - every call returns an exf_status; on error exf_last_error() (thread
 *    local) carries the message. Status values mirror the reference's error
 *    classes: EXF_INVALID <-> std::invalid_argument (CLI exit 2,
 *    proj/tools/exflow.cpp:646-652), EXF_RUNTIME <-> std::runtime_error /
 *    ParseError (exit 1).
 *  - all layouts are row-major:
 *      paths  [T][L] int32          (reference PathMatrix, trace.hpp:23)
 *      counts [L-gap][E][E] int64   (reference CountMatrix (a,b) of pair j;
 *                                    the reference stores it column-major)
 *      assign [L][E] int32 GPU ids  (reference Placement::assign(j, e))
 */
#ifndef EXFLOW_C_H
#define EXFLOW_C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* exf_stream_t;

typedef enum {
    EXF_OK = 0,
    EXF_RUNTIME = 1,  /* std::runtime_error / ParseError            */
    EXF_INVALID = 2,  /* std::invalid_argument                      */
    EXF_CUDA = 3,     /* CUDA runtime / launch / kernel fault        */
    EXF_COMM = 4      /* peer (NVLink) exchange failure or timeout   */
} exf_status;

/* Thread-local message of the last failing call on this thread. */
const char* exf_last_error(void);
/* Library version (major*10000 + minor*100 + patch). */
int32_t exf_version(void);
/* 1 if the library was built for sm_100a and a compute-capability-10.0 GPU is
 * visible, 0 otherwise (no error). */
int32_t exf_device_ok(void);

/* ------------------------------------------------------------------------
 * Kernel (5) -- inter-layer affinity histogram (bulk rebuild).
 * Replaces exflow::count_transitions (proj/include/exflow/trace.hpp:71,
 * proj/src/trace.cpp:191-215): counts[j][a][b] = #{t : paths[t][j] == a and
 * paths[t][j+gap] == b}, row_totals[j][a] = sum_b counts[j][a][b].
 * Bit-exact (integer). Validation errors match trace.cpp:53-70 / :193-196.
 * d_workspace must hold exf_count_transitions_workspace_bytes(...) bytes.
 * ---------------------------------------------------------------------- */
int64_t exf_count_transitions_workspace_bytes(int64_t T, int32_t L, int32_t E, int32_t gap);
exf_status exf_count_transitions(const int32_t* d_paths, int64_t T, int32_t L, int32_t E,
                                 int32_t gap, int64_t* d_counts, int64_t* d_row_totals,
                                 void* d_workspace, exf_stream_t stream);
/* Host-buffer convenience (H2D, kernel, D2H inside; synchronous).
 * Validates ids on the host first, like RoutingTrace::validate. */
exf_status exf_count_transitions_host(const int32_t* h_paths, int64_t T, int32_t L, int32_t E,
                                      int32_t gap, int64_t* h_counts, int64_t* h_row_totals);

/* ------------------------------------------------------------------------
 * Routing replay -- the per-token/per-layer hot loop of exflow::simulate
 * (proj/src/sim.cpp:110-145). Counters are exact integer sums; the ratios and
 * collective counts of SimReport (sim.cpp:147-167) are derived on the host
 * (exf_sim_report_from_counters).
 * homes may be NULL (round-robin t % G, sim.cpp:111). mode: 0 vanilla,
 * 1 coherent (sim.hpp:14).
 * ---------------------------------------------------------------------- */
typedef struct {
    int64_t gpu_local_events;
    int64_t node_local_events;
    int64_t away_from_home_events;
    int64_t coherent_moves;
    int64_t hops_intra_node;
    int64_t hops_inter_node;
} exf_sim_counters;

typedef struct { /* proj/include/exflow/sim.hpp:49-63 */
    int64_t hops_intra_node;
    int64_t hops_inter_node;
    double locality_gpu;
    double locality_node;
    double p;
    double p_star;
    int64_t alltoall_count;
    int64_t allgather_count;
    int64_t setup_allgather_count;
    double volume_units;
    double estimated_latency;
} exf_sim_report;

exf_status exf_route_replay(const int32_t* d_paths, const int32_t* d_homes,
                            const int32_t* d_assign, int64_t T, int32_t L, int32_t E,
                            int32_t num_nodes, int32_t gpus_per_node, int32_t mode,
                            exf_sim_counters* d_out, exf_stream_t stream);
exf_status exf_sim_report_from_counters(const exf_sim_counters* counters, int64_t T,
                                        int32_t L, int32_t num_nodes, int32_t gpus_per_node,
                                        double intra_node_hop_cost,
                                        double inter_node_hop_cost, int32_t tokens_per_gpu,
                                        int32_t mode, exf_sim_report* out);
/* Host-buffer convenience: validates like simulate (sim.cpp:78-105), runs the
 * replay kernel, fills the report. homes may be NULL. */
exf_status exf_simulate_host(const int32_t* h_paths, int64_t T, int32_t L, int32_t E,
                             const int32_t* h_assign, int32_t num_nodes, int32_t gpus_per_node,
                             double intra_node_hop_cost, double inter_node_hop_cost,
                             int32_t tokens_per_gpu, int32_t mode, const int32_t* h_homes,
                             exf_sim_report* out);

/* ------------------------------------------------------------------------
 * Host (CPU) placement table and integer-program placement solver. These
 * stay on the CPU (BASELINE.json north_star); they consume the GPU
 * histogram. counts are gap-1 counts [L-1][E][E]; assign is [L][E].
 * ---------------------------------------------------------------------- */
typedef struct { /* proj/include/exflow/placement.hpp:106-114 */
    int32_t restarts;           /* 8 */
    int64_t max_iters;          /* 0 -> 20000*L */
    double initial_temperature; /* 0 -> mean positive weight */
    double cooling;             /* 0.999 */
    uint64_t seed;
} exf_anneal_params;

typedef struct { /* proj/include/exflow/placement.hpp:120-130 */
    char solver[32];
    double objective;
    uint64_t seed;
    int64_t iterations;
    int32_t restarts;
    int32_t has_optimality_gap;
    double optimality_gap;
    int32_t has_tiers;
    double inter_node_crossings;
    double intra_node_crossings;
    double weighted_cost;
} exf_solve_report;

/* contiguous_placement, proj/src/placement.cpp:482-502 */
exf_status exf_contiguous_placement(int32_t E, int32_t L, int32_t num_nodes,
                                    int32_t gpus_per_node, int32_t* h_assign);
/* random_placement, proj/src/placement.cpp:504-526 */
exf_status exf_random_placement(int32_t E, int32_t L, int32_t num_nodes, int32_t gpus_per_node,
                                uint64_t seed, int32_t* h_assign);
/* Placement::validate, proj/src/placement.cpp:434-470 */
exf_status exf_validate_placement(const int32_t* h_assign, int32_t L, int32_t E,
                                  int32_t num_nodes, int32_t gpus_per_node);
/* objective_crossings, proj/src/placement.cpp:618-643; level 0 node, 1 gpu */
exf_status exf_objective_crossings(const int64_t* h_counts, int32_t L, int32_t E, int32_t gap,
                                   const int32_t* h_assign, int32_t num_nodes,
                                   int32_t gpus_per_node, int32_t level, double* out);
/* balanced_assignment_count, proj/src/placement.cpp:645-667 (-1 on bad args) */
int64_t exf_balanced_assignment_count(int32_t items, int32_t parts, int64_t cap);
/* solve_exact_dp, proj/src/placement.cpp:684-700 */
exf_status exf_solve_exact_dp(const int64_t* h_counts, int32_t L, int32_t E, int32_t partitions,
                              int64_t state_cap, int32_t* h_assign, exf_solve_report* report);
/* solve_local_search, proj/src/placement.cpp:702-718 */
exf_status exf_solve_local_search(const int64_t* h_counts, int32_t L, int32_t E,
                                  int32_t partitions, const exf_anneal_params* params,
                                  int32_t* h_assign, exf_solve_report* report);
/* solve_staged, proj/src/placement.cpp:720-821 */
exf_status exf_solve_staged(const int64_t* h_counts, int32_t L, int32_t E, int32_t num_nodes,
                            int32_t gpus_per_node, double intra_node_hop_cost,
                            double inter_node_hop_cost, const exf_anneal_params* params,
                            int64_t state_cap, int32_t* h_assign, exf_solve_report* report);
/* generate_markov_trace, proj/src/synth.cpp:30-53 (forced-routing inputs) */
exf_status exf_generate_markov_trace(int32_t E, int32_t L, int64_t T, double alpha,
                                     int32_t planted_groups, uint64_t seed, int32_t* h_paths);

#ifdef __cplusplus
}
#endif
#endif /* EXFLOW_C_H */
