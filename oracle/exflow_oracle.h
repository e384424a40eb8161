/*
 * exflow_oracle.h -- CPU restatement of the ExFlow reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in paper_2401_08383_b200/ links, imports
 * or calls this code; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, and only as the checker or as
 * the timed CPU baseline.
 *
 * The reference (/root/reference/proj) cannot be built here: it needs Eigen3
 * (proj/CMakeLists.txt:12) and vendored CLI11/doctest headers that are not
 * shipped. This file restates the reference's own loops in plain C; every
 * function cites the file:line it follows. Parity of this restatement is
 * pinned against the reference's golden vectors (tests/test_oracle_golden.py).
 *
 * Layouts (all row-major, plain pointers):
 *   paths   : [T][L] int32               (reference PathMatrix, RowMajor)
 *   counts  : [L-gap][E][E] int64        (reference CountMatrix is col-major;
 *                                         element (a,b) of pair j is
 *                                         counts[(j*E + a)*E + b] here)
 *   assign  : [L][E] int32 GPU ids       (reference MatrixXi assign(j, e))
 */
#ifndef EXFLOW_ORACLE_H
#define EXFLOW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng: proj/include/exflow/rng.hpp:17-98 ---------------------------- */
typedef struct { uint64_t s[4]; } orc_rng;
void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
uint64_t orc_rng_below(orc_rng* r, uint64_t bound);
double orc_rng_uniform01(orc_rng* r);
uint64_t orc_splitmix64(uint64_t* x);
uint64_t orc_seed_stream(uint64_t seed, uint64_t stream);
void orc_shuffle_int(int32_t* v, int64_t n, orc_rng* r);

/* ---- synth: proj/src/synth.cpp:11-58 ----------------------------------- */
int orc_generate_markov_trace(int32_t E, int32_t L, int64_t T, double alpha,
                              int32_t groups, uint64_t seed, int32_t* paths);
double orc_expected_planted_locality(double alpha, int32_t groups);

/* ---- trace: proj/src/trace.cpp ------------------------------------------ */
int orc_validate_trace(const int32_t* paths, int64_t T, int32_t L, int32_t E);
int orc_count_transitions(const int32_t* paths, int64_t T, int32_t L, int32_t E,
                          int32_t gap, int64_t* counts, int64_t* row_totals);
int orc_count_transitions_mt(const int32_t* paths, int64_t T, int32_t L, int32_t E,
                             int32_t gap, int64_t* counts, int64_t* row_totals,
                             int32_t threads);
void orc_conditional_probabilities(const int64_t* counts, const int64_t* row_totals,
                                   int32_t pairs, int32_t E, double* probs,
                                   uint8_t* seen);
int orc_most_affiliated(const double* probs, const uint8_t* seen, int32_t pairs,
                        int32_t E, int32_t source_layer, int32_t expert);
int orc_permute_experts(const int32_t* paths, int64_t T, int32_t L, int32_t E,
                        const int32_t* perm, int32_t* out);

/* ---- placement: proj/src/placement.cpp:425-526, 618-667 ---------------- */
int orc_validate_placement(const int32_t* assign, int32_t L, int32_t E, int32_t gpus);
int orc_contiguous_placement(int32_t E, int32_t L, int32_t gpus, int32_t* assign);
int orc_random_placement(int32_t E, int32_t L, int32_t gpus, uint64_t seed,
                         int32_t* assign);
double orc_objective_crossings(const int64_t* counts, int32_t pairs, int32_t E,
                               int32_t gap, const int32_t* assign,
                               int32_t gpus_per_node, int32_t level_node);
int64_t orc_balanced_assignment_count(int32_t items, int32_t parts, int64_t cap);
/* test-only brute force: proj/tests/oracle_util.hpp:18-65 */
double orc_brute_force_optimum(const int64_t* counts, int32_t L, int32_t E,
                               int32_t parts);

/* ---- comm simulator: proj/src/sim.cpp:34-191 --------------------------- */
enum { ORC_VANILLA = 0, ORC_COHERENT = 1 };
typedef struct {
    int64_t hops_intra_node;
    int64_t hops_inter_node;
    int64_t gpu_local_events;
    int64_t node_local_events;
    int64_t away_from_home_events;
    int64_t coherent_moves;
    double locality_gpu;
    double locality_node;
    double p;
    double p_star;
    int64_t alltoall_count;
    int64_t allgather_count;
    int64_t setup_allgather_count;
    double volume_units;
    double estimated_latency;
} orc_sim_report;

/* hops_out[j] = hop count, crossed_out[j] = 0/1, tier_out[j] = 0/1/2 */
int orc_token_hops(const int32_t* path, int32_t L, int32_t home,
                   const int32_t* assign, int32_t E, int32_t num_nodes,
                   int32_t gpus_per_node, int32_t mode, int32_t* hops_out,
                   int32_t* crossed_out, int32_t* tier_out);
int orc_simulate(const int32_t* paths, int64_t T, int32_t L, int32_t E,
                 const int32_t* assign, int32_t num_nodes, int32_t gpus_per_node,
                 double intra_cost, double inter_cost, int32_t tokens_per_gpu,
                 int32_t mode, const int32_t* homes, orc_sim_report* out);
int orc_simulate_mt(const int32_t* paths, int64_t T, int32_t L, int32_t E,
                    const int32_t* assign, int32_t num_nodes, int32_t gpus_per_node,
                    double intra_cost, double inter_cost, int32_t tokens_per_gpu,
                    int32_t mode, const int32_t* homes, orc_sim_report* out,
                    int32_t threads);
/* gating: 0 top1, 1 top2; method: 0 deepspeed 1 fastermoe 2 tamoe 3 exflow */
double orc_volume_table1(int32_t gpus, int32_t tokens_per_gpu, int32_t layers,
                         double ratio, int32_t gating, int32_t method);

/* ---- model oracle (no reference implementation: SPEC.md:8, :108) ------- */
/* See exflow_model_oracle.c for the arithmetic contract. */
float orc_bf16_to_f32(uint16_t v);
uint16_t orc_f32_to_bf16(float f);
void orc_gate_logits(const uint16_t* x, const uint16_t* wg, int32_t d, int32_t E,
                     float* logits);
int orc_gate_top1(const float* logits, int32_t E, float* prob);
void orc_expert_ffn(const uint16_t* x, const uint16_t* w1, const uint16_t* b1,
                    const uint16_t* w2, const uint16_t* b2, int32_t d, int32_t dff,
                    float prob, uint16_t* out, float* out_f32);
/* fp32 mode: the same fixed-order fmaf gate on fp32 inputs (products are
 * rounded inside the fused multiply-add exactly as on the device), and the
 * expert FFN on fp32 inputs evaluated in fp64 with no intermediate rounding
 * (the reference the 1e-5 fp32 bar is measured against). */
void orc_gate_logits_f32(const float* x, const float* wg, int32_t d, int32_t E, float* logits);
void orc_expert_ffn_f32(const float* x, const float* w1, const float* b1, const float* w2,
                        const float* b2, int32_t d, int32_t dff, float prob, double* out);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
