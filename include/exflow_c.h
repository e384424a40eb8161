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
 * d_workspace: exf_count_transitions_workspace_bytes(...) bytes: 0 (may be
 * NULL) when the per-CTA counters flush with exact 64-bit atomics, else the
 * per-CTA u16 partials summed by a second kernel (large E).
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

/* token_hops, proj/src/sim.cpp:34-76 (proj/include/exflow/sim.hpp:28-30):
 * the per-token hop semantics the replay kernel sums. h_path [L] expert ids
 * of one token, its home GPU, h_assign [L][E]; per layer j: h_crossed[j]
 * (0/1), h_tier[j] (0 intra-GPU, 1 intra-node, 2 inter-node) and h_hops[j]
 * (vanilla: 2 when the expert is away from home; coherent: 1 when it is
 * away from the token's current GPU, which then becomes the token's GPU).
 * Host-only; validation and messages as the reference. */
exf_status exf_token_hops(const int32_t* h_path, int32_t L, int32_t home, const int32_t* h_assign,
                          int32_t E, int32_t num_nodes, int32_t gpus_per_node, int32_t mode,
                          int32_t* h_crossed, int32_t* h_tier, int32_t* h_hops);

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

/* ------------------------------------------------------------------------
 * Context-coherent expert-parallel MoE decode (the model surface the
 * reference leaves out; protocol of proj/src/sim.cpp:65-71
 * and :159-162). One handle per rank/GPU. Per MoE layer: fused gate +
 * top-1 + affinity histogram (kernel 1+5), atomic-free bucketing fused with
 * the single dispatch exchange over NVLink (kernels 2+3), grouped expert FFN
 * on tcgen05 (kernel 4); tokens stay on their expert's GPU (no combine).
 * Per step: context AllGather of the step's token states (kernel 3b).
 * Tokens: rank r owns home tokens r + G*i, i < tokens_per_gpu (round robin,
 * sim.cpp:111). x_in is this rank's [B][d] home tokens; the output is the
 * [G*B][d] final states of ALL tokens, indexed by token id. Element type:
 * bf16, or fp32 with dtype = EXF_DTYPE_F32 (every "bf16" buffer below --
 * x_in, output, weights, resident rows -- is then fp32).
 * ---------------------------------------------------------------------- */
typedef struct exf_model exf_model;

typedef struct { /* in the style of SynthConfig (proj/include/exflow/synth.hpp:13-23) */
    int32_t num_experts;     /* E (divisible by world_size, <= 64) */
    int32_t num_layers;      /* L MoE layers (>= 2) */
    int32_t d_model;         /* d (multiple of 256) */
    int32_t d_ffn;           /* expert hidden width (multiple of 128) */
    int32_t top_k;           /* must be 1 (all paper models are top-1) */
    int32_t tokens_per_gpu;  /* B decode sequences per rank */
    int32_t world_size;      /* G ranks (<= 8, one node) */
    int32_t rank;
    uint64_t seed;           /* weight-init seed */
    float init_std;          /* expert weight std (0.02) */
    float gate_affinity;     /* planted inter-layer gate correlation rho in [0,1] */
    int32_t ep_mode;         /* EXF_EP_COHERENT (ExFlow: tokens stay on their expert's GPU,
                                one exchange per layer) or EXF_EP_VANILLA (dispatch + combine
                                back to the home GPU every layer, proj/src/sim.cpp:60-64) */
    int32_t dtype;           /* EXF_DTYPE_BF16 (tcgen05 path) or EXF_DTYPE_F32 (fp32 mode:
                                fp32 weights, token states, gate and FFN; SIMT FFN) */
    int32_t attn_heads;      /* H > 0: every layer starts with the coherent attention block
                                (QKV projection, K/V append into every replica, attention over
                                the token's sequence in the local replica, output projection +
                                residual; bf16 only); 0: MoE layers only */
    int32_t context_len;     /* replicated context capacity per sequence (keys) */
    int32_t context_prefix;  /* prompt length written by exf_model_context_setup */
} exf_model_config;
#define EXF_EP_COHERENT 0
#define EXF_EP_VANILLA 1
#define EXF_DTYPE_BF16 0
#define EXF_DTYPE_F32 1

/* assign: [L][E] placement table (exf_contiguous_placement = vanilla,
 * exf_solve_staged = affinity). Allocates weights (generated on device from
 * the seed; identical for a (layer, expert) on whichever rank holds it). */
exf_status exf_model_create(const exf_model_config* config, const int32_t* h_assign,
                            exf_model** out);
exf_status exf_model_destroy(exf_model* model);
/* Peer wiring. Multi-process: exchange 64-byte CUDA-IPC handles (e.g. with
 * torch.distributed) and pass all G of them (own included) in rank order.
 * Single process emulating G ranks on one GPU: exf_model_connect_local. */
exf_status exf_model_ipc_handle(exf_model* model, void* h_handle64);
exf_status exf_model_connect(exf_model* model, const void* h_handles);
exf_status exf_model_connect_local(exf_model* const* models, int32_t count);
/* One decode step (L layers + context AllGather) on `stream`, asynchronous.
 * d_x_in: [B][d] bf16 device pointer. */
exf_status exf_model_step(exf_model* model, const void* d_x_in, exf_stream_t stream);
/* Phased form for lock-step emulation of G ranks in one stream:
 * phase 0 begin(x_in) | 1 gate+dispatch(layer) | 2 ffn(layer) |
 * 5 fused layer (gate..GEMM2 in one launch; needs every rank's kernel to run
 * concurrently, i.e. one process or GPU per rank) |
 * 3 gather send | 4 gather wait |
 * 6 combine send(layer) | 7 combine wait(layer) (ep_mode EXF_EP_VANILLA, after
 * each layer: outputs back to the tokens' home ranks) |
 * 8 attention block(layer) (attn_heads > 0: runs before the layer's MoE). */
exf_status exf_model_step_phase(exf_model* model, int32_t phase, int32_t layer,
                                const void* d_x_in, exf_stream_t stream);
/* Setup AllGather of the replicated context (attention block; once before
 * decoding, proj/src/sim.cpp:162): every rank writes the prompt's K/V
 * (context_prefix positions, synthetic and seeded) of its home sequences
 * into EVERY rank's replica over NVLink, sets the lengths, then flags every
 * peer and waits for all of them on `stream`. All ranks must call it. */
exf_status exf_model_context_setup(exf_model* model, exf_stream_t stream);
/* The same in two halves for G ranks emulated in one stream (lock-step):
 * phase 1 writes + flags the peers, phase 2 waits (0 = both); phase 3 writes
 * every sequence's (deterministic) prompt into this rank's replica only --
 * the same resulting state without NVLink traffic, for long-context benches. */
exf_status exf_model_context_setup_phase(exf_model* model, int32_t phase, exf_stream_t stream);
/* Replicated context rows of this rank's replica (synchronous, diagnostics /
 * tests): K and V of (layer, seq) at positions [pos0, pos0+count), each
 * [count][H][Dh] bf16 bits; lengths [S] int32 of a layer. */
exf_status exf_model_read_kv(exf_model* model, int32_t layer, int32_t seq, int32_t pos0,
                             int32_t count, uint16_t* h_k, uint16_t* h_v);
exf_status exf_model_read_kv_len(exf_model* model, int32_t layer, int32_t* h_len);
/* Attention-block weights of a layer (bf16 bits): Wqkv [3d][d], bqkv [3d],
 * Wo [d][d], bo [d] (replicated on every rank). */
exf_status exf_model_read_attn(exf_model* model, int32_t layer, uint16_t* h_wqkv, uint16_t* h_bqkv,
                               uint16_t* h_wo, uint16_t* h_bo);
/* Device pointer to the [G*B][d] bf16 step output (token-id order). */
exf_status exf_model_output(exf_model* model, void** d_out);
/* Forced routing (routes from a trace, e.g. generate_markov_trace): h_routes
 * is [G*B][L] int32 indexed by token id; NULL disables. */
exf_status exf_model_set_forced_routes(exf_model* model, const int32_t* h_routes);
/* Cumulative statistics since the last reset (synchronous):
 *  routes  [G*B][L] int32: expert of each token at each layer in the LAST
 *          step (entries of tokens not resident here are -1 unless the
 *          rank saw them),
 *  crossed [L] int64: tokens that changed GPU at each layer (this rank's
 *          outgoing moves; sum over ranks = SimReport coherent moves),
 *  counts  [L-1][E][E] int64: fused affinity histogram (sum over ranks =
 *          count_transitions of the emitted trace). */
exf_status exf_model_read_routes(exf_model* model, int32_t* h_routes);
exf_status exf_model_read_crossed(exf_model* model, int64_t* h_crossed);
exf_status exf_affinity_snapshot(exf_model* model, int64_t* h_counts);
exf_status exf_model_reset_stats(exf_model* model);
/* Device error word (0 = ok); non-zero after a peer timeout or capacity fault. */
exf_status exf_model_check(exf_model* model);
/* Weights of (layer, global expert) if it is placed on this rank:
 * w1 [dff][d], b1 [dff], w2 [d][dff], b2 [d], bf16 bits. */
exf_status exf_model_read_expert(exf_model* model, int32_t layer, int32_t expert, uint16_t* h_w1,
                                 uint16_t* h_b1, uint16_t* h_w2, uint16_t* h_b2);
exf_status exf_model_read_gate(exf_model* model, int32_t layer, uint16_t* h_wg /* [E][d] */);
/* Expert migration (online placement change): device
 * pointers of local weight slot `slot` of `layer` (W1 [d_ffn][d], b1, W2
 * [d][d_ffn], b2, bf16; slot k holds the k-th expert of this rank in expert
 * order), so a caller can move weights between ranks (NCCL send/recv or
 * peer copies) into the slots of a new placement, then install the new
 * table with exf_model_set_placement on every rank (validated like
 * Placement::validate, proj/src/placement.cpp:434-470; between steps only;
 * captured graphs stay valid: the tables are updated in place). */
exf_status exf_model_expert_storage(exf_model* model, int32_t layer, int32_t slot, void** d_w1,
                                    void** d_b1, void** d_w2, void** d_b2);
exf_status exf_model_set_placement(exf_model* model, const int32_t* h_assign /* [L][E] */);
/* Resident tokens of buffer `which` (layer j reads buffer j%2 and writes
 * (j+1)%2): h_x [n][d] bf16 bits, h_meta [n][2] int32 {token, prev_expert},
 * *n_out = n. Buffers must hold G*B rows. Synchronous (tests/diagnostics). */
exf_status exf_model_read_resident(exf_model* model, int32_t which, uint16_t* h_x,
                                   int32_t* h_meta, int32_t* n_out);
/* CUDA-graph capture of one full step reading d_x_in; replay launches it. */
exf_status exf_model_capture(exf_model* model, const void* d_x_in, exf_stream_t stream);
exf_status exf_model_replay(exf_model* model, exf_stream_t stream);
/* Kernel launches one step issues (for bench accounting). */
int32_t exf_model_launches_per_step(exf_model* model);
/* JSON description of the launch plan (token tile, split-K, persistent
 * clusters per GEMM) into buf (NUL-terminated, truncated to len). */
exf_status exf_model_describe(exf_model* model, char* buf, int32_t len);
/* Diagnostics: per-CTA globaltimer stamps of the last launches ([6][ctas][16]
 * u64; rows 0/1 = GEMM1/GEMM2 of the two-kernel path or expert-phase stamps
 * of the fused kernel, rows 2/3 = fused token-phase stamps of even/odd layers;
 * requires EXF_FFN_TIMELINE=1 at create time). */
exf_status exf_model_read_ffn_timeline(exf_model* model, uint64_t* h_stamps, int32_t ctas);
/* Diagnostics: the last spin timeout of the fused layer kernel, read from
 * host-mapped memory (valid even after the CUDA context is lost):
 * out12 = {timed out?, site code (101..112, see csrc/layer_fused.cu), block,
 * thread, then 8 progress words of that CTA's roles}. Returns 0 if the
 * channel is not set up (no fused launch yet). */
int32_t exf_debug_last_timeout(int32_t* out12);
/* Diagnostics: per (layer, kernel in {gate_dispatch, GEMM1, GEMM2}) globaltimer
 * [first CTA entry, first wait-return, last wait-return, last CTA exit,
 * phase marks 4..7] ([L][3][8] u64); reset != 0 re-arms the timeline. */
exf_status exf_model_read_step_timeline(exf_model* model, uint64_t* h_stamps, int32_t reset);

/* ------------------------------------------------------------------------
 * Coherent decode attention over the replicated context cache (SURVEY §8(f)
 * rank 1). No reference code: the protocol is PAPER.md:180-184 and the
 * per-step context AllGather it relies on is counted at proj/src/sim.cpp:
 * 161-162. Every GPU holds the whole K/V cache, so a token the dispatch left
 * on this GPU attends over its own sequence's rows here (no combine).
 *   d_q   [N][H][Dh] bf16     d_seq [N] int32 sequence id of each token
 *   d_ctx_len [S] int32 (<= C) d_k, d_v [S][H][C][Dh] bf16 (head-major)
 *   d_out [N][H][Dh] bf16 = softmax(scale * q k^T) v over keys < ctx_len;
 *   an empty context gives 0. Dh in {64, 128}. fp32 scores/softmax/accum.
 * d_workspace: exf_coherent_attention_workspace_bytes(N, H, Dh, C) bytes
 * (0 -> may be NULL); no initialisation needed: the call zeroes the split
 * arrival counters at the front of it on `stream` (one memset node) and
 * the same workspace may be reused across calls of any N, H, C.
 * Deterministic (fixed merge order). One kernel launch per call.
 * ---------------------------------------------------------------------- */
int64_t exf_coherent_attention_workspace_bytes(int64_t N, int32_t H, int32_t Dh, int32_t C);
exf_status exf_coherent_attention(const void* d_q, const int32_t* d_seq, const int32_t* d_ctx_len,
                                  const void* d_k, const void* d_v, int64_t N, int32_t S,
                                  int32_t H, int32_t Dh, int32_t C, float scale,
                                  void* d_workspace, void* d_out, exf_stream_t stream);

/* Per-step K/V append into every replica of the context cache (the data the
 * context AllGather moves, proj/src/sim.cpp:161-162). For each token n (one
 * token per sequence per call): pos = ctx_len[seq[n]] of replica 0; the rows
 * d_k_new/d_v_new [N][H][Dh] bf16 are written at [seq][h][pos][:] of every
 * replica's [S][H][C][Dh] cache, then each replica's ctx_len[seq] = pos + 1.
 * Replicas are device pointers reachable from this GPU (local buffers or
 * CUDA-IPC-mapped NVLink peers), up to 8; h_* arrays hold `replicas` entries,
 * replica 0 is the local one. Tokens whose sequence is full (pos == C) are
 * skipped and counted in *d_overflow (nullable). Cross-GPU readers must
 * synchronise (stream sync + barrier) before attending. */
exf_status exf_kv_append(const void* d_k_new, const void* d_v_new, const int32_t* d_seq,
                         int64_t N, int32_t S, int32_t H, int32_t Dh, int32_t C,
                         int32_t replicas, void* const* h_k_caches, void* const* h_v_caches,
                         int32_t* const* h_ctx_lens, int32_t* d_overflow, exf_stream_t stream);

/* Replica wiring for exf_kv_append across processes: export a device buffer
 * as a 64-byte CUDA-IPC handle + byte offset inside its allocation, import it
 * on the caller's current device (peer access enabled lazily), close it. */
exf_status exf_ipc_export(const void* d_ptr, void* h_handle64, int64_t* h_offset);
exf_status exf_ipc_import(const void* h_handle64, int64_t offset, void** d_ptr);
exf_status exf_ipc_close(void* d_ptr, int64_t offset);

#ifdef __cplusplus
}
#endif
#endif /* EXFLOW_C_H */
