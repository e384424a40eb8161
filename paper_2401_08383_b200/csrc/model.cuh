// model.cuh -- device data layout of one rank of the ExFlow MoE decode step.
//
// HBM layout per rank (G ranks, B home tokens per rank, C = G*B capacity):
//  symmetric region (one cudaMalloc, IPC-shared, identical offsets on every rank)
//    recv_x    [2 parity][G src][C][d]   bf16  tokens dispatched to this rank
//    recv_meta [2][G][C]                 RecvMeta {token, expert, prob}
//    recv_cnt  [2][G][E_loc]             int32 per-(src, local expert) counts
//    flags     [2][G]                    u64   dispatch epoch per src
//    gather_x  [C][d]                    bf16  context AllGather output (by token id)
//    gflags    [G]                       u64   AllGather epoch per src
//  private
//    res_x[2][C][d], res_meta[2][C], n_res[2]  resident tokens (ping-pong)
//    expert[C], prob[C]                         gate outputs
//    H[C][dff]                                  FFN hidden (canonical order)
//    weights: Wg[L][E][d]; W1[L][E_loc][dff][d]; b1[L][E_loc][dff];
//             W2[L][E_loc][d][dff]; b2[L][E_loc][d]       (all bf16)
//    gpu_of/slot_of [L][E], hist[L-1][E][E] i64, crossed[L] i64,
//    trace[C][L] i32 (token-id indexed), step counter, error word
#pragma once

#include <cuda_bf16.h>

#include <cstdint>

namespace exf {

struct RecvMeta {
    int32_t token;   // global token id (home rank = token % G)
    int32_t expert;  // global expert id chosen at this layer
    float prob;      // softmax probability of that expert (output scale)
    int32_t pad;
};

struct ResMeta {
    int32_t token;
    int32_t prev_expert;  // expert of the previous layer (-1 before layer 0)
};

struct Symm {  // byte offsets inside the symmetric region
    int64_t recv_x, recv_meta, recv_cnt, flags, gather_x, gflags, cflags;
    int64_t comb_x, comb_meta, comb_flags;  // vanilla-EP combine: [2 layer parity][B] home slots
    // replicated context (attention block): K, V [L][S][H][Cctx][Dh] bf16,
    // lengths [L][S] int32, setup-AllGather flags [G] u64 (0 when disabled)
    int64_t kv_k, kv_v, kv_len, sflags;
    int64_t total;
};
// fused layer kernel: per-(parity, src rank, src CTA) dispatch-complete flags
constexpr int kMaxCtas = 256;

// Everything a kernel needs, passed by value.
struct LayerArgs {
    int32_t G, rank, E, E_loc, d, dff, C, L, layer, forced;
    int32_t esz;                    // bytes per element of rows and gate: 2 (bf16) or 4 (fp32 mode)
    // rank-local
    const void* wg;                 // [E][d] of this layer
    const int32_t* gpu_of;          // [E] of this layer
    const int32_t* slot_of;         // [E] of this layer
    const void* res_x_in;           // [C][d]
    const ResMeta* res_meta_in;     // [C]
    const int32_t* n_res_in;        // device scalar
    int32_t* expert;                // [C]
    float* prob;                    // [C]
    unsigned long long* hist;       // [L-1][E][E] (nullptr -> no fused histogram)
    unsigned long long* crossed;    // [L]
    int32_t* trace;                 // [C][L] token-id indexed (nullptr -> off)
    const int32_t* forced_routes;   // [C][L] token-id indexed forced experts
    const uint64_t* step;           // device step counter
    int32_t* err;
    int32_t* done_ctr;              // last-CTA-done counter for dispatch
    int32_t* cta_cnt;               // [grid][E] per-CTA key counts (gate_dispatch)
    uint32_t* gbar;                 // [2] grid barrier {count, generation}
    int32_t tpc;                    // tokens per CTA of gate_dispatch
    // peers' symmetric regions (index = rank), and this layer's parity
    uint8_t* const* peers;          // device array [G]
    Symm sym;
    int32_t parity;
    unsigned long long* tl;         // optional step timeline [4] (diagnostics)
};

// Step timeline (diagnostics, EXF_FFN_TIMELINE=1): per (layer, kernel)
// [0] min CTA entry, [1] min wait-return, [2] max wait-return, [3] max exit.
__device__ __forceinline__ void tl_mark(unsigned long long* tl, int which) {
    if (!tl) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (which == 0 || which == 1) atomicMin(tl + which, t);
    if (which == 1) atomicMax(tl + 2, t);
    if (which >= 3) atomicMax(tl + which, t);  // 3 = exit, 4..7 = phase marks
}

// Arguments of one grouped-FFN GEMM launch (ffn_tcgen05.cu).
struct FfnArgs {
    int32_t G, rank, E_loc, C, d, dff, K, M_total, ksplit, L, layer, mode;
    uint8_t* own_sym;
    Symm sym;
    const uint64_t* step;
    __nv_bfloat16* H;            // [C][dff]
    const __nv_bfloat16* bias;   // [E_loc][M_total] of this layer
    __nv_bfloat16* res_x_out;    // [C][d]  (GEMM2)
    ResMeta* res_meta_out;       // [C]     (GEMM2)
    int32_t* n_res_out;          //         (GEMM2)
    int32_t* err;
    uint64_t* tstamp;            // optional per-CTA globaltimer stamps [grid][16] (diagnostics)
    unsigned long long* tl;      // optional step timeline [4] (diagnostics)
};

// Arguments of one dense decode GEMM of the attention block (attn_block.cu).
struct DenseArgs {
    int32_t M, K, d, ksplit;
    const int32_t* n_dev;          // resident tokens (device scalar)
    const __nv_bfloat16* bias;     // [M]
    __nv_bfloat16* out[3];         // MODE 0: q, k, v [C][d]; MODE 1: out[0] = x [C][d] (in place)
    int32_t* err;
    // K/V append folded into the projection (replicas > 0): MODE 0 stores each
    // resident token's k and v rows at position lens[0][seq] of every replica
    // (instead of out[1] / out[2]); MODE 1 then advances every replica's length
    // of each resident token's sequence (after the attention has read it)
    int32_t replicas, kv_H, kv_Dh, kv_C;
    const int32_t* seq;            // resident row -> sequence (ResMeta.token, stride 2)
    __nv_bfloat16* kc[8];
    __nv_bfloat16* vc[8];
    int32_t* lens[8];              // per replica [S] lengths of this layer; [0] = local
    int32_t* overflow;
};

// Arguments of the setup AllGather of the replicated context (attn_block.cu).
struct ContextSetupArgs {
    int32_t G, rank, L, S, H, Dh, Cctx, prefix;
    int32_t local;  // 1: every sequence into this rank's replica only (no exchange)
    uint64_t seed;
    uint8_t* const* peers;  // device array [G] of symmetric-region bases
    int64_t kv_k, kv_v, kv_len;
};

// Arguments of one fp32-mode FFN GEMM launch (ffn_f32.cu).
struct FfnF32Args {
    int32_t G, rank, E_loc, C, d, dff, L, layer;
    uint8_t* own_sym;
    Symm sym;
    const uint64_t* step;
    const float* w;        // [E_loc][M][K] of this layer (W1: M = dff, K = d; W2: M = d, K = dff)
    const float* bias;     // [E_loc][M] of this layer
    float* H;              // [C][dff] canonical token order
    float* res_x_out;      // [C][d]  (GEMM2)
    ResMeta* res_meta_out; //         (GEMM2)
    int32_t* n_res_out;    //         (GEMM2)
    int32_t* err;
};

// One piece of the fused kernel's static stream-K schedule: a contiguous run
// of 64-wide k-blocks of one (gemm, local expert, 128-row tile). Every CTA
// owns an equal share of GEMM1's and of GEMM2's k-blocks, cut at tile edges;
// a tile's contributors (S, in k order kidx) park fp32 partials and the last
// to arrive sums them in k order.
struct Piece {
    int16_t g, e, mt, kb0;
    int16_t nkb, kidx, S, pad;
};
constexpr int kMaxPieces = 64;  // per CTA (static smem: 1 KB)

// Arguments of the fused per-layer kernel (layer_fused.cu).
struct FusedArgs {
    // token side
    int32_t G, rank, E, E_loc, d, dff, C, L, layer, forced, tpc;
    const __nv_bfloat16* wg;
    const int32_t* gpu_of;
    const int32_t* slot_of;
    const __nv_bfloat16* res_x_in;
    const ResMeta* res_meta_in;
    const int32_t* n_res_in;
    unsigned long long* hist;
    unsigned long long* crossed;
    int32_t* trace;
    const int32_t* forced_routes;
    const uint64_t* step;
    int32_t* err;
    int32_t* done_ctr;
    int32_t* cta_cnt;
    uint32_t* gbar;
    uint8_t* const* peers;
    uint8_t* own_sym;
    Symm sym;
    // expert side
    __nv_bfloat16* H;
    const __nv_bfloat16* b1;  // [E_loc][dff] of this layer
    const __nv_bfloat16* b2;  // [E_loc][d] of this layer
    __nv_bfloat16* res_x_out;
    ResMeta* res_meta_out;
    int32_t* n_res_out;
    float* ws;           // split-K partials
    int32_t* item_ctr;   // arrivals per (gemm, expert, tile, chunk)
    int32_t* hdone;      // [2 parity][E_loc] completed GEMM1 (tile, chunk) units
    const Piece* pieces;       // stream-K schedule, CTA c owns [piece_off[c], piece_off[c+1])
    const int32_t* piece_off;  // [grid + 1]
    int32_t max_contrib, max_chunks;
    // dense single-GPU mode (G == 1, one token per CTA): GEMM1's MMAs run over
    // every resident token from the PDL wait on, while each token's CTA gates
    // it and publishes {epoch, slot, prob} in one 64-bit route flag; GEMM1's
    // epilogue keeps routed rows only, GEMM2 runs on the compact H
    int32_t dense;
    int32_t xpre;  // dense: pieces whose weights are L2-prefetched before the PDL wait
    int32_t hbox;  // dense: GEMM2 H tiles in 16/32-row boxes when the expert has few tokens
    // dispatch path, few tokens per local expert: the schedule's expert ids are
    // virtual slots, bound to the local experts in descending token count once
    // the counts are in (no weight prefetch before the PDL wait)
    int32_t remap;
    int32_t chain;      // previous kernel in the stream = this model's previous layer (see fin_gen)
    uint64_t* fin_gen;  // [ctas] exit generation (global layer index + 1) per CTA
    int32_t ctas;  // grid size (the schedule's CTA count; <= #SMs, all co-resident)
    unsigned long long* tl;
    uint64_t* tstamp;    // optional per-CTA stamps [grid][16] (diagnostics)
};

__host__ __device__ inline int64_t bytes_bf16(int64_t n) { return n * 2; }

// GELU(v) = v/2 (1 + erf(v/sqrt2)) with erf from Abramowitz-Stegun 7.1.26
// (|error| <= 1.5e-7, far below the bf16 rounding of H; the oracle uses exact
// erf, oracle/exflow_model_oracle.c): one reciprocal, one exp2, five FMAs.
// libdevice erff's branchy polynomial cost ~190 cycles per value on the one
// epilogue warp of each SM sub-partition (~3000 cycles per 16-token group),
// which made the expert epilogues the critical path.
__device__ __forceinline__ float gelu_erf(float v) {
    const float z = fabsf(v) * 0.70710678118654752440f;
    // single MUFU ops (flush-to-zero approximations; the 7.1.26 polynomial's
    // own error, 1.5e-7, dominates): __fdividef / exp2f carried denormal
    // fix-up code into the epilogue loops
    float t, e;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.0f)));
    float p = fmaf(1.061405429f, t, -1.453152027f);
    p = fmaf(p, t, 1.421413741f);
    p = fmaf(p, t, -0.284496736f);
    p = fmaf(p, t, 0.254829592f);
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-z * z * 1.44269504088896341f));
    const float erf_abs = fmaf(-p * t, e, 1.0f);
    return 0.5f * v * (1.0f + copysignf(erf_abs, v));
}

// error codes written to the device error word before a trap
enum : int {
    ERR_NONE = 0,
    ERR_TIMEOUT_DISPATCH = 1,
    ERR_TIMEOUT_GATHER = 2,
    ERR_TIMEOUT_PIPE = 3,
    ERR_CAPACITY = 4,
    ERR_BAD_EXPERT = 5,
};

}  // namespace exf
