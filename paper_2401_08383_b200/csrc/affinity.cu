// affinity.cu -- kernel (5): inter-layer expert-affinity histogram, bulk
// rebuild from a routing trace.
//
// Replaces exflow::count_transitions (proj/src/trace.cpp:191-215; hot loop
// :205-209 does counts[j](p(t,j), p(t,j+gap)) += 1 with scattered int64 RMW).
//
// Design (HBM-bound integer scatter; v2 after the round-1
// ncu capture: 212 us for 201 MB of ids = 0.15 of HBM, of which 70 us was a
// serial split reduction):
//  * persistent CTAs, each owning a contiguous token range (<= 65535 tokens)
//    and privatising the (pairs x E x E) histogram in shared memory as packed
//    u16 counters (two bins per 32-bit word; a per-CTA count never exceeds
//    65535, so a 32-bit atomicAdd of 1<<16 never carries). Each pair's block
//    of words has an odd stride, so lanes counting the same (a, b) transition
//    of different layer pairs hit different banks;
//  * the trace streams through a software pipeline: the next tile's rows
//    (a contiguous chunk of the row-major [T][L] trace) are loaded into
//    registers with 16-byte non-allocating loads while the current tile is
//    counted from shared memory;
//  * work items are (token, pair) with the pair fixed per thread (no integer
//    division in the loop);
//  * the merge is a flush of the CTA's non-zero bins with 64-bit global
//    atomics into zeroed counts: integer sums are exact in any order, so the
//    result is bit-identical to the reference loop and
//    there is no second pass over split partials.
// Algorithmic bytes per launch: 4*T*L (ids) + 8*(L-gap)*E*E (+8*(L-gap)*E).
#include "common.cuh"

#include <algorithm>
#include <vector>

namespace exf {
namespace {

constexpr int kHistThreads = 512;
constexpr int kTileTokens = 256;
constexpr int kMaxTokensPerCta = 65535;
constexpr int64_t kCounterSmemBudget = 190 * 1024;
constexpr int kPrefetchVec = 4;  // int4 per thread per tile in registers (tile <= 512*4*4 ints)

int g_num_sms = 0;

int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

struct HistPlan {
    int32_t pairs;
    int32_t pair_group;   // pairs per CTA pass (all pairs when they fit)
    int32_t groups;
    int64_t splits;       // token ranges
    int32_t pair_words;   // odd stride of one pair's packed counters (u32 words)
    int32_t tile_tokens;  // tokens per pipeline tile
    size_t smem_bytes;
    int64_t workspace_bytes;
};

HistPlan plan_hist(int64_t T, int32_t L, int32_t E, int32_t gap) {
    HistPlan p{};
    p.pairs = L - gap;
    const int64_t bins_per_pair = (int64_t)E * E;
    p.pair_words = (int32_t)(((bins_per_pair + 1) / 2) | 1);
    // the tile must fit the register prefetch (kPrefetchVec int4 per thread)
    p.tile_tokens = (int32_t)std::min<int64_t>(kTileTokens, (int64_t)kHistThreads * kPrefetchVec * 4 / L);
    p.tile_tokens = std::max(1, p.tile_tokens & ~3);
    const int64_t tile_bytes = (int64_t)p.tile_tokens * L * 4;
    // pair groups sized for two CTAs per SM (the counting is latency-bound on
    // shared-memory atomics; one 188 KB CTA per SM at E = 64 left 3/4 of the
    // warp slots empty), balanced across groups; every group re-reads its
    // token range (L2 hits: the groups of a range run side by side)
    const int64_t per_cta = 110 * 1024 - tile_bytes - 64;
    const int64_t all_bytes = (int64_t)p.pairs * p.pair_words * 4;
    int64_t groups = std::max<int64_t>(1, (all_bytes + per_cta - 1) / per_cta);
    groups = std::min<int64_t>(groups, p.pairs);
    p.pair_group = (int32_t)((p.pairs + groups - 1) / groups);
    if ((int64_t)p.pair_group * p.pair_words * 4 + tile_bytes > kCounterSmemBudget + 32 * 1024)
        p.pair_group = (int32_t)std::max<int64_t>(1, (kCounterSmemBudget + 32 * 1024 - tile_bytes) / ((int64_t)p.pair_words * 4));
    p.groups = (p.pairs + p.pair_group - 1) / p.pair_group;
    // token ranges: about two CTAs per SM over all groups, <= 65535 tokens each
    const int64_t min_splits = (T + kMaxTokensPerCta - 1) / kMaxTokensPerCta;
    const int64_t target = std::max<int64_t>(1, 2 * (int64_t)num_sms() / p.groups);
    int64_t splits = std::max(target, min_splits);
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, (T + 63) / 64));
    p.splits = std::max<int64_t>(std::max(splits, min_splits), 1);
    p.smem_bytes = (size_t)p.pair_group * p.pair_words * 4 + (size_t)tile_bytes + 16;
    // few bins x CTAs: exact 64-bit atomic flush, no workspace; many (E >= 32):
    // u16 partials in a workspace summed by hist_sum_kernel
    const int64_t total_bins = (int64_t)p.pairs * E * E;
    p.workspace_bytes = total_bins * p.splits > (4LL << 20) ? total_bins * p.splits * 2 : 0;
    return p;
}

// One CTA: one token range x one pair group.
__global__ void __launch_bounds__(kHistThreads)
hist_kernel(const int32_t* __restrict__ paths, int64_t T, int32_t L, int32_t E, int32_t gap,
            int32_t pairs, int32_t pair_group, int32_t pair_words, int32_t tile_tokens, int64_t splits,
            unsigned long long* __restrict__ counts, unsigned long long* __restrict__ row_totals,
            uint16_t* __restrict__ partials) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
    const int32_t group = blockIdx.x;
    const int32_t j0 = group * pair_group;
    const int32_t pg = min(pair_group, pairs - j0);
    int32_t* tile = reinterpret_cast<int32_t*>(smem + (((int64_t)pair_group * pair_words * 4 + 15) & ~15ll));
    const int64_t split = blockIdx.y;
    const int64_t t_begin = T * split / splits;
    const int64_t t_end = T * (split + 1) / splits;
    const int32_t EE = E * E;
    const int32_t tid = threadIdx.x;

    for (int32_t w = tid; w < pg * pair_words; w += kHistThreads) cnt[w] = 0u;
    // pair handled by this thread, token stride
    const int32_t lanes = (kHistThreads / pg) * pg;  // threads in use
    const int32_t jj = tid % pg, tstep = kHistThreads / pg, tfirst = tid / pg;
    const bool counting = tid < lanes;
    uint32_t* my_cnt = cnt + jj * pair_words;
    const int32_t ja = j0 + jj, jb = ja + gap;

    const bool aligned = ((reinterpret_cast<uintptr_t>(paths) | (uintptr_t)(L * 4)) & 15) == 0;
    int4 pre[kPrefetchVec];
    auto fetch = [&](int64_t t0) {  // tile starting at token t0 into registers
        const int32_t nt = (int32_t)imin64(tile_tokens, t_end - t0);
        if (aligned) {
            const int32_t nvec = nt * L / 4;
            const int4* s4 = reinterpret_cast<const int4*>(paths + t0 * L);
#pragma unroll
            for (int u = 0; u < kPrefetchVec; ++u) {
                const int32_t i = tid + u * kHistThreads;
                if (i < nvec) pre[u] = ld_nc_v4(s4 + i);
            }
        }
    };
    auto stage = [&](int64_t t0) {  // registers (or global, unaligned) -> shared tile
        const int32_t nt = (int32_t)imin64(tile_tokens, t_end - t0);
        if (aligned) {
            const int32_t nvec = nt * L / 4;
            int4* d4 = reinterpret_cast<int4*>(tile);
#pragma unroll
            for (int u = 0; u < kPrefetchVec; ++u) {
                const int32_t i = tid + u * kHistThreads;
                if (i < nvec) d4[i] = pre[u];
            }
        } else {
            for (int32_t i = tid; i < nt * L; i += kHistThreads) tile[i] = __ldg(paths + t0 * L + i);
        }
    };
    if (t_begin < t_end) fetch(t_begin);
    for (int64_t t0 = t_begin; t0 < t_end; t0 += tile_tokens) {
        const int32_t nt = (int32_t)imin64(tile_tokens, t_end - t0);
        __syncthreads();  // previous tile fully counted (and the zeroing done)
        stage(t0);
        if (t0 + tile_tokens < t_end) fetch(t0 + tile_tokens);  // in flight while counting
        __syncthreads();
        if (counting) {
            for (int32_t t = tfirst; t < nt; t += tstep) {
                const int32_t a = tile[t * L + ja];
                const int32_t b = tile[t * L + jb];
                if ((unsigned)a < (unsigned)E && (unsigned)b < (unsigned)E) {
                    const int32_t bin = a * E + b;
                    atomicAdd(&my_cnt[bin >> 1], 1u << ((bin & 1) * 16));
                }
            }
        }
    }
    __syncthreads();
    const uint16_t* c16 = reinterpret_cast<const uint16_t*>(cnt);
    if (partials) {
        // many bins x many CTAs (E >= 32): the CTA's u16 partials go to a
        // workspace [split][pair][E][E] with coalesced stores; hist_sum_kernel
        // adds them up (one 64-bit atomic per bin and CTA would be ~10^7
        // global atomics at E = 64)
        uint16_t* dst = partials + split * (int64_t)pairs * EE + (int64_t)j0 * EE;
        for (int32_t i = tid; i < pg * EE; i += kHistThreads) {
            const int32_t q = i / EE, bin = i - q * EE;
            dst[i] = c16[(int64_t)q * pair_words * 2 + bin];
        }
        return;
    }
    // flush: non-zero bins into the exact 64-bit result; row totals per (pair, a)
    for (int32_t i = tid; i < pg * EE; i += kHistThreads) {
        const int32_t q = i / EE, bin = i - q * EE;
        const uint32_t c = c16[(int64_t)q * pair_words * 2 + bin];
        if (c) atomicAdd(&counts[(int64_t)(j0 + q) * EE + bin], (unsigned long long)c);
    }
    if (row_totals)
        for (int32_t r = tid; r < pg * E; r += kHistThreads) {
            const int32_t q = r / E, a = r - q * E;
            const uint16_t* row = c16 + (int64_t)q * pair_words * 2 + (int64_t)a * E;
            uint32_t sum = 0;
            for (int32_t b = 0; b < E; ++b) sum += row[b];
            if (sum) atomicAdd(&row_totals[(int64_t)(j0 + q) * E + a], (unsigned long long)sum);
        }
}

// Sum of the per-CTA u16 partials, bin by bin: a block covers 64 consecutive
// bins x 8 split groups (coalesced loads), integer sums (order-free, exact).
__global__ void __launch_bounds__(512) hist_sum_kernel(const uint16_t* __restrict__ partials, int64_t splits,
                                                       int64_t total_bins, unsigned long long* __restrict__ counts) {
    __shared__ unsigned long long s_acc[8][64];
    const int lane_bin = threadIdx.x & 63, grp = threadIdx.x >> 6;
    const int64_t bin = (int64_t)blockIdx.x * 64 + lane_bin;
    unsigned long long acc = 0;
    if (bin < total_bins) {
#pragma unroll 8
        for (int64_t sp = grp; sp < splits; sp += 8) acc += partials[sp * total_bins + bin];
    }
    s_acc[grp][lane_bin] = acc;
    __syncthreads();
    if (grp == 0 && bin < total_bins) {
        unsigned long long t = 0;
#pragma unroll
        for (int g = 0; g < 8; ++g) t += s_acc[g][lane_bin];
        counts[bin] = t;
    }
}

// Row totals from the final counts (proj/src/trace.cpp:210-213): one warp per row.
__global__ void hist_rows_kernel(const unsigned long long* __restrict__ counts, int64_t rows, int32_t E,
                                 unsigned long long* __restrict__ row_totals) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= rows) return;
    unsigned long long s = 0;
    for (int32_t b = threadIdx.x & 31; b < E; b += 32) s += counts[row * E + b];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) row_totals[row] = s;
}

exf_status check_hist_args(int64_t T, int32_t L, int32_t E, int32_t gap) {
    // RoutingTrace::validate (proj/src/trace.cpp:53-70) and the gap check (:193-196)
    if (E < 1) return invalid("num_experts must be >= 1, got " + std::to_string(E));
    if (L < 2) return invalid("num_layers must be >= 2, got " + std::to_string(L));
    if (T < 1) return invalid("trace contains no token paths");
    if (gap < 1 || gap > L - 1)
        return invalid("gap " + std::to_string(gap) + " out of range [1," + std::to_string(L - 1) +
                       "]");
    if ((((int64_t)E * E + 1) / 2 | 1) * 4 > kCounterSmemBudget)
        return invalid("num_experts " + std::to_string(E) + " exceeds the histogram kernel limit");
    if ((int64_t)L * 4 > (int64_t)kHistThreads * kPrefetchVec * 16) return invalid("num_layers too large");
    return EXF_OK;
}

}  // namespace
}  // namespace exf

using namespace exf;

extern "C" int64_t exf_count_transitions_workspace_bytes(int64_t T, int32_t L, int32_t E,
                                                         int32_t gap) {
    if (check_hist_args(T, L, E, gap) != EXF_OK) return -1;
    return plan_hist(T, L, E, gap).workspace_bytes;
}

extern "C" exf_status exf_count_transitions(const int32_t* d_paths, int64_t T, int32_t L,
                                            int32_t E, int32_t gap, int64_t* d_counts,
                                            int64_t* d_row_totals, void* d_workspace,
                                            exf_stream_t stream) {
    exf::NvtxRange nvtx_range("exf.count_transitions");
    EXF_TRY(check_hist_args(T, L, E, gap));
    if (!d_paths || !d_counts) return invalid("null device pointer");
    // (d_workspace: NULL allowed when exf_count_transitions_workspace_bytes == 0)
    const HistPlan p = plan_hist(T, L, E, gap);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    static size_t attr_bytes = 0;
    if (p.smem_bytes > attr_bytes) {
        EXF_CUDA_TRY(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)std::max<size_t>(p.smem_bytes, 48 * 1024)));
        attr_bytes = std::max<size_t>(p.smem_bytes, 48 * 1024);
    }
    const int64_t pairs_bins = (int64_t)p.pairs * E * E;
    auto* counts = reinterpret_cast<unsigned long long*>(d_counts);
    auto* totals = reinterpret_cast<unsigned long long*>(d_row_totals);
    dim3 grid(p.groups, (unsigned)p.splits);
    if (p.workspace_bytes > 0) {
        if (!d_workspace) return invalid("workspace required (exf_count_transitions_workspace_bytes)");
        auto* ws = static_cast<uint16_t*>(d_workspace);
        hist_kernel<<<grid, kHistThreads, p.smem_bytes, s>>>(d_paths, T, L, E, gap, p.pairs, p.pair_group,
                                                             p.pair_words, p.tile_tokens, p.splits, counts,
                                                             totals, ws);
        EXF_LAUNCH_CHECK("hist_kernel");
        hist_sum_kernel<<<(unsigned)((pairs_bins + 63) / 64), 512, 0, s>>>(ws, p.splits, pairs_bins, counts);
        EXF_LAUNCH_CHECK("hist_sum_kernel");
        if (d_row_totals) {
            const int64_t rows = (int64_t)p.pairs * E;
            hist_rows_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(counts, rows, E, totals);
            EXF_LAUNCH_CHECK("hist_rows_kernel");
        }
        return EXF_OK;
    }
    EXF_CUDA_TRY(cudaMemsetAsync(d_counts, 0, (size_t)pairs_bins * 8, s));
    if (d_row_totals) EXF_CUDA_TRY(cudaMemsetAsync(d_row_totals, 0, (size_t)p.pairs * E * 8, s));
    hist_kernel<<<grid, kHistThreads, p.smem_bytes, s>>>(d_paths, T, L, E, gap, p.pairs, p.pair_group,
                                                         p.pair_words, p.tile_tokens, p.splits, counts, totals,
                                                         nullptr);
    EXF_LAUNCH_CHECK("hist_kernel");
    return EXF_OK;
}

extern "C" exf_status exf_count_transitions_host(const int32_t* h_paths, int64_t T, int32_t L,
                                                 int32_t E, int32_t gap, int64_t* h_counts,
                                                 int64_t* h_row_totals) {
    exf::NvtxRange nvtx_range("exf.count_transitions_host");
    EXF_TRY(check_hist_args(T, L, E, gap));
    for (int64_t i = 0; i < T * (int64_t)L; ++i)
        if (h_paths[i] < 0 || h_paths[i] >= E)
            return invalid("expert id out of range [0," + std::to_string(E) + ")");
    const HistPlan p = plan_hist(T, L, E, gap);
    const size_t paths_b = (size_t)T * L * 4;
    const size_t counts_b = (size_t)p.pairs * E * E * 8;
    const size_t tot_b = (size_t)p.pairs * E * 8;
    const size_t total = paths_b + counts_b + tot_b + (size_t)p.workspace_bytes + 64;
    HostScratch* hs = nullptr;  // cached per thread and device: no per-call cudaMalloc
    EXF_TRY(host_scratch(total, std::max(paths_b, counts_b), &hs));
    uint8_t* buf = hs->dev;
    int32_t* d_paths = reinterpret_cast<int32_t*>(buf);
    int64_t* d_counts = reinterpret_cast<int64_t*>(buf + ((paths_b + 15) & ~size_t(15)));
    int64_t* d_tot = d_counts + (size_t)p.pairs * E * E;
    void* d_ws = d_tot + (size_t)p.pairs * E;
    EXF_TRY(hs->h2d(d_paths, h_paths, paths_b));
    EXF_TRY(exf_count_transitions(d_paths, T, L, E, gap, d_counts, d_tot, d_ws, hs->stream));
    EXF_TRY(hs->d2h(h_counts, d_counts, counts_b));
    if (h_row_totals) EXF_TRY(hs->d2h(h_row_totals, d_tot, tot_b));
    return EXF_OK;
}
