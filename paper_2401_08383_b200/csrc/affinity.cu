// affinity.cu -- kernel (5): inter-layer expert-affinity histogram, bulk
// rebuild from a routing trace.
//
// Replaces exflow::count_transitions (proj/src/trace.cpp:191-215; hot loop
// :205-209 does counts[j](p(t,j), p(t,j+gap)) += 1 with scattered int64 RMW).
//
// Design (HBM-bound integer scatter):
//  * grid = splits x 1: each CTA owns a contiguous token range (<= 65535
//    tokens) and privatises the WHOLE (pairs x E x E) histogram in shared
//    memory as packed u16 counters (two bins per 32-bit word; a per-CTA count
//    never exceeds 65535, so a 32-bit atomicAdd of 1<<16 never carries).
//  * token rows are staged through shared memory with coalesced 16-byte loads
//    (a token range of the row-major [T][L] trace is one contiguous chunk);
//    work items are flattened (token, pair) so consecutive lanes touch
//    consecutive columns (conflict-free reads) and different pair matrices
//    (low atomic contention).
//  * global merge is atomic-free and deterministic: each CTA streams its u16
//    partials to a workspace; a second kernel sums the splits per bin into the
//    int64 result and forms row totals (trace.cpp:210-213).
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
    int32_t pair_group;  // pairs per CTA pass (all pairs when they fit)
    int32_t groups;
    int64_t splits;
    int64_t counter_words;  // u32 words of packed u16 counters per CTA
    size_t smem_bytes;
    int64_t workspace_bytes;
};

HistPlan plan_hist(int64_t T, int32_t L, int32_t E, int32_t gap) {
    HistPlan p{};
    p.pairs = L - gap;
    const int64_t bins_per_pair = (int64_t)E * E;
    p.pair_group = (int32_t)std::max<int64_t>(
        1, std::min<int64_t>(p.pairs, kCounterSmemBudget / (bins_per_pair * 2)));
    p.groups = (p.pairs + p.pair_group - 1) / p.pair_group;
    const int64_t group_bins = bins_per_pair * p.pair_group;
    p.counter_words = (group_bins + 1) / 2;
    // splits: enough CTAs to fill the machine, few enough that the flush of
    // private histograms (splits * bins * 2 B) stays well below the id bytes.
    const int64_t total_bins = bins_per_pair * p.pairs;
    const int64_t min_splits = (T + kMaxTokensPerCta - 1) / kMaxTokensPerCta;
    const int64_t by_traffic = std::max<int64_t>(1, (4 * T * L) / (total_bins * 2 * 4));
    const int64_t target = std::max<int64_t>(1, 2 * (int64_t)num_sms() / p.groups);
    int64_t splits = std::min(target, by_traffic);
    splits = std::max(splits, min_splits);
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, (T + 31) / 32));
    p.splits = std::max<int64_t>(splits, 1);
    p.smem_bytes = (size_t)p.counter_words * 4 + (size_t)kTileTokens * L * 4 + 16;
    p.workspace_bytes = p.splits * total_bins * 2;
    return p;
}

// Each CTA: one token range x one pair group. Writes packed u16 partials to
// ws[split][pair][E][E] (u16 view).
__global__ void __launch_bounds__(kHistThreads)
hist_partial_kernel(const int32_t* __restrict__ paths, int64_t T, int32_t L, int32_t E,
                    int32_t gap, int32_t pairs, int32_t pair_group, int64_t splits,
                    int64_t counter_words, uint16_t* __restrict__ ws) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
    int32_t* tile = reinterpret_cast<int32_t*>(smem + ((counter_words * 4 + 15) & ~15ll));

    const int32_t group = blockIdx.x;
    const int64_t split = blockIdx.y;
    const int32_t j0 = group * pair_group;
    const int32_t pg = min(pair_group, pairs - j0);
    const int64_t t_begin = T * split / splits;
    const int64_t t_end = T * (split + 1) / splits;
    const int32_t EE = E * E;

    for (int64_t w = threadIdx.x; w < counter_words; w += blockDim.x) cnt[w] = 0u;

    for (int64_t t0 = t_begin; t0 < t_end; t0 += kTileTokens) {
        const int32_t nt = (int32_t)imin64(kTileTokens, t_end - t0);
        const int32_t nints = nt * L;
        const int32_t* src = paths + t0 * L;
        __syncthreads();  // previous tile fully consumed
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            const int32_t nvec = nints >> 2;
            const int4* s4 = reinterpret_cast<const int4*>(src);
            int4* d4 = reinterpret_cast<int4*>(tile);
            for (int32_t i = threadIdx.x; i < nvec; i += blockDim.x) d4[i] = ld_nc_v4(s4 + i);
            for (int32_t i = (nvec << 2) + threadIdx.x; i < nints; i += blockDim.x) tile[i] = src[i];
        } else {
            for (int32_t i = threadIdx.x; i < nints; i += blockDim.x) tile[i] = __ldg(src + i);
        }
        __syncthreads();
        const int32_t items = nt * pg;
        for (int32_t w = threadIdx.x; w < items; w += blockDim.x) {
            const int32_t t = w / pg;
            const int32_t jj = w - t * pg;
            const int32_t j = j0 + jj;
            const int32_t a = tile[t * L + j];
            const int32_t b = tile[t * L + j + gap];
            if ((unsigned)a < (unsigned)E && (unsigned)b < (unsigned)E) {
                const int32_t bin = jj * EE + a * E + b;
                atomicAdd(&cnt[bin >> 1], 1u << ((bin & 1) * 16));
            }
        }
    }
    __syncthreads();
    // stream the packed partial histogram of this group to the workspace
    const int64_t total_bins = (int64_t)pairs * EE;
    uint16_t* dst = ws + split * total_bins + (int64_t)j0 * EE;
    const uint16_t* c16 = reinterpret_cast<const uint16_t*>(cnt);
    const int64_t nb = (int64_t)pg * EE;
    for (int64_t i = threadIdx.x; i < nb; i += blockDim.x) dst[i] = c16[i];
}

// One CTA per (pair j, source expert a): sums the splits of each bin (fixed
// order, exact) and forms the row total.
__global__ void hist_reduce_kernel(const uint16_t* __restrict__ ws, int64_t splits,
                                   int32_t pairs, int32_t E, int64_t* __restrict__ counts,
                                   int64_t* __restrict__ row_totals) {
    const int32_t row = blockIdx.x;  // j*E + a
    const int64_t total_bins = (int64_t)pairs * E * E;
    __shared__ int64_t warp_tot[32];
    int64_t mine = 0;
    for (int32_t b = threadIdx.x; b < E; b += blockDim.x) {
        const int64_t bin = (int64_t)row * E + b;
        int64_t s = 0;
        for (int64_t sp = 0; sp < splits; ++sp) s += ws[sp * total_bins + bin];
        counts[bin] = s;
        mine += s;
    }
    mine = warp_sum(mine);
    if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = mine;
    __syncthreads();
    if (threadIdx.x == 0 && row_totals) {
        int64_t t = 0;
        for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) t += warp_tot[w];
        row_totals[row] = t;
    }
}

exf_status check_hist_args(int64_t T, int32_t L, int32_t E, int32_t gap) {
    // RoutingTrace::validate (proj/src/trace.cpp:53-70) and the gap check (:193-196)
    if (E < 1) return invalid("num_experts must be >= 1, got " + std::to_string(E));
    if (L < 2) return invalid("num_layers must be >= 2, got " + std::to_string(L));
    if (T < 1) return invalid("trace contains no token paths");
    if (gap < 1 || gap > L - 1)
        return invalid("gap " + std::to_string(gap) + " out of range [1," + std::to_string(L - 1) +
                       "]");
    if ((int64_t)E * E * 2 > kCounterSmemBudget)
        return invalid("num_experts " + std::to_string(E) + " exceeds the histogram kernel limit");
    if ((int64_t)kTileTokens * L * 4 > 32 * 1024) return invalid("num_layers too large");
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
    EXF_TRY(check_hist_args(T, L, E, gap));
    if (!d_paths || !d_counts || !d_workspace) return invalid("null device pointer");
    const HistPlan p = plan_hist(T, L, E, gap);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    EXF_CUDA_TRY(cudaFuncSetAttribute(hist_partial_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)p.smem_bytes));
    dim3 grid(p.groups, (unsigned)p.splits);
    hist_partial_kernel<<<grid, kHistThreads, p.smem_bytes, s>>>(
        d_paths, T, L, E, gap, p.pairs, p.pair_group, p.splits, p.counter_words,
        static_cast<uint16_t*>(d_workspace));
    EXF_LAUNCH_CHECK("hist_partial_kernel");
    const int threads = std::max(32, std::min(256, ((E + 31) / 32) * 32));
    hist_reduce_kernel<<<p.pairs * E, threads, 0, s>>>(static_cast<uint16_t*>(d_workspace),
                                                       p.splits, p.pairs, E, d_counts,
                                                       d_row_totals);
    EXF_LAUNCH_CHECK("hist_reduce_kernel");
    return EXF_OK;
}

extern "C" exf_status exf_count_transitions_host(const int32_t* h_paths, int64_t T, int32_t L,
                                                 int32_t E, int32_t gap, int64_t* h_counts,
                                                 int64_t* h_row_totals) {
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
