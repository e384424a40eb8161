// replay.cu -- routing replay: the per-token, per-layer hot loop of
// exflow::simulate (proj/src/sim.cpp:110-145), as exact integer counters.
//
// One thread follows one token through the L layers (the coherent location is
// a sequential dependency). v2 after the round-1 capture (239 us for 201 MB
// of ids, 0.13 of HBM): persistent CTAs stream the trace through a software
// pipeline (the next tile's rows in flight as 16-byte non-allocating loads
// while the current tile is replayed from shared memory, rows padded to L|1
// words so per-thread column reads are bank-conflict free); the placement
// table lives in shared memory with each entry packed as {gpu, node} so the
// loop does no integer division; counters are reduced warp -> CTA -> one
// 64-bit atomic per counter per CTA (integer sums: order-independent,
// bit-exact).
// Algorithmic bytes per launch: 4*T*L (+4*T homes when given).
#include "common.cuh"

#include <algorithm>
#include <string>
#include <vector>

namespace exf {
namespace {

constexpr int kReplayThreads = 256;
constexpr int kReplayPrefetch = 8;  // int4 per thread per tile (tile <= 256 tokens x 32 layers)

// MODE 1 (coherent) / 0 (vanilla). Per token and layer only the comparisons
// that cannot be derived are counted (entries packed as gpu | node << 16; the
// current GPU is tracked in both modes, sim.cpp:112/:143):
//   same  = #(expert GPU == current GPU)       -> gpu_local, and moves = L - same
//   snode = #(expert node == current node)     -> node_local
//   away  = #(expert GPU != home)              -> away_from_home
//   anode = #(expert node != home node)        (vanilla)
// coherent: hops_inter = #(node changes) = L - snode, hops_intra = snode - same;
// vanilla: hops_inter = 2 anode, hops_intra = 2 (away - anode) (sim.cpp:60-71)
template <int MODE>
__global__ void __launch_bounds__(kReplayThreads)
route_replay_kernel(const int32_t* __restrict__ paths, const int32_t* __restrict__ homes,
                    const int32_t* __restrict__ assign, int64_t T, int32_t L, int32_t E,
                    int32_t gpus_per_node, int32_t gpus, unsigned long long* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int32_t stride = L | 1;
    int32_t* s_tab = reinterpret_cast<int32_t*>(smem);  // [L][E] gpu | node << 16
    int32_t* tile = s_tab + ((L * E + 3) & ~3);
    __shared__ unsigned long long s_cnt[6];
    const int tid = threadIdx.x;
    for (int32_t i = tid; i < L * E; i += blockDim.x) {
        const int32_t g = assign[i];
        s_tab[i] = g | ((g / gpus_per_node) << 16);
    }
    if (tid < 6) s_cnt[tid] = 0ull;

    const bool vec = ((reinterpret_cast<uintptr_t>(paths) | (uintptr_t)(L * 4)) & 15) == 0 &&
                     L * kReplayThreads <= kReplayPrefetch * 4 * kReplayThreads;
    const int64_t tiles = (T + kReplayThreads - 1) / kReplayThreads;
    int4 pre[kReplayPrefetch];
    auto fetch = [&](int64_t tile_id) {
        const int64_t t0 = tile_id * kReplayThreads;
        const int32_t nvec = (int32_t)imin64(kReplayThreads, T - t0) * L / 4;
        const int4* s4 = reinterpret_cast<const int4*>(paths + t0 * L);
#pragma unroll
        for (int u = 0; u < kReplayPrefetch; ++u) {
            const int32_t i = tid + u * kReplayThreads;
            if (i < nvec) pre[u] = ld_nc_v4(s4 + i);
        }
    };
    int64_t c_same = 0, c_snode = 0, c_away = 0, c_anode = 0, c_tok = 0;
    if (vec && blockIdx.x < tiles) fetch(blockIdx.x);
    for (int64_t tile_id = blockIdx.x; tile_id < tiles; tile_id += gridDim.x) {
        const int64_t t0 = tile_id * kReplayThreads;
        const int32_t nt = (int32_t)imin64(kReplayThreads, T - t0);
        __syncthreads();  // previous tile replayed (and the table built)
        if (vec) {
            const int32_t nvec = nt * L / 4;
#pragma unroll
            for (int u = 0; u < kReplayPrefetch; ++u) {
                const int32_t i = tid + u * kReplayThreads;
                if (i < nvec) {
                    const int32_t e0 = 4 * i, r = e0 / L, c = e0 - r * L;  // L % 4 == 0: no row straddle
                    int32_t* d = tile + r * stride + c;
                    d[0] = pre[u].x;
                    d[1] = pre[u].y;
                    d[2] = pre[u].z;
                    d[3] = pre[u].w;
                }
            }
            if (tile_id + gridDim.x < tiles) fetch(tile_id + gridDim.x);  // in flight during the replay
        } else {
            const int32_t* src = paths + t0 * L;
            for (int32_t i = tid; i < nt * L; i += blockDim.x) {
                const int32_t r = i / L;
                tile[r * stride + (i - r * L)] = __ldg(src + i);
            }
        }
        __syncthreads();
        if (tid < nt) {
            const int64_t t = t0 + tid;
            const int32_t home = homes ? __ldg(homes + t) : (int32_t)(t % gpus);
            const int32_t home_ent = home | ((home / gpus_per_node) << 16);
            int32_t loc_ent = home_ent;
            int32_t same = 0, snode = 0, away = 0, anode = 0;  // per tile: <= L each
            const int32_t* p = tile + tid * stride;
            const int32_t* tab = s_tab;
            for (int32_t j = 0; j < L; ++j, tab += E) {
                const int32_t e = p[j];
                const int32_t ent = ((unsigned)e < (unsigned)E) ? tab[e] : loc_ent;
                // the current GPU is tracked in both modes (sim.cpp:112, :143)
                same += (ent == loc_ent);
                snode += ((ent ^ loc_ent) >> 16) == 0;
                if (MODE == 0) anode += ((ent ^ home_ent) >> 16) != 0;
                loc_ent = ent;
                away += ((ent ^ home_ent) & 0xFFFF) != 0;
            }
            c_same += same;
            c_snode += snode;
            c_away += away;
            c_anode += anode;
            ++c_tok;
        }
    }
    // gpu_local, node_local, away, coherent moves, hops intra, hops inter
    const int64_t tl = c_tok * L;
    int64_t v[6];
    v[0] = c_same;
    v[1] = c_snode;
    v[2] = c_away;
    v[3] = tl - c_same;
    if (MODE == 1) {
        v[4] = c_snode - c_same;
        v[5] = tl - c_snode;
    } else {
        v[4] = 2 * (c_away - c_anode);
        v[5] = 2 * c_anode;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const int64_t sm = warp_sum(v[k]);
        if ((tid & 31) == 0 && sm) atomicAdd(&s_cnt[k], (unsigned long long)sm);
    }
    __syncthreads();
    if (tid < 6 && s_cnt[tid]) atomicAdd(&out[tid], s_cnt[tid]);
}

}  // namespace
}  // namespace exf

using namespace exf;

extern "C" exf_status exf_route_replay(const int32_t* d_paths, const int32_t* d_homes,
                                       const int32_t* d_assign, int64_t T, int32_t L, int32_t E,
                                       int32_t num_nodes, int32_t gpus_per_node, int32_t mode,
                                       exf_sim_counters* d_out, exf_stream_t stream) {
    if (num_nodes < 1 || gpus_per_node < 1)
        return invalid("topology must have at least one node and one GPU per node");
    if (E < 1 || L < 1 || T < 1) return invalid("replay needs T, L, E >= 1");
    if (mode != 0 && mode != 1) return invalid("mode must be 0 (vanilla) or 1 (coherent)");
    if ((int64_t)L * E * 4 + (int64_t)kReplayThreads * (L | 1) * 4 > 200 * 1024)
        return invalid("placement table too large for the replay kernel");
    if (num_nodes * gpus_per_node > 0x7FFF) return invalid("too many GPUs for the replay kernel");
    if (!d_paths || !d_assign || !d_out) return invalid("null device pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t smem = (size_t)((L * E + 3) & ~3) * 4 + (size_t)kReplayThreads * (L | 1) * 4;
    auto kern = mode == 1 ? route_replay_kernel<1> : route_replay_kernel<0>;
    EXF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    EXF_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(exf_sim_counters), s));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = (T + kReplayThreads - 1) / kReplayThreads;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 4LL * sms));
    kern<<<blocks, kReplayThreads, smem, s>>>(d_paths, d_homes, d_assign, T, L, E, gpus_per_node,
                                              num_nodes * gpus_per_node,
                                              reinterpret_cast<unsigned long long*>(d_out));
    EXF_LAUNCH_CHECK("route_replay_kernel");
    return EXF_OK;
}

extern "C" exf_status exf_sim_report_from_counters(const exf_sim_counters* c, int64_t T,
                                                   int32_t L, int32_t num_nodes,
                                                   int32_t gpus_per_node, double intra_cost,
                                                   double inter_cost, int32_t tokens_per_gpu,
                                                   int32_t mode, exf_sim_report* out) {
    if (!c || !out) return invalid("null pointer");
    if (tokens_per_gpu < 1) return invalid("tokens_per_gpu must be >= 1");
    const int32_t gpus = num_nodes * gpus_per_node;
    *out = exf_sim_report{};
    out->hops_intra_node = c->hops_intra_node;
    out->hops_inter_node = c->hops_inter_node;
    const double events = (double)T * L;  // sim.cpp:147-151
    out->locality_gpu = c->gpu_local_events / events;
    out->locality_node = c->node_local_events / events;
    out->p = c->away_from_home_events / events;
    out->p_star = c->coherent_moves / events;
    const double g = gpus, n = tokens_per_gpu, l = L;
    if (mode == 0) {  // sim.cpp:153-157, volume_table1 deepspeed top-1 (:171-191)
        out->alltoall_count = 2LL * L;
        out->volume_units = 2.0 * g * n * l * out->p;
    } else {  // sim.cpp:158-165, exflow top-1
        out->alltoall_count = L;
        out->allgather_count = 1;
        out->setup_allgather_count = 1;
        out->volume_units = g * n * (l * out->p_star + g);
    }
    out->estimated_latency = c->hops_intra_node * intra_cost + c->hops_inter_node * inter_cost;
    return EXF_OK;
}

extern "C" exf_status exf_simulate_host(const int32_t* h_paths, int64_t T, int32_t L,
                                        int32_t E, const int32_t* h_assign, int32_t num_nodes,
                                        int32_t gpus_per_node, double intra_cost,
                                        double inter_cost, int32_t tokens_per_gpu, int32_t mode,
                                        const int32_t* h_homes, exf_sim_report* out) {
    exf::NvtxRange nvtx_range("exf.simulate_host");
    // validation order follows simulate (proj/src/sim.cpp:78-105): the trace
    // (trace.cpp:53-70), then the placement (placement.cpp:434-470), then the
    // config (topology, then tokens_per_gpu; sim.cpp:24-32), then the homes
    if (E < 1) return invalid("num_experts must be >= 1, got " + std::to_string(E));
    if (L < 2) return invalid("num_layers must be >= 2, got " + std::to_string(L));
    if (T < 1) return invalid("trace contains no token paths");
    for (int64_t i = 0; i < T * (int64_t)L; ++i)
        if (h_paths[i] < 0 || h_paths[i] >= E)
            return invalid("expert id out of range [0," + std::to_string(E) + ")");
    if (num_nodes < 1 || gpus_per_node < 1) return invalid("placement grid must be at least 1x1");
    const int32_t gpus = num_nodes * gpus_per_node;
    if (E % gpus != 0)
        return invalid("num_experts " + std::to_string(E) + " not divisible by total GPUs " +
                       std::to_string(gpus));
    const int32_t cap = E / gpus;
    std::vector<int32_t> load(gpus);
    for (int32_t j = 0; j < L; ++j) {
        std::fill(load.begin(), load.end(), 0);
        for (int32_t e = 0; e < E; ++e) {
            const int32_t g = h_assign[j * E + e];
            if (g < 0 || g >= gpus)
                return invalid("gpu id " + std::to_string(g) + " out of range [0," +
                               std::to_string(gpus) + ") at layer " + std::to_string(j));
            load[g]++;
        }
        for (int32_t g = 0; g < gpus; ++g)
            if (load[g] != cap)
                return invalid("layer " + std::to_string(j) + " places " + std::to_string(load[g]) +
                               " experts on gpu " + std::to_string(g) + ", expected " +
                               std::to_string(cap));
    }
    if (intra_cost < 0.0 || inter_cost < intra_cost)
        return invalid("hop costs must satisfy inter >= intra >= 0");
    if (tokens_per_gpu < 1) return invalid("tokens_per_gpu must be >= 1");
    if (h_homes)
        for (int64_t t = 0; t < T; ++t)
            if (h_homes[t] < 0 || h_homes[t] >= gpus) return invalid("home gpu out of range");
    const size_t paths_b = (size_t)T * L * 4, assign_b = (size_t)L * E * 4;
    const size_t homes_b = h_homes ? (size_t)T * 4 : 0;
    const size_t cnt_off = (paths_b + assign_b + homes_b + 15) & ~size_t(15);
    HostScratch* hs = nullptr;  // cached per thread and device: no per-call cudaMalloc
    EXF_TRY(host_scratch(cnt_off + sizeof(exf_sim_counters) + 64, paths_b, &hs));
    uint8_t* buf = hs->dev;
    int32_t* d_paths = reinterpret_cast<int32_t*>(buf);
    int32_t* d_assign = reinterpret_cast<int32_t*>(buf + paths_b);
    int32_t* d_homes = h_homes ? reinterpret_cast<int32_t*>(buf + paths_b + assign_b) : nullptr;
    exf_sim_counters* d_out = reinterpret_cast<exf_sim_counters*>(buf + cnt_off);
    exf_sim_counters c{};
    EXF_TRY(hs->h2d(d_paths, h_paths, paths_b));
    EXF_TRY(hs->h2d(d_assign, h_assign, assign_b));
    if (h_homes) EXF_TRY(hs->h2d(d_homes, h_homes, homes_b));
    EXF_TRY(exf_route_replay(d_paths, d_homes, d_assign, T, L, E, num_nodes, gpus_per_node, mode,
                             d_out, hs->stream));
    EXF_TRY(hs->d2h(&c, d_out, sizeof(c)));
    return exf_sim_report_from_counters(&c, T, L, num_nodes, gpus_per_node, intra_cost,
                                        inter_cost, tokens_per_gpu, mode, out);
}
