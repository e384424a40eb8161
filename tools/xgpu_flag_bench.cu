// xgpu_flag_bench.cu -- diagnostics: latency of ONE dispatch exchange round
// between G GPUs of one node (one process, P2P over NVLink), the pattern of
// the fused layer kernel's token phase at configs[1] (B tokens per GPU, C =
// G*B slots, 148 CTAs x tpc slots, 2 KB token rows), for several
// publish/poll protocols. Rounds run back to back inside one persistent
// kernel per GPU (epoch-tagged flags, parity double buffers); per-round time
// = kernel time / rounds.
//
// Variants
//   0  per-slot flags at every destination, each st.release.sys by its own
//      thread; every CTA polls all G*C flags (relaxed spin + ld.acquire.sys)
//      [the round-1 kernel]
//   1  as 0, but each writer warp issues one fence.acq_rel.sys after its row
//      stores, then bar.sync, then relaxed.sys flag stores; pollers spin
//      relaxed and fence once at the end
//   2  as 1, but ONE flag per (source CTA, destination) carrying the CTA's
//      slot bitmask: G*148 flags per destination instead of G*C
//   3  as 2, but only tokens that changed GPU are signalled remotely: a
//      CTA's local routes go through a GPU-scope flag (relaxed.gpu) and only
//      CTAs with remote tokens for a destination set a .sys flag there; the
//      destination learns which source CTAs will signal from a per-source
//      CTA-presence bitmask published once per round by the last arriving
//      source CTA (one .sys flag per (source, destination))
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//        -I../paper_2401_08383_b200/csrc xgpu_flag_bench.cu -o xgpu_flag_bench
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"

using namespace exf;

constexpr int kThreads = 256;
constexpr int kCtas = 148;

struct Args {
    int G, me, B, C, tpc, d, rounds, variant;
    float cross;                 // fraction of tokens routed to another GPU
    uint8_t* peers[8];           // per-GPU symmetric buffers
    long long* out;              // [0] ns total
};

// symmetric layout (same offsets on every GPU)
//   rows  [2][G][C][d] bf16
//   sflag [2][G][C]    u64   per-slot flags (variants 0, 1)
//   cflag [2][G][kCtas] u64  per-(source CTA) flags (variants 2, 3)
//   pres  [2][G]       u64   per-source presence masks + epoch (variant 3, 64-bit epoch | count)
//   ctr   [2]          u32   local arrival counters (variant 3)
struct Layout {
    size_t rows, sflag, cflag, pres, pacc, ctr, total;
};
__host__ __device__ inline Layout layout(int G, int C, int d) {
    Layout l{};
    size_t o = 0;
    auto take = [&](size_t b) { size_t at = o; o += (b + 255) & ~size_t(255); return at; };
    l.rows = take((size_t)2 * G * C * d * 2);
    l.sflag = take((size_t)2 * G * C * 8);
    l.cflag = take((size_t)2 * G * kCtas * 8);
    l.pres = take((size_t)2 * G * 8 * 8);
    l.pacc = take((size_t)2 * 8 * 4 * 8);
    l.ctr = take(64);
    l.total = o;
    return l;
}

__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys64(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// destination of token t at round r (deterministic; `cross` of them remote)
__device__ __forceinline__ int dest_of(const Args& a, int t, int r) {
    const uint32_t h = (uint32_t)(t * 2654435761u) ^ (uint32_t)(r * 40503u) ^ (uint32_t)(a.me * 97u);
    const float u = (float)(h & 0xFFFF) / 65536.f;
    if (u >= a.cross || a.G == 1) return a.me;
    return (a.me + 1 + (int)((h >> 16) % (uint32_t)(a.G - 1))) % a.G;
}

__global__ void __launch_bounds__(kThreads, 1) exchange_kernel(Args a) {
    const Layout L = layout(a.G, a.C, a.d);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int t0 = blockIdx.x * a.tpc;
    const int K = a.G * a.C;
    uint8_t* own = a.peers[a.me];
    __shared__ int s_dest[32];
    const uint64_t t_start = ptx::globaltimer();
    for (int r = 0; r < a.rounds; ++r) {
        const int par = r & 1;
        const uint64_t ep = (uint64_t)r + 1;
        if (tid < a.tpc) s_dest[tid] = (t0 + tid < a.B) ? dest_of(a, t0 + tid, r) : -1;  // B real tokens
        __syncthreads();
        // ---- rows: warp i copies token i of this CTA to its destination slot
        for (int i = warp; i < a.tpc; i += kThreads / 32) {
            const int g = s_dest[i];
            if (g < 0) continue;
            int4* dst = reinterpret_cast<int4*>(a.peers[g] + L.rows +
                                                 (((size_t)par * a.G + a.me) * a.C + t0 + i) * a.d * 2);
            const int4 v = make_int4(r, t0 + i, a.me, 7);
            for (int u = lane; u < a.d / 8; u += 32) dst[u] = v;
        }
        if (a.variant >= 1) fence_sys();  // each writer warp: its rows visible system-wide
        __syncthreads();
        // ---- publish
        if (a.variant <= 1) {
            for (int q = kThreads - 1 - tid; q < a.tpc * a.G; q += kThreads) {
                const int i = q / a.G, g = q - i * a.G;
                if (t0 + i >= a.C) continue;
                const uint64_t slotv = (s_dest[i] == g) ? 1u : 0xFFu;
                uint64_t* f = reinterpret_cast<uint64_t*>(a.peers[g] + L.sflag) + ((size_t)par * a.G + a.me) * a.C + t0 + i;
                if (a.variant == 0) st_release_sys64(f, (ep << 40) | (slotv << 32));
                else st_relaxed_sys(f, (ep << 40) | (slotv << 32));
            }
        } else {
            if (tid < a.G) {
                const int g = tid;
                uint32_t mask = 0;
                for (int i = 0; i < a.tpc; ++i)
                    if (s_dest[i] == g) mask |= 1u << i;
                uint64_t* f = reinterpret_cast<uint64_t*>(a.peers[g] + L.cflag) + ((size_t)par * a.G + a.me) * kCtas + blockIdx.x;
                if (a.variant == 2 || mask != 0 || g == a.me)
                    st_relaxed_sys(f, (ep << 40) | mask);
                if (a.variant == 3 && g != a.me && mask == 0) {
                    // no remote tokens for g from this CTA: the presence mask says so
                }
            }
            if (a.variant == 3) {
                // per-source presence masks: bit c set if CTA c sends to g;
                // published by the last arriving CTA of this GPU
                __shared__ int s_last;
                uint32_t* ctr = reinterpret_cast<uint32_t*>(own + L.ctr) + par;
                unsigned long long* pm = reinterpret_cast<unsigned long long*>(own + L.pacc) + (size_t)par * 8 * 4;
                if (tid < a.G) {
                    uint32_t mask = 0;
                    for (int i = 0; i < a.tpc; ++i)
                        if (s_dest[i] == tid) mask |= 1u << i;
                    if (mask && tid != a.me) atomicOr(&pm[tid * 4 + blockIdx.x / 64], 1ull << (blockIdx.x % 64));
                }
                __syncthreads();
                if (tid == 0) {
                    __threadfence();
                    const uint32_t prev = atomicAdd(ctr, 1u);
                    s_last = prev == (uint32_t)(gridDim.x - 1);
                }
                __syncthreads();
                if (s_last && tid == 0) *ctr = 0;  // next use: round r+2 (after the peers' round r+1)
                if (s_last && tid < a.G && tid != a.me) {
                    __threadfence();
                    const int g = tid;
                    uint64_t w3[3];
                    for (int w = 0; w < 3; ++w) {  // take and clear before publishing
                        w3[w] = pm[g * 4 + w];
                        pm[g * 4 + w] = 0;
                    }
                    uint64_t* dstp = reinterpret_cast<uint64_t*>(a.peers[g] + L.pres) + ((size_t)par * a.G + a.me) * 8;
                    for (int w = 0; w < 3; ++w) dstp[1 + w] = w3[w];
                    fence_sys();
                    st_relaxed_sys(dstp, ep);
                }
            }
        }
        // ---- poll
        if (a.variant <= 1) {
            const uint64_t* f = reinterpret_cast<const uint64_t*>(own + L.sflag) + (size_t)par * K;
            for (int k = tid; k < K; k += kThreads) {
                ptx::SpinGuard g;
                while ((ptx::ld_relaxed_u64(f + k, true) >> 40) != ep) g.step(nullptr, 0, 2000000000ull);
                if (a.variant == 0) (void)ld_acquire_sys64(f + k);
            }
            if (a.variant == 1) fence_sys();
        } else if (a.variant == 2) {
            const uint64_t* f = reinterpret_cast<const uint64_t*>(own + L.cflag) + (size_t)par * a.G * kCtas;
            for (int k = tid; k < a.G * kCtas; k += kThreads) {
                if (k % kCtas >= (int)gridDim.x) continue;
                ptx::SpinGuard g;
                while ((ptx::ld_relaxed_u64(f + k, true) >> 40) != ep) g.step(nullptr, 0, 2000000000ull);
            }
            fence_sys();
        } else {
            // presence masks first (one per remote source), then the flagged CTAs
            const uint64_t* p = reinterpret_cast<const uint64_t*>(own + L.pres) + (size_t)par * a.G * 8;
            const uint64_t* f = reinterpret_cast<const uint64_t*>(own + L.cflag) + (size_t)par * a.G * kCtas;
            for (int src = 0; src < a.G; ++src) {
                if (src == a.me) continue;
                if (tid == 0) {
                    ptx::SpinGuard g;
                    while (ptx::ld_relaxed_u64(p + src * 8, true) != ep) g.step(nullptr, 0, 2000000000ull);
                }
            }
            fence_sys();
            __syncthreads();
            for (int k = tid; k < a.G * kCtas; k += kThreads) {
                const int src = k / kCtas, c = k % kCtas;
                if (src == a.me || c >= (int)gridDim.x) continue;
                const uint64_t bits = ptx::ld_relaxed_u64(p + src * 8 + 1 + c / 64, true);
                if (!((bits >> (c % 64)) & 1)) continue;
                ptx::SpinGuard g;
                while ((ptx::ld_relaxed_u64(f + k, true) >> 40) != ep) g.step(nullptr, 0, 2000000000ull);
            }
            fence_sys();
        }
        __syncthreads();
    }
    if (tid == 0 && blockIdx.x == 0) a.out[0] = (long long)(ptx::globaltimer() - t_start);
}


// ---------------------------------------------------------------------------
// Protocol matrix (variant = 100 + rows*100 + pub*10 + poll):
//   rows  0 none, 1 token rows stored first
//   pub   0 per-slot st.release.sys by distinct threads after bar.sync
//         1 per-slot st.relaxed.sys
//         2 per-(CTA, dest) st.release.sys by thread 0..G-1 after bar.sync
//         3 per-(CTA, dest) st.relaxed.sys
//         4 per-slot st.release.sys by the warp that wrote the row (lane 0)
//   poll  0 every thread: relaxed spin + ld.acquire.sys per flag
//         1 every thread: relaxed spin only
//         2 warp 0 of each CTA polls, bar.sync releases the rest
//         3 CTA 0 polls everything, then a GPU-scope broadcast flag
__global__ void __launch_bounds__(kThreads, 1) matrix_kernel(Args a, int rows_on, int pub, int poll,
                                                             uint64_t* bcast) {
    const Layout L = layout(a.G, a.C, a.d);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int t0 = blockIdx.x * a.tpc;
    uint8_t* own = a.peers[a.me];
    __shared__ int s_dest[32];
    const bool per_cta = pub == 2 || pub == 3;
    const int nflags = per_cta ? a.G * (int)gridDim.x : a.G * a.C;
    const uint64_t t_start = ptx::globaltimer();
    for (int r = 0; r < a.rounds; ++r) {
        const int par = r & 1;
        const uint64_t ep = (uint64_t)r + 1;
        if (tid < a.tpc) s_dest[tid] = (t0 + tid < a.B) ? dest_of(a, t0 + tid, r) : -1;
        __syncthreads();
        for (int i = warp; i < a.tpc; i += kThreads / 32) {
            const int g = s_dest[i];
            if (rows_on && g >= 0) {
                int4* dst = reinterpret_cast<int4*>(a.peers[g] + L.rows +
                                                     (((size_t)par * a.G + a.me) * a.C + t0 + i) * a.d * 2);
                const int4 v = make_int4(r, t0 + i, a.me, 7);
                for (int u = lane; u < a.d / 8; u += 32) dst[u] = v;
            }
            if (pub == 4 && t0 + i < a.C) {
                __syncwarp();
                if (lane < a.G) {
                    const uint64_t slotv = (g == lane) ? 1u : 0xFFu;
                    uint64_t* f = reinterpret_cast<uint64_t*>(a.peers[lane] + L.sflag) +
                                  ((size_t)par * a.G + a.me) * a.C + t0 + i;
                    st_release_sys64(f, (ep << 40) | (slotv << 32));
                }
            }
        }
        __syncthreads();
        if (pub == 0 || pub == 1) {
            for (int q = kThreads - 1 - tid; q < a.tpc * a.G; q += kThreads) {
                const int i = q / a.G, g = q - i * a.G;
                if (t0 + i >= a.C) continue;
                const uint64_t slotv = (s_dest[i] == g) ? 1u : 0xFFu;
                uint64_t* f = reinterpret_cast<uint64_t*>(a.peers[g] + L.sflag) + ((size_t)par * a.G + a.me) * a.C + t0 + i;
                if (pub == 0) st_release_sys64(f, (ep << 40) | (slotv << 32));
                else st_relaxed_sys(f, (ep << 40) | (slotv << 32));
            }
        } else if (per_cta && tid < a.G) {
            const int g = tid;
            uint32_t mask = 0;
            for (int i = 0; i < a.tpc; ++i)
                if (s_dest[i] == g) mask |= 1u << i;
            uint64_t* f = reinterpret_cast<uint64_t*>(a.peers[g] + L.cflag) + ((size_t)par * a.G + a.me) * kCtas + blockIdx.x;
            if (pub == 2) st_release_sys64(f, (ep << 40) | mask);
            else st_relaxed_sys(f, (ep << 40) | mask);
        }
        const uint64_t* f = reinterpret_cast<const uint64_t*>(own + (per_cta ? L.cflag : L.sflag)) +
                            (size_t)par * (per_cta ? a.G * kCtas : a.G * a.C);
        auto flag_at = [&](int k) {
            return per_cta ? f + (k / (int)gridDim.x) * kCtas + (k % (int)gridDim.x) : f + k;
        };
        if (poll == 0 || poll == 1) {
            for (int k = tid; k < nflags; k += kThreads) {
                ptx::SpinGuard g;
                while ((ptx::ld_relaxed_u64(flag_at(k), true) >> 40) != ep) g.step(nullptr, 0, 2000000000ull);
                if (poll == 0) (void)ld_acquire_sys64(flag_at(k));
            }
        } else if (poll == 2) {
            if (warp == 0) {
                for (int k = lane; k < nflags; k += 32) {
                    ptx::SpinGuard g;
                    while ((ptx::ld_relaxed_u64(flag_at(k), true) >> 40) != ep) g.step(nullptr, 0, 2000000000ull);
                    (void)ld_acquire_sys64(flag_at(k));
                }
            }
        } else {
            if (blockIdx.x == 0) {
                for (int k = tid; k < nflags; k += kThreads) {
                    ptx::SpinGuard g;
                    while ((ptx::ld_relaxed_u64(flag_at(k), true) >> 40) != ep) g.step(nullptr, 0, 2000000000ull);
                    (void)ld_acquire_sys64(flag_at(k));
                }
                __syncthreads();
                if (tid == 0) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(bcast), "l"(ep) : "memory");
            } else if (tid == 0) {
                ptx::SpinGuard g;
                while (ptx::ld_relaxed_u64(bcast, false) < ep) g.step(nullptr, 0, 2000000000ull);
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
        __syncthreads();
    }
    if (tid == 0 && blockIdx.x == 0) a.out[0] = (long long)(ptx::globaltimer() - t_start);
}

int main(int argc, char** argv) {
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    const int G = argc > 1 ? atoi(argv[1]) : ndev;
    const int B = argc > 2 ? atoi(argv[2]) : 64;
    const float cross = argc > 3 ? (float)atof(argv[3]) : 0.75f;
    if (G > ndev || G < 1) {
        printf("need %d GPUs, have %d\n", G, ndev);
        return 1;
    }
    const int C = G * B, d = 1024, tpc = (C + kCtas - 1) / kCtas;
    const Layout L = layout(G, C, d);
    std::vector<uint8_t*> bufs(G);
    std::vector<long long*> outs(G);
    std::vector<cudaStream_t> streams(G);
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(g);
        for (int h = 0; h < G; ++h)
            if (h != g) cudaDeviceEnablePeerAccess(h, 0);
        cudaMalloc(&bufs[g], L.total);
        cudaMemset(bufs[g], 0, L.total);
        cudaMalloc(&outs[g], 64);
        cudaStreamCreate(&streams[g]);
        cudaFuncSetAttribute(exchange_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(exchange_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    }
    printf("G=%d B=%d C=%d tpc=%d cross=%.2f (%s)\n", G, B, C, tpc, cross,
           cudaGetErrorString(cudaGetLastError()));
    const char* names[] = {"per-slot flags, st.release.sys each, poll all G*C",
                           "per-slot flags, warp fence + relaxed, poll all G*C",
                           "per-(CTA, dest) mask flags, G*148 polled",
                           "presence masks + flags only from sending CTAs"};
    for (int variant = 0; variant < 4; ++variant) {
        for (int rep = 0; rep < 2; ++rep) {
            const int rounds = rep == 0 ? 20 : 400;
            for (int g = 0; g < G; ++g) {  // fresh epochs per run
                cudaSetDevice(g);
                cudaMemset(bufs[g], 0, L.total);
            }
            for (int g = 0; g < G; ++g) cudaSetDevice(g), cudaDeviceSynchronize();
            for (int g = 0; g < G; ++g) {
                cudaSetDevice(g);
                Args a{};
                a.G = G;
                a.me = g;
                a.B = B;
                a.C = C;
                a.tpc = tpc;
                a.d = d;
                a.rounds = rounds;
                a.variant = variant;
                a.cross = cross;
                for (int h = 0; h < G; ++h) a.peers[h] = bufs[h];
                a.out = outs[g];
                exchange_kernel<<<kCtas, kThreads, 150 * 1024, streams[g]>>>(a);  // one CTA per SM
            }
            long long worst = 0;
            for (int g = 0; g < G; ++g) {
                cudaSetDevice(g);
                cudaError_t e = cudaStreamSynchronize(streams[g]);
                if (e != cudaSuccess) {
                    printf("variant %d: %s\n", variant, cudaGetErrorString(e));
                    return 1;
                }
                long long ns = 0;
                cudaMemcpy(&ns, outs[g], 8, cudaMemcpyDeviceToHost);
                worst = ns > worst ? ns : worst;
            }
            if (rep == 1) printf("  v%d %-52s %.2f us per exchange round\n", variant, names[variant],
                                 worst / 1000.0 / rounds);
        }
    }
    // protocol matrix
    std::vector<uint64_t*> bc(G);
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(g);
        cudaMalloc(&bc[g], 64);
        cudaFuncSetAttribute(matrix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    }
    const int combos[][3] = {{0, 0, 0}, {0, 1, 1}, {1, 0, 0}, {1, 0, 1}, {1, 0, 2}, {1, 0, 3}, {1, 4, 0},
                             {1, 4, 2}, {1, 2, 0}, {1, 2, 2}, {1, 2, 3}, {0, 3, 1}, {1, 3, 1}};
    for (const auto& cb : combos) {
        double per = 0;
        for (int rep = 0; rep < 2; ++rep) {
            const int rounds = rep == 0 ? 20 : 400;
            for (int g = 0; g < G; ++g) {
                cudaSetDevice(g);
                cudaMemset(bufs[g], 0, L.total);
                cudaMemset(bc[g], 0, 64);
            }
            for (int g = 0; g < G; ++g) cudaSetDevice(g), cudaDeviceSynchronize();
            for (int g = 0; g < G; ++g) {
                cudaSetDevice(g);
                Args a{};
                a.G = G; a.me = g; a.B = B; a.C = C; a.tpc = tpc; a.d = d; a.rounds = rounds; a.cross = cross;
                for (int h = 0; h < G; ++h) a.peers[h] = bufs[h];
                a.out = outs[g];
                matrix_kernel<<<kCtas, kThreads, 150 * 1024, streams[g]>>>(a, cb[0], cb[1], cb[2], bc[g]);
            }
            long long worst = 0;
            for (int g = 0; g < G; ++g) {
                cudaSetDevice(g);
                cudaError_t e = cudaStreamSynchronize(streams[g]);
                if (e != cudaSuccess) {
                    printf("matrix %d%d%d: %s\n", cb[0], cb[1], cb[2], cudaGetErrorString(e));
                    return 1;
                }
                long long ns = 0;
                cudaMemcpy(&ns, outs[g], 8, cudaMemcpyDeviceToHost);
                worst = ns > worst ? ns : worst;
            }
            per = worst / 1000.0 / rounds;
        }
        printf("  rows=%d pub=%d poll=%d  %.2f us per round\n", cb[0], cb[1], cb[2], per);
    }
    return 0;
}
