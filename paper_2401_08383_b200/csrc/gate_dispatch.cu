// gate_dispatch.cu -- per-layer token-side kernel of the ExFlow decode step,
// plus step begin and the context AllGather.
//
// gate_dispatch_kernel (kernels 1 + 5' + 2 + 3 fused, latency-optimised):
//  (1) gate: the layer's gate matrix Wg [E][d] is staged in shared memory;
//      one warp per token computes the logits in the fixed fp32 reduction
//      order documented in oracle/exflow_model_oracle.c (32 lane partials,
//      c-major / i-minor FMA, xor-butterfly), so routing is bit-identical to
//      the CPU oracle; top-1 ties -> lowest expert index; softmax prob.
//  (5') fused affinity histogram hist[j-1][prev][e] += 1 and trace emission.
//  (2) deterministic, atomic-free bucketing by (destination GPU, local slot):
//      each CTA owns a contiguous token slice; warp-aggregated ranks
//      (__match_any_sync + popc(lanemask_lt)) give per-CTA key counts; one
//      grid barrier publishes them; every CTA prefix-sums the counts of the
//      CTAs before it -> stable global positions (token order within a key).
//  (3) ExFlow's single dispatch exchange: rows are stored straight into the
//      destination rank's symmetric receive region over NVLink (P2P stores
//      through CUDA-IPC mapped pointers); the last CTA writes the per-(src,
//      slot) counts and release-flags every destination. Tokens stay on their
//      expert's GPU (coherent mode, proj/src/sim.cpp:65-71; no combine).
// gather_send/gather_wait (3b): the per-step context AllGather; every rank
// scatters its resident tokens' states into every peer's token-id-indexed
// output buffer, then waits for all peers' flags.
#include "common.cuh"
#include "model.cuh"
#include "ptx.cuh"

#include <cuda_bf16.h>

#include <algorithm>

namespace exf {

namespace {

__device__ __forceinline__ void unpack8(const int4& v, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 p = __bfloat1622float2(h[i]);
        f[2 * i] = p.x;
        f[2 * i + 1] = p.y;
    }
}

// 8 consecutive elements as fp32 (bf16 rows: one 16-byte load; fp32 rows: two)
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&f)[8]) {
    unpack8(*reinterpret_cast<const int4*>(p), f);
}
__device__ __forceinline__ void load8(const float* p, float (&f)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w;
    f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Sense-reversal grid barrier over all CTAs of the launch (they are all
// co-resident: the grid is capped well below one CTA per SM).
__device__ void grid_barrier(uint32_t* gbar, uint32_t nctas, int32_t* err) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t gen = ld_acquire_gpu_u32(gbar + 1);
        __threadfence();
        const uint32_t prev = atomicAdd(gbar, 1u);
        if (prev == nctas - 1) {
            gbar[0] = 0;
            __threadfence();
            atomicAdd(gbar + 1, 1u);
        } else {
            ptx::SpinGuard g;
            while (ld_acquire_gpu_u32(gbar + 1) == gen) g.step(err, ERR_TIMEOUT_PIPE);
        }
        __threadfence();
    }
    __syncthreads();
}

}  // namespace

constexpr int kGdThreads = 512;
constexpr int kGdWarps = kGdThreads / 32;
constexpr int kMaxKeys = 64;

// T: element type of the token rows and the gate (bf16, or fp32 in the fp32
// mode); the gate reduction order is the same for both (fixed-order fmaf)
template <int EMAX, typename T>
__global__ void __launch_bounds__(kGdThreads) gate_dispatch_kernel(LayerArgs a, int wg_in_smem) {
    // dynamic smem: X [tpc][d] T | meta [tpc] ResMeta | Wg [E][d] T (when it fits)
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int32_t s_exp[256];
    __shared__ float s_prob[256];
    __shared__ int32_t s_pos[256];
    __shared__ int32_t s_cnt[kMaxKeys];   // this CTA's per-key counts (running)
    __shared__ int32_t s_tot[kMaxKeys];   // all CTAs
    __shared__ int32_t s_before[kMaxKeys];
    __shared__ int32_t s_start[kMaxKeys + 1];
    __shared__ int32_t s_last;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) tl_mark(a.tl, 0);
    ptx::pdl_wait();
    ptx::pdl_trigger();  // GEMM1 may start its prologue + weight prefetch now
    if (tid == 0) tl_mark(a.tl, 1);

    const int n = *a.n_res_in;
    const uint64_t q = *a.step * (uint64_t)a.L + (uint64_t)a.layer;
    const int parity = (int)(q & 1);
    const uint64_t epoch = q + 1;
    const int t0 = blockIdx.x * a.tpc;
    const int nt = max(0, min(a.tpc, n - t0));
    const int E = a.E;
    if (n > a.C) {
        if (tid == 0) atomicExch(a.err, ERR_CAPACITY);
        return;  // uniform: every CTA reads the same n
    }
    // only CTAs that own tokens take part (CTA 0 always: it publishes counts
    // and flags even when no token is resident)
    const uint32_t nactive = (uint32_t)max(1, (n + a.tpc - 1) / a.tpc);
    if (blockIdx.x >= nactive) return;

    // ---- stage this CTA's token rows, their metadata and Wg in shared memory
    //      with one batch of independent 16-byte loads
    const int vec = a.d * (int)sizeof(T) / 16;  // int4 per row
    T* sx = reinterpret_cast<T*>(smem);
    ResMeta* smeta = reinterpret_cast<ResMeta*>(smem + (size_t)a.tpc * a.d * sizeof(T));
    const T* wg = static_cast<const T*>(a.wg);
    {
        const int4* xs = reinterpret_cast<const int4*>(static_cast<const T*>(a.res_x_in) + (int64_t)t0 * a.d);
        int4* xd = reinterpret_cast<int4*>(sx);
        for (int i = tid; i < nt * vec; i += kGdThreads) xd[i] = xs[i];
        for (int i = tid; i < nt; i += kGdThreads) smeta[i] = a.res_meta_in[t0 + i];
        if (wg_in_smem && nt > 0) {
            T* swg = reinterpret_cast<T*>(smem + (size_t)a.tpc * (a.d * sizeof(T) + 8));
            const int4* src = reinterpret_cast<const int4*>(a.wg);
            int4* dst = reinterpret_cast<int4*>(swg);
            for (int i = tid; i < E * vec; i += kGdThreads) dst[i] = __ldg(src + i);
            wg = swg;
        }
    }
    if (tid < kMaxKeys) s_cnt[tid] = 0;
    __syncthreads();
    if (tid == 0) tl_mark(a.tl, 4);

    // ---- (1) gate, one warp per token
    const int chunks = a.d >> 8;
    for (int i = warp; i < nt; i += kGdWarps) {
        const int t = t0 + i;
        const T* x = sx + (int64_t)i * a.d;
        float acc[EMAX];
#pragma unroll
        for (int e = 0; e < EMAX; ++e) acc[e] = 0.f;
        for (int c = 0; c < chunks; ++c) {
            float xf[8];
            load8(x + c * 256 + lane * 8, xf);
#pragma unroll
            for (int e = 0; e < EMAX; ++e) {
                if (e < E) {
                    float wf[8];
                    load8(wg + (int64_t)e * a.d + c * 256 + lane * 8, wf);
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc[e] = fmaf(xf[k], wf[k], acc[e]);
                }
            }
        }
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], off);
        }
        if (lane == 0) {
            int best = 0;
            float mx = acc[0];
#pragma unroll
            for (int e = 1; e < EMAX; ++e)
                if (e < E && acc[e] > mx) {
                    mx = acc[e];
                    best = e;
                }
            float s = 0.f;
#pragma unroll
            for (int e = 0; e < EMAX; ++e)
                if (e < E) s += expf(acc[e] - mx);
            const ResMeta m = smeta[i];
            int sel = best;
            float p = 1.f / s;
            if (a.forced) {
                sel = a.forced_routes[(int64_t)m.token * a.L + a.layer];
                if ((unsigned)sel >= (unsigned)E) {
                    atomicExch(a.err, ERR_BAD_EXPERT);
                    sel = best;
                }
                float ls = acc[0];
#pragma unroll
                for (int e = 0; e < EMAX; ++e)
                    if (e == sel) ls = acc[e];
                p = expf(ls - mx) / s;
            }
            s_exp[i] = sel;
            s_prob[i] = p;
            a.expert[t] = sel;
            a.prob[t] = p;
            if (a.hist && a.layer > 0 && m.prev_expert >= 0)
                atomicAdd(&a.hist[((int64_t)(a.layer - 1) * E + m.prev_expert) * E + sel], 1ull);
            if (a.trace) a.trace[(int64_t)m.token * a.L + a.layer] = sel;
        }
    }
    __syncthreads();
    if (tid == 0) tl_mark(a.tl, 5);

    // ---- (2a) stable ranks inside this CTA's slice (warp 0, 32 tokens at a
    //      time, atomic-free) and per-key counts
    if (warp == 0) {
        for (int b = 0; b < nt; b += 32) {
            const int i = b + lane;
            int key = -1;
            if (i < nt) {
                const int e = s_exp[i];
                key = a.gpu_of[e] * a.E_loc + a.slot_of[e];
            }
            const uint32_t peers = __match_any_sync(0xffffffffu, key);
            const int rank = __popc(peers & lanemask_lt());
            if (key >= 0) s_pos[i] = (s_cnt[key] + rank) | (key << 20);  // in-CTA rank | key
            __syncwarp();
            if (key >= 0 && rank == 0) s_cnt[key] += __popc(peers);
            __syncwarp();
        }
        for (int k = lane; k < E; k += 32) a.cta_cnt[blockIdx.x * E + k] = s_cnt[k];
    }
    // ---- (2b) publish counts, barrier over the active CTAs, key offsets
    if (nactive > 1) grid_barrier(a.gbar, nactive, a.err);
    else __syncthreads();
    if (tid == 0) tl_mark(a.tl, 6);
    if (tid < E) {
        int tot = 0, before = 0;
        for (int c = 0; c < (int)nactive; ++c) {
            const int v = a.cta_cnt[c * E + tid];
            tot += v;
            before += (c < (int)blockIdx.x) ? v : 0;
        }
        s_tot[tid] = tot;
        s_before[tid] = before;
    }
    __syncthreads();
    if (tid == 0) {
        int acc = 0;
        for (int k = 0; k < E; ++k) {
            s_start[k] = acc;
            acc += s_tot[k];
        }
        s_start[E] = acc;
    }
    __syncthreads();

    // ---- (3) rows straight from shared memory into the destination's
    //      receive region (P2P stores for remote destinations)
    const int64_t row_bytes = (int64_t)a.d * sizeof(T);
    for (int i = warp; i < nt; i += kGdWarps) {
        const int key = s_pos[i] >> 20;
        const int dest = key / a.E_loc;
        const int pos = s_start[key] + s_before[key] + (s_pos[i] & 0xFFFFF);
        const int local = pos - s_start[dest * a.E_loc];
        uint8_t* pbase = a.peers[dest];
        const int64_t slot_row = ((int64_t)(parity * a.G + a.rank) * a.C + local);
        int4* dst = reinterpret_cast<int4*>(pbase + a.sym.recv_x + slot_row * row_bytes);
        const int4* src = reinterpret_cast<const int4*>(sx + (int64_t)i * a.d);
        for (int v = lane; v < vec; v += 32) dst[v] = src[v];
        if (lane == 0) {
            RecvMeta m;
            m.token = smeta[i].token;
            m.expert = s_exp[i];
            m.prob = s_prob[i];
            m.pad = 0;
            reinterpret_cast<RecvMeta*>(pbase + a.sym.recv_meta)[slot_row] = m;
        }
    }
    __syncthreads();
    if (tid == 0) tl_mark(a.tl, 7);
    // completion: one fence per CTA (cumulative over the CTA's stores through
    // the barrier above) before the done-counter; the last CTA publishes
    if (tid == 0) {
        if (nactive == 1) {
            s_last = 1;
        } else {
            if (a.G > 1) __threadfence_system(); else __threadfence();
            s_last = atomicAdd(a.done_ctr, 1) == (int)nactive - 1;
            if (s_last) __threadfence();
        }
    }
    __syncthreads();
    if (tid == 0) tl_mark(a.tl, 3);
    if (!s_last) return;
    // ---- last CTA: per-(src = me, slot) counts, stats, release flags
    if (tid < E) {
        const int dest = tid / a.E_loc, slot = tid - dest * a.E_loc;
        int32_t* cnt = reinterpret_cast<int32_t*>(a.peers[dest] + a.sym.recv_cnt);
        cnt[((int64_t)parity * a.G + a.rank) * a.E_loc + slot] = s_tot[tid];
    }
    if (tid == 0) {
        int stay = 0;
        for (int s = 0; s < a.E_loc; ++s) stay += s_tot[a.rank * a.E_loc + s];
        atomicAdd(&a.crossed[a.layer], (unsigned long long)(n - stay));
    }
    __syncthreads();  // counts and rows precede the release stores below
    if (tid < a.G) {
        uint64_t* f = reinterpret_cast<uint64_t*>(a.peers[tid] + a.sym.flags);
        ptx::flag_publish(f + parity * a.G + a.rank, epoch, a.G > 1);  // .gpu scope on one GPU
    }
    if (tid == 0 && nactive > 1) *a.done_ctr = 0;
    if (tid == 0) tl_mark(a.tl, 3);
}

// ------------------------------------------------------------------ step begin
// Home tokens of this rank: global ids rank + G*i (round-robin homes, t % G;
// proj/src/sim.cpp:111).
// (rows are copied as 16-byte vectors: vec = row bytes / 16, bf16 or fp32)
__global__ void step_begin_kernel(const void* __restrict__ x_in, void* res_x,
                                  ResMeta* res_meta, int32_t* n_res, int B, int vec, int G,
                                  int rank) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)B * vec;
         i += (int64_t)gridDim.x * blockDim.x)
        reinterpret_cast<int4*>(res_x)[i] = reinterpret_cast<const int4*>(x_in)[i];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B; i += gridDim.x * blockDim.x) {
        res_meta[i].token = rank + G * i;
        res_meta[i].prev_expert = -1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_res = B;
}

// ------------------------------------------------------------------ context AllGather
__global__ void __launch_bounds__(512) gather_send_kernel(
    const void* __restrict__ res_x, const ResMeta* __restrict__ res_meta,
    const int32_t* n_res, uint8_t* const* peers, Symm sym, int G, int rank, int vec, int C,
    const uint64_t* step, int32_t* done_ctr, int32_t* err) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    const int n = *n_res;
    for (int64_t w = (int64_t)blockIdx.x * nwarp + warp; w < (int64_t)n * G;
         w += (int64_t)gridDim.x * nwarp) {
        const int r = (int)(w / G), p = (int)(w - (int64_t)r * G);
        const int tok = res_meta[r].token;
        if ((unsigned)tok >= (unsigned)C) {
            if (lane == 0) atomicExch(err, ERR_CAPACITY);
            continue;
        }
        int4* dst = reinterpret_cast<int4*>(peers[p] + sym.gather_x) + (int64_t)tok * vec;
        const int4* src = reinterpret_cast<const int4*>(res_x) + (int64_t)r * vec;
        for (int v = lane; v < vec; v += 32) dst[v] = src[v];
    }
    if (G > 1) __threadfence_system(); else __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int prev = atomicAdd(done_ctr, 1);
        if (prev == (int)gridDim.x - 1) {
            if (G > 1) __threadfence_system(); else __threadfence();
            const uint64_t epoch = *step + 1;
            for (int p = 0; p < G; ++p)  // .gpu scope on one GPU (a .sys release costs ~4 us)
                ptx::flag_publish(reinterpret_cast<uint64_t*>(peers[p] + sym.gflags) + rank, epoch, G > 1);
            *done_ctr = 0;
        }
    }
}

__global__ void gather_wait_kernel(uint8_t* own_sym, Symm sym, int G, uint64_t* step,
                                   int32_t* err) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const uint64_t epoch = *step + 1;
    if ((int)threadIdx.x < G) {
        const uint64_t* f = reinterpret_cast<const uint64_t*>(own_sym + sym.gflags) + threadIdx.x;
        ptx::SpinGuard g;
        while (ptx::flag_read(f, G > 1) < epoch) g.step(err, ERR_TIMEOUT_GATHER);
    }
    __syncthreads();
    if (threadIdx.x == 0) *step = epoch;
}

// ------------------------------------------------------------------ vanilla-EP combine
// Vanilla expert parallelism (the DeepSpeed-MoE-style baseline ExFlow is
// compared against): after every layer each token's output row goes back to
// its home rank (proj/src/sim.cpp:60-64: 2 hops per crossed token, dispatch +
// combine; collective counts :153-157). Row of token t lands in slot t / G of
// home rank t % G's combine buffer (double-buffered by layer parity), followed
// by a per-slot release flag {epoch = step * L + layer + 1}: the home rank
// needs no counts, it waits for its B slots.
__global__ void __launch_bounds__(256) combine_send_kernel(
    const void* __restrict__ res_x, const ResMeta* __restrict__ res_meta, const int32_t* n_res,
    uint8_t* const* peers, Symm sym, int G, int B, int vec, int L, int layer, const uint64_t* step,
    int32_t* err) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    const int n = *n_res;
    const uint64_t epoch = *step * (uint64_t)L + (uint64_t)layer + 1;
    const int par = layer & 1;
    for (int r = blockIdx.x * nwarp + warp; r < n; r += gridDim.x * nwarp) {
        const ResMeta m = res_meta[r];
        if ((unsigned)m.token >= (unsigned)(B * G)) {
            if (lane == 0) atomicExch(err, ERR_CAPACITY);
            continue;
        }
        const int home = m.token % G, slot = m.token / G;
        uint8_t* base = peers[home];
        int4* dst = reinterpret_cast<int4*>(base + sym.comb_x) + ((int64_t)par * B + slot) * vec;
        const int4* src = reinterpret_cast<const int4*>(res_x) + (int64_t)r * vec;
        for (int v = lane; v < vec; v += 32) dst[v] = src[v];
        if (lane == 0) reinterpret_cast<ResMeta*>(base + sym.comb_meta)[par * B + slot] = m;
        __syncwarp();  // the warp's row stores precede lane 0's release
        if (lane == 0) {
            uint64_t* f = reinterpret_cast<uint64_t*>(base + sym.comb_flags) + par * B + slot;
            if (G > 1) ptx::st_release_sys(f, epoch); else ptx::st_release_gpu_u64(f, epoch);
        }
    }
}

// Home side: wait for the B slots, then copy them (home order) into the
// resident buffers the next layer reads.
__global__ void __launch_bounds__(256) combine_wait_kernel(
    const uint8_t* own_sym, Symm sym, int G, int B, int vec, int L, int layer, const uint64_t* step,
    void* res_x_next, ResMeta* res_meta_next, int32_t* n_res_next, int32_t* err) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    const uint64_t epoch = *step * (uint64_t)L + (uint64_t)layer + 1;
    const int par = layer & 1;
    for (int slot = blockIdx.x * nwarp + warp; slot < B; slot += gridDim.x * nwarp) {
        const uint64_t* f = reinterpret_cast<const uint64_t*>(own_sym + sym.comb_flags) + par * B + slot;
        if (lane == 0) {
            ptx::SpinGuard g;
            while (ptx::ld_relaxed_u64(f, G > 1) < epoch) g.step(err, ERR_TIMEOUT_GATHER);
            (void)ptx::flag_read(f, G > 1);  // acquire on the flag itself
        }
        __syncwarp();
        const int4* src = reinterpret_cast<const int4*>(own_sym + sym.comb_x) + ((int64_t)par * B + slot) * vec;
        int4* dst = reinterpret_cast<int4*>(res_x_next) + (int64_t)slot * vec;
        for (int v = lane; v < vec; v += 32) dst[v] = src[v];
        if (lane == 0) res_meta_next[slot] = reinterpret_cast<const ResMeta*>(own_sym + sym.comb_meta)[par * B + slot];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_res_next = B;
}

// ------------------------------------------------------------------ launchers
// Tokens per CTA of gate_dispatch: the CTA stages its token rows (and, when
// they fit, Wg) in shared memory; at most 128 CTAs so that all active CTAs
// are co-resident for the grid barrier (model creation enforces C <= 128*tpc).
constexpr size_t kGdSmemBudget = 200 * 1024;
// one token per warp (16) so the gate spreads over ceil(n/16) SMs; larger
// capacities grow the slice so the grid stays <= 128 CTAs
int gate_dispatch_tpc(int C) {
    int tpc = (C + 127) / 128;
    tpc = ((tpc + 15) / 16) * 16;
    return std::max(16, std::min(tpc, 256));
}

template <typename T>
exf_status launch_gate_dispatch_t(const LayerArgs& a, cudaStream_t s) {
    if (a.E > kMaxKeys) return invalid("at most 64 experts");
    if (a.tpc < 16 || a.tpc > 256) return invalid("bad gate_dispatch tile");
    const int grid = (a.C + a.tpc - 1) / a.tpc;
    if (grid > 128) return invalid("G*B exceeds the gate_dispatch capacity (128 CTAs)");
    const size_t x_bytes = (size_t)a.tpc * (sizeof(T) * a.d + 8);
    if (x_bytes > kGdSmemBudget) return invalid("gate_dispatch token slice does not fit in shared memory");
    const size_t wg_bytes = (size_t)a.E * a.d * sizeof(T);
    const int in_smem = x_bytes + wg_bytes <= kGdSmemBudget ? 1 : 0;
    const size_t smem = x_bytes + (in_smem ? wg_bytes : 0);
    void (*k)(LayerArgs, int) = a.E <= 8    ? gate_dispatch_kernel<8, T>
                                : a.E <= 16 ? gate_dispatch_kernel<16, T>
                                : a.E <= 32 ? gate_dispatch_kernel<32, T>
                                            : gate_dispatch_kernel<64, T>;
    static bool attr = false;
    if (!attr) {
        for (auto kk : {gate_dispatch_kernel<8, T>, gate_dispatch_kernel<16, T>, gate_dispatch_kernel<32, T>,
                        gate_dispatch_kernel<64, T>}) {
            EXF_CUDA_TRY(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)kGdSmemBudget));
            max_carveout(kk);
        }
        max_carveout(step_begin_kernel);
        max_carveout(gather_send_kernel);
        max_carveout(gather_wait_kernel);
        attr = true;
    }
    EXF_CUDA_TRY(launch_pdl(k, dim3(grid), dim3(kGdThreads), smem, s, 0, a, in_smem));
    return EXF_OK;
}

exf_status launch_gate_dispatch(const LayerArgs& a, cudaStream_t s) {
    return a.esz == 4 ? launch_gate_dispatch_t<float>(a, s) : launch_gate_dispatch_t<__nv_bfloat16>(a, s);
}

exf_status launch_step_begin(const void* x_in, void* res_x, ResMeta* res_meta,
                             int32_t* n_res, int B, int vec, int G, int rank, cudaStream_t s) {
    const int blocks = std::max(1, std::min(148, (int)(((int64_t)B * vec + 255) / 256)));
    EXF_CUDA_TRY(launch_pdl(step_begin_kernel, dim3(blocks), dim3(256), 0, s, 0, x_in, res_x,
                            res_meta, n_res, B, vec, G, rank));
    return EXF_OK;
}

exf_status launch_gather_send(const void* res_x, const ResMeta* res_meta,
                              const int32_t* n_res, uint8_t* const* peers, const Symm& sym, int G,
                              int rank, int vec, int C, const uint64_t* step, int32_t* done_ctr,
                              int32_t* err, cudaStream_t s) {
    const int blocks = std::max(1, std::min(132, (C * G + 15) / 16));
    EXF_CUDA_TRY(launch_pdl(gather_send_kernel, dim3(blocks), dim3(512), 0, s, 0, res_x, res_meta,
                            n_res, peers, sym, G, rank, vec, C, step, done_ctr, err));
    return EXF_OK;
}

exf_status launch_combine(const void* res_x_out, const ResMeta* res_meta_out, const int32_t* n_res_out,
                          uint8_t* const* peers, uint8_t* own_sym, const Symm& sym, int G, int B, int vec, int L,
                          int layer, const uint64_t* step, void* res_x_next, ResMeta* res_meta_next,
                          int32_t* n_res_next, int32_t* err, int part, cudaStream_t s) {
    const int blocks = std::max(1, std::min(148, (B * G + 7) / 8));
    if (part == 0) {
        EXF_CUDA_TRY(launch_pdl(combine_send_kernel, dim3(blocks), dim3(256), 0, s, 0, res_x_out, res_meta_out,
                                n_res_out, peers, sym, G, B, vec, L, layer, step, err));
        return EXF_OK;
    }
    EXF_CUDA_TRY(launch_pdl(combine_wait_kernel, dim3(std::max(1, std::min(148, (B + 7) / 8))), dim3(256), 0, s, 0,
                            (const uint8_t*)own_sym, sym, G, B, vec, L, layer, step, res_x_next, res_meta_next,
                            n_res_next, err));
    return EXF_OK;
}

exf_status launch_gather_wait(uint8_t* own_sym, const Symm& sym, int G, uint64_t* step,
                              int32_t* err, cudaStream_t s) {
    EXF_CUDA_TRY(launch_pdl(gather_wait_kernel, dim3(1), dim3(32 * ((G + 31) / 32)), 0, s, 0,
                            own_sym, sym, G, step, err));
    return EXF_OK;
}

}  // namespace exf
