// gate_dispatch.cu -- per-layer token-side kernels of the ExFlow decode step.
//
//  (1) gate_kernel: fused gate GEMM + softmax/top-1 + affinity histogram
//      (kernel 5, fused form) + routing-trace emission. One warp per token;
//      the logits use the fixed fp32 reduction order documented in
//      oracle/exflow_model_oracle.c (32 lane partials accumulated c-major /
//      i-minor with FMA, then a xor-butterfly), so routing is bit-identical
//      to the CPU oracle. Top-1 ties -> lowest expert index.
//  (2)+(3) dispatch_kernel: deterministic, atomic-free bucketing of the
//      resident tokens by (destination GPU, local expert slot) with a
//      warp-aggregated prefix scan (__match_any_sync + popc(lanemask_lt),
//      then a per-key scan over warps), fused with ExFlow's single dispatch
//      "Alltoall": rows are stored straight into the destination rank's
//      symmetric receive region over NVLink (P2P stores through CUDA-IPC
//      mapped pointers), followed by a system-scope release flag. Tokens stay
//      on their expert's GPU afterwards (coherent mode, no combine step;
//      proj/src/sim.cpp:65-71).
//  (3b) gather_send/gather_wait: the per-step context AllGather; every rank
//      scatters its resident tokens' hidden states into every peer's
//      token-id-indexed output buffer, then waits for all peers' flags.
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

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace

// ------------------------------------------------------------------ gate
template <int EMAX>
__global__ void __launch_bounds__(256) gate_kernel(LayerArgs a) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int n = *a.n_res_in;
    const int chunks = a.d >> 8;
    for (int t = gw; t < n; t += nw) {
        const __nv_bfloat16* x = a.res_x_in + (int64_t)t * a.d;
        float acc[EMAX];
#pragma unroll
        for (int e = 0; e < EMAX; ++e) acc[e] = 0.f;
        for (int c = 0; c < chunks; ++c) {
            float xf[8];
            unpack8(*reinterpret_cast<const int4*>(x + c * 256 + lane * 8), xf);
#pragma unroll
            for (int e = 0; e < EMAX; ++e) {
                if (e < a.E) {
                    float wf[8];
                    unpack8(__ldg(reinterpret_cast<const int4*>(a.wg + (int64_t)e * a.d + c * 256 +
                                                                 lane * 8)),
                            wf);
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[e] = fmaf(xf[i], wf[i], acc[e]);
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
                if (e < a.E && acc[e] > mx) {
                    mx = acc[e];
                    best = e;
                }
            float s = 0.f;
#pragma unroll
            for (int e = 0; e < EMAX; ++e)
                if (e < a.E) s += expf(acc[e] - mx);
            const ResMeta m = a.res_meta_in[t];
            int sel = best;
            float p = 1.f / s;
            if (a.forced) {
                sel = a.forced_routes[(int64_t)m.token * a.L + a.layer];
                if ((unsigned)sel >= (unsigned)a.E) {
                    atomicExch(a.err, ERR_BAD_EXPERT);
                    sel = best;
                }
                float ls = acc[0];
#pragma unroll
                for (int e = 0; e < EMAX; ++e)
                    if (e == sel) ls = acc[e];
                p = expf(ls - mx) / s;
            }
            a.expert[t] = sel;
            a.prob[t] = p;
            if (a.hist && a.layer > 0 && m.prev_expert >= 0)
                atomicAdd(&a.hist[((int64_t)(a.layer - 1) * a.E + m.prev_expert) * a.E + sel], 1ull);
            if (a.trace) a.trace[(int64_t)m.token * a.L + a.layer] = sel;
        }
    }
}

// ------------------------------------------------------------------ dispatch
// Dynamic smem: key[C] (int16 packed in int32), pos[C], warp counts, per-key
// running totals. Every CTA runs the (cheap) scan redundantly, then copies its
// share of rows; the last CTA to finish releases the per-destination flags.
constexpr int kDispThreads = 512;
constexpr int kDispWarps = kDispThreads / 32;
constexpr int kMaxKeys = 64;

__global__ void __launch_bounds__(kDispThreads) dispatch_kernel(LayerArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    int32_t* s_pos = reinterpret_cast<int32_t*>(smem);        // [C]
    int32_t* s_key = s_pos + a.C;                              // [C]
    __shared__ int32_t s_wcnt[kDispWarps][kMaxKeys];
    __shared__ int32_t s_run[kMaxKeys];
    __shared__ int32_t s_start[kMaxKeys + 1];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = *a.n_res_in;
    const int K = a.E;  // keys = G * E_loc = E
    const uint64_t step = *a.step;
    const int64_t q = (int64_t)step * a.L + a.layer;
    const int parity = (int)(q & 1);
    const uint64_t epoch = (uint64_t)q + 1;
    if (n > a.C) {
        if (tid == 0) atomicExch(a.err, ERR_CAPACITY);
        return;
    }

    if (tid < kMaxKeys) s_run[tid] = 0;
    // pass 1: keys and per-key totals (warp-aggregated, atomic-free)
    for (int base = 0; base < n; base += kDispThreads) {
        const int t = base + tid;
        int key = -1;
        if (t < n) {
            const int e = a.expert[t];
            key = a.gpu_of[e] * a.E_loc + a.slot_of[e];
            s_key[t] = key;
        }
        for (int k = lane; k < kMaxKeys; k += 32) s_wcnt[warp][k] = 0;
        __syncwarp();
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        if (key >= 0 && (peers & lanemask_lt()) == 0) s_wcnt[warp][key] = __popc(peers);
        __syncthreads();
        if (tid < K) {
            int s = 0;
            for (int w = 0; w < kDispWarps; ++w) s += s_wcnt[w][tid];
            s_run[tid] += s;
        }
        __syncthreads();
    }
    if (tid == 0) {
        int acc = 0;
        for (int k = 0; k < K; ++k) {
            s_start[k] = acc;
            acc += s_run[k];
        }
        s_start[K] = acc;
    }
    __syncthreads();
    // keep the per-key totals, reuse s_run as the running write cursor
    int my_total = 0;
    if (tid < K) {
        my_total = s_run[tid];
        s_run[tid] = s_start[tid];
    }
    __syncthreads();
    // pass 2: stable positions = start[key] + tokens of this key in earlier
    // chunks + earlier warps of this chunk + rank within the warp
    for (int base = 0; base < n; base += kDispThreads) {
        const int t = base + tid;
        const int key = t < n ? s_key[t] : -1;
        for (int k = lane; k < kMaxKeys; k += 32) s_wcnt[warp][k] = 0;
        __syncwarp();
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        const int rank = __popc(peers & lanemask_lt());
        if (key >= 0 && rank == 0) s_wcnt[warp][key] = __popc(peers);
        __syncthreads();
        if (tid < K) {  // exclusive prefix over warps for key `tid`
            int run = s_run[tid];
            for (int w = 0; w < kDispWarps; ++w) {
                const int c = s_wcnt[w][tid];
                s_wcnt[w][tid] = run;
                run += c;
            }
            s_run[tid] = run;
        }
        __syncthreads();
        if (key >= 0) s_pos[t] = s_wcnt[warp][key] + rank;
        __syncthreads();
    }

    // copy rows: warp-granular, tokens strided over the whole grid
    const int64_t row_bytes = (int64_t)a.d * 2;
    const int vec_per_row = a.d >> 3;  // int4 per row
    for (int t = blockIdx.x * kDispWarps + warp; t < n; t += gridDim.x * kDispWarps) {
        const int key = s_key[t];
        const int dest = key / a.E_loc;
        const int local = s_pos[t] - s_start[dest * a.E_loc];
        uint8_t* pbase = a.peers[dest];
        const int64_t slot_row = ((int64_t)(parity * a.G + a.rank) * a.C + local);
        int4* dst = reinterpret_cast<int4*>(pbase + a.sym.recv_x + slot_row * row_bytes);
        const int4* src = reinterpret_cast<const int4*>(a.res_x_in + (int64_t)t * a.d);
        for (int v = lane; v < vec_per_row; v += 32) dst[v] = src[v];
        if (lane == 0) {
            RecvMeta m;
            m.token = a.res_meta_in[t].token;
            m.expert = a.expert[t];
            m.prob = a.prob[t];
            m.pad = 0;
            reinterpret_cast<RecvMeta*>(pbase + a.sym.recv_meta)[slot_row] = m;
        }
    }
    // per-(src = me, slot) counts into every destination
    if (blockIdx.x == 0 && tid < K) {
        const int dest = tid / a.E_loc, slot = tid - dest * a.E_loc;
        int32_t* cnt = reinterpret_cast<int32_t*>(a.peers[dest] + a.sym.recv_cnt);
        cnt[((int64_t)parity * a.G + a.rank) * a.E_loc + slot] = my_total;
    }
    if (blockIdx.x == 0 && tid == 0) {
        int stay = 0;
        for (int s = 0; s < a.E_loc; ++s) stay += s_run[a.rank * a.E_loc + s] - s_start[a.rank * a.E_loc + s];
        atomicAdd(&a.crossed[a.layer], (unsigned long long)(n - stay));
    }
    __threadfence_system();
    __syncthreads();
    if (tid == 0) {
        const int prev = atomicAdd(a.done_ctr, 1);
        if (prev == (int)gridDim.x - 1) {
            __threadfence_system();
            for (int p = 0; p < a.G; ++p) {
                uint64_t* f = reinterpret_cast<uint64_t*>(a.peers[p] + a.sym.flags);
                ptx::st_release_sys(f + parity * a.G + a.rank, epoch);
            }
            *a.done_ctr = 0;
        }
    }
}

// ------------------------------------------------------------------ step begin
// Home tokens of this rank: global ids rank + G*i (round-robin homes, t % G;
// proj/src/sim.cpp:111).
__global__ void step_begin_kernel(const __nv_bfloat16* __restrict__ x_in, __nv_bfloat16* res_x,
                                  ResMeta* res_meta, int32_t* n_res, int B, int d, int G,
                                  int rank) {
    const int vec = d >> 3;
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
    const __nv_bfloat16* __restrict__ res_x, const ResMeta* __restrict__ res_meta,
    const int32_t* n_res, uint8_t* const* peers, Symm sym, int G, int rank, int d, int C,
    const uint64_t* step, int32_t* done_ctr, int32_t* err) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    const int n = *n_res;
    const int vec = d >> 3;
    for (int64_t w = (int64_t)blockIdx.x * nwarp + warp; w < (int64_t)n * G;
         w += (int64_t)gridDim.x * nwarp) {
        const int r = (int)(w / G), p = (int)(w - (int64_t)r * G);
        const int tok = res_meta[r].token;
        if ((unsigned)tok >= (unsigned)C) {
            if (lane == 0) atomicExch(err, ERR_CAPACITY);
            continue;
        }
        int4* dst = reinterpret_cast<int4*>(peers[p] + sym.gather_x + (int64_t)tok * d * 2);
        const int4* src = reinterpret_cast<const int4*>(res_x + (int64_t)r * d);
        for (int v = lane; v < vec; v += 32) dst[v] = src[v];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int prev = atomicAdd(done_ctr, 1);
        if (prev == (int)gridDim.x - 1) {
            __threadfence_system();
            const uint64_t epoch = *step + 1;
            for (int p = 0; p < G; ++p)
                ptx::st_release_sys(reinterpret_cast<uint64_t*>(peers[p] + sym.gflags) + rank, epoch);
            *done_ctr = 0;
        }
    }
}

__global__ void gather_wait_kernel(uint8_t* own_sym, Symm sym, int G, uint64_t* step,
                                   int32_t* err) {
    const uint64_t epoch = *step + 1;
    if ((int)threadIdx.x < G) {
        const uint64_t* f = reinterpret_cast<const uint64_t*>(own_sym + sym.gflags) + threadIdx.x;
        ptx::SpinGuard g;
        while (ptx::ld_acquire_sys(f) < epoch) g.step(err, ERR_TIMEOUT_GATHER);
    }
    __syncthreads();
    if (threadIdx.x == 0) *step = epoch;
}

// ------------------------------------------------------------------ launchers
exf_status launch_gate(const LayerArgs& a, cudaStream_t s) {
    const int blocks = (int)std::min<int64_t>(4 * 148, ((int64_t)a.C + 7) / 8);
    const int bl = blocks < 1 ? 1 : blocks;
    if (a.E <= 8) gate_kernel<8><<<bl, 256, 0, s>>>(a);
    else if (a.E <= 16) gate_kernel<16><<<bl, 256, 0, s>>>(a);
    else if (a.E <= 32) gate_kernel<32><<<bl, 256, 0, s>>>(a);
    else gate_kernel<64><<<bl, 256, 0, s>>>(a);
    EXF_LAUNCH_CHECK("gate_kernel");
    return EXF_OK;
}

int dispatch_grid(int C) {
    int g = (C + kDispWarps - 1) / kDispWarps;  // ~1 row per warp
    return g < 1 ? 1 : (g > 132 ? 132 : g);
}

exf_status launch_dispatch(const LayerArgs& a, cudaStream_t s) {
    const size_t smem = (size_t)a.C * 8;
    static bool attr_done = false;
    if (!attr_done) {
        EXF_CUDA_TRY(cudaFuncSetAttribute(dispatch_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        attr_done = true;
    }
    dispatch_kernel<<<dispatch_grid(a.C), kDispThreads, smem, s>>>(a);
    EXF_LAUNCH_CHECK("dispatch_kernel");
    return EXF_OK;
}

exf_status launch_step_begin(const __nv_bfloat16* x_in, __nv_bfloat16* res_x, ResMeta* res_meta,
                             int32_t* n_res, int B, int d, int G, int rank, cudaStream_t s) {
    const int blocks = std::max(1, std::min(148, (int)(((int64_t)B * (d >> 3) + 255) / 256)));
    step_begin_kernel<<<blocks, 256, 0, s>>>(x_in, res_x, res_meta, n_res, B, d, G, rank);
    EXF_LAUNCH_CHECK("step_begin_kernel");
    return EXF_OK;
}

exf_status launch_gather_send(const __nv_bfloat16* res_x, const ResMeta* res_meta,
                              const int32_t* n_res, uint8_t* const* peers, const Symm& sym, int G,
                              int rank, int d, int C, const uint64_t* step, int32_t* done_ctr,
                              int32_t* err, cudaStream_t s) {
    const int blocks = std::max(1, std::min(132, (C * G + 15) / 16));
    gather_send_kernel<<<blocks, 512, 0, s>>>(res_x, res_meta, n_res, peers, sym, G, rank, d, C,
                                              step, done_ctr, err);
    EXF_LAUNCH_CHECK("gather_send_kernel");
    return EXF_OK;
}

exf_status launch_gather_wait(uint8_t* own_sym, const Symm& sym, int G, uint64_t* step,
                              int32_t* err, cudaStream_t s) {
    gather_wait_kernel<<<1, 32 * ((G + 31) / 32), 0, s>>>(own_sym, sym, G, step, err);
    EXF_LAUNCH_CHECK("gather_wait_kernel");
    return EXF_OK;
}

}  // namespace exf
