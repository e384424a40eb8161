// attention.cu -- coherent decode attention over the replicated context cache
// (SURVEY.md §8(f) rank 1).
//
// ExFlow drops the combine Alltoall because every GPU holds the whole context
// (one AllGather per step, proj/src/sim.cpp:161-162; protocol PAPER.md:180-184):
// a token that the dispatch left on GPU X attends over ITS OWN sequence's K/V
// rows in X's replica. The kernel therefore takes a per-token sequence id
// (tokens arrive in dispatch order, not sequence order).
//
// Layouts (row-major, bf16):
//   q     [N][H][Dh]       one decode query per resident token
//   seq   [N] int32        sequence (context row) of each token
//   ctx   [S] int32        valid context length of each sequence (<= C)
//   k, v  [S][H][C][Dh]    head-major so one (sequence, head) is one contiguous
//                          C*Dh*2-byte stream
//   out   [N][H][Dh]
// HBM-bound (AI ~ 1 flop/B): every K/V byte is read once, 16 B per lane,
// a lane group of Dh/8 lanes per key, 4 keys in flight per group. Long
// contexts are split across CTAs (flash-decoding) so the grid covers the
// 148 SMs in one wave; the last CTA of each (token, head) to arrive merges
// the partial (m, l, acc) in split order (deterministic, no second launch).
#include "common.cuh"

#include <algorithm>

#include <cuda_bf16.h>
#include <math_constants.h>

#include <cstring>

namespace exf {
namespace {

constexpr int kThreads = 128;
constexpr int kUnroll = 4;

// workspace layout: [N*H] u32 split-arrival counters (fixed offset 0, zeroed
// per call), then the fp32 partials {m, l, acc[Dh]} per (token, head, split),
// 16-byte aligned
__host__ __device__ inline size_t ws_partials_off(int64_t N, int H) {
    return (((size_t)N * H + 3) / 4) * 4;  // in floats
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// grid (H, N, splits). Partial results go to ws (splits > 1) or straight to out.
template <int Dh>
__global__ void __launch_bounds__(kThreads) coherent_attn_kernel(
    const __nv_bfloat16* __restrict__ q, const int32_t* __restrict__ seq,
    const int32_t* __restrict__ ctx, const __nv_bfloat16* __restrict__ k,
    const __nv_bfloat16* __restrict__ v, int32_t H, int32_t C, int32_t chunk, float scale_log2,
    float* __restrict__ ws, __nv_bfloat16* __restrict__ out, int32_t seq_stride,
    const int32_t* __restrict__ n_dev, int32_t len_add) {
    constexpr int LPK = Dh / 8;                  // lanes per key
    constexpr int GROUPS = kThreads / LPK;       // keys in flight per CTA step
    const int h = blockIdx.x, n = blockIdx.y, split = blockIdx.z, splits = gridDim.z;
    // decode-step form: the grid covers the capacity, the resident count is
    // on the device (uniform per CTA: every split of token n leaves together)
    if (n_dev && n >= *n_dev) return;
    const int s = seq[(size_t)n * seq_stride];
    // len_add = 1: the step's own K/V row was stored at position ctx[s] by the
    // projection (folded append) and the length advances after this kernel
    const int len = min(ctx[s] + len_add, C);
    const int lane_in = threadIdx.x % LPK, grp = threadIdx.x / LPK;
    const int k_begin = split * chunk;
    const int k_end = min(len, k_begin + chunk);

    float qf[8];
    bf16x8_to_f32(reinterpret_cast<const uint4*>(q + ((size_t)n * H + h) * Dh)[lane_in], qf);
#pragma unroll
    for (int i = 0; i < 8; ++i) qf[i] *= scale_log2;

    const size_t base = ((size_t)s * H + h) * (size_t)C * Dh;
    const uint4* kp = reinterpret_cast<const uint4*>(k + base) + lane_in;
    const uint4* vp = reinterpret_cast<const uint4*>(v + base) + lane_in;

    float m = -CUDART_INF_F, l = 0.f, acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;

    // CTA-uniform trip count: the lane groups of a warp share the shuffles
    // below, so keys past k_end are masked rather than skipped
    for (int kb = k_begin; kb < k_end; kb += GROUPS * kUnroll) {
        const int key0 = kb + grp;
        uint4 kr[kUnroll], vr[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int key = key0 + u * GROUPS;
            kr[u] = make_uint4(0, 0, 0, 0);
            vr[u] = make_uint4(0, 0, 0, 0);
            if (key < k_end) {
                kr[u] = ld_stream(kp + (size_t)key * LPK);
                vr[u] = ld_stream(vp + (size_t)key * LPK);
            }
        }
        float sc[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            float kf[8];
            bf16x8_to_f32(kr[u], kf);
            float d = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) d = fmaf(qf[i], kf[i], d);
#pragma unroll
            for (int o = LPK / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            sc[u] = (key0 + u * GROUPS < k_end) ? d : -CUDART_INF_F;
        }
        float mx = m;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) mx = fmaxf(mx, sc[u]);
        // no valid key for this group yet (mx = -inf): keep the state as is
        const float corr = (mx == -CUDART_INF_F) ? 1.f : exp2f(m - mx);  // m = -inf -> 0
        l *= corr;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] *= corr;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (key0 + u * GROUPS < k_end) {
                const float p = exp2f(sc[u] - mx);
                l += p;
                float vf[8];
                bf16x8_to_f32(vr[u], vf);
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] = fmaf(p, vf[i], acc[i]);
            }
        }
        m = mx;
    }

    // merge the GROUPS lane groups of this CTA (fixed order -> deterministic)
    __shared__ float s_m[GROUPS], s_l[GROUPS];
    __shared__ float s_acc[GROUPS][Dh];
    if (lane_in == 0) {
        s_m[grp] = m;
        s_l[grp] = l;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s_acc[grp][lane_in * 8 + i] = acc[i];
    __syncthreads();
    if (threadIdx.x < Dh) {
        const int c = threadIdx.x;
        float M = -CUDART_INF_F;
        for (int g = 0; g < GROUPS; ++g) M = fmaxf(M, s_m[g]);
        float L = 0.f, A = 0.f;
        if (M != -CUDART_INF_F) {
            for (int g = 0; g < GROUPS; ++g) {
                const float w = exp2f(s_m[g] - M);
                L += s_l[g] * w;
                A += s_acc[g][c] * w;
            }
        }
        const size_t nh = (size_t)n * H + h;
        if (splits == 1) {
            out[nh * Dh + c] = __float2bfloat16(L > 0.f ? A / L : 0.f);
        } else {
            float* p = ws + ws_partials_off(gridDim.y, H) + (nh * splits + split) * (Dh + 2);
            p[2 + c] = A;
            if (c == 0) {
                p[0] = M;
                p[1] = L;
            }
        }
    }
    if (splits == 1) return;
    // the last CTA of this (token, head) to finish merges all splits, in split
    // order (deterministic). The arrival counters sit at the FRONT of the
    // workspace (offset independent of N and splits) and are zeroed by the
    // host wrapper on the launching stream before every call.
    __shared__ int s_last;
    unsigned int* counters = reinterpret_cast<unsigned int*>(ws);
    const size_t nh = (size_t)n * H + h;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&counters[nh], 1u) == (unsigned)(splits - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x < Dh) {
        const int c = threadIdx.x;
        const float* p = ws + ws_partials_off(gridDim.y, H) + nh * splits * (Dh + 2);
        float M = -CUDART_INF_F;
        for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(p + sp * (Dh + 2)));
        float L = 0.f, A = 0.f;
        if (M != -CUDART_INF_F) {
            for (int sp = 0; sp < splits; ++sp) {
                const float* ps = p + sp * (Dh + 2);
                const float w = exp2f(__ldcg(ps) - M);
                L += __ldcg(ps + 1) * w;
                A += __ldcg(ps + 2 + c) * w;
            }
        }
        out[nh * Dh + c] = __float2bfloat16(L > 0.f ? A / L : 0.f);
    }
}

int attn_splits(int64_t N, int32_t H, int32_t Dh, int32_t C) {
    int dev = 0, sms = 148, per_sm = 8;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int b = 0;
        const cudaError_t e =
            Dh == 128 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, coherent_attn_kernel<128>,
                                                                      kThreads, 0)
                      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, coherent_attn_kernel<64>,
                                                                      kThreads, 0);
        if (e == cudaSuccess && b > 0) per_sm = b;
    }
    cudaGetLastError();
    const int64_t heads = N * (int64_t)H;
    const int64_t target = (int64_t)sms * per_sm;  // one full wave of resident CTAs
    int64_t splits = target / heads;  // round down: one full wave, no tail
    const int64_t max_splits = (C + 255) / 256;  // at least 256 keys per split
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    return (int)splits;
}

}  // namespace

// n_plan: the token count the split plan is made for (a decode rank holds
// about tokens_per_gpu tokens, the grid covers the capacity N; planning for N
// left 3/4 of the GPU idle at N = 4 GPUs)
int64_t attention_workspace_bytes(int64_t N, int32_t H, int32_t Dh, int32_t C, int64_t n_plan) {
    const int splits = attn_splits(std::max<int64_t>(1, std::min(n_plan, N)), H, Dh, C);
    cudaGetLastError();
    if (splits <= 1) return 0;
    return (int64_t)ws_partials_off(N, H) * (int64_t)sizeof(float) +
           N * (int64_t)H * (int64_t)splits * (Dh + 2) * (int64_t)sizeof(float);
}

exf_status launch_attention_model(const void* q, const int32_t* seq, int32_t seq_stride,
                                  const int32_t* n_dev, int64_t n_max, const int32_t* ctx,
                                  const void* k, const void* v, int32_t H, int32_t Dh, int32_t C,
                                  float scale, void* ws, void* out, int64_t n_plan, int32_t len_add,
                                  cudaStream_t st) {
    if (n_max <= 0) return EXF_OK;
    if (Dh != 64 && Dh != 128) return invalid("attention: head dim must be 64 or 128");
    const int splits = attn_splits(std::max<int64_t>(1, std::min(n_plan, n_max)), H, Dh, C);
    if (splits > 1 && !ws) return invalid("attention: workspace required");
    const int chunk = ((C + splits - 1) / splits + 63) / 64 * 64;
    const float scale_log2 = scale * 1.4426950408889634f;
    const dim3 grid(H, (unsigned)n_max, splits);
    if (splits > 1) EXF_CUDA_TRY(cudaMemsetAsync(ws, 0, (size_t)n_max * H * sizeof(unsigned int), st));
    auto qq = static_cast<const __nv_bfloat16*>(q);
    auto kk = static_cast<const __nv_bfloat16*>(k);
    auto vv = static_cast<const __nv_bfloat16*>(v);
    auto oo = static_cast<__nv_bfloat16*>(out);
    auto w = static_cast<float*>(ws);
    if (Dh == 64)
        coherent_attn_kernel<64><<<grid, kThreads, 0, st>>>(qq, seq, ctx, kk, vv, H, C, chunk, scale_log2, w, oo,
                                                            seq_stride, n_dev, len_add);
    else
        coherent_attn_kernel<128><<<grid, kThreads, 0, st>>>(qq, seq, ctx, kk, vv, H, C, chunk, scale_log2, w,
                                                             oo, seq_stride, n_dev, len_add);
    EXF_LAUNCH_CHECK("attention_model");
    return EXF_OK;
}

}  // namespace exf

extern "C" int64_t exf_coherent_attention_workspace_bytes(int64_t N, int32_t H, int32_t Dh,
                                                          int32_t C) {
    if (N <= 0 || H <= 0 || Dh <= 0 || C <= 0) return 0;
    int splits = exf::attn_splits(N, H, Dh, C);
    cudaGetLastError();
    if (splits <= 1) return 0;
    return (int64_t)exf::ws_partials_off(N, H) * (int64_t)sizeof(float) +
           N * (int64_t)H * (int64_t)splits * (Dh + 2) * (int64_t)sizeof(float);
}

extern "C" exf_status exf_coherent_attention(const void* d_q, const int32_t* d_seq,
                                             const int32_t* d_ctx_len, const void* d_k,
                                             const void* d_v, int64_t N, int32_t S, int32_t H,
                                             int32_t Dh, int32_t C, float scale,
                                             void* d_workspace, void* d_out,
                                             exf_stream_t stream) {
    using namespace exf;
    if (N < 0 || S <= 0 || H <= 0 || C <= 0) {
        set_error("coherent_attention: N >= 0, S, H, C > 0 required");
        return EXF_INVALID;
    }
    if (Dh != 64 && Dh != 128) {
        set_error("coherent_attention: head dim " + std::to_string(Dh) + " unsupported (64, 128)");
        return EXF_INVALID;
    }
    if (N > 65535) {
        set_error("coherent_attention: at most 65535 tokens per call");
        return EXF_INVALID;
    }
    if (N == 0) return EXF_OK;
    if (!d_q || !d_seq || !d_ctx_len || !d_k || !d_v || !d_out) {
        set_error("coherent_attention: null buffer");
        return EXF_INVALID;
    }
    const int splits = attn_splits(N, H, Dh, C);
    if (splits > 1 && !d_workspace) {
        set_error("coherent_attention: workspace required (exf_coherent_attention_workspace_bytes)");
        return EXF_INVALID;
    }
    const int chunk = ((C + splits - 1) / splits + 63) / 64 * 64;
    const float scale_log2 = scale * 1.4426950408889634f;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const dim3 grid(H, (unsigned)N, splits);
    auto q = static_cast<const __nv_bfloat16*>(d_q);
    auto k = static_cast<const __nv_bfloat16*>(d_k);
    auto v = static_cast<const __nv_bfloat16*>(d_v);
    auto o = static_cast<__nv_bfloat16*>(d_out);
    auto ws = static_cast<float*>(d_workspace);
    if (splits > 1) {  // arrival counters (front of the workspace) start from zero
        const cudaError_t ze = cudaMemsetAsync(ws, 0, (size_t)N * H * sizeof(unsigned int), st);
        if (ze != cudaSuccess) return cuda_status(ze, "coherent_attention counter reset");
    }
    if (Dh == 64) {
        coherent_attn_kernel<64><<<grid, kThreads, 0, st>>>(q, d_seq, d_ctx_len, k, v, H, C, chunk,
                                                            scale_log2, ws, o, 1, nullptr, 0);
    } else {
        coherent_attn_kernel<128><<<grid, kThreads, 0, st>>>(q, d_seq, d_ctx_len, k, v, H, C,
                                                             chunk, scale_log2, ws, o, 1, nullptr, 0);
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_status(err, "coherent_attention launch");
    return EXF_OK;
}

// ---------------------------------------------------------------------------
// Per-step K/V append into every replica of the context cache: the data the
// ExFlow context AllGather moves (proj/src/sim.cpp:161-162). The rank that
// holds a token writes its new K/V rows at position ctx_len[seq] of each
// replica (local or NVLink peer pointers, up to 8) and advances ctx_len there.
// One token per sequence per call (decode), so positions are race-free and
// every replica stays identical.
namespace exf {
namespace {

constexpr int kMaxReplicas = 8;
struct KvReplicas {
    __nv_bfloat16* k[kMaxReplicas];
    __nv_bfloat16* v[kMaxReplicas];
    int32_t* ctx[kMaxReplicas];
};

// grid (N), 128 threads: one token's H*Dh K and V values per block.
__global__ void __launch_bounds__(128) kv_append_kernel(const uint4* __restrict__ k_new,
                                                        const uint4* __restrict__ v_new,
                                                        const int32_t* __restrict__ seq,
                                                        int32_t H, int32_t Dh, int32_t C,
                                                        int32_t replicas, KvReplicas rep,
                                                        int32_t* overflow, int32_t seq_stride,
                                                        const int32_t* __restrict__ n_dev,
                                                        int64_t new_stride) {
    const int n = blockIdx.x;
    if (n_dev && n >= *n_dev) return;
    const int s = seq[(size_t)n * seq_stride];
    const int pos = rep.ctx[0][s];
    if (pos >= C) {
        if (threadIdx.x == 0 && overflow) atomicAdd(overflow, 1);
        return;
    }
    const int vec_per_head = Dh / 8;
    const int vecs = H * vec_per_head;
    for (int i = threadIdx.x; i < vecs; i += blockDim.x) {
        const int h = i / vec_per_head, c = i % vec_per_head;
        const uint4 kv = k_new[(size_t)n * new_stride + i];
        const uint4 vv = v_new[(size_t)n * new_stride + i];
        const size_t off = (((size_t)s * H + h) * C + pos) * vec_per_head + c;
        for (int r = 0; r < replicas; ++r) {
            reinterpret_cast<uint4*>(rep.k[r])[off] = kv;
            reinterpret_cast<uint4*>(rep.v[r])[off] = vv;
        }
    }
    // rows visible before the new length: system scope when replicas live on
    // peer GPUs, device scope when the only replica is local
    if (replicas > 1)
        __threadfence_system();
    else
        __threadfence();
    __syncthreads();
    if (threadIdx.x == 0)
        for (int r = 0; r < replicas; ++r) rep.ctx[r][s] = pos + 1;
}

}  // namespace

// Decode-step forms used by the model (attn_block.cu): token count on the
// device (grid over the capacity), sequence id = the token id of each
// resident row (ResMeta stride 2), rows of the projection buffers with their
// own stride (int4 units).
exf_status launch_kv_append_model(const void* k_new, const void* v_new, int64_t new_stride_vec,
                                  const int32_t* seq, int32_t seq_stride, const int32_t* n_dev,
                                  int64_t n_max, int32_t H, int32_t Dh, int32_t C, int32_t replicas,
                                  void* const* k_caches, void* const* v_caches,
                                  int32_t* const* lens, int32_t* overflow, cudaStream_t st) {
    if (replicas < 1 || replicas > kMaxReplicas) return invalid("kv_append: replicas must be in [1, 8]");
    KvReplicas rep{};
    for (int r = 0; r < replicas; ++r) {
        rep.k[r] = static_cast<__nv_bfloat16*>(k_caches[r]);
        rep.v[r] = static_cast<__nv_bfloat16*>(v_caches[r]);
        rep.ctx[r] = lens[r];
    }
    if (n_max <= 0) return EXF_OK;
    kv_append_kernel<<<(unsigned)n_max, 128, 0, st>>>(static_cast<const uint4*>(k_new),
                                                      static_cast<const uint4*>(v_new), seq, H, Dh, C,
                                                      replicas, rep, overflow, seq_stride, n_dev,
                                                      new_stride_vec);
    EXF_LAUNCH_CHECK("kv_append_model");
    return EXF_OK;
}

}  // namespace exf

extern "C" exf_status exf_kv_append(const void* d_k_new, const void* d_v_new,
                                    const int32_t* d_seq, int64_t N, int32_t S, int32_t H,
                                    int32_t Dh, int32_t C, int32_t replicas,
                                    void* const* h_k_caches, void* const* h_v_caches,
                                    int32_t* const* h_ctx_lens, int32_t* d_overflow,
                                    exf_stream_t stream) {
    using namespace exf;
    if (N < 0 || S <= 0 || H <= 0 || C <= 0) {
        set_error("kv_append: N >= 0, S, H, C > 0 required");
        return EXF_INVALID;
    }
    if (Dh <= 0 || Dh % 8 != 0) {
        set_error("kv_append: head dim must be a positive multiple of 8");
        return EXF_INVALID;
    }
    if (replicas < 1 || replicas > kMaxReplicas) {
        set_error("kv_append: replicas must be in [1, 8]");
        return EXF_INVALID;
    }
    if (N > S) {
        set_error("kv_append: more tokens than sequences (one token per sequence per call)");
        return EXF_INVALID;
    }
    if (N == 0) return EXF_OK;
    if (!d_k_new || !d_v_new || !d_seq || !h_k_caches || !h_v_caches || !h_ctx_lens) {
        set_error("kv_append: null buffer");
        return EXF_INVALID;
    }
    KvReplicas rep{};
    for (int r = 0; r < replicas; ++r) {
        if (!h_k_caches[r] || !h_v_caches[r] || !h_ctx_lens[r]) {
            set_error("kv_append: null replica " + std::to_string(r));
            return EXF_INVALID;
        }
        rep.k[r] = static_cast<__nv_bfloat16*>(h_k_caches[r]);
        rep.v[r] = static_cast<__nv_bfloat16*>(h_v_caches[r]);
        rep.ctx[r] = h_ctx_lens[r];
    }
    kv_append_kernel<<<(unsigned)N, 128, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(d_k_new), static_cast<const uint4*>(d_v_new), d_seq, H, Dh, C,
        replicas, rep, d_overflow, 1, nullptr, (int64_t)H * Dh / 8);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_status(err, "kv_append launch");
    return EXF_OK;
}

// ---------------------------------------------------------------------------
// Buffer sharing for the cache replicas: a 64-byte CUDA-IPC handle plus the
// byte offset of the pointer inside its allocation (caching allocators hand
// out sub-ranges), opened on the CALLER's current device so that kernels
// launched there can store into the peer's HBM over NVLink.
#include <cuda.h>

extern "C" exf_status exf_ipc_export(const void* d_ptr, void* h_handle64, int64_t* h_offset) {
    using namespace exf;
    if (!d_ptr || !h_handle64 || !h_offset) return invalid("ipc_export: null argument");
    // driver entry point resolved at run time (no link-time libcuda dependency)
    using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static RangeFn range_fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<RangeFn>(p);
        return static_cast<RangeFn>(nullptr);
    }();
    if (!range_fn) return runtime_err("ipc_export: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS)
        return runtime_err("ipc_export: pointer is not a device allocation");
    cudaIpcMemHandle_t h;
    EXF_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
    memcpy(h_handle64, &h, 64);
    *h_offset = (int64_t)(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
    return EXF_OK;
}

extern "C" exf_status exf_ipc_import(const void* h_handle64, int64_t offset, void** d_ptr) {
    using namespace exf;
    if (!h_handle64 || !d_ptr || offset < 0) return invalid("ipc_import: bad argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, h_handle64, 64);
    void* base = nullptr;
    EXF_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *d_ptr = static_cast<char*>(base) + offset;
    return EXF_OK;
}

extern "C" exf_status exf_ipc_close(void* d_ptr, int64_t offset) {
    using namespace exf;
    if (!d_ptr) return invalid("ipc_close: null pointer");
    EXF_CUDA_TRY(cudaIpcCloseMemHandle(static_cast<char*>(d_ptr) - offset));
    return EXF_OK;
}
