// ffn_f32.cu -- the grouped expert FFN of the fp32 mode (BASELINE.json
// north_star: layer outputs within 1e-5 relative error in fp32 mode; the
// bf16 mode runs on tcgen05, layer_fused.cu / ffn_tcgen05.cu).
//
// fp32 has no dense tensor-core path that keeps 1e-5 (kind::tf32 rounds the
// operands to 10-bit mantissas), so this is a SIMT kernel shaped for the
// roofline that binds it: at decode batch sizes an expert sees a handful of
// tokens, so the work is weight streaming (2 x d x d_ffn x 4 B per active
// expert) with ~2 x tokens flops per weight -- far below the fp32 FMA ridge.
//
// One launch per GEMM (MODE 0: H = gelu(X W1^T + b1); MODE 1:
// out = x + prob * (H W2^T + b2)), grid (M / RB, E_loc), 256 threads:
//   * the K dimension streams through a 4-stage cp.async ring of chunks of
//     32 columns: the CTA's RB weight rows (16-byte copies, 128 contiguous
//     bytes per row and chunk, rows padded to 36 floats so that the
//     per-thread 16-byte row reads are bank-conflict free) and the same 32
//     columns of the expert's <= 16 tokens (canonical (slot, source, order)
//     rows of the receive region for GEMM1, H rows for GEMM2);
//   * TPR threads share a weight row, each owning 16/TPR tokens; a warp's
//     lanes hold 32 different rows and the same tokens, so every token read
//     is a shared-memory broadcast and every weight read a conflict-free
//     vector;
//   * each thread accumulates its row x tokens in k order with fmaf:
//     deterministic fp32 accumulation (the fp64 oracle sits within ~1e-6).
// Version history: one thread per row reading global memory directly (0.05 of
// HBM: uncoalesced), then one warp per row with a butterfly per row (0.19:
// every token read was a 512-byte non-broadcast shared load).
// Tokens of expert e come from the dispatch exactly as on the bf16 two-kernel
// path: per-(source, slot) counts in recv_cnt, rows of source s for slot e at
// [seg_start, +cnt) of s's receive region, flags per source (GEMM1 waits).
#include "common.cuh"
#include "model.cuh"
#include "ptx.cuh"

#include <algorithm>

namespace exf {

namespace {

constexpr int kF32Threads = 256;
constexpr int kF32TokTile = 16;  // tokens per pass
constexpr int kKC = 32;          // k columns per pipeline chunk
constexpr int kWStride = 36;     // floats per staged weight row (144 B: 16-byte aligned, odd granules)
constexpr int kStages = 4;

__device__ __forceinline__ float gelu_exact(float v) { return 0.5f * v * (1.0f + erff(v * 0.70710678118654752440f)); }

template <int TPR>
struct F32Smem {
    static constexpr int kRB = kF32Threads / TPR;     // weight rows per CTA
    static constexpr int kW = kRB * kWStride * 4;     // bytes of one weight chunk
    static constexpr int kX = kF32TokTile * kKC * 4;  // bytes of one token chunk (2 KB)
    static constexpr int kStage = kW + kX;
    static constexpr int kBytes = kStages * kStage;
};

}  // namespace

template <int MODE, int TPR>
__global__ void __launch_bounds__(kF32Threads) ffn_f32_kernel(FfnF32Args a) {
    using S = F32Smem<TPR>;
    constexpr int RB = S::kRB;
    constexpr int TPT = kF32TokTile / TPR;  // tokens per thread
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int32_t s_prefix[9], s_start[8];
    __shared__ int32_t s_ne, s_off;
    __shared__ int64_t s_src[kF32TokTile];  // first float of each token row of the tile
    const int tid = threadIdx.x;
    const int e = blockIdx.y;
    const int M = MODE == 0 ? a.dff : a.d;
    const int K = MODE == 0 ? a.d : a.dff;
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const uint64_t q = *a.step * (uint64_t)a.L + (uint64_t)a.layer;
    const int parity = (int)(q & 1);
    if (MODE == 0 && tid < a.G) {  // every source's dispatch of this layer
        const uint64_t epoch = q + 1;
        const uint64_t* f = reinterpret_cast<const uint64_t*>(a.own_sym + a.sym.flags) + parity * a.G + tid;
        ptx::SpinGuard g;
        while (ptx::flag_read(f, a.G > 1) < epoch) g.step(a.err, ERR_TIMEOUT_DISPATCH);
    }
    __syncthreads();
    const int32_t* cnt = reinterpret_cast<const int32_t*>(a.own_sym + a.sym.recv_cnt) +
                         (int64_t)parity * a.G * a.E_loc;
    if (tid == 0) {
        int n = 0, off = 0;
        for (int s = 0; s < a.G; ++s) {
            int st = 0;
            for (int x = 0; x < e; ++x) st += cnt[s * a.E_loc + x];
            off += st;
            s_prefix[s] = n;
            s_start[s] = st;
            n += cnt[s * a.E_loc + e];
        }
        s_prefix[a.G] = n;
        s_ne = n;
        s_off = off;
        if (MODE == 1 && e == 0 && blockIdx.x == 0) {
            int total = 0;
            for (int i = 0; i < a.G * a.E_loc; ++i) total += cnt[i];
            *a.n_res_out = total;
        }
    }
    __syncthreads();
    const int n_e = s_ne, off_e = s_off;
    if (n_e == 0) return;  // an expert without tokens costs no weight traffic
    const float* rx = reinterpret_cast<const float*>(a.own_sym + a.sym.recv_x);
    const RecvMeta* rmeta = reinterpret_cast<const RecvMeta*>(a.own_sym + a.sym.recv_meta);
    auto recv_row = [&](int i) -> int64_t {  // token i of this expert (canonical) -> receive row
        int s = 0;
        while (s + 1 < a.G && s_prefix[s + 1] <= i) ++s;
        return ((int64_t)parity * a.G + s) * a.C + s_start[s] + (i - s_prefix[s]);
    };
    const int row_l = tid % RB, part = tid / RB;  // a warp: 32 rows, one token group
    const int r0 = blockIdx.x * RB;
    const float* wbase = a.w + ((int64_t)e * M + r0) * K;
    const float* tbase = MODE == 0 ? rx : a.H;
    const int nchunks = K / kKC;
    for (int t0 = 0; t0 < n_e; t0 += kF32TokTile) {
        const int nt = min(kF32TokTile, n_e - t0);
        if (tid < kF32TokTile)
            s_src[tid] = tid < nt ? (MODE == 0 ? recv_row(t0 + tid) * (int64_t)a.d
                                               : (int64_t)(off_e + t0 + tid) * a.dff)
                                  : -1;
        __syncthreads();
        auto stage_chunk = [&](int c) {  // cp.async of chunk c into ring slot c % kStages
            uint8_t* sb = smem + (c % kStages) * S::kStage;
            float* sw = reinterpret_cast<float*>(sb);
            float* sx = reinterpret_cast<float*>(sb + S::kW);
            const int k0 = c * kKC;
            for (int i = tid; i < RB * (kKC / 4); i += kF32Threads) {  // 8 x 16 B per row
                const int r = i >> 3, g = i & 7;
                ptx::cp_async16(sw + r * kWStride + g * 4, wbase + (int64_t)r * K + k0 + g * 4);
            }
            if (tid < kF32TokTile * (kKC / 4)) {
                const int t = tid >> 3, g = tid & 7;
                if (t < nt) ptx::cp_async16(sx + t * kKC + g * 4, tbase + s_src[t] + k0 + g * 4);
            }
        };
        for (int c = 0; c < kStages - 1; ++c) {
            if (c < nchunks) stage_chunk(c);
            ptx::cp_async_commit();
        }
        float acc[TPT];
#pragma unroll
        for (int t = 0; t < TPT; ++t) acc[t] = 0.f;
        for (int c = 0; c < nchunks; ++c) {
            asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 2) : "memory");
            __syncthreads();  // chunk c visible to every thread; slot (c-1) % kStages free
            if (c + kStages - 1 < nchunks) stage_chunk(c + kStages - 1);
            ptx::cp_async_commit();
            const uint8_t* sb = smem + (c % kStages) * S::kStage;
            const float* sw = reinterpret_cast<const float*>(sb) + row_l * kWStride;
            const float* sx = reinterpret_cast<const float*>(sb + S::kW) + (part * TPT) * kKC;
#pragma unroll
            for (int k4 = 0; k4 < kKC / 4; ++k4) {
                const float4 w = *reinterpret_cast<const float4*>(sw + k4 * 4);
#pragma unroll
                for (int t = 0; t < TPT; ++t) {
                    const float4 x = *reinterpret_cast<const float4*>(sx + t * kKC + k4 * 4);
                    acc[t] = fmaf(w.x, x.x, acc[t]);
                    acc[t] = fmaf(w.y, x.y, acc[t]);
                    acc[t] = fmaf(w.z, x.z, acc[t]);
                    acc[t] = fmaf(w.w, x.w, acc[t]);
                }
            }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        const int r = r0 + row_l;
        const float bias = a.bias[(int64_t)e * M + r];
#pragma unroll
        for (int t = 0; t < TPT; ++t) {
            const int tt = part * TPT + t;
            if (tt < nt) {
                const int i = t0 + tt;  // canonical index within the expert
                if (MODE == 0) {
                    a.H[(int64_t)(off_e + i) * a.dff + r] = gelu_exact(acc[t] + bias);
                } else {
                    const int64_t rrow = recv_row(i);
                    const float p = rmeta[rrow].prob;
                    a.res_x_out[(int64_t)(off_e + i) * a.d + r] = rx[rrow * a.d + r] + p * (acc[t] + bias);
                }
            }
        }
        if (MODE == 1 && blockIdx.x == 0)
            for (int t = tid; t < nt; t += kF32Threads) {
                const RecvMeta m = rmeta[recv_row(t0 + t)];
                a.res_meta_out[off_e + t0 + t] = ResMeta{m.token, m.expert};
            }
        __syncthreads();  // the ring and s_src are reused by the next token tile
    }
}

exf_status launch_ffn_f32(const FfnF32Args& a, int mode, cudaStream_t s) {
    const int M = mode == 0 ? a.dff : a.d;
    const int K = mode == 0 ? a.d : a.dff;
    if (a.G > 8) return invalid("fp32 FFN supports up to 8 ranks");
    // GEMM1 (M = d_ffn rows): 2 threads per row, 128 rows per CTA; GEMM2
    // (M = d rows, 4x fewer): 4 threads per row, 64 rows per CTA (8 threads
    // per row, 32 rows, measured slower: every CTA re-reads the token chunk)
    const int tpr = mode == 0 ? 2 : 4;
    const int rb = kF32Threads / tpr;
    if (M % rb != 0 || K % kKC != 0) return invalid("fp32 FFN needs d_model, d_ffn multiples of 128");
    auto k0 = ffn_f32_kernel<0, 2>;
    auto k1 = ffn_f32_kernel<1, 4>;
    static bool attr = false;
    if (!attr) {
        EXF_CUDA_TRY(cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, F32Smem<2>::kBytes));
        EXF_CUDA_TRY(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, F32Smem<4>::kBytes));
        max_carveout(k0);
        max_carveout(k1);
        attr = true;
    }
    const dim3 grid(M / rb, a.E_loc);
    if (mode == 0) EXF_CUDA_TRY(launch_pdl(k0, grid, dim3(kF32Threads), F32Smem<2>::kBytes, s, 0, a));
    else EXF_CUDA_TRY(launch_pdl(k1, grid, dim3(kF32Threads), F32Smem<4>::kBytes, s, 0, a));
    return EXF_OK;
}

}  // namespace exf
