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
// out = x + prob * (H W2^T + b2)), grid (M / RB, E_loc):
//   * a CTA owns RB output features (weight rows) of one local expert; S
//     threads share a row, each streaming K/S consecutive weights with 32 B
//     loads (4 in flight per thread), L1-bypassing;
//   * the expert's tokens are staged per tile of <= 16 in shared memory
//     (canonical (slot, source, order) rows of the receive region for GEMM1,
//     H rows for GEMM2) and read as broadcasts;
//   * each thread accumulates its k-range in order with fmaf; the S partials
//     of a row are summed in k order through shared memory: deterministic,
//     fp32 accumulation (the fp64 oracle sits within ~1e-6 relative).
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
constexpr int kF32TokTile = 16;          // tokens per pass (accumulators per thread)
constexpr size_t kF32SmemBudget = 200 * 1024;

__device__ __forceinline__ float4 ld_stream4(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ float gelu_exact(float v) { return 0.5f * v * (1.0f + erff(v * 0.70710678118654752440f)); }

}  // namespace

template <int MODE, int S>
__global__ void __launch_bounds__(kF32Threads) ffn_f32_kernel(FfnF32Args a) {
    constexpr int RB = kF32Threads / S;  // weight rows per CTA
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int32_t s_prefix[9], s_start[8];
    __shared__ int32_t s_ne, s_off;
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
        while (ptx::ld_acquire_sys(f) < epoch) g.step(a.err, ERR_TIMEOUT_DISPATCH);
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
    const int tile = min(kF32TokTile, (int)(kF32SmemBudget / ((size_t)K * 4)));
    float* sx = reinterpret_cast<float*>(smem);                           // [tile][K]
    float* red = reinterpret_cast<float*>(smem + (size_t)tile * K * 4);  // [RB][S][tile]
    const int row_l = tid / S, ks = tid - row_l * S;
    const int r = blockIdx.x * RB + row_l;  // weight row == output feature
    const int kn = K / S, k0 = ks * kn;
    const float* wr = a.w + ((int64_t)e * M + r) * K + k0;
    const float bias = a.bias[(int64_t)e * M + r];
    for (int t0 = 0; t0 < n_e; t0 += tile) {
        const int nt = min(tile, n_e - t0);
        // ---- stage the tile's token rows (float4 copies)
        const int vec = K / 4;
        for (int i = tid; i < nt * vec; i += kF32Threads) {
            const int t = i / vec, v = i - t * vec;
            const float* src = MODE == 0 ? rx + recv_row(t0 + t) * (int64_t)a.d
                                         : a.H + (int64_t)(off_e + t0 + t) * a.dff;
            reinterpret_cast<float4*>(sx)[i] = reinterpret_cast<const float4*>(src)[v];
        }
        __syncthreads();
        float acc[kF32TokTile];
#pragma unroll
        for (int t = 0; t < kF32TokTile; ++t) acc[t] = 0.f;
        // ---- stream this thread's k-range of its weight row, 32 floats per
        // round in flight, each 8-float group applied to every token in order
        for (int k = 0; k < kn; k += 32) {
            float4 w[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) w[u] = ld_stream4(wr + k + 4 * u);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
#pragma unroll
                for (int t = 0; t < kF32TokTile; ++t) {
                    if (t < nt) {
                        const float4 x = *reinterpret_cast<const float4*>(sx + (int64_t)t * K + k0 + k + 4 * u);
                        acc[t] = fmaf(w[u].x, x.x, acc[t]);
                        acc[t] = fmaf(w[u].y, x.y, acc[t]);
                        acc[t] = fmaf(w[u].z, x.z, acc[t]);
                        acc[t] = fmaf(w[u].w, x.w, acc[t]);
                    }
                }
            }
        }
        // ---- the S partials of each row, summed in k order
        if (S > 1) {
#pragma unroll
            for (int t = 0; t < kF32TokTile; ++t)
                if (t < nt) red[((int64_t)row_l * S + ks) * tile + t] = acc[t];
            __syncthreads();
        }
        if (ks == 0) {
            for (int t = 0; t < nt; ++t) {
                float v = acc[t];
                if (S > 1) {
                    v = red[((int64_t)row_l * S) * tile + t];
                    for (int j = 1; j < S; ++j) v += red[((int64_t)row_l * S + j) * tile + t];
                }
                const int i = t0 + t;  // canonical index within the expert
                if (MODE == 0) {
                    a.H[(int64_t)(off_e + i) * a.dff + r] = gelu_exact(v + bias);
                } else {
                    const int64_t rr = recv_row(i);
                    const float p = rmeta[rr].prob;
                    a.res_x_out[(int64_t)(off_e + i) * a.d + r] = rx[rr * a.d + r] + p * (v + bias);
                }
            }
        }
        if (MODE == 1 && blockIdx.x == 0)
            for (int t = tid; t < nt; t += kF32Threads) {
                const RecvMeta m = rmeta[recv_row(t0 + t)];
                a.res_meta_out[off_e + t0 + t] = ResMeta{m.token, m.expert};
            }
        __syncthreads();  // the tile buffer is reused
    }
}

exf_status launch_ffn_f32(const FfnF32Args& a, int mode, cudaStream_t s) {
    const int M = mode == 0 ? a.dff : a.d;
    const int K = mode == 0 ? a.d : a.dff;
    if (a.G > 8) return invalid("fp32 FFN supports up to 8 ranks");
    // GEMM1 (K = d): 2 threads per row; GEMM2 (K = d_ffn): 8 per row
    const int S = mode == 0 ? 2 : 8;
    const int RB = kF32Threads / S;
    if (M % RB != 0 || K % (32 * S) != 0)
        return invalid("fp32 FFN needs d_model, d_ffn multiples of 256 and of 32 x threads per row");
    const int tile = std::min<int>(kF32TokTile, (int)(kF32SmemBudget / ((size_t)K * 4)));
    if (tile < 1) return invalid("fp32 FFN: a token row does not fit in shared memory");
    const size_t smem = (size_t)tile * K * 4 + (size_t)RB * S * tile * 4;
    auto k0 = ffn_f32_kernel<0, 2>;
    auto k1 = ffn_f32_kernel<1, 8>;
    static bool attr = false;
    if (!attr) {
        EXF_CUDA_TRY(cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, 216 * 1024));
        EXF_CUDA_TRY(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, 216 * 1024));
        max_carveout(k0);
        max_carveout(k1);
        attr = true;
    }
    const dim3 grid(M / RB, a.E_loc);
    if (mode == 0) EXF_CUDA_TRY(launch_pdl(k0, grid, dim3(kF32Threads), smem, s, 0, a));
    else EXF_CUDA_TRY(launch_pdl(k1, grid, dim3(kF32Threads), smem, s, 0, a));
    return EXF_OK;
}

}  // namespace exf
