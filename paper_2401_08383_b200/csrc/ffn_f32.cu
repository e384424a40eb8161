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
// out = x + prob * (H W2^T + b2)), grid (M / kRowsPerCta, E_loc):
//   * each warp owns whole weight rows (output features); its 32 lanes read
//     one row as consecutive 16-byte vectors (512 B per warp instruction,
//     fully coalesced, L1-bypassing), a 1024-float chunk in flight at a time
//     with the next chunk prefetched;
//   * the expert's tokens are staged per tile of <= 16 in shared memory
//     (canonical (slot, source, order) rows of the receive region for GEMM1,
//     H rows for GEMM2); lane l reads token columns k = 4l + 128c (conflict-
//     free vectors);
//   * per token, each lane accumulates its columns in order with fmaf, then a
//     fixed xor butterfly sums the 32 lanes: deterministic fp32 accumulation
//     (the fp64 oracle sits within ~1e-6 relative).
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

constexpr int kRowsPerWarp = 8;
constexpr int kRowsPerCta = kRowsPerWarp * (kF32Threads / 32);  // 64

template <int MODE>
__global__ void __launch_bounds__(kF32Threads, 1) ffn_f32_kernel(FfnF32Args a) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int32_t s_prefix[9], s_start[8];
    __shared__ int32_t s_ne, s_off;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
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
    float* sx = reinterpret_cast<float*>(smem);  // [tile][K]
    const int nv = K / 128;                      // float4 per lane per row
    const int kchunks = (nv + 7) / 8;            // 32 lanes x 8 float4 per chunk
    for (int t0 = 0; t0 < n_e; t0 += tile) {
        const int nt = min(tile, n_e - t0);
        const int vec = K / 4;
        for (int i = tid; i < nt * vec; i += kF32Threads) {
            const int t = i / vec, v = i - t * vec;
            const float* src = MODE == 0 ? rx + recv_row(t0 + t) * (int64_t)a.d
                                         : a.H + (int64_t)(off_e + t0 + t) * a.dff;
            reinterpret_cast<float4*>(sx)[i] = reinterpret_cast<const float4*>(src)[v];
        }
        __syncthreads();
        // the warp's (row, chunk) items as one stream: the next item's weights
        // are always in flight while the current one is applied
        const int items = kRowsPerWarp * kchunks;
        auto row_of = [&](int it) { return blockIdx.x * kRowsPerCta + (it / kchunks) * (kF32Threads / 32) + warp; };
        auto load_item = [&](int it, float4 (&w)[8]) {
            const int c = it % kchunks;
            const float* wr = a.w + ((int64_t)e * M + row_of(it)) * K + c * 1024 + lane * 4;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                w[u] = c * 8 + u < nv ? ld_stream4(wr + u * 128) : make_float4(0.f, 0.f, 0.f, 0.f);
        };
        float acc[kF32TokTile];
#pragma unroll
        for (int t = 0; t < kF32TokTile; ++t) acc[t] = 0.f;
        float4 w[8];
        load_item(0, w);
        for (int it = 0; it < items; ++it) {
            const int c = it % kchunks;
            float4 wn[8];
            if (it + 1 < items) load_item(it + 1, wn);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int k = c * 1024 + u * 128 + lane * 4;
#pragma unroll
                for (int t = 0; t < kF32TokTile; ++t) {
                    if (t < nt && c * 8 + u < nv) {
                        const float4 x = *reinterpret_cast<const float4*>(sx + (int64_t)t * K + k);
                        acc[t] = fmaf(w[u].x, x.x, acc[t]);
                        acc[t] = fmaf(w[u].y, x.y, acc[t]);
                        acc[t] = fmaf(w[u].z, x.z, acc[t]);
                        acc[t] = fmaf(w[u].w, x.w, acc[t]);
                    }
                }
            }
            if (c == kchunks - 1) {  // the row is complete: reduce, write, restart
                const int r = row_of(it);
                // fixed xor butterfly over the 32 lanes (deterministic)
#pragma unroll
                for (int t = 0; t < kF32TokTile; ++t) {
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
                }
                const float bias = a.bias[(int64_t)e * M + r];
                // lane t writes token t (static register indexing via a select chain)
                float mine = acc[0];
#pragma unroll
                for (int t = 1; t < kF32TokTile; ++t)
                    if (lane == t) mine = acc[t];
                if (lane < nt) {
                    const int i = t0 + lane;  // canonical index within the expert
                    if (MODE == 0) {
                        a.H[(int64_t)(off_e + i) * a.dff + r] = gelu_exact(mine + bias);
                    } else {
                        const int64_t rrow = recv_row(i);
                        const float p = rmeta[rrow].prob;
                        a.res_x_out[(int64_t)(off_e + i) * a.d + r] = rx[rrow * a.d + r] + p * (mine + bias);
                    }
                }
#pragma unroll
                for (int t = 0; t < kF32TokTile; ++t) acc[t] = 0.f;
            }
            if (it + 1 < items) {
#pragma unroll
                for (int u = 0; u < 8; ++u) w[u] = wn[u];
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
    if (M % kRowsPerCta != 0 || K % 128 != 0)
        return invalid("fp32 FFN needs d_model, d_ffn multiples of 128 (and of 64 output rows)");
    const int tile = std::min<int>(kF32TokTile, (int)(kF32SmemBudget / ((size_t)K * 4)));
    if (tile < 1) return invalid("fp32 FFN: a token row does not fit in shared memory");
    const size_t smem = (size_t)tile * K * 4;
    auto k0 = ffn_f32_kernel<0>;
    auto k1 = ffn_f32_kernel<1>;
    static bool attr = false;
    if (!attr) {
        EXF_CUDA_TRY(cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF32SmemBudget));
        EXF_CUDA_TRY(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF32SmemBudget));
        max_carveout(k0);
        max_carveout(k1);
        attr = true;
    }
    const dim3 grid(M / kRowsPerCta, a.E_loc);
    if (mode == 0) EXF_CUDA_TRY(launch_pdl(k0, grid, dim3(kF32Threads), smem, s, 0, a));
    else EXF_CUDA_TRY(launch_pdl(k1, grid, dim3(kF32Threads), smem, s, 0, a));
    return EXF_OK;
}

}  // namespace exf
