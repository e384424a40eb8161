// attn_block.cu -- the attention block of the context-coherent decode layer
// (SURVEY §8(f) rank 1): the token a dispatch left on this GPU attends over
// its own sequence in this GPU's replica of the context,
// so the layer needs no combine exchange.
//
// Per layer, on the resident tokens of this rank (n <= capacity, on device):
//   dense_gemm_kernel<MODE 0>  q, k, v = x Wqkv^T + bqkv        (tcgen05)
//   kv append                  k, v rows of every resident token into EVERY
//                              replica of the layer's K/V cache over NVLink
//                              (attention.cu; the per-step context AllGather
//                              of the new tokens' context, one row per layer)
//   coherent attention         softmax(q K^T / sqrt(Dh)) V over the token's
//                              own sequence in the local replica (attention.cu)
//   dense_gemm_kernel<MODE 1>  x = x + attn Wo^T + bo, in place (tcgen05)
// then the MoE layer (layer_fused.cu) routes the updated x.
//
// dense_gemm_kernel is the decode-shaped dense GEMM: swap-AB,
//   D[m][n] = sum_k W[m][k] X[n][k]   M = output features (128 per tile),
//                                     N = resident tokens (NT per chunk)
// weights by TMA (SWIZZLE_128B, evict-first) in an mbarrier ring, token rows
// by TMA tile boxes (rows past the resident count are ignored), one elected
// thread issues tcgen05.mma kind::f16 into a double-buffered TMEM accumulator.
// Split-K over a thread-block cluster of KS CTAs: the fp32 partials meet in
// distributed shared memory and each CTA finishes 128/KS rows, summing the
// partials in CTA order (deterministic). HBM-bound at decode batch sizes
// (weights 6 d^2 + 2 d^2 bytes per layer, ~2 x tokens flops per weight byte).
//
// The setup AllGather (context_setup_kernel, once before decoding,
// proj/src/sim.cpp:162): every rank writes the prefix of its home sequences'
// context into every replica, then flags every peer and waits for all.
#include "common.cuh"
#include "model.cuh"
#include "ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>

namespace exf {

namespace {

constexpr int kDBM = 128;
constexpr int kDBK = 64;
constexpr int kDThreads = 192;  // w0 TMA, w1 MMA + TMEM, w2..w5 epilogue (TMEM lane quarters 2,3,0,1)

template <int NT, int STAGES>
struct DenseSmem {
    static constexpr int kA = kDBM * kDBK * 2;  // 16 KB of weights per k-block
    static constexpr int kB = NT * kDBK * 2;    // token rows per k-block
    static constexpr int kP = NT * kDBM * 4;    // fp32 partial [NT][128]
    static constexpr int kOffA = 0;
    static constexpr int kOffB = STAGES * kA;
    static constexpr int kOffP = kOffB + STAGES * kB;
    static constexpr int kOffBar = kOffP + kP;
    // full[S], empty[S], tmem_full[2], tmem_empty[2], red_full, red_empty
    static constexpr int kOffMisc = kOffBar + (2 * STAGES + 6) * 8;
    static constexpr int kBytes = kOffMisc + 64 + 1024;
};

}  // namespace

template <int NT, int STAGES, int MODE>
__global__ void __launch_bounds__(kDThreads, 1)
dense_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                  const DenseArgs a) {
    using S = DenseSmem<NT, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint64_t* tmem_empty = tmem_full + 2;
    uint64_t* red_full = tmem_empty + 2;
    uint64_t* red_empty = red_full + 1;
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + S::kOffMisc);
    float* P = reinterpret_cast<float*>(smem + S::kOffP);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ks = a.ksplit;
    const uint32_t crank = ptx::cluster_ctarank();
    const int mt = blockIdx.x / ks;          // 128-row tile of the output features
    const int kbs = a.K / kDBK / ks;         // k-blocks of this split
    const int kb0 = (int)crank * kbs;

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tmem_full[b], 1);
            ptx::mbar_init(&tmem_empty[b], 128);
        }
        ptx::mbar_init(red_full, ks);
        ptx::mbar_init(red_empty, ks);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&misc[0], 2 * NT);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = misc[0];
    // the token count comes from the previous kernel (the MoE layer / step
    // begin); weights do not: their first stages are issued before the wait
    const uint64_t pol_w = ptx::policy_evict_first();
    const int npre = min(kbs, STAGES);
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmW);
        ptx::tma_prefetch_desc(&tmX);
        for (int kb = 0; kb < npre; ++kb) {
            ptx::mbar_arrive_expect_tx(&full[kb], S::kA + S::kB);
            ptx::tma_load_2d(smem + S::kOffA + kb * S::kA, &tmW, &full[kb], (kb0 + kb) * kDBK, mt * kDBM, pol_w);
        }
    }
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int n = *a.n_dev;
    if (MODE == 1 && a.replicas > 0 && blockIdx.x == 0) {
        // folded K/V append, second half: the attention (previous kernel) has
        // read every length; advance each resident token's sequence in every
        // replica (rows were stored two kernels earlier, in stream order)
        for (int t = tid; t < n; t += kDThreads) {
            const int sq = a.seq[(int64_t)t * 2];
            if (a.lens[0][sq] >= a.kv_C) {
                if (a.overflow) atomicAdd(a.overflow, 1);
                continue;
            }
            for (int r = 0; r < a.replicas; ++r) a.lens[r][sq] += 1;
        }
    }
    const int chunks = max(1, (n + NT - 1) / NT);  // >= 1: the prefetched stages are consumed

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_x = ptx::policy_evict_last();  // every m-tile re-reads the rows
            int it = 0;
            for (int c = 0; c < chunks; ++c)
                for (int kb = 0; kb < kbs; ++kb, ++it) {
                    const int st = it % STAGES;
                    if (it >= npre) {
                        ptx::mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1, a.err, 121);
                        ptx::mbar_arrive_expect_tx(&full[st], S::kA + S::kB);
                        ptx::tma_load_2d(smem + S::kOffA + st * S::kA, &tmW, &full[st], (kb0 + kb) * kDBK,
                                         mt * kDBM, pol_w);
                    }
                    ptx::tma_load_2d(smem + S::kOffB + st * S::kB, &tmX, &full[st], (kb0 + kb) * kDBK, c * NT,
                                     pol_x);
                }
        }
    } else if (warp == 1) {
        int it = 0;
        for (int c = 0; c < chunks; ++c) {
            const int nc = max(0, min(NT, n - c * NT));
            const int ncol = max(16, (nc + 15) & ~15);
            const uint32_t idesc = ptx::umma_idesc_bf16(kDBM, ncol);
            const int buf = c & 1;
            if (c >= 2) ptx::mbar_wait(&tmem_empty[buf], ((c >> 1) - 1) & 1, a.err, 122);
            ptx::tc_fence_after();
            const uint32_t d_tmem = tmem + buf * NT;
            for (int kb = 0; kb < kbs; ++kb, ++it) {
                const int st = it % STAGES;
                ptx::mbar_wait(&full[st], (it / STAGES) & 1, a.err, 123);
                ptx::tc_fence_after();
                if (lane == 0) {
                    const uint64_t da = ptx::umma_desc_sw128(ptx::smem_u32(smem + S::kOffA + st * S::kA));
                    const uint64_t db = ptx::umma_desc_sw128(ptx::smem_u32(smem + S::kOffB + st * S::kB));
#pragma unroll
                    for (int kk = 0; kk < kDBK / 16; ++kk)
                        ptx::umma_bf16(d_tmem, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) ? 1u : 0u);
                    ptx::umma_commit(&empty[st]);
                    if (kb + 1 == kbs) ptx::umma_commit(&tmem_full[buf]);
                }
                __syncwarp();
            }
        }
    } else {
        // ================= epilogue (warps 2..5 = TMEM lane quarters 2,3,0,1)
        const int et = (warp & 3) * 32 + lane;  // TMEM lane == weight row in the tile
        const int rows_per = kDBM / ks;
        const int r_lo = (int)crank * rows_per;
        const int tpr = kDBM / rows_per;
        const int my_row = r_lo + (et % rows_per);
        const int my_n0 = et / rows_per;
        const int m_glob = mt * kDBM + my_row;
        const float bias = __bfloat162float(a.bias[m_glob]);
        for (int c = 0; c < chunks; ++c) {
            const int nc = max(0, min(NT, n - c * NT));
            const int buf = c & 1;
            ptx::mbar_wait(&tmem_full[buf], (c >> 1) & 1, a.err, 124);
            ptx::tc_fence_after();
            if (c > 0) ptx::mbar_wait_cluster(red_empty, (c - 1) & 1, a.err, 125);
            const uint32_t t_base = tmem + buf * NT + ((uint32_t)((warp & 3) * 32) << 16);
            for (int col = 0; col < nc; col += 16) {
                uint32_t r[16];
                ptx::tmem_ld_32x32b_x16(t_base + col, r);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 16; ++i) P[(col + i) * kDBM + et] = __uint_as_float(r[i]);
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tmem_empty[buf]);
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (et == 0) {
                ptx::fence_acq_rel_cluster();
                for (int qc = 0; qc < ks; ++qc) ptx::mbar_arrive_remote(red_full, qc);
            }
            ptx::mbar_wait_cluster(red_full, c & 1, a.err, 126);
            for (int t = my_n0; t < nc; t += tpr) {
                float acc = 0.f;
                for (int qc = 0; qc < ks; ++qc) {  // CTA order: deterministic
                    const uint32_t ad = ptx::dsmem_addr(&P[t * kDBM + my_row], qc);
                    float v;
                    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ad) : "memory");
                    acc += v;
                }
                acc += bias;
                const int64_t row = (int64_t)c * NT + t;  // resident row
                if (MODE == 0) {
                    // q | k | v column ranges of the fused projection
                    const int which = m_glob / a.d, col = m_glob - which * a.d;
                    if (which > 0 && a.replicas > 0) {
                        // k / v row straight into every replica of the context
                        // cache at the sequence's current length
                        const int sq = a.seq[row * 2];
                        const int pos = a.lens[0][sq];
                        if (pos < a.kv_C) {
                            const int h = col / a.kv_Dh, dc = col - h * a.kv_Dh;
                            const int64_t off = (((int64_t)sq * a.kv_H + h) * a.kv_C + pos) * a.kv_Dh + dc;
                            const __nv_bfloat16 v = __float2bfloat16(acc);
                            for (int r = 0; r < a.replicas; ++r) (which == 1 ? a.kc[r] : a.vc[r])[off] = v;
                        }
                    } else {
                        __nv_bfloat16* dst = which == 0 ? a.out[0] : (which == 1 ? a.out[1] : a.out[2]);
                        dst[row * a.d + col] = __float2bfloat16(acc);
                    }
                } else {
                    __nv_bfloat16* x = a.out[0] + row * a.d + m_glob;
                    *x = __float2bfloat16(__bfloat162float(*x) + acc);
                }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (et == 0) {
                ptx::fence_acq_rel_cluster();
                for (int qc = 0; qc < ks; ++qc) ptx::mbar_arrive_remote(red_empty, qc);
            }
        }
        // peers must be done reading this CTA's partial before it exits
        ptx::mbar_wait_cluster(red_empty, (chunks - 1) & 1, a.err, 127);
    }
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 2 * NT);
    }
}

// ------------------------------------------------------------------ setup AllGather
// Deterministic synthetic prefix context of sequence s (the prompt's K/V,
// identical on every replica): N(0, 1) bf16 from (seed, layer, s, k|v, index).
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

__global__ void __launch_bounds__(256) context_setup_kernel(ContextSetupArgs a) {
    // grid (pos blocks, home sequences, layers)
    const int j = blockIdx.z;
    const int home_i = blockIdx.y;
    // AllGather: home sequence (round robin, sim.cpp:111) into every replica;
    // local: every sequence into this rank's replica only (same contents)
    const int s = a.local ? home_i : a.rank + a.G * home_i;
    const int row_elems = a.H * a.Dh;     // per position, all heads
    const int64_t per_head = (int64_t)a.Cctx * a.Dh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)a.prefix * row_elems;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int pos = (int)(i / row_elems), rem = (int)(i - (int64_t)pos * row_elems);
        const int h = rem / a.Dh, c = rem - h * a.Dh;
        const uint64_t key = (((uint64_t)j * 1000003u + (uint64_t)s) * 31u + (uint64_t)h) * 65537u + (uint64_t)pos;
        const uint64_t hk = mix64(a.seed ^ mix64(key * 2u + 0u) ^ (uint64_t)c * 0x9E37u);
        const uint64_t hv = mix64(a.seed ^ mix64(key * 2u + 1u) ^ (uint64_t)c * 0x9E37u);
        // sum of 4 uniforms, centred and scaled: unit variance, bounded
        auto draw = [](uint64_t hsh) {
            float t = 0.f;
            for (int q = 0; q < 4; ++q) t += (float)((hsh >> (16 * q)) & 0xFFFF) * (1.f / 65536.f);
            return (t - 2.0f) * 1.7320508f;
        };
        const __nv_bfloat16 kv = __float2bfloat16(draw(hk)), vv = __float2bfloat16(draw(hv));
        const int64_t off = (((int64_t)j * a.S + s) * a.H + h) * per_head + (int64_t)pos * a.Dh + c;
        for (int r = a.local ? a.rank : 0; r < (a.local ? a.rank + 1 : a.G); ++r) {
            __nv_bfloat16* base_k = reinterpret_cast<__nv_bfloat16*>(a.peers[r] + a.kv_k);
            __nv_bfloat16* base_v = reinterpret_cast<__nv_bfloat16*>(a.peers[r] + a.kv_v);
            base_k[off] = kv;
            base_v[off] = vv;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int r = a.local ? a.rank : 0; r < (a.local ? a.rank + 1 : a.G); ++r)
            reinterpret_cast<int32_t*>(a.peers[r] + a.kv_len)[(int64_t)j * a.S + s] = a.prefix;
}

// every rank: rows + lengths visible system-wide, flag every peer (publish),
// wait for all peers' flags (wait)
__global__ void context_setup_sync_kernel(uint8_t* const* peers, int64_t flag_off, int G, int rank,
                                          uint64_t epoch, int32_t* err, int publish, int wait) {
    __threadfence_system();
    if (publish && (int)threadIdx.x < G) {
        uint64_t* f = reinterpret_cast<uint64_t*>(peers[threadIdx.x] + flag_off) + rank;
        ptx::st_release_sys(f, epoch);
    }
    __syncthreads();
    if (wait && (int)threadIdx.x < G) {
        const uint64_t* f = reinterpret_cast<const uint64_t*>(peers[rank] + flag_off) + threadIdx.x;
        ptx::SpinGuard g;
        while (ptx::ld_acquire_sys(f) < epoch) g.step(err, ERR_TIMEOUT_GATHER);
    }
}

// ------------------------------------------------------------------ host side
namespace {

template <int NT, int STAGES, int MODE>
struct DenseLauncher {
    using Sm = DenseSmem<NT, STAGES>;
    static constexpr auto kern = dense_gemm_kernel<NT, STAGES, MODE>;
    bool ready = false;
    exf_status launch(const CUtensorMap& w, const CUtensorMap& x, const DenseArgs& a, cudaStream_t s) {
        if (!ready) {
            EXF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Sm::kBytes));
            EXF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            max_carveout(kern);
            ready = true;
        }
        const int tiles = a.M / kDBM;
        EXF_CUDA_TRY(launch_pdl(kern, dim3(tiles * a.ksplit), dim3(kDThreads), Sm::kBytes, s, a.ksplit, w, x, a));
        return EXF_OK;
    }
};

}  // namespace

// split-K so the grid covers about one wave of the 148 SMs
int dense_gemm_ksplit(int M, int K) {
    const int tiles = M / kDBM, kblocks = K / kDBK;
    int ks = 1;
    while (ks < 8 && tiles * ks * 2 <= 148 && kblocks % (ks * 2) == 0 && kblocks / (ks * 2) >= 2) ks *= 2;
    return ks;
}

exf_status launch_dense_gemm(const CUtensorMap& w, const CUtensorMap& x, const DenseArgs& a, int nt, int mode,
                             cudaStream_t s) {
    if (a.M % kDBM || a.K % (kDBK * a.ksplit)) return invalid("dense GEMM shape not tileable");
    static DenseLauncher<64, 6, 0> q64;
    static DenseLauncher<64, 6, 1> o64;
    static DenseLauncher<128, 4, 0> q128;
    static DenseLauncher<128, 4, 1> o128;
    if (nt <= 64) return mode == 0 ? q64.launch(w, x, a, s) : o64.launch(w, x, a, s);
    return mode == 0 ? q128.launch(w, x, a, s) : o128.launch(w, x, a, s);
}

exf_status launch_context_setup(const ContextSetupArgs& a, int64_t flag_off, uint64_t epoch, int32_t* err,
                                int phase, cudaStream_t s) {
    const int B = a.local ? a.S : a.S / a.G;  // sequences this rank writes
    if (phase != 2 && B > 0) {
        const int64_t elems = (int64_t)a.prefix * a.H * a.Dh;
        const int bx = (int)std::min<int64_t>(64, (elems + 255) / 256);
        context_setup_kernel<<<dim3(std::max(bx, 1), B, a.L), 256, 0, s>>>(a);
        EXF_LAUNCH_CHECK("context_setup_kernel");
    }
    if (a.local) return EXF_OK;  // nothing crossed GPUs: no flags
    context_setup_sync_kernel<<<1, 32, 0, s>>>(a.peers, flag_off, a.G, a.rank, epoch, err, phase != 2,
                                               phase != 1);
    EXF_LAUNCH_CHECK("context_setup_sync_kernel");
    return EXF_OK;
}

}  // namespace exf
