// ffn_tcgen05.cu -- kernel (4): grouped expert FFN on the 5th-gen tensor
// cores (tcgen05.mma kind::f16, bf16 in / fp32 accumulate in TMEM).
//
// Decode is weight-streaming: tokens per expert are few (8..256), weights are
// 16*d^2 bytes per expert, so every configured shape sits far below the ridge
// (SURVEY.md §8d, H4). The kernel is built around streaming weights at HBM
// rate with swap-AB:
//   D[m][n] = sum_k W[m][k] * X[n][k]     M = weight rows (128 per tile),
//                                         N = tokens of the expert (<= NMAX)
//   A = weight tile, TMA (SWIZZLE_128B, evict-first), multi-stage mbarrier ring
//   B = token rows, GATHERED by two producer warps straight from the
//       per-source receive regions the dispatch kernel wrote (no permutation
//       copy), stored in the same 128-byte swizzle, fence.proxy.async
//   MMA = one elected thread, 4 x (M128 x N x K16) per 64-wide k-block
//   split-K across a thread-block cluster; partial accumulators are reduced
//   through distributed shared memory (DSMEM) in a fixed CTA order
//   (deterministic), each CTA finishing 128/KS rows.
// Warp roles (256 threads): w0 TMA(A) | w1 MMA + TMEM alloc | w2-3 B gather |
// w4-7 epilogue (TMEM -> regs -> smem partial -> DSMEM reduce -> epilogue).
// Epilogues: GEMM1 h = bf16(gelu(acc + b1)) -> H (canonical token order);
//            GEMM2 out = x + prob*(acc + b2) -> next-layer resident rows.
#include "common.cuh"
#include "model.cuh"
#include "ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>

namespace exf {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 256;
constexpr int kMaxSrc = 8;

template <int NMAX, int STAGES>
struct FfnSmem {
    static constexpr int kA = kBM * kBK * 2;     // 16 KB
    static constexpr int kB = NMAX * kBK * 2;    // NMAX * 128 B
    static constexpr int kP = NMAX * kBM * 4;    // fp32 partial [NMAX][128]
    static constexpr int kOffA = 0;
    static constexpr int kOffB = kOffA + STAGES * kA;
    static constexpr int kOffP = kOffB + STAGES * kB;
    static constexpr int kOffBar = kOffP + kP;
    // full[S], empty[S], tmem_full, tmem_empty, red_full, red_empty
    static constexpr int kOffMisc = kOffBar + (2 * STAGES + 4) * 8;
    static constexpr int kBytes = kOffMisc + 256 + 1024;  // + alignment slack
};

__device__ __forceinline__ float gelu_erf(float v) {
    return 0.5f * v * (1.0f + erff(v * 0.70710678118654752440f));
}

template <int NMAX, int STAGES, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
ffn_gemm_kernel(const __grid_constant__ CUtensorMap tmapA, const FfnArgs a) {
    using S = FfnSmem<NMAX, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint64_t* tmem_empty = tmem_full + 1;
    uint64_t* red_full = tmem_empty + 1;
    uint64_t* red_empty = red_full + 1;
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + S::kOffMisc);
    // misc: [0] tmem base, [1] n_e, [2] off_e, [3] total tokens,
    //       [8..16] seg_prefix[G+1], [24..31] seg_start[G]
    int32_t* seg_prefix = reinterpret_cast<int32_t*>(misc + 8);
    int32_t* seg_start = reinterpret_cast<int32_t*>(misc + 24);
    float* P = reinterpret_cast<float*>(smem + S::kOffP);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ks = a.ksplit;
    const uint32_t crank = ptx::cluster_ctarank();
    const int unit = blockIdx.x / ks;
    const int mtiles = a.M_total / kBM;
    const int e = unit / mtiles;
    const int mt = unit - e * mtiles;
    const int kbs = a.K / kBK / ks;           // k-blocks of this split
    const int kb0 = (int)crank * kbs;

    const uint64_t q = *a.step * (uint64_t)a.L + (uint64_t)a.layer;
    const int parity = (int)(q & 1);
    const uint64_t epoch = q + 1;

    // ---- wait for every source's dispatch of this layer (GEMM1 only)
    if (MODE == 0 && tid < a.G) {
        const uint64_t* f = reinterpret_cast<const uint64_t*>(a.own_sym + a.sym.flags) + parity * a.G + tid;
        ptx::SpinGuard g;
        while (ptx::ld_acquire_sys(f) < epoch) g.step(a.err, ERR_TIMEOUT_DISPATCH);
    }
    __syncthreads();
    // ---- segment table of expert e: tokens from source s occupy rows
    //      [seg_start[s], +cnt) of recv region s; canonical order is source-major
    if (tid == 0) {
        const int32_t* cnt = reinterpret_cast<const int32_t*>(a.own_sym + a.sym.recv_cnt) +
                             (int64_t)parity * a.G * a.E_loc;
        int n_e = 0, off = 0, total = 0;
        for (int s = 0; s < a.G; ++s) {
            int st = 0;
            for (int x = 0; x < a.E_loc; ++x) {
                const int c = cnt[s * a.E_loc + x];
                if (x < e) {
                    st += c;
                    off += c;
                }
                total += c;
            }
            seg_start[s] = st;
            seg_prefix[s] = n_e;
            n_e += cnt[s * a.E_loc + e];
        }
        seg_prefix[a.G] = n_e;
        misc[1] = n_e;
        misc[2] = off;
        misc[3] = total;
    }
    __syncthreads();
    const int n_e = (int)misc[1];
    const int off_e = (int)misc[2];
    if (MODE == 1 && blockIdx.x == 0 && tid == 0) *a.n_res_out = (int)misc[3];
    if (n_e == 0) return;  // uniform across the cluster (same expert)

    const RecvMeta* rmeta = reinterpret_cast<const RecvMeta*>(a.own_sym + a.sym.recv_meta);
    const __nv_bfloat16* rx = reinterpret_cast<const __nv_bfloat16*>(a.own_sym + a.sym.recv_x);
    // token i of expert e -> row index in the [2][G][C] receive arrays
    auto recv_row = [&](int i) -> int64_t {
        int s = 0;
        while (s + 1 < a.G && seg_prefix[s + 1] <= i) ++s;
        return ((int64_t)parity * a.G + s) * a.C + seg_start[s] + (i - seg_prefix[s]);
    };
    if (MODE == 1 && mt == 0 && crank == 0) {
        for (int i = tid; i < n_e; i += kThreads) {
            const RecvMeta m = rmeta[recv_row(i)];
            a.res_meta_out[off_e + i] = ResMeta{m.token, m.expert};
        }
    }

    const int nchunks = (n_e + NMAX - 1) / NMAX;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1 + 64);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(tmem_full, 1);
        ptx::mbar_init(tmem_empty, 128);
        ptx::mbar_init(red_full, ks);
        ptx::mbar_init(red_empty, ks);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&misc[0], NMAX);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = misc[0];

    if (warp == 0) {
        // ================= A producer (weights via TMA) =================
        if (lane == 0) {
            ptx::tma_prefetch_desc(&tmapA);
            const uint64_t pol = ptx::policy_evict_first();
            const int row0 = e * a.M_total + mt * kBM;
            int it = 0;
            for (int c = 0; c < nchunks; ++c)
                for (int kb = 0; kb < kbs; ++kb, ++it) {
                    const int st = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    ptx::mbar_wait(&empty[st], ph ^ 1, a.err, ERR_TIMEOUT_PIPE);
                    ptx::mbar_arrive_expect_tx(&full[st], S::kA);
                    ptx::tma_load_2d(smem + S::kOffA + st * S::kA, &tmapA, &full[st],
                                     (kb0 + kb) * kBK, row0, pol);
                }
        }
    } else if (warp == 1) {
        // ================= MMA issuer =================
        int it = 0;
        for (int c = 0; c < nchunks; ++c) {
            const int nc = min(NMAX, n_e - c * NMAX);
            const int ncol = (nc + 15) & ~15;
            const uint32_t idesc = ptx::umma_idesc_bf16(kBM, ncol);
            if (c > 0) ptx::mbar_wait(tmem_empty, (c - 1) & 1, a.err, ERR_TIMEOUT_PIPE);
            ptx::tc_fence_after();
            for (int kb = 0; kb < kbs; ++kb, ++it) {
                const int st = it % STAGES;
                const uint32_t ph = (it / STAGES) & 1;
                ptx::mbar_wait(&full[st], ph, a.err, ERR_TIMEOUT_PIPE);
                ptx::tc_fence_after();
                if (lane == 0) {
                    const uint64_t da = ptx::umma_desc_sw128(ptx::smem_u32(smem + S::kOffA + st * S::kA));
                    const uint64_t db = ptx::umma_desc_sw128(ptx::smem_u32(smem + S::kOffB + st * S::kB));
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk)
                        ptx::umma_bf16(tmem, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) ? 1u : 0u);
                    ptx::umma_commit(&empty[st]);
                    if (kb == kbs - 1) ptx::umma_commit(tmem_full);
                }
                __syncwarp();
            }
        }
    } else if (warp < 4) {
        // ================= B producer: gather token rows =================
        const int t64 = tid - 64;
        int it = 0;
        for (int c = 0; c < nchunks; ++c) {
            const int cb = c * NMAX;
            const int nc = min(NMAX, n_e - cb);
            const int ncol = (nc + 15) & ~15;
            for (int kb = 0; kb < kbs; ++kb, ++it) {
                const int st = it % STAGES;
                const uint32_t ph = (it / STAGES) & 1;
                ptx::mbar_wait(&empty[st], ph ^ 1, a.err, ERR_TIMEOUT_PIPE);
                uint8_t* bs = smem + S::kOffB + st * S::kB;
                const int kcol = (kb0 + kb) * kBK;
                for (int qd = t64; qd < ncol * 8; qd += 64) {
                    const int r = qd >> 3, cc = qd & 7;
                    int4 v = make_int4(0, 0, 0, 0);
                    if (r < nc) {
                        const __nv_bfloat16* src;
                        if (MODE == 0) src = rx + recv_row(cb + r) * a.d + kcol + cc * 8;
                        else src = a.H + (int64_t)(off_e + cb + r) * a.dff + kcol + cc * 8;
                        v = *reinterpret_cast<const int4*>(src);
                    }
                    *reinterpret_cast<int4*>(bs + r * 128 + ((cc ^ (r & 7)) << 4)) = v;
                }
                ptx::fence_proxy_async_smem();
                ptx::mbar_arrive(&full[st]);
            }
        }
    } else {
        // ================= epilogue =================
        const int et = tid - 128;          // TMEM lane == weight row within the tile
        const int lane_base = (warp & 3) * 32;
        const int rows_per = kBM / ks;     // rows this CTA finishes
        const int r_lo = (int)crank * rows_per;
        const int tpr = kThreads / 2 / rows_per;  // threads per row group (128/rows_per)
        const int my_row = r_lo + (et % rows_per);
        const int my_n0 = et / rows_per;
        const int m_glob = mt * kBM + my_row;
        const float bias = __bfloat162float(a.bias[(int64_t)e * a.M_total + m_glob]);
        for (int c = 0; c < nchunks; ++c) {
            const int cb = c * NMAX;
            const int nc = min(NMAX, n_e - cb);
            const int ncol = (nc + 15) & ~15;
            ptx::mbar_wait(tmem_full, c & 1, a.err, ERR_TIMEOUT_PIPE);
            ptx::tc_fence_after();
            if (c > 0) ptx::mbar_wait_cluster(red_empty, (c - 1) & 1, a.err, ERR_TIMEOUT_PIPE);
            for (int col = 0; col < ncol; col += 16) {
                uint32_t r[16];
                ptx::tmem_ld_32x32b_x16(tmem + ((uint32_t)lane_base << 16) + col, r);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 16; ++i) P[(col + i) * kBM + et] = __uint_as_float(r[i]);
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(tmem_empty);
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (et == 0) {
                ptx::fence_acq_rel_cluster();
                for (int qc = 0; qc < ks; ++qc) ptx::mbar_arrive_remote(red_full, qc);
            }
            ptx::mbar_wait_cluster(red_full, c & 1, a.err, ERR_TIMEOUT_PIPE);
            // reduce rows [r_lo, r_lo + rows_per) over the cluster in CTA order
            for (int n = my_n0; n < nc; n += tpr) {
                float acc = 0.f;
                for (int qc = 0; qc < ks; ++qc) {
                    const uint32_t ad = ptx::dsmem_addr(&P[n * kBM + my_row], qc);
                    float v;
                    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ad) : "memory");
                    acc += v;
                }
                acc += bias;
                const int i = cb + n;  // token index within expert e
                if (MODE == 0) {
                    a.H[(int64_t)(off_e + i) * a.dff + m_glob] = __float2bfloat16(gelu_erf(acc));
                } else {
                    const int64_t rr = recv_row(i);
                    const float xin = __bfloat162float(rx[rr * a.d + m_glob]);
                    const float p = rmeta[rr].prob;
                    a.res_x_out[(int64_t)(off_e + i) * a.d + m_glob] = __float2bfloat16(xin + p * acc);
                }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (et == 0) {
                ptx::fence_acq_rel_cluster();
                for (int qc = 0; qc < ks; ++qc) ptx::mbar_arrive_remote(red_empty, qc);
            }
        }
        // peers must be done reading this CTA's partial before it exits
        ptx::mbar_wait_cluster(red_empty, (nchunks - 1) & 1, a.err, ERR_TIMEOUT_PIPE);
    }
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, NMAX);
    }
}

// ------------------------------------------------------------------ host side
namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

}  // namespace

// Row-major [rows][cols] bf16 matrix, box = 128 rows x 64 cols, SWIZZLE_128B.
exf_status make_weight_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t cols) {
    EncodeFn fn = encode_fn();
    if (!fn) return runtime_err("cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)kBM};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return runtime_err("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return EXF_OK;
}

template <int NMAX, int STAGES, int MODE>
static exf_status launch_one(const CUtensorMap& map, const FfnArgs& a, int units, cudaStream_t s) {
    using S = FfnSmem<NMAX, STAGES>;
    auto kern = ffn_gemm_kernel<NMAX, STAGES, MODE>;
    static bool attr = false;
    if (!attr) {
        EXF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes));
        EXF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(units * a.ksplit);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = S::kBytes;
    cfg.stream = s;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = a.ksplit;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    EXF_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, map, a));
    return EXF_OK;
}

exf_status launch_ffn_gemm(const CUtensorMap& map, const FfnArgs& a, int nmax, cudaStream_t s) {
    if (a.M_total % kBM != 0) return invalid("FFN rows must be a multiple of 128");
    if (a.K % (kBK * a.ksplit) != 0) return invalid("FFN K must be a multiple of 64*ksplit");
    if (a.G > kMaxSrc) return invalid("at most 8 ranks per dispatch group");
    const int units = a.E_loc * (a.M_total / kBM);
    if (nmax <= 64) {
        return a.mode == 0 ? launch_one<64, 6, 0>(map, a, units, s) : launch_one<64, 6, 1>(map, a, units, s);
    }
    return a.mode == 0 ? launch_one<128, 4, 0>(map, a, units, s) : launch_one<128, 4, 1>(map, a, units, s);
}

}  // namespace exf
