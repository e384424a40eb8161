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
// PERSISTENT: one CTA per SM (grid <= co-resident clusters x KS); each
// cluster walks the (expert, m-tile) work items round-robin, the TMA ring
// never drains between items, and the TMEM accumulator is double-buffered so
// the epilogue of item i overlaps the MMAs of item i+1.
// Split-K across a thread-block cluster of KS CTAs: partial accumulators are
// exchanged through DSMEM with cluster-scope mbarriers and summed in CTA order
// (deterministic); each CTA finishes 128/KS rows.
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
constexpr int kMaxLocal = 64;

template <int NMAX, int STAGES>
struct FfnSmem {
    static constexpr int kA = kBM * kBK * 2;     // 16 KB
    static constexpr int kB = NMAX * kBK * 2;    // NMAX * 128 B
    static constexpr int kP = NMAX * kBM * 4;    // fp32 partial [NMAX][128]
    static constexpr int kOffA = 0;
    static constexpr int kOffB = kOffA + STAGES * kA;
    static constexpr int kOffP = kOffB + STAGES * kB;
    static constexpr int kOffTab = kOffP + kP;
    // per local expert: n, off, seg_prefix[9], seg_start[8]
    static constexpr int kTabInts = 20;
    static constexpr int kOffBar = kOffTab + kMaxLocal * kTabInts * 4;
    // full[S], empty[S], tmem_full[2], tmem_empty[2], red_full, red_empty
    static constexpr int kOffMisc = kOffBar + (2 * STAGES + 6) * 8;
    static constexpr int kBytes = kOffMisc + 64 + 1024;  // + alignment slack
};


template <int NMAX, int STAGES, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
ffn_gemm_kernel(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB,
                const FfnArgs a) {
    using S = FfnSmem<NMAX, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;  // [2]
    uint64_t* tmem_empty = tmem_full + 2;  // [2]
    uint64_t* red_full = tmem_empty + 2;
    uint64_t* red_empty = red_full + 1;
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + S::kOffMisc);  // [0] tmem base
    int32_t* tab = reinterpret_cast<int32_t*>(smem + S::kOffTab);
    float* P = reinterpret_cast<float*>(smem + S::kOffP);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ks = a.ksplit;
    const uint32_t crank = ptx::cluster_ctarank();
    const int cluster_id = blockIdx.x / ks;
    const int num_clusters = gridDim.x / ks;
    const int mtiles = a.M_total / kBM;
    const int items = a.E_loc * mtiles;
    const int kbs = a.K / kBK / ks;  // k-blocks of this split
    const int kb0 = (int)crank * kbs;

    uint64_t* ts = a.tstamp ? a.tstamp + (int64_t)blockIdx.x * 16 : nullptr;
    if (ts && tid == 0) ts[0] = ptx::globaltimer();
    if (tid == 0) tl_mark(a.tl, 0);

    // ---- independent prologue (overlaps the previous kernel under PDL):
    //      barriers, TMEM, and the first weight stages of this CTA's first item
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 2);  // A producer + B producer (expect_tx each)
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
    if (warp == 1) ptx::tmem_alloc(&misc[0], 2 * NMAX);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = misc[0];
    // weights do not depend on the previous kernel: prefetch the first
    // min(kbs, STAGES) k-blocks of the first item (its first chunk always runs)
    const int npre = cluster_id < items ? min(kbs, STAGES) : 0;
    const uint64_t pol_a = ptx::policy_evict_first();
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmapA);
        const int e0 = cluster_id / mtiles, mt0 = cluster_id - e0 * mtiles;
        for (int kb = 0; kb < npre; ++kb) {
            ptx::mbar_arrive_expect_tx(&full[kb], S::kA);
            ptx::tma_load_2d(smem + S::kOffA + kb * S::kA, &tmapA, &full[kb], (kb0 + kb) * kBK,
                             e0 * a.M_total + mt0 * kBM, pol_a);
        }
    }

    // ---- dependent part: the previous kernel's outputs become visible here
    ptx::pdl_wait();
    ptx::pdl_trigger();
    if (tid == 0) tl_mark(a.tl, 1);
    const uint64_t q = *a.step * (uint64_t)a.L + (uint64_t)a.layer;
    const int parity = (int)(q & 1);
    const uint64_t epoch = q + 1;

    // ---- wait for every source's dispatch of this layer (GEMM1 only)
    if (MODE == 0 && tid < a.G) {
        const uint64_t* f = reinterpret_cast<const uint64_t*>(a.own_sym + a.sym.flags) + parity * a.G + tid;
        ptx::SpinGuard g;
        while (ptx::flag_read(f, a.G > 1) < epoch) g.step(a.err, ERR_TIMEOUT_DISPATCH);
    }
    __syncthreads();
    // ---- per-expert segment tables: tokens of expert e from source s occupy
    //      rows [seg_start, +cnt) of recv region s; canonical order is
    //      source-major within the expert, experts in slot order
    const int32_t* cnt = reinterpret_cast<const int32_t*>(a.own_sym + a.sym.recv_cnt) +
                         (int64_t)parity * a.G * a.E_loc;
    if (tid < a.E_loc) {
        const int e = tid;
        int32_t* t = tab + e * S::kTabInts;
        int n = 0, off = 0;
        for (int s = 0; s < a.G; ++s) {
            int st = 0;
            for (int x = 0; x < e; ++x) st += cnt[s * a.E_loc + x];
            off += st;
            t[2 + s] = n;        // seg_prefix[s]
            t[11 + s] = st;      // seg_start[s]
            n += cnt[s * a.E_loc + e];
        }
        t[2 + a.G] = n;
        t[0] = n;
        t[1] = off;
    }
    if (MODE == 1 && blockIdx.x == 0 && tid == 0) {
        int total = 0;
        for (int i = 0; i < a.G * a.E_loc; ++i) total += cnt[i];
        *a.n_res_out = total;
    }

    const RecvMeta* rmeta = reinterpret_cast<const RecvMeta*>(a.own_sym + a.sym.recv_meta);
    const __nv_bfloat16* rx = reinterpret_cast<const __nv_bfloat16*>(a.own_sym + a.sym.recv_x);
    // token i of local expert e -> row index in the [2][G][C] receive arrays
    auto recv_row = [&](int e, int i) -> int64_t {
        const int32_t* t = tab + e * S::kTabInts;
        int s = 0;
        while (s + 1 < a.G && t[2 + s + 1] <= i) ++s;
        return ((int64_t)parity * a.G + s) * a.C + t[11 + s] + (i - t[2 + s]);
    };
    // chunks of item w: the CTA's first item always runs >= 1 chunk (its first
    // weight stages were prefetched before the token counts were known)
    auto nchunks = [&](int w, int n_e) {
        const int c = (n_e + NMAX - 1) / NMAX;
        return (w == cluster_id && c == 0) ? 1 : c;
    };
    __syncthreads();  // tables visible to every role of this CTA
    if (ts && tid == 0) ts[1] = ptx::globaltimer();

    if (warp == 0) {
        // ================= A producer (weights via TMA) =================
        if (lane == 0) {
            int it = 0;
            for (int w = cluster_id; w < items; w += num_clusters) {
                const int e = w / mtiles, mt = w - e * mtiles;
                const int nch = nchunks(w, tab[e * S::kTabInts]);
                const int row0 = e * a.M_total + mt * kBM;
                for (int c = 0; c < nch; ++c)
                    for (int kb = 0; kb < kbs; ++kb, ++it) {
                        if (it < npre) continue;  // prefetched in the prologue
                        const int st = it % STAGES;
                        const uint32_t ph = (it / STAGES) & 1;
                        ptx::mbar_wait(&empty[st], ph ^ 1, a.err, ERR_TIMEOUT_PIPE);
                        ptx::mbar_arrive_expect_tx(&full[st], S::kA);
                        ptx::tma_load_2d(smem + S::kOffA + st * S::kA, &tmapA, &full[st],
                                         (kb0 + kb) * kBK, row0, pol_a);
                    }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer =================
        int it = 0, job = 0;
        for (int w = cluster_id; w < items; w += num_clusters) {
            const int e = w / mtiles;
            const int n_e = tab[e * S::kTabInts];
            const int nch = nchunks(w, n_e);
            for (int c = 0; c < nch; ++c, ++job) {
                const int nc = max(0, min(NMAX, n_e - c * NMAX));
                const int ncol = max(16, (nc + 15) & ~15);
                const uint32_t idesc = ptx::umma_idesc_bf16(kBM, ncol);
                const int buf = job & 1;
                if (job >= 2) ptx::mbar_wait(&tmem_empty[buf], ((job >> 1) - 1) & 1, a.err, ERR_TIMEOUT_PIPE);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem + buf * NMAX;
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
                            ptx::umma_bf16(d_tmem, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) ? 1u : 0u);
                        ptx::umma_commit(&empty[st]);
                        if (kb == kbs - 1) ptx::umma_commit(&tmem_full[buf]);
                        if (ts && kb == 0 && job < 6) ts[2 + 2 * job] = ptx::globaltimer();
                        if (ts && kb == kbs - 1 && job < 6) ts[3 + 2 * job] = ptx::globaltimer();
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 2) {
        // ========== B producer: TMA gather4 of the expert's token rows ==========
        // lane l loads rows 4l..4l+3 of the token tile (row indices into the
        // receive region for GEMM1, into H for GEMM2); padding rows repeat the
        // chunk's first row and are discarded by the epilogue.
        if (lane == 0) ptx::tma_prefetch_desc(&tmapB);
        int it = 0;
        for (int w = cluster_id; w < items; w += num_clusters) {
            const int e = w / mtiles;
            const int n_e = tab[e * S::kTabInts];
            const int off_e = tab[e * S::kTabInts + 1];
            const int nch = nchunks(w, n_e);
            const int row_lim = MODE == 0 ? 2 * a.G * a.C : a.C;
            for (int c = 0; c < nch; ++c) {
                const int cb = c * NMAX;
                const int nc = max(0, min(NMAX, n_e - cb));
                const int ncol = max(16, (nc + 15) & ~15);
                const int ng = ncol >> 2;
                int32_t rows[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int r = 4 * lane + u;
                    const int i = cb + (r < nc ? r : 0);
                    const int64_t row = MODE == 0 ? recv_row(e, i) : (int64_t)(off_e + i);
                    rows[u] = (int32_t)(row < 0 ? 0 : (row >= row_lim ? row_lim - 1 : row));
                }
                for (int kb = 0; kb < kbs; ++kb, ++it) {
                    const int st = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    ptx::mbar_wait(&empty[st], ph ^ 1, a.err, ERR_TIMEOUT_PIPE);
                    if (lane == 0) ptx::mbar_arrive_expect_tx(&full[st], (uint32_t)ncol * 128u);
                    __syncwarp();
                    if (lane < ng)
                        ptx::tma_gather4(smem + S::kOffB + st * S::kB + lane * 512, &tmapB, &full[st],
                                         (kb0 + kb) * kBK, rows[0], rows[1], rows[2], rows[3]);
                }
            }
        }
    } else if (warp == 3) {
        // idle warp (keeps the epilogue warps aligned to TMEM lane quarters)
    } else {
        // ================= epilogue =================
        const int et = tid - 128;          // TMEM lane == weight row within the tile
        const int lane_base = (warp & 3) * 32;
        const int rows_per = kBM / ks;     // rows this CTA finishes
        const int r_lo = (int)crank * rows_per;
        const int tpr = kBM / rows_per;    // threads sharing one row
        const int my_row = r_lo + (et % rows_per);
        const int my_n0 = et / rows_per;
        int job = 0;
        for (int w = cluster_id; w < items; w += num_clusters) {
            const int e = w / mtiles, mt = w - e * mtiles;
            const int n_e = tab[e * S::kTabInts];
            const int off_e = tab[e * S::kTabInts + 1];
            if (MODE == 1 && mt == 0 && crank == 0) {
                for (int i = et; i < n_e; i += 128) {
                    const RecvMeta m = rmeta[recv_row(e, i)];
                    a.res_meta_out[off_e + i] = ResMeta{m.token, m.expert};
                }
            }
            const int m_glob = mt * kBM + my_row;
            const float bias = n_e ? __bfloat162float(a.bias[(int64_t)e * a.M_total + m_glob]) : 0.f;
            const int nch = nchunks(w, n_e);
            for (int c = 0; c < nch; ++c, ++job) {
                const int cb = c * NMAX;
                const int nc = max(0, min(NMAX, n_e - cb));
                const int ncol = max(16, (nc + 15) & ~15);
                const int buf = job & 1;
                ptx::mbar_wait(&tmem_full[buf], (job >> 1) & 1, a.err, ERR_TIMEOUT_PIPE);
                ptx::tc_fence_after();
                // peers must have finished reading the previous partial
                if (job > 0) ptx::mbar_wait_cluster(red_empty, (job - 1) & 1, a.err, ERR_TIMEOUT_PIPE);
                const uint32_t t_base = tmem + buf * NMAX + ((uint32_t)lane_base << 16);
                for (int col = 0; col < ncol; col += 16) {
                    uint32_t r[16];
                    ptx::tmem_ld_32x32b_x16(t_base + col, r);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) P[(col + i) * kBM + et] = __uint_as_float(r[i]);
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive(&tmem_empty[buf]);
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (et == 0) {
                    ptx::fence_acq_rel_cluster();
                    for (int qc = 0; qc < ks; ++qc) ptx::mbar_arrive_remote(red_full, qc);
                }
                ptx::mbar_wait_cluster(red_full, job & 1, a.err, ERR_TIMEOUT_PIPE);
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
                        const int64_t rr = recv_row(e, i);
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
        }
        // peers must be done reading this CTA's partial before it exits
        if (job > 0) ptx::mbar_wait_cluster(red_empty, (job - 1) & 1, a.err, ERR_TIMEOUT_PIPE);
        if (ts && et == 0) ts[14] = ptx::globaltimer();
    }
    __syncthreads();
    if (ts && tid == 0) ts[15] = ptx::globaltimer();
    if (tid == 0) tl_mark(a.tl, 3);
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 2 * NMAX);
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

template <int NMAX, int STAGES, int MODE>
struct Launcher {
    using S = FfnSmem<NMAX, STAGES>;
    static constexpr auto kern = ffn_gemm_kernel<NMAX, STAGES, MODE>;
    int max_clusters[17] = {0};  // co-resident clusters per cluster size

    exf_status prepare() {
        if (max_clusters[1]) return EXF_OK;
        EXF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes));
        EXF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        max_carveout(kern);
        for (int ks = 1; ks <= 16; ks *= 2) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(ks * 148);
            cfg.blockDim = dim3(kThreads);
            cfg.dynamicSmemBytes = S::kBytes;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = ks;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
                cudaGetLastError();
                n = 0;
            }
            max_clusters[ks] = n;
        }
        if (max_clusters[1] <= 0) return runtime_err("ffn kernel cannot be resident (smem/regs)");
        return EXF_OK;
    }

    // split-K / grid choice: minimise rounds x (K-blocks per split) with the
    // number of co-resident clusters of that size (cluster placement strands
    // SMs at larger sizes), tie -> smaller split.
    void plan(int items, int kblocks, int* ks_out, int* clusters_out) const {
        int best_ks = 1, best_cl = std::max(1, std::min(items, max_clusters[1]));
        long best = -1;
        for (int ks = 1; ks <= 16; ks *= 2) {
            if (kblocks % ks != 0 || max_clusters[ks] <= 0) continue;
            const int cl = std::max(1, std::min(items, max_clusters[ks]));
            const long rounds = (items + cl - 1) / cl;
            const long cost = rounds * (kblocks / ks) + (ks > 1 ? 1 : 0);
            if (best < 0 || cost < best) {
                best = cost;
                best_ks = ks;
                best_cl = cl;
            }
        }
        *ks_out = best_ks;
        *clusters_out = best_cl;
    }

    exf_status launch(const CUtensorMap& map, const CUtensorMap& mapB, FfnArgs a, int clusters,
                      cudaStream_t s) {
        EXF_CUDA_TRY(launch_pdl(kern, dim3(clusters * a.ksplit), dim3(kThreads), S::kBytes, s,
                                a.ksplit, map, mapB, a));
        return EXF_OK;
    }
};

// token tile x ring depth: smaller token tiles leave room for more weight
// stages in flight (A bytes in flight per SM = STAGES * 16 KB)
Launcher<32, 10, 0> g_l32_0;
Launcher<32, 10, 1> g_l32_1;
Launcher<64, 7, 0> g_l64_0;
Launcher<64, 7, 1> g_l64_1;
Launcher<128, 4, 0> g_l128_0;
Launcher<128, 4, 1> g_l128_1;

template <class F>
exf_status with_launcher(int nmax, int mode, F&& f) {
    if (nmax <= 32) return mode == 0 ? f(g_l32_0) : f(g_l32_1);
    if (nmax <= 64) return mode == 0 ? f(g_l64_0) : f(g_l64_1);
    return mode == 0 ? f(g_l128_0) : f(g_l128_1);
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

// Row-major [rows][cols] bf16 token matrix as UMMA B tiles: box = box_rows
// rows x 64 cols, SWIZZLE_128B (the K-major layout of one k-block), rows past
// the end zero-filled. Used where a tile's rows are contiguous (dense fused mode).
exf_status make_tile_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
    EncodeFn fn = encode_fn();
    if (!fn) return runtime_err("cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return runtime_err("cuTensorMapEncodeTiled (tile) failed: " + std::to_string((int)r));
    return EXF_OK;
}

// Row-major [rows][cols] bf16 token matrix for TMA gather4: box = 1 row x 64
// cols (128 B), SWIZZLE_128B, so four gathered rows land as one swizzled
// 4-row slab of the UMMA K-major B tile.
exf_status make_gather_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t cols) {
    EncodeFn fn = encode_fn();
    if (!fn) return runtime_err("cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kBK, 1};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return runtime_err("cuTensorMapEncodeTiled (gather) failed: " + std::to_string((int)r));
    return EXF_OK;
}

// Chooses (split-K, clusters) for a GEMM of `items` 128-row tiles over `K`.
exf_status plan_ffn_gemm(int nmax, int mode, int items, int K, int* ksplit, int* clusters) {
    const int kblocks = K / kBK;
    return with_launcher(nmax, mode, [&](auto& l) {
        EXF_TRY(l.prepare());
        l.plan(items, kblocks, ksplit, clusters);
        return EXF_OK;
    });
}

exf_status launch_ffn_gemm(const CUtensorMap& map, const CUtensorMap& mapB, const FfnArgs& a,
                           int nmax, int clusters,
                           cudaStream_t s) {
    if (a.M_total % kBM != 0) return invalid("FFN rows must be a multiple of 128");
    if (a.K % (kBK * a.ksplit) != 0) return invalid("FFN K must be a multiple of 64*ksplit");
    if (a.G > kMaxSrc) return invalid("at most 8 ranks per dispatch group");
    if (a.E_loc > kMaxLocal) return invalid("at most 64 local experts");
    return with_launcher(nmax, a.mode, [&](auto& l) {
        EXF_TRY(l.prepare());
        return l.launch(map, mapB, a, clusters, s);
    });
}

}  // namespace exf
