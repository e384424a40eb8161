// tma_stream_bench.cu -- diagnostics: HBM streaming ceiling of the fused
// kernel's weight-operand pattern. Every CTA (one per SM) walks its own
// contiguous range of 128-row x 64-col bf16 boxes (SW128, K-major, like the
// A operand of layer_fused_kernel) through an mbarrier ring of S stages; a
// consumer thread just waits and frees each stage (no MMA). Prints GB/s per
// (stages, box rows). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -I../paper_2401_08383_b200/csrc tma_stream_bench.cu -o tma_stream_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"

using namespace exf;

template <int S>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, int rows_per_cta,
                                                       int box_rows, int kblocks, int* err) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int box_bytes = box_rows * 128;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * box_bytes);
    uint64_t* empty = full + S;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const int row0 = blockIdx.x * rows_per_cta;
    const int tiles = (rows_per_cta / box_rows) * kblocks;
    const uint64_t pol = ptx::policy_evict_first();
    if (threadIdx.x == 0) {
        for (int it = 0; it < tiles; ++it) {
            const int st = it % S;
            ptx::mbar_wait(&empty[st], ((it / S) & 1) ^ 1, err, 1);
            const int rt = it / kblocks, kb = it % kblocks;
            ptx::mbar_arrive_expect_tx(&full[st], box_bytes);
            ptx::tma_load_2d(smem + st * box_bytes, &tm, &full[st], kb * 64, row0 + rt * box_rows, pol);
        }
    } else if (threadIdx.x == 32) {
        for (int it = 0; it < tiles; ++it) {
            const int st = it % S;
            ptx::mbar_wait(&full[st], (it / S) & 1, err, 1);
            ptx::mbar_arrive(&empty[st]);
        }
    }
    __syncthreads();
}

// The same weight stream plus the dense-mode token operand: per weight box, a
// 64-row x 64-col box of a small L2-resident token matrix (B) through its own
// ring, like the fused kernel's GEMM1 (does B traffic slow the weight stream?)
template <int S, int SB>
__global__ void __launch_bounds__(96, 1) stream_ab_kernel(const __grid_constant__ CUtensorMap tm,
                                                          const __grid_constant__ CUtensorMap tx, int rows_per_cta,
                                                          int kblocks, int with_b, int* err) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int a_bytes = 128 * 128, b_bytes = 64 * 128;
    uint8_t* sb = smem + S * a_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sb + SB * b_bytes);
    uint64_t* empty = full + S;
    uint64_t* fullb = empty + S;
    uint64_t* emptyb = fullb + SB;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < SB; ++s) {
            ptx::mbar_init(&fullb[s], 1);
            ptx::mbar_init(&emptyb[s], 1);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const int row0 = blockIdx.x * rows_per_cta;
    const int tiles = (rows_per_cta / 128) * kblocks;
    const uint64_t pol = ptx::policy_evict_first(), polx = ptx::policy_evict_last();
    if (threadIdx.x == 0) {
        for (int it = 0; it < tiles; ++it) {
            const int st = it % S;
            ptx::mbar_wait(&empty[st], ((it / S) & 1) ^ 1, err, 1);
            const int rt = it / kblocks, kb = it % kblocks;
            ptx::mbar_arrive_expect_tx(&full[st], a_bytes);
            ptx::tma_load_2d(smem + st * a_bytes, &tm, &full[st], kb * 64, row0 + rt * 128, pol);
        }
    } else if (threadIdx.x == 64 && with_b) {
        for (int it = 0; it < tiles; ++it) {
            const int st = it % SB;
            ptx::mbar_wait(&emptyb[st], ((it / SB) & 1) ^ 1, err, 1);
            ptx::mbar_arrive_expect_tx(&fullb[st], b_bytes);
            ptx::tma_load_2d(sb + st * b_bytes, &tx, &fullb[st], (it % kblocks) * 64, 0, polx);
        }
    } else if (threadIdx.x == 32) {
        for (int it = 0; it < tiles; ++it) {
            const int st = it % S, stb = it % SB;
            ptx::mbar_wait(&full[st], (it / S) & 1, err, 1);
            if (with_b) ptx::mbar_wait(&fullb[stb], (it / SB) & 1, err, 1);
            ptx::mbar_arrive(&empty[st]);
            if (with_b) ptx::mbar_arrive(&emptyb[stb]);
        }
    }
    __syncthreads();
}

template <int S, int SB>
float run_ab(CUtensorMap* tm, CUtensorMap* tx, int ctas, int rows_per_cta, int kblocks, int with_b, int* err) {
    const int smem = S * 128 * 128 + SB * 64 * 128 + 2 * (S + SB) * 8 + 1024;
    cudaFuncSetAttribute(stream_ab_kernel<S, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    stream_ab_kernel<S, SB><<<ctas, 96, smem>>>(*tm, *tx, rows_per_cta, kblocks, with_b, err);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) stream_ab_kernel<S, SB><<<ctas, 96, smem>>>(*tm, *tx, rows_per_cta, kblocks, with_b, err);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

template <int S>
float run(CUtensorMap* tm, int ctas, int rows_per_cta, int box_rows, int kblocks, int* err) {
    const int smem = S * box_rows * 128 + 2 * S * 8 + 1024;
    cudaFuncSetAttribute(stream_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    stream_kernel<S><<<ctas, 64, smem>>>(*tm, rows_per_cta, box_rows, kblocks, err);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) stream_kernel<S><<<ctas, 64, smem>>>(*tm, rows_per_cta, box_rows, kblocks, err);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int K = 1024;            // row length (bf16): like W1 (d = 1024)
    const int kblocks = K / 64;    // 16 boxes along K per row block
    const long rows = 1L << 16;    // 65536 rows x 2 KB = 128 MB (> L2)
    void* buf = nullptr;
    cudaMalloc(&buf, rows * K * 2);
    cudaMemset(buf, 1, rows * K * 2);
    int* err = nullptr;
    cudaMalloc(&err, 4);
    cudaMemset(err, 0, 4);
    typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<EncodeFn>(fn);
    for (int box_rows : {128, 256}) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)K * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
        cuuint32_t es[2] = {1, 1};
        if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed (box rows %d)\n", box_rows);
            continue;
        }
        for (int ctas : {sms, sms / 2}) {
            const int rows_per_cta = (int)(rows / sms) / box_rows * box_rows;
            const double bytes = (double)ctas * rows_per_cta * K * 2;
            auto report = [&](int S, float ms) {
                printf("box %3d rows  ctas %3d  stages %2d (%3d KB in flight): %7.1f GB/s  (%5.1f GB/s per SM)\n",
                       box_rows, ctas, S, S * box_rows * 128 / 1024, bytes / (ms * 1e-3) / 1e9,
                       bytes / (ms * 1e-3) / 1e9 / ctas);
            };
            if (box_rows == 128) {
                report(4, run<4>(&tm, ctas, rows_per_cta, box_rows, kblocks, err));
                report(8, run<8>(&tm, ctas, rows_per_cta, box_rows, kblocks, err));
                report(10, run<10>(&tm, ctas, rows_per_cta, box_rows, kblocks, err));
                report(12, run<12>(&tm, ctas, rows_per_cta, box_rows, kblocks, err));
            } else {
                report(5, run<5>(&tm, ctas, rows_per_cta, box_rows, kblocks, err));
                report(6, run<6>(&tm, ctas, rows_per_cta, box_rows, kblocks, err));
            }
        }
    }
    {  // weight stream with / without the token operand (dense GEMM1 pattern)
        CUtensorMap tm, tx;
        cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)K * 2};
        cuuint32_t box[2] = {64, 128};
        cuuint32_t es[2] = {1, 1};
        encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        void* xb = nullptr;
        cudaMalloc(&xb, 64 * K * 2);
        cudaMemset(xb, 2, 64 * K * 2);
        cuuint64_t xdims[2] = {(cuuint64_t)K, 64};
        cuuint32_t xbox[2] = {64, 64};
        encode(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xb, xdims, strides, xbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int rows_per_cta = (int)(rows / sms) / 128 * 128;
        const double bytes = (double)sms * rows_per_cta * K * 2;
        for (int wb = 0; wb < 2; ++wb) {
            const float m8 = run_ab<8, 10>(&tm, &tx, sms, rows_per_cta, kblocks, wb, err);
            const float m10 = run_ab<10, 10>(&tm, &tx, sms, rows_per_cta, kblocks, wb, err);
            printf("A 8 x 16 KB + B 10 x 8 KB, token operand %s: %7.1f GB/s of weights; A 10 stages: %7.1f GB/s\n",
                   wb ? "ON " : "off", bytes / (m8 * 1e-3) / 1e9, bytes / (m10 * 1e-3) / 1e9);
        }
    }
    cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
