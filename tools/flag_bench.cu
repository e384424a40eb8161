// flag_bench.cu -- diagnostics: latency of a grid-wide flag barrier across
// 148 co-resident CTAs (each CTA release-stores its epoch slot, then threads
// poll all slots), idle GPU, several publish/poll variants.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I../paper_2401_08383_b200/csrc flag_bench.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"

using namespace exf;

template <int MODE>
__global__ void __launch_bounds__(256, 1) barrier_kernel(uint64_t* slots, int rounds, uint64_t base, long long* out) {
    __shared__ uint64_t pad[20000];  // one CTA per SM, like the fused kernel
    if (threadIdx.x == 0) pad[0] = 0;
    const long long t0 = clock64();
    for (int r = 1; r <= rounds; ++r) {
        const uint64_t ep = base + r;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) {
            if (MODE == 2)
                asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(slots + blockIdx.x), "l"(ep) : "memory");
            else
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(slots + blockIdx.x), "l"(ep) : "memory");
        }
        if (MODE >= 3) {  // one warp polls every slot, coalesced, optional back-off
            if (threadIdx.x < 32) {
                for (int c = threadIdx.x; c < (int)gridDim.x; c += 32) {
                    while (ptx::ld_relaxed_u64(slots + c, false) < ep) {
                        if (MODE == 4) __nanosleep(32);
                    }
                }
                ptx::fence_acquire(false);
            }
        } else if (threadIdx.x < gridDim.x) {
            if (MODE == 0) {
                uint64_t v;
                do {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(slots + threadIdx.x) : "memory");
                } while (v < ep);
            } else {
                while (ptx::ld_relaxed_u64(slots + threadIdx.x, false) < ep) {
                }
                ptx::fence_acquire(false);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = clock64() - t0;
}

template <int MODE>
void run(const char* name, uint64_t* slots, long long* d_out, int sms, uint64_t& base) {
    const int rounds = 2000;
    barrier_kernel<MODE><<<sms, 256>>>(slots, rounds, base, d_out);
    base += rounds;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    barrier_kernel<MODE><<<sms, 256>>>(slots, rounds, base, d_out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    base += rounds;
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-48s %.3f us per barrier\n", name, ms * 1e3 / rounds);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint64_t* slots = nullptr;
    long long* d_out = nullptr;
    cudaMalloc(&slots, 256 * 8);
    cudaMemset(slots, 0, 256 * 8);
    cudaMalloc(&d_out, 8);
    uint64_t base = 0;
    run<0>("st.release + ld.acquire poll", slots, d_out, sms, base);
    run<1>("st.release + relaxed poll + fence", slots, d_out, sms, base);
    run<2>("st.relaxed + relaxed poll + fence", slots, d_out, sms, base);
    run<3>("st.release + one polling warp per CTA", slots, d_out, sms, base);
    run<4>("st.release + one polling warp, nanosleep(32)", slots, d_out, sms, base);
    cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
