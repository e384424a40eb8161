// common.cuh -- shared host/device plumbing for the exflow sm_100a library:
// status/error propagation for the C-ABI and small device helpers.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <utility>
#include <string>

#include "exflow_c.h"

#include <nvtx3/nvToolsExt.h>

namespace exf {

// NVTX range over a host entry point (header-only NVTX v3: a no-op unless a
// tool such as nsys/ncu attaches). Names are "exf.<what>"; the step phases
// carry the layer in the payload.
struct NvtxRange {
    explicit NvtxRange(const char* name, int64_t payload = -1) {
        nvtxEventAttributes_t ev{};
        ev.version = NVTX_VERSION;
        ev.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
        ev.messageType = NVTX_MESSAGE_TYPE_ASCII;
        ev.message.ascii = name;
        if (payload >= 0) {
            ev.payloadType = NVTX_PAYLOAD_TYPE_INT64;
            ev.payload.llValue = payload;
        }
        nvtxRangePushEx(&ev);
    }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Thread-local last-error message behind exf_last_error().
void set_error(const std::string& msg);
const std::string& last_error();

struct Status {
    exf_status code;
    explicit Status(exf_status c) : code(c) {}
};

// Returns EXF_INVALID with a message (reference std::invalid_argument).
inline exf_status invalid(const std::string& msg) {
    set_error(msg);
    return EXF_INVALID;
}
inline exf_status runtime_err(const std::string& msg) {
    set_error(msg);
    return EXF_RUNTIME;
}
exf_status cuda_status(cudaError_t err, const char* what);

// Per-(host thread, device) scratch of the synchronous host-buffer entry
// points (exf_count_transitions_host, exf_simulate_host): a device buffer and
// a pinned staging buffer, both grown on demand and kept, plus a non-blocking
// stream, so a decode-sized call costs no cudaMalloc/cudaFree/cudaHostAlloc.
struct HostScratch {
    uint8_t* dev = nullptr;
    size_t dev_cap = 0;
    uint8_t* pin = nullptr;
    size_t pin_cap = 0;
    cudaStream_t stream = nullptr;
    // pageable host <-> device through the pinned buffer, on `stream`
    exf_status h2d(void* d, const void* src, size_t bytes);
    exf_status d2h(void* dst, const void* d, size_t bytes);  // synchronous
};
exf_status host_scratch(size_t dev_bytes, size_t pin_bytes, HostScratch** out);

}  // namespace exf

#define EXF_CUDA_TRY(expr)                                                   \
    do {                                                                     \
        cudaError_t _e = (expr);                                             \
        if (_e != cudaSuccess) return ::exf::cuda_status(_e, #expr);         \
    } while (0)

#define EXF_TRY(expr)                                                        \
    do {                                                                     \
        exf_status _s = (expr);                                              \
        if (_s != EXF_OK) return _s;                                         \
    } while (0)

// Launch check: catches configuration errors right after a <<<>>> launch.
#define EXF_LAUNCH_CHECK(what) EXF_CUDA_TRY(cudaPeekAtLastError())

namespace exf {
// Kernel launch with programmatic dependent launch (PDL) enabled: the grid may
// start while the previous grid in the stream finishes; kernels call
// griddepcontrol.wait before consuming the previous grid's output. Optional
// thread-block cluster dimension.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, int cluster, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    int n = 0;
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
    if (cluster > 0) {
        at[n].id = cudaLaunchAttributeClusterDimension;
        at[n].val.clusterDim.x = cluster;
        at[n].val.clusterDim.y = 1;
        at[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
// One fixed L1/shared carveout (max shared) for every step kernel, so the SMs
// never reconfigure between back-to-back kernels of a decode step.
template <typename K>
inline void max_carveout(K kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
}  // namespace exf

namespace exf {

__device__ __forceinline__ int4 ld_nc_v4(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

}  // namespace exf
