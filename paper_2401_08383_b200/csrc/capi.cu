// capi.cu -- C-ABI error plumbing and device probing.
#include "common.cuh"

#include <cstring>
#include <string>

namespace exf {

namespace {
thread_local std::string t_last_error;
constexpr int kMaxDevices = 16;
constexpr size_t kPinChunk = 8u << 20;
// grown on demand, never shrunk; freed with the process (a thread-exit
// destructor could run after the CUDA context is gone)
thread_local HostScratch t_scratch[kMaxDevices];
}

exf_status host_scratch(size_t dev_bytes, size_t pin_bytes, HostScratch** out) {
    int dev = 0;
    EXF_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDevices) return runtime_err("device ordinal out of range");
    HostScratch& h = t_scratch[dev];
    if (!h.stream) EXF_CUDA_TRY(cudaStreamCreateWithFlags(&h.stream, cudaStreamNonBlocking));
    if (dev_bytes > h.dev_cap) {
        const size_t cap = std::max(dev_bytes, h.dev_cap * 2);
        if (h.dev) cudaFree(h.dev);
        h.dev = nullptr;
        h.dev_cap = 0;
        EXF_CUDA_TRY(cudaMalloc(&h.dev, cap));
        h.dev_cap = cap;
    }
    pin_bytes = std::min<size_t>(pin_bytes, kPinChunk);  // larger copies go in chunks
    if (pin_bytes > h.pin_cap) {
        if (h.pin) cudaFreeHost(h.pin);
        h.pin = nullptr;
        h.pin_cap = 0;
        const size_t cap = std::max<size_t>(pin_bytes, 1 << 16);
        EXF_CUDA_TRY(cudaHostAlloc(&h.pin, cap, cudaHostAllocDefault));
        h.pin_cap = cap;
    }
    *out = &h;
    return EXF_OK;
}

exf_status HostScratch::h2d(void* d, const void* src, size_t bytes) {
    // through the pinned staging buffer in chunks (one DMA per chunk, the
    // next chunk's host copy overlapping nothing: calls are synchronous)
    const uint8_t* p = static_cast<const uint8_t*>(src);
    uint8_t* q = static_cast<uint8_t*>(d);
    for (size_t o = 0; o < bytes; o += pin_cap) {
        const size_t n = std::min(pin_cap, bytes - o);
        EXF_CUDA_TRY(cudaStreamSynchronize(stream));  // staging buffer free again
        std::memcpy(pin, p + o, n);
        EXF_CUDA_TRY(cudaMemcpyAsync(q + o, pin, n, cudaMemcpyHostToDevice, stream));
    }
    return EXF_OK;
}

exf_status HostScratch::d2h(void* dst, const void* d, size_t bytes) {
    uint8_t* p = static_cast<uint8_t*>(dst);
    const uint8_t* q = static_cast<const uint8_t*>(d);
    for (size_t o = 0; o < bytes; o += pin_cap) {
        const size_t n = std::min(pin_cap, bytes - o);
        EXF_CUDA_TRY(cudaMemcpyAsync(pin, q + o, n, cudaMemcpyDeviceToHost, stream));
        EXF_CUDA_TRY(cudaStreamSynchronize(stream));
        std::memcpy(p + o, pin, n);
    }
    return EXF_OK;
}

void set_error(const std::string& msg) { t_last_error = msg; }
const std::string& last_error() { return t_last_error; }

exf_status cuda_status(cudaError_t err, const char* what) {
    set_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorName(err) + ": " +
              cudaGetErrorString(err));
    return EXF_CUDA;
}

}  // namespace exf

extern "C" const char* exf_last_error(void) { return exf::last_error().c_str(); }

extern "C" int32_t exf_version(void) { return 100; }

extern "C" int32_t exf_device_ok(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return 0;
    }
    int dev = 0, major = 0, minor = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return (major == 10 && minor == 0) ? 1 : 0;
}
