// capi.cu -- C-ABI error plumbing and device probing.
#include "common.cuh"

#include <string>

namespace exf {

namespace {
thread_local std::string t_last_error;
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
