// hmc_host.h -- host-side pieces shared by the C-ABI translation units
// (hmc_api.cu, hmc_api_surface.cu, hmc_api_exact.cu): the thread-local
// error string, the CUDA-error macro, workspace alignment and the per-call
// preparation of the kernel arguments and step tables.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "hmc_device.cuh"
#include "hmc_launch.h"
#include "hmc_path32.cuh"

namespace hmc_host {

using hmc::KernelArgs;
using hmc::StepD;

extern thread_local std::string g_err;  // hmc_last_error()

int fail(int code, const std::string& msg);

#define HMC_CK(expr)                                                                  \
    do {                                                                              \
        cudaError_t e_ = (expr);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return fail(e_ == cudaErrorNoDevice || e_ == cudaErrorInsufficientDriver  \
                            ? HMC_E_NODEVICE                                          \
                            : HMC_E_CUDA,                                             \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));          \
    } while (0)

// The one-call entry points select their device; restore the caller's
// current device on return (a library call must not move it).
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            prev = -1;
            cudaGetLastError();
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// The one-call entry points run on a per-thread, per-device non-blocking
// stream created on first use and destroyed at thread exit (creating and
// destroying a stream per call costs more than a small job's kernel).
cudaError_t call_stream(int device, cudaStream_t* out);

// stream-ordered allocation from libhmc's private per-device pool (hmc_api.cu);
// release with cudaFreeAsync
cudaError_t pool_alloc(int dev, void** p, size_t bytes, cudaStream_t s);

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
inline long long n_tiles_of(long long n) { return (n + HMC_TILE - 1) / HMC_TILE; }
inline long long n_chunks_of(long long n) { return (n + HMC_CHUNK - 1) / HMC_CHUNK; }

struct Prepared {
    KernelArgs a{};
    std::vector<StepD> st64;
    std::vector<float4> st32;
    std::vector<hmc::BridgeNodeD> bn64;
    std::vector<hmc::BridgeStepD> bs64;
    std::vector<hmc::BridgeNode> bn32;
    std::vector<hmc::BridgeStep> bs32;
    long long n_tiles = 0, n_chunks = 0;
    size_t off_st64 = 0, off_st32 = 0, off_sobol = 0, off_bridge = 0, bytes = 0;
};

int check_model(const hmc_model* m);

// validate one single-product job and build its arguments and tables
int prepare(const hmc_model* m, const hmc_product* pr, const hmc_sim* sim, Prepared& P);
// workspace bytes of the Brownian-bridge tables
size_t bridge_bytes(int S, int n_steps);

}  // namespace hmc_host
