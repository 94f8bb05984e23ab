// hmc_launch.h -- host-side launchers implemented by the kernel TUs.
#pragma once

#include <cuda_runtime.h>

#include "hmc_device.cuh"

namespace hmc {

// fp32 production kernel (hmc_fast.cu): tiles[run][tile][HMC_NW]
cudaError_t launch_fast_greeks(const KernelArgs& a, double* d_tiles, long long n_tiles,
                               cudaStream_t s);

// fp64 replay kernels (hmc_replay.cu)
cudaError_t launch_replay_greeks(const KernelArgs& a, double* d_tiles, long long n_tiles,
                                 cudaStream_t s);
cudaError_t launch_replay_batch(const KernelArgs& a, unsigned long long key_run,
                                const double* d_uniforms, double* d_out, cudaStream_t s);

// reductions (hmc_api.cu)
cudaError_t launch_tiles_to_chunks(const double* d_tiles, long long n_tiles, int n_runs,
                                   double* d_chunks, long long n_chunks, cudaStream_t s);
cudaError_t launch_chunks_to_runs(const double* d_chunks, long long n_chunks, int n_runs,
                                  double* d_out, cudaStream_t s);

}  // namespace hmc
