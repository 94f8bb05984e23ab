// hmc_launch.h -- host-side launchers implemented by the kernel TUs.
#pragma once

#include <cuda_runtime.h>

#include "hmc_device.cuh"

namespace hmc {

// ---- strike x maturity surface (hmc_surface.cu) ---------------------------
#ifndef HMC_SURF_THREADS
#define HMC_SURF_THREADS 1024
#endif
#ifndef HMC_SURF_MINB
#define HMC_SURF_MINB 1
#endif
constexpr int kSurfThreads = HMC_SURF_THREADS;  // paths per tile (one block)
constexpr int kSurfMinBlocks = HMC_SURF_MINB;   // resident blocks per SM
constexpr int kSurfMaxStrikes = HMC_SURF_MAX_STRIKES;
constexpr int kSurfMaxMats = HMC_SURF_MAX_MATS;
// Per (style, maturity): kSurfVals rows of nK + 1 columns.
// Rows 0..14 are bucketed moments, column = strike bucket c(x) = #{K_j < x};
// a strike's sum over {x > K_j} is the suffix sum over columns > j:
//    0 sum A    (key A(1+e))   1 sum A^2   (key A(1+e))
//    2 N        (key A)        3 sum A      4 sum A^2     5 sum w   6 sum w^2   (w = tw - T A)
//    7 N        (key A(1-e))   8 sum A      9 sum A^2
//   10 sum g    (key min(Au, Ad), g = d (Au - Ad)/dv)   11 sum g^2
//   12 N        (key Rm)      13 sum a     14 sum a^2  (a = (d+ Rp - d- Rm)/2h_r)
// Rows 15..22 are per-STRIKE band moments (column = strike j), added for
// every strike a path's bumped pair straddles -- the only regions where a
// finite difference is not a K-free or K-linear function of the path:
//   15/16 sum x, x^2, x = A(1+e) - K_j,  A(1-e) <= K_j < A(1+e)   (FD delta)
//   17/18 sum x, x^2, x = Au - K_j,      Ad <= K_j < Au           (vega)
//   19/20 sum x, x^2, x = Ad - K_j,      Au <= K_j < Ad           (vega)
//   21/22 sum x, x^2, x = Rp - K_j,      Rm <= K_j < Rp           (FD rho)
constexpr int kSurfVals = 23;
constexpr int kSurfBucketRows = 15;
constexpr float kSurfLinScale = 1024.0f;      // 2^10 fixed point for linear moments
constexpr float kSurfQuadScale = 4.0f;        // 2^2 for quadratic moments (A^2 >= 2^18 escapes to int64)
constexpr float kSurfBandScale = 1048576.0f;  // 2^20 for the (small, <= ~1) band moments

struct SurfMat {
    int step;      // grid index of the maturity
    float inv_n;   // 1 / step (daily-average weight)
    float T;       // t_step
    float ehp, ehm;  // e^{+h_r T}, e^{-h_r T}
    float d, dp, dm; // e^{-r T}, e^{-(r +- h_r) T}
    float ddisc;     // dp - dm formed in fp64 (rounding dp and dm separately
                     // and subtracting biases the Asian FD Rho by ~3e-5)
};

struct SurfArgs {
    const float* strikes;
    int nK;
    const SurfMat* mats;
    int n_mats;
    unsigned long long* acc;  // [run][2][n_mats][kSurfVals][nK + 1] int64 fixed point
    float eps_up, eps_dn;     // 1 +- h_spot / S0
    float inv_dv;             // 1 / (v0_up - v0_dn)
    int uniform;              // strikes equally spaced: k0 + j / inv_dk
    float k0, inv_dk;
    float inv_2hr;            // 1 / (2 h_r)
};

cudaError_t launch_surface(const KernelArgs& a, const SurfArgs& s, long long n_tiles, int grid_x,
                           cudaStream_t stream);

// ---- Broadie-Kaya exact simulation (hmc_exact.cu) --------------------------
constexpr int kExactThreads = 128;
constexpr int kExactCacheNodes = 256;  // Re Phi nodes cached per thread (rest recomputed)

struct ExactArgs {
    double kappa, theta, sigma, rho, r, v0, dof, s0;
    const double* times;     // [n_steps + 1] step endpoints, times[0] = 0
    const long long* flags;  // [n_steps] 1 if the step's end is an averaging date
    int n_steps;
    long long n_dates;
    long long path_lo, path_hi;
    const unsigned long long* key_runs;  // [n_runs] per-run stream keys (device)
    int n_runs;
    int run_offset;          // global index of run 0 of this launch (Sobol blocks)
    const double* uniforms;  // [n_runs][n][3 n_steps] or null
    const uint32_t* sobol_v; // [30][3 n_steps] Sobol direction numbers (device) or null
    int sobol_scramble;      // digital shifts per (run, dimension)
    long long sobol_n_paths; // N of the run blocks 1 + run N + path
    double* out;             // [n_runs][n][3], or [n_runs][n][5] with rbump
    const double* rbump;     // [n_steps + 1][2] expm1(+-h_r t_k), or null: the r +- h_r
                             // averages as extra columns (see exact_batch_kernel)
    double* scratch;         // [kExactCacheNodes][grid threads]
    int* err_flag;           // max reference error code seen
};

// grid (one resident wave, grid-stride) and register variant for `rows`
// (run, path) pairs; the node cache is sized by grid * kExactThreads
cudaError_t exact_plan(long long rows, int sms, int* grid, int* variant);
cudaError_t launch_exact(const ExactArgs& e, int grid, int variant, cudaStream_t s);
// per-path exact-scheme estimators -> tiles[run0 + run][tile][HMC_NW]
cudaError_t launch_exact_estimators(const KernelArgs& a, const double* const obs[3], long long n, int n_runs,
                                    double ehT, double emhT, double* tiles, long long n_tiles, int run0,
                                    cudaStream_t s);

// the production step arithmetic on given normals (hmc_fast.cu), per path
cudaError_t launch_given_normals(const KernelArgs& a, const float2* d_z, long long n, double* d_out,
                                 cudaStream_t s);

// fp32 production kernel (hmc_fast.cu): tiles[run][tile][HMC_NW]
cudaError_t launch_fast_greeks(const KernelArgs& a, double* d_tiles, long long n_tiles,
                               cudaStream_t s);

// fp64 replay kernels (hmc_replay.cu)
cudaError_t launch_replay_greeks(const KernelArgs& a, double* d_tiles, long long n_tiles,
                                 cudaStream_t s);
// elementwise reference primitives (hmc_replay.cu): uniform_at, ndtri, one step
cudaError_t launch_uniforms(const unsigned long long* d_keys, long long n_keys,
                            const unsigned long long* d_draws, long long n, double* d_out, cudaStream_t s);
cudaError_t launch_ndtri(const double* d_u, long long n, double* d_out, cudaStream_t s);
// Marsaglia-Tsang Gamma on the reference stream (hmc_exact.cu)
// the reference's exact-scheme host modules on the device (hmc_exact.cu)
cudaError_t launch_bessel(int mode, double nu, const double* d_z, const double* d_aux, long long n, double* d_out,
                          int* d_err, cudaStream_t s);
cudaError_t launch_ivlaw_phi(double kappa, double sigma, double dof, double v_u, double v_t, double dt,
                             const double* d_a, long long n, double* d_out, int* d_err, cudaStream_t s);
cudaError_t launch_ivlaw_eval(int mode, double kappa, double theta, double sigma, double dof, double v_u,
                              double v_t, double dt, const double* d_in, long long n, double* d_out, double* d_info,
                              double* d_scratch, int* d_err, cudaStream_t s);
cudaError_t launch_exact_step(int full, const hmc_model& m, double s_u, double v_u, double dt, const double* d_draws,
                              long long n, double* d_out, double* d_scratch, int* d_err, cudaStream_t s);
cudaError_t launch_gamma(const unsigned long long* d_keys, const unsigned long long* d_start, long long n,
                         double shape, double scale, double* d_out, unsigned long long* d_used, cudaStream_t s);
cudaError_t launch_steps(const KernelArgs& a, const double* d_s, const double* d_v, const double* d_u,
                         long long n, double* d_s_out, double* d_v_out, cudaStream_t s);
cudaError_t launch_replay_batch(const KernelArgs& a, unsigned long long key_run,
                                const double* d_uniforms, double* d_out, cudaStream_t s);

// reductions (hmc_api.cu)
cudaError_t launch_tiles_to_chunks(const double* d_tiles, long long n_tiles, int n_runs,
                                   double* d_chunks, long long n_chunks, cudaStream_t s);
cudaError_t launch_chunks_to_runs(const double* d_chunks, long long n_chunks, int n_runs,
                                  double* d_out, cudaStream_t s);

}  // namespace hmc
