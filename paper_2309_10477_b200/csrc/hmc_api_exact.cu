// hmc_api_exact.cu -- C ABI of the Broadie-Kaya exact scheme
// (hmc_exact_batch_f64, hmc_exact_runs_f64) and the Sobol direction-number construction
// (hmc_sobol_init_directions).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "hmc_host.h"

using namespace hmc_host;

extern "C" {

int hmc_exact_runs_f64(const hmc_model* model, double s0, const double* step_times,
                       int32_t n_steps, const int64_t* avg_flags, int64_t path_lo, int64_t path_hi,
                       const uint64_t* key_runs, int32_t n_runs, const double* uniforms,
                       const uint32_t* sobol_v, int32_t sobol_scramble, int64_t sobol_n_paths,
                       double* out, int32_t device) {
    int rc = check_model(model);
    if (rc) return rc;
    if (!(s0 > 0.0) || !std::isfinite(s0) || n_steps < 1 || !step_times || !avg_flags)
        return fail(HMC_E_INVALID, "need finite s0 > 0, n_steps >= 1, step_times and avg_flags");
    for (int k = 0; k < n_steps; ++k)
        if (!(step_times[k + 1] > step_times[k]) || !std::isfinite(step_times[k + 1]))
            return fail(HMC_E_INVALID, "step_times must be finite and increase");
    if (path_hi < path_lo) return fail(HMC_E_INVALID, "path_hi < path_lo");
    if (n_runs < 1 || !key_runs) return fail(HMC_E_INVALID, "need n_runs >= 1 and key_runs");
    if (sobol_v && uniforms) return fail(HMC_E_INVALID, "pass uniforms or sobol_v, not both");
    if (sobol_v) {
        const double blocks = sobol_scramble ? 1.0 : (double)n_runs;
        if (sobol_n_paths < path_hi || 1.0 + blocks * (double)sobol_n_paths > 1073741824.0)
            return fail(HMC_E_INVALID, "sobol index range exceeds 2^30 points (or n_paths < path_hi)");
    }
    const long long n = path_hi - path_lo;
    if (n == 0) return HMC_OK;
    const long long rows = n * n_runs;
    if (!out) return fail(HMC_E_INVALID, "out is NULL");
    long long n_dates = 0;
    for (int k = 0; k < n_steps; ++k) n_dates += avg_flags[k] ? 1 : 0;

    hmc::ExactArgs e{};
    e.kappa = model->kappa; e.theta = model->theta; e.sigma = model->sigma; e.rho = model->rho;
    e.r = model->r; e.v0 = model->v0;
    e.dof = 4.0 * model->kappa * model->theta / (model->sigma * model->sigma);  // model.py:43-45
    e.s0 = s0;
    e.n_steps = n_steps;
    e.n_dates = n_dates;
    e.path_lo = path_lo;
    e.path_hi = path_hi;
    e.n_runs = n_runs;

    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(device));
    HMC_CK(keep_pool_memory(device));
    int dev = 0, sms = 148;
    HMC_CK(cudaGetDevice(&dev));
    HMC_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int grid = 0, variant = 4;
    HMC_CK(hmc::exact_plan(rows, sms, &grid, &variant));
    const size_t threads = (size_t)grid * hmc::kExactThreads;
    cudaStream_t st;
    HMC_CK(call_stream(device, &st));
    const size_t tb = ((size_t)n_steps + 1) * sizeof(double), fb = (size_t)n_steps * sizeof(long long);
    const size_t ub = uniforms ? (size_t)rows * 3 * n_steps * sizeof(double) : 0;
    const size_t ob = (size_t)rows * 3 * sizeof(double);
    const size_t sb = (size_t)hmc::kExactCacheNodes * threads * sizeof(double);
    const size_t kb = (size_t)n_runs * sizeof(uint64_t);
    const size_t vb = sobol_v ? (size_t)30 * 3 * n_steps * sizeof(uint32_t) : 0;
    const size_t total = align_up(tb) + align_up(fb) + align_up(ub) + align_up(ob) + align_up(sb) +
                         align_up(kb) + align_up(vb) + 256;
    char* buf = nullptr;
    int h_err = 0;
    cudaError_t ce = cudaMallocAsync((void**)&buf, total, st);
    if (ce == cudaSuccess) {
        size_t off = 0;
        double* d_t = (double*)(buf + off); off += align_up(tb);
        long long* d_f = (long long*)(buf + off); off += align_up(fb);
        double* d_u = uniforms ? (double*)(buf + off) : nullptr; off += align_up(ub);
        double* d_o = (double*)(buf + off); off += align_up(ob);
        double* d_s = (double*)(buf + off); off += align_up(sb);
        unsigned long long* d_k = (unsigned long long*)(buf + off); off += align_up(kb);
        uint32_t* d_v = sobol_v ? (uint32_t*)(buf + off) : nullptr; off += align_up(vb);
        int* d_err = (int*)(buf + off);
        std::vector<long long> flags(avg_flags, avg_flags + n_steps);
        ce = cudaMemcpyAsync(d_t, step_times, tb, cudaMemcpyHostToDevice, st);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(d_f, flags.data(), fb, cudaMemcpyHostToDevice, st);
        if (ce == cudaSuccess && uniforms) ce = cudaMemcpyAsync(d_u, uniforms, ub, cudaMemcpyHostToDevice, st);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(d_k, key_runs, kb, cudaMemcpyHostToDevice, st);
        if (ce == cudaSuccess && sobol_v) ce = cudaMemcpyAsync(d_v, sobol_v, vb, cudaMemcpyHostToDevice, st);
        e.sobol_v = d_v;
        e.sobol_scramble = sobol_scramble ? 1 : 0;
        e.sobol_n_paths = sobol_n_paths;
        if (ce == cudaSuccess) ce = cudaMemsetAsync(d_err, 0, sizeof(int), st);
        e.key_runs = d_k;
        e.times = d_t;
        e.flags = d_f;
        e.uniforms = d_u;
        e.out = d_o;
        e.scratch = d_s;
        e.err_flag = d_err;
        if (ce == cudaSuccess) ce = hmc::launch_exact(e, grid, variant, st);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(out, d_o, ob, cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        cudaFreeAsync(buf, st);
    }
    cudaError_t ce2 = cudaStreamSynchronize(st);
    HMC_CK(ce);
    HMC_CK(ce2);
    switch (h_err) {  // _core.pyx:508-520
        case 0: return HMC_OK;
        case 1: return fail(HMC_E_BESSEL, "|z| exceeds the series validity bound 50");
        case 2: return fail(HMC_E_BESSEL, "Bessel series did not converge");
        case 3: return fail(HMC_E_QUAD, "characteristic-function tail did not fall below tolerance");
        default: return fail(HMC_E_ROOT, "CDF inversion failed to reach tolerance");
    }
}

int hmc_exact_batch_f64(const hmc_model* model, double s0, const double* step_times,
                        int32_t n_steps, const int64_t* avg_flags, int64_t path_lo, int64_t path_hi,
                        uint64_t key_run, const double* uniforms, double* out, int32_t device) {
    return hmc_exact_runs_f64(model, s0, step_times, n_steps, avg_flags, path_lo, path_hi, &key_run, 1,
                              uniforms, nullptr, 0, 0, out, device);
}

// Bratley-Fox / Joe-Kuo recurrence on the m-values, then the 2^(bits-1-b)
// column scaling -- the construction scipy.stats.qmc.Sobol uses for its
// unscrambled 30-bit direction numbers.
int hmc_sobol_init_directions(const int64_t* poly, const int64_t* vinit, int32_t dim, uint32_t* v_out) {
    const int bits = 30;
    if (!poly || !vinit || !v_out || dim < 1 || dim > 21201)
        return fail(HMC_E_INVALID, "bad sobol direction arguments");
    std::vector<uint64_t> row(bits);
    for (int d = 0; d < dim; ++d) {
        if (d == 0) {
            for (int b = 0; b < bits; ++b) row[b] = 1;
        } else {
            const uint64_t p = (uint64_t)poly[d];
            int m = 0;
            while ((p >> (m + 1)) != 0) ++m;  // degree = bit_length - 1
            if (m < 1 || m > 18) return fail(HMC_E_INVALID, "bad sobol polynomial");
            for (int j = 0; j < m && j < bits; ++j) row[j] = (uint64_t)vinit[(size_t)d * 18 + j];
            for (int j = m; j < bits; ++j) {
                uint64_t nv = row[j - m];
                uint64_t pow2 = 1;
                for (int k = 0; k < m; ++k) {
                    pow2 <<= 1;
                    if ((p >> (m - 1 - k)) & 1) nv ^= pow2 * row[j - k - 1];
                }
                row[j] = nv;
            }
        }
        for (int b = 0; b < bits; ++b)
            v_out[(size_t)b * dim + d] = (uint32_t)(row[b] << (bits - 1 - b));
    }
    return HMC_OK;
}
}  // extern "C"
