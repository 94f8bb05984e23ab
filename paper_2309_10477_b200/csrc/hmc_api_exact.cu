// hmc_api_exact.cu -- C ABI of the Broadie-Kaya exact scheme
// (hmc_exact_batch_f64, hmc_exact_runs_f64) and the Sobol direction-number construction
// (hmc_sobol_init_directions).
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
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
    int dev = 0, sms = 148;
    HMC_CK(cudaGetDevice(&dev));
    HMC_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int grid = 0, variant = 1;
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
    cudaError_t ce = pool_alloc(device, (void**)&buf, total, st);
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

int hmc_exact_greeks_chunks(const hmc_model* model, const hmc_product* product, const hmc_sim* sim,
                            const double* step_times, int32_t n_steps, const int64_t* avg_flags,
                            double* d_chunks, void* stream) {
    int rc = check_model(model);
    if (rc) return rc;
    if (!product || !sim || !d_chunks) return fail(HMC_E_INVALID, "product / sim / d_chunks is NULL");
    if (!(product->strike > 0.0) || !(product->maturity > 0.0) || !(product->spot > 0.0) ||
        !std::isfinite(product->strike) || !std::isfinite(product->maturity) || !std::isfinite(product->spot))
        return fail(HMC_E_INVALID, "strike, maturity and spot must be finite and > 0");
    if (product->style != HMC_STYLE_EUROPEAN && product->style != HMC_STYLE_ASIAN)
        return fail(HMC_E_INVALID, "unknown option style");
    if (product->right != HMC_CALL && product->right != HMC_PUT) return fail(HMC_E_INVALID, "unknown option right");
    if (sim->want_greeks && product->right != HMC_CALL)
        return fail(HMC_E_UNSUPPORTED, "pathwise Greeks are derived for calls only");
    if (sim->n_runs < 1 || sim->n_paths < 1)
        return fail(HMC_E_INVALID, "need n_runs >= 1 and n_paths >= 1");
    if (sim->path_lo < 0 || sim->path_hi > sim->n_paths || sim->path_lo >= sim->path_hi ||
        sim->path_lo % HMC_CHUNK != 0)
        return fail(HMC_E_INVALID, "path slice must be chunk aligned within [0, n_paths)");
    if (sim->want_greeks && (!(sim->h_spot > 0.0 && sim->h_spot < product->spot) ||
                             !(sim->v0_up > sim->v0_dn && sim->v0_dn >= 0.0) || !(sim->h_r > 0.0) ||
                             !std::isfinite(sim->v0_up) || !std::isfinite(sim->h_r)))
        return fail(HMC_E_INVALID, "bad bump sizes");
    if (sim->sampler != HMC_SAMPLER_PSEUDO && sim->sampler != HMC_SAMPLER_SOBOL)
        return fail(HMC_E_INVALID, "unknown sampler");
    if (!step_times || !avg_flags || n_steps < 1) return fail(HMC_E_INVALID, "need step_times and avg_flags");
    for (int k = 0; k < n_steps; ++k)
        if (!(step_times[k + 1] > step_times[k]) || !std::isfinite(step_times[k + 1]))
            return fail(HMC_E_INVALID, "step_times must be finite and increase");
    const bool sob = sim->sampler == HMC_SAMPLER_SOBOL;
    if (sob) {
        if (!sim->sobol_v) return fail(HMC_E_INVALID, "sobol sampler needs direction numbers");
        const double blocks = sim->sobol_scramble ? 1.0 : (double)sim->n_runs;
        if (1.0 + blocks * (double)sim->n_paths > 1073741824.0)
            return fail(HMC_E_INVALID, "sobol index range exceeds 2^30 points");
    }
    const long long n = sim->path_hi - sim->path_lo, R = sim->n_runs;
    long long n_dates = 0;
    for (int k = 0; k < n_steps; ++k) n_dates += avg_flags[k] ? 1 : 0;
    const bool asian = product->style == HMC_STYLE_ASIAN, greeks = sim->want_greeks != 0;
    const double T = product->maturity, r = model->r;

    // model variants simulated on the same streams: base, v0 +-.  The r +- h_r
    // underlyings are the base paths rescaled (exact_estimator_kernel): the
    // base run of an Asian carries sum S_k expm1(+-h_r t_k) as two more columns
    hmc_model var[3] = {*model, *model, *model};
    var[1].v0 = sim->v0_up;
    var[2].v0 = sim->v0_dn;
    const int n_var = greeks ? 3 : 1;
    const bool rcols = greeks && asian;

    // epilogue arguments (hmc_device.cuh greeks_epilogue)
    KernelArgs a{};
    a.K = product->strike;
    a.s0 = product->spot;
    a.T = T;
    a.r = r;
    a.disc = std::exp(-r * T);
    a.h_spot = greeks ? sim->h_spot : 0.0;
    a.h_r = greeks ? sim->h_r : 0.0;
    a.v0_up = greeks ? sim->v0_up : model->v0;
    a.v0_dn = greeks ? sim->v0_dn : model->v0;
    a.disc_up = std::exp(-(r + a.h_r) * T);
    a.disc_dn = std::exp(-(r - a.h_r) * T);
    a.is_asian = asian;
    a.is_call = product->right == HMC_CALL;
    a.want_greeks = greeks;

    std::vector<unsigned long long> keys((size_t)R);
    const unsigned long long root = hmc::mix64(sim->seed ^ 0x8CB92BA72F3D8DD7ULL);  // rng.py:46-47
    for (long long q = 0; q < R; ++q) keys[(size_t)q] = hmc::derive(root, (unsigned long long)q);

    int dev = 0, sms = 148;
    HMC_CK(cudaGetDevice(&dev));
    HMC_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // runs go through in batches so the observables of all variants stay
    // within ~2 GB of device memory
    const long long per_run = n * (long long)sizeof(double) * (3 * n_var + (rcols ? 2 : 0));
    const long long batch = std::max(1LL, std::min({R, (long long)hmc::kMaxRunsPerLaunch,
                                                     (2LL << 30) / std::max(per_run, 1LL)}));
    int grid = 0, variant = 1;
    HMC_CK(hmc::exact_plan(n * batch, sms, &grid, &variant));
    const long long n_tiles = n_tiles_of(n), n_chunks = n_chunks_of(n);
    const size_t tb = ((size_t)n_steps + 1) * sizeof(double), fb = (size_t)n_steps * sizeof(long long);
    const size_t kb = (size_t)R * sizeof(uint64_t);
    const size_t vb = sob && !sim->sobol_v_on_device ? (size_t)30 * 3 * n_steps * sizeof(uint32_t) : 0;
    const size_t sb = (size_t)hmc::kExactCacheNodes * grid * hmc::kExactThreads * sizeof(double);
    const size_t ob = (size_t)batch * n * 3 * sizeof(double);
    const size_t ob0 = (size_t)batch * n * (rcols ? 5 : 3) * sizeof(double);
    const size_t eb = rcols ? ((size_t)n_steps + 1) * 2 * sizeof(double) : 0;
    const size_t lb = (size_t)R * n_tiles * HMC_NW * sizeof(double);
    const size_t total = align_up(tb) + align_up(fb) + align_up(kb) + align_up(vb) + align_up(sb) +
                         align_up(ob0) + (n_var - 1) * align_up(ob) + align_up(eb) + align_up(lb) + 256;
    cudaStream_t st = (cudaStream_t)stream;
    char* buf = nullptr;
    HMC_CK(pool_alloc(dev, (void**)&buf, total, st));
    size_t off = 0;
    auto take = [&](size_t bytes) { char* p = buf + off; off += align_up(bytes); return p; };
    double* d_t = (double*)take(tb);
    long long* d_f = (long long*)take(fb);
    unsigned long long* d_k = (unsigned long long*)take(kb);
    uint32_t* d_v = vb ? (uint32_t*)take(vb) : nullptr;
    double* d_s = (double*)take(sb);
    double* d_obs[3] = {nullptr, nullptr, nullptr};
    for (int v = 0; v < n_var; ++v) d_obs[v] = (double*)take(v == 0 ? ob0 : ob);
    double* d_e = eb ? (double*)take(eb) : nullptr;
    std::vector<double> em(rcols ? 2 * ((size_t)n_steps + 1) : 0);
    for (size_t k = 0; rcols && k <= (size_t)n_steps; ++k) {
        em[2 * k] = std::expm1(sim->h_r * step_times[k]);
        em[2 * k + 1] = std::expm1(-sim->h_r * step_times[k]);
    }
    double* d_tiles = (double*)take(lb);
    int* d_err = (int*)(buf + off);
    std::vector<long long> flags(avg_flags, avg_flags + n_steps);
    cudaError_t ce = cudaMemcpyAsync(d_t, step_times, tb, cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(d_f, flags.data(), fb, cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(d_k, keys.data(), kb, cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess && vb) ce = cudaMemcpyAsync(d_v, sim->sobol_v, vb, cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess && eb) ce = cudaMemcpyAsync(d_e, em.data(), eb, cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(d_err, 0, sizeof(int), st);
    for (long long r0 = 0; ce == cudaSuccess && r0 < R; r0 += batch) {
        const int nb = (int)std::min(batch, R - r0);
        for (int v = 0; v < n_var && ce == cudaSuccess; ++v) {
            hmc::ExactArgs e{};
            e.kappa = var[v].kappa; e.theta = var[v].theta; e.sigma = var[v].sigma; e.rho = var[v].rho;
            e.r = var[v].r; e.v0 = var[v].v0;
            e.dof = 4.0 * var[v].kappa * var[v].theta / (var[v].sigma * var[v].sigma);  // model.py:43-45
            e.s0 = product->spot;
            e.n_steps = n_steps;
            e.n_dates = n_dates;
            e.path_lo = sim->path_lo;
            e.path_hi = sim->path_hi;
            e.key_runs = d_k + r0;
            e.n_runs = nb;
            e.run_offset = (int)r0;
            e.times = d_t;
            e.flags = d_f;
            e.sobol_v = sob ? (sim->sobol_v_on_device ? sim->sobol_v : d_v) : nullptr;
            e.sobol_scramble = sim->sobol_scramble ? 1 : 0;
            e.sobol_n_paths = sim->n_paths;
            e.out = d_obs[v];
            e.rbump = v == 0 ? d_e : nullptr;
            e.scratch = d_s;
            e.err_flag = d_err;
            ce = hmc::launch_exact(e, grid, variant, st);
        }
        if (ce == cudaSuccess)
            ce = hmc::launch_exact_estimators(a, d_obs, n, nb, std::exp(a.h_r * T), std::exp(-a.h_r * T),
                                              d_tiles, n_tiles, (int)r0, st);
    }
    if (ce == cudaSuccess) ce = hmc::launch_tiles_to_chunks(d_tiles, n_tiles, (int)R, d_chunks, n_chunks, st);
    int h_err = 0;
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(buf, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);  // error codes need the kernels done
    HMC_CK(ce);
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
