// hmc_api_surface.cu -- C ABI of the strike x maturity surface
// (include/hmc.h hmc_surface*): spec validation, per-call tables, the
// kernel launch and the host finalisation (suffix sums of the bucketed
// fixed-point moments -> per-strike {sum, sum of squares}).
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "hmc_host.h"

using namespace hmc_host;

namespace {

struct SurfPrepared {
    Prepared P;                    // single-product args: asian call, fixings 1..n
    std::vector<int64_t> fix_idx;  // 1..n_steps
    std::vector<float> strikes;
    std::vector<hmc::SurfMat> mats;
    hmc::SurfArgs s{};
    size_t off_st64 = 0, off_st32 = 0, off_k = 0, off_m = 0, off_sobol = 0, bytes = 0;
};

int check_surface_spec(const hmc_surface_spec* sp, const hmc_sim* sim) {
    if (!sp || !sim) return fail(HMC_E_INVALID, "surface spec / sim is NULL");
    if (!(sp->spot > 0.0) || !(sp->dt > 0.0) || !std::isfinite(sp->spot) || !std::isfinite(sp->dt))
        return fail(HMC_E_INVALID, "need finite spot > 0 and dt > 0");
    if (!sp->strikes || sp->n_strikes < 1 || sp->n_strikes > HMC_SURF_MAX_STRIKES)
        return fail(HMC_E_INVALID, "need 1..HMC_SURF_MAX_STRIKES strikes");
    for (int j = 0; j < sp->n_strikes; ++j)
        if (!(sp->strikes[j] > 0.0) || !std::isfinite(sp->strikes[j]) ||
            (j > 0 && !(sp->strikes[j] > sp->strikes[j - 1])))
            return fail(HMC_E_INVALID, "strikes must be positive and strictly increasing");
    if (!sp->mat_idx || sp->n_mats < 1 || sp->n_mats > HMC_SURF_MAX_MATS)
        return fail(HMC_E_INVALID, "need 1..HMC_SURF_MAX_MATS maturities");
    for (int m = 0; m < sp->n_mats; ++m)
        if (sp->mat_idx[m] < 1 || (m > 0 && sp->mat_idx[m] <= sp->mat_idx[m - 1]))
            return fail(HMC_E_INVALID, "maturity grid indices must be >= 1 and strictly increasing");
    if (sim->n_steps != sp->mat_idx[sp->n_mats - 1])
        return fail(HMC_E_INVALID, "sim->n_steps must equal the last maturity's grid index");
    if (sim->precision != HMC_PREC_FP32)
        return fail(HMC_E_UNSUPPORTED, "surfaces run on the fp32 path (pseudo or Sobol)");
    if (sim->sobol_bridge != 0)
        return fail(HMC_E_UNSUPPORTED, "surfaces take time-ordered Sobol dimensions (no bridge)");
    return HMC_OK;
}

int prepare_surface(const hmc_model* m, const hmc_surface_spec* sp, const hmc_sim* sim_in,
                    SurfPrepared& S) {
    int rc = check_surface_spec(sp, sim_in);
    if (rc) return rc;
    hmc_sim sim = *sim_in;
    sim.want_greeks = 1;
    S.fix_idx.resize((size_t)sim.n_steps);
    for (int k = 0; k < sim.n_steps; ++k) S.fix_idx[k] = k + 1;
    hmc_product pr{};
    pr.style = HMC_STYLE_ASIAN;
    pr.right = HMC_CALL;
    pr.strike = sp->strikes[0];
    pr.maturity = sp->dt * sim.n_steps;
    pr.spot = sp->spot;
    pr.avg_idx = S.fix_idx.data();
    pr.n_avg = sim.n_steps;
    rc = prepare(m, &pr, &sim, S.P);
    if (rc) return rc;
    const KernelArgs& a = S.P.a;
    S.strikes.assign(sp->strikes, sp->strikes + sp->n_strikes);
    for (int k = 0; k < sp->n_mats; ++k) {
        const int step = (int)sp->mat_idx[k];
        const double T = S.P.st64[step].t;
        const double dp = std::exp(-(a.r + a.h_r) * T), dm = std::exp(-(a.r - a.h_r) * T);
        S.mats.push_back({step, (float)(1.0 / step), (float)T, (float)std::exp(a.h_r * T),
                          (float)std::exp(-a.h_r * T), (float)std::exp(-a.r * T), (float)dp, (float)dm,
                          (float)(dp - dm)});
    }
    S.s.nK = sp->n_strikes;
    S.s.n_mats = sp->n_mats;
    S.s.eps_up = (float)(1.0 + a.h_spot / a.s0);
    S.s.eps_dn = (float)(1.0 - a.h_spot / a.s0);
    S.s.inv_dv = (float)(1.0 / (a.v0_up - a.v0_dn));
    S.s.uniform = 0;
    if (sp->n_strikes >= 2) {
        const double k0 = sp->strikes[0], dk = (sp->strikes[sp->n_strikes - 1] - k0) / (sp->n_strikes - 1);
        bool uni = dk > 0.0;
        for (int j = 0; j < sp->n_strikes && uni; ++j)
            uni = std::fabs(sp->strikes[j] - (k0 + j * dk)) <= 1e-9 * std::fabs(sp->strikes[j]);
        if (uni) {
            S.s.uniform = 1;
            S.s.k0 = (float)k0;
            S.s.inv_dk = (float)(1.0 / dk);
        }
    }
    S.s.inv_2hr = (float)(0.5 / a.h_r);
    size_t off = 0;
    S.off_st64 = off;
    off += align_up(S.P.st64.size() * sizeof(StepD));
    S.off_st32 = off;
    off += align_up(S.P.st32.size() * sizeof(float4));
    S.off_k = off;
    off += align_up(S.strikes.size() * sizeof(float));
    S.off_m = off;
    off += align_up(S.mats.size() * sizeof(hmc::SurfMat));
    S.off_sobol = off;
    if (sim.sampler == HMC_SAMPLER_SOBOL && !sim.sobol_v_on_device)
        off += align_up((size_t)30 * 2 * sim.n_steps * sizeof(uint32_t));
    S.bytes = off;
    return HMC_OK;
}

double suffix(const std::vector<double>& col, int nb, int from) {
    double acc = 0.0;
    for (int c = nb - 1; c >= from; --c) acc += col[c];
    return acc;
}

}  // namespace

extern "C" {

int64_t hmc_surface_acc_words(const hmc_surface_spec* spec, int32_t n_runs) {
    if (!spec || n_runs < 1) return 0;
    return (int64_t)n_runs * 2 * spec->n_mats * HMC_SURF_VALS * (spec->n_strikes + 1);
}

int64_t hmc_surface_workspace_bytes(const hmc_surface_spec* spec, const hmc_sim* sim) {
    if (!spec || !sim || sim->n_steps < 1) return 0;
    size_t b = align_up(((size_t)sim->n_steps + 1) * sizeof(StepD)) +
               align_up(((size_t)sim->n_steps + 1) * sizeof(float4)) +
               align_up((size_t)spec->n_strikes * sizeof(float)) +
               align_up((size_t)spec->n_mats * sizeof(hmc::SurfMat));
    if (sim->sampler == HMC_SAMPLER_SOBOL && !sim->sobol_v_on_device)
        b += align_up((size_t)30 * 2 * sim->n_steps * sizeof(uint32_t));
    return (int64_t)b;
}

int hmc_surface_partials(const hmc_model* model, const hmc_surface_spec* spec, const hmc_sim* sim,
                         int64_t* d_acc, void* d_work, void* stream) {
    SurfPrepared S;
    int rc = prepare_surface(model, spec, sim, S);
    if (rc) return rc;
    if (!d_acc || !d_work) return fail(HMC_E_INVALID, "d_acc / d_work is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    char* w = (char*)d_work;
    HMC_CK(cudaMemcpyAsync(w + S.off_st64, S.P.st64.data(), S.P.st64.size() * sizeof(StepD),
                           cudaMemcpyHostToDevice, st));
    HMC_CK(cudaMemcpyAsync(w + S.off_st32, S.P.st32.data(), S.P.st32.size() * sizeof(float4),
                           cudaMemcpyHostToDevice, st));
    HMC_CK(cudaMemcpyAsync(w + S.off_k, S.strikes.data(), S.strikes.size() * sizeof(float),
                           cudaMemcpyHostToDevice, st));
    HMC_CK(cudaMemcpyAsync(w + S.off_m, S.mats.data(), S.mats.size() * sizeof(hmc::SurfMat),
                           cudaMemcpyHostToDevice, st));
    S.P.a.steps64 = (const StepD*)(w + S.off_st64);
    S.P.a.steps32 = (const float4*)(w + S.off_st32);
    S.s.strikes = (const float*)(w + S.off_k);
    S.s.mats = (const hmc::SurfMat*)(w + S.off_m);
    S.s.acc = (unsigned long long*)d_acc;
    if (sim->sampler == HMC_SAMPLER_SOBOL) {
        if (sim->sobol_v_on_device) {
            S.P.a.sobol_v = sim->sobol_v;
        } else {
            HMC_CK(cudaMemcpyAsync(w + S.off_sobol, sim->sobol_v, (size_t)30 * S.P.a.sobol_dim * sizeof(uint32_t),
                                   cudaMemcpyHostToDevice, st));
            S.P.a.sobol_v = (const uint32_t*)(w + S.off_sobol);
        }
    }
    const long long n_tiles = (sim->path_hi - sim->path_lo + hmc::kSurfThreads - 1) / hmc::kSurfThreads;
    int dev = 0, sms = 148;
    HMC_CK(cudaGetDevice(&dev));
    HMC_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const long long slots = (long long)sms * hmc::kSurfMinBlocks;
    const int grid_x = (int)(n_tiles < slots ? n_tiles : slots);
    HMC_CK(hmc::launch_surface(S.P.a, S.s, n_tiles, grid_x, st));
    return HMC_OK;
}

int hmc_surface_finalize(const hmc_model* model, const hmc_surface_spec* spec, const hmc_sim* sim,
                         const int64_t* h_acc, double* out) {
    SurfPrepared S;
    int rc = prepare_surface(model, spec, sim, S);
    if (rc) return rc;
    if (!h_acc || !out) return fail(HMC_E_INVALID, "h_acc / out is NULL");
    const KernelArgs& a = S.P.a;
    const int nK = spec->n_strikes, nb = nK + 1, V = HMC_SURF_VALS;
    // row kind: 0 count, 1 linear, 2 quadratic, 3 band (layout: hmc_launch.h)
    static const int kind[HMC_SURF_VALS] = {1, 2, 0, 1, 2, 1, 2, 0, 1, 2, 1, 2, 0, 1, 2,
                                            3, 3, 3, 3, 3, 3, 3, 3};
    const double inv_scale[4] = {1.0, 1.0 / hmc::kSurfLinScale, 1.0 / hmc::kSurfQuadScale,
                                 1.0 / hmc::kSurfBandScale};
    const double S0 = a.s0, h = a.h_spot, hr = a.h_r, dv = a.v0_up - a.v0_dn;
    const int R = hmc::kSurfBucketRows;
    std::vector<std::vector<double>> col(V, std::vector<double>(nb));
    for (int run = 0; run < sim->n_runs; ++run)
        for (int style = 0; style < 2; ++style)
            for (int mi = 0; mi < spec->n_mats; ++mi) {
                const int64_t* hst = h_acc + (((size_t)run * 2 + style) * spec->n_mats + mi) * V * nb;
                for (int v = 0; v < V; ++v)
                    for (int c = 0; c < nb; ++c)
                        col[v][c] = (double)hst[(size_t)v * nb + c] * inv_scale[kind[v]];
                const double T = S.P.st64[S.mats[mi].step].t;
                const double d = std::exp(-a.r * T), dp = std::exp(-(a.r + hr) * T),
                             dm = std::exp(-(a.r - hr) * T);
                for (int j = 0; j < nK; ++j) {
                    const double K = spec->strikes[j];
                    double f[HMC_SURF_VALS];
                    for (int v = 0; v < R; ++v) f[v] = suffix(col[v], nb, j + 1);  // {x > K_j}
                    for (int v = R; v < V; ++v) f[v] = col[v][j];                   // bands at K_j
                    double* o = out + ((((size_t)run * 2 + style) * spec->n_mats + mi) * nK + j) * HMC_NW;
                    // price, pathwise delta, pathwise rho over {A > K}
                    o[0] = d * (f[3] - K * f[2]);
                    o[1] = d * d * (f[4] - 2 * K * f[3] + K * K * f[2]);
                    o[2] = d / S0 * f[3];
                    o[3] = (d / S0) * (d / S0) * f[4];
                    o[4] = d * (f[5] + T * K * f[2]);
                    o[5] = d * d * (f[6] + 2 * T * K * f[5] + T * T * K * K * f[2]);
                    // gamma: (d/S0) A / 2h on the band A(1-e) <= K < A(1+e)
                    const double cg = d / (S0 * 2 * h);
                    o[6] = cg * (f[0] - f[8]);
                    o[7] = cg * cg * (f[1] - f[9]);
                    // FD delta: d A / S0 where A(1-e) > K, d (A(1+e) - K)/2h on the band
                    const double cd = d / (2 * h);
                    o[10] = d / S0 * f[8] + cd * f[15];
                    o[11] = (d / S0) * (d / S0) * f[9] + cd * cd * f[16];
                    // vega: g where both bumped paths are ITM, +-d (x - K)/dv on the bands
                    const double cv = d / dv;
                    o[8] = f[10] + cv * (f[17] - f[19]);
                    o[9] = f[11] + cv * cv * (f[18] + f[20]);
                    // FD rho: a - K b where Rm > K, d+ (Rp - K)/2h_r on the band
                    const double b = (dp - dm) / (2 * hr), ap = dp / (2 * hr);
                    o[12] = (f[13] - K * b * f[12]) + ap * f[21];
                    o[13] = (f[14] - 2 * K * b * f[13] + K * K * b * b * f[12]) + ap * ap * f[22];
                }
            }
    return HMC_OK;
}

int hmc_surface(const hmc_model* model, const hmc_surface_spec* spec, const hmc_sim* sim_in,
                double* h_out, int32_t device) {
    if (!sim_in || !h_out) return fail(HMC_E_INVALID, "sim / h_out is NULL");
    hmc_sim sim = *sim_in;
    sim.path_lo = 0;
    sim.path_hi = sim.n_paths;
    SurfPrepared S;
    int rc = prepare_surface(model, spec, &sim, S);
    if (rc) return rc;
    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(device));
    cudaStream_t st;
    HMC_CK(call_stream(device, &st));
    const size_t acc_bytes = (size_t)hmc_surface_acc_words(spec, sim.n_runs) * sizeof(int64_t);
    const size_t work = (size_t)hmc_surface_workspace_bytes(spec, &sim);
    std::vector<int64_t> h_acc(acc_bytes / sizeof(int64_t));
    char* buf = nullptr;
    cudaError_t e = pool_alloc(device, (void**)&buf, align_up(acc_bytes) + work, st);
    if (e == cudaSuccess) {
        int64_t* d_acc = (int64_t*)buf;
        e = cudaMemsetAsync(d_acc, 0, acc_bytes, st);
        if (e == cudaSuccess) rc = hmc_surface_partials(model, spec, &sim, d_acc, buf + align_up(acc_bytes), st);
        if (e == cudaSuccess && rc == HMC_OK) {
            e = cudaMemcpyAsync(h_acc.data(), d_acc, acc_bytes, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        }
        cudaFreeAsync(buf, st);
    }
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (rc) return rc;
    HMC_CK(e);
    HMC_CK(e2);
    return hmc_surface_finalize(model, spec, &sim, h_acc.data(), h_out);
}
}  // extern "C"
