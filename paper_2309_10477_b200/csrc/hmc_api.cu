// hmc_api.cu -- the C ABI (include/hmc.h): argument validation, per-call
// step tables, kernel dispatch, and the fixed-order reductions
//   tile partials (128 paths)  ->  chunk partials (16384 paths)  ->  per run.
// Chunks are the unit exchanged between GPUs, so a job split across any
// number of devices at chunk boundaries reduces in exactly the single-GPU
// order (bit-identical results, the reference's determinism contract,
// engine.py:5-9).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <utility>
#include <vector>

#include "hmc_host.h"

namespace hmc_host {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

namespace {
struct ThreadStreams {
    std::vector<cudaStream_t> by_device;
    ~ThreadStreams() {
        for (cudaStream_t st : by_device)
            if (st) cudaStreamDestroy(st);
    }
};
thread_local ThreadStreams t_streams;
}  // namespace

cudaError_t call_stream(int device, cudaStream_t* out) {
    if (device < 0 || device >= 1024) return cudaErrorInvalidDevice;
    if ((size_t)device >= t_streams.by_device.size()) t_streams.by_device.resize((size_t)device + 1, nullptr);
    cudaStream_t& st = t_streams.by_device[device];
    if (!st) {
        cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            st = nullptr;
            return e;
        }
    }
    *out = st;
    return cudaSuccess;
}

// The one-call entry points allocate their device buffers from a
// stream-ordered pool PRIVATE to libhmc (one per device, created on first
// use).  The default pool is left untouched, so torch's caching allocator
// and every other user of it keep their own release policy.  The private
// pool keeps up to kPoolKeepBytes of freed blocks across synchronizes: the
// exact scheme's node cache (up to ~310 MB: 256 fp64 nodes per resident
// thread) is re-mapped on every call otherwise -- measured 310 ms per
// 2^17-path exact price with a 256 MB threshold, 0.8 ms with 1 GiB --
// while a one-off multi-GB buffer (a caller's replay uniforms) above the
// threshold goes back to the driver instead of being held for the life of
// the process.
constexpr uint64_t kPoolKeepBytes = 1ull << 30;

namespace {
std::mutex g_pool_mu;
std::vector<cudaMemPool_t> g_pools;  // by device ordinal
}  // namespace

cudaError_t pool_alloc(int dev, void** p, size_t bytes, cudaStream_t s) {
    if (dev < 0 || dev >= 1024) return cudaErrorInvalidDevice;
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if ((size_t)dev >= g_pools.size()) g_pools.resize((size_t)dev + 1, nullptr);
        if (!g_pools[dev]) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.handleTypes = cudaMemHandleTypeNone;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            cudaMemPool_t created = nullptr;
            cudaError_t e = cudaMemPoolCreate(&created, &props);
            if (e != cudaSuccess) return e;
            uint64_t keep = kPoolKeepBytes;
            e = cudaMemPoolSetAttribute(created, cudaMemPoolAttrReleaseThreshold, &keep);
            if (e != cudaSuccess) {
                cudaMemPoolDestroy(created);
                return e;
            }
            g_pools[dev] = created;
        }
        pool = g_pools[dev];
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

// workspace bytes of the bridge tables (S nodes, n_steps + 1 steps, both precisions)
size_t bridge_bytes(int S, int n_steps) {
    if (S <= 0) return 0;
    const size_t n = (size_t)n_steps + 1;
    return align_up(S * sizeof(hmc::BridgeNodeD)) + align_up(n * sizeof(hmc::BridgeStepD)) +
           align_up(S * sizeof(hmc::BridgeNode)) + align_up(n * sizeof(hmc::BridgeStep));
}

// Brownian-bridge tables over steps 1..n_sim with S segments (layout and
// formulas: hmc_device.cuh BridgeNodeD).  Level order: the root (W at the
// horizon) first, then the midpoint of every interval of the previous level,
// left to right -- the coarsest scales get the lowest Sobol dimensions.
void build_bridge(int S, int n_sim, double dt, Prepared& P) {
    std::vector<long long> b((size_t)S + 1);
    for (int j = 0; j <= S; ++j) b[j] = (long long)j * n_sim / S;
    auto t = [&](int j) { return (double)b[j] * dt; };
    P.bn64.clear();
    P.bn64.push_back({0.0, std::sqrt(t(S)), S, 0, 0, 0});
    std::vector<std::pair<int, int>> level{{0, S}};
    while (!level.empty()) {
        std::vector<std::pair<int, int>> next;
        for (auto [l, r] : level) {
            if (r - l < 2) continue;
            const int m = (l + r) / 2;
            const double tl = t(l), tm = t(m), tr = t(r);
            P.bn64.push_back({(tm - tl) / (tr - tl), std::sqrt((tm - tl) * (tr - tm) / (tr - tl)), m, l, r, 0});
            next.push_back({l, m});
            next.push_back({m, r});
        }
        level.swap(next);
    }
    P.bs64.assign((size_t)n_sim + 1, hmc::BridgeStepD{0.0, 0.0, 0, 0});
    for (int j = 1; j <= S; ++j)
        for (long long k = b[j - 1] + 1; k <= b[j]; ++k) {
            const double left = (double)(b[j] - k);  // steps after k inside the segment
            P.bs64[k] = {1.0 / (left + 1.0), std::sqrt(dt * left / (left + 1.0)), j, k < b[j] ? 1 : 0};
        }
    P.bn32.clear();
    // fp32 tables: the kernel's Sobol normals come as z / sqrt(2) (hmc_path32.cuh
    // sobol_normal_u), so the noise coefficients carry the sqrt(2)
    const double r2 = std::sqrt(2.0);
    for (const auto& n : P.bn64) P.bn32.push_back({(float)n.a, (float)(n.sd * r2), n.m, n.l | (n.r << 16)});
    P.bs32.clear();
    for (const auto& st : P.bs64) P.bs32.push_back({(float)st.alpha, (float)(st.beta * r2)});
}

int check_model(const hmc_model* m) {
    if (!m) return fail(HMC_E_INVALID, "model is NULL");
    if (!std::isfinite(m->kappa) || !std::isfinite(m->theta) || !std::isfinite(m->sigma) ||
        !std::isfinite(m->rho) || !std::isfinite(m->r) || !std::isfinite(m->v0))
        return fail(HMC_E_INVALID, "model parameters must be finite");
    if (!(m->kappa > 0.0) || !(m->theta > 0.0) || !(m->sigma > 0.0))
        return fail(HMC_E_INVALID, "kappa, theta and sigma must be > 0");
    if (!(m->rho >= -1.0 && m->rho <= 1.0)) return fail(HMC_E_INVALID, "rho must lie in [-1, 1]");
    if (!(m->v0 >= 0.0)) return fail(HMC_E_INVALID, "v0 must be >= 0");
    return HMC_OK;
}

// step tables shared by every kernel: t_k = k*T/n_steps computed exactly as
// _core.pyx:406 (int k promoted to double, times T, divided by n_steps);
// the fp32 table holds the fixing weights (E_k, E_k t_k, E_k expm1(+-h t_k))
// with E_k = S0 e^{r t_k}, zero on non-fixing steps.
void build_steps(int n_steps, double T, double h_r, double s0, double r,
                 const unsigned char* fix, Prepared& P) {
    P.st64.resize((size_t)n_steps + 1);
    P.st32.resize((size_t)n_steps + 1);
    for (int k = 0; k <= n_steps; ++k) {
        const double t = k * T / n_steps;
        StepD s{t, std::expm1(h_r * t), std::expm1(-h_r * t), fix[k] ? 1.0 : 0.0};
        P.st64[k] = s;
        const double E = fix[k] ? s0 * std::exp(r * t) : 0.0;
        P.st32[k] = make_float4((float)E, (float)(E * t), (float)(E * s.e1p), (float)(E * s.e1m));
    }
}

void fill_fp32_constants(KernelArgs& a) {
    const double log2e = 1.4426950408889634074, ln2 = 0.69314718055994530942;
    const double mil = a.milstein ? 1.0 : 0.0;
    a.f_omkdt = (float)(1.0 - a.kappa * a.dt);
    a.f_ck0 = (float)(a.kappa * a.theta * a.dt - mil * 0.25 * a.sigma * a.sigma * a.dt);
    a.f_cmil = (float)(mil * 0.25 * a.sigma * a.sigma);
    a.f_sigma = (float)a.sigma;
    a.f_nhdt2 = (float)(-0.5 * a.dt * log2e);
    a.f_bm2 = (float)(-2.0 * ln2 * a.dt * log2e * log2e);
    a.f_cA = (float)(a.sigma * a.rho / log2e);
    a.f_cB = (float)(a.sigma * a.sq1mr2 / log2e);
    a.f_cmil2 = (float)(0.25 * mil);
    a.f_log2e = (float)log2e;
    a.f_rho = (float)a.rho;
    a.f_sq1mr2 = (float)a.sq1mr2;
    a.f_sqdt = (float)std::sqrt(a.dt);
    {
        const float sq2 = 1.41421356237309504880f;   // hmc_path32.cuh kSqrt2f
        a.f_sob_k.x = sq2 * a.f_sqdt * a.f_log2e;
        a.f_sob_k.y = sq2 * a.f_sigma * a.f_sqdt * a.f_sq1mr2;
        a.f_sob_k2.x = -2.0f * a.f_sob_k.x;
        a.f_sob_k2.y = -2.0f * a.f_sob_k.y;
        a.f_sob_crho = a.f_sigma * a.f_rho / a.f_log2e;
    }
    a.f_v0 = (float)a.v0;
    a.f_vu = (float)a.v0_up;
    a.f_vd = (float)a.v0_dn;
    a.f_K = (float)a.K;
    a.f_T = (float)a.T;
    a.f_disc = (float)a.disc;
    a.f_disc_up = (float)a.disc_up;
    a.f_disc_dn = (float)a.disc_dn;
    a.f_ddisc = (float)(a.disc_up - a.disc_dn);
    a.f_inv_s0 = (float)(1.0 / a.s0);
    a.f_up_ratio = (float)((a.s0 + a.h_spot) / a.s0);
    a.f_dn_ratio = (float)((a.s0 - a.h_spot) / a.s0);
    a.f_inv_2h = a.h_spot > 0.0 ? (float)(0.5 / a.h_spot) : 0.0f;
    a.f_inv_dv = a.v0_up > a.v0_dn ? (float)(1.0 / (a.v0_up - a.v0_dn)) : 0.0f;
    a.f_inv_2hr = a.h_r > 0.0 ? (float)(0.5 / a.h_r) : 0.0f;
    a.f_inv_navg = (float)(1.0 / a.n_avg);
}

int prepare(const hmc_model* m, const hmc_product* pr, const hmc_sim* sim, Prepared& P) {
    int rc = check_model(m);
    if (rc) return rc;
    if (!pr || !sim) return fail(HMC_E_INVALID, "product/sim is NULL");
    if (!(pr->strike > 0.0) || !(pr->maturity > 0.0) || !(pr->spot > 0.0) || !std::isfinite(pr->strike) ||
        !std::isfinite(pr->maturity) || !std::isfinite(pr->spot))
        return fail(HMC_E_INVALID, "strike, maturity and spot must be finite and > 0");
    if (pr->style != HMC_STYLE_EUROPEAN && pr->style != HMC_STYLE_ASIAN)
        return fail(HMC_E_INVALID, "unknown option style");
    if (pr->right != HMC_CALL && pr->right != HMC_PUT) return fail(HMC_E_INVALID, "unknown option right");
    if (sim->scheme != HMC_SCHEME_EULER && sim->scheme != HMC_SCHEME_MILSTEIN)
        return fail(HMC_E_UNSUPPORTED, "only the euler and milstein schemes run on the GPU");
    if (sim->sampler != HMC_SAMPLER_PSEUDO && sim->sampler != HMC_SAMPLER_SOBOL)
        return fail(HMC_E_INVALID, "unknown sampler");
    if (sim->precision != HMC_PREC_FP32 && sim->precision != HMC_PREC_FP64)
        return fail(HMC_E_INVALID, "unknown precision");
    if (sim->n_steps < 1 || sim->n_runs < 1 || sim->n_paths < 1)
        return fail(HMC_E_INVALID, "need n_steps >= 1, n_runs >= 1, n_paths >= 1");
    if (sim->path_lo < 0 || sim->path_hi > sim->n_paths || sim->path_lo >= sim->path_hi)
        return fail(HMC_E_INVALID, "path slice must satisfy 0 <= path_lo < path_hi <= n_paths");
    if (sim->path_lo % HMC_CHUNK != 0) return fail(HMC_E_INVALID, "path_lo must be a multiple of HMC_CHUNK");
    if (sim->want_greeks && pr->right != HMC_CALL)
        return fail(HMC_E_UNSUPPORTED, "pathwise Greeks are derived for calls only");
    if (!pr->avg_idx || pr->n_avg < 1) return fail(HMC_E_INVALID, "avg_idx must hold >= 1 index");
    for (long long i = 0; i < pr->n_avg; ++i) {
        if (pr->avg_idx[i] < 1 || pr->avg_idx[i] > sim->n_steps ||
            (i > 0 && pr->avg_idx[i] <= pr->avg_idx[i - 1]))
            return fail(HMC_E_INVALID, "avg_idx must be strictly increasing in [1, n_steps]");
    }
    if (pr->style == HMC_STYLE_EUROPEAN && (pr->n_avg != 1 || pr->avg_idx[0] != sim->n_steps))
        return fail(HMC_E_INVALID, "european products fix once, at n_steps");
    if (sim->want_greeks) {
        if (!std::isfinite(sim->v0_up) || !std::isfinite(sim->h_r))
            return fail(HMC_E_INVALID, "bump sizes must be finite");
        if (!(sim->h_spot > 0.0 && sim->h_spot < pr->spot)) return fail(HMC_E_INVALID, "need 0 < h_spot < spot");
        if (!(sim->v0_up > sim->v0_dn && sim->v0_dn >= 0.0)) return fail(HMC_E_INVALID, "need v0_up > v0_dn >= 0");
        if (!(sim->h_r > 0.0)) return fail(HMC_E_INVALID, "need h_r > 0");
    }
    if (sim->sampler == HMC_SAMPLER_PSEUDO && sim->precision == HMC_PREC_FP32 &&
        sim->n_paths > 4294967296LL)
        return fail(HMC_E_INVALID, "the Philox counter addresses at most 2^32 paths per run");
    if (sim->sampler == HMC_SAMPLER_SOBOL) {
        if (!sim->sobol_v) return fail(HMC_E_INVALID, "sobol sampler needs direction numbers");
        const double blocks = sim->sobol_scramble ? 1.0 : (double)sim->n_runs;
        if (1.0 + blocks * (double)sim->n_paths > 1073741824.0)
            return fail(HMC_E_INVALID, "sobol index range exceeds 2^30 points");
    }
    if (sim->sobol_bridge != 0) {
        if (sim->sampler != HMC_SAMPLER_SOBOL)
            return fail(HMC_E_INVALID, "the Brownian bridge orders Sobol dimensions (sampler must be sobol)");
        if (sim->sobol_bridge < 0 || sim->sobol_bridge > HMC_BRIDGE_MAX_SEGMENTS ||
            sim->sobol_bridge > pr->avg_idx[pr->n_avg - 1])
            return fail(HMC_E_INVALID, "sobol_bridge must lie in [1, min(HMC_BRIDGE_MAX_SEGMENTS, simulated steps)]");
    }

    KernelArgs& a = P.a;
    a.kappa = m->kappa; a.theta = m->theta; a.sigma = m->sigma; a.rho = m->rho;
    a.r = m->r; a.v0 = m->v0;
    a.s0 = pr->spot; a.T = pr->maturity; a.K = pr->strike;
    a.v0_up = sim->want_greeks ? sim->v0_up : m->v0;
    a.v0_dn = sim->want_greeks ? sim->v0_dn : m->v0;
    a.h_spot = sim->want_greeks ? sim->h_spot : 0.0;
    a.h_r = sim->want_greeks ? sim->h_r : 0.0;
    a.dt = pr->maturity / sim->n_steps;                    // _core.pyx:378
    a.sq1mr2 = std::sqrt(1.0 - m->rho * m->rho);           // _core.pyx:379
    a.disc = std::exp(-m->r * pr->maturity);               // engine.py:50
    a.disc_up = std::exp(-(m->r + a.h_r) * pr->maturity);
    a.disc_dn = std::exp(-(m->r - a.h_r) * pr->maturity);
    a.n_steps = sim->n_steps;
    a.n_avg = (int)pr->n_avg;
    a.n_sim = (int)pr->avg_idx[pr->n_avg - 1];
    bool every = (long long)a.n_sim == pr->n_avg;          // 1..n_sim all fixings
    a.fix_mode = pr->n_avg == 1 ? hmc::kFixLast : (every ? hmc::kFixEvery : hmc::kFixTable);
    a.is_asian = pr->style == HMC_STYLE_ASIAN;
    a.is_call = pr->right == HMC_CALL;
    a.want_greeks = sim->want_greeks ? 1 : 0;
    a.milstein = sim->scheme == HMC_SCHEME_MILSTEIN;
    a.sampler = sim->sampler;
    a.n_runs = sim->n_runs;
    a.n_paths = sim->n_paths;
    a.path_lo = sim->path_lo;
    a.path_hi = sim->path_hi;
    a.root_key = hmc_root_key(sim->seed);
    a.sobol_dim = 2 * sim->n_steps;
    a.sobol_scramble = sim->sampler == HMC_SAMPLER_SOBOL && sim->sobol_scramble ? 1 : 0;

    fill_fp32_constants(a);
    std::vector<unsigned char> fix((size_t)sim->n_steps + 1, 0);
    for (long long i = 0; i < pr->n_avg; ++i) fix[pr->avg_idx[i]] = 1;
    build_steps(sim->n_steps, pr->maturity, a.h_r, pr->spot, m->r, fix.data(), P);
    a.bridge_segments = sim->sobol_bridge;
    if (a.bridge_segments > 0) {
        build_bridge(a.bridge_segments, a.n_sim, a.dt, P);
        for (size_t k = 1; k < P.bs64.size(); ++k)  // fp32 kernel: beta == 0 marks segment ends
            if (P.bs64[k].consume && P.bs32[k].beta == 0.0f)
                return fail(HMC_E_INVALID, "time step too small for the fp32 Brownian bridge");
    }

    const long long n = sim->path_hi - sim->path_lo;
    P.n_tiles = n_tiles_of(n);
    P.n_chunks = n_chunks_of(n);
    size_t off = align_up((size_t)sim->n_runs * P.n_tiles * HMC_NW * sizeof(double));
    P.off_st64 = off;
    off += align_up(P.st64.size() * sizeof(StepD));
    P.off_st32 = off;
    off += align_up(P.st32.size() * sizeof(float4));
    P.off_sobol = off;
    if (sim->sampler == HMC_SAMPLER_SOBOL && !sim->sobol_v_on_device)
        off += align_up((size_t)30 * a.sobol_dim * sizeof(uint32_t));
    P.off_bridge = off;
    off += bridge_bytes(a.bridge_segments, sim->n_steps);
    P.bytes = off;
    return HMC_OK;
}


}  // namespace hmc_host

using namespace hmc_host;

namespace hmc {

__global__ void tiles_to_chunks_kernel(const double* __restrict__ tiles, long long n_tiles,
                                       double* __restrict__ chunks, long long n_chunks) {
    const int w = threadIdx.x;
    if (w >= kNW) return;
    const int run = blockIdx.y;
    const long long c = blockIdx.x;
    const long long t0 = c * HMC_CHUNK_TILES;
    const long long t1 = t0 + HMC_CHUNK_TILES < n_tiles ? t0 + HMC_CHUNK_TILES : n_tiles;
    const double* src = tiles + (size_t)run * n_tiles * kNW;
    double s = 0.0;
    for (long long t = t0; t < t1; ++t) s += src[t * kNW + w];
    chunks[((size_t)run * n_chunks + c) * kNW + w] = s;
}

// Sum over chunks in global path order with a FIXED shape: thread t owns
// chunks t, t + 512, ... (sequential), then a fixed 512-way tree.  The shape
// depends only on the global chunk count, never on how the chunks were
// produced, so 1 GPU and N GPUs give bit-identical results.
constexpr int kRunThreads = 512;

__global__ void __launch_bounds__(kRunThreads) chunks_to_runs_kernel(const double* __restrict__ chunks,
                                                                    long long n_chunks,
                                                                    double* __restrict__ out) {
    __shared__ double red[kRunThreads];
    const int run = blockIdx.x;
    const double* src = chunks + (size_t)run * n_chunks * kNW;
    double acc[kNW];
#pragma unroll
    for (int w = 0; w < kNW; ++w) acc[w] = 0.0;
    for (long long c = threadIdx.x; c < n_chunks; c += kRunThreads) {
#pragma unroll
        for (int w = 0; w < kNW; ++w) acc[w] += src[c * kNW + w];
    }
    for (int w = 0; w < kNW; ++w) {
        red[threadIdx.x] = acc[w];
        __syncthreads();
        for (int s = kRunThreads / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[(size_t)run * kNW + w] = red[0];
        __syncthreads();
    }
}

cudaError_t launch_tiles_to_chunks(const double* d_tiles, long long n_tiles, int n_runs,
                                   double* d_chunks, long long n_chunks, cudaStream_t s) {
    for (int r0 = 0; r0 < n_runs; r0 += kMaxRunsPerLaunch) {
        const int nb = min(kMaxRunsPerLaunch, n_runs - r0);
        tiles_to_chunks_kernel<<<dim3((unsigned)n_chunks, (unsigned)nb), 32, 0, s>>>(
            d_tiles + (size_t)r0 * n_tiles * kNW, n_tiles, d_chunks + (size_t)r0 * n_chunks * kNW, n_chunks);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

__global__ void philox_kat_kernel(const uint4* __restrict__ ctr, uint4* __restrict__ out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const uint4 c = ctr[i];
        out[i] = philox4x32_10(c.x, c.y, c.z, c.w);
    }
}

// the production kernels' Box-Muller on given Philox blocks: three (z1, z2)
// standard-normal pairs per block (KernelArgs set so the folded constants
// reduce to sqrt(-2 ln u1) (cos, sin))
__global__ void box_muller_kat_kernel(const uint4* __restrict__ w, int n, KernelArgs a,
                                      float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const uint4 x = w[i];
        float fr[3], fa[3];
        tri_unpack(x, fr, fa);
        for (int k = 0; k < 3; ++k) {
            float z1, z2;
            box_muller_f(fr[k], fa[k], a, z1, z2);
            out[6 * i + 2 * k] = z1;
            out[6 * i + 2 * k + 1] = z2;
        }
    }
}

// the production kernels' Sobol quantile on given 30-bit coordinates: the
// paired form (x[i], x[n-1-i]) as the path kernels use it, its second lane
// checked bit for bit against the scalar form (a mismatch writes NaN).
// Every lane of a warp runs the quantile (its tail branches are warp votes).
__global__ void sobol_quantile_kernel(const uint32_t* __restrict__ x, int n, float half,
                                      float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = min(i, n - 1);
    const uint32_t mid = half != 0.0f ? 2u : 0u;           // left-aligned coordinates
    const uint32_t Xa = (x[j] << 2) | mid, Xb = (x[n - 1 - j] << 2) | mid;
    const float2 z = sobol_normal_X2(Xa, Xb, f2(1.0f));
    const float s = sobol_normal_X(Xb, 1.0f);
    if (i < n) out[i] = __float_as_uint(s) == __float_as_uint(z.y) ? kSqrt2f * z.x : __int_as_float(0x7fffffff);
}

cudaError_t launch_chunks_to_runs(const double* d_chunks, long long n_chunks, int n_runs,
                                  double* d_out, cudaStream_t s) {
    chunks_to_runs_kernel<<<(unsigned)n_runs, kRunThreads, 0, s>>>(d_chunks, n_chunks, d_out);
    return cudaGetLastError();
}

}  // namespace hmc

extern "C" {

int hmc_abi_version(void) { return HMC_ABI_VERSION; }

const char* hmc_last_error(void) { return g_err.c_str(); }

int hmc_device_count(int32_t* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        if (count) *count = 0;
        cudaGetLastError();
        return fail(HMC_E_NODEVICE, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    if (count) *count = n;
    return HMC_OK;
}

uint64_t hmc_root_key(uint64_t seed) { return hmc::mix64(seed ^ 0x8CB92BA72F3D8DD7ULL); }

uint64_t hmc_derive_key(uint64_t parent, uint64_t index) { return hmc::derive(parent, index); }

int64_t hmc_chunks_in_slice(const hmc_sim* sim) {
    if (!sim || sim->path_hi <= sim->path_lo) return 0;
    return n_chunks_of(sim->path_hi - sim->path_lo);
}

int64_t hmc_workspace_bytes(const hmc_sim* sim) {
    if (!sim || sim->path_hi <= sim->path_lo || sim->n_steps < 1 || sim->n_runs < 1) return 0;
    const long long n = sim->path_hi - sim->path_lo;
    size_t b = align_up((size_t)sim->n_runs * n_tiles_of(n) * HMC_NW * sizeof(double));
    b += align_up(((size_t)sim->n_steps + 1) * sizeof(StepD));
    b += align_up(((size_t)sim->n_steps + 1) * sizeof(float4));
    if (sim->sampler == HMC_SAMPLER_SOBOL && !sim->sobol_v_on_device)
        b += align_up((size_t)30 * 2 * sim->n_steps * sizeof(uint32_t));
    if (sim->sobol_bridge > 0 && sim->sobol_bridge <= HMC_BRIDGE_MAX_SEGMENTS)
        b += bridge_bytes(sim->sobol_bridge, sim->n_steps);
    return (int64_t)b;
}

int hmc_greeks_chunks(const hmc_model* model, const hmc_product* product, const hmc_sim* sim,
                      double* d_chunks, void* d_work, void* stream) {
    Prepared P;
    int rc = prepare(model, product, sim, P);
    if (rc) return rc;
    if (!d_chunks || !d_work) return fail(HMC_E_INVALID, "d_chunks / d_work is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    char* w = (char*)d_work;
    double* d_tiles = (double*)w;
    {   // both step tables in one host->device copy (they are adjacent in the workspace)
        const size_t b64 = P.st64.size() * sizeof(StepD), b32 = P.st32.size() * sizeof(float4);
        std::vector<char> img(P.off_st32 - P.off_st64 + b32);
        std::memcpy(img.data(), P.st64.data(), b64);
        std::memcpy(img.data() + (P.off_st32 - P.off_st64), P.st32.data(), b32);
        HMC_CK(cudaMemcpyAsync(w + P.off_st64, img.data(), img.size(), cudaMemcpyHostToDevice, s));
    }
    P.a.steps64 = (const StepD*)(w + P.off_st64);
    P.a.steps32 = (const float4*)(w + P.off_st32);
    if (sim->sampler == HMC_SAMPLER_SOBOL) {
        if (sim->sobol_v_on_device) {
            P.a.sobol_v = sim->sobol_v;
        } else {
            HMC_CK(cudaMemcpyAsync(w + P.off_sobol, sim->sobol_v,
                                   (size_t)30 * P.a.sobol_dim * sizeof(uint32_t),
                                   cudaMemcpyHostToDevice, s));
            P.a.sobol_v = (const uint32_t*)(w + P.off_sobol);
        }
    }
    if (P.a.bridge_segments > 0) {
        char* b = w + P.off_bridge;
        const size_t sz[4] = {P.bn64.size() * sizeof(hmc::BridgeNodeD), P.bs64.size() * sizeof(hmc::BridgeStepD),
                              P.bn32.size() * sizeof(hmc::BridgeNode), P.bs32.size() * sizeof(hmc::BridgeStep)};
        const void* src[4] = {P.bn64.data(), P.bs64.data(), P.bn32.data(), P.bs32.data()};
        // region strides as bridge_bytes(): S node slots, n_steps + 1 step slots
        const size_t S = (size_t)P.a.bridge_segments, n1 = (size_t)sim->n_steps + 1;
        const size_t stride[4] = {align_up(S * sizeof(hmc::BridgeNodeD)), align_up(n1 * sizeof(hmc::BridgeStepD)),
                                  align_up(S * sizeof(hmc::BridgeNode)), align_up(n1 * sizeof(hmc::BridgeStep))};
        char* dst[4];
        for (int i = 0; i < 4; ++i) {
            dst[i] = b;
            HMC_CK(cudaMemcpyAsync(b, src[i], sz[i], cudaMemcpyHostToDevice, s));
            b += stride[i];
        }
        P.a.bridge_nodes64 = (const hmc::BridgeNodeD*)dst[0];
        P.a.bridge_steps64 = (const hmc::BridgeStepD*)dst[1];
        P.a.bridge_nodes32 = (const hmc::BridgeNode*)dst[2];
        P.a.bridge_steps32 = (const hmc::BridgeStep*)dst[3];
    }
    if (sim->precision == HMC_PREC_FP64)
        HMC_CK(hmc::launch_replay_greeks(P.a, d_tiles, P.n_tiles, s));
    else
        HMC_CK(hmc::launch_fast_greeks(P.a, d_tiles, P.n_tiles, s));
    HMC_CK(hmc::launch_tiles_to_chunks(d_tiles, P.n_tiles, sim->n_runs, d_chunks, P.n_chunks, s));
    return HMC_OK;
}

int hmc_reduce_chunks(const double* d_chunks, int32_t n_runs, int64_t n_chunks, double* d_out,
                      void* stream) {
    if (!d_chunks || !d_out || n_runs < 1 || n_chunks < 1)
        return fail(HMC_E_INVALID, "bad reduce arguments");
    HMC_CK(hmc::launch_chunks_to_runs(d_chunks, n_chunks, n_runs, d_out, (cudaStream_t)stream));
    return HMC_OK;
}

int hmc_greeks(const hmc_model* model, const hmc_product* product, const hmc_sim* sim_in,
               double* h_out, int32_t device) {
    if (!sim_in || !h_out) return fail(HMC_E_INVALID, "sim / h_out is NULL");
    hmc_sim sim = *sim_in;
    sim.path_lo = 0;
    sim.path_hi = sim.n_paths;
    Prepared P;
    int rc = prepare(model, product, &sim, P);
    if (rc) return rc;
    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(device));
    cudaStream_t s;
    HMC_CK(call_stream(device, &s));
    const size_t work = (size_t)hmc_workspace_bytes(&sim);
    const size_t chunk_bytes = (size_t)sim.n_runs * P.n_chunks * HMC_NW * sizeof(double);
    const size_t out_bytes = (size_t)sim.n_runs * HMC_NW * sizeof(double);
    char* buf = nullptr;
    cudaError_t e = pool_alloc(device, (void**)&buf, work + align_up(chunk_bytes) + out_bytes, s);
    if (e == cudaSuccess) {
        double* d_chunks = (double*)(buf + work);
        double* d_out = (double*)(buf + work + align_up(chunk_bytes));
        rc = hmc_greeks_chunks(model, product, &sim, d_chunks, buf, s);
        if (rc == HMC_OK) rc = hmc_reduce_chunks(d_chunks, sim.n_runs, P.n_chunks, d_out, s);
        if (rc == HMC_OK) {
            e = cudaMemcpyAsync(h_out, d_out, out_bytes, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        }
        cudaFreeAsync(buf, s);
    }
    cudaError_t e2 = cudaStreamSynchronize(s);
    if (rc) return rc;
    HMC_CK(e);
    HMC_CK(e2);
    return HMC_OK;
}

int hmc_greeks_multi(const hmc_model* model, const hmc_product* product, const hmc_sim* sim_in,
                     double* h_out, const int32_t* devices, int32_t n_devices) {
    if (!sim_in || !h_out) return fail(HMC_E_INVALID, "sim / h_out is NULL");
    if (!devices || n_devices < 1 || n_devices > 1024) return fail(HMC_E_INVALID, "need 1..1024 devices");
    if (sim_in->sobol_v_on_device)
        return fail(HMC_E_INVALID, "hmc_greeks_multi needs a host Sobol direction table "
                                   "(sobol_v_on_device = 0): a device pointer belongs to one GPU");
    hmc_sim sim = *sim_in;
    sim.path_lo = 0;
    sim.path_hi = sim.n_paths;
    Prepared P;
    int rc = prepare(model, product, &sim, P);  // validates the whole job before any device work
    if (rc) return rc;
    const long long C = P.n_chunks, R = sim.n_runs;
    const size_t row = (size_t)HMC_NW * sizeof(double);

    struct Part {
        int dev = 0;
        long long c_lo = 0, c_hi = 0;
        hmc_sim sim{};
        cudaStream_t st = nullptr;
        cudaEvent_t done = nullptr;
        char* buf = nullptr;
    };
    std::vector<Part> parts((size_t)n_devices);
    const long long base = C / n_devices, extra = C % n_devices;
    for (int r = 0; r < n_devices; ++r) {  // parallel.shard
        Part& q = parts[r];
        q.dev = devices[r];
        q.c_lo = r * base + (r < extra ? r : extra);
        q.c_hi = q.c_lo + base + (r < extra ? 1 : 0);
        q.sim = sim;
        q.sim.path_lo = std::min(q.c_lo * (long long)HMC_CHUNK, (long long)sim.n_paths);
        q.sim.path_hi = std::min(q.c_hi * (long long)HMC_CHUNK, (long long)sim.n_paths);
    }
    // the gather buffer [run][C][HMC_NW] + the result live on devices[0]
    const int root = devices[0];
    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(root));
    cudaStream_t rs;
    HMC_CK(cudaStreamCreateWithFlags(&rs, cudaStreamNonBlocking));
    char* gbuf = nullptr;
    const size_t gbytes = align_up((size_t)R * C * row) + (size_t)R * row;
    // plain cudaMalloc: the peer copies of the other devices write into it
    cudaError_t e = cudaMalloc((void**)&gbuf, gbytes);
    double* g_chunks = (double*)gbuf;
    double* g_out = (double*)(gbuf + align_up((size_t)R * C * row));

    // launch every slice (asynchronous: the devices run concurrently)
    for (Part& q : parts) {
        if (e != cudaSuccess || rc != HMC_OK) break;
        if (q.c_hi <= q.c_lo) continue;
        if ((e = cudaSetDevice(q.dev)) != cudaSuccess) break;
        if ((e = cudaStreamCreateWithFlags(&q.st, cudaStreamNonBlocking)) != cudaSuccess) break;
        if ((e = cudaEventCreateWithFlags(&q.done, cudaEventDisableTiming)) != cudaSuccess) break;
        const long long nc = q.c_hi - q.c_lo;
        const size_t work = (size_t)hmc_workspace_bytes(&q.sim);
        if ((e = pool_alloc(q.dev, (void**)&q.buf, work + (size_t)R * nc * row, q.st)) != cudaSuccess) break;
        double* loc = (double*)(q.buf + work);
        rc = hmc_greeks_chunks(model, product, &q.sim, loc, q.buf, q.st);
        if (rc != HMC_OK) break;
        for (long long r = 0; r < R && e == cudaSuccess; ++r)  // run r's rows, in path order
            e = cudaMemcpyPeerAsync(g_chunks + ((size_t)r * C + q.c_lo) * HMC_NW, root,
                                    loc + (size_t)r * nc * HMC_NW, q.dev, (size_t)nc * row, q.st);
        if (e == cudaSuccess) e = cudaEventRecord(q.done, q.st);
    }
    if (e == cudaSuccess && rc == HMC_OK) e = cudaSetDevice(root);
    for (Part& q : parts)
        if (e == cudaSuccess && rc == HMC_OK && q.done) e = cudaStreamWaitEvent(rs, q.done, 0);
    if (e == cudaSuccess && rc == HMC_OK) {
        rc = hmc_reduce_chunks(g_chunks, (int32_t)R, C, g_out, rs);
        if (rc == HMC_OK) e = cudaMemcpyAsync(h_out, g_out, (size_t)R * row, cudaMemcpyDeviceToHost, rs);
        if (e == cudaSuccess && rc == HMC_OK) e = cudaStreamSynchronize(rs);
    }
    // teardown on every path (errors included)
    for (Part& q : parts) {
        if (!q.st) continue;
        cudaSetDevice(q.dev);
        if (q.buf) cudaFreeAsync(q.buf, q.st);
        cudaStreamSynchronize(q.st);
        cudaStreamDestroy(q.st);
        if (q.done) cudaEventDestroy(q.done);
    }
    cudaSetDevice(root);
    cudaError_t e2 = cudaStreamSynchronize(rs);
    if (gbuf) cudaFree(gbuf);
    cudaStreamDestroy(rs);
    if (rc) return rc;
    HMC_CK(e);
    HMC_CK(e2);
    return HMC_OK;
}

int hmc_discretised_batch_f64(const hmc_model* model, double s0, double T, int32_t n_steps,
                              int32_t milstein, int64_t path_lo, int64_t path_hi,
                              uint64_t key_run, const double* uniforms, const int64_t* avg_idx,
                              int64_t n_avg, double* out, int32_t device) {
    int rc = check_model(model);
    if (rc) return rc;
    if (n_steps < 1 || !(T > 0.0) || !(s0 > 0.0) || !std::isfinite(T) || !std::isfinite(s0))
        return fail(HMC_E_INVALID, "need n_steps >= 1, finite T > 0 and s0 > 0");
    if (path_hi < path_lo) return fail(HMC_E_INVALID, "path_hi < path_lo");
    if (!avg_idx || n_avg < 1) return fail(HMC_E_INVALID, "avg_idx must hold >= 1 index");
    for (int64_t i = 0; i < n_avg; ++i)
        if (avg_idx[i] < 0 || avg_idx[i] > n_steps) return fail(HMC_E_INVALID, "avg index outside [0, n_steps]");
    const long long n = path_hi - path_lo;
    if (n == 0) return HMC_OK;
    if (!out) return fail(HMC_E_INVALID, "out is NULL");

    Prepared P;
    KernelArgs& a = P.a;
    a.kappa = model->kappa; a.theta = model->theta; a.sigma = model->sigma;
    a.rho = model->rho; a.r = model->r; a.v0 = model->v0;
    a.s0 = s0; a.T = T;
    a.dt = T / n_steps;
    a.sq1mr2 = std::sqrt(1.0 - model->rho * model->rho);
    a.n_steps = n_steps;
    a.n_avg = (int)n_avg;  // the reference divides by len(avg_idx) (_core.pyx:370)
    a.milstein = milstein ? 1 : 0;
    a.path_lo = path_lo;
    a.path_hi = path_hi;
    std::vector<unsigned char> fix((size_t)n_steps + 1, 0);
    for (int64_t i = 0; i < n_avg; ++i) fix[avg_idx[i]] = 1;
    build_steps(n_steps, T, 0.0, s0, model->r, fix.data(), P);

    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(device));
    cudaStream_t s;
    HMC_CK(call_stream(device, &s));
    const size_t ub = uniforms ? (size_t)n * 2 * n_steps * sizeof(double) : 0;
    const size_t ob = (size_t)n * 3 * sizeof(double);
    const size_t tb = P.st64.size() * sizeof(StepD);
    char* buf = nullptr;
    cudaError_t e = pool_alloc(device, (void**)&buf, align_up(ub) + align_up(ob) + tb, s);
    if (e == cudaSuccess) {
        double* d_u = uniforms ? (double*)buf : nullptr;
        double* d_out = (double*)(buf + align_up(ub));
        StepD* d_tab = (StepD*)(buf + align_up(ub) + align_up(ob));
        if (uniforms) e = cudaMemcpyAsync(d_u, uniforms, ub, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_tab, P.st64.data(), tb, cudaMemcpyHostToDevice, s);
        a.steps64 = d_tab;
        if (e == cudaSuccess) e = hmc::launch_replay_batch(a, key_run, d_u, d_out, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(out, d_out, ob, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFreeAsync(buf, s);
    }
    cudaError_t e2 = cudaStreamSynchronize(s);
    HMC_CK(e);
    HMC_CK(e2);
    return HMC_OK;
}

}  // extern "C"

namespace {
// device round trip of one elementwise primitive on the per-thread stream:
// `host_in` (bytes each) -> device, launch, device -> `host_out`
template <class Launch>
int elementwise_call(int32_t device, const std::vector<std::pair<const void*, size_t>>& host_in,
                     const std::vector<std::pair<void*, size_t>>& host_out, Launch launch) {
    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(device));
    cudaStream_t s;
    HMC_CK(call_stream(device, &s));
    size_t total = 0;
    for (auto& b : host_in) total += align_up(b.second);
    for (auto& b : host_out) total += align_up(b.second);
    char* buf = nullptr;
    HMC_CK(pool_alloc(device, (void**)&buf, std::max<size_t>(total, 256), s));
    std::vector<void*> dev;
    size_t off = 0;
    cudaError_t e = cudaSuccess;
    for (auto& b : host_in) {
        dev.push_back(buf + off);
        if (e == cudaSuccess && b.second) e = cudaMemcpyAsync(buf + off, b.first, b.second, cudaMemcpyHostToDevice, s);
        off += align_up(b.second);
    }
    for (auto& b : host_out) {
        dev.push_back(buf + off);
        off += align_up(b.second);
    }
    if (e == cudaSuccess) e = launch(dev, s);
    for (size_t j = 0; j < host_out.size() && e == cudaSuccess; ++j)
        if (host_out[j].second)
            e = cudaMemcpyAsync(host_out[j].first, dev[host_in.size() + j], host_out[j].second,
                                cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(buf, s);
    const cudaError_t e2 = cudaStreamSynchronize(s);
    HMC_CK(e);
    HMC_CK(e2);
    return HMC_OK;
}
}  // namespace

extern "C" {

int hmc_uniforms_f64(const uint64_t* keys, int64_t n_keys, const uint64_t* draws, int64_t n, double* out,
                     int32_t device) {
    if (n < 0 || (n > 0 && (!keys || !draws || !out)) || (n_keys != 1 && n_keys != n))
        return fail(HMC_E_INVALID, "need keys (1 or n of them), draws[n] and out[n]");
    if (n == 0) return HMC_OK;
    const size_t kb = (size_t)n_keys * 8, db = (size_t)n * 8;
    return elementwise_call(device, {{keys, kb}, {draws, db}}, {{out, db}}, [&](auto& d, cudaStream_t s) {
        return hmc::launch_uniforms((const unsigned long long*)d[0], n_keys, (const unsigned long long*)d[1], n,
                                    (double*)d[2], s);
    });
}

int hmc_ndtri_f64(const double* u, int64_t n, double* out, int32_t device) {
    if (n < 0 || (n > 0 && (!u || !out))) return fail(HMC_E_INVALID, "need u[n] and out[n]");
    if (n == 0) return HMC_OK;
    const size_t b = (size_t)n * 8;
    return elementwise_call(device, {{u, b}}, {{out, b}}, [&](auto& d, cudaStream_t s) {
        return hmc::launch_ndtri((const double*)d[0], n, (double*)d[1], s);
    });
}

int hmc_gamma_f64(const uint64_t* keys, const uint64_t* start, int64_t n, double shape, double scale,
                  double* out, uint64_t* used, int32_t device) {
    if (!(shape > 0.0) || !(scale > 0.0) || !std::isfinite(shape) || !std::isfinite(scale))
        return fail(HMC_E_INVALID, "gamma shape and scale must be finite and > 0");
    if (n < 0 || (n > 0 && (!keys || !start || !out || !used)))
        return fail(HMC_E_INVALID, "need keys[n], start[n], out[n], used[n]");
    if (n == 0) return HMC_OK;
    const size_t b = (size_t)n * 8;
    return elementwise_call(device, {{keys, b}, {start, b}}, {{out, b}, {used, b}}, [&](auto& d, cudaStream_t s) {
        return hmc::launch_gamma((const unsigned long long*)d[0], (const unsigned long long*)d[1], n, shape, scale,
                                 (double*)d[2], (unsigned long long*)d[3], s);
    });
}

int hmc_steps_f64(const hmc_model* model, int32_t milstein, double dt, const double* s, const double* v,
                  const double* u, int64_t n, double* s_out, double* v_out, int32_t device) {
    int rc = check_model(model);
    if (rc) return rc;
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(HMC_E_INVALID, "dt must be finite and > 0");
    if (n < 0 || (n > 0 && (!s || !v || !u || !s_out || !v_out)))
        return fail(HMC_E_INVALID, "need s[n], v[n], u[n][2], s_out[n], v_out[n]");
    for (int64_t i = 0; i < n; ++i)
        if (!(v[i] >= 0.0) || !(s[i] > 0.0)) return fail(HMC_E_INVALID, "states need s > 0 and v >= 0");
    if (n == 0) return HMC_OK;
    KernelArgs a{};
    a.kappa = model->kappa; a.theta = model->theta; a.sigma = model->sigma;
    a.rho = model->rho; a.r = model->r; a.v0 = model->v0;
    a.dt = dt;
    a.sq1mr2 = std::sqrt(1.0 - model->rho * model->rho);   // _core.pyx:379, rng.py:235
    a.milstein = milstein ? 1 : 0;
    const size_t b = (size_t)n * 8;
    return elementwise_call(device, {{s, b}, {v, b}, {u, 2 * b}}, {{s_out, b}, {v_out, b}},
                            [&](auto& d, cudaStream_t st) {
                                return hmc::launch_steps(a, (const double*)d[0], (const double*)d[1],
                                                         (const double*)d[2], n, (double*)d[3], (double*)d[4], st);
                            });
}

// the exact kernel's error codes (_core.pyx:36-40, 508-520) as ABI codes
static int exact_error(int code) {
    switch (code) {
        case 0: return HMC_OK;
        case 1: return fail(HMC_E_BESSEL, "|z| exceeds the series validity bound 50");
        case 2: return fail(HMC_E_BESSEL, "Bessel series did not converge");
        case 3: return fail(HMC_E_QUAD, "characteristic-function tail did not fall below tolerance");
        default: return fail(HMC_E_ROOT, "CDF inversion failed to reach tolerance");
    }
}

int hmc_bessel_f64(int32_t mode, double nu, const double* z, const double* aux, int64_t n, double* out,
                   int32_t device) {
    if (mode != HMC_BESSEL_SERIES && mode != HMC_BESSEL_I && mode != HMC_BESSEL_RATIO)
        return fail(HMC_E_INVALID, "unknown Bessel mode");
    if (!(nu > -1.0) || !std::isfinite(nu)) return fail(HMC_E_INVALID, "need a finite order nu > -1");
    if (n < 0 || (n > 0 && (!z || !out || (mode == HMC_BESSEL_RATIO && !aux))))
        return fail(HMC_E_INVALID, "need z[n][2], out[n][2] (and aux[n][4] for the ratio)");
    if (n == 0) return HMC_OK;
    int h_err = 0;
    const size_t zb = (size_t)n * 16, ab = mode == HMC_BESSEL_RATIO ? (size_t)n * 32 : 0;
    int rc = elementwise_call(device, {{z, zb}, {aux, ab}}, {{out, zb}, {&h_err, sizeof(int)}},
                              [&](auto& d, cudaStream_t s) {
        cudaError_t e = cudaMemsetAsync(d[3], 0, sizeof(int), s);
        if (e == cudaSuccess)
            e = hmc::launch_bessel(mode, nu, (const double*)d[0], (const double*)d[1], n, (double*)d[2], (int*)d[3], s);
        return e;
    });
    return rc ? rc : exact_error(h_err);
}

int hmc_ivlaw_phi_f64(const hmc_model* model, double v_u, double v_t, double dt, const double* a, int64_t n,
                      double* out, int32_t device) {
    int rc = check_model(model);
    if (rc) return rc;
    if (!(dt > 0.0) || !std::isfinite(dt) || !(v_u >= 0.0) || !(v_t >= 0.0))
        return fail(HMC_E_INVALID, "need dt > 0 and v_u, v_t >= 0");
    if (n < 0 || (n > 0 && (!a || !out))) return fail(HMC_E_INVALID, "need a[n] and out[n][2]");
    if (n == 0) return HMC_OK;
    int h_err = 0;
    const double dof = 4.0 * model->kappa * model->theta / (model->sigma * model->sigma);  // model.py:43-45
    rc = elementwise_call(device, {{a, (size_t)n * 8}}, {{out, (size_t)n * 16}, {&h_err, sizeof(int)}},
                          [&](auto& d, cudaStream_t s) {
        cudaError_t e = cudaMemsetAsync(d[2], 0, sizeof(int), s);
        if (e == cudaSuccess)
            e = hmc::launch_ivlaw_phi(model->kappa, model->sigma, dof, v_u, v_t, dt, (const double*)d[0], n,
                                      (double*)d[1], (int*)d[2], s);
        return e;
    });
    return rc ? rc : exact_error(h_err);
}

int hmc_ivlaw_eval_f64(const hmc_model* model, double v_u, double v_t, double dt, int32_t mode,
                       const double* in, int64_t n, double* out, double* info, int32_t device) {
    int rc = check_model(model);
    if (rc) return rc;
    if (!(dt > 0.0) || !std::isfinite(dt) || !(v_u >= 0.0) || !(v_t >= 0.0))
        return fail(HMC_E_INVALID, "need dt > 0 and v_u, v_t >= 0");
    if (mode < HMC_IVLAW_INFO || mode > HMC_IVLAW_INVERSE) return fail(HMC_E_INVALID, "unknown ivlaw mode");
    if (n < 0 || (n > 0 && (!in || !out)) || !info) return fail(HMC_E_INVALID, "need in[n], out[n] and info[4]");
    int h_err = 0;
    const double dof = 4.0 * model->kappa * model->theta / (model->sigma * model->sigma);
    const long long threads = n > 0 ? n : 1;
    // node-cache scratch: kExactCacheNodes doubles per thread, so inputs go in
    // batches of at most kBatch (~128 MB of scratch)
    constexpr long long kBatch = 1LL << 16;
    const long long batch = std::min(threads, kBatch);
    rc = elementwise_call(device, {{in, (size_t)n * 8}}, {{out, (size_t)n * 8}, {info, 32}, {&h_err, sizeof(int)}},
                          [&](auto& d, cudaStream_t s) {
        double* scratch = nullptr;
        cudaError_t e = hmc_host::pool_alloc(device, (void**)&scratch,
                                             (size_t)hmc::kExactCacheNodes * batch * sizeof(double), s);
        if (e == cudaSuccess) e = cudaMemsetAsync(d[3], 0, sizeof(int), s);
        for (long long off = 0; e == cudaSuccess && (off < n || (n == 0 && off == 0)); off += batch) {
            const long long m = n == 0 ? 0 : std::min(batch, n - off);
            e = hmc::launch_ivlaw_eval(mode, model->kappa, model->theta, model->sigma, dof, v_u, v_t, dt,
                                       (const double*)d[0] + off, m, (double*)d[1] + off, (double*)d[2], scratch,
                                       (int*)d[3], s);
            if (n == 0) break;
        }
        if (scratch) cudaFreeAsync(scratch, s);
        return e;
    });
    return rc ? rc : exact_error(h_err);
}

int hmc_exact_step_f64(const hmc_model* model, int32_t full, double s_u, double v_u, double dt,
                       const double* draws, int64_t n, double* out, int32_t device) {
    int rc = check_model(model);
    if (rc) return rc;
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(HMC_E_INVALID, "dt must be finite and > 0");
    if (!(s_u > 0.0) || !(v_u >= 0.0)) return fail(HMC_E_INVALID, "need s_u > 0 and v_u >= 0");
    if (n < 0 || (n > 0 && (!draws || !out))) return fail(HMC_E_INVALID, "need draws[n][4] and out[n][3]");
    if (n == 0) return HMC_OK;
    int h_err = 0;
    constexpr long long kBatch = 1LL << 16;   // node-cache scratch per batch (as hmc_ivlaw_eval_f64)
    const long long batch = std::min((long long)n, kBatch);
    rc = elementwise_call(device, {{draws, (size_t)n * 32}}, {{out, (size_t)n * 24}, {&h_err, sizeof(int)}},
                          [&](auto& d, cudaStream_t s) {
        double* scratch = nullptr;
        cudaError_t e = full ? hmc_host::pool_alloc(device, (void**)&scratch,
                                                    (size_t)hmc::kExactCacheNodes * batch * sizeof(double), s)
                             : cudaSuccess;
        if (e == cudaSuccess) e = cudaMemsetAsync(d[2], 0, sizeof(int), s);
        for (long long off = 0; e == cudaSuccess && off < n; off += batch)
            e = hmc::launch_exact_step(full ? 1 : 0, *model, s_u, v_u, dt, (const double*)d[0] + 4 * off,
                                       std::min(batch, n - off), (double*)d[1] + 3 * off, scratch, (int*)d[2], s);
        if (scratch) cudaFreeAsync(scratch, s);
        return e;
    });
    return rc ? rc : exact_error(h_err);
}

int hmc_philox_check(const uint32_t* ctr, int32_t n, uint32_t* out, int32_t device) {
    if (!ctr || !out || n < 1) return fail(HMC_E_INVALID, "bad philox check arguments");
    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(device));
    uint4 *d_c = nullptr, *d_o = nullptr;
    HMC_CK(cudaMalloc((void**)&d_c, (size_t)n * sizeof(uint4)));
    cudaError_t e = cudaMalloc((void**)&d_o, (size_t)n * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMemcpy(d_c, ctr, (size_t)n * sizeof(uint4), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        hmc::philox_kat_kernel<<<(n + 127) / 128, 128>>>(d_c, d_o, n);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, d_o, (size_t)n * sizeof(uint4), cudaMemcpyDeviceToHost);
    cudaFree(d_c);
    cudaFree(d_o);
    HMC_CK(e);
    return HMC_OK;
}

int hmc_fp32_paths_check(const hmc_model* model, const hmc_product* product, const hmc_sim* sim_in,
                         const float* normals, int64_t n, double* out, int32_t device) {
    if (!sim_in || !normals || !out || n < 1) return fail(HMC_E_INVALID, "bad paths check arguments");
    hmc_sim sim = *sim_in;
    sim.want_greeks = 1;
    sim.sampler = HMC_SAMPLER_PSEUDO;
    sim.precision = HMC_PREC_FP32;
    sim.sobol_bridge = 0;
    sim.n_runs = 1;
    sim.n_paths = n;
    sim.path_lo = 0;
    sim.path_hi = n;
    Prepared P;
    int rc = prepare(model, product, &sim, P);
    if (rc) return rc;
    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(device));
    const size_t zb = align_up((size_t)n * P.a.n_sim * sizeof(float2));
    const size_t ob = align_up((size_t)n * HMC_NQ * sizeof(double));
    const size_t t64 = align_up(P.st64.size() * sizeof(StepD)), t32 = P.st32.size() * sizeof(float4);
    char* buf = nullptr;
    HMC_CK(cudaMalloc((void**)&buf, zb + ob + t64 + t32));
    cudaError_t e = cudaMemcpy(buf, normals, (size_t)n * P.a.n_sim * sizeof(float2), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(buf + zb + ob, P.st64.data(), P.st64.size() * sizeof(StepD), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(buf + zb + ob + t64, P.st32.data(), t32, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        P.a.steps64 = (const StepD*)(buf + zb + ob);
        P.a.steps32 = (const float4*)(buf + zb + ob + t64);
        e = hmc::launch_given_normals(P.a, (const float2*)buf, n, (double*)(buf + zb), 0);
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, buf + zb, (size_t)n * HMC_NQ * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(buf);
    HMC_CK(e);
    return HMC_OK;
}

int hmc_box_muller_check(const uint32_t* words, int32_t n, float* out, int32_t device) {
    if (!words || !out || n < 1) return fail(HMC_E_INVALID, "bad box-muller check arguments");
    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(device));
    KernelArgs a{};
    a.f_bm2 = (float)(-2.0 * std::log(2.0));  // R = sqrt(-2 ln u1)
    a.f_cA = 0.0f;                            // second output = R sin
    a.f_cB = 1.0f;
    char* buf = nullptr;
    const size_t wb = align_up((size_t)n * sizeof(uint4)), ob = (size_t)n * 6 * sizeof(float);
    HMC_CK(cudaMalloc((void**)&buf, wb + ob));
    cudaError_t e = cudaMemcpy(buf, words, (size_t)n * sizeof(uint4), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        hmc::box_muller_kat_kernel<<<(n + 127) / 128, 128>>>((const uint4*)buf, n, a, (float*)(buf + wb));
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, buf + wb, ob, cudaMemcpyDeviceToHost);
    cudaFree(buf);
    HMC_CK(e);
    return HMC_OK;
}

int hmc_sobol_quantile_check(const uint32_t* x, int32_t n, int32_t scrambled, float* out,
                             int32_t device) {
    if (!x || !out || n < 1) return fail(HMC_E_INVALID, "bad quantile check arguments");
    for (int32_t i = 0; i < n; ++i)
        if (x[i] >= (1u << 30) || (!scrambled && x[i] == 0))
            return fail(HMC_E_INVALID, "coordinates are 30-bit, and >= 1 unless scrambled");
    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(device));
    char* buf = nullptr;
    const size_t xb = align_up((size_t)n * sizeof(uint32_t)), ob = align_up((size_t)n * sizeof(float));
    HMC_CK(cudaMalloc((void**)&buf, xb + ob));
    cudaError_t e = cudaMemcpy(buf, x, (size_t)n * sizeof(uint32_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        hmc::sobol_quantile_kernel<<<(n + 127) / 128, 128>>>((const uint32_t*)buf, n, scrambled ? 0.5f : 0.0f,
                                                            (float*)(buf + xb));
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, buf + xb, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost);
    cudaFree(buf);
    HMC_CK(e);
    return HMC_OK;
}

}  // extern "C"
