// hmc_device.cuh -- device building blocks shared by the sm_100a path kernels.
//
//   * KernelArgs: everything a path kernel reads (by value -> constant bank)
//   * Philox4x32-10 counter RNG (production stream)
//   * SplitMix64 counter RNG + Acklam/Halley inverse normal in fp64
//     (the reference stream, rng.py:38-132 / _core.pyx:57-109)
//   * Gray-code Sobol coordinate (scipy.stats.qmc.Sobol, unscrambled, 30 bit)
//   * fixed-order tile reduction of per-path quantities to fp64 partials
#pragma once

#include <cstdint>

#include "../../include/hmc.h"

// Device-side bounds checks of every data- or table-dependent index
// (shared tables, histograms, skeletons, node caches, step tables, tile
// writes), compiled in only for the checked build (HMC_DEBUG_BOUNDS=1,
// paper_2309_10477_b200/_variants/libhmc_checked.so, tests/test_gpu_checked.py):
// the stand-in for compute-sanitizer, which is closed on this GPU pool.
#if defined(HMC_DEBUG_BOUNDS) && HMC_DEBUG_BOUNDS
#include <cassert>
#define HMC_DCHECK(cond) assert(cond)
#else
#define HMC_DCHECK(cond) ((void)0)
#endif

namespace hmc {

constexpr int kTile = HMC_TILE;
// runs map to gridDim.y; longer run lists go out in launches of this many
constexpr int kMaxRunsPerLaunch = 65535;
constexpr int kNQ = HMC_NQ;
constexpr int kNW = HMC_NW;
constexpr int kWarps = kTile / 32;
constexpr int kSobolBits = 30;

enum FixMode : int {
    kFixLast = 0,   // one fixing at the last simulated step (european)
    kFixEvery = 1,  // every step is a fixing date (daily-fixing asian)
    kFixTable = 2   // fixing flags from the step table
};

// Per-step table entry, built on the host in fp64 (t_k = k*T/n_steps exactly
// as _core.pyx:406), also shipped as fp32.
//   x = t_k, y = expm1(+h_r t_k), z = expm1(-h_r t_k), w = 1 if k is a fixing
struct StepD {
    double t, e1p, e1m, fix;
};

// Sobol Brownian bridge (hmc_sim.sobol_bridge = S > 0).  Skeleton points
// j = 0..S sit at steps b_j = floor(j n_sim / S) (point 0 = origin, W = 0);
// node i (level order, dimension pair i) sets
//   W(b_m) = W(b_l) + a (W(b_r) - W(b_l)) + sd z      (root: l = r = 0)
// and step k of segment j (b_{j-1} < k <= b_j) draws its increment as
//   dW_k = (W(b_j) - W_{k-1}) alpha_k + beta_k z
// with alpha_k = 1 / (b_j - k + 1), beta_k = sqrt(dt (b_j - k) / (b_j - k + 1));
// segment ends (k = b_j) have alpha = 1, beta = 0 and consume no pair; the
// other steps take the next pair S, S+1, ... in time order.
struct BridgeNodeD {
    double a, sd;
    int m, l, r, pad;
};
struct BridgeStepD {
    double alpha, beta;
    int j, consume;
};
struct BridgeNode {
    float a, sd;
    int m, lr;  // l | r << 16
};
struct BridgeStep {  // fp32: the segment index and the pair flag are implied
    float alpha, beta;  // (beta == 0 exactly at segment ends)
};

struct KernelArgs {
    // model (HestonParams) and product (OptionSpec)
    double kappa, theta, sigma, rho, r, v0;
    double s0, T, K;
    double v0_up, v0_dn, h_spot, h_r;
    double dt, sq1mr2;
    double disc, disc_up, disc_dn;  // exp(-r T), exp(-(r +- h_r) T)  (host libm)
    int n_steps;     // grid size (dt = T / n_steps)
    int n_sim;       // steps actually simulated (last fixing for asians)
    int n_avg;       // number of fixing dates
    int fix_mode;
    int is_asian, is_call, want_greeks, milstein;
    int sampler;
    int n_runs;
    int run0;        // global index of the launch's first run (blockIdx.y = run - run0)
    long long n_paths, path_lo, path_hi;
    // root_key(seed) (rng.py:46-47): per-run stream key derivation for both
    // the Philox counter (fp32) and the SplitMix64 stream (fp64)
    unsigned long long root_key;
    // tables (device pointers)
    const StepD* steps64;       // [n_steps + 1]
    const float4* steps32;      // [n_steps + 1] fixing weights, see FixW
    const uint32_t* sobol_v;    // [30][sobol_dim]
    int sobol_dim;
    int sobol_scramble;         // random digital shift per (run, dimension)
    int bridge_segments;        // S: Sobol Brownian bridge (0 = time order)
    const BridgeNodeD* bridge_nodes64;  // [S]
    const BridgeStepD* bridge_steps64;  // [n_sim + 1]
    const BridgeNode* bridge_nodes32;   // [S]
    const BridgeStep* bridge_steps32;   // [n_sim + 1]
    // fp32 derived constants (host-computed in fp64, rounded once)
    float f_omkdt;   // 1 - kappa dt
    float f_ck0;     // kappa theta dt - milstein * sigma^2 dt / 4
    float f_cmil;    // milstein * sigma^2 / 4
    float f_sigma;
    float f_nhdt2;   // -0.5 dt log2(e)
    float f_bm2;     // -2 ln(2) dt log2(e)^2: R' = sqrt(f_bm2 lg2 u1) = sqrt(dt) |z| log2 e
    float f_cA;      // sigma rho / log2(e)
    float f_cB;      // sigma sqrt(1 - rho^2) / log2(e)
    float f_cmil2;   // milstein / 4  (multiplies (sigma sqrt(dt) z2)^2)
    float f_log2e;
    float f_rho, f_sq1mr2;
    float f_sqdt;    // sqrt(dt)
    // Sobol drivers: the quantile's per-coordinate scales k (sqrt(2) folded in:
    // .x -> z1l, .y -> sigma sqrt(dt) sqrt(1 - rho^2) z_b), -2k, and
    // sigma rho / log2(e); host-computed in the float order the kernel used
    float2 f_sob_k, f_sob_k2;
    float f_sob_crho;
    // fp32 epilogue constants (no double->float conversions or divisions on
    // the device: F2F and MUFU.RCP share the MIO queue with the path MUFUs)
    float f_v0, f_vu, f_vd;
    float f_K, f_T, f_disc, f_disc_up, f_disc_dn, f_ddisc;  // f_ddisc = disc_up - disc_dn (fp64)
    float f_inv_s0, f_up_ratio, f_dn_ratio;   // 1/S0, (S0 +- h)/S0
    float f_inv_2h, f_inv_dv, f_inv_2hr;      // 1/(2 h_S), 1/(v0u - v0d), 1/(2 h_r)
    float f_inv_navg;
};

// fp32 fixing weights of step k (host-computed in fp64):
//   x = E_k = S0 e^{r t_k},  y = E_k t_k,  z = E_k expm1(h_r t_k),
//   w = E_k expm1(-h_r t_k);  all zero when k is not a fixing date.
// With P = 2^{L_k} (L = r-free log2 price ratio), S_k = P E_k.

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11) with a fixed key: the
// round keys are compile-time immediates of the LOP3s (no constant loads in
// the step loop).  Streams are separated through the counter instead:
//   (c0, c1, c2, c3) = (step pair, path, lo32, hi32 of key_run),
//   key_run = derive(root_key(seed), run)  -- the reference's per-run key
//   derivation (engine.py:96, rng.py:46-52), 64 bits of stream id.
// ---------------------------------------------------------------------------
constexpr uint32_t kPhiloxK0 = 0xA4093822u, kPhiloxK1 = 0x299F31D0u;

// 32x32 -> 64 multiply as ONE IMAD.WIDE.U32 (the plain C++ form makes ptxas
// add a zero high word after every multiply)
__device__ __forceinline__ void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
    asm("{\n\t.reg .b64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%1, %0}, t;\n\t}"
        : "=r"(hi), "=r"(lo) : "r"(a), "r"(b));
}


__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                               uint32_t c3) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t k0 = kPhiloxK0 + (uint32_t)i * 0x9E3779B9u;
        const uint32_t k1 = kPhiloxK1 + (uint32_t)i * 0xBB67AE85u;
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo32(0xD2511F53u, c0, hi0, lo0);
        mulhilo32(0xCD9E8D57u, c2, hi1, lo1);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

// ---------------------------------------------------------------------------
// Reference stream: SplitMix64 (rng.py:38-65, _core.pyx:57-68)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ unsigned long long derive(unsigned long long parent,
                                                              unsigned long long index) {
    return mix64(parent ^ mix64(index + 0xD1B54A32D192ED03ULL));
}
__host__ __device__ __forceinline__ double uniform_at(unsigned long long key,
                                                      unsigned long long i) {
    return (double)(mix64(key + (i + 1) * 0x9E3779B97F4A7C15ULL) >> 11) *
           (1.0 / 9007199254740992.0);
}

// random digital shift (30 bits) of dimension d for the run with key key_run
__host__ __device__ __forceinline__ uint32_t sobol_shift(unsigned long long key_run, int d) {
    return (uint32_t)(mix64(key_run ^ ((unsigned long long)(d + 1) * 0x9E3779B97F4A7C15ULL)) >> 34);
}

// ---------------------------------------------------------------------------
// Sobol coordinate d of Gray-code point n: XOR of v[b][d] over the set bits
// of gray(n) = n ^ (n >> 1), as 30-bit integer.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t sobol_coord(uint32_t gray, const uint32_t* __restrict__ v,
                                                int dim, int d) {
    uint32_t x = 0;
#pragma unroll
    for (int b = 0; b < kSobolBits; ++b) {
        if ((gray >> b) & 1u) x ^= __ldg(v + b * dim + d);
    }
    return x;
}

// ---------------------------------------------------------------------------
// Fixed-order tile reduction: every thread holds kNQ per-path values; write
// {sum x, sum x^2} per quantity for the tile.  Butterfly shuffles then warps
// in index order -- deterministic for a given tile content.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tile_reduce_store(const double (&q)[kNQ], double* __restrict__ out) {
    __shared__ double red[kWarps][kNW];
    double w[kNW];
#pragma unroll
    for (int i = 0; i < kNQ; ++i) {
        w[2 * i] = q[i];
        w[2 * i + 1] = q[i] * q[i];
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
#pragma unroll
        for (int i = 0; i < kNW; ++i) w[i] += __shfl_xor_sync(0xffffffffu, w[i], off);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kNW; ++i) red[warp][i] = w[i];
    }
    __syncthreads();
    HMC_DCHECK(blockDim.x == kTile);
    if (threadIdx.x < kNW) {
        double s = red[0][threadIdx.x];
#pragma unroll
        for (int k = 1; k < kWarps; ++k) s += red[k][threadIdx.x];
        out[threadIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------
// Per-path estimators (engine.py:47-68 for price / pathwise Delta / pathwise
// Rho; CRN finite differences for the rest, test_products.py:101-137).
//   A      underlying: average over fixings (asian) or S_T (european)
//   tw     (1/N) sum S_k t_k                     (Asian pathwise Rho)
//   Au/Ad  underlyings of the v0 +/- trajectories (Vega)
//   Rp/Rm  underlyings under r +/- h_r by exact rescaling:
//          S_k(r+h) = S_k(r) e^{h t_k}  (r enters the log-Euler drift only)
// S0 +/- h is an exact rescaling too: S_k(S0+h) = S_k (S0+h)/S0, so the
// pathwise Delta of the bumped path equals disc*A/S0 on its exercise set.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T pos_part(T x) {
    return x > T(0) ? x : T(0);
}

template <typename T>
__device__ __forceinline__ void greeks_epilogue(const KernelArgs& a, T A, T tw, T Au, T Ad,
                                                T Rp, T Rm, double (&q)[kNQ]) {
    const T K = (T)a.K, disc = (T)a.disc;
    auto payoff = [&](T x, T d) -> T { return a.is_call ? d * pos_part(x - K) : d * pos_part(K - x); };
    q[HMC_Q_PRICE] = (double)payoff(A, disc);
#pragma unroll
    for (int i = 1; i < kNQ; ++i) q[i] = 0.0;
    if (!a.want_greeks) return;
    const T S0 = (T)a.s0, h = (T)a.h_spot;
    const bool itm = A > K;
    if (itm) {
        q[HMC_Q_DELTA] = (double)(disc * A / S0);
        q[HMC_Q_RHO] = a.is_asian ? (double)(disc * (tw - (T)a.T * (A - K)))
                                  : (double)(disc * K * (T)a.T);
    }
    const T Aup = A * ((S0 + h) / S0), Adn = A * ((S0 - h) / S0);
    const T ind = (T)((Aup > K) ? 1 : 0) - (T)((Adn > K) ? 1 : 0);
    q[HMC_Q_GAMMA] = (double)(ind * (disc * A / S0) / (T(2) * h));
    q[HMC_Q_DELTA_FD] = (double)((payoff(Aup, disc) - payoff(Adn, disc)) / (T(2) * h));
    q[HMC_Q_VEGA] = (double)((payoff(Au, disc) - payoff(Ad, disc)) / (T)(a.v0_up - a.v0_dn));
    q[HMC_Q_RHO_FD] = (double)((payoff(Rp, (T)a.disc_up) - payoff(Rm, (T)a.disc_dn)) /
                               (T(2) * (T)a.h_r));
}

// fp32 twin of greeks_epilogue: same estimators, host-precomputed
// reciprocals instead of divisions
// fp32 per-path estimators.  Au, Ad are the v0-bumped averages; dp, dm the
// r-bumped underlyings' offsets Rp - A, Rm - A (accumulated directly).  The FD Greeks of
// a call are evaluated in cancellation-free form: where both bumped
// underlyings are in the money the finite difference is linear in the path,
//   delta_fd = d A / S0                     ((A(1+e) - A(1-e)) / 2h = A / S0)
//   rho_fd   = ((A - K) (d+ - d-) + d+ dp - d- dm) / 2h_r
// with d+ - d- from the host in fp64 (rounding d+ and d- separately and
// subtracting cost ~3e-5 relative bias in rho_fd); on the band where only
// the up-bumped one is, it is the single term d+ (Rp - K) / 2h.
__device__ __forceinline__ void greeks_epilogue_f32(const KernelArgs& a, float A, float tw, float Au,
                                                    float Ad, float dp, float dm, double (&q)[kNQ]) {
    const float K = a.f_K, disc = a.f_disc;
    auto payoff = [&](float x, float d) -> float {
        return a.is_call ? d * pos_part(x - K) : d * pos_part(K - x);
    };
    q[HMC_Q_PRICE] = (double)payoff(A, disc);
    const float dA = disc * A * a.f_inv_s0;
    const bool itm = A > K;
    q[HMC_Q_DELTA] = itm ? (double)dA : 0.0;
    q[HMC_Q_RHO] = itm ? (a.is_asian ? (double)(disc * (tw - a.f_T * (A - K))) : (double)(disc * K * a.f_T))
                       : 0.0;
    const float Aup = A * a.f_up_ratio, Adn = A * a.f_dn_ratio;
    const float ind = (float)((Aup > K) ? 1 : 0) - (float)((Adn > K) ? 1 : 0);
    q[HMC_Q_GAMMA] = (double)(ind * dA * a.f_inv_2h);
    const float Rp = A + dp, Rm = A + dm;
    if (a.is_call) {
        // both v0-bumped averages in the money: d (Au - Ad) / dv, the
        // difference taken before scaling (as the surface kernel does)
        q[HMC_Q_VEGA] = (Au > K && Ad > K) ? (double)(disc * (Au - Ad) * a.f_inv_dv)
                                           : (double)((payoff(Au, disc) - payoff(Ad, disc)) * a.f_inv_dv);
        q[HMC_Q_DELTA_FD] = Adn > K ? (double)dA : (double)(disc * pos_part(Aup - K) * a.f_inv_2h);
        q[HMC_Q_RHO_FD] =
            Rm > K ? (double)(fmaf(A - K, a.f_ddisc, fmaf(a.f_disc_up, dp, -a.f_disc_dn * dm)) * a.f_inv_2hr)
                   : (double)(a.f_disc_up * pos_part(Rp - K) * a.f_inv_2hr);
    } else {
        q[HMC_Q_VEGA] = (double)((payoff(Au, disc) - payoff(Ad, disc)) * a.f_inv_dv);
        q[HMC_Q_DELTA_FD] = (double)((payoff(Aup, disc) - payoff(Adn, disc)) * a.f_inv_2h);
        q[HMC_Q_RHO_FD] = (double)((payoff(Rp, a.f_disc_up) - payoff(Rm, a.f_disc_dn)) * a.f_inv_2hr);
    }
}

}  // namespace hmc
