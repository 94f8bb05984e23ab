// hmc_fast.cu -- the production sm_100a path kernel (fp32 state, fp64 sums).
//
// One Monte Carlo path per thread; all state lives in registers for all
// time steps, nothing but the final fp64 tile partials touches HBM:
//
//   per path:  3 variance trajectories (v0, v0 + h, v0 - h) driven by the
//              same normals (common random numbers); log-price of each in
//              log2 units; running fixing sums; for the base trajectory also
//              sum S t (Asian pathwise Rho) and sum S expm1(+-h t) (r bumps)
//   per step:  2 correlated normals -- Box-Muller on Philox4x32-10 (pseudo)
//              or Giles' erfinv on an on-the-fly Gray-code Sobol point (QMC)
//              Milstein/Euler full-truncation update (_core.pyx:399-404),
//              algebraically regrouped so the step-shared terms are computed
//              once per thread, not once per trajectory:
//                v' = max(v (1 - k dt) + c_k + (sigma sqrt(dt) z2) sqrt(v), 0)
//                c_k = k theta dt + sigma^2/4 (dt z2^2 - dt)      (Milstein)
//                L' = L + sqrt(v) (sqrt(dt) z1 log2 e) - v dt/2 log2 e
//              S_k = 2^(L_k + log2 S0 + r t_k log2 e) only at fixing dates
//
// Bound: the MUFU (XU) pipe -- per Asian daily-fixing step 4 (lg2, sqrt,
// sin, cos) + 3 x (sqrt, ex2) = 10 MUFU ops vs ~70 other issue slots
// (DESIGN.md "roofline").
#include <cuda_runtime.h>

#include "hmc_device.cuh"
#include "hmc_launch.h"

namespace hmc {

__device__ __forceinline__ float ex2a(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2a(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sqrta(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// uniform in [1, 2) from 23 random bits (no int->float conversion on the XU pipe)
__device__ __forceinline__ float one_to_two(uint32_t x) {
    return __uint_as_float((x & 0x007fffffu) | 0x3f800000u);
}

// Box-Muller: radius from xr, angle from xa; returns the step shocks
//   z1l = sqrt(dt) z1 log2(e),   z2s = sqrt(dt) (rho z1 + sqrt(1-rho^2) zb)
__device__ __forceinline__ void box_muller(uint32_t xr, uint32_t xa, const KernelArgs& a,
                                           float& z1l, float& z2s) {
    const float u1 = 2.0f - one_to_two(xr);                 // (0, 1]
    const float R = sqrta(lg2a(u1) * a.f_bm);               // sqrt(dt) sqrt(-2 ln u1)
    const float th = fmaf(one_to_two(xa), 6.28318530717958647692f, -9.42477796076937971538f);
    const float sn = __sinf(th), cs = __cosf(th);           // th in [-pi, pi)
    z1l = (R * a.f_log2e) * cs;
    z2s = fmaf(R * a.f_rho, cs, (R * a.f_sq1mr2) * sn);
}

// Standard-normal quantile of the Sobol coordinate x * 2^-30 (x in [1, 2^30)):
// Giles' single-precision erfinv, z = sqrt(2) erfinv(2u - 1), with 4u(1-u)
// formed from the distance to the nearer end so the tails keep precision.
__device__ __forceinline__ float sobol_normal(uint32_t x) {
    const int m = (int)(2u * x) - (1 << 30);                // (2u - 1) 2^30
    const uint32_t t = min(x, (1u << 30) - x);              // min(u, 1-u) 2^30
    const float xs = (float)m * 9.31322574615478515625e-10f;
    const float tf = (float)t * 9.31322574615478515625e-10f;
    float w = -0.69314718055994530942f * lg2a(4.0f * tf * (1.0f - tf));
    float p;
    if (w < 5.0f) {
        w = w - 2.5f;
        p = 2.81022636e-08f;
        p = fmaf(p, w, 3.43273939e-07f);
        p = fmaf(p, w, -3.5233877e-06f);
        p = fmaf(p, w, -4.39150654e-06f);
        p = fmaf(p, w, 0.00021858087f);
        p = fmaf(p, w, -0.00125372503f);
        p = fmaf(p, w, -0.00417768164f);
        p = fmaf(p, w, 0.246640727f);
        p = fmaf(p, w, 1.50140941f);
    } else {
        w = sqrta(w) - 3.0f;
        p = -0.000200214257f;
        p = fmaf(p, w, 0.000100950558f);
        p = fmaf(p, w, 0.00134934322f);
        p = fmaf(p, w, -0.00367342844f);
        p = fmaf(p, w, 0.00573950773f);
        p = fmaf(p, w, -0.0076224613f);
        p = fmaf(p, w, 0.00943887047f);
        p = fmaf(p, w, 1.00167406f);
        p = fmaf(p, w, 2.83297682f);
    }
    return 1.41421356237309504880f * p * xs;
}

struct PathState32 {
    float v0, L0, A0;  // base trajectory
    float vu, Lu, Au;  // v0 + h
    float vd, Ld, Ad;  // v0 - h (floored at 0)
    float T1, Dp, Dm;  // base: sum S t, sum S expm1(h t), sum S expm1(-h t)
};

template <bool GREEKS>
__device__ __forceinline__ void traj_step(float& v, float& L, float z1l, float sz2, float ck,
                                          const KernelArgs& a) {
    const float s = sqrta(v);
    L = fmaf(s, z1l, L);
    L = fmaf(v, a.f_nhdt2, L);
    v = fmaxf(fmaf(s, sz2, fmaf(v, a.f_omkdt, ck)), 0.0f);
}

template <bool GREEKS>
__device__ __forceinline__ void advance(PathState32& st, float z1l, float z2s, const KernelArgs& a) {
    const float sz2 = a.f_sigma * z2s;
    const float ck = fmaf(z2s * z2s, a.f_cmil, a.f_ck0);
    traj_step<GREEKS>(st.v0, st.L0, z1l, sz2, ck, a);
    if (GREEKS) {
        traj_step<GREEKS>(st.vu, st.Lu, z1l, sz2, ck, a);
        traj_step<GREEKS>(st.vd, st.Ld, z1l, sz2, ck, a);
    }
}

template <bool GREEKS>
__device__ __forceinline__ void fixing(PathState32& st, const float4 tab, const KernelArgs& a) {
    const float rt2 = fmaf(tab.x, a.f_rl2, a.f_l2s0);
    const float S = ex2a(st.L0 + rt2);
    st.A0 += S;
    if (GREEKS) {
        st.T1 = fmaf(S, tab.x, st.T1);
        st.Dp = fmaf(S, tab.y, st.Dp);
        st.Dm = fmaf(S, tab.z, st.Dm);
        st.Au += ex2a(st.Lu + rt2);
        st.Ad += ex2a(st.Ld + rt2);
    }
}

template <int FIX, bool GREEKS>
__device__ __forceinline__ void step(PathState32& st, int k, float z1l, float z2s,
                                     const KernelArgs& a) {
    advance<GREEKS>(st, z1l, z2s, a);
    if (FIX == kFixEvery) {
        fixing<GREEKS>(st, __ldg(a.steps32 + k), a);
    } else if (FIX == kFixTable) {
        const float4 tab = __ldg(a.steps32 + k);
        if (tab.w != 0.0f) fixing<GREEKS>(st, tab, a);
    }
}

template <int FIX, bool GREEKS, int SAMPLER>
__global__ void __launch_bounds__(kTile) fast_greeks_kernel(const KernelArgs a,
                                                            double* __restrict__ tiles,
                                                            long long n_tiles) {
    const int run = blockIdx.y;
    const long long path = a.path_lo + (long long)blockIdx.x * kTile + threadIdx.x;
    const bool live = path < a.path_hi;
    const long long p = live ? path : a.path_lo;

    PathState32 st;
    st.v0 = (float)a.v0;
    st.vu = (float)a.v0_up;
    st.vd = (float)a.v0_dn;
    st.L0 = st.Lu = st.Ld = 0.0f;
    st.A0 = st.Au = st.Ad = 0.0f;
    st.T1 = st.Dp = st.Dm = 0.0f;

    if (SAMPLER == HMC_SAMPLER_PSEUDO) {
        // Philox counter (pair j, path lo, path hi, run); key = root_key(seed)
        const uint32_t c1 = (uint32_t)p, c2 = (uint32_t)((unsigned long long)p >> 32);
        const uint32_t c3 = (uint32_t)run;
        const int npairs = a.n_sim >> 1;
        int k = 1;
#pragma unroll 1
        for (int j = 0; j < npairs; ++j) {
            const uint4 x = philox4x32_10((uint32_t)j, c1, c2, c3, a);
            float z1l, z2s;
            box_muller(x.x, x.y, a, z1l, z2s);
            step<FIX, GREEKS>(st, k, z1l, z2s, a);
            box_muller(x.z, x.w, a, z1l, z2s);
            step<FIX, GREEKS>(st, k + 1, z1l, z2s, a);
            k += 2;
        }
        if (a.n_sim & 1) {
            const uint4 x = philox4x32_10((uint32_t)npairs, c1, c2, c3, a);
            float z1l, z2s;
            box_muller(x.x, x.y, a, z1l, z2s);
            step<FIX, GREEKS>(st, k, z1l, z2s, a);
        }
    } else {
        // engine.py:100: run r uses Sobol rows 1 + r*n_paths + path
        const uint32_t n = (uint32_t)(1 + (long long)run * a.n_paths + p);
        const uint32_t gray = n ^ (n >> 1);
        const float c1 = a.f_sqdt * a.f_log2e;
#pragma unroll 1
        for (int k = 1; k <= a.n_sim; ++k) {
            const float za = sobol_normal(sobol_coord(gray, a.sobol_v, a.sobol_dim, 2 * (k - 1)));
            const float zb = sobol_normal(sobol_coord(gray, a.sobol_v, a.sobol_dim, 2 * k - 1));
            const float z1l = c1 * za;
            const float z2s = a.f_sqdt * fmaf(a.f_rho, za, a.f_sq1mr2 * zb);
            step<FIX, GREEKS>(st, k, z1l, z2s, a);
        }
    }
    if (FIX == kFixLast) fixing<GREEKS>(st, __ldg(a.steps32 + a.n_sim), a);

    const float inv_n = 1.0f / (float)a.n_avg;
    const float A = st.A0 * inv_n;
    double q[kNQ];
    if (GREEKS) {
        greeks_epilogue<float>(a, A, st.T1 * inv_n, st.Au * inv_n, st.Ad * inv_n,
                               fmaf(st.Dp, inv_n, A), fmaf(st.Dm, inv_n, A), q);
    } else {
        const float K = (float)a.K, disc = (float)a.disc;
        q[0] = (double)(a.is_call ? disc * pos_part(A - K) : disc * pos_part(K - A));
#pragma unroll
        for (int i = 1; i < kNQ; ++i) q[i] = 0.0;
    }
    if (!live) {
#pragma unroll
        for (int i = 0; i < kNQ; ++i) q[i] = 0.0;
    }
    tile_reduce_store(q, tiles + ((size_t)run * n_tiles + blockIdx.x) * kNW);
}

template <int FIX, bool GREEKS>
static void launch_sampler(const KernelArgs& a, double* d_tiles, long long n_tiles, dim3 grid,
                           cudaStream_t s) {
    if (a.sampler == HMC_SAMPLER_PSEUDO)
        fast_greeks_kernel<FIX, GREEKS, HMC_SAMPLER_PSEUDO><<<grid, kTile, 0, s>>>(a, d_tiles, n_tiles);
    else
        fast_greeks_kernel<FIX, GREEKS, HMC_SAMPLER_SOBOL><<<grid, kTile, 0, s>>>(a, d_tiles, n_tiles);
}

template <int FIX>
static void launch_greeks_flag(const KernelArgs& a, double* d_tiles, long long n_tiles,
                               dim3 grid, cudaStream_t s) {
    if (a.want_greeks)
        launch_sampler<FIX, true>(a, d_tiles, n_tiles, grid, s);
    else
        launch_sampler<FIX, false>(a, d_tiles, n_tiles, grid, s);
}

cudaError_t launch_fast_greeks(const KernelArgs& a, double* d_tiles, long long n_tiles,
                               cudaStream_t s) {
    dim3 grid((unsigned)n_tiles, (unsigned)a.n_runs);
    switch (a.fix_mode) {
        case kFixLast: launch_greeks_flag<kFixLast>(a, d_tiles, n_tiles, grid, s); break;
        case kFixEvery: launch_greeks_flag<kFixEvery>(a, d_tiles, n_tiles, grid, s); break;
        default: launch_greeks_flag<kFixTable>(a, d_tiles, n_tiles, grid, s); break;
    }
    return cudaGetLastError();
}

}  // namespace hmc
