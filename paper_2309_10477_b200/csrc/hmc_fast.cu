// hmc_fast.cu -- the production sm_100a path kernel (fp32 state, fp64 sums).
//
// One Monte Carlo path per thread; all state lives in registers for all
// time steps, nothing but the final fp64 tile partials touches HBM:
//
//   per path:  3 variance trajectories (v0, v0 + h, v0 - h) driven by the
//              same normals (common random numbers); r-free log2 price ratio
//              L of each; running fixing sums; for the base trajectory also
//              sum S t (Asian pathwise Rho) and sum S expm1(+-h t) (r bumps)
//   per step:  2 correlated normals -- Box-Muller on Philox4x32-10 (pseudo)
//              or Giles' erfinv on an on-the-fly Gray-code Sobol point (QMC)
//              Milstein/Euler full-truncation update (_core.pyx:399-404),
//              algebraically regrouped so the step-shared terms are computed
//              once per thread, not once per trajectory:
//                v' = max(v (1 - k dt) + c_k + (sigma sqrt(dt) z2) sqrt(v), 0)
//                c_k = k theta dt + sigma^2/4 ((sqrt(dt) z2)^2 - dt)  (Milstein)
//                L' = L + sqrt(v) (sqrt(dt) z1 log2 e) - v dt/2 log2 e
//              S_k = E_k 2^{L_k}, E_k = S0 e^{r t_k}, only at fixing dates
//
// The loop is bound jointly by instruction issue and the MUFU (XU) pipe
// (DESIGN.md "roofline").  Build-time switches trade MUFU ops for FMA-pipe
// polynomials:
//   HMC_SINCOS_POLY  Box-Muller angle via sin/cos polynomials (-2 MUFU/step)
//   HMC_EX2_POLY     number of trajectories (0..3) whose 2^L uses a
//                    polynomial instead of MUFU.EX2 (-1 MUFU/step each)
#include <cuda_runtime.h>

#include "hmc_device.cuh"
#include "hmc_launch.h"

#ifndef HMC_SINCOS_POLY
#define HMC_SINCOS_POLY 0
#endif
#ifndef HMC_EX2_POLY
#define HMC_EX2_POLY 0
#endif
#ifndef HMC_SQRT_RSQ
#define HMC_SQRT_RSQ 0
#endif
#ifndef HMC_PIPELINE_RNG
#define HMC_PIPELINE_RNG 0   // generate step pair j+1's Philox block during pair j
#endif
#ifndef HMC_TRIPACK
#define HMC_TRIPACK 1        // 3 steps per Philox block (23-bit radius, 19/18-bit angle)
#endif
#ifndef HMC_UNROLL_PAIRS
#define HMC_UNROLL_PAIRS 1
#endif
#define HMC_PRAGMA_(x) _Pragma(#x)
#define HMC_UNROLL_(n) HMC_PRAGMA_(unroll n)
#define HMC_UNROLL(n) HMC_UNROLL_(n)
#ifndef HMC_MIN_BLOCKS
// 7 resident blocks (28 warps) per SM, up to 72 registers: fewer warps
// contend less for the MIO/MUFU queue (tools/kernel_variants.py sweep:
// 48 warps 11.1 ms, 28 warps 10.76 ms per 2^24 x 252 launch)
#define HMC_MIN_BLOCKS 7
#endif
#define HMC_BOUNDS __launch_bounds__(kTile, HMC_MIN_BLOCKS)

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
__device__ __forceinline__ float rsqrta(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// sqrt(v) of a variance (v >= 0): MUFU.SQRT, or v * MUFU.RSQ(v) (exact 0 at v = 0)
__device__ __forceinline__ float sqrt_var(float v) {
#if HMC_SQRT_RSQ
    return v * rsqrta(fmaxf(v, 1e-30f));
#else
    return sqrta(v);
#endif
}

// 2^x on the FMA pipe: x = j + f, |f| <= 1/2, 2^f by a degree-6 Taylor
// polynomial (rel. err 1.6e-7), exponent added with one LEA.
__device__ __forceinline__ float ex2_poly(float x) {
    const float magic = 12582912.0f;  // 1.5 * 2^23: rounds to integer
    x = fmaxf(x, -125.0f);            // keep the exponent add in range
    const float m = x + magic;
    const float f = x - (m - magic);
    float p = 1.5403530393381606e-4f;
    p = fmaf(p, f, 1.3333558146428441e-3f);
    p = fmaf(p, f, 9.6181291076284772e-3f);
    p = fmaf(p, f, 5.5504108664821576e-2f);
    p = fmaf(p, f, 2.4022650695910071e-1f);
    p = fmaf(p, f, 6.9314718055994531e-1f);
    p = fmaf(p, f, 1.0f);
    return __uint_as_float(__float_as_uint(p) + (__float_as_uint(m) << 23));
}

template <int POLY>
__device__ __forceinline__ float ex2_sel(float x) {
    if (POLY) return ex2_poly(x);
    return ex2a(x);
}

// uniform in [1, 2) from the top 23 bits of x: one LEA.HI
__device__ __forceinline__ float one_to_two(uint32_t x) {
    return __uint_as_float((x >> 9) + 0x3f800000u);
}

// Box-Muller on two Philox words; returns the step shocks
//   z1l = sqrt(dt) z1 log2(e),   sz2 = sigma sqrt(dt) (rho z1 + sqrt(1-rho^2) zb)
__device__ __forceinline__ void sincos_turns(float fa, uint32_t sgn, float& sn, float& cs) {
#if HMC_SINCOS_POLY
    // angle in [-pi/2, pi/2) from fa in [1, 2), sin/cos by Taylor polynomials
    // (abs err 6e-8); a random sign bit (bit 31 of sgn) flips cos to cover
    // the left half circle
    const float r = fmaf(fa, 2.0f, -3.0f);                   // [-1, 1)
    const float r2 = r * r;
    float ps = -3.598843235212084e-06f;
    ps = fmaf(ps, r2, 1.6044118478735975e-04f);
    ps = fmaf(ps, r2, -4.681754135318687e-03f);
    ps = fmaf(ps, r2, 7.969262624616703e-02f);
    ps = fmaf(ps, r2, -6.459640975062462e-01f);
    ps = fmaf(ps, r2, 1.5707963267948966f);
    sn = ps * r;
    float pc = 4.710874778818169e-07f;
    pc = fmaf(pc, r2, -2.5202042373060596e-05f);
    pc = fmaf(pc, r2, 9.192602748394263e-04f);
    pc = fmaf(pc, r2, -2.0863480763352957e-02f);
    pc = fmaf(pc, r2, 2.53669507901048e-01f);
    pc = fmaf(pc, r2, -1.2337005501361697f);
    pc = fmaf(pc, r2, 1.0f);
    cs = __uint_as_float(__float_as_uint(pc) ^ (sgn & 0x80000000u));
#else
    const float th = fmaf(fa, 6.28318530717958647692f, -9.42477796076937971538f);
    sn = __sinf(th);                                         // th in [-pi, pi)
    cs = __cosf(th);
    (void)sgn;
#endif
}

__device__ __forceinline__ void box_muller_f(float fr, float fa, uint32_t sgn, const KernelArgs& a,
                                             float& z1l, float& sz2) {
    const float u1 = 2.0f - fr;                              // (0, 1]
    const float R = sqrta(lg2a(u1) * a.f_bm2);               // sqrt(dt) sqrt(-2 ln u1) log2 e
    float sn, cs;
    sincos_turns(fa, sgn, sn, cs);
    z1l = R * cs;
    sz2 = R * fmaf(a.f_cA, cs, a.f_cB * sn);
}

// three Box-Muller steps from one 128-bit Philox block: radii from the top
// 23 bits of w0, w1, w2; angles from w3[31:13], w3[12:0]|w0[8:3],
// w1[8:0]|w2[8:0] (19, 19 and 18 bits); w0[2:0] left as spare sign bits
__device__ __forceinline__ void tri_unpack(const uint4 w, float (&fr)[3], float (&fa)[3]) {
    fr[0] = one_to_two(w.x);
    fr[1] = one_to_two(w.y);
    fr[2] = one_to_two(w.z);
    fa[0] = __uint_as_float(((w.w >> 9) & 0x007FFFF0u) | 0x3f800000u);
    fa[1] = __uint_as_float(((w.w << 10) & 0x007FFC00u) | ((w.x << 1) & 0x000003F0u) | 0x3f800000u);
    fa[2] = __uint_as_float(((w.y << 14) & 0x007FC000u) | ((w.z << 5) & 0x00003FE0u) | 0x3f800000u);
}

__device__ __forceinline__ void box_muller(uint32_t xr, uint32_t xa, const KernelArgs& a,
                                           float& z1l, float& sz2) {
    const float u1 = 2.0f - one_to_two(xr);                  // (0, 1]
    const float R = sqrta(lg2a(u1) * a.f_bm2);               // sqrt(dt) sqrt(-2 ln u1) log2 e
    float sn, cs;
#if HMC_SINCOS_POLY
    // angle in [-pi/2, pi/2) from the top 23 bits, sin/cos by Taylor
    // polynomials (abs err 6e-8), cos sign from a spare (low) bit of xr
    const float r = fmaf(one_to_two(xa), 2.0f, -3.0f);       // [-1, 1)
    const float r2 = r * r;
    float ps = -3.598843235212084e-06f;
    ps = fmaf(ps, r2, 1.6044118478735975e-04f);
    ps = fmaf(ps, r2, -4.681754135318687e-03f);
    ps = fmaf(ps, r2, 7.969262624616703e-02f);
    ps = fmaf(ps, r2, -6.459640975062462e-01f);
    ps = fmaf(ps, r2, 1.5707963267948966f);
    sn = ps * r;
    float pc = 4.710874778818169e-07f;
    pc = fmaf(pc, r2, -2.5202042373060596e-05f);
    pc = fmaf(pc, r2, 9.192602748394263e-04f);
    pc = fmaf(pc, r2, -2.0863480763352957e-02f);
    pc = fmaf(pc, r2, 2.53669507901048e-01f);
    pc = fmaf(pc, r2, -1.2337005501361697f);
    pc = fmaf(pc, r2, 1.0f);
    cs = __uint_as_float(__float_as_uint(pc) ^ (xr << 31));
#else
    const float th = fmaf(one_to_two(xa), 6.28318530717958647692f, -9.42477796076937971538f);
    sn = __sinf(th);                                         // th in [-pi, pi)
    cs = __cosf(th);
#endif
    z1l = R * cs;
    sz2 = R * fmaf(a.f_cA, cs, a.f_cB * sn);
}

// Standard-normal quantile of the Sobol coordinate u = (x + half) 2^-30:
// Giles' single-precision erfinv, z = sqrt(2) erfinv(2u - 1), with 4u(1-u)
// formed from the distance to the nearer end so the tails keep precision.
// half = 0 for the reference's unscrambled points (x >= 1 always); half = 1/2
// for digitally shifted points, where x = 0 can occur.
__device__ __forceinline__ float sobol_normal(uint32_t x, float half) {
    const int m = (int)(2u * x) - (1 << 30);                // (2u - 1) 2^30 - 2 half
    const uint32_t t = min(x, (1u << 30) - x);              // min(u, 1-u) 2^30 (- half)
    const float xs = fmaf((float)m, 9.31322574615478515625e-10f, half * 1.86264514923095703125e-09f);
    const float tf = ((float)t + half) * 9.31322574615478515625e-10f;
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

__device__ __forceinline__ void traj_step(float& v, float& L, float z1l, float sz2, float ck,
                                          const KernelArgs& a) {
    const float s = sqrt_var(v);
    L = fmaf(s, z1l, L);
    L = fmaf(v, a.f_nhdt2, L);
    v = fmaxf(fmaf(s, sz2, fmaf(v, a.f_omkdt, ck)), 0.0f);
}

template <bool GREEKS>
__device__ __forceinline__ void advance(PathState32& st, float z1l, float sz2, const KernelArgs& a) {
    const float ck = fmaf(sz2 * sz2, a.f_cmil2, a.f_ck0);
    traj_step(st.v0, st.L0, z1l, sz2, ck, a);
    if (GREEKS) {
        traj_step(st.vu, st.Lu, z1l, sz2, ck, a);
        traj_step(st.vd, st.Ld, z1l, sz2, ck, a);
    }
}

template <bool GREEKS>
__device__ __forceinline__ void fixing(PathState32& st, const float4 w) {
    const float P = ex2_sel<(HMC_EX2_POLY >= 3)>(st.L0);
    st.A0 = fmaf(P, w.x, st.A0);
    if (GREEKS) {
        st.T1 = fmaf(P, w.y, st.T1);
        st.Dp = fmaf(P, w.z, st.Dp);
        st.Dm = fmaf(P, w.w, st.Dm);
        st.Au = fmaf(ex2_sel<(HMC_EX2_POLY >= 1)>(st.Lu), w.x, st.Au);
        st.Ad = fmaf(ex2_sel<(HMC_EX2_POLY >= 2)>(st.Ld), w.x, st.Ad);
    }
}

template <int FIX, bool GREEKS>
__device__ __forceinline__ void step(PathState32& st, int k, float z1l, float sz2,
                                     const KernelArgs& a) {
    advance<GREEKS>(st, z1l, sz2, a);
    if (FIX == kFixEvery) {
        fixing<GREEKS>(st, __ldg(a.steps32 + k));
    } else if (FIX == kFixTable) {
        const float4 w = __ldg(a.steps32 + k);
        if (w.x != 0.0f) fixing<GREEKS>(st, w);
    }
}

// ---------------------------------------------------------------------------
// Sobol QMC driver (engine.py:97-101: run r uses points 1 + r*N + path).
//
// gray(n) = gray(n & ~31) ^ gray(n & 31) (no carries between the parts), so
// the XOR of direction numbers splits into a warp-uniform high part U (the
// warp's <= 2 aligned 32-point blocks) and a lane part T indexed by the
// lane's 5-bit Gray code.  Both are rebuilt in shared memory for every
// 64-step chunk of dimensions; the per-step cost is two LDS.64 + two XORs
// instead of a 30-bit XOR per coordinate.  Optional random digital shift
// (a.sobol_shift) per (run, dimension) for randomised QMC.
// ---------------------------------------------------------------------------
constexpr int kSobolSteps = 64;  // steps per table refill (128 dimensions)

struct SobolTables {
    uint2 T[kSobolSteps][32];          // lane parts, (dim 2q, dim 2q+1)
    uint2 U[kWarps][2][kSobolSteps];   // per warp: blocks B1, B2
};

template <int FIX, bool GREEKS>
__device__ __forceinline__ void sobol_paths(PathState32& st, int run, long long p, const KernelArgs& a) {
    __shared__ SobolTables tab;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // scrambled (randomised QMC): every run re-uses points 1..N under its own shifts
        const uint32_t n = (uint32_t)(1 + (a.sobol_scramble ? 0LL : (long long)run * a.n_paths) + p);
    const uint32_t n0 = __shfl_sync(0xffffffffu, n, 0);
    const uint32_t B1 = n0 & ~31u;
    const uint32_t gB1 = B1 ^ (B1 >> 1), gB2 = (B1 + 32) ^ ((B1 + 32) >> 1);
    const int which = ((n & ~31u) != B1) ? 1 : 0;
    const uint32_t c = n & 31u, jl = c ^ (c >> 1);
    const unsigned long long key_run = derive(a.root_key, (unsigned long long)run);
    const uint32_t* __restrict__ V = a.sobol_v;
    const int dim = a.sobol_dim;
    const float c1 = a.f_sqdt * a.f_log2e;
    const float cs = a.f_sigma * a.f_sqdt;
    const float half = a.sobol_scramble ? 0.5f : 0.0f;

#pragma unroll 1
    for (int k0 = 1; k0 <= a.n_sim; k0 += kSobolSteps) {
        const int m = min(kSobolSteps, a.n_sim - k0 + 1);
        const int d0 = 2 * (k0 - 1);
        __syncthreads();  // previous chunk fully consumed
        // lane-part table: thread t owns dimension d0 + t, all 32 Gray codes
        if (threadIdx.x < 2 * m) {
            const int d = d0 + threadIdx.x;
            uint32_t v[5];
#pragma unroll
            for (int b = 0; b < 5; ++b) v[b] = __ldg(V + b * dim + d);
            uint32_t x[32];
            x[0] = 0;
#pragma unroll
            for (int j = 1; j < 32; ++j) x[j] = x[j & (j - 1)] ^ v[__ffs(j) - 1];
            uint32_t* col = reinterpret_cast<uint32_t*>(&tab.T[threadIdx.x >> 1][0]) + (threadIdx.x & 1);
#pragma unroll
            for (int j = 0; j < 32; ++j) col[2 * j] = x[j];
        }
        // warp-uniform parts for this warp's two aligned blocks
        for (int dd = lane; dd < 2 * m; dd += 32) {
            const int d = d0 + dd;
            uint32_t u1 = 0, u2d = 0;
            for (int b = 4; b < kSobolBits; ++b) {
                const uint32_t vb = ((gB1 | (gB1 ^ gB2)) >> b) & 1u ? __ldg(V + b * dim + d) : 0u;
                if ((gB1 >> b) & 1u) u1 ^= vb;
                if (((gB1 ^ gB2) >> b) & 1u) u2d ^= vb;
            }
            if (a.sobol_scramble) u1 ^= sobol_shift(key_run, d);
            reinterpret_cast<uint32_t*>(&tab.U[warp][0][dd >> 1])[dd & 1] = u1;
            reinterpret_cast<uint32_t*>(&tab.U[warp][1][dd >> 1])[dd & 1] = u1 ^ u2d;
        }
        __syncthreads();
#pragma unroll 1
        for (int q = 0; q < m; ++q) {
            const uint2 t = tab.T[q][jl];
            const uint2 u = tab.U[warp][which][q];
            const float za = sobol_normal(t.x ^ u.x, half);
            const float zb = sobol_normal(t.y ^ u.y, half);
            const float z1l = c1 * za;
            const float sz2 = cs * fmaf(a.f_rho, za, a.f_sq1mr2 * zb);
            step<FIX, GREEKS>(st, k0 + q, z1l, sz2, a);
        }
    }
}

template <int FIX, bool GREEKS, int SAMPLER>
__global__ void HMC_BOUNDS fast_greeks_kernel(const KernelArgs a,
                                                            double* __restrict__ tiles,
                                                            long long n_tiles) {
    const int run = blockIdx.y;
    const long long path = a.path_lo + (long long)blockIdx.x * kTile + threadIdx.x;
    const bool live = path < a.path_hi;
    const long long p = live ? path : a.path_lo;

#ifdef HMC_SMEM_PAD
    // experiments: cap resident blocks per SM through shared memory
    __shared__ volatile char occupancy_pad[HMC_SMEM_PAD];
    if (threadIdx.x == 0) occupancy_pad[0] = 0;
#endif
    PathState32 st;
    st.v0 = a.f_v0;
    st.vu = a.f_vu;
    st.vd = a.f_vd;
    st.L0 = st.Lu = st.Ld = 0.0f;
    st.A0 = st.Au = st.Ad = 0.0f;
    st.T1 = st.Dp = st.Dm = 0.0f;

    if (SAMPLER == HMC_SAMPLER_PSEUDO) {
        // counter (step pair, path, key_run lo, key_run hi), fixed key
        const unsigned long long key_run = derive(a.root_key, (unsigned long long)run);
        const uint32_t c1 = (uint32_t)p;
        const uint32_t c2 = (uint32_t)key_run, c3 = (uint32_t)(key_run >> 32);
#if HMC_TRIPACK
        const int ntri = a.n_sim / 3;
        int k = 1;
#pragma unroll 1
        for (int j = 0; j < ntri; ++j) {
            const uint4 x = philox4x32_10((uint32_t)j, c1, c2, c3);
            float fr[3], fa[3];
            tri_unpack(x, fr, fa);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                float z1l, sz2;
                box_muller_f(fr[i], fa[i], x.x << (31 - i), a, z1l, sz2);
                step<FIX, GREEKS>(st, k + i, z1l, sz2, a);
            }
            k += 3;
        }
        if (k <= a.n_sim) {
            const uint4 x = philox4x32_10((uint32_t)ntri, c1, c2, c3);
            float fr[3], fa[3];
            tri_unpack(x, fr, fa);
            for (int i = 0; k + i <= a.n_sim; ++i) {
                float z1l, sz2;
                box_muller_f(fr[i], fa[i], x.x << (31 - i), a, z1l, sz2);
                step<FIX, GREEKS>(st, k + i, z1l, sz2, a);
            }
        }
#else
        const int npairs = a.n_sim >> 1;
        int k = 1;
#if HMC_PIPELINE_RNG
        uint4 xn = philox4x32_10(0u, c1, c2, c3);
#endif
        HMC_UNROLL(HMC_UNROLL_PAIRS)
        for (int j = 0; j < npairs; ++j) {
#if HMC_PIPELINE_RNG
            const uint4 x = xn;
            xn = philox4x32_10((uint32_t)(j + 1), c1, c2, c3);
#else
            const uint4 x = philox4x32_10((uint32_t)j, c1, c2, c3);
#endif
            float z1l, sz2;
            box_muller(x.x, x.y, a, z1l, sz2);
            step<FIX, GREEKS>(st, k, z1l, sz2, a);
            box_muller(x.z, x.w, a, z1l, sz2);
            step<FIX, GREEKS>(st, k + 1, z1l, sz2, a);
            k += 2;
        }
        if (a.n_sim & 1) {
            const uint4 x = philox4x32_10((uint32_t)npairs, c1, c2, c3);
            float z1l, sz2;
            box_muller(x.x, x.y, a, z1l, sz2);
            step<FIX, GREEKS>(st, k, z1l, sz2, a);
        }
#endif
    } else {
        sobol_paths<FIX, GREEKS>(st, run, p, a);
    }
    if (FIX == kFixLast) fixing<GREEKS>(st, __ldg(a.steps32 + a.n_sim));

    const float inv_n = a.f_inv_navg;
    const float A = st.A0 * inv_n;
    double q[kNQ];
    if (GREEKS) {
        greeks_epilogue_f32(a, A, st.T1 * inv_n, st.Au * inv_n, st.Ad * inv_n,
                            fmaf(st.Dp, inv_n, A), fmaf(st.Dm, inv_n, A), q);
    } else {
        const float K = a.f_K, disc = a.f_disc;
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
