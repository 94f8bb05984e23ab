// hmc_surface.cu -- strike x maturity surfaces of European and daily-average
// Asian calls with full Greeks from ONE set of simulated paths
// (BASELINE config 5: 64 strikes x 8 maturities, both styles, 2^22 paths).
//
// Every (strike, maturity, style) shares the same paths (common random
// numbers): the paths are simulated once to the last maturity with the
// production step (hmc_path32.cuh); at each maturity checkpoint every path
// drops its observables into per-maturity HISTOGRAMS keyed by the strike
// bucket c(x) = #{j : K_j < x}.  Because a call payoff is linear in the
// underlying above the strike,
//     sum_paths (A - K_j)^+ = S1(A > K_j) - K_j N(A > K_j),
// every per-strike sum and sum of squares of every estimator (price,
// pathwise Delta/Rho, FD Gamma/Delta/Vega/Rho) follows from suffix sums of a
// few bucketed moments (hmc_api.cu surface_finalize).  Cost per path and
// maturity is O(log K) instead of O(K).
//
// Histograms are integer fixed point (linear moments to 2^-10, quadratic to 2^-2,
// counts exact; int32 per block, int64 per run): integer addition is
// associative, so block order, grid size and GPU count cannot change a
// single bit of the result -- multi-GPU runs all-reduce the integer
// histograms.  Rounding to the grid is unbiased (round to nearest) and
// ~1e-3 of a per-path value, far below the Monte Carlo noise.
#include <cuda_runtime.h>

#include "hmc_device.cuh"
#include "hmc_launch.h"

#include "hmc_path32.cuh"
#include "hmc_sobol32.cuh"

namespace hmc {

// number of strikes strictly below x.  Uniform strike grids (the usual
// surface) take an arithmetic guess and one exact correction step each way
// against the stored strikes; otherwise an unrolled branch-free lower-bound
// descent over <= 128 strikes.
__device__ __forceinline__ int strike_bucket(const float* sK, int pow2, int nK, float x,
                                             const SurfArgs& s) {
    if (s.uniform) {
        int c = (int)floorf((x - s.k0) * s.inv_dk) + 1;
        c = min(max(c, 0), nK);
        if (c > 0 && !(sK[c - 1] < x)) --c;
        if (c < nK && sK[c] < x) ++c;
        return c;
    }
    int pos = 0;
#pragma unroll
    for (int step = 128; step > 0; step >>= 1) {
        const int cand = pos + step;
        if (step <= pow2 && cand <= nK && sK[cand - 1] < x) pos = cand;
    }
    return pos;
}

// Block histograms are int32 fixed point updated with native shared-memory
// atomics (64-bit shared atomics are CAS loops on sm_100).  A value whose
// scaled magnitude reaches 2^20 bypasses the block histogram and goes
// straight to the int64 run accumulator (native global RED), so 1024 paths
// can never overflow an int32 bucket (1024 * 2^20 = 2^30).  The float ->
// int conversion is the 1.5*2^23 magic add (FMA pipe, no XU conversion).
__device__ __forceinline__ void hist_add(int* h, unsigned long long* gdirect, int nb, int v, int c,
                                         float x, float scale) {
    HMC_DCHECK(v >= 0 && v < kSurfVals && c >= 0 && c < nb);
    const float y = x * scale;
    if (fabsf(y) < 1048576.0f) {
        const int q = __float_as_int(y + 12582912.0f) - 0x4B400000;  // round to nearest
        if (q) atomicAdd(h + v * nb + c, q);
    } else {
        atomicAdd(gdirect + v * nb + c, (unsigned long long)__float2ll_rn(y));
    }
}

__device__ __forceinline__ void hist_count(int* h, int nb, int v, int c) {
    HMC_DCHECK(v >= 0 && v < kSurfVals && c >= 0 && c < nb);
    atomicAdd(h + v * nb + c, 1);
}

// add moments of x - K_j for every strike j in [lo, hi) (a bumped pair
// straddling those strikes; usually zero or one strike)
__device__ __forceinline__ void band_add(int* h, unsigned long long* g64, int nb, const float* sK,
                                         int row, int lo, int hi, float x) {
    HMC_DCHECK(lo >= 0 && hi <= nb - 1);
    for (int j = lo; j < hi; ++j) {
        const float e = x - sK[j];
        hist_add(h, g64, nb, row, j, e, kSurfBandScale);
        hist_add(h, g64, nb, row + 1, j, e * e, kSurfBandScale);
    }
}

// one style at one maturity (row layout in hmc_launch.h)
#ifndef HMC_SURF_NOINLINE
#define HMC_SURF_NOINLINE 1   // out of line: 12.5K -> 3K instructions in the kernel, 7.47 -> 7.29 ms (config 5)
#endif
#if HMC_SURF_NOINLINE
#define HMC_SURF_UPDATE_FN __device__ __noinline__
#else
#define HMC_SURF_UPDATE_FN __device__ __forceinline__
#endif
HMC_SURF_UPDATE_FN void surface_update(int* h, unsigned long long* g64, int nb, const float* sK,
                                               int pow2, int nK, const SurfArgs& s, float d, float A,
                                               float Au, float Ad, float Rp, float Rm, float w,
                                               float al) {
    const float L = kSurfLinScale, Q = kSurfQuadScale;
    const float Aup = A * s.eps_up, Adn = A * s.eps_dn;
    const int cu = strike_bucket(sK, pow2, nK, Aup, s);
    hist_add(h, g64, nb, 0, cu, A, L); hist_add(h, g64, nb, 1, cu, A * A, Q);
    const int c1 = strike_bucket(sK, pow2, nK, A, s);
    hist_count(h, nb, 2, c1); hist_add(h, g64, nb, 3, c1, A, L); hist_add(h, g64, nb, 4, c1, A * A, Q);
    hist_add(h, g64, nb, 5, c1, w, L); hist_add(h, g64, nb, 6, c1, w * w, Q);
    const int cd = strike_bucket(sK, pow2, nK, Adn, s);
    hist_count(h, nb, 7, cd); hist_add(h, g64, nb, 8, cd, A, L); hist_add(h, g64, nb, 9, cd, A * A, Q);
    band_add(h, g64, nb, sK, 15, cd, cu, Aup);
    const int cvu = strike_bucket(sK, pow2, nK, Au, s), cvd = strike_bucket(sK, pow2, nK, Ad, s);
    const float gv = d * (Au - Ad) * s.inv_dv;
    const int cmin = min(cvu, cvd);
    hist_add(h, g64, nb, 10, cmin, gv, L); hist_add(h, g64, nb, 11, cmin, gv * gv, Q);
    band_add(h, g64, nb, sK, 17, cvd, cvu, Au);
    band_add(h, g64, nb, sK, 19, cvu, cvd, Ad);
    const int cp = strike_bucket(sK, pow2, nK, Rp, s), cm = strike_bucket(sK, pow2, nK, Rm, s);
    hist_count(h, nb, 12, cm); hist_add(h, g64, nb, 13, cm, al, L); hist_add(h, g64, nb, 14, cm, al * al, Q);
    band_add(h, g64, nb, sK, 21, cm, cp, Rp);
}

__device__ __forceinline__ void surface_checkpoint(const PathState32& st, const KernelArgs& a,
                                                   const SurfArgs& s, int m, bool live, int* hist,
                                                   const float* sK, int pow2,
                                                   unsigned long long* gacc) {
    const int nb = s.nK + 1;
    const int per_style = kSurfVals * nb;
    unsigned long long* g_euro = gacc + ((size_t)0 * s.n_mats + m) * per_style;
    unsigned long long* g_asian = gacc + ((size_t)1 * s.n_mats + m) * per_style;
    HMC_DCHECK(m >= 0 && m < s.n_mats);
    if (live) {
        const SurfMat mc = s.mats[m];
        HMC_DCHECK(mc.step >= 1 && mc.step <= a.n_sim);
        const float E = __ldg(a.steps32 + mc.step).x;       // S0 e^{r T_m}
        // European: S_T of each trajectory; r bumps by e^{+-h T}, for which
        // d+ Rp - d- Rm = 0 exactly (the FD numerator is -K (d+ - d-))
        const float Ae = E * ex2a(st.L0);
        surface_update(hist, g_euro, nb, sK, pow2, s.nK, s, mc.d, Ae, E * ex2a(st.Lb.x), E * ex2a(st.Lb.y),
                       Ae * mc.ehp, Ae * mc.ehm, 0.0f, 0.0f);
        // Asian: average of S over grid dates t_1..t_m;
        // a = [A (d+ - d-) + (d+ D+ - d- D-)/N] / 2h_r, both terms same sign
        const float inv = mc.inv_n;
        const float Aa = st.AT.x * inv;
        const float al = (Aa * mc.ddisc + (mc.dp * st.D.x - mc.dm * st.D.y) * inv) * s.inv_2hr;
        surface_update(hist + per_style, g_asian, nb, sK, pow2, s.nK, s, mc.d, Aa, st.Ab.x * inv, st.Ab.y * inv,
                       fmaf(st.D.x, inv, Aa), fmaf(st.D.y, inv, Aa), fmaf(st.AT.y, inv, -mc.T * Aa), al);
    }
    __syncthreads();
    // flush this maturity's block histograms into the run accumulators
    for (int i = threadIdx.x; i < 2 * per_style; i += blockDim.x) {
        const int v = hist[i];
        if (v) {
            const int style = i / per_style, rest = i - style * per_style;
            atomicAdd(gacc + ((size_t)style * s.n_mats + m) * per_style + rest,
                      (unsigned long long)(long long)v);
            hist[i] = 0;
        }
    }
    __syncthreads();
}

// Sobol surfaces: the path kernel's Gray-code tables sized for the
// surface block (kSurfThreads / 32 warps), 32 steps per refill (the static
// shared-memory budget is 48 KB)
constexpr int kSurfSobolSteps = 32;
using SurfSobolTables = SobolTablesT<kSurfSobolSteps, kSurfThreads / 32>;

template <int SAMPLER>
__global__ void __launch_bounds__(kSurfThreads, kSurfMinBlocks) surface_kernel(const KernelArgs a, const SurfArgs s,
                                                                  long long n_tiles) {
    extern __shared__ int hist[];  // [2][kSurfVals][nK + 1] int32 fixed point
    __shared__ float sK[kSurfMaxStrikes];
    const int nb = s.nK + 1;
    HMC_DCHECK(s.nK >= 1 && s.nK <= kSurfMaxStrikes && s.n_mats >= 1);
    for (int i = threadIdx.x; i < s.nK; i += blockDim.x) sK[i] = s.strikes[i];
    for (int i = threadIdx.x; i < 2 * kSurfVals * nb; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    int pow2 = 1;
    while (pow2 * 2 <= s.nK) pow2 *= 2;

    const int run = a.run0 + (int)blockIdx.y;
    unsigned long long* gacc = s.acc + (size_t)run * 2 * s.n_mats * kSurfVals * nb;
    const unsigned long long key_run = derive(a.root_key, (unsigned long long)run);
    const uint32_t c2 = (uint32_t)key_run, c3 = (uint32_t)(key_run >> 32);

#pragma unroll 1
    for (long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const long long path = a.path_lo + tile * kSurfThreads + threadIdx.x;
        const bool live = path < a.path_hi;
        const uint32_t c1 = (uint32_t)(live ? path : a.path_lo);
        PathState32 st;
        st.init(a.f_v0, make_float2(a.f_vu, a.f_vd));
        int m = 0, next = s.mats[0].step;
        if (SAMPLER == HMC_SAMPLER_SOBOL) {
            // the single-product Sobol driver's points and quantile (same
            // dimensions 2(k-1), 2(k-1)+1 per step), checkpoints in between
            __shared__ SurfSobolTables tab;
            const SobolLane sl(run, path, a.path_lo + tile * kSurfThreads, kSurfThreads / 32, a);
            const float c1 = kSqrt2f * a.f_sqdt * a.f_log2e, cs = kSqrt2f * a.f_sigma * a.f_sqdt;
#pragma unroll 1
            for (int k0 = 1; k0 <= a.n_sim; k0 += kSurfSobolSteps) {
                const int mq = min(kSurfSobolSteps, a.n_sim - k0 + 1);
                sobol_refill(tab, k0 - 1, mq, sl, a);
#pragma unroll 1
                for (int q = 0; q < mq; ++q) {
                    const int k = k0 + q;
                    float za, zb;
                    sobol_pair(tab, q, sl, za, zb);
                    step<kFixEvery, true, true>(st, k, c1 * za, cs * fmaf(a.f_rho, za, a.f_sq1mr2 * zb), a);
                    if (k == next) {
                        surface_checkpoint(st, a, s, m, live, hist, sK, pow2, gacc);
                        ++m;
                        next = m < s.n_mats ? s.mats[m].step : 0x7fffffff;
                    }
                }
            }
            continue;
        }
#pragma unroll 1
        for (int k0 = 1; k0 <= a.n_sim; k0 += 3) {
            // same Philox counters as fast_greeks_kernel: (step triple, path, key_run)
            const uint4 x = philox4x32_10((uint32_t)((k0 - 1) / 3), c1, c2, c3);
            float fr[3], fa[3];
            tri_unpack(x, fr, fa);
            if (k0 + 2 < next) {
                // no maturity inside this triple (next <= n_sim always): plain steps
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    float z1l, sz2;
                    box_muller_f(fr[i], fa[i], a, z1l, sz2);
                    step<kFixEvery, true>(st, k0 + i, z1l, sz2, a);
                }
                continue;
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int k = k0 + i;
                if (k > a.n_sim) break;
                float z1l, sz2;
                box_muller_f(fr[i], fa[i], a, z1l, sz2);
                step<kFixEvery, true>(st, k, z1l, sz2, a);
                if (k == next) {
                    surface_checkpoint(st, a, s, m, live, hist, sK, pow2, gacc);
                    ++m;
                    next = m < s.n_mats ? s.mats[m].step : 0x7fffffff;
                }
            }
        }
    }
}

cudaError_t launch_surface(const KernelArgs& a, const SurfArgs& s, long long n_tiles, int grid_x,
                           cudaStream_t stream) {
    const size_t smem = (size_t)2 * kSurfVals * (s.nK + 1) * sizeof(int);
    auto k = a.sampler == HMC_SAMPLER_SOBOL ? surface_kernel<HMC_SAMPLER_SOBOL> : surface_kernel<HMC_SAMPLER_PSEUDO>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    for (int r0 = 0; r0 < a.n_runs; r0 += kMaxRunsPerLaunch) {
        KernelArgs b = a;
        b.run0 = r0;
        dim3 grid((unsigned)grid_x, (unsigned)min(kMaxRunsPerLaunch, a.n_runs - r0));
        k<<<grid, kSurfThreads, smem, stream>>>(b, s, n_tiles);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace hmc
