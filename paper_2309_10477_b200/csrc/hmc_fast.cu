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
// The loop is bound by the MUFU (XU) pipe at ~86 %;
// the FMA-pipe substitutions tried against it (sin/cos and ex2 polynomials,
// scalar and paired FFMA2) are recorded with their timings in DESIGN.md.
#include <cuda_runtime.h>

#include "hmc_device.cuh"
#include "hmc_launch.h"

#include "hmc_path32.cuh"
#include "hmc_sobol32.cuh"

// Resident blocks per SM (register budget) by fixing mode, from
// tools/kernel_variants.py sweeps on 2^24 x 252 full-Greeks launches:
// daily-fixing Asian is MUFU-queue bound and prefers 7 blocks (28 warps,
// 72 regs: 48 warps 11.1 ms -> 28 warps 10.7 ms); the European (one ex2 at
// the end) prefers 10 blocks (8.55 -> 8.40 ms).
// The time-ordered Sobol Asian kernel runs 8 blocks (60 registers, no spills):
// RQMC Asian 2^22 x 252 3.28 -> 3.18 ms against 7 blocks (6: 3.28).
// The Brownian-bridge Sobol kernel keeps its skeleton in shared memory
// (10 KB tables + (S + 1) KB skeleton per block), 7 blocks at S = 16.
#ifdef HMC_MIN_BLOCKS
#define HMC_BOUNDS __launch_bounds__(kTile, HMC_MIN_BLOCKS)
#else
#define HMC_BOUNDS \
    __launch_bounds__(kTile, (SAMPLER == kSamplerBridge ? 7 : (FIX == kFixLast ? 10 : SAMPLER == HMC_SAMPLER_SOBOL ? 8 : 7)))
#endif

namespace hmc {

// Sobol driver pieces: hmc_sobol32.cuh
// the bridge driver also holds the skeleton in shared memory: half-size
// tables keep it at 7 blocks per SM
#ifndef HMC_BRIDGE_TABLE_STEPS
#define HMC_BRIDGE_TABLE_STEPS 32
#endif
constexpr int kBridgeTableSteps = HMC_BRIDGE_TABLE_STEPS;
// steps of the time-ordered Sobol loop unrolled together: the quantiles of
// later steps overlap the trajectory updates of earlier ones (RQMC Asian
// 2^22 x 252 Greeks: 1 -> 3.71 ms, 2 -> 3.53, 4 -> 3.43, 8 -> 3.33, 16 -> 3.66)
#ifndef HMC_SOBOL_UNROLL
#define HMC_SOBOL_UNROLL 8
#endif
// fine steps of a bridge segment unrolled together (RQMC Asian 2^22 x 252,
// S = 16: per-step loop 4.85 ms; segment loops 4.47, unrolled x2 4.25,
// x4 4.19, x8 4.33)
#ifndef HMC_BRIDGE_UNROLL
#define HMC_BRIDGE_UNROLL 4
#endif
#define HMC_PRAGMA(x) _Pragma(#x)
#define HMC_UNROLL(n) HMC_PRAGMA(unroll n)
using SobolTables = SobolTablesT<kSobolSteps, kWarps>;

constexpr int kSamplerBridge = 2;  // internal: Sobol with Brownian-bridge ordering

template <int FIX, bool GREEKS>
__device__ __forceinline__ void sobol_paths(PathState32& st, int run, long long p, const KernelArgs& a) {
    __shared__ SobolTables tab;
    const SobolLane sl(run, p, a.path_lo + (long long)blockIdx.x * kTile, kWarps, a);
    // the quantile returns k z / sqrt(2): fold the step constants into k so
    //   .x = sqrt(dt) log2(e) z_a                        (= z1l)
    //   .y = sigma sqrt(dt) sqrt(1 - rho^2) z_b
    // and sz2 = sigma sqrt(dt) (rho z_a + sqrt(1 - rho^2) z_b) = .y + z1l sigma rho / log2(e)
    // (host-computed: a.f_sob_k, a.f_sob_k2 = -2k, a.f_sob_crho = sigma rho / log2(e))

#pragma unroll 1
    for (int k0 = 1; k0 <= a.n_sim; k0 += kSobolSteps) {
        const int m = min(kSobolSteps, a.n_sim - k0 + 1);
        sobol_refill(tab, k0 - 1, m, sl, a);
        // the next step's table coordinates are loaded one step ahead (the
        // XOR consuming the LDS was the top stall site; 3.33 -> 3.29 ms;
        // two steps ahead: 3.45) -- unconditionally, into the tables' pad
        // step at the end of a chunk; the fixing weights through a chunk
        // pointer, so the unrolled loads take immediate offsets
        HMC_DCHECK(k0 + m - 1 <= a.n_sim);
        const float4* __restrict__ wk = per_thread_ptr(a.steps32 + k0);
        uint2 Xn = sobol_coords(tab, 0, sl);
        HMC_UNROLL(HMC_SOBOL_UNROLL)
        for (int q = 0; q < m; ++q) {
            const uint2 X = Xn;
            Xn = sobol_coords(tab, q + 1, sl);
            const float2 z = sobol_normal_X2(X.x, X.y, a.f_sob_k, a.f_sob_k2);
            step_w<FIX, GREEKS, true>(st, wk + q, z.x, fmaf(z.x, a.f_sob_crho, z.y), a);
        }
    }
}

// Sobol with Brownian-bridge ordering (hmc_sim.sobol_bridge, tables:
// hmc_device.cuh BridgeNode): pairs 0..S-1 build this path's skeleton of
// both Brownian motions in shared memory (dynamic, [S + 1][kTile] float2,
// conflict-free), then the steps run in time order, each increment drawn
// conditionally on the segment's right end.  Same dimensions, same table
// refills as the time-ordered driver; the increments replace sqrt(dt) z.
template <int FIX, bool GREEKS>
__device__ __forceinline__ void sobol_bridge_paths(PathState32& st, int run, long long p,
                                                   const KernelArgs& a) {
    constexpr int kQ = kBridgeTableSteps;
    __shared__ SobolTablesT<kQ, kWarps> tab;
    extern __shared__ float2 skel[];
    float2* my = skel + threadIdx.x;  // point j at my[j * kTile]
    const SobolLane sl(run, p, a.path_lo + (long long)blockIdx.x * kTile, kWarps, a);
    const int S = a.bridge_segments;
    // The bridge runs on the step-shock channels directly: every bridge
    // formula is linear, so instead of (W1, W2) it carries
    //   B = (log2(e) W1, sigma (rho W1 + sqrt(1 - rho^2) W2))
    // whose increments ARE the step shocks (z1l, sz2) of step(): the
    // quantile takes the scales k = (log2 e, sigma sqrt(1 - rho^2)) and
    // z'.y += (sigma rho / log2 e) z'.x correlates them.  Per fine step that
    // is one FADD2 + FMUL2 + FFMA2 + FADD2 instead of ~12 scalar instructions.
    const float2 kq = make_float2(a.f_log2e, a.f_sigma * a.f_sq1mr2);
    const float crho = a.f_sob_crho;
    auto shocks = [&](int q) {
        const uint2 X = sobol_coords(tab, q, sl);
        float2 z = sobol_normal_X2(X.x, X.y, kq);
        z.y = fmaf(z.x, crho, z.y);
        return z;
    };

    int c0 = 0;  // first pair of the loaded chunk
    sobol_refill(tab, 0, min(kQ, a.n_sim), sl, a);
    my[0] = make_float2(0.0f, 0.0f);
#pragma unroll 1
    for (int i = 0; i < S; ++i) {
        if (i == c0 + kQ) {
            c0 = i;
            sobol_refill(tab, c0, min(kQ, a.n_sim - c0), sl, a);
        }
        const float2 z = shocks(i - c0);
        const BridgeNode nd = a.bridge_nodes32[i];
        HMC_DCHECK(nd.m >= 1 && nd.m <= S && (nd.lr & 0xffff) <= S && (nd.lr >> 16) <= S);
        const float2 wl = my[(nd.lr & 0xffff) * kTile], wr = my[(nd.lr >> 16) * kTile];
        my[nd.m * kTile] = __ffma2_rn(f2(nd.sd), z, __ffma2_rn(f2(nd.a), sub2(wr, wl), wl));
    }
    // time order, segment by segment: segment j covers steps b_{j-1}+1 .. b_j,
    // b_j = j n_sim / S (the host's build_bridge); its fine steps draw the
    // next pairs and move towards the skeleton point R, the last step lands
    // on it (alpha = 1, beta = 0: d = R - B).  The fine steps run as a
    // regular loop between table refills, unrolled so the quantiles of
    // later steps overlap the trajectory updates of earlier ones.
    int pc = S;  // next pair
    float2 B = make_float2(0.0f, 0.0f);
    int k = 1;
#pragma unroll 1
    for (int j = 1; j <= S; ++j) {
        const float2 R = my[j * kTile];
        const int kend = (int)(((long long)j * a.n_sim) / S);
#pragma unroll 1
        while (k < kend) {
            if (pc == c0 + kQ) {
                c0 = pc;
                sobol_refill(tab, c0, min(kQ, a.n_sim - c0), sl, a);
            }
            const int run = min(kend - k, c0 + kQ - pc);
            const int q0 = pc - c0;
            HMC_DCHECK(run >= 1 && q0 >= 0 && q0 + run <= kQ && k + run - 1 <= a.n_sim);
            // as the time-ordered driver: per-step tables through per-thread
            // pointers (immediate offsets)
            const BridgeStep* __restrict__ bsp = per_thread_ptr(a.bridge_steps32 + k);
            const float4* __restrict__ wk = per_thread_ptr(a.steps32 + k);
            HMC_UNROLL(HMC_BRIDGE_UNROLL)
            for (int i = 0; i < run; ++i) {
                const BridgeStep bs = bsp[i];
                const float2 z = shocks(q0 + i);
                const float2 d = __ffma2_rn(sub2(R, B), f2(bs.alpha), __fmul2_rn(f2(bs.beta), z));
                B = __fadd2_rn(B, d);
                step_w<FIX, GREEKS, true>(st, wk + i, d.x, d.y, a);
            }
            k += run;
            pc += run;
        }
        const float2 d = sub2(R, B);    // segment end
        B = R;
        step<FIX, GREEKS, true>(st, k, d.x, d.y, a);
        ++k;
    }
}

template <int FIX, bool GREEKS, int SAMPLER>
__global__ void HMC_BOUNDS fast_greeks_kernel(const KernelArgs a,
                                                            double* __restrict__ tiles,
                                                            long long n_tiles) {
    const int run = a.run0 + (int)blockIdx.y;
    const long long path = a.path_lo + (long long)blockIdx.x * kTile + threadIdx.x;
    const bool live = path < a.path_hi;
    const long long p = live ? path : a.path_lo;

    PathState32 st;
    st.init(a.f_v0, make_float2(a.f_vu, a.f_vd));

    if (SAMPLER == HMC_SAMPLER_PSEUDO) {
        // counter (step triple, path, key_run lo, key_run hi), fixed key;
        // one Philox block feeds three Box-Muller steps (tri_unpack)
        const unsigned long long key_run = derive(a.root_key, (unsigned long long)run);
        const uint32_t c1 = (uint32_t)p;
        const uint32_t c2 = (uint32_t)key_run, c3 = (uint32_t)(key_run >> 32);
        const int ntri = a.n_sim / 3;
        int k = 1;
#pragma unroll 1
        for (int j = 0; j < ntri; ++j) {
            const uint4 x = philox4x32_10((uint32_t)j, c1, c2, c3);
            float fr[3], fa[3];
            tri_unpack(x, fr, fa);
            HMC_DCHECK(k + 2 <= a.n_sim);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                float z1l, sz2;
                box_muller_f(fr[i], fa[i], a, z1l, sz2);
                step<FIX, GREEKS, FIX == kFixLast>(st, k + i, z1l, sz2, a);
            }
            k += 3;
        }
        if (k <= a.n_sim) {
            const uint4 x = philox4x32_10((uint32_t)ntri, c1, c2, c3);
            float fr[3], fa[3];
            tri_unpack(x, fr, fa);
            for (int i = 0; k + i <= a.n_sim; ++i) {
                float z1l, sz2;
                box_muller_f(fr[i], fa[i], a, z1l, sz2);
                step<FIX, GREEKS, FIX == kFixLast>(st, k + i, z1l, sz2, a);
            }
        }
    } else if (SAMPLER == HMC_SAMPLER_SOBOL) {
        sobol_paths<FIX, GREEKS>(st, run, p, a);
    } else {
        sobol_bridge_paths<FIX, GREEKS>(st, run, p, a);
    }
    if (FIX == kFixLast) fixing<GREEKS>(st, __ldg(a.steps32 + a.n_sim));

    const float inv_n = a.f_inv_navg;
    const float A = st.AT.x * inv_n;
    double q[kNQ];
    if (GREEKS) {
        greeks_epilogue_f32(a, A, st.AT.y * inv_n, st.Ab.x * inv_n, st.Ab.y * inv_n, st.D.x * inv_n,
                            st.D.y * inv_n, q);
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
    HMC_DCHECK((long long)blockIdx.x < n_tiles && run < a.n_runs);
    tile_reduce_store(q, tiles + ((size_t)run * n_tiles + blockIdx.x) * kNW);
}

template <int FIX, bool GREEKS>
static void launch_sampler(const KernelArgs& a, double* d_tiles, long long n_tiles, dim3 grid,
                           cudaStream_t s) {
    if (a.sampler == HMC_SAMPLER_PSEUDO)
        fast_greeks_kernel<FIX, GREEKS, HMC_SAMPLER_PSEUDO><<<grid, kTile, 0, s>>>(a, d_tiles, n_tiles);
    else if (a.bridge_segments == 0)
        fast_greeks_kernel<FIX, GREEKS, HMC_SAMPLER_SOBOL><<<grid, kTile, 0, s>>>(a, d_tiles, n_tiles);
    else {
        const int smem = (a.bridge_segments + 1) * kTile * (int)sizeof(float2);
        auto k = fast_greeks_kernel<FIX, GREEKS, kSamplerBridge>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);  // launch reports failure
        k<<<grid, kTile, smem, s>>>(a, d_tiles, n_tiles);
    }
}

template <int FIX>
static void launch_greeks_flag(const KernelArgs& a, double* d_tiles, long long n_tiles,
                               dim3 grid, cudaStream_t s) {
    if (a.want_greeks)
        launch_sampler<FIX, true>(a, d_tiles, n_tiles, grid, s);
    else
        launch_sampler<FIX, false>(a, d_tiles, n_tiles, grid, s);
}

// Known-answer path of the production arithmetic: the same state, step,
// fixing and epilogue code as fast_greeks_kernel, driven by GIVEN standard
// normals z[path][k] = (z1, z2) (z2 independent of z1; correlated as in
// the kernels), per-path quantities out[path][HMC_NQ] (no reduction).
template <int FIX>
__global__ void __launch_bounds__(kTile) given_normals_kernel(const KernelArgs a, const float2* __restrict__ z,
                                                              long long n, double* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    PathState32 st;
    st.init(a.f_v0, make_float2(a.f_vu, a.f_vd));
    const float c1 = a.f_sqdt * a.f_log2e, cs = a.f_sigma * a.f_sqdt;
    for (int k = 1; k <= a.n_sim; ++k) {
        const float2 w = z[(size_t)i * a.n_sim + (k - 1)];
        step<FIX, true>(st, k, c1 * w.x, cs * fmaf(a.f_rho, w.x, a.f_sq1mr2 * w.y), a);
    }
    if (FIX == kFixLast) fixing<true>(st, __ldg(a.steps32 + a.n_sim));
    const float inv_n = a.f_inv_navg;
    const float A = st.AT.x * inv_n;
    double q[kNQ];
    greeks_epilogue_f32(a, A, st.AT.y * inv_n, st.Ab.x * inv_n, st.Ab.y * inv_n, st.D.x * inv_n, st.D.y * inv_n,
                        q);
#pragma unroll
    for (int j = 0; j < kNQ; ++j) out[(size_t)i * kNQ + j] = q[j];
}

cudaError_t launch_given_normals(const KernelArgs& a, const float2* d_z, long long n, double* d_out,
                                 cudaStream_t s) {
    const unsigned grid = (unsigned)((n + kTile - 1) / kTile);
    switch (a.fix_mode) {
        case kFixLast: given_normals_kernel<kFixLast><<<grid, kTile, 0, s>>>(a, d_z, n, d_out); break;
        case kFixEvery: given_normals_kernel<kFixEvery><<<grid, kTile, 0, s>>>(a, d_z, n, d_out); break;
        default: given_normals_kernel<kFixTable><<<grid, kTile, 0, s>>>(a, d_z, n, d_out); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_fast_greeks(const KernelArgs& a, double* d_tiles, long long n_tiles,
                               cudaStream_t s) {
    // runs map to gridDim.y (<= 65535 per launch): batches carry run0
    for (int r0 = 0; r0 < a.n_runs; r0 += kMaxRunsPerLaunch) {
        KernelArgs b = a;
        b.run0 = r0;
        dim3 grid((unsigned)n_tiles, (unsigned)min(kMaxRunsPerLaunch, a.n_runs - r0));
        switch (a.fix_mode) {
            case kFixLast: launch_greeks_flag<kFixLast>(b, d_tiles, n_tiles, grid, s); break;
            case kFixEvery: launch_greeks_flag<kFixEvery>(b, d_tiles, n_tiles, grid, s); break;
            default: launch_greeks_flag<kFixTable>(b, d_tiles, n_tiles, grid, s); break;
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace hmc
