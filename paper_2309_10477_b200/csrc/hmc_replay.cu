// hmc_replay.cu -- fp64 "replay" kernels: the reference's own random stream
// and arithmetic, one path per thread, on sm_100a.
//
// Compiled with -fmad=false: the reference's C build (-O3, x86-64 baseline,
// pkg/setup.py:11) has no FMA, so the GPU follows the same rounding sequence
// operation for operation (_core.pyx:384-411).  Remaining differences are the
// last-ulp behaviour of CUDA's exp/log/erfc vs glibc's, i.e. ~1e-16 relative
// per step; the parity gate is 1e-12 per path (tests/test_gpu_replay.py).
//
//   replay_batch_kernel   backend discretised_batch: per-path (s_T, avg, tw)
//   replay_greeks_kernel  engine path: base + v0 +/- trajectories per thread,
//                         per-path estimators, fp64 tile partials
#include <cuda_runtime.h>

#include "hmc_device.cuh"
#include "hmc_launch.h"
#include "hmc_ndtri64.cuh"

namespace hmc {

struct TrajD {
    double s, v, ps, tw;
};

// one Euler/Milstein full-truncation step (_core.pyx:399-404)
__device__ __forceinline__ void ref_step(TrajD& t, double z1, double z2, const KernelArgs& a) {
    const double sqv = sqrt(t.v * a.dt);
    t.s = t.s * exp((a.r - 0.5 * t.v) * a.dt + sqv * z1);
    double v_new = t.v + a.kappa * (a.theta - t.v) * a.dt + a.sigma * sqv * z2;
    if (a.milstein) v_new = v_new + 0.25 * a.sigma * a.sigma * a.dt * (z2 * z2 - 1.0);
    t.v = v_new > 0.0 ? v_new : 0.0;
}

// the two uniforms of step k (1-based) for this path: reference layout
// u[2(k-1)] -> asset, u[2(k-1)+1] -> variance (_core.pyx:391-396)
struct RefDraws {
    int sampler;
    unsigned long long key;         // pseudo: per-path main key
    uint32_t gray;                  // sobol: Gray code of the point index
    const uint32_t* v;
    int dim;
    const double* row;              // supplied uniforms (replay batch) or null
    int scramble;                   // sobol: random digital shift (hmc_fast.cu sobol_shift)
    unsigned long long key_run;
    __device__ __forceinline__ void get(int k, double& u1, double& u2) const {
        const int i = 2 * (k - 1);
        if (row) {
            u1 = row[i];
            u2 = row[i + 1];
        } else if (sampler == HMC_SAMPLER_PSEUDO) {
            u1 = uniform_at(key, (unsigned long long)i);
            u2 = uniform_at(key, (unsigned long long)(i + 1));
        } else {
            uint32_t x1 = sobol_coord(gray, v, dim, i), x2 = sobol_coord(gray, v, dim, i + 1);
            double half = 0.0;  // reference points: x * 2^-30 exactly (x >= 1)
            if (scramble) {     // shifted points can hit x = 0: cell midpoints
                x1 ^= sobol_shift(key_run, i);
                x2 ^= sobol_shift(key_run, i + 1);
                half = 0.5;
            }
            u1 = ((double)x1 + half) * (1.0 / 1073741824.0);
            u2 = ((double)x2 + half) * (1.0 / 1073741824.0);
        }
    }
};

__global__ void __launch_bounds__(kTile) replay_batch_kernel(const KernelArgs a,
                                                             unsigned long long key_run,
                                                             const double* __restrict__ uniforms,
                                                             double* __restrict__ out) {
    const long long n = a.path_hi - a.path_lo;
    const long long i = (long long)blockIdx.x * kTile + threadIdx.x;
    if (i >= n) return;
    RefDraws dr{};
    dr.sampler = HMC_SAMPLER_PSEUDO;
    dr.key = derive(derive(key_run, (unsigned long long)(a.path_lo + i)), 0ULL);
    dr.row = uniforms ? uniforms + (size_t)i * 2 * a.n_steps : nullptr;
    TrajD t{a.s0, a.v0, 0.0, 0.0};
    for (int k = 1; k <= a.n_steps; ++k) {
        double u1, u2;
        dr.get(k, u1, u2);
        const double z1 = ndtri_ref(u1);
        const double z2 = a.rho * z1 + a.sq1mr2 * ndtri_ref(u2);
        ref_step(t, z1, z2, a);
        const StepD st = a.steps64[k];
        if (st.fix != 0.0) {
            t.ps += t.s;
            t.tw += t.s * st.t;
        }
    }
    out[3 * i + 0] = t.s;
    out[3 * i + 1] = t.ps / a.n_avg;
    out[3 * i + 2] = t.tw / a.n_avg;
}

// 8 resident blocks (64 registers, the rest spilled to L1-resident local
// memory): the fp64 pipe needs the warps to hide its latency.  Full-Greeks
// replay, Asian daily fixings, 2^20 x 252 (tools/kernel_variants.py set
// "replay"): unbounded (168-255 registers, 3 blocks) 14.1-18.0 ms, 4 blocks
// 12.4, 5 12.05, 6 12.02, 8 11.93 ms; results identical.
#ifndef HMC_REPLAY_MINB
#define HMC_REPLAY_MINB 8
#endif
template <bool GREEKS>
__global__ void __launch_bounds__(kTile, HMC_REPLAY_MINB) replay_greeks_kernel(const KernelArgs a,
                                                              double* __restrict__ tiles,
                                                              long long n_tiles) {
    const int run = a.run0 + (int)blockIdx.y;
    const long long path = a.path_lo + (long long)blockIdx.x * kTile + threadIdx.x;
    const bool live = path < a.path_hi;
    const long long p = live ? path : a.path_lo;
    RefDraws dr{};
    dr.sampler = a.sampler;
    if (a.sampler == HMC_SAMPLER_PSEUDO) {
        // engine.py:96 key_run = derive(root(seed), run); _core.pyx:385
        const unsigned long long key_run = derive(a.root_key, (unsigned long long)run);
        dr.key = derive(derive(key_run, (unsigned long long)p), 0ULL);
    } else {
        // engine.py:100: run r uses Sobol rows 1 + r*n_paths + path
        // scrambled (randomised QMC): every run re-uses points 1..N under its own shifts
        const uint32_t n = (uint32_t)(1 + (a.sobol_scramble ? 0LL : (long long)run * a.n_paths) + p);
        dr.gray = n ^ (n >> 1);
        dr.v = a.sobol_v;
        dr.dim = a.sobol_dim;
        dr.scramble = a.sobol_scramble;
        dr.key_run = derive(a.root_key, (unsigned long long)run);
    }
    TrajD t0{a.s0, a.v0, 0.0, 0.0};
    TrajD tu{a.s0, a.v0_up, 0.0, 0.0};
    TrajD td{a.s0, a.v0_dn, 0.0, 0.0};
    double dp = 0.0, dm = 0.0;
    auto advance = [&](int k, double z1, double z2) {
        ref_step(t0, z1, z2, a);
        if (GREEKS) {
            ref_step(tu, z1, z2, a);
            ref_step(td, z1, z2, a);
        }
        HMC_DCHECK(k >= 1 && k <= a.n_sim);
        const StepD st = a.steps64[k];
        if (st.fix != 0.0) {
            t0.ps += t0.s;
            t0.tw += t0.s * st.t;
            if (GREEKS) {
                tu.ps += tu.s;
                td.ps += td.s;
                dp += t0.s * st.e1p;
                dm += t0.s * st.e1m;
            }
        }
    };
    if (a.bridge_segments == 0) {
        for (int k = 1; k <= a.n_sim; ++k) {
            double u1, u2;
            dr.get(k, u1, u2);
            const double z1 = ndtri_ref(u1);
            const double z2 = a.rho * z1 + a.sq1mr2 * ndtri_ref(u2);
            advance(k, z1, z2);
        }
    } else {
        // Sobol Brownian bridge (tables and formulas: hmc_device.cuh
        // BridgeNodeD); fp64 twin of hmc_fast.cu sobol_bridge_paths
        double W1s[HMC_BRIDGE_MAX_SEGMENTS + 1], W2s[HMC_BRIDGE_MAX_SEGMENTS + 1];
        W1s[0] = W2s[0] = 0.0;
        for (int i = 0; i < a.bridge_segments; ++i) {
            double u1, u2;
            dr.get(i + 1, u1, u2);  // dimension pair i
            const BridgeNodeD nd = a.bridge_nodes64[i];
            HMC_DCHECK(nd.m >= 1 && nd.m <= a.bridge_segments && nd.l <= a.bridge_segments &&
                       nd.r <= a.bridge_segments);
            W1s[nd.m] = W1s[nd.l] + nd.a * (W1s[nd.r] - W1s[nd.l]) + nd.sd * ndtri_ref(u1);
            W2s[nd.m] = W2s[nd.l] + nd.a * (W2s[nd.r] - W2s[nd.l]) + nd.sd * ndtri_ref(u2);
        }
        int pc = a.bridge_segments;
        double W1 = 0.0, W2 = 0.0;
        const double isq = 1.0 / sqrt(a.dt);
        for (int k = 1; k <= a.n_sim; ++k) {
            const BridgeStepD bs = a.bridge_steps64[k];
            HMC_DCHECK(bs.j >= 1 && bs.j <= a.bridge_segments);
            double za = 0.0, zb = 0.0;
            if (bs.consume) {
                double u1, u2;
                dr.get(++pc, u1, u2);  // pair pc - 1
                za = ndtri_ref(u1);
                zb = ndtri_ref(u2);
            }
            const double d1 = (W1s[bs.j] - W1) * bs.alpha + bs.beta * za;
            const double d2 = (W2s[bs.j] - W2) * bs.alpha + bs.beta * zb;
            W1 = bs.consume ? W1 + d1 : W1s[bs.j];
            W2 = bs.consume ? W2 + d2 : W2s[bs.j];
            const double z1 = d1 * isq;
            advance(k, z1, a.rho * z1 + a.sq1mr2 * (d2 * isq));
        }
    }
    // european: the one fixing is t_n = T, so ps = s_T and the reference's
    // obs[:, 0] == obs[:, 1] (engine.py:51)
    const double A = t0.ps / a.n_avg;
    double q[kNQ];
    HMC_DCHECK((long long)blockIdx.x < n_tiles);
    greeks_epilogue<double>(a, A, t0.tw / a.n_avg, tu.ps / a.n_avg, td.ps / a.n_avg,
                            A + dp / a.n_avg, A + dm / a.n_avg, q);
    if (!live) {
#pragma unroll
        for (int i = 0; i < kNQ; ++i) q[i] = 0.0;
    }
    tile_reduce_store(q, tiles + ((size_t)run * n_tiles + blockIdx.x) * kNW);
}

cudaError_t launch_replay_batch(const KernelArgs& a, unsigned long long key_run,
                                const double* d_uniforms, double* d_out, cudaStream_t s) {
    const long long n = a.path_hi - a.path_lo;
    const unsigned grid = (unsigned)((n + kTile - 1) / kTile);
    replay_batch_kernel<<<grid, kTile, 0, s>>>(a, key_run, d_uniforms, d_out);
    return cudaGetLastError();
}

cudaError_t launch_replay_greeks(const KernelArgs& a, double* d_tiles, long long n_tiles,
                                 cudaStream_t s) {
    for (int r0 = 0; r0 < a.n_runs; r0 += kMaxRunsPerLaunch) {
        KernelArgs b = a;
        b.run0 = r0;
        dim3 grid((unsigned)n_tiles, (unsigned)min(kMaxRunsPerLaunch, a.n_runs - r0));
        if (a.want_greeks)
            replay_greeks_kernel<true><<<grid, kTile, 0, s>>>(b, d_tiles, n_tiles);
        else
            replay_greeks_kernel<false><<<grid, kTile, 0, s>>>(b, d_tiles, n_tiles);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// ---- the reference's RNG / step primitives, elementwise (the drop-in's
// rng / schemes modules: rng.uniform_at / _uniform_keys (rng.py:63-65,
// 356-361), rng.inverse_normal_cdf (rng.py:95-132), schemes.euler_step /
// milstein_step (schemes.py:33-61)) -- the SAME device functions the replay
// kernels run, so each is pinned on its own by the reference's vectors.

__global__ void uniforms_kernel(const unsigned long long* __restrict__ keys, long long n_keys,
                                const unsigned long long* __restrict__ draws, long long n,
                                double* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = uniform_at(keys[n_keys == 1 ? 0 : i], draws[i]);
}

__global__ void ndtri_kernel(const double* __restrict__ u, long long n, double* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = ndtri_ref(u[i]);
}

// one step per element from state (s, v) and the step's two uniforms
// (asset, variance), correlated as rng.correlated_pair (rng.py:226-235)
__global__ void steps_kernel(const KernelArgs a, const double* __restrict__ s, const double* __restrict__ v,
                             const double* __restrict__ u, long long n, double* __restrict__ s_out,
                             double* __restrict__ v_out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double z1 = ndtri_ref(u[2 * i]);
    const double z2 = a.rho * z1 + a.sq1mr2 * ndtri_ref(u[2 * i + 1]);
    TrajD t{s[i], v[i], 0.0, 0.0};
    ref_step(t, z1, z2, a);
    s_out[i] = t.s;
    v_out[i] = t.v;
}

cudaError_t launch_uniforms(const unsigned long long* d_keys, long long n_keys,
                            const unsigned long long* d_draws, long long n, double* d_out, cudaStream_t s) {
    uniforms_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(d_keys, n_keys, d_draws, n, d_out);
    return cudaGetLastError();
}

cudaError_t launch_ndtri(const double* d_u, long long n, double* d_out, cudaStream_t s) {
    ndtri_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(d_u, n, d_out);
    return cudaGetLastError();
}

cudaError_t launch_steps(const KernelArgs& a, const double* d_s, const double* d_v, const double* d_u,
                         long long n, double* d_s_out, double* d_v_out, cudaStream_t s) {
    steps_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(a, d_s, d_v, d_u, n, d_s_out, d_v_out);
    return cudaGetLastError();
}

}  // namespace hmc
