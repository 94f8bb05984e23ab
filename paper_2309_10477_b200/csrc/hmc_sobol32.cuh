// hmc_sobol32.cuh -- the fp32 kernels' on-the-fly Sobol driver pieces
// (shared-memory Gray-code tables, per-lane point decomposition, quantile),
// used by the path kernel (hmc_fast.cu) and the surface kernel
// (hmc_surface.cu).
#pragma once

#include "hmc_device.cuh"
#include "hmc_path32.cuh"

namespace hmc {

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

template <int STEPS, int WARPS>
struct SobolTablesT {
    static constexpr int kSteps = STEPS;
    uint2 T[STEPS][32];          // lane parts, (dim 2q, dim 2q+1)
    uint2 U[WARPS][2][STEPS];    // per warp: blocks B1, B2
};

// Gray-code split of this thread's point index (see above)
struct SobolLane {
    uint32_t gB1, gB2;  // Gray codes of the warp's two aligned 32-point blocks
    int which;          // this lane's block
    uint32_t jl;        // Gray code of the lane part
    unsigned long long key_run;
    float hx, ht;       // half 2^-29, half 2^-30 (half = 0.5: cell midpoints of shifted points)

    __device__ __forceinline__ SobolLane(int run, long long p, const KernelArgs& a) {
        // scrambled (randomised QMC): every run re-uses points 1..N under its own shifts
        const uint32_t n = (uint32_t)(1 + (a.sobol_scramble ? 0LL : (long long)run * a.n_paths) + p);
        const uint32_t n0 = __shfl_sync(0xffffffffu, n, 0);
        const uint32_t B1 = n0 & ~31u;
        gB1 = B1 ^ (B1 >> 1);
        gB2 = (B1 + 32) ^ ((B1 + 32) >> 1);
        which = ((n & ~31u) != B1) ? 1 : 0;
        const uint32_t c = n & 31u;
        jl = c ^ (c >> 1);
        key_run = derive(a.root_key, (unsigned long long)run);
        const float half = a.sobol_scramble ? 0.5f : 0.0f;
        hx = half * 1.86264514923095703125e-09f;
        ht = half * 9.31322574615478515625e-10f;
    }
};

// (re)build the tables for dimension pairs [q0, q0 + m); block-wide
template <class Tab>
__device__ __forceinline__ void sobol_refill(Tab& tab, int q0, int m, const SobolLane& sl,
                                             const KernelArgs& a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t* __restrict__ V = a.sobol_v;
    const int dim = a.sobol_dim;
    const int d0 = 2 * q0;
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
            const uint32_t vb = ((sl.gB1 | (sl.gB1 ^ sl.gB2)) >> b) & 1u ? __ldg(V + b * dim + d) : 0u;
            if ((sl.gB1 >> b) & 1u) u1 ^= vb;
            if (((sl.gB1 ^ sl.gB2) >> b) & 1u) u2d ^= vb;
        }
        if (a.sobol_scramble) u1 ^= sobol_shift(sl.key_run, d);
        reinterpret_cast<uint32_t*>(&tab.U[warp][0][dd >> 1])[dd & 1] = u1;
        reinterpret_cast<uint32_t*>(&tab.U[warp][1][dd >> 1])[dd & 1] = u1 ^ u2d;
    }
    __syncthreads();
}

// the two standard normals (divided by sqrt(2)) of pair q of the loaded chunk
template <class Tab>
__device__ __forceinline__ void sobol_pair(const Tab& tab, int q, const SobolLane& sl,
                                           float& za, float& zb) {
    const uint2 t = tab.T[q][sl.jl];
    const uint2 u = tab.U[threadIdx.x >> 5][sl.which][q];
    za = sobol_normal_u(t.x ^ u.x, sl.hx, sl.ht);
    zb = sobol_normal_u(t.y ^ u.y, sl.hx, sl.ht);
}


}  // namespace hmc
