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
// the XOR of direction numbers splits into a high part U, shared by the 32
// points of an aligned 32-point block, and a lane part T indexed by the
// lane's 5-bit Gray code.  A thread block's consecutive points span at most
// WARPS + 1 aligned blocks; the refill builds T and those U rows in shared
// memory for every chunk of STEPS steps (2 STEPS dimensions): the first row
// from the direction numbers, each next row by XORing the (two) direction
// numbers in which consecutive blocks' Gray codes differ.  Per step a lane
// then does two LDS.64 + two XORs.  Optional random digital shift
// (a.sobol_shift) per (run, dimension) for randomised QMC, folded into U.
// ---------------------------------------------------------------------------
#ifndef HMC_SOBOL_STEPS
#define HMC_SOBOL_STEPS 64
#endif
constexpr int kSobolSteps = HMC_SOBOL_STEPS;  // steps per table refill (2 dimensions each, <= 64)

// One pad step per row: a driver may load pair q + 1 = STEPS unconditionally
// (its one-ahead prefetch at the end of a chunk; the value is never used),
// which keeps the unrolled step loop free of predicates and register copies.
template <int STEPS, int WARPS>
struct SobolTablesT {
    static constexpr int kSteps = STEPS;
    static constexpr int kRows = WARPS + 1;
    uint2 T[STEPS + 1][32];      // lane parts, (dim 2q, dim 2q+1)
    uint2 U[kRows][STEPS + 1];   // high parts of the block's aligned 32-point blocks
};

// Gray-code split of this thread's point index (see above)
struct SobolLane {
    uint32_t B0;        // first aligned 32-point block of the thread block
    int row;            // this lane's block, relative to B0
    uint32_t jl;        // Gray code of the lane part
    unsigned long long key_run;
    uint32_t mid;       // 2: left-aligned coordinates are cell midpoints (digitally shifted points)

    // p: this thread's path; p_first: the thread block's first path (its
    // paths are consecutive; a dead lane's row is clamped, its values unused)
    __device__ __forceinline__ SobolLane(int run, long long p, long long p_first, int max_row,
                                         const KernelArgs& a) {
        // scrambled (randomised QMC): every run re-uses points 1..N under its own shifts
        const long long off = 1 + (a.sobol_scramble ? 0LL : (long long)run * a.n_paths);
        const uint32_t n = (uint32_t)(off + p);
        B0 = (uint32_t)(off + p_first) & ~31u;
        row = (int)min(max(((long long)(n & ~31u) - (long long)B0) >> 5, 0LL), (long long)max_row);
        const uint32_t c = n & 31u;
        jl = c ^ (c >> 1);
        key_run = derive(a.root_key, (unsigned long long)run);
        mid = a.sobol_scramble ? 2u : 0u;
    }
};

// (re)build the tables for dimension pairs [q0, q0 + m); block-wide
template <class Tab>
__device__ __forceinline__ void sobol_refill(Tab& tab, int q0, int m, const SobolLane& sl,
                                             const KernelArgs& a) {
    const uint32_t* __restrict__ V = a.sobol_v;
    const int dim = a.sobol_dim;
    const int d0 = 2 * q0;
    const int nd = 2 * m;
    HMC_DCHECK(m >= 1 && m <= Tab::kSteps && d0 + nd <= dim && nd <= (int)blockDim.x);
    __syncthreads();  // previous chunk fully consumed
    // lane-part table: thread t owns dimension d0 + t, all 32 Gray codes
    if (threadIdx.x < nd) {
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
        for (int j = 0; j < 32; ++j) col[2 * j] = x[j] << 2;   // left-aligned (sobol_normal_X)
    }
    // high parts: (dimension, group of rows) per thread; a group's first row
    // from the direction numbers, the others incrementally
    const int groups = max(1, (int)blockDim.x / nd);
    const int rows_per = (Tab::kRows + groups - 1) / groups;
    if (threadIdx.x < nd * groups) {
        const int dd = threadIdx.x % nd, r0 = (threadIdx.x / nd) * rows_per;
        const int r1 = min(r0 + rows_per, Tab::kRows);
        const int d = d0 + dd;
        uint32_t B = sl.B0 + 32u * (uint32_t)r0;
        uint32_t g = B ^ (B >> 1);
        uint32_t u = 0;
        for (uint32_t bits = g & ~15u; bits; bits &= bits - 1) u ^= __ldg(V + (__ffs(bits) - 1) * dim + d);
        const uint32_t sh = a.sobol_scramble ? sobol_shift(sl.key_run, d) : 0u;
        uint32_t* out = reinterpret_cast<uint32_t*>(&tab.U[0][0]) + (dd >> 1) * 2 + (dd & 1);
        for (int r = r0; r < r1; ++r) {
            HMC_DCHECK(r < Tab::kRows && (dd >> 1) < Tab::kSteps);
            if (r > r0) {
                B += 32u;
                const uint32_t g2 = B ^ (B >> 1);
                for (uint32_t bits = g ^ g2; bits; bits &= bits - 1)
                    u ^= __ldg(V + (__ffs(bits) - 1) * dim + d);
                g = g2;
            }
            out[r * 2 * (Tab::kSteps + 1)] = ((u ^ sh) << 2) | sl.mid;   // left-aligned, midpoint bit
        }
    }
    __syncthreads();
}

// the two left-aligned coordinates X = x << 2 | mid of pair q of the loaded chunk
template <class Tab>
__device__ __forceinline__ uint2 sobol_coords(const Tab& tab, int q, const SobolLane& sl) {
    HMC_DCHECK(q >= 0 && q <= Tab::kSteps && sl.row >= 0 && sl.row < Tab::kRows && sl.jl < 32u);
    const uint2 t = tab.T[q][sl.jl];
    const uint2 u = tab.U[sl.row][q];
    return make_uint2(t.x ^ u.x, t.y ^ u.y);
}

// the two standard normals (divided by sqrt(2)) of pair q of the loaded chunk
template <class Tab>
__device__ __forceinline__ void sobol_pair(const Tab& tab, int q, const SobolLane& sl,
                                           float& za, float& zb) {
    const uint2 X = sobol_coords(tab, q, sl);
    const float2 z = sobol_normal_X2(X.x, X.y, f2(1.0f));
    za = z.x;
    zb = z.y;
}

// pair q as scaled shocks (k.x z_a, k.y z_b) / sqrt(2): the caller's step
// constants folded into the quantile's last FFMA
template <class Tab>
__device__ __forceinline__ float2 sobol_pair_scaled(const Tab& tab, int q, const SobolLane& sl, float2 k) {
    const uint2 X = sobol_coords(tab, q, sl);
    return sobol_normal_X2(X.x, X.y, k);
}


}  // namespace hmc
