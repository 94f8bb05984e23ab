// hmc_path32.cuh -- fp32 path building blocks shared by the production
// kernels (hmc_fast.cu: single-product Greeks; hmc_surface.cu: strike x
// maturity surfaces): MUFU wrappers, Philox -> Box-Muller step shocks, the
// Giles quantile for Sobol coordinates, and the regrouped Milstein/Euler
// trajectory update with fixing accumulation.  See hmc_fast.cu for the
// algebra and DESIGN.md section 4 for the measurements behind each choice.
#pragma once

#include <cuda_runtime.h>

#include "hmc_device.cuh"


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
// p, opaque to the compiler's uniformity analysis: a block-uniform table
// pointer then stays in vector registers and unrolled loads through it take
// immediate offsets (a uniform one costs a uniform-datapath address
// computation plus two MOVs per load)
template <class T>
__device__ __forceinline__ const T* per_thread_ptr(const T* p) {
    asm("mov.b64 %0, %0;" : "+l"(p));
    return p;
}

// a float2 with both halves x (scalar operand of the paired FFMA2/FMUL2)
__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }
// paired a - b (one FFMA2 with b * -1: exact product, one rounding, = a - b)
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, f2(-1.0f), a); }

// uniform in [1, 2) from the top 23 bits of x: one LEA.HI
__device__ __forceinline__ float one_to_two(uint32_t x) {
    return __uint_as_float((x >> 9) + 0x3f800000u);
}

// Box-Muller on two Philox words; returns the step shocks
//   z1l = sqrt(dt) z1 log2(e),   sz2 = sigma sqrt(dt) (rho z1 + sqrt(1-rho^2) zb)
__device__ __forceinline__ void sincos_turns(float fa, float& sn, float& cs) {
    const float th = fmaf(fa, 6.28318530717958647692f, -9.42477796076937971538f);
    sn = __sinf(th);                                         // th in [-pi, pi)
    cs = __cosf(th);
}

__device__ __forceinline__ void box_muller_f(float fr, float fa, const KernelArgs& a,
                                             float& z1l, float& sz2) {
    const float u1 = 2.0f - fr;                              // (0, 1]
    const float R = sqrta(lg2a(u1) * a.f_bm2);               // sqrt(dt) sqrt(-2 ln u1) log2 e
    float sn, cs;
    sincos_turns(fa, sn, cs);
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

// Standard-normal quantile of a Sobol coordinate, Giles' single-precision
// erfinv: z = sqrt(2) erfinv(2u - 1).  Coordinates arrive LEFT-ALIGNED:
// X = x << 2 | mid, u = X 2^-32, with mid = 0 for the reference's
// unscrambled points (u = x 2^-30, x >= 1) and mid = 2 for digitally
// shifted points (cell midpoints (x + 1/2) 2^-30, x = 0 possible).  Then
//   t = min(X, 2^32 - X) = (X ^ m) - m,  m = X >> 31 (arithmetic)
// is exact integer work (2^32 - X = ~X + 1), tf = t 2^-32 = min(u, 1 - u)
// keeps full relative precision in both tails, w = -ln(4 tf (1 - tf)) and
// |2u - 1| = 1 - 2 tf with the sign of 2u - 1 = the top bit of X.
// Returns k z / sqrt(2): callers fold sqrt(2) and their own scale k > 0 in.
// The tail polynomial (w >= 5, 0.3 % of draws) runs only in warps where a
// lane needs it (warp vote), the extreme cells (w >= 16, t < ~3e-8, where
// Giles' float erfinv is out of range) take Acklam's lower-tail rational
// (the reference's ndtri, _core.pyx:75-109) on tf.
constexpr float kTwoM32 = 2.3283064365386962890625e-10f;   // 2^-32
constexpr float kLn2 = 0.69314718055994530942f;

// min(X, 2^32 - X) 2^-32 = min(u, 1 - u).  umin(X, -X) is at most 2^31 (at
// u = 1/2), which ptxas 12.9 computes as IABS and then converts as a SIGNED
// integer (X = 2^31 -> -2^31) even through an explicit cvt.rn.f32.u32; the
// |.| of the converted value (a free FMUL operand modifier) makes the result
// exact for every X.
__device__ __forceinline__ float sobol_tail_frac(uint32_t X) {
    const uint32_t t = min(X, 0u - X);
    return fabsf(__int2float_rn((int)t)) * kTwoM32;
}

__device__ __forceinline__ float sobol_sign(float v, uint32_t X) {   // v with the sign of 2u - 1
    return __uint_as_float(__float_as_uint(v) ^ (~X & 0x80000000u));
}

// Acklam lower tail on tf (z < 0), the extreme cells
__device__ __forceinline__ float acklam_lower_tail(float tf) {
    const float qa = sqrta(-1.38629436111989061883f * lg2a(tf));   // sqrt(-2 ln t)
    const float num = fmaf(fmaf(fmaf(fmaf(fmaf(-7.784894002430293e-03f, qa, -3.223964580411365e-01f), qa,
                                         -2.400758277161838e+00f), qa, -2.549732539343734e+00f), qa,
                               4.374664141464968e+00f), qa, 2.938163982698783e+00f);
    const float den = fmaf(fmaf(fmaf(fmaf(7.784695709041462e-03f, qa, 3.224671290700398e-01f), qa,
                                    2.445134137142996e+00f), qa, 3.754408661907416e+00f), qa, 1.0f);
    return __fdividef(num, den) * 0.70710678118654752440f;
}

__device__ __forceinline__ float giles_central(float wc) {   // wc = w - 2.5
    float p = 2.81022636e-08f;
    p = fmaf(p, wc, 3.43273939e-07f);
    p = fmaf(p, wc, -3.5233877e-06f);
    p = fmaf(p, wc, -4.39150654e-06f);
    p = fmaf(p, wc, 0.00021858087f);
    p = fmaf(p, wc, -0.00125372503f);
    p = fmaf(p, wc, -0.00417768164f);
    p = fmaf(p, wc, 0.246640727f);
    return fmaf(p, wc, 1.50140941f);
}

__device__ __forceinline__ float giles_tail(float wt) {      // wt = sqrt(w) - 3
    float q = -0.000200214257f;
    q = fmaf(q, wt, 0.000100950558f);
    q = fmaf(q, wt, 0.00134934322f);
    q = fmaf(q, wt, -0.00367342844f);
    q = fmaf(q, wt, 0.00573950773f);
    q = fmaf(q, wt, -0.0076224613f);
    q = fmaf(q, wt, 0.00943887047f);
    q = fmaf(q, wt, 1.00167406f);
    return fmaf(q, wt, 2.83297682f);
}

// scalar form: k z / sqrt(2) of one left-aligned coordinate
__device__ __forceinline__ float sobol_normal_X(uint32_t X, float k) {
    const float tf = sobol_tail_frac(X);
    const float pr = fmaf(-tf, tf, tf);                                  // tf (1 - tf)
    const float wc = fmaf(lg2a(pr), -kLn2, -2.0f * kLn2 - 2.5f);         // w - 2.5
    float p = giles_central(wc);
    if (__any_sync(0xffffffffu, wc >= 2.5f)) {
        const float q = giles_tail(sqrta(wc + 2.5f) - 3.0f);
        p = wc >= 2.5f ? q : p;
        if (__any_sync(0xffffffffu, wc >= 13.5f)) {
            const float z = acklam_lower_tail(tf) * k;
            if (wc >= 13.5f) return sobol_sign(-z, X);
        }
    }
    return p * sobol_sign(fmaf(tf, -2.0f * k, k), X);
}

// the rare part of sobol_normal_X2 (a lane of the warp has w >= 5): Giles'
// tail polynomial, and for the extreme cells the scalar path.  (Out of line
// it would keep the unrolled step loop small, but the call costs more than
// the instruction-cache misses it saves: RQMC Asian 2^22 x 252, 8-step
// unroll, 3.51 vs 3.33 ms.)  done: the value is the final result; else it
// is the corrected polynomial value.
struct SobolTail {
    float2 v;   // the final result (done) or the corrected polynomial value
    bool done;
};

__device__ __forceinline__ SobolTail sobol_tail2(float2 wc, float2 tf, uint32_t Xa, uint32_t Xb, float2 k, float2 p) {
    const float2 wt = __fadd2_rn(make_float2(sqrta(wc.x + 2.5f), sqrta(wc.y + 2.5f)), f2(-3.0f));
    float2 q = f2(-0.000200214257f);
    q = __ffma2_rn(q, wt, f2(0.000100950558f));
    q = __ffma2_rn(q, wt, f2(0.00134934322f));
    q = __ffma2_rn(q, wt, f2(-0.00367342844f));
    q = __ffma2_rn(q, wt, f2(0.00573950773f));
    q = __ffma2_rn(q, wt, f2(-0.0076224613f));
    q = __ffma2_rn(q, wt, f2(0.00943887047f));
    q = __ffma2_rn(q, wt, f2(1.00167406f));
    q = __ffma2_rn(q, wt, f2(2.83297682f));
    p.x = wc.x >= 2.5f ? q.x : p.x;
    p.y = wc.y >= 2.5f ? q.y : p.y;
    if (__any_sync(0xffffffffu, fmaxf(wc.x, wc.y) >= 13.5f)) {   // extreme cells: the scalar path
        const float2 xk = __ffma2_rn(tf, make_float2(-2.0f * k.x, -2.0f * k.y), k);
        const float2 r = __fmul2_rn(p, make_float2(sobol_sign(xk.x, Xa), sobol_sign(xk.y, Xb)));
        const float sa = sobol_normal_X(Xa, k.x), sb = sobol_normal_X(Xb, k.y);   // all lanes
        return {make_float2(wc.x >= 13.5f ? sa : r.x, wc.y >= 13.5f ? sb : r.y), true};
    }
    return {p, false};
}

// both coordinates of a step at once: the same per-lane arithmetic as the
// scalar form (bit-identical), the float work as paired FFMA2/FMUL2; k is
// the per-coordinate scale
// k2 = -2k (callers in hot loops pass it precomputed)
__device__ __forceinline__ float2 sobol_normal_X2(uint32_t Xa, uint32_t Xb, float2 k, float2 k2) {
    const float2 tf = make_float2(sobol_tail_frac(Xa), sobol_tail_frac(Xb));
    const float2 pr = __ffma2_rn(make_float2(-tf.x, -tf.y), tf, tf);
    const float2 wc = __ffma2_rn(make_float2(lg2a(pr.x), lg2a(pr.y)), f2(-kLn2), f2(-2.0f * kLn2 - 2.5f));
    float2 p = f2(2.81022636e-08f);
    p = __ffma2_rn(p, wc, f2(3.43273939e-07f));
    p = __ffma2_rn(p, wc, f2(-3.5233877e-06f));
    p = __ffma2_rn(p, wc, f2(-4.39150654e-06f));
    p = __ffma2_rn(p, wc, f2(0.00021858087f));
    p = __ffma2_rn(p, wc, f2(-0.00125372503f));
    p = __ffma2_rn(p, wc, f2(-0.00417768164f));
    p = __ffma2_rn(p, wc, f2(0.246640727f));
    p = __ffma2_rn(p, wc, f2(1.50140941f));
    if (__builtin_expect(__any_sync(0xffffffffu, fmaxf(wc.x, wc.y) >= 2.5f), 0)) {
        const SobolTail r = sobol_tail2(wc, tf, Xa, Xb, k, p);
        if (r.done) return r.v;
        p = r.v;
    }
    const float2 xk = __ffma2_rn(tf, k2, k);   // k |2u - 1|
    return __fmul2_rn(p, make_float2(sobol_sign(xk.x, Xa), sobol_sign(xk.y, Xb)));
}

__device__ __forceinline__ float2 sobol_normal_X2(uint32_t Xa, uint32_t Xb, float2 k) {
    return sobol_normal_X2(Xa, Xb, k, make_float2(-2.0f * k.x, -2.0f * k.y));
}

constexpr float kSqrt2f = 1.41421356237309504880f;


// The two v0-bumped trajectories run as one float2 pair (.x: v0 + h, .y:
// v0 - h floored at 0) so their updates issue as sm_100 paired FFMA2 --
// the same IEEE fma per lane, half the issue slots.
struct PathState32 {
    float v0, L0;          // base trajectory
    float2 AT;             // base: (fixing sum A0, sum S t)
    float2 D;              // base: (sum S expm1(h t), sum S expm1(-h t))
    float2 vb, Lb, Ab;     // bumped pair

    __device__ __forceinline__ void init(float v0_, float2 vb_) {
        v0 = v0_;
        vb = vb_;
        L0 = 0.0f;
        AT = D = Lb = Ab = make_float2(0.0f, 0.0f);
    }
};

__device__ __forceinline__ void traj_step(float& v, float& L, float z1l, float sz2, float ck,
                                          const KernelArgs& a) {
    const float s = sqrta(v);
    L = fmaf(s, z1l, L);
    L = fmaf(v, a.f_nhdt2, L);
    v = fmaxf(fmaf(s, sz2, fmaf(v, a.f_omkdt, ck)), 0.0f);
}

// traj_step on the bumped pair, operation for operation; PAIR issues it as
// paired FFMA2 (bit-identical).  Measured (tools/kernel_variants.py, 2^24 x
// 252): European 8.44 -> 8.20 ms, RQMC Sobol Asian 3.98 -> 3.93 ms; the
// MUFU-bound daily-fixing pseudo-random Asian loses 0.3 % and keeps scalar.
template <bool PAIR>
__device__ __forceinline__ void traj_step2(float2& v, float2& L, float z1l, float sz2, float ck,
                                           const KernelArgs& a) {
    if (PAIR) {
    const float2 s = make_float2(sqrta(v.x), sqrta(v.y));
    L = __ffma2_rn(s, f2(z1l), L);
    L = __ffma2_rn(v, f2(a.f_nhdt2), L);
    const float2 t = __ffma2_rn(s, f2(sz2), __ffma2_rn(v, f2(a.f_omkdt), f2(ck)));
    v = make_float2(fmaxf(t.x, 0.0f), fmaxf(t.y, 0.0f));
    } else {
    traj_step(v.x, L.x, z1l, sz2, ck, a);
    traj_step(v.y, L.y, z1l, sz2, ck, a);
    }
}

template <bool GREEKS, bool PAIR>
__device__ __forceinline__ void advance(PathState32& st, float z1l, float sz2, const KernelArgs& a) {
    const float ck = fmaf(sz2 * sz2, a.f_cmil2, a.f_ck0);
    traj_step(st.v0, st.L0, z1l, sz2, ck, a);
    if (GREEKS) traj_step2<PAIR>(st.vb, st.Lb, z1l, sz2, ck, a);
}

template <bool GREEKS, bool PAIR = false>
__device__ __forceinline__ void fixing(PathState32& st, const float4 w) {
    const float P = ex2a(st.L0);
    if (!GREEKS) {
        st.AT.x = fmaf(P, w.x, st.AT.x);
    } else if (PAIR) {   // the same four fmas as paired FFMA2 (issue-bound drivers)
        st.AT = __ffma2_rn(f2(P), make_float2(w.x, w.y), st.AT);
        st.D = __ffma2_rn(f2(P), make_float2(w.z, w.w), st.D);
    } else {
        st.AT.x = fmaf(P, w.x, st.AT.x);
        st.AT.y = fmaf(P, w.y, st.AT.y);
        st.D.x = fmaf(P, w.z, st.D.x);
        st.D.y = fmaf(P, w.w, st.D.y);
    }
    if (GREEKS) {
        // (carrying Au - A0 instead -- one more FADD per trajectory and
        // fixing -- shrinks Vega's fp32 error ~40x but costs 4 % of the
        // daily-fixing kernel: 10.66 -> 11.08 ms; not taken)
        if (PAIR) {
            st.Ab = __ffma2_rn(make_float2(ex2a(st.Lb.x), ex2a(st.Lb.y)), f2(w.x), st.Ab);
        } else {
            st.Ab.x = fmaf(ex2a(st.Lb.x), w.x, st.Ab.x);
            st.Ab.y = fmaf(ex2a(st.Lb.y), w.x, st.Ab.y);
        }
    }
}

// PAIR: the bumped trajectories as paired FFMA2 (see traj_step2); wk: this
// step's fixing-weight entry (a.steps32 + k)
template <int FIX, bool GREEKS, bool PAIR = false>
__device__ __forceinline__ void step_w(PathState32& st, const float4* wk, float z1l, float sz2,
                                       const KernelArgs& a) {
    advance<GREEKS, PAIR>(st, z1l, sz2, a);
    if (FIX == kFixEvery) {
        fixing<GREEKS, PAIR>(st, __ldg(wk));
    } else if (FIX == kFixTable) {
        const float4 w = __ldg(wk);
        if (w.x != 0.0f) fixing<GREEKS, PAIR>(st, w);
    }
}

template <int FIX, bool GREEKS, bool PAIR = false>
__device__ __forceinline__ void step(PathState32& st, int k, float z1l, float sz2,
                                     const KernelArgs& a) {
    HMC_DCHECK(k >= 1 && k <= a.n_sim);
    step_w<FIX, GREEKS, PAIR>(st, a.steps32 + k, z1l, sz2, a);
}

}  // namespace hmc
