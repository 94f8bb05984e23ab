// hmc_exact.cu -- Broadie-Kaya exact simulation on sm_100a.
//
// The reference's exact scheme (_core.pyx:112-347, 415-521; exact.py;
// ivlaw.py) one path per thread in fp64, same random stream, same algorithm:
//   variance transition  v_t = c (Gamma(d/2 - 1/2, 2) + (Z + sqrt(lambda))^2)
//                        Gamma by Marsaglia-Tsang on the path's gamma substream
//   integrated variance  inverse of the Fourier-series CDF
//                        F(x) = h x / pi + 2/pi sum_j sin(j h x)/j Re Phi(j h)
//                        of the conditional characteristic function Phi
//                        (modified Bessel series of complex argument), nodes
//                        added until a tail criterion holds, second-order
//                        Newton with bracketing and a bisection fallback
//   log price            ln S += r dt - iv/2 + rho W2 + sqrt((1-rho^2) iv) Z3
// Compiled with -fmad=false like the replay kernels.  Error codes follow
// _core.pyx:36-40 and surface as BesselNonConvergence /
// QuadratureNonConvergence / RootNotBracketed in Python.
//
// The reference caches Re Phi at up to MAX_NODES = 20000 nodes per call;
// here the first kCacheNodes live in a per-thread slice of a device scratch
// buffer (node-major, coalesced) and any further node is recomputed on the
// fly -- identical values, bounded memory.  Typical node counts are 20-130.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "hmc_device.cuh"
#include "hmc_launch.h"
#include "hmc_ndtri64.cuh"

namespace hmc {

#ifndef HMC_EXACT_NOINLINE
#define HMC_EXACT_NOINLINE 1
#endif
#if HMC_EXACT_NOINLINE
#define HMC_EXACT_FN __device__ __noinline__
#else
#define HMC_EXACT_FN __device__
#endif

namespace {

constexpr int kMaxNodes = 20000;
constexpr double kTailTol = 1e-7;
constexpr int kTailRun = 3;
constexpr double kNewtonTol = 1e-7;
constexpr int kNewtonMaxIter = 100;
constexpr int kBisectMaxIter = 200;
constexpr double kPeriodStds = 12.0;
constexpr double kDegenerateRelStd = 1e-5;
constexpr double kPi = 3.14159265358979323846;
constexpr int kRotSeed = 32;

struct cplx {
    double re, im;
};
__device__ __forceinline__ cplx cx(double re, double im = 0.0) { return {re, im}; }
__device__ __forceinline__ cplx operator+(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx operator-(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cplx operator*(cplx a, cplx b) {
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__device__ __forceinline__ cplx operator*(double s, cplx a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cplx operator/(cplx a, double s) {
    const double r = 1.0 / s;  // one division
    return {a.re * r, a.im * r};
}
// Smith's algorithm (robust complex division)
__device__ __forceinline__ cplx operator/(cplx a, cplx b) {
    // (one reciprocal of d instead of two divisions by it)
    if (fabs(b.re) >= fabs(b.im)) {
        const double r = b.im / b.re, id = 1.0 / (b.re + b.im * r);
        return {(a.re + a.im * r) * id, (a.im - a.re * r) * id};
    }
    const double r = b.re / b.im, id = 1.0 / (b.re * r + b.im);
    return {(a.re * r + a.im) * id, (a.im * r - a.re) * id};
}
// |a|: the magnitudes here are moderate (Bessel arguments <= 50, series
// values <= e^50), so sqrt(re^2 + im^2) cannot over/underflow where hypot's
// scaling would matter; within an ulp of hypot at a third of the cost
__device__ __forceinline__ double norm2_(cplx a) { return a.re * a.re + a.im * a.im; }
__device__ __forceinline__ double cabs_(cplx a) { return sqrt(norm2_(a)); }
__device__ __forceinline__ cplx cexp_(cplx a) {
    const double e = exp(a.re);
    double s, c;
    sincos(a.im, &s, &c);
    return {e * c, e * s};
}
// principal square root
__device__ __forceinline__ cplx csqrt_(cplx a) {
    if (a.re == 0.0 && a.im == 0.0) return {0.0, a.im};
    const double t = sqrt(0.5 * (cabs_(a) + fabs(a.re)));
    if (a.re >= 0.0) return {t, a.im / (2.0 * t)};
    return {fabs(a.im) / (2.0 * t), copysign(t, a.im)};
}

enum { kErrNone = 0, kErrBesselRange = 1, kErrBesselConv = 2, kErrQuad = 3, kErrRoot = 4 };

// power series of the modified Bessel function I_nu(z) / ((z/2)^nu / Gamma(nu+1))
// (_core.pyx:143-159)
// inv_kn: optional table of 1 / (k (nu + k)), k = 1..kBesselTerms, for the
// kernels whose nu is fixed per launch (the same IEEE quotient the division
// computes -- bit-identical -- but a shared-memory load instead of a fp64
// reciprocal per term)
constexpr int kBesselTerms = 400;
HMC_EXACT_FN cplx bessel_series(double nu, cplx z, int* err, const double* inv_kn = nullptr) {
    if (cabs_(z) > 50.0) {
        *err = kErrBesselRange;
        return cx(0.0);
    }
    const cplx q = 0.25 * (z * z);
    cplx term = cx(1.0), total = cx(1.0);
    for (int k = 1; k <= kBesselTerms; ++k) {
        term = inv_kn ? inv_kn[k - 1] * (term * q) : term * q / (k * (nu + k));
        total = total + term;
        // |term| < 1e-12 |total|, compared squared (no square roots)
        if (norm2_(term) < 1e-24 * norm2_(total)) return total;
    }
    *err = kErrBesselConv;
    return total;
}

// conditional characteristic function of the integrated variance
// (_core.pyx:162-188), split into the per-path constants (PhiPath: every
// term that does not depend on the transform variable a, including the
// denominator Bessel series of real argument) and the per-node part.  The
// reference re-evaluates all of it at every node; hoisting is bit-identical
// (same operations on the same inputs) and removes one of the two series.
struct PhiPath {
    double kappa, sigma2, nu, tau;
    double ek, one_m_ek, kb, vs, w, log1m_ek, ekh_inv;  // ekh_inv = e^{kappa tau / 2}
    cplx den;      // bessel_series(nu, w coeff_k)
    int den_err;   // its error code (kErrNone = 0)
    const double* inv_kn;  // bessel_series' optional 1 / (k (nu + k)) table
    // per-path quotients of phi_node, hoisted (the same IEEE operations on
    // the same inputs: bit-identical to evaluating them at every node)
    double inv_kappa;   // 1 / kappa                  (g / kappa)
    double lead_c;      // e^{kappa tau/2} (1 - e^{-kappa tau}) / kappa
    double four_s2;     // 4 / sigma^2
    double inv_den;     // 1 / den.re                 (ser / den.re)
};

HMC_EXACT_FN PhiPath phi_path(double kappa, double sigma2, double nu, double v_u, double v_t, double tau,
                              const double* inv_kn = nullptr) {
    PhiPath P;
    P.inv_kn = inv_kn;
    P.kappa = kappa;
    P.sigma2 = sigma2;
    P.nu = nu;
    P.tau = tau;
    P.ek = exp(-kappa * tau);
    P.one_m_ek = 1.0 - P.ek;
    P.kb = kappa * (1.0 + P.ek) / (1.0 - P.ek);
    P.vs = (v_u + v_t) / sigma2;
    const double ekh = exp(-0.5 * kappa * tau);
    P.ekh_inv = exp(0.5 * kappa * tau);
    const double coeff_k = 4.0 * kappa * ekh / (sigma2 * (1.0 - ekh * ekh));
    P.w = sqrt(v_u * v_t);
    P.log1m_ek = log(1.0 - P.ek);
    P.den_err = 0;
    P.den = bessel_series(nu, cx(P.w * coeff_k), &P.den_err, inv_kn);
    P.inv_kappa = 1.0 / kappa;
    P.lead_c = P.ekh_inv * P.one_m_ek / kappa;
    P.four_s2 = 4.0 / sigma2;
    P.inv_den = 1.0 / P.den.re;
    return P;
}

HMC_EXACT_FN cplx phi_node(const PhiPath& P, double a, int* err) {
    if (a == 0.0) return cx(1.0);
    const double kappa = P.kappa, sigma2 = P.sigma2, nu = P.nu, tau = P.tau;
    const cplx g = csqrt_(cx(kappa * kappa, -2.0 * sigma2 * a));
    // The reference's formula, regrouped (same mathematics, last-ulp
    // differences): e^{-g tau / 2} once -- e^{-g tau} is its square and the
    // lead factor's e^{-(g - kappa) tau / 2} is it times e^{kappa tau / 2};
    // the three quotients by 1 - e^{-g tau} share one reciprocal (the
    // Bessel argument's 1 - e^{-g tau}... is the same 1 - egh^2), and
    // g e^{-g tau / 2} / (1 - e^{-g tau}) is shared by the lead factor and
    // the Bessel argument; the two outer exponentials are one.
    const cplx egh = cexp_(-0.5 * (g * cx(tau)));
    const cplx eg = egh * egh;
    const cplx one = cx(1.0);
    const cplx ome = one - eg;
    const cplx inv_ome = one / ome;
    const cplx ge = (g * egh) * inv_ome;
    const cplx lead = P.lead_c * ge;
    const cplx bracket = cx(P.kb) - (g * (one + eg)) * inv_ome;
    const cplx coeff_g = P.four_s2 * ge;
    // log q = log(g / kappa) - (g - kappa) tau / 2 + log(1 - e^{-kappa tau}) - log(1 - e^{-g tau}),
    // the two real logarithms merged into one, and the two arguments too:
    // Re g > 0 (principal root), so |e^{-g tau}| < 1 and Re(1 - e^{-g tau}) > 0
    // -- both principal arguments lie in (-pi/2, pi/2), their difference in
    // (-pi, pi), so arg(g/kappa) - arg(ome) = arg(g/kappa conj(ome)) exactly
    // (one atan2 instead of two: they were ~11 % of the kernel's samples)
    const cplx gk = {g.re * P.inv_kappa, g.im * P.inv_kappa};   // g / kappa (operator/ is r = 1/s, then a r)
    const cplx half_gt = 0.5 * ((g - cx(kappa)) * cx(tau));
    const cplx gko = gk * cx(ome.re, -ome.im);
    const cplx log_q = {0.5 * log(norm2_(gk) / norm2_(ome)) - half_gt.re + P.log1m_ek,
                        atan2(gko.im, gko.re) - half_gt.im};
    const cplx expo = cexp_(P.vs * bracket + nu * log_q);   // e^{vs bracket} q^nu
    const cplx ser = bessel_series(nu, P.w * coeff_g, err, P.inv_kn);
    if (P.den_err != kErrNone) *err = P.den_err;
    // the denominator series has a real argument: real (ser / den.re, as r = 1/s then ser r)
    return lead * expo * cx(ser.re * P.inv_den, ser.im * P.inv_den);
}

// Marsaglia-Tsang on the reference stream (_core.pyx:116-136), from draw
// ctr0 of the stream; *used = draws consumed
HMC_EXACT_FN double sample_gamma_from(unsigned long long key, unsigned long long ctr0, double shape,
                                      double scale, unsigned long long* used) {
    double boost = 1.0, alpha = shape;
    unsigned long long ctr = ctr0;
    if (alpha < 1.0) {
        boost = pow(uniform_at(key, ctr), 1.0 / alpha);
        alpha += 1.0;
        ctr += 1;
    }
    const double d = alpha - 1.0 / 3.0;
    const double c = 1.0 / sqrt(9.0 * d);
    while (true) {
        const double x = ndtri_ref(uniform_at(key, ctr));
        double u = uniform_at(key, ctr + 1);
        ctr += 2;
        double v = 1.0 + c * x;
        if (v <= 0.0) continue;
        v = v * v * v;
        if (u < 1e-300) u = 1e-300;
        if (log(u) < 0.5 * x * x + d - d * v + d * log(v)) {
            *used = ctr - ctr0;
            return boost * d * v * scale;
        }
    }
}

HMC_EXACT_FN double sample_gamma(unsigned long long key, double shape, double scale) {
    unsigned long long used;
    return sample_gamma_from(key, 0ULL, shape, scale, &used);
}

struct NodeCache {
    double* base;  // scratch + thread slot; node j at base[j * stride]
    long long stride;
    int cap;
    // for recomputation past the cache
    const PhiPath* P;
    double h;
    __device__ double re(int j, int* err) const {  // j 0-based
        HMC_DCHECK(j >= 0);
        if (j < cap) return base[(size_t)j * stride];
        return phi_node(*P, (j + 1) * h, err).re;
    }
};

// 1 / j for the Fourier-series weights: a constant-memory table (the node
// index is warp-uniform, so the load broadcasts) instead of a division
constexpr int kInvTable = 512;
struct InvIntTable {
    double v[kInvTable];
    constexpr InvIntTable() : v() {
        for (int j = 1; j < kInvTable; ++j) v[j] = 1.0 / j;  // IEEE quotient, as __drcp_rn
    }
};
__constant__ InvIntTable c_inv_int = InvIntTable();
__device__ __forceinline__ double inv_int(int j) { return j < kInvTable ? c_inv_int.v[j] : __drcp_rn((double)j); }

// F(x) - the CDF of the Fourier-series inversion -- and its first two
// derivatives accumulated node by node (the reference's Newton sums,
// _core.pyx:276-287); sin / cos (j h x) by rotation from (h x), re-seeded
// from sincos every kRotSeed nodes (drift ~1e-16 per node: the reference's
// per-node sin / cos to ~1e-15)
struct NewtonSums {
    double h, x, f, d1, d2, sr, cr, sx, cxv;
    int seed;
    __device__ NewtonSums(double h_, double x_) : h(h_), x(x_), f(h_ * x_ / kPi), d1(h_ / kPi), d2(0.0),
                                                  sx(0.0), cxv(1.0), seed(0) {
        sincos(h * x, &sr, &cr);
    }
    __device__ __forceinline__ void add(int j, double rp) {
        const double s_j = j * h;
        if (seed == 0) {
            sincos(s_j * x, &sx, &cxv);
            seed = kRotSeed;
        } else {
            const double sn = sx * cr + cxv * sr;
            cxv = cxv * cr - sx * sr;
            sx = sn;
        }
        --seed;
        f += (2.0 / kPi) * sx * inv_int(j) * rp;
        d1 += (2.0 * h / kPi) * cxv * rp;
        d2 -= (2.0 * h / kPi) * s_j * sx * rp;
    }
};

__device__ double cdf_at(double x, double h, int n, const NodeCache& nc, int* err) {
    double f = h * x / kPi;
    for (int j = 1; j <= n; ++j) f += (2.0 / kPi) * sin(j * h * x) / j * nc.re(j - 1, err);
    return f;
}

HMC_EXACT_FN double bisect_iv(double u, double lo, double hi, double h, int n, const NodeCache& nc,
                            int* err) {
    const double f_hi = cdf_at(hi, h, n, nc, err);
    if (f_hi < u - kNewtonTol) {
        if (f_hi < u - 1e-4) {
            *err = kErrRoot;
            return 0.0;
        }
        return hi;
    }
    double x = 0.5 * (lo + hi);
    for (int it = 0; it < kBisectMaxIter; ++it) {
        const double f = cdf_at(x, h, n, nc, err);
        if (fabs(f - u) < kNewtonTol) return x;
        if (f > u)
            hi = x;
        else
            lo = x;
        x = 0.5 * (lo + hi);
        if (hi - lo < 1e-16 * (1.0 + hi)) break;
    }
    if (fabs(cdf_at(x, h, n, nc, err) - u) < 1e-6) return x;
    *err = kErrRoot;
    return 0.0;
}

// The law of the conditional integrated variance (ivlaw.py
// IntegratedVarianceLaw.__post_init__ / _moments, _core.pyx:195-240): the
// point-mass and degenerate regimes, else the moments from Phi at a small
// frequency and the quadrature step h; P is the per-path part of Phi.
enum { kLawQuadrature = 0, kLawPointMass = 1, kLawDegenerate = 2 };
struct IvLaw {
    double mean, std, h;
    int kind;
};

__device__ __forceinline__ IvLaw iv_law(double kappa, double theta, double sigma, double dof, double v_u,
                                        double v_t, double dt, PhiPath& P, int* err,
                                        const double* inv_kn = nullptr) {
    const double sigma2 = sigma * sigma;
    const double nu = 0.5 * dof - 1.0;
    IvLaw L{0.0, 0.0, 0.0, kLawQuadrature};
    if (sigma < 1e-4 * kappa) {
        L.mean = theta * dt + (v_u - theta) * (1.0 - exp(-kappa * dt)) / kappa;
        L.kind = kLawPointMass;
        return L;
    }
    double scale = 0.5 * (v_u + v_t);
    if (scale < 0.01 * theta) scale = 0.01 * theta;
    scale *= dt;
    double m1 = scale, eps;
    cplx phi;
    P = phi_path(kappa, sigma2, nu, v_u, v_t, dt, inv_kn);
    for (int it = 0; it < 2; ++it) {
        eps = 0.05 / m1;
        phi = phi_node(P, eps, err);
        const double m1_new = phi.im / eps;
        if (!(m1_new > 0.0) || !isfinite(m1_new)) break;
        m1 = m1_new;
    }
    eps = 0.05 / m1;
    phi = phi_node(P, eps, err);
    m1 = phi.im / eps;
    const double m2 = -2.0 * (phi.re - 1.0) / (eps * eps);
    double var = m2 - m1 * m1;
    if (var < 0.0) var = 0.0;
    L.mean = m1;
    L.std = sqrt(var);
    if (L.std < kDegenerateRelStd * L.mean) L.kind = kLawDegenerate;
    L.h = 2.0 * kPi / (L.mean + kPeriodStds * L.std);
    return L;
}

// Re Phi at the quadrature nodes j h, j = 1.., into the cache until the tail
// criterion holds (_core.pyx: (2/pi) |Phi(j h)| / j below tolerance for
// kTailRun nodes in a row); on_node(j, Re Phi) sees every node.  Returns
// the node count (0 with *err set past kMaxNodes).
template <class OnNode>
__device__ __forceinline__ int iv_nodes(const PhiPath& P, double h, const NodeCache& nc, OnNode on_node,
                                        int* err) {
    int n = 0, run = 0;
    while (run < kTailRun) {
        if (n >= kMaxNodes) {
            *err = kErrQuad;
            return 0;
        }
        const int j = n + 1;
        const cplx p = phi_node(P, j * h, err);
        if (*err != kErrNone) return 0;
        if (n < nc.cap) nc.base[(size_t)n * nc.stride] = p.re;
        on_node(j, p.re);
        // (2/pi) |p| / j < tol, compared squared
        const double tj = kTailTol * j;
        if ((4.0 / (kPi * kPi)) * norm2_(p) < tj * tj)
            ++run;
        else
            run = 0;
        ++n;
    }
    return n;
}

// inverse-CDF draw of the conditional integrated variance (_core.pyx:195-310)
__device__ double sample_iv(double kappa, double theta, double sigma, double dof, double v_u,
                            double v_t, double dt, double u, NodeCache& nc, int* err,
                            const double* inv_kn = nullptr) {
    if (u < 1e-12) u = 1e-12;
    if (u > 1.0 - 1e-12) u = 1.0 - 1e-12;
    PhiPath P;
    const IvLaw L = iv_law(kappa, theta, sigma, dof, v_u, v_t, dt, P, err, inv_kn);
    if (L.kind == kLawPointMass) return L.mean;
    if (*err != kErrNone) return 0.0;
    if (L.kind == kLawDegenerate) {
        const double r = L.mean + L.std * ndtri_ref(u);
        return r > 0.0 ? r : 0.0;
    }
    const double h = L.h, mean = L.mean;
    nc.P = &P;
    nc.h = h;

    // the first Newton iterate is known before the nodes: its sums are
    // accumulated while the nodes are generated (same order, same
    // arithmetic as a separate pass), saving one pass over the nodes
    double lo = 0.0, hi = 2.0 * kPi / h, x = mean;
    if (x < 1e-3 * hi) x = 1e-3 * hi;
    if (x > 0.9 * hi) x = 0.9 * hi;
    NewtonSums first(h, x);
    const int n = iv_nodes(P, h, nc, [&](int j, double re) { first.add(j, re); }, err);
    if (*err != kErrNone) return 0.0;

    for (int it = 0; it < kNewtonMaxIter; ++it) {
        NewtonSums ns = first;
        if (it > 0) {
            ns = NewtonSums(h, x);
            double rp_next = nc.re(0, err);  // node loads issue one node ahead
            for (int j = 1; j <= n; ++j) {
                const double rp = rp_next;
                if (j < n) rp_next = nc.re(j, err);
                ns.add(j, rp);
            }
        }
        const double f = ns.f, d1 = ns.d1, d2 = ns.d2;
        const double efun = f - u;
        if (fabs(efun) < kNewtonTol) return x;
        if (efun > 0.0) {
            if (x < hi) hi = x;
        } else {
            if (x > lo) lo = x;
        }
        bool have_step = false;
        double step = 0.0;
        if (d1 > 0.0) {
            const double disc = 1.0 - 2.0 * efun * d2 / (d1 * d1);
            if (fabs(d2) < 1e-300 || fabs(2.0 * efun * d2) < 1e-12 * d1 * d1) {
                step = -efun / d1;
                have_step = true;
            } else if (disc > 0.0) {
                step = -(d1 / d2) * (1.0 - sqrt(disc));
                have_step = true;
            }
        }
        if (!have_step || x + step <= lo || x + step >= hi)
            x = 0.5 * (lo + hi);
        else
            x = x + step;
    }
    return bisect_iv(u, lo, hi, h, n, nc, err);
}

}  // namespace

// Two register budgets, picked per launch by exact_plan: a wide one for jobs
// of a few waves and a deep one for long grid-stride loops.  The series,
// characteristic-function, Gamma and bisection routines are out-of-line
// calls (HMC_EXACT_NOINLINE): inlined at every call site the kernel was
// 431 KB of SASS and stalled on instruction fetch; out of line it is 136 KB
// and 2^20 paths run in 28.6 instead of 33.1 ms (tools/exact_prof.py).  With
// call frames on the stack, higher occupancy then pays a little: 8 / 6
// blocks per SM (64 / 80 registers) against the inlined kernel's 4 / 3
// (128 / 158): 2^17 paths 4.3 ms, 2^20 26-28 ms (noise +-5 %).
template <int MINB>
__global__ void __launch_bounds__(kExactThreads, MINB) exact_batch_kernel(const ExactArgs e) {
    const long long n = e.path_hi - e.path_lo;
    const long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    // the Bessel series' 1 / (k (nu + k)) for this launch's nu, once per block
    __shared__ double inv_kn[kBesselTerms];
    {
        const double nu = 0.5 * e.dof - 1.0;
        for (int k = threadIdx.x + 1; k <= kBesselTerms; k += blockDim.x) inv_kn[k - 1] = 1.0 / (k * (nu + k));
        __syncthreads();
    }
    NodeCache nc{};
    nc.base = e.scratch + slot;
    nc.stride = stride;
    nc.cap = kExactCacheNodes;
    const bool point_mass = e.sigma < 1e-4 * e.kappa;
    const long long total = n * e.n_runs;  // (run, path) pairs; row i of uniforms / out
    for (long long i = slot; i < total; i += stride) {
        int err = kErrNone;
        const long long run = i / n, p = i - run * n;
        HMC_DCHECK(run < e.n_runs && slot < stride);
        const unsigned long long key_path = derive(e.key_runs[run], (unsigned long long)(e.path_lo + p));
        const unsigned long long main_key = derive(key_path, 0ULL);
        const unsigned long long gamma_root = derive(key_path, 1ULL);
        double ln_s = log(e.s0), v = e.v0, price_sum = 0.0, tw_sum = 0.0, dp_sum = 0.0, dm_sum = 0.0;
        const double* urow = e.uniforms ? e.uniforms + (size_t)i * 3 * e.n_steps : nullptr;
        // on-device Sobol (engine.py:97-101): point 1 + run N + path, or points
        // 1..N under per-(run, dimension) digital shifts (randomised QMC)
        uint32_t gray = 0;
        if (e.sobol_v) {
            const uint32_t idx = (uint32_t)(1 + (e.sobol_scramble ? 0LL : (e.run_offset + run) * e.sobol_n_paths) +
                                            e.path_lo + p);
            gray = idx ^ (idx >> 1);
        }
        for (int k = 0; k < e.n_steps; ++k) {
            const double dt = e.times[k + 1] - e.times[k];
            double u1, u2, u3;
            if (urow) {
                u1 = urow[3 * k];
                u2 = urow[3 * k + 1];
                u3 = urow[3 * k + 2];
            } else if (e.sobol_v) {
                double uu[3];
                for (int j = 0; j < 3; ++j) {
                    uint32_t x = sobol_coord(gray, e.sobol_v, 3 * e.n_steps, 3 * k + j);
                    double half = 0.0;
                    if (e.sobol_scramble) {
                        x ^= sobol_shift(e.key_runs[run], 3 * k + j);
                        half = 0.5;
                    }
                    uu[j] = ((double)x + half) * (1.0 / 1073741824.0);
                }
                u1 = uu[0];
                u2 = uu[1];
                u3 = uu[2];
            } else {
                u1 = uniform_at(main_key, (unsigned long long)(3 * k));
                u2 = uniform_at(main_key, (unsigned long long)(3 * k + 1));
                u3 = uniform_at(main_key, (unsigned long long)(3 * k + 2));
            }
            const double ek = exp(-e.kappa * dt);
            const double c = e.sigma * e.sigma * (1.0 - ek) / (4.0 * e.kappa);
            const double lam = 4.0 * e.kappa * ek * v / (e.sigma * e.sigma * (1.0 - ek));
            const double z1 = ndtri_ref(u1);
            const double g = sample_gamma(derive(gamma_root, (unsigned long long)k), 0.5 * (e.dof - 1.0), 2.0);
            const double shifted = z1 + sqrt(lam);
            const double v_new = c * (g + shifted * shifted);
            const double iv = sample_iv(e.kappa, e.theta, e.sigma, e.dof, v, v_new, dt, u2, nc, &err, inv_kn);
            if (err != kErrNone) break;
            double int_w2;
            if (point_mass)
                int_w2 = sqrt(iv) * ndtri_ref(u2);
            else
                int_w2 = (v_new - v - e.kappa * e.theta * dt + e.kappa * iv) / e.sigma;
            const double z3 = ndtri_ref(u3);
            double var_ln = (1.0 - e.rho * e.rho) * iv;
            if (var_ln < 0.0) var_ln = 0.0;
            ln_s = ln_s + e.r * dt - 0.5 * iv + e.rho * int_w2 + sqrt(var_ln) * z3;
            v = v_new;
            if (e.flags[k]) {
                const double s_now = exp(ln_s);
                price_sum += s_now;
                tw_sum += s_now * e.times[k + 1];
                if (e.rbump) {
                    dp_sum += s_now * e.rbump[2 * (k + 1)];
                    dm_sum += s_now * e.rbump[2 * (k + 1) + 1];
                }
            }
        }
        const int cols = e.rbump ? 5 : 3;
        double* o = e.out + (size_t)i * cols;
        if (err != kErrNone) {
            atomicMax(e.err_flag, err);
            for (int c = 0; c < cols; ++c) o[c] = 0.0;
            continue;
        }
        o[0] = exp(ln_s);
        o[1] = price_sum / e.n_dates;
        o[2] = tw_sum / e.n_dates;
        if (e.rbump) {  // the r +- h_r averages are A + these (r enters only the drift)
            o[3] = dp_sum / e.n_dates;
            o[4] = dm_sum / e.n_dates;
        }
    }
}

// Per-path estimators of the exact scheme on the device (the engine's
// greeks_epilogue, fp64) from the observables of the base and bumped
// simulations, reduced per 128-path tile like the discretised kernels --
// so exact-scheme jobs use the same chunk exchange and fixed-shape run
// reduction (bit-identical for any number of GPUs).
//   obs*: [run][n][3] (s_T, avg, tw_sum); U/D: v0 +- bumps.  The r +- h_r
//   underlyings need no extra simulation: r enters the scheme only through
//   the log-price drift (_core.pyx exact step), so S_k(r +- h) = S_k e^{+-h t_k}
//   exactly -- European: S_T e^{+-h T}; Asian: A + (1/N) sum S_k expm1(+-h t_k),
//   the base run's columns 3 and 4 ([run][n][5]), as the discretised kernels do.
__global__ void __launch_bounds__(kTile) exact_estimator_kernel(const KernelArgs a, const double* __restrict__ o0,
                                                                const double* __restrict__ oU,
                                                                const double* __restrict__ oD, long long n,
                                                                double ehT, double emhT, double* __restrict__ tiles,
                                                                long long n_tiles, int run0) {
    const int run = blockIdx.y;
    const long long i = (long long)blockIdx.x * kTile + threadIdx.x;
    const bool live = i < n;
    const size_t idx = (size_t)run * n + (live ? i : 0);
    const bool rcols = a.want_greeks && a.is_asian;
    const size_t row = idx * (rcols ? 5 : 3);
    const int col = a.is_asian ? 1 : 0;
    const double A = o0[row + col], tw = o0[row + 2];
    double Au = A, Ad = A, Rp = A * ehT, Rm = A * emhT;
    if (a.want_greeks) {
        Au = oU[idx * 3 + col];
        Ad = oD[idx * 3 + col];
        if (a.is_asian) {
            Rp = A + o0[row + 3];
            Rm = A + o0[row + 4];
        }
    }
    double q[kNQ];
    greeks_epilogue<double>(a, A, tw, Au, Ad, Rp, Rm, q);
    if (!live) {
#pragma unroll
        for (int k = 0; k < kNQ; ++k) q[k] = 0.0;
    }
    tile_reduce_store(q, tiles + ((size_t)(run0 + run) * n_tiles + blockIdx.x) * kNW);
}

cudaError_t launch_exact_estimators(const KernelArgs& a, const double* const obs[3], long long n, int n_runs,
                                    double ehT, double emhT, double* tiles, long long n_tiles, int run0,
                                    cudaStream_t s) {
    dim3 grid((unsigned)((n + kTile - 1) / kTile), (unsigned)n_runs);
    exact_estimator_kernel<<<grid, kTile, 0, s>>>(a, obs[0], obs[1], obs[2], n, ehT, emhT, tiles, n_tiles, run0);
    return cudaGetLastError();
}

#ifndef HMC_EXACT_MINB_WIDE
#define HMC_EXACT_MINB_WIDE 8
#endif
#ifndef HMC_EXACT_MINB_DEEP
#define HMC_EXACT_MINB_DEEP 6
#endif
constexpr int kMinBWide = HMC_EXACT_MINB_WIDE, kMinBDeep = HMC_EXACT_MINB_DEEP;

// variant 1: the wide budget (jobs of a few waves), 0: the deep one
cudaError_t exact_plan(long long rows, int sms, int* grid, int* variant) {
    int occ_wide = 0, occ_deep = 0;
    cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_wide, exact_batch_kernel<kMinBWide>,
                                                                    kExactThreads, 0);
    if (err == cudaSuccess)
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_deep, exact_batch_kernel<kMinBDeep>,
                                                            kExactThreads, 0);
    if (err != cudaSuccess) return err;
    const long long wave = (long long)sms * (occ_wide > 0 ? occ_wide : kMinBWide) * kExactThreads;
    *variant = rows > 4 * wave ? 0 : 1;  // deep loops: fewer, fatter threads
    const long long per_sm = *variant == 0 ? (occ_deep > 0 ? occ_deep : kMinBDeep)
                                           : (occ_wide > 0 ? occ_wide : kMinBWide);
    const long long blocks = (rows + kExactThreads - 1) / kExactThreads;
    const long long max_blocks = (long long)sms * per_sm;  // grid-stride: one resident wave
    *grid = (int)(blocks < max_blocks ? blocks : max_blocks);
    return cudaSuccess;
}

cudaError_t launch_exact(const ExactArgs& e, int grid, int variant, cudaStream_t s) {
    if (variant == 0)
        exact_batch_kernel<kMinBDeep><<<grid, kExactThreads, 0, s>>>(e);
    else
        exact_batch_kernel<kMinBWide><<<grid, kExactThreads, 0, s>>>(e);
    return cudaGetLastError();
}

// one Gamma(shape, scale) draw per (key, start draw) -- rng.gamma_batch /
// sample_gamma (rng.py:238-262, 308-343) on the device
__global__ void gamma_kernel(const unsigned long long* __restrict__ keys,
                             const unsigned long long* __restrict__ start, long long n, double shape,
                             double scale, double* __restrict__ out, unsigned long long* __restrict__ used) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned long long u = 0;
    out[i] = sample_gamma_from(keys[i], start[i], shape, scale, &u);
    used[i] = u;
}

cudaError_t launch_gamma(const unsigned long long* d_keys, const unsigned long long* d_start, long long n,
                         double shape, double scale, double* d_out, unsigned long long* d_used, cudaStream_t s) {
    gamma_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(d_keys, d_start, n, shape, scale, d_out, d_used);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// The reference's exact-scheme host modules (bessel.py, ivlaw.py, exact.py)
// as elementwise kernels over the exact kernel's own device routines: the
// Bessel series, the characteristic function, the law's moments, nodes,
// CDF and Newton inversion, and one exact step on given draws.  One thread
// per input; the law's nodes live in a per-thread scratch slice like the
// batch kernel's.  Errors: the batch kernel's codes, max over threads.
// ---------------------------------------------------------------------------
namespace {
__device__ __forceinline__ cplx clog_(cplx a) { return {log(cabs_(a)), atan2(a.im, a.re)}; }
}  // namespace

// bessel.py: mode 0 bessel_i_series, 1 bessel_i, 2 bessel_i_ratio (z =
// coeff_num; aux[4 i ..] = coeff_den, w, log_coeff_ratio re / im, re NaN for
// the principal log of coeff_num / coeff_den)
__global__ void bessel_kernel(int mode, double nu, const double* __restrict__ z, const double* __restrict__ aux,
                              long long n, double* __restrict__ out, int* err) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int e = kErrNone;
    const cplx zz = cx(z[2 * i], z[2 * i + 1]);
    cplx r;
    if (mode == HMC_BESSEL_SERIES) {
        r = bessel_series(nu, zz, &e);
    } else if (mode == HMC_BESSEL_I) {
        const cplx ser = bessel_series(nu, zz, &e);
        if (zz.re == 0.0 && zz.im == 0.0)   // the limits at z = 0 (bessel.py bessel_i)
            r = nu > 0.0 ? cx(0.0) : (nu == 0.0 ? ser / exp(lgamma(nu + 1.0)) : cx(CUDART_INF));
        else
            r = cexp_(nu * clog_(0.5 * zz) - cx(lgamma(nu + 1.0))) * ser;
    } else {
        const double cd = aux[4 * i], w = aux[4 * i + 1];
        const cplx s_num = bessel_series(nu, w * zz, &e);
        const cplx s_den = bessel_series(nu, cx(w * cd), &e);
        const cplx lr = isnan(aux[4 * i + 2]) ? clog_(zz / cd) : cx(aux[4 * i + 2], aux[4 * i + 3]);
        r = (cexp_(nu * lr) * s_num) / s_den;
    }
    out[2 * i] = r.re;
    out[2 * i + 1] = r.im;
    if (e != kErrNone) atomicMax(err, e);
}

cudaError_t launch_bessel(int mode, double nu, const double* d_z, const double* d_aux, long long n, double* d_out,
                          int* d_err, cudaStream_t s) {
    bessel_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(mode, nu, d_z, d_aux, n, d_out, d_err);
    return cudaGetLastError();
}

// ivlaw.py characteristic_fn_raw / _characteristic_fn_vec: Phi(a) at each a
__global__ void ivlaw_phi_kernel(double kappa, double sigma, double dof, double v_u, double v_t, double dt,
                                 const double* __restrict__ a, long long n, double* __restrict__ out, int* err) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int e = kErrNone;
    cplx p = cx(1.0);
    if (a[i] != 0.0) {   // Phi(0) = 1 exactly, no series evaluated
        const PhiPath P = phi_path(kappa, sigma * sigma, 0.5 * dof - 1.0, v_u, v_t, dt);
        p = phi_node(P, a[i], &e);
    }
    out[2 * i] = p.re;
    out[2 * i + 1] = p.im;
    if (e != kErrNone) atomicMax(err, e);
}

cudaError_t launch_ivlaw_phi(double kappa, double sigma, double dof, double v_u, double v_t, double dt,
                             const double* d_a, long long n, double* d_out, int* d_err, cudaStream_t s) {
    ivlaw_phi_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(kappa, sigma, dof, v_u, v_t, dt, d_a, n, d_out,
                                                                 d_err);
    return cudaGetLastError();
}

// ivlaw.py IntegratedVarianceLaw: info[0..3] = mean, std, h, node count
// (thread 0), and per input (mode) cdf_raw(x), cdf(x) or inverse_cdf(u)
__global__ void ivlaw_eval_kernel(int mode, double kappa, double theta, double sigma, double dof, double v_u,
                                  double v_t, double dt, const double* __restrict__ in, long long n,
                                  double* __restrict__ out, double* __restrict__ info, double* scratch,
                                  long long stride, int* err) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (n > 0 ? n : 1)) return;
    int e = kErrNone;
    NodeCache nc{};
    nc.base = scratch + i;
    nc.stride = stride;
    nc.cap = kExactCacheNodes;
    PhiPath P;
    const IvLaw L = iv_law(kappa, theta, sigma, dof, v_u, v_t, dt, P, &e);
    const bool degenerate = L.std < kDegenerateRelStd * L.mean;   // ivlaw.py is_degenerate
    // nodes: for cdf_raw always (the reference evaluates its quadrature even
    // in a degenerate regime), for cdf and the info (the converged node
    // count) outside the degenerate regimes
    const bool want_nodes = e == kErrNone && L.kind != kLawPointMass &&
                            (mode == HMC_IVLAW_CDF_RAW || ((mode == HMC_IVLAW_CDF || mode == HMC_IVLAW_INFO) &&
                                                           !degenerate));
    int n_nodes = 0;
    if (want_nodes) {
        nc.P = &P;
        nc.h = L.h;
        n_nodes = iv_nodes(P, L.h, nc, [](int, double) {}, &e);
    }
    if (i == 0) {
        info[0] = L.mean;
        info[1] = L.std;
        info[2] = L.h;
        info[3] = (double)n_nodes;
    }
    if (n > 0 && e == kErrNone) {
        const double x = in[i];
        double r = 0.0;
        if (mode == HMC_IVLAW_INVERSE) {
            r = sample_iv(kappa, theta, sigma, dof, v_u, v_t, dt, x, nc, &e);
        } else if (mode == HMC_IVLAW_CDF && degenerate) {
            if (L.std == 0.0)
                r = x < L.mean ? 0.0 : 1.0;
            else
                r = x > 0.0 ? 0.5 * erfc(-((x - L.mean) / L.std) / sqrt(2.0)) : 0.0;
        } else if (x > 0.0) {
            r = cdf_at(x, L.h, n_nodes, nc, &e);
            if (mode == HMC_IVLAW_CDF) r = fmin(fmax(r, 0.0), 1.0);
        }
        out[i] = r;
    }
    if (e != kErrNone) atomicMax(err, e);
}

cudaError_t launch_ivlaw_eval(int mode, double kappa, double theta, double sigma, double dof, double v_u,
                              double v_t, double dt, const double* d_in, long long n, double* d_out, double* d_info,
                              double* d_scratch, int* d_err, cudaStream_t s) {
    const long long threads = n > 0 ? n : 1;
    ivlaw_eval_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(
        mode, kappa, theta, sigma, dof, v_u, v_t, dt, d_in, n, d_out, d_info, d_scratch, threads, d_err);
    return cudaGetLastError();
}

// exact.py variance_transition (full = 0) / exact_step (full = 1) on given
// draws [z1, gamma, u_iv, z3] per row: the batch kernel's step arithmetic
__global__ void exact_step_kernel(int full, hmc_model m, double dof, double s_u, double v_u, double dt,
                                  const double* __restrict__ draws, long long n, double* __restrict__ out,
                                  double* scratch, int* err) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int e = kErrNone;
    const double* d = draws + 4 * i;
    const double ek = exp(-m.kappa * dt);
    const double c = m.sigma * m.sigma * (1.0 - ek) / (4.0 * m.kappa);
    const double lam = 4.0 * m.kappa * ek * v_u / (m.sigma * m.sigma * (1.0 - ek));
    const double shifted = d[0] + sqrt(lam);
    const double v_t = c * (d[1] + shifted * shifted);
    double s_t = s_u, iv = 0.0;
    if (full) {
        NodeCache nc{};
        nc.base = scratch + i;
        nc.stride = n;
        nc.cap = kExactCacheNodes;
        iv = sample_iv(m.kappa, m.theta, m.sigma, dof, v_u, v_t, dt, d[2], nc, &e);
        const double int_w2 = m.sigma < 1e-4 * m.kappa ? sqrt(iv) * ndtri_ref(d[2])
                                                       : (v_t - v_u - m.kappa * m.theta * dt + m.kappa * iv) / m.sigma;
        double var_ln = (1.0 - m.rho * m.rho) * iv;
        if (var_ln < 0.0) var_ln = 0.0;
        s_t = exp(log(s_u) + m.r * dt - 0.5 * iv + m.rho * int_w2 + sqrt(var_ln) * d[3]);
    }
    out[3 * i] = s_t;
    out[3 * i + 1] = v_t;
    out[3 * i + 2] = iv;
    if (e != kErrNone) atomicMax(err, e);
}

cudaError_t launch_exact_step(int full, const hmc_model& m, double s_u, double v_u, double dt, const double* d_draws,
                              long long n, double* d_out, double* d_scratch, int* d_err, cudaStream_t s) {
    const double dof = 4.0 * m.kappa * m.theta / (m.sigma * m.sigma);  // model.py:43-45
    exact_step_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(full, m, dof, s_u, v_u, dt, d_draws, n, d_out,
                                                                  d_scratch, d_err);
    return cudaGetLastError();
}

}  // namespace hmc
