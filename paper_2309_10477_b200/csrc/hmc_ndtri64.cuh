// hmc_ndtri64.cuh -- the reference's fp64 inverse normal CDF on the device,
// shared by every fp64 kernel that replays the reference's stream
// (hmc_replay.cu, hmc_exact.cu).  Include ONLY from translation units built
// with -fmad=false (paper_2309_10477_b200/_build.py): the reference's C build
// has no FMA, and parity to 1e-12 per path relies on the same rounding
// sequence.
#pragma once

#include <cuda_runtime.h>

namespace hmc {

// Acklam rational approximation + one Halley step on erfc
// (_core.pyx:75-109, rng.py:82-132)
static __device__ __noinline__ double ndtri_ref(double u) {
    double q, s, num, den, x, e, corr, p, sign;
    if (u < 1e-300) u = 1e-300;
    if (u > 1.0 - 1e-16) u = 1.0 - 1e-16;
    if (0.02425 <= u && u <= 0.97575) {
        q = u - 0.5;
        s = q * q;
        num = ((((-3.969683028665376e+01 * s + 2.209460984245205e+02) * s
                 - 2.759285104469687e+02) * s + 1.383577518672690e+02) * s
               - 3.066479806614716e+01) * s + 2.506628277459239e+00;
        den = ((((-5.447609879822406e+01 * s + 1.615858368580409e+02) * s
                 - 1.556989798598866e+02) * s + 6.680131188771972e+01) * s
               - 1.328068155288572e+01) * s + 1.0;
        x = q * num / den;
    } else {
        if (u < 0.02425) {
            p = u;
            sign = 1.0;
        } else {
            p = 1.0 - u;
            sign = -1.0;
        }
        q = sqrt(-2.0 * log(p));
        num = ((((-7.784894002430293e-03 * q - 3.223964580411365e-01) * q
                 - 2.400758277161838e+00) * q - 2.549732539343734e+00) * q
               + 4.374664141464968e+00) * q + 2.938163982698783e+00;
        den = (((7.784695709041462e-03 * q + 3.224671290700398e-01) * q
                + 2.445134137142996e+00) * q + 3.754408661907416e+00) * q + 1.0;
        x = sign * num / den;
    }
    e = 0.5 * erfc(-x / sqrt(2.0)) - u;
    corr = e * 2.5066282746310002 * exp(0.5 * x * x);
    x -= corr / (1.0 + 0.5 * x * corr);
    return x;
}

}  // namespace hmc
