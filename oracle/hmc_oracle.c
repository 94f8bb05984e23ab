/*
 * oracle/hmc_oracle.c -- CPU restatement of the reference's discretised
 * Heston path kernel, used ONLY AS TEST INFRASTRUCTURE.
 *
 *   This file is the checker, never the product.  Only tests/,
 *   __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 *   leg may load it.  The shipped engine (paper_2309_10477_b200) never links
 *   or calls it; it fails loudly when its CUDA library is missing.
 *
 * What it restates (reference = /root/reference/pkg/src/hestonmc):
 *   - SplitMix64 counter RNG        _core.pyx:57-68, rng.py:38-65
 *   - Acklam + one Halley step       _core.pyx:75-109, rng.py:82-132
 *   - Euler / Milstein full-truncation path loop with Asian accumulation
 *                                    _core.pyx:354-412, _batch_py.py:36-81
 *   - per-path payoff / pathwise Delta / pathwise Rho
 *                                    engine.py:47-68, products.py:23-51
 *   - Gamma / Vega / FD-Rho by re-simulating bumped inputs under common
 *     random numbers, the reference's own finite-difference method
 *                                    tests/test_products.py:101-137,
 *                                    SPEC.md:294
 *
 * Parity pin: compiled with gcc -O2 -ffp-contract=off against the same glibc
 * libm as the reference's _core, so discretised_batch is bit-identical to
 * the reference (checked against tests/golden/ fixtures produced by the
 * reference itself, tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL     /* _core.pyx:31 */
#define ROOT_SALT 0x8CB92BA72F3D8DD7ULL  /* _core.pyx:32, rng.py:27 */
#define INDEX_SALT 0xD1B54A32D192ED03ULL /* _core.pyx:33, rng.py:28 */
static const double INV53 = 1.0 / 9007199254740992.0; /* _core.pyx:34 */

typedef struct {
    double kappa, theta, sigma, rho, r, v0;
} hmo_params;

typedef struct {
    int is_asian;
    int is_call;
    double strike, maturity, spot;
} hmo_product;

typedef struct {
    double h_spot; /* absolute S0 bump            (test_products.py:105) */
    double v0_up;  /* v0 of the up-bumped variance trajectory          */
    double v0_dn;  /* v0 of the down-bumped variance trajectory        */
    double h_r;    /* absolute r bump             (test_products.py:118) */
} hmo_bumps;

/* ---- RNG: SplitMix64 (rng.py:38-65, _core.pyx:57-68) -------------------- */

uint64_t hmo_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t hmo_root_key(uint64_t seed) { return hmo_mix64(seed ^ ROOT_SALT); } /* rng.py:46-47 */

uint64_t hmo_derive(uint64_t parent, uint64_t index) { /* rng.py:50-52 */
    return hmo_mix64(parent ^ hmo_mix64(index + INDEX_SALT));
}

double hmo_uniform_at(uint64_t key, uint64_t i) { /* rng.py:63-65 */
    return (double)(hmo_mix64(key + (i + 1) * GOLDEN) >> 11) * INV53;
}

void hmo_uniforms_vec(uint64_t key, uint64_t start, int64_t count, double* out) {
    for (int64_t i = 0; i < count; ++i) out[i] = hmo_uniform_at(key, start + (uint64_t)i);
}

/* ---- inverse normal CDF: Acklam + one Halley step (_core.pyx:75-109) ----- */

double hmo_ndtri(double u) {
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

void hmo_ndtri_vec(const double* u, double* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = hmo_ndtri(u[i]);
}

/* ---- one path (_core.pyx:384-411) --------------------------------------- */

typedef struct {
    double s_T, avg, tw;
} hmo_obs;

/* zrow (optional): the step normals themselves, (z1, z2) per step with z2
 * already correlated -- for samplers that build normals some other way
 * (oracle/bridge.py: Sobol Brownian-bridge ordering) */
static hmo_obs simulate_one(const hmo_params* p, double s0, double v0, double r,
                            double T, int n_steps, int milstein, uint64_t main_key,
                            const double* urow, const double* zrow,
                            const unsigned char* is_avg, int64_t n_dates) {
    const double kappa = p->kappa, theta = p->theta, sigma = p->sigma, rho = p->rho;
    const double dt = T / n_steps;
    const double sq1mr2 = sqrt(1.0 - rho * rho);
    double s = s0, v = v0, price_sum = 0.0, tw_sum = 0.0;
    for (int k = 1; k <= n_steps; ++k) {
        double u1 = 0.0, u2 = 0.0;
        if (zrow) {
        } else if (urow) {
            u1 = urow[2 * (k - 1)];
            u2 = urow[2 * (k - 1) + 1];
        } else {
            u1 = hmo_uniform_at(main_key, (uint64_t)(2 * (k - 1)));
            u2 = hmo_uniform_at(main_key, (uint64_t)(2 * (k - 1) + 1));
        }
        double z1, z2;
        if (zrow) {
            z1 = zrow[2 * (k - 1)];
            z2 = zrow[2 * (k - 1) + 1];
        } else {
            z1 = hmo_ndtri(u1);
            z2 = rho * z1 + sq1mr2 * hmo_ndtri(u2);
        }
        double sqv = sqrt(v * dt);
        s = s * exp((r - 0.5 * v) * dt + sqv * z1);
        double v_new = v + kappa * (theta - v) * dt + sigma * sqv * z2;
        if (milstein) v_new = v_new + 0.25 * sigma * sigma * dt * (z2 * z2 - 1.0);
        v = v_new > 0.0 ? v_new : 0.0;
        if (is_avg[k]) {
            double t_k = k * T / n_steps;
            price_sum += s;
            tw_sum += s * t_k;
        }
    }
    hmo_obs o = {s, price_sum / n_dates, tw_sum / n_dates};
    return o;
}

static unsigned char* avg_mask(int n_steps, const int64_t* avg_idx, int64_t n_avg) {
    unsigned char* m = (unsigned char*)calloc((size_t)n_steps + 1, 1);
    for (int64_t i = 0; i < n_avg; ++i) m[avg_idx[i]] = 1;
    return m;
}

/* Reference backend entry discretised_batch (_core.pyx:354-412): out is
 * (path_hi - path_lo, 3) row-major [s_T, avg, tw_sum]. uniforms, when not
 * NULL, is (path_hi - path_lo, 2*n_steps) row-major. */
int hmo_discretised_batch(const hmo_params* p, double s0, double T, int n_steps,
                          int milstein, int64_t path_lo, int64_t path_hi,
                          uint64_t key_run, const double* uniforms,
                          const int64_t* avg_idx, int64_t n_avg, double* out) {
    unsigned char* m = avg_mask(n_steps, avg_idx, n_avg);
    if (!m) return 1;
    for (int64_t i = 0; i < path_hi - path_lo; ++i) {
        uint64_t main_key = hmo_derive(hmo_derive(key_run, (uint64_t)(path_lo + i)), 0);
        const double* urow = uniforms ? uniforms + (size_t)i * 2 * n_steps : NULL;
        hmo_obs o = simulate_one(p, s0, p->v0, p->r, T, n_steps, milstein, main_key,
                                 urow, NULL, m, n_avg);
        out[3 * i + 0] = o.s_T;
        out[3 * i + 1] = o.avg;
        out[3 * i + 2] = o.tw;
    }
    free(m);
    return 0;
}

/* ---- per-path estimators (engine.py:47-68, products.py:23-51) ----------- */

static double disc_payoff(const hmo_product* pr, double a, double disc) {
    return pr->is_call ? disc * fmax(a - pr->strike, 0.0) : disc * fmax(pr->strike - a, 0.0);
}

static double underlying(const hmo_product* pr, hmo_obs o) { return pr->is_asian ? o.avg : o.s_T; }

static double pw_delta(const hmo_product* pr, hmo_obs o, double disc, double spot) {
    double a = underlying(pr, o);
    return a > pr->strike ? disc * a / spot : 0.0;
}

static double pw_rho(const hmo_product* pr, hmo_obs o, double disc) {
    double a = underlying(pr, o);
    if (!(a > pr->strike)) return 0.0;
    if (pr->is_asian) return disc * (o.tw - pr->maturity * (a - pr->strike));
    return disc * pr->strike * pr->maturity;
}

/* Per-path quantities, out is (n, 7) row-major:
 *   0 price   discounted payoff                          engine.py:53-56
 *   1 delta   pathwise                                   engine.py:58-59
 *   2 rho     pathwise                                   engine.py:60-67
 *   3 gamma   central FD of pathwise delta, S0 +/- h
 *   4 vega    central FD of price in v0 (CRN)            (new; north_star)
 *   5 delta_fd  central FD of price, S0 +/- h            test_products.py:101-112
 *   6 rho_fd    central FD of price, r +/- h             test_products.py:114-125
 * Every bumped value is a full re-simulation with the same uniforms (common
 * random numbers), exactly as the reference's FD tests do.  With
 * want_greeks == 0 only column 0 is filled (the rest are 0). */
static int greeks_impl(const hmo_params* p, const hmo_product* pr, int n_steps, int milstein,
                       int64_t path_lo, int64_t path_hi, uint64_t key_run,
                       const double* uniforms, const double* normals, const int64_t* avg_idx,
                       int64_t n_avg, const hmo_bumps* b, int want_greeks, double* out) {
    unsigned char* m = avg_mask(n_steps, avg_idx, n_avg);
    if (!m) return 1;
    const double T = pr->maturity, S0 = pr->spot, r = p->r;
    const double disc = exp(-r * T);
    for (int64_t i = 0; i < path_hi - path_lo; ++i) {
        uint64_t key = hmo_derive(hmo_derive(key_run, (uint64_t)(path_lo + i)), 0);
        const double* urow = uniforms ? uniforms + (size_t)i * 2 * n_steps : NULL;
        const double* zrow = normals ? normals + (size_t)i * 2 * n_steps : NULL;
        double* o = out + 7 * i;
        memset(o, 0, 7 * sizeof(double));
        hmo_obs base = simulate_one(p, S0, p->v0, r, T, n_steps, milstein, key, urow, zrow, m, n_avg);
        o[0] = disc_payoff(pr, underlying(pr, base), disc);
        if (!want_greeks) continue;
        o[1] = pw_delta(pr, base, disc, S0);
        o[2] = pw_rho(pr, base, disc);
        const double h = b->h_spot;
        hmo_obs su = simulate_one(p, S0 + h, p->v0, r, T, n_steps, milstein, key, urow, zrow, m, n_avg);
        hmo_obs sd = simulate_one(p, S0 - h, p->v0, r, T, n_steps, milstein, key, urow, zrow, m, n_avg);
        o[3] = (pw_delta(pr, su, disc, S0 + h) - pw_delta(pr, sd, disc, S0 - h)) / (2.0 * h);
        o[5] = (disc_payoff(pr, underlying(pr, su), disc) -
                disc_payoff(pr, underlying(pr, sd), disc)) / (2.0 * h);
        hmo_obs vu = simulate_one(p, S0, b->v0_up, r, T, n_steps, milstein, key, urow, zrow, m, n_avg);
        hmo_obs vd = simulate_one(p, S0, b->v0_dn, r, T, n_steps, milstein, key, urow, zrow, m, n_avg);
        o[4] = (disc_payoff(pr, underlying(pr, vu), disc) -
                disc_payoff(pr, underlying(pr, vd), disc)) / (b->v0_up - b->v0_dn);
        const double hr = b->h_r;
        hmo_obs ru = simulate_one(p, S0, p->v0, r + hr, T, n_steps, milstein, key, urow, zrow, m, n_avg);
        hmo_obs rd = simulate_one(p, S0, p->v0, r - hr, T, n_steps, milstein, key, urow, zrow, m, n_avg);
        o[6] = (disc_payoff(pr, underlying(pr, ru), exp(-(r + hr) * T)) -
                disc_payoff(pr, underlying(pr, rd), exp(-(r - hr) * T))) / (2.0 * hr);
    }
    free(m);
    return 0;
}

int hmo_greeks_paths(const hmo_params* p, const hmo_product* pr, int n_steps, int milstein,
                     int64_t path_lo, int64_t path_hi, uint64_t key_run,
                     const double* uniforms, const int64_t* avg_idx, int64_t n_avg,
                     const hmo_bumps* b, int want_greeks, double* out) {
    return greeks_impl(p, pr, n_steps, milstein, path_lo, path_hi, key_run, uniforms, NULL,
                       avg_idx, n_avg, b, want_greeks, out);
}

/* same, driven by given step normals (n, 2*n_steps) row-major [z1, z2] */
int hmo_greeks_paths_z(const hmo_params* p, const hmo_product* pr, int n_steps, int milstein,
                       int64_t n, const double* normals, const int64_t* avg_idx, int64_t n_avg,
                       const hmo_bumps* b, int want_greeks, double* out) {
    return greeks_impl(p, pr, n_steps, milstein, 0, n, 0, NULL, normals, avg_idx, n_avg, b,
                       want_greeks, out);
}

int hmo_abi_version(void) { return 1; }
