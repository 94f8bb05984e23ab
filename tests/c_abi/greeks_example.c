/* Plain-C host of libhmc.so (include/hmc.h): the INTEGRATION.md example.
 * Prints one line per quantity: name mean path_se.
 * cc -I include tests/c_abi/greeks_example.c -L paper_2309_10477_b200 -lhmc -Wl,-rpath,... */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "hmc.h"

int main(int argc, char** argv) {
    const int64_t n_paths = argc > 1 ? atoll(argv[1]) : (1 << 20);
    hmc_model m = {2.0, 0.04, 0.3, -0.7, 0.03, 0.04};
    int64_t idx[252];
    for (int k = 0; k < 252; ++k) idx[k] = k + 1;
    hmc_product p = {HMC_STYLE_ASIAN, HMC_CALL, 100.0, 1.0, 100.0, idx, 252};
    hmc_sim s = {0};
    s.scheme = HMC_SCHEME_MILSTEIN;
    s.sampler = HMC_SAMPLER_PSEUDO;
    s.precision = HMC_PREC_FP32;
    s.want_greeks = 1;
    s.n_steps = 252;
    s.n_runs = 1;
    s.n_paths = n_paths;
    s.seed = 42;
    s.h_spot = 0.5;
    s.v0_up = 0.0404;
    s.v0_dn = 0.0396;
    s.h_r = 1e-4;
    double out[HMC_NW];
    if (hmc_greeks(&m, &p, &s, out, 0) != HMC_OK) {
        fprintf(stderr, "hmc_greeks: %s\n", hmc_last_error());
        return 1;
    }
    static const char* names[HMC_NQ] = {"price", "delta", "rho", "gamma", "vega", "delta_fd", "rho_fd"};
    for (int q = 0; q < HMC_NQ; ++q) {
        const double mean = out[2 * q] / n_paths;
        const double var = (out[2 * q + 1] - out[2 * q] * mean) / (n_paths - 1);
        printf("%s %.17g %.6g\n", names[q], mean, sqrt(var > 0 ? var / n_paths : 0));
    }
    /* the same job dealt over three slices (one GPU here, three streams):
       bit-identical sums */
    const int32_t devs[3] = {0, 0, 0};
    double multi[HMC_NW];
    if (hmc_greeks_multi(&m, &p, &s, multi, devs, 3) != HMC_OK) {
        fprintf(stderr, "hmc_greeks_multi: %s\n", hmc_last_error());
        return 1;
    }
    int same = 1;
    for (int w = 0; w < HMC_NW; ++w) same &= multi[w] == out[w];
    printf("multi_bit_identical %d\n", same);
    /* a usage error never touches the device */
    p.right = HMC_PUT;
    int rc = hmc_greeks(&m, &p, &s, out, 0);
    printf("put_greeks_rc %d %s\n", rc, hmc_last_error());
    return 0;
}
