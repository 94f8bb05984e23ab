"""Every kernel on small and ragged shapes, for the bounds-checked build
(HMC_LIB_PATH=paper_2309_10477_b200/_variants/libhmc_checked.so; device
asserts on every table / histogram / skeleton / cache index, see
csrc/hmc_device.cuh HMC_DCHECK).  A failed check aborts the kernel and the
call raises; every result must also be finite.  Prints one line per group
and "checked suite ok" at the end (tests/test_gpu_checked.py)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from paper_2309_10477_b200 import (BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, cuda_backend,
                                   daily_fixings, greeks, price, surface)

p = HestonParams(**BENCH_PARAMS)
n_calls = 0


def finite(x, what):
    global n_calls
    n_calls += 1
    arr = np.asarray(x, dtype=np.float64)
    if not np.all(np.isfinite(arr)):
        raise SystemExit(f"non-finite result: {what}")


def specs(n_steps):
    out = [OptionSpec("european", "call", 100.0, 1.0, 100.0),
           OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, n_steps))]
    if n_steps >= 4:
        k = [max(1, n_steps // 4), max(2, n_steps // 2), n_steps]
        out.append(OptionSpec("asian_arithmetic", "call", 95.0, 1.0, 100.0,
                              averaging_times=tuple(sorted({i / n_steps for i in k}))))
    return out


# backend seam (fp64 replay of the reference stream; given uniforms)
rng = np.random.default_rng(0)
for n_steps, lo, hi in ((1, 0, 1), (3, 5, 133), (7, 0, 300), (20, 127, 16513)):
    finite(cuda_backend.discretised_batch(p, 100.0, 1.0, n_steps, True, lo, hi, 12345, None,
                                          np.array([n_steps])), "discretised_batch")
    u = rng.random((hi - lo, 2 * n_steps))
    finite(cuda_backend.discretised_batch(p, 100.0, 1.0, n_steps, False, lo, hi, 7, u,
                                          np.arange(1, n_steps + 1)), "discretised_batch uniforms")
print("backend ok", flush=True)

# single-product engine: precision x sampler x bridge x product x ragged sizes
for n_steps in (1, 2, 7, 65, 130):
    for spec in specs(n_steps):
        for n_paths, n_runs in ((1, 1), (129, 2), (16385, 3)):
            for prec in ("fp32", "fp64"):
                samplers = [("pseudo", False, 0), ("sobol", False, 0), ("sobol", True, 0)]
                if n_steps >= 2:
                    samplers += [("sobol", True, 1), ("sobol", True, min(5, n_steps)), ("sobol", False, min(16, n_steps))]
                for sampler, scr, S in samplers:
                    cfg = SimConfig(scheme="milstein" if n_steps % 2 else "euler", sampler=sampler,
                                    sobol_highdim_ack=True, sobol_scramble=scr, sobol_bridge=S,
                                    n_paths=n_paths, n_steps=n_steps, n_runs=n_runs, seed=3, precision=prec)
                    g = greeks(p, spec, cfg)
                    finite([v.estimate for v in g.values()], f"greeks {n_steps} {spec.style} {n_paths} {prec} {sampler} {S}")
                    finite(price(p, spec, cfg).estimate, "price")
    print("engine ok", n_steps, flush=True)

# surfaces: uniform and irregular strike grids, one to many maturities
for strikes, mats, n_steps in (([100.0], [1.0], 8),
                               (np.arange(70.0, 134.0, 1.0), [0.25 * i for i in range(1, 9)], 64),
                               ([80.0, 93.5, 100.0, 101.0, 140.0], [0.5, 1.0], 20),
                               (np.linspace(50.0, 160.0, 128), [1.0 / 16 * i for i in range(1, 17)], 32)):
    for sampler in ("pseudo", "sobol"):
        for n_paths in (1, 1500, 20000):
            cfg = SimConfig(scheme="milstein", sampler=sampler, sobol_highdim_ack=True, sobol_scramble=True,
                            n_paths=n_paths, n_steps=n_steps, n_runs=2, seed=5)
            res = surface(p, strikes, mats, cfg)
            for style in res.estimate.values():
                for arr in style.values():
                    finite(arr, "surface")
print("surface ok", flush=True)

# Broadie-Kaya exact scheme (pseudo and Sobol, European and Asian)
for spec in (OptionSpec("european", "call", 100.0, 1.0, 100.0),
             OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=(0.25, 0.5, 1.0))):
    for sampler in ("pseudo", "sobol"):
        for n_paths in (1, 300, 16390):
            cfg = SimConfig(scheme="exact", sampler=sampler, n_paths=n_paths, n_steps=1, n_runs=2, seed=9)
            finite([v.estimate for v in greeks(p, spec, cfg).values()], "exact greeks")
finite(cuda_backend.exact_batch(p, 100.0, np.array([0.0, 0.5, 1.0]), np.array([1, 1]), 3, 2000, 11, None),
       "exact_batch")
# the exact scheme's host modules (bessel / ivlaw / exact step) on the device
from paper_2309_10477_b200 import bessel, exact, ivlaw, rng
finite([abs(bessel.bessel_i(nu, z)) for nu in (-0.37, 0.0, 1.5) for z in (0.5 + 1j, 20.0 + 0j, 45 - 3j)], "bessel_i")
finite(np.abs(bessel.bessel_i_series_vec(-0.37, np.array([0.1 + 0j, 3 - 2j, 40 + 10j]))), "bessel series")
finite(abs(bessel.bessel_i_ratio(-0.37, 2 + 1.5j, 2.4, 0.8)), "bessel ratio")
for v_u, v_t, dt in ((0.010201, 0.010201, 1.0), (0.04, 0.01, 0.25), (0.0, 0.02, 1.0 / 252)):
    law = ivlaw.IntegratedVarianceLaw(p, v_u, v_t, dt)
    finite([law.mean, law.std, law.cdf(law.mean), law.cdf_raw(0.5 * law.mean), law.inverse_cdf(0.3)], "ivlaw")
    finite(np.abs(ivlaw._characteristic_fn_vec(p, v_u, v_t, dt, np.array([0.0, 0.3, 30.0, 3000.0]))), "phi")
st = rng.UniformStream(seed=4)
res = exact.exact_step(st, p, 100.0, 0.010201, 1.0, gamma_stream=rng.UniformStream(seed=4, stream_index=1))
finite([res.s_t, res.v_t, res.integrated_variance], "exact_step")
finite(exact.variance_transition(rng.UniformStream(seed=5), p, 0.02, 0.5), "variance_transition")
print("exact ok", flush=True)
print(f"checked suite ok ({n_calls} checked calls)")
