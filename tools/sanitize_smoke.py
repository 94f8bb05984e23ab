"""Small invocation of every kernel (for compute-sanitizer memcheck)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2309_10477_b200 import (BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, cuda_backend,
                                   daily_fixings, greeks, price, surface)
p = HestonParams(**BENCH_PARAMS)
euro = OptionSpec("european", "call", 100.0, 1.0, 100.0)
asian = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 20))
sparse = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=(0.25, 0.5, 1.0))
print(cuda_backend.discretised_batch(p, 100.0, 1.0, 20, True, 3, 300, 12345, None, np.array([5, 20])).sum())
print(cuda_backend.discretised_batch(p, 100.0, 1.0, 4, True, 0, 37, 1, np.random.default_rng(0).random((37, 8)), np.array([4])).sum())
for spec in (euro, asian, sparse):
    for prec in ("fp32", "fp64"):
        for sampler in ("pseudo", "sobol"):
            kw = dict(scheme="milstein", sampler=sampler, sobol_highdim_ack=True, n_paths=16500, n_steps=20,
                      n_runs=2, seed=3, precision=prec)
            print(spec.style, prec, sampler, greeks(p, spec, SimConfig(**kw))["price"].estimate,
                  price(p, spec, SimConfig(**kw)).estimate)
res = surface(p, [90.0, 100.0, 110.0, 125.0], [0.5, 1.0], SimConfig(scheme="milstein", n_paths=3000, n_steps=20, n_runs=2))
print(res.estimate["european"]["price"])
res = surface(p, [90.0, 97.0, 100.0], [0.25, 1.0], SimConfig(scheme="euler", n_paths=1500, n_steps=20, n_runs=1))
print(res.estimate["asian_arithmetic"]["vega"])
