"""One exact_batch call (BASELINE params, European, one [0, T] step) for
timing / ncu: python tools/exact_prof.py [n_paths]."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2309_10477_b200 import HestonParams, cuda_backend
from paper_2309_10477_b200.model import BENCH_PARAMS
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 17
p = HestonParams(**BENCH_PARAMS)
for rep in range(2):
    t0 = time.perf_counter()
    out = cuda_backend.exact_batch(p, 100.0, np.array([0.0, 1.0]), np.array([1]), 0, n, 7, None)
    dt = time.perf_counter() - t0
print(n, "paths %.1f ms  %.3f us/path" % (dt * 1e3, dt / n * 1e6))
if len(sys.argv) > 2:   # engine-level greeks (3 kernel passes + reference per-run procedure)
    from paper_2309_10477_b200 import OptionSpec, SimConfig, greeks
    cfg = SimConfig(scheme="exact", n_paths=n, n_steps=1, n_runs=1, seed=7)
    euro = OptionSpec("european", "call", 100.0, 1.0, 100.0)
    for rep in range(3):
        t0 = time.perf_counter()
        g = greeks(p, euro, cfg)
        dt = time.perf_counter() - t0
    print("greeks e2e %.1f ms" % (dt * 1e3), g["price"].estimate, g["vega"].estimate)
