"""Seed sweep of the reference test test_engine.py::test_se_scaling_one_over_sqrt_n
(SE ratio of 8000- vs 2000-path runs, 30 runs, 64 steps; bound 0.35..0.65) on
the fp32 Philox stream and the reference's own stream (precision fp64)."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2309_10477_b200 import *
p = HestonParams(**DEFAULT_PARAMS)
euro = OptionSpec("european", "call", 100.0, 1.0, 100.0)
def cfg(**kw):
    base = dict(scheme="milstein", sampler="pseudo", n_paths=8192, n_steps=32, n_runs=3, seed=42); base.update(kw); return SimConfig(**base)
for prec in ("fp32", "fp64"):
    rs = []
    for seed in range(40):
        small = price(p, euro, cfg(n_paths=2000, n_steps=64, n_runs=30, seed=seed, precision=prec))
        large = price(p, euro, cfg(n_paths=8000, n_steps=64, n_runs=30, seed=seed, precision=prec))
        rs.append(large.std_error / small.std_error)
    rs = np.array(rs)
    print(prec, "seeds 0..39: mean", rs.mean(), "sd", rs.std(), "min", rs.min(), "max", rs.max(), "frac_fail", np.mean((rs < 0.35) | (rs > 0.65)))
    print(np.round(rs, 3).tolist())
s42 = [price(p, euro, cfg(n_paths=n, n_steps=64, n_runs=30, seed=42, precision=pr)).std_error for pr in ("fp32","fp64") for n in (2000, 8000)]
print("seed 42 fp32 small/large, fp64 small/large", s42)
# per-path SE consistency
s = price(p, euro, cfg(n_paths=2000, n_steps=64, n_runs=30, seed=42))
print("path SE * sqrt(runs)", s.path_std_error*np.sqrt(30), "run SD", s.std_error)
s = price(p, euro, cfg(n_paths=8000, n_steps=64, n_runs=30, seed=42))
print("path SE * sqrt(runs)", s.path_std_error*np.sqrt(30), "run SD", s.std_error)
