"""fp32 production estimates over many seeds vs the semi-analytic price:
z-score distribution (bias check, dev tool)."""
import math, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, price
from oracle.semi_analytic import call_price
p = HestonParams(**BENCH_PARAMS); spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
sa = call_price(100, 100, 1, p.r, p.kappa, p.theta, p.sigma, p.rho, p.v0)
for prec in ("fp32", "fp64"):
    zs = []
    for seed in range(0, 32):
        s = price(p, spec, SimConfig(scheme="milstein", n_paths=2**22, n_steps=252, n_runs=1, seed=seed, precision=prec))
        zs.append((s.estimate - sa) / s.path_std_error)
    zs = np.array(zs)
    print(prec, "z mean %.3f sd %.3f min %.2f max %.2f" % (zs.mean(), zs.std(ddof=1), zs.min(), zs.max()), np.round(zs, 2).tolist(), flush=True)
# high-precision fp32 vs fp64 at 64 steps
res = {}
for prec in ("fp32", "fp64"):
    s = price(p, spec, SimConfig(scheme="milstein", n_paths=2**24, n_steps=64, n_runs=16, seed=123, precision=prec))
    res[prec] = (s.estimate, s.path_std_error)
d = res["fp32"][0] - res["fp64"][0]
print("fp32-fp64 @2^28x64: %.6f +- %.6f z=%.2f" % (d, math.hypot(res["fp32"][1], res["fp64"][1]), d / math.hypot(res["fp32"][1], res["fp64"][1])), res)
