"""Independence of per-run estimates on the production stream: correlation
between runs derived from one seed (dev tool)."""
import math, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, price
p = HestonParams(**BENCH_PARAMS); spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
for prec in ("fp32", "fp64"):
    for n_paths, steps in ((2**18, 64), (2**20, 64), (2**16, 252)):
        s = price(p, spec, SimConfig(scheme="milstein", n_paths=n_paths, n_steps=steps, n_runs=64, seed=1, precision=prec))
        exp = s.path_std_error * math.sqrt(64)
        r = np.array(s.per_run_values)
        # lag-1 correlation of run values
        c = np.corrcoef(r[:-1], r[1:])[0, 1]
        print(prec, n_paths, steps, "run sd %.5f expected %.5f ratio %.3f mean %.5f lag1 %.3f" % (s.std_error, exp, s.std_error / exp, s.estimate, c), flush=True)
