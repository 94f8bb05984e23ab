"""Diagnostic: fp32 production path vs fp64 replay (reference stream) and the
semi-analytic price, pooled over seeds (dev tool)."""
import json, math, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, price, greeks
from oracle.semi_analytic import call_price

p = HestonParams(**BENCH_PARAMS)
spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
sa = call_price(100, 100, 1, p.r, p.kappa, p.theta, p.sigma, p.rho, p.v0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2**22
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 252
res = {"semi_analytic": sa}
for prec in ("fp32", "fp64"):
    for scheme in ("milstein", "euler"):
        ests, ses = [], []
        t0 = time.time()
        for seed in range(1, 5):
            s = price(p, spec, SimConfig(scheme=scheme, n_paths=n, n_steps=steps, n_runs=1, seed=seed, precision=prec))
            ests.append(s.estimate); ses.append(s.path_std_error)
        m = sum(ests) / 4; se = math.sqrt(sum(x * x for x in ses)) / 4
        res[f"{prec}_{scheme}"] = {"mean": m, "se": se, "z_vs_sa": (m - sa) / se, "runs": ests, "sec": time.time() - t0}
        print(prec, scheme, m, se, (m - sa) / se, f"{time.time()-t0:.1f}s", flush=True)
print(json.dumps(res))
