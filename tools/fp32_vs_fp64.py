"""fp32 production vs the fp64 replay of the reference stream at the headline
configuration (Asian, 252 daily fixings, full Greeks), pooled over runs:
python tools/fp32_vs_fp64.py [log2_paths_per_run] [runs]."""
import json, math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, daily_fixings, greeks
e = int(sys.argv[1]) if len(sys.argv) > 1 else 24
R = int(sys.argv[2]) if len(sys.argv) > 2 else 16
p = HestonParams(**BENCH_PARAMS)
spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 252))
res = {prec: greeks(p, spec, SimConfig(scheme="milstein", n_paths=2**e, n_steps=252, n_runs=R, seed=2024,
                                       precision=prec)) for prec in ("fp32", "fp64")}
out = {"paths": R * 2**e, "steps": 252, "rows": {}}
for q in res["fp32"]:
    a, b = res["fp32"][q], res["fp64"][q]
    se = math.hypot(a.path_std_error, b.path_std_error)
    out["rows"][q] = {"fp32": a.estimate, "fp64": b.estimate, "diff": a.estimate - b.estimate, "z": (a.estimate - b.estimate) / se,
                      "rel_diff": (a.estimate - b.estimate) / abs(b.estimate), "combined_se": se}
print(json.dumps(out, indent=1))
