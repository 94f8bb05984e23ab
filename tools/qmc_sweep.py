"""BASELINE config 4: error-vs-N of randomised Sobol QMC vs pseudo-random MC
for European and Asian (daily fixings) full Greeks, 2^20 .. 2^26 points,
R independent replications each (digital shifts for QMC, seeds for MC)."""
import json, math, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, greeks, daily_fixings

p = HestonParams(**BENCH_PARAMS)
specs = {"euro": OptionSpec("european", "call", 100.0, 1.0, 100.0),
         "asian": OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                             averaging_times=daily_fixings(1.0, 252))}
R = int(os.environ.get("QMC_R", "16"))
lo, hi = int(os.environ.get("QMC_LO", "20")), int(os.environ.get("QMC_HI", "26"))
out = {"runs": R, "steps": 252, "params": BENCH_PARAMS, "rows": []}
for name, spec in specs.items():
    for e in range(lo, hi + 1):
        for sampler, S in (("pseudo", 0), ("sobol", 0), ("sobol", 16)):
            cfg = SimConfig(scheme="milstein", sampler=sampler, sobol_highdim_ack=True, sobol_scramble=True,
                            sobol_bridge=S, n_paths=2 ** e, n_steps=252, n_runs=R, seed=2024)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            g = greeks(p, spec, cfg)
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
            row = {"product": name, "log2_n": e, "sampler": sampler + ("+bridge16" if S else ""),
                   "seconds": dt,
                   "path_steps_per_s": R * 2 ** e * 252 / dt}
            for q in ("price", "delta", "gamma", "vega", "rho"):
                row[q] = [g[q].estimate, g[q].std_error / math.sqrt(R)]
            out["rows"].append(row)
            print(json.dumps(row), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "qmc_sweep.json"), "w") as f:
    json.dump(out, f, indent=1)
