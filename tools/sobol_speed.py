"""Device time of one 2^22 x 252 Asian full-Greeks call per sampler
(pseudo, time-ordered RQMC Sobol, bridge-ordered RQMC Sobol); CUDA events,
median of 7."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, greeks, daily_fixings
p = HestonParams(**BENCH_PARAMS)
specs = {"asian": OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                             averaging_times=daily_fixings(1.0, 252)),
         "euro": OptionSpec("european", "call", 100.0, 1.0, 100.0)}
for name, spec in specs.items():
    for sampler, S in (("pseudo", 0), ("sobol", 0), ("sobol", 16), ("sobol", 64)):
        cfg = SimConfig(scheme="milstein", sampler=sampler, sobol_highdim_ack=True, sobol_scramble=sampler == "sobol",
                        sobol_bridge=S, n_paths=2**22, n_steps=252, n_runs=1, seed=1)
        greeks(p, spec, cfg)
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g = greeks(p, spec, cfg); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(name, sampler, S, "%.2f ms" % sorted(ts)[3], g["price"].estimate, g["price"].path_std_error, flush=True)
