import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, greeks, price, daily_fixings
p = HestonParams(**BENCH_PARAMS)
spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 252))
for sampler in ("pseudo", "sobol"):
    cfg = SimConfig(scheme="milstein", sampler=sampler, sobol_highdim_ack=True, n_paths=2**22, n_steps=252, n_runs=1, seed=1)
    greeks(p, spec, cfg)
    torch.cuda.synchronize(); t = time.perf_counter()
    g = greeks(p, spec, cfg)
    print(sampler, "%.2f ms" % ((time.perf_counter() - t) * 1e3), g["price"].estimate, g["price"].path_std_error)
