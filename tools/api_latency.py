"""Host-side latency of the public API (greeks()) for small and large jobs, with a
cProfile of the Python layer (dev tool; run on the GPU box)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, greeks, price
p = HestonParams(**BENCH_PARAMS); spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
from paper_2309_10477_b200 import daily_fixings
asian = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 252))
for n, steps, runs in ((1024, 8, 1), (32000, 128, 30), (2**20, 252, 1)):
    cfg = SimConfig(scheme="milstein", n_paths=n, n_steps=steps, n_runs=runs, seed=1)
    for _ in range(3): greeks(p, spec, cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); greeks(p, spec, cfg); ts.append(time.perf_counter() - t0)
    ts.sort()
    print(n, steps, runs, "median %.1f us  min %.1f us" % (ts[10] * 1e6, ts[0] * 1e6))
import cProfile, pstats
cfg = SimConfig(scheme="milstein", n_paths=16384, n_steps=252, n_runs=1, seed=1)
for _ in range(3): greeks(p, asian, cfg)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    t0 = time.perf_counter(); greeks(p, asian, cfg); ts.append(time.perf_counter() - t0)
ts.sort(); print("asian 16384 x 252 daily fixings: median %.1f us" % (ts[10] * 1e6))
pr = cProfile.Profile(); pr.enable()
for _ in range(200): greeks(p, asian, cfg)
pr.disable(); pstats.Stats(pr).sort_stats("cumtime").print_stats(15)
