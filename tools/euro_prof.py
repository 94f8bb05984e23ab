"""One European full-Greeks call (BASELINE config 2: 2^22 x 252, Philox) for
timing / ncu: python tools/euro_prof.py [n_paths]."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, greeks
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 22
p = HestonParams(**BENCH_PARAMS)
spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
cfg = SimConfig(scheme="milstein", n_paths=n, n_steps=252, n_runs=1, seed=7)
g = greeks(p, spec, cfg)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g = greeks(p, spec, cfg); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("european", n, "paths: %.3f ms" % min(ts), g["price"].estimate)
