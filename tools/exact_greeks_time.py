"""Exact-scheme (Broadie-Kaya) full Greeks through the public API, European
and 4-date Asian, CUDA events (dev tool; HMC_LIB_PATH picks the library):
python tools/exact_greeks_time.py [n_paths]."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, greeks
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 17
p = HestonParams(**BENCH_PARAMS)
specs = {"european": OptionSpec("european", "call", 100.0, 1.0, 100.0),
         "asian4": OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=(0.25, 0.5, 0.75, 1.0))}
out = {}
for name, spec in specs.items():
    cfg = SimConfig(scheme="exact", n_paths=n, n_steps=1, n_runs=1, seed=7)
    g = greeks(p, spec, cfg)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g = greeks(p, spec, cfg); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[name] = {"ms": sorted(ts)[2], "est": {q: g[q].estimate for q in ("price", "delta", "rho", "vega", "rho_fd")}}
print(json.dumps({"n_paths": n, **out}))
