"""One Sobol RQMC Asian full-Greeks call (2^22 x 252) for ncu:
python tools/sobol_prof.py [bridge_segments]."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, greeks, daily_fixings
S = int(sys.argv[1]) if len(sys.argv) > 1 else 0
p = HestonParams(**BENCH_PARAMS)
spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 252))
cfg = SimConfig(scheme="milstein", sampler="sobol", sobol_highdim_ack=True, sobol_scramble=True,
                sobol_bridge=S, n_paths=2**22, n_steps=252, n_runs=1, seed=1)
for _ in range(2):
    g = greeks(p, spec, cfg)
torch.cuda.synchronize()
print("ok", g["price"].estimate)
