"""Per-path fp32 production arithmetic vs the fp64 oracle on identical
normals (hmc_fp32_paths_check): max / mean absolute differences per column."""
import ctypes, json, math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import oracle
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, _lib, daily_fixings, engine
p = HestonParams(**BENCH_PARAMS)
out = {}
K = float(sys.argv[1]) if len(sys.argv) > 1 else 100.0
for name, spec in (("european", OptionSpec("european", "call", K, 1.0, 100.0)),
                   ("asian_daily", OptionSpec("asian_arithmetic", "call", K, 1.0, 100.0,
                                              averaging_times=daily_fixings(1.0, 252)))):
    cfg = SimConfig(scheme="milstein", n_paths=16384, n_steps=252, n_runs=1, seed=1)
    job = engine.Job(p, spec, cfg, True)
    n, n_sim = 16384, int(job.avg_idx[-1])
    z = np.random.default_rng(3).standard_normal((n, n_sim, 2)).astype(np.float32)
    got = np.empty((n, 7))
    _lib.check(_lib.lib().hmc_fp32_paths_check(ctypes.byref(job.model), ctypes.byref(job.product),
                                               ctypes.byref(job.sim), z.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                               n, got.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 0))
    zz = np.zeros((n, 504))
    zz[:, 0::2] = z[:, :, 0]
    zz[:, 1::2] = p.rho * z[:, :, 0].astype(np.float64) + math.sqrt(1 - p.rho ** 2) * z[:, :, 1]
    ref = oracle.greeks_paths_z(p, spec, 252, True, zz, job.avg_idx, engine.bump_sizes(p, spec, cfg))
    d = np.abs(got - ref)
    out[name] = {q: {"max_abs": float(d[:, i].max()), "median_abs": float(np.median(d[:, i])),
                     "mean_got": float(got[:, i].mean()), "mean_ref": float(ref[:, i].mean())}
                 for i, q in enumerate(oracle.QUANTITIES)}
print(json.dumps(out, indent=1))
