"""The backend-plugin seam (INTEGRATION.md level 2): the reference engine's
orchestration (oracle.engine, a line-by-line restatement of engine.py,
4096-path jobs on a thread pool) driven through cuda_backend.discretised_batch
vs the reference's own compiled kernel, same workload:
European, 252 steps, price + pathwise Greeks, 2^18 paths, 1 run."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import json
import numpy as np
from oracle import engine as oe
import oracle
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, cuda_backend

p = HestonParams(**BENCH_PARAMS)
spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 18
cfg = SimConfig(scheme="milstein", n_paths=n, n_steps=252, n_runs=1, seed=42)
workers = os.cpu_count() or 1
out = {"paths": n, "steps": 252, "workers": workers}
orig = oe._kernel
try:
    oe._kernel = lambda kind: cuda_backend.discretised_batch
    oe.per_run_values(p, spec, SimConfig(scheme="milstein", n_paths=8192, n_steps=252, n_runs=1), True, "port", workers)
    for w in (1, 8, workers):
        t0 = time.perf_counter()
        gpu = oe.per_run_values(p, spec, cfg, True, "port", w)
        out[f"gpu_plugin_w{w}_s"] = time.perf_counter() - t0
finally:
    oe._kernel = orig
if oracle.ref_core() is not None:
    t0 = time.perf_counter()
    ref = oe.per_run_values(p, spec, cfg, True, "reference", workers)
    out["cpu_reference_s"] = time.perf_counter() - t0
    out["max_rel_diff_vs_reference"] = float(np.max(np.abs(gpu - ref) / np.abs(ref)))
print(json.dumps(out))
