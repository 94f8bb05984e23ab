"""BASELINE config 5: 64 strikes x 8 maturities (0.25..2.0, dt = 1/252),
European + daily-average Asian calls, full Greeks, 2^22 paths -- one pass."""
import ctypes, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, SimConfig, surface, _lib
from paper_2309_10477_b200.surface import SurfaceJob

p = HestonParams(**BENCH_PARAMS)
strikes = np.arange(70.0, 134.0, 1.0)          # 64 strikes
mats = [0.25 * i for i in range(1, 9)]          # 8 maturities
n_paths = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 22
cfg = SimConfig(scheme="milstein", n_paths=n_paths, n_steps=504, n_runs=1, seed=42)
job = SurfaceJob(p, strikes, mats, cfg)
L = _lib.lib()
words = L.hmc_surface_acc_words(ctypes.byref(job.spec), 1)
acc = torch.zeros(words, dtype=torch.int64, device="cuda")
work = torch.empty(L.hmc_surface_workspace_bytes(ctypes.byref(job.spec), ctypes.byref(job.sim)),
                   dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
def run():
    acc.zero_()
    _lib.check(L.hmc_surface_partials(ctypes.byref(job.model), ctypes.byref(job.spec), ctypes.byref(job.sim),
                                      ctypes.c_void_p(acc.data_ptr()), ctypes.c_void_p(work.data_ptr()),
                                      ctypes.c_void_p(s.cuda_stream)))
for _ in range(3): run()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
dev_ms = sorted(ts)[2]
t0 = time.perf_counter(); res = surface(p, strikes, mats, cfg); e2e_ms = (time.perf_counter() - t0) * 1e3
path_steps = n_paths * 504
out = {"workload": "surface_64K_x_8T_euro_asian_full_greeks", "paths": n_paths, "steps": 504,
       "options": 2 * 64 * 8, "device_ms": dev_ms, "e2e_ms": e2e_ms,
       "path_steps_per_s": path_steps / (dev_ms / 1e3),
       "option_greeks_per_s": 2 * 64 * 8 * 7 / (e2e_ms / 1e3),
       "sample": {"euro_T1_K100_price": float(res.estimate["european"]["price"][3, 30]),
                  "asian_T1_K100_price": float(res.estimate["asian_arithmetic"]["price"][3, 30]),
                  "euro_T1_K100_vega": float(res.estimate["european"]["vega"][3, 30]),
                  "euro_T1_K100_price_se": float(res.path_std_error["european"]["price"][3, 30])}}
print(json.dumps(out))
