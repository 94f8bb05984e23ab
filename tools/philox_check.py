"""Device Philox4x32-10 against a host restatement and a price probe on the
production stream (dev tool)."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_10477_b200 import _lib, BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, price
ctr = np.array([[0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0, 0, 0, 0], [1, 2, 3, 4], [5, 7, 0x1234, 0x99]], dtype=np.uint32)
out = np.zeros_like(ctr)
_lib.check(_lib.lib().hmc_philox_check(ctr.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), len(ctr), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), 0))
print([[hex(x) for x in r] for r in out])
p = HestonParams(**BENCH_PARAMS); spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
for prec in ("fp32", "fp64"):
    s = price(p, spec, SimConfig(scheme="milstein", n_paths=2**20, n_steps=64, n_runs=8, seed=1, precision=prec))
    print(prec, "runs", [round(x, 4) for x in s.per_run_values], "sd", s.std_error, "path se", s.path_std_error * 8 ** 0.5)
    vals = [price(p, spec, SimConfig(scheme="milstein", n_paths=2**20, n_steps=64, n_runs=1, seed=sd, precision=prec)).estimate for sd in range(1, 9)]
    print(prec, "seeds", [round(x, 4) for x in vals])
