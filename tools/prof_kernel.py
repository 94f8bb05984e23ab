"""Run the bench workload kernel a few times (for ncu); HMC_LIB_PATH selects a variant."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2309_10477_b200 import _lib, engine
import bench
p, spec, cfg = bench.workload()
if len(sys.argv) > 1:
    import dataclasses
    cfg = dataclasses.replace(cfg, n_paths=int(sys.argv[1]))
job = engine.Job(p, spec, cfg, True)
L = _lib.lib()
work = torch.empty(L.hmc_workspace_bytes(ctypes.byref(job.sim)), dtype=torch.uint8, device="cuda")
loc = torch.zeros((1, -(-cfg.n_paths // 16384), 14), dtype=torch.float64, device="cuda")
for _ in range(2):
    _lib.check(L.hmc_greeks_chunks(ctypes.byref(job.model), ctypes.byref(job.product), ctypes.byref(job.sim),
               ctypes.c_void_p(loc.data_ptr()), ctypes.c_void_p(work.data_ptr()), None))
torch.cuda.synchronize()
print("ok")
