"""Latency of the reference's default call price(params, spec, SimConfig()) (exact scheme, 30 runs x 2048 paths) on the GPU engine (dev tool)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2309_10477_b200 import DEFAULT_PARAMS, HestonParams, OptionSpec, SimConfig, price, greeks
p = HestonParams(**DEFAULT_PARAMS)
spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
for cfg in (SimConfig(), SimConfig(sampler="sobol")):
    for _ in range(3): price(p, spec, cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); s = price(p, spec, cfg); ts.append(time.perf_counter() - t0)
    ts.sort(); print(cfg.sampler, "default exact price(): median %.2f ms" % (ts[10] * 1e3), s.estimate, s.std_error)
