#!/usr/bin/env python
"""Build / time build-time variants of the production kernel (dev tool).

    python tools/kernel_variants.py build          # here (nvcc, no GPU)
    python tools/kernel_variants.py time [K]       # on the GPU box

Each variant is a full libhmc.so built with different HMC_* switches into
paper_2309_10477_b200/_variants/ and timed in a fresh process (HMC_LIB_PATH)
on the bench workload (2^24-path Asian daily-fixing full Greeks).
"""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2309_10477_b200", "_variants")

VARIANT_SETS = {
    "occupancy": {"base": {}, "lb6": {"HMC_MIN_BLOCKS": 6}, "lb8": {"HMC_MIN_BLOCKS": 8}},
    # RQMC Sobol driver (time with HMC_VARIANT_SOBOL=1)
    "sobol": {"u8": {}, "u4": {"HMC_SOBOL_UNROLL": 4}, "u16": {"HMC_SOBOL_UNROLL": 16},
              "u8lb8": {"HMC_MIN_BLOCKS": 8}, "u8lb6": {"HMC_MIN_BLOCKS": 6}},
    # bridge-ordered Sobol (time with HMC_VARIANT_SOBOL=1 HMC_VARIANT_BRIDGE=16)
    "bridge": {"b1": {}, "b2": {"HMC_BRIDGE_UNROLL": 2}, "b4": {"HMC_BRIDGE_UNROLL": 4},
               "b8": {"HMC_BRIDGE_UNROLL": 8}},
    # European (time with HMC_VARIANT_EURO=1): resident blocks per SM
    "euro": {"e10": {}, "e8": {"HMC_MIN_BLOCKS": 8}, "e12": {"HMC_MIN_BLOCKS": 12}, "e14": {"HMC_MIN_BLOCKS": 14}},
    # fp64 replay greeks (time with HMC_VARIANT_FP64=1): resident blocks per SM
    "replay": {"r1": {}, "r4": {"HMC_REPLAY_MINB": 4}, "r5": {"HMC_REPLAY_MINB": 5},
               "r6": {"HMC_REPLAY_MINB": 6}, "r8": {"HMC_REPLAY_MINB": 8}},
    # A/B of two prebuilt libraries dropped into _variants/ as libhmc_a.so / libhmc_b.so
    "ab": {"a": None, "b": None},
}
VARIANTS = VARIANT_SETS[os.environ.get("HMC_VARIANT_SET", "occupancy")]


def build():
    from paper_2309_10477_b200 import _build
    os.makedirs(VDIR, exist_ok=True)
    for name, d in VARIANTS.items():
        lib = os.path.join(VDIR, f"libhmc_{name}.so")
        _build.build(defines=d, lib=lib, objdir=os.path.join(VDIR, f"obj_{name}"))
        sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
        print(name, lib, "MUFU:", sass.count("MUFU."))


CHILD = r"""
import ctypes, json, sys, time
import torch
sys.path.insert(0, %(root)r)
from paper_2309_10477_b200 import _lib, engine, greeks
import bench
p, spec, cfg = bench.workload()
import os as _os, dataclasses as _dc
if _os.environ.get("HMC_VARIANT_EURO"):
    from paper_2309_10477_b200 import OptionSpec as _OS
    spec = _OS("european", "call", 100.0, 1.0, 100.0)
if _os.environ.get("HMC_VARIANT_FP64"):
    cfg = _dc.replace(cfg, precision="fp64", n_paths=2**20)
if _os.environ.get("HMC_VARIANT_SOBOL"):
    cfg = _dc.replace(cfg, sampler="sobol", sobol_highdim_ack=True, sobol_scramble=True, n_paths=2**22,
                      sobol_bridge=int(_os.environ.get("HMC_VARIANT_BRIDGE", "0")))
job = engine.Job(p, spec, cfg, True)
if job.sobol_host is not None:
    import numpy as _np
    _v = _np.ascontiguousarray(job.sobol_host)
    job.sim.sobol_v = _v.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
    job.sim.sobol_v_on_device = 0
L = _lib.lib()
work = torch.empty(L.hmc_workspace_bytes(ctypes.byref(job.sim)), dtype=torch.uint8, device="cuda")
loc = torch.zeros((1, -(-cfg.n_paths // 16384), 14), dtype=torch.float64, device="cuda")
def run():
    _lib.check(L.hmc_greeks_chunks(ctypes.byref(job.model), ctypes.byref(job.product), ctypes.byref(job.sim),
        ctypes.c_void_p(loc.data_ptr()), ctypes.c_void_p(work.data_ptr()), None))
for _ in range(3): run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(%(k)d):
    e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
g = greeks(p, spec, cfg)
print(json.dumps({"ms": sorted(ts)[len(ts)//2], "min": min(ts),
                  "est": {q: [g[q].estimate, g[q].path_std_error] for q in ("price","delta","gamma","vega","rho")}}))
"""


def time_all(k=10):
    out = {}
    for name in VARIANTS:
        lib = os.path.join(VDIR, f"libhmc_{name}.so")
        env = dict(os.environ, HMC_LIB_PATH=lib)
        r = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT, "k": k}], env=env,
                           capture_output=True, text=True, cwd=ROOT)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-2000:]
        print(name, line, flush=True)
        try:
            out[name] = json.loads(line)
        except Exception:
            out[name] = {"error": line}
    return out


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        res = time_all(int(sys.argv[2]) if len(sys.argv) > 2 else 10)
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", "variants.json"), "w") as f:
            json.dump(res, f, indent=1)
