#!/usr/bin/env python
"""Build / time block-shape variants of the surface kernel (dev tool).

    python tools/surface_variants.py build     # here (nvcc, no GPU)
    python tools/surface_variants.py time      # on the GPU box

Each variant is a full libhmc.so with different HMC_SURF_THREADS /
HMC_SURF_MINB, timed in a fresh process (HMC_LIB_PATH) by
tools/surface_bench.py (BASELINE config 5).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2309_10477_b200", "_variants")

VARIANTS = {
    "s1024x1": {},
    "noinline": {"HMC_SURF_NOINLINE": 1},
    "s512x2": {"HMC_SURF_THREADS": 512, "HMC_SURF_MINB": 2},
    "s256x4": {"HMC_SURF_THREADS": 256, "HMC_SURF_MINB": 4},
    "s768x1": {"HMC_SURF_THREADS": 768, "HMC_SURF_MINB": 1},
    "s384x2": {"HMC_SURF_THREADS": 384, "HMC_SURF_MINB": 2},
    "s896x1": {"HMC_SURF_THREADS": 896, "HMC_SURF_MINB": 1},
}
if os.environ.get("SURF_VARIANTS"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["SURF_VARIANTS"].split(",")}


def build():
    from paper_2309_10477_b200 import _build
    os.makedirs(VDIR, exist_ok=True)
    for name, d in VARIANTS.items():
        lib = os.path.join(VDIR, f"libhmc_{name}.so")
        _build.build(defines=d, lib=lib, objdir=os.path.join(VDIR, f"obj_{name}"))
        print(name, lib)


def time_all():
    out = {}
    for name in VARIANTS:
        env = dict(os.environ, HMC_LIB_PATH=os.path.join(VDIR, f"libhmc_{name}.so"))
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "surface_bench.py")],
                           capture_output=True, text=True, env=env, timeout=600)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        out[name] = json.loads(line[-1]) if line else {"error": r.stderr[-400:]}
        print(name, json.dumps(out[name]), flush=True)
    return out


if __name__ == "__main__":
    build() if sys.argv[1] == "build" else time_all()
