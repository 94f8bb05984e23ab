"""In-tree build of libhmc.so for sm_100a (nvcc, no torch extension machinery).

``python -m paper_2309_10477_b200._build [--verbose]`` compiles each CUDA
translation unit with ``-gencode arch=compute_100a,code=sm_100a -lineinfo``
and links ``paper_2309_10477_b200/libhmc.so``.  The replay TU is compiled
with ``-fmad=false`` so its fp64 arithmetic follows the reference's
FMA-free rounding sequence ("replay parity").
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_objs")
LIB = os.path.join(PKG, "libhmc.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2",
          f"-I{os.path.join(ROOT, 'include')}"]


def nccl_dirs() -> tuple[str, str]:
    """(include, lib) directories of the torch-bundled NCCL (nvidia-nccl wheel)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia.nccl (torch's NCCL) not found: libhmc's comm unit needs nccl.h")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


_NCCL_INC, _NCCL_LIB = nccl_dirs()
UNITS = {
    "hmc_api.cu": [],
    "hmc_comm.cu": [f"-I{_NCCL_INC}", f'-DHMC_NCCL_LIB_DIR="{_NCCL_LIB}"'],
    "hmc_api_surface.cu": [],
    "hmc_api_exact.cu": [],
    "hmc_fast.cu": [],
    "hmc_replay.cu": ["-fmad=false"],
    "hmc_surface.cu": [],
    "hmc_exact.cu": ["-fmad=false"],
}


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines: dict | None = None,
          lib: str = LIB, objdir: str = BUILD) -> str:
    """Compile and link; ``defines`` (e.g. {"HMC_SINCOS_POLY": 1}) build a
    kernel variant into ``lib`` / ``objdir`` (used by tools/kernel_variants.py)."""
    os.makedirs(objdir, exist_ok=True)
    dflags = [f"-D{k}={v}" for k, v in (defines or {}).items()]
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "hmc.h"))
    objs, cmds = [], []
    for unit, extra in UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(objdir, unit.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [src, __file__] + headers):
            cmd = [nvcc(), *ARCH, *COMMON, *dflags, *extra, "-c", src, "-o", obj]
            if verbose:
                cmd += ["-Xptxas", "-v"]
                print(" ".join(cmd), flush=True)
            cmds.append(cmd)
    # translation units compile independently: run them concurrently
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max(1, min(len(cmds), os.cpu_count() or 1))) as pool:
        for fut in [pool.submit(subprocess.run, c, check=True) for c in cmds]:
            fut.result()
    if force or _stale(lib, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return lib


CHECKED_LIB = os.path.join(PKG, "_variants", "libhmc_checked.so")


def build_checked(verbose: bool = False, force: bool = False) -> str:
    """The bounds-checked build (device asserts on every data- or
    table-dependent index, csrc/hmc_device.cuh HMC_DCHECK) -- the stand-in
    for compute-sanitizer (tests/test_gpu_checked.py); never the product."""
    return build(verbose=verbose, force=force, defines={"HMC_DEBUG_BOUNDS": 1}, lib=CHECKED_LIB,
                 objdir=os.path.join(PKG, "_variants", "obj_checked"))


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force="--force" in sys.argv)
    print(LIB)
