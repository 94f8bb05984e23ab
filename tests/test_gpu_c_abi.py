"""The C ABI from a plain C host: compile
tests/c_abi/greeks_example.c against include/hmc.h, link libhmc.so, run it,
and compare with the Python engine on the same job (same Philox stream)."""

import os
import shutil
import subprocess

import pytest

from conftest import ROOT
from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, daily_fixings, greeks

pytestmark = pytest.mark.gpu


def test_plain_c_host(tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lib_dir = os.path.join(ROOT, "paper_2309_10477_b200")
    exe = tmp_path / "greeks_example"
    # libhmc.so has no SONAME prefix 'lib' issue: link by full path
    subprocess.run([cc, "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c_abi", "greeks_example.c"),
                    os.path.join(lib_dir, "libhmc.so"), f"-Wl,-rpath,{lib_dir}", "-lm",
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), str(2**20)], check=True, capture_output=True, text=True).stdout
    rows = {ln.split()[0]: ln.split()[1:] for ln in out.strip().splitlines()}
    p = HestonParams(**BENCH_PARAMS)
    spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 252))
    g = greeks(p, spec, SimConfig(scheme="milstein", n_paths=2**20, n_steps=252, n_runs=1, seed=42))
    for q in ("price", "delta", "rho", "gamma", "vega", "delta_fd", "rho_fd"):
        assert float(rows[q][0]) == pytest.approx(g[q].estimate, rel=1e-12, abs=1e-14), q
    assert rows["multi_bit_identical"][0] == "1"
    assert rows["put_greeks_rc"][0] == "-4"


@pytest.mark.parametrize("n_paths,n_runs,n_dev,qmc", [
    (70001, 3, 3, {}), (40000, 2, 7, {}), (2**20, 1, 2, {}),
    # Sobol: slices start at chunk boundaries, runs at 1 + r N (unaligned
    # 32-point blocks for the Gray-code tables), or every run at point 1
    (70001, 3, 3, dict(sampler="sobol", sobol_highdim_ack=True)),
    (40000, 2, 3, dict(sampler="sobol", sobol_highdim_ack=True, sobol_scramble=True))])
def test_greeks_multi_bit_identical(n_paths, n_runs, n_dev, qmc):
    """hmc_greeks_multi deals chunk-aligned slices over a device list (here
    the one GPU repeated: separate streams and buffers, the same code path
    as distinct GPUs) and must reproduce hmc_greeks bit for bit, including
    device lists longer than the chunk count (empty slices)."""
    import ctypes
    import numpy as np
    from paper_2309_10477_b200 import _lib, engine
    p = HestonParams(**BENCH_PARAMS)
    spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 64))
    job = engine.Job(p, spec, SimConfig(scheme="milstein", n_paths=n_paths, n_steps=64, n_runs=n_runs,
                                        seed=5, **qmc), True)
    if job.sobol_host is not None:       # host direction numbers for the one-call entries
        v = np.ascontiguousarray(job.sobol_host)
        job.sim.sobol_v = v.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
        job.sim.sobol_v_on_device = 0
    L = _lib.lib()
    one = np.zeros((n_runs, _lib.HMC_NW))
    multi = np.zeros((n_runs, _lib.HMC_NW))
    pd = ctypes.POINTER(ctypes.c_double)
    _lib.check(L.hmc_greeks(ctypes.byref(job.model), ctypes.byref(job.product), ctypes.byref(job.sim),
                            one.ctypes.data_as(pd), 0))
    devs = (ctypes.c_int32 * n_dev)(*([0] * n_dev))
    _lib.check(L.hmc_greeks_multi(ctypes.byref(job.model), ctypes.byref(job.product), ctypes.byref(job.sim),
                                  multi.ctypes.data_as(pd), devs, n_dev))
    assert np.array_equal(one, multi)
    assert np.all(one[:, 0] > 0)


def test_integration_md_ctypes_stub_runs():
    """The plain-ctypes backend stub printed in INTEGRATION.md (what a
    reference maintainer would paste into hestonmc/backend.py) is executable
    and returns what cuda_backend.discretised_batch returns."""
    import re
    import numpy as np
    from paper_2309_10477_b200 import cuda_backend
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    stub = next(b for b in blocks if "hmc_discretised_batch_f64" in b and "argtypes" in b)
    lib = os.path.join(ROOT, "paper_2309_10477_b200", "libhmc.so")
    ns = {}
    exec(compile(stub.replace('"libhmc.so"', repr(lib)), "INTEGRATION.md", "exec"), ns)
    p = HestonParams(**BENCH_PARAMS)
    avg = np.array([8, 16, 24, 32])
    got = ns["discretised_batch"](p, 100.0, 1.0, 32, True, 0, 256, 12345, None, avg)
    ref = cuda_backend.discretised_batch(p, 100.0, 1.0, 32, True, 0, 256, 12345, None, avg)
    assert ns["BACKEND_NAME"] == "cuda"
    np.testing.assert_array_equal(got, ref)

