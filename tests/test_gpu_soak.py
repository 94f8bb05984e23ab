"""Repeated calls: every public entry point returns bit-identical results
call after call, and neither torch's caching allocator nor the device's
free memory drifts (libhmc's private pool keeps at most its 1 GiB release
threshold mapped; nothing else is retained between calls)."""
import numpy as np
import pytest
import torch

from paper_2309_10477_b200 import (BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, cuda_backend,
                                   daily_fixings, greeks, price, surface)

pytestmark = pytest.mark.gpu


def _calls():
    p = HestonParams(**BENCH_PARAMS)
    euro = OptionSpec("european", "call", 100.0, 1.0, 100.0)
    asian = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 64))
    return [
        lambda: [v.estimate for v in greeks(p, asian, SimConfig(scheme="milstein", n_paths=50_000, n_steps=64,
                                                               n_runs=2, seed=1)).values()],
        lambda: [v.estimate for v in greeks(p, asian, SimConfig(scheme="milstein", sampler="sobol",
                                                               sobol_highdim_ack=True, sobol_scramble=True,
                                                               sobol_bridge=8, n_paths=20_000, n_steps=64,
                                                               n_runs=2, seed=2)).values()],
        lambda: [price(p, euro, SimConfig(scheme="milstein", n_paths=30_000, n_steps=32, n_runs=1, seed=3,
                                          precision="fp64")).estimate],
        lambda: [price(p, euro, SimConfig(scheme="exact", n_paths=4096, n_steps=1, n_runs=2, seed=4)).estimate],
        lambda: list(surface(p, [90.0, 100.0, 110.0], [0.5, 1.0],
                             SimConfig(scheme="milstein", n_paths=20_000, n_steps=32, n_runs=1, seed=5)
                             ).estimate["asian_arithmetic"]["price"].ravel()),
        lambda: list(cuda_backend.discretised_batch(p, 100.0, 1.0, 16, True, 0, 2000, 77, None,
                                                    np.array([16])).ravel()[:50]),
    ]


def test_repeated_calls_are_bit_identical_and_leak_free():
    calls = _calls()
    first = [f() for f in calls]                       # warm: pools and caches settle
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    alloc0 = torch.cuda.memory_allocated()
    for it in range(40):
        for f, want in zip(calls, first):
            assert f() == want, it
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert torch.cuda.memory_allocated() == alloc0
    assert free0 - free1 < 64 * 2**20, (free0, free1)   # nothing accumulates on the device


def test_missing_extension_fails_loudly_on_a_gpu_box(tmp_path):
    """With a GPU visible but libhmc.so missing, every entry point raises
    DeviceError -- there is no CPU path to fall back to."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {root!r})\n"
        "from paper_2309_10477_b200 import DeviceError, HestonParams, OptionSpec, SimConfig, greeks, cuda_backend\n"
        "p = HestonParams(2.0, 0.04, 0.3, -0.7, 0.03, 0.04)\n"
        "spec = OptionSpec('european', 'call', 100.0, 1.0, 100.0)\n"
        "n = 0\n"
        "for f in (lambda: greeks(p, spec, SimConfig(scheme='milstein', n_paths=1024, n_steps=8, n_runs=1)),\n"
        "          lambda: cuda_backend.discretised_batch(p, 100.0, 1.0, 8, True, 0, 16, 1, None, np.array([8]))):\n"
        "    try:\n"
        "        f()\n"
        "    except DeviceError:\n"
        "        n += 1\n"
        "print('raised', n)\n")
    env = dict(os.environ, HMC_LIB_PATH=str(tmp_path / "no_such_libhmc.so"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "raised 2" in r.stdout, (r.stdout, r.stderr[-2000:])
