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
