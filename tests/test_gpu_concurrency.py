"""Re-entrancy of the C ABI under concurrent host threads (the
reference engine calls its backend from up to `workers` pool threads on
disjoint path ranges, with no global mutable state).  Each calling thread
gets its own cached stream and thread-local error slot; results must equal
the single-threaded ones bit for bit."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2309_10477_b200 import (BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, cuda_backend,
                                   daily_fixings, greeks)

pytestmark = pytest.mark.gpu


def test_backend_plugin_from_pool_threads():
    """The reference engine's pattern: 4096-path jobs on 8 threads."""
    p = HestonParams(**BENCH_PARAMS)
    idx = np.arange(1, 65, dtype=np.int64)
    key = 0x1234_5678_9ABC_DEF0
    n, job = 8 * 4096 + 123, 4096
    whole = cuda_backend.discretised_batch(p, 100.0, 1.0, 64, True, 0, n, key, None, idx)
    ranges = [(lo, min(lo + job, n)) for lo in range(0, n, job)]
    with ThreadPoolExecutor(max_workers=8) as pool:
        parts = list(pool.map(lambda r: cuda_backend.discretised_batch(p, 100.0, 1.0, 64, True, r[0], r[1],
                                                                       key, None, idx), ranges * 3))
    for i, (lo, hi) in enumerate(ranges * 3):
        assert np.array_equal(parts[i], whole[lo:hi]), (lo, hi)


def test_engine_calls_from_threads():
    """Concurrent greeks() calls (different configurations) give exactly the
    serial results."""
    p = HestonParams(**BENCH_PARAMS)
    spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 32))
    cfgs = [SimConfig(scheme="milstein", n_paths=20_000 + 1000 * i, n_steps=32, n_runs=2, seed=i,
                      **({"sampler": "sobol", "sobol_highdim_ack": True} if i % 3 == 2 else {}))
            for i in range(9)]
    serial = [greeks(p, spec, c) for c in cfgs]
    with ThreadPoolExecutor(max_workers=6) as pool:
        threaded = list(pool.map(lambda c: greeks(p, spec, c), cfgs))
    for a, b in zip(serial, threaded):
        for q in a:
            assert a[q].per_run_values == b[q].per_run_values, q


def test_errors_stay_on_their_thread():
    """A failing call on one thread (exact scheme outside the Bessel range)
    raises there while concurrent valid calls succeed."""
    from paper_2309_10477_b200 import BesselNonConvergence
    p = HestonParams(**BENCH_PARAMS)
    bad_times = np.linspace(0.0, 1.0, 13)

    def bad():
        with pytest.raises(BesselNonConvergence):
            cuda_backend.exact_batch(p, 100.0, bad_times, np.ones(12, dtype=np.int64), 0, 64, 12345, None)
        return "raised"

    def good():
        out = cuda_backend.exact_batch(p, 100.0, np.array([0.0, 1.0]), np.array([1]), 0, 256, 7, None)
        return bool(np.all(np.isfinite(out)))

    with ThreadPoolExecutor(max_workers=8) as pool:
        res = list(pool.map(lambda f: f(), [bad, good] * 8))
    assert res == ["raised", True] * 8
