"""Broadie-Kaya exact simulation on the GPU against golden
vectors the reference's exact_batch produced (tests/golden/make_golden.py):
same stream, same algorithm, fp64."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2309_10477_b200 import (BesselNonConvergence, HestonParams, OptionSpec, SimConfig,
                                   UnsupportedProduct, cuda_backend, greeks, price)
from paper_2309_10477_b200.model import BENCH_PARAMS

pytestmark = pytest.mark.gpu


def _cases():
    z = np.load(os.path.join(GOLDEN, "exact_cases.npz"))
    meta = json.loads(bytes(z["__meta__"]).decode())
    for name, m in meta.items():
        yield name, m, z[f"{name}__out"], (z[f"{name}__uniforms"] if m["has_uniforms"] else None)


def test_exact_batch_golden():
    for name, m, ref, u in _cases():
        got = cuda_backend.exact_batch(HestonParams(**m["params"]), m["s0"], np.array(m["times"]),
                                       np.array(m["flags"]), m["path_lo"], m["path_hi"],
                                       int(m["key_run"]), u)
        rel = np.abs(got - ref) / np.abs(ref)
        # CUDA vs glibc last-ulp differences in exp/sin/erfc can move a Newton
        # stop by one iterate (|F - u| < 1e-7 criterion): most paths agree to
        # ~1e-13, every path within the inversion tolerance
        assert np.median(rel) < 1e-11, (name, np.median(rel))
        assert rel.max() < 1e-5, (name, rel.max())


def test_exact_errors_like_reference():
    # reference: BesselNonConvergence at >= 12 steps for the BASELINE params
    p = HestonParams(**BENCH_PARAMS)
    times = np.linspace(0.0, 1.0, 13)
    with pytest.raises(BesselNonConvergence):
        cuda_backend.exact_batch(p, 100.0, times, np.ones(12, dtype=np.int64), 0, 64, 12345, None)


def test_exact_engine_vs_golden_bk_price(golden_stats):
    """engine.price(scheme='exact') on the GPU vs the reference's 2^15-path
    Broadie-Kaya estimate (different seed) within 3 combined SE."""
    p = HestonParams(**golden_stats["params"])
    spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
    s = price(p, spec, SimConfig(scheme="exact", n_paths=2**16, n_steps=1, n_runs=1, seed=5))
    bk, bk_se = golden_stats["bk_exact_euro"]["price"]
    assert abs(s.estimate - bk) <= 3 * (s.path_std_error ** 2 + bk_se ** 2) ** 0.5


def test_exact_scrambled_sobol_unbiased_and_tighter(params, euro_call):
    """Randomised QMC on the exact scheme: per-run digital shifts of points
    1..N give independent unbiased runs (vs the semi-analytic price) whose
    spread is well below the pseudo-random runs'."""
    from oracle.semi_analytic import call_price
    ref = call_price(100.0, 100.0, 1.0, params.r, params.kappa, params.theta, params.sigma,
                     params.rho, params.v0)
    base = dict(scheme="exact", n_paths=2048, n_steps=1, n_runs=30, seed=42)
    rq = price(params, euro_call, SimConfig(sampler="sobol", sobol_scramble=True, **base))
    ps = price(params, euro_call, SimConfig(sampler="pseudo", **base))
    assert np.all(np.isfinite(rq.per_run_values))
    assert len(set(rq.per_run_values)) == 30            # runs are distinct randomisations
    assert abs(rq.estimate - ref) <= 4 * rq.std_error, (rq.estimate, ref, rq.std_error)
    assert rq.std_error / ps.std_error < 0.5


def test_exact_runs_equal_per_run_batches(params):
    """hmc_exact_runs_f64 (all runs in one launch) reproduces one
    exact_batch call per run exactly, with and without supplied uniforms."""
    import oracle
    times, flags = np.array([0.0, 0.25, 0.5]), np.array([1, 1])
    keys = [oracle.derive_key(oracle.root_key(77), r) for r in range(3)]
    many = cuda_backend.exact_runs(params, 100.0, times, flags, 10, 1010, keys, None)
    for r, k in enumerate(keys):
        one = cuda_backend.exact_batch(params, 100.0, times, flags, 10, 1010, k, None)
        np.testing.assert_array_equal(many[r], one)
    rng = np.random.default_rng(3)
    u = rng.random((3, 500, 6))
    many = cuda_backend.exact_runs(params, 100.0, times, flags, 0, 500, keys, u)
    for r, k in enumerate(keys):
        np.testing.assert_array_equal(many[r], cuda_backend.exact_batch(params, 100.0, times, flags, 0, 500,
                                                                        k, u[r]))


@pytest.mark.parametrize("scramble", [False, True])
def test_exact_device_sobol_equals_host_points(params, scramble):
    """Sobol points generated inside the exact kernel equal the host's
    sobol.points (reference block 1 + run N + path, or points 1..N under
    per-run digital shifts): per-path outputs identical."""
    import oracle
    from paper_2309_10477_b200 import sobol
    times, flags = np.array([0.0, 0.25, 0.5, 0.75, 1.0]), np.array([1, 1, 1, 1])
    N, lo, hi = 3000, 1000, 2500
    keys = [oracle.derive_key(oracle.root_key(5), r) for r in range(2)]
    dev = cuda_backend.exact_runs(params, 100.0, times, flags, lo, hi, keys, None,
                                  sobol=(sobol.directions(12), scramble, N))
    for r, k in enumerate(keys):
        if scramble:
            u = sobol.points(12, 1 + lo, hi - lo, key_run=k)
        else:
            u = sobol.points(12, 1 + r * N + lo, hi - lo)
        host = cuda_backend.exact_batch(params, 100.0, times, flags, lo, hi, k, u)
        np.testing.assert_array_equal(dev[r], host)


@pytest.mark.parametrize("sampler", ["pseudo", "sobol"])
def test_exact_put_call_parity_and_price_only(params, sampler):
    """Puts price on the exact scheme (price only, like the reference);
    with common random numbers C - P = disc (S_T - K) path by path, so the
    parity gap is the martingale error of the discounted S_T."""
    cfg = SimConfig(scheme="exact", sampler=sampler, n_paths=2**15, n_steps=1, n_runs=4, seed=3)
    c = price(params, OptionSpec("european", "call", 100.0, 1.0, 100.0), cfg)
    p = price(params, OptionSpec("european", "put", 100.0, 1.0, 100.0), cfg)
    gap = np.array(c.per_run_values) - np.array(p.per_run_values)
    fwd = 100.0 - 100.0 * np.exp(-params.r)
    assert np.all(np.abs(gap - fwd) < 0.5), gap
    with pytest.raises(UnsupportedProduct):       # reference engine.py:120-121
        greeks(params, OptionSpec("european", "put", 100.0, 1.0, 100.0), cfg)


def test_exact_chunks_split_bit_identical(params):
    """hmc_exact_greeks_chunks on chunk-aligned slices produces the same
    chunk partials as on the whole range: the exact scheme inherits the
    engine's bit-identical multi-GPU reduction."""
    import ctypes
    import torch
    from paper_2309_10477_b200 import _lib, engine, exact
    spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=(0.25, 0.5, 0.75, 1.0))
    cfg = SimConfig(scheme="exact", n_paths=3 * 16384 + 1000, n_steps=1, n_runs=2, seed=9)
    h, vu, vd, hr = engine.bump_sizes(params, spec, cfg)
    times = exact.exact_step_times(spec)
    flags = np.ones(times.size - 1, dtype=np.int64)
    L = _lib.lib()
    m = _lib.Model(params.kappa, params.theta, params.sigma, params.rho, params.r, params.v0)
    idx = np.zeros(1, dtype=np.int64)
    pr = _lib.Product(1, 0, 100.0, 1.0, 100.0, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 1)
    stream = torch.cuda.current_stream()

    def chunks(lo, hi):
        sim = _lib.Sim(scheme=2, sampler=0, precision=1, want_greeks=1, n_steps=4, n_runs=2,
                       n_paths=cfg.n_paths, path_lo=lo, path_hi=hi, seed=9, h_spot=h, v0_up=vu, v0_dn=vd,
                       h_r=hr)
        nc = -(-(hi - lo) // 16384)
        out = torch.empty((2, nc, _lib.HMC_NW), dtype=torch.float64, device="cuda")
        _lib.check(L.hmc_exact_greeks_chunks(ctypes.byref(m), ctypes.byref(pr), ctypes.byref(sim),
                                             times.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 4,
                                             flags.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                             ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))
        return out.cpu().numpy()

    whole = chunks(0, cfg.n_paths)
    parts = np.concatenate([chunks(0, 16384), chunks(16384, 3 * 16384), chunks(3 * 16384, cfg.n_paths)], axis=1)
    np.testing.assert_array_equal(whole, parts)


# ---------------------------------------------------------------------------
# The reference's own exact-scheme properties (tests/test_exact.py:75-96,
# tests/test_ivlaw.py:122-137), run through the GPU backend plugin.
# ---------------------------------------------------------------------------
def _key(seed):
    from oracle import derive_key, root_key
    return int(derive_key(root_key(seed), 0))


def test_exact_martingale(params):
    """Discounted terminal mean over 10^5 exact paths equals S0 within 3 SE."""
    import math
    obs = cuda_backend.exact_batch(params, 100.0, np.array([0.0, 1.0]), np.array([1], dtype=np.int64),
                                   0, 100_000, _key(11), None)
    disc = math.exp(-params.r) * obs[:, 0]
    assert abs(disc.mean() - 100.0) < 3.0 * disc.std(ddof=1) / math.sqrt(disc.size)


def test_exact_composability_across_partitions(params):
    """One step over [0, 1] and two steps over [0, .5], [.5, 1] give the same
    law of S_T (two-sample KS)."""
    from scipy import stats
    one = cuda_backend.exact_batch(params, 100.0, np.array([0.0, 1.0]), np.array([1], dtype=np.int64),
                                   0, 50_000, _key(21), None)[:, 0]
    two = cuda_backend.exact_batch(params, 100.0, np.array([0.0, 0.5, 1.0]), np.array([0, 1], dtype=np.int64),
                                   0, 50_000, _key(22), None)[:, 0]
    assert stats.ks_2samp(one, two).pvalue > 0.01


def test_exact_tiny_dt_exceeds_series_validity(params):
    """The Bessel argument grows like 1/dt: a 1e-4 step is reported, not
    returned as garbage (the reference raises BesselNonConvergence)."""
    with pytest.raises(BesselNonConvergence):
        cuda_backend.exact_batch(params, 100.0, np.array([0.0, 1e-4]), np.array([1], dtype=np.int64),
                                 0, 64, _key(5), None)


def test_exact_vanishing_vol_of_vol_collapses_to_mean_path():
    """sigma -> 0: the integrated variance is the deterministic mean path, so
    S_T is lognormal with that variance (the reference's degenerate branch)."""
    import math
    from paper_2309_10477_b200 import DEFAULT_PARAMS
    p = HestonParams(**dict(DEFAULT_PARAMS, sigma=1e-7))
    obs = cuda_backend.exact_batch(p, 100.0, np.array([0.0, 1.0]), np.array([1], dtype=np.int64),
                                   0, 50_000, _key(3), None)
    iv = p.theta + (p.v0 - p.theta) * (1.0 - math.exp(-p.kappa)) / p.kappa
    logs = np.log(obs[:, 0] / 100.0)
    assert abs(logs.var(ddof=1) - iv) < 0.03 * iv
    assert abs(logs.mean() - (p.r - 0.5 * iv)) < 3.0 * math.sqrt(iv / logs.size)


def test_exact_zero_start_variance():
    """v0 = 0 is a valid start (reference test_exact.py:45-47)."""
    from paper_2309_10477_b200 import DEFAULT_PARAMS
    p = HestonParams(**dict(DEFAULT_PARAMS, v0=0.0))
    obs = cuda_backend.exact_batch(p, 100.0, np.array([0.0, 0.5]), np.array([1], dtype=np.int64),
                                   0, 4096, _key(9), None)
    assert np.all(np.isfinite(obs)) and np.all(obs[:, 0] > 0.0)
