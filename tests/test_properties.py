"""Property-based checks (hypothesis) of the CPU-side pieces: the oracle's
inverse normal (reference tests/test_rng.py:98-104 style monotonicity and
symmetry), the key derivation of the C ABI against the oracle, the host
Sobol points, and the Brownian-bridge construction -- CPU only."""


import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
from oracle import bridge
from paper_2309_10477_b200 import _lib, sobol

U = st.floats(min_value=1e-12, max_value=1 - 1e-12, allow_nan=False)


@settings(max_examples=200, deadline=None)
@given(U, U)
def test_inverse_normal_monotone(a, b):
    lo, hi = min(a, b), max(a, b)
    z = oracle.inverse_normal_cdf([lo, hi])
    assert z[0] <= z[1]


@settings(max_examples=200, deadline=None)
@given(st.floats(min_value=1e-6, max_value=0.5, allow_nan=False))
def test_inverse_normal_symmetric(u):
    # (1 - u is exact to ~1e-16 absolute; below u ~ 1e-6 that rounding, not
    # the quantile, dominates the asymmetry)
    z = oracle.inverse_normal_cdf([u, 1.0 - u])
    assert abs(z[0] + z[1]) <= 1e-9 * max(1.0, abs(z[0]))


@settings(max_examples=100, deadline=None)
@given(st.integers(min_value=0, max_value=2**64 - 1), st.integers(min_value=0, max_value=2**64 - 1))
def test_c_abi_keys_equal_oracle(seed, index):
    L = _lib.lib()
    rk = L.hmc_root_key(seed)
    assert rk == oracle.root_key(seed)
    assert L.hmc_derive_key(rk, index) == oracle.derive_key(rk, index)


@settings(max_examples=40, deadline=None)
@given(st.integers(min_value=1, max_value=64), st.integers(min_value=0, max_value=5000),
       st.integers(min_value=1, max_value=64))
def test_sobol_points_in_unit_cube(dim, start, count):
    x = sobol.points(dim, start, count)
    assert x.shape == (count, dim)
    assert np.all((x >= 0.0) & (x < 1.0))
    # Gray-code order: consecutive points differ in exactly one direction
    # number per dimension, so a point never repeats within a 2^k block
    if start % 64 == 0 and count == 64 and start > 0:
        assert len({tuple(r) for r in x}) == 64


@settings(max_examples=30, deadline=None)
@given(st.integers(min_value=1, max_value=64), st.integers(min_value=1, max_value=300))
def test_bridge_is_brownian_motion(S, n):
    S = min(S, n)
    dt = 1.0 / 252
    t = np.arange(1, n + 1) * dt
    C = bridge.covariance_matrix(S, n, dt)
    assert np.max(np.abs(C - np.minimum.outer(t, t))) <= 1e-14 * max(1.0, n * dt)


BAD = st.sampled_from([float("nan"), float("inf"), -float("inf")])


@settings(max_examples=60, deadline=None)
@given(st.sampled_from(["kappa", "theta", "sigma", "rho", "r", "v0", "strike", "maturity", "spot",
                        "h_r", "v0_up"]), BAD)
def test_c_abi_rejects_non_finite_inputs(field, bad):
    """Every floating-point input of a pricing call is validated on the host:
    NaN / inf never reach a kernel (HMC_E_INVALID, no device work)."""
    import ctypes
    m = _lib.Model(2.0, 0.04, 0.3, -0.7, 0.03, 0.04)
    avg = np.array([64], dtype=np.int64)
    pr = _lib.Product(0, 0, 100.0, 1.0, 100.0, avg.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 1)
    sim = _lib.Sim(scheme=2, sampler=0, precision=0, want_greeks=1, n_steps=64, n_runs=1, n_paths=4096,
                   path_lo=0, path_hi=4096, seed=1, h_spot=0.5, v0_up=0.0404, v0_dn=0.0396, h_r=1e-4)
    for obj in (m, pr, sim):
        if hasattr(obj, field) and field in dict(obj._fields_):
            setattr(obj, field, bad)
    buf = ctypes.create_string_buffer(64)
    rc = _lib.lib().hmc_greeks_chunks(ctypes.byref(m), ctypes.byref(pr), ctypes.byref(sim), buf, buf, None)
    assert rc == _lib.HMC_E_INVALID
