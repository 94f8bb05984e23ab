"""Sobol Brownian-bridge ordering (SimConfig.sobol_bridge): the CPU
restatement (oracle/bridge.py) and the host-side contract (CPU only)."""

import ctypes

import numpy as np
import pytest

from oracle import bridge
from paper_2309_10477_b200 import ConfigInvalid, SimConfig, _lib


@pytest.mark.parametrize("S,n", [(1, 1), (1, 7), (4, 16), (16, 252), (7, 100), (64, 64), (16, 17)])
def test_construction_is_exact_brownian_motion(S, n):
    """The construction is linear in the normals; its implied covariance
    must be min(t_k, t_l) exactly (up to rounding) for every (S, n)."""
    dt = 1.0 / 252
    t = np.arange(1, n + 1) * dt
    np.testing.assert_allclose(bridge.covariance_matrix(S, n, dt), np.minimum.outer(t, t), atol=1e-15)


def test_skeleton_level_order():
    b, nodes = bridge.skeleton(16, 252)
    assert b[0] == 0 and b[-1] == 252 and all(x < y for x, y in zip(b, b[1:]))
    assert nodes[0] == (16, 0, 0)                       # horizon first
    assert nodes[1] == (8, 0, 16)                        # then the midpoint
    assert sorted(m for m, _, _ in nodes) == list(range(1, 17))
    for i, (m, lo, hi) in enumerate(nodes[1:], 1):       # parents come first
        seen = {x for x, _, _ in nodes[:i]} | {0}
        assert lo in seen and hi in seen and lo < m < hi


def test_step_normals_consume_every_pair_once():
    """Each Sobol pair drives exactly one Brownian degree of freedom: the
    normals -> increments map is invertible (full rank), so no dimension is
    skipped or reused."""
    n, S, dt = 40, 8, 0.025
    A = np.diff(bridge.construct(np.eye(n), S, n, dt), axis=1)   # rows: Z_i, columns: dW_k
    assert np.linalg.matrix_rank(A) == n


def test_config_validation():
    ok = SimConfig(scheme="milstein", sampler="sobol", sobol_highdim_ack=True, sobol_bridge=16)
    assert ok.sobol_bridge == 16
    for bad in (dict(sampler="pseudo", scheme="milstein", sobol_bridge=16),
                dict(scheme="exact", sampler="sobol", sobol_bridge=4),
                dict(scheme="milstein", sampler="sobol", sobol_highdim_ack=True, sobol_bridge=65),
                dict(scheme="milstein", sampler="sobol", sobol_highdim_ack=True, sobol_bridge=-1)):
        with pytest.raises(ConfigInvalid):
            SimConfig(**bad)


def _sim(**over):
    m = _lib.Model(2.0, 0.04, 0.3, -0.7, 0.03, 0.04)
    avg = np.array([over.pop("n_avg_last", 64)], dtype=np.int64)
    pr = _lib.Product(0, 0, 100.0, 1.0, 100.0, avg.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 1)
    v = np.zeros((30, 128), dtype=np.uint32)
    kw = dict(scheme=2, sampler=1, precision=0, want_greeks=1, n_steps=64, n_runs=1, n_paths=4096,
              path_lo=0, path_hi=4096, seed=1, h_spot=0.5, v0_up=0.0404, v0_dn=0.0396, h_r=1e-4,
              sobol_v=v.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), sobol_bridge=16)
    kw.update(over)
    return m, pr, _lib.Sim(**kw), (avg, v)


@pytest.mark.parametrize("over", [dict(sampler=0, sobol_v=None), dict(sobol_bridge=65),
                                  dict(sobol_bridge=-2),
                                  dict(sobol_bridge=65, n_steps=128, n_avg_last=128),
                                  dict(sobol_bridge=9, n_steps=8, n_avg_last=8)])
def test_c_abi_rejects_bad_bridge(over):
    L = _lib.lib()
    m, pr, sim, _keep = _sim(**over)
    buf = ctypes.create_string_buffer(64)
    rc = L.hmc_greeks_chunks(ctypes.byref(m), ctypes.byref(pr), ctypes.byref(sim), buf, buf, None)
    assert rc == _lib.HMC_E_INVALID
    assert b"bridge" in L.hmc_last_error()


def test_workspace_counts_bridge_tables():
    L = _lib.lib()
    _, _, a, _k1 = _sim(sobol_bridge=0)
    _, _, b, _k2 = _sim(sobol_bridge=16)
    assert L.hmc_workspace_bytes(ctypes.byref(b)) > L.hmc_workspace_bytes(ctypes.byref(a))
