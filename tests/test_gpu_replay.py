"""fp64 replay parity on the GPU: the backend entry ``discretised_batch``
(reference _core.pyx:354-412) must reproduce the reference's per-path
(s_T, avg, tw_sum) within 1e-12 relative (north star, check (a)), on the
golden vectors the reference produced and on fresh inputs against the
bit-exact C oracle."""

import math

import numpy as np
import pytest
from scipy.special import ndtr

import oracle
from paper_2309_10477_b200 import cuda_backend
from paper_2309_10477_b200.model import DEFAULT_PARAMS, HestonParams

pytestmark = pytest.mark.gpu

RTOL = 1e-12


def _rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def test_golden_vectors(golden_replay):
    for name, c in golden_replay.items():
        got = cuda_backend.discretised_batch(HestonParams(**c["params"]), c["s0"], c["T"],
                                             c["n_steps"], c["milstein"], c["path_lo"],
                                             c["path_hi"], c["key_run"], c["uniforms"], c["avg"])
        assert got.shape == c["out"].shape, name
        assert _rel(got, c["out"]) <= RTOL, (name, _rel(got, c["out"]))


@pytest.mark.parametrize("milstein", [False, True])
@pytest.mark.parametrize("avg", ["euro", "daily", "sparse"])
def test_fresh_inputs_vs_oracle(milstein, avg, bench_params):
    n_steps = 252
    idx = {"euro": np.array([252]), "daily": np.arange(1, 253),
           "sparse": np.array([21, 63, 126, 189, 252])}[avg]
    kr = oracle.derive_key(oracle.root_key(2024), 3)
    a = cuda_backend.discretised_batch(bench_params, 100.0, 1.0, n_steps, milstein, 77, 4173, kr,
                                       None, idx)
    b = oracle.discretised_batch(bench_params, 100.0, 1.0, n_steps, milstein, 77, 4173, kr, None, idx)
    assert _rel(a, b) <= RTOL


def test_path_range_offsets_bit_exact(params):
    # reference tests/test_backends.py:53-60
    kr = oracle.derive_key(oracle.root_key(42), 0)
    avg = np.array([16], dtype=np.int64)
    full = cuda_backend.discretised_batch(params, 100.0, 1.0, 16, True, 0, 64, kr, None, avg)
    tail = cuda_backend.discretised_batch(params, 100.0, 1.0, 16, True, 32, 64, kr, None, avg)
    np.testing.assert_array_equal(full[32:], tail)


def test_empty_range(params):
    out = cuda_backend.discretised_batch(params, 100.0, 1.0, 16, True, 10, 10, 1, None, np.array([16]))
    assert out.shape == (0, 3)


class TestKnownAnswers:
    """Forced-uniform known answers (reference tests/test_schemes.py:34-110)
    through the GPU kernel's supplied-uniforms path."""

    def test_single_drift_step_terminal(self, params):
        u = np.full((4, 2), 0.5)
        out = cuda_backend.discretised_batch(params, 100.0, 1.0, 1, False, 0, 4, 0, u, np.array([1]))
        assert out[:, 0] == pytest.approx(100.0 * math.exp(params.r - 0.5 * params.v0), rel=1e-14)

    def test_multi_step_drift_only(self, params):
        """z1 = z2 = 0 (uniforms 1/2): the variance follows the deterministic
        recursion and S the drift exp((r - v/2) dt) (reference
        tests/test_schemes.py:34-46), Euler and Milstein."""
        n, T = 8, 1.0
        dt = T / n
        u = np.full((3, 2 * n), 0.5)
        for milstein in (False, True):
            out = cuda_backend.discretised_batch(params, 100.0, T, n, milstein, 0, 3, 0, u, np.array([n]))
            s, v = 100.0, params.v0
            for _ in range(n):
                s = s * math.exp((params.r - 0.5 * v) * dt)
                vn = v + params.kappa * (params.theta - v) * dt
                if milstein:
                    vn += 0.25 * params.sigma ** 2 * dt * (0.0 - 1.0)
                v = max(vn, 0.0)
            np.testing.assert_allclose(out[:, 0], s, rtol=1e-14)

    def test_euler_equals_milstein_as_sigma_vanishes(self):
        """reference tests/test_schemes.py:80-88: the Milstein correction is
        O(sigma^2), so with sigma -> 0 both schemes give the same paths."""
        p = HestonParams(**{**DEFAULT_PARAMS, "sigma": 1e-7})
        kr = oracle.derive_key(oracle.root_key(3), 0)
        a = cuda_backend.discretised_batch(p, 100.0, 1.0, 64, False, 0, 512, kr, None, np.array([64]))
        b = cuda_backend.discretised_batch(p, 100.0, 1.0, 64, True, 0, 512, kr, None, np.array([64]))
        np.testing.assert_allclose(a, b, rtol=1e-10)

    def test_milstein_equals_euler_when_z2_is_one(self):
        p = HestonParams(**{**DEFAULT_PARAMS, "rho": 0.0})
        u = np.array([[0.31, float(ndtr(1.0))]] * 8)
        a = cuda_backend.discretised_batch(p, 100.0, 0.125, 1, False, 0, 8, 0, u, np.array([1]))
        b = cuda_backend.discretised_batch(p, 100.0, 0.125, 1, True, 0, 8, 0, u, np.array([1]))
        np.testing.assert_array_equal(a[:, 0], b[:, 0])

    def test_truncation_clamps_to_zero(self):
        # v = 0 and the Milstein -sigma^2 dt / 4 term drive v negative -> clamp,
        # so the asset path is deterministic drift afterwards
        p = HestonParams(**{**DEFAULT_PARAMS, "theta": 0.001, "v0": 0.0})
        u = np.full((2, 8), 0.5)
        out = cuda_backend.discretised_batch(p, 100.0, 1.0, 4, True, 0, 2, 0, u, np.array([4]))
        assert np.all(out[:, 0] > 0.0)
        assert out[0, 0] == pytest.approx(100.0 * math.exp(p.r), rel=1e-13)

    def test_terminal_date_average_equals_european(self, params):
        kr = oracle.derive_key(oracle.root_key(8), 0)
        a = cuda_backend.discretised_batch(params, 100.0, 1.0, 16, True, 0, 256, kr, None, np.array([16]))
        np.testing.assert_array_equal(a[:, 0], a[:, 1])
        np.testing.assert_allclose(a[:, 2], a[:, 0] * 1.0, rtol=0, atol=0)

    @pytest.mark.parametrize("milstein", [False, True])
    def test_martingale_32k_paths(self, params, milstein):
        # reference tests/test_schemes.py:111-119
        kr = oracle.derive_key(oracle.root_key(13), 0)
        obs = cuda_backend.discretised_batch(params, 100.0, 1.0, 128, milstein, 0, 32_000, kr, None,
                                             np.array([128]))
        disc = math.exp(-params.r) * obs[:, 0]
        se = disc.std(ddof=1) / math.sqrt(disc.size)
        assert abs(disc.mean() - 100.0) < 3.0 * se

    def test_variance_stress_finite(self):
        p = HestonParams(kappa=2.0, theta=0.01, sigma=2.0, rho=-0.5, r=0.0, v0=1e-6)
        kr = oracle.derive_key(oracle.root_key(99), 0)
        out = cuda_backend.discretised_batch(p, 100.0, 1.0, 512, True, 0, 4096, kr, None, np.array([512]))
        assert np.all(np.isfinite(out)) and np.all(out[:, 0] > 0.0)


def test_reference_engine_runs_on_gpu_backend(golden_engine):
    """The reference engine's orchestration (restated in oracle.engine, which
    reproduces the reference bit for bit) driven through the cuda backend --
    the plugin swap of reference tests/test_backends.py:63-71."""
    from oracle import engine as oe
    from conftest import spec_from
    from paper_2309_10477_b200.model import SimConfig
    c = golden_engine["paper_euro_mil"]
    p, spec, cfg = HestonParams(**c["params"]), spec_from(c["spec"]), SimConfig(**c["config"])
    orig = oe._kernel
    oe._kernel = lambda kind: cuda_backend.discretised_batch
    try:
        runs = oe.per_run_values(p, spec, cfg, True, "port", workers=4)
    finally:
        oe._kernel = orig
    np.testing.assert_allclose(runs[:, 0], c["greeks_price"], rtol=1e-12)
    np.testing.assert_allclose(runs[:, 1], c["greeks_delta"], rtol=1e-12)
    np.testing.assert_allclose(runs[:, 2], c["greeks_rho"], rtol=1e-12)
