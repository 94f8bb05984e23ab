"""Pin the CPU oracle to the reference before trusting it (CPU only).

The C restatement (oracle/hmc_oracle.c) must reproduce, bit for bit, the
golden vectors the reference produced (tests/golden/make_golden.py) and, when
oracle/_ref was built here, the reference kernel itself on fresh inputs.
"""


import numpy as np
import pytest

import oracle
from oracle import engine as oengine
from conftest import spec_from
from paper_2309_10477_b200.model import HestonParams, SimConfig


def _p(d):
    return HestonParams(**d)


class TestRngPinned:
    def test_key_derivation(self, golden_rng):
        for seed, row in golden_rng["keys"].items():
            rk = oracle.root_key(int(seed))
            assert rk == int(row["root"])
            idx = (0, 1, 2, 1000, 2**40)
            assert [oracle.derive_key(rk, i) for i in idx] == [int(x) for x in row["derived"]]

    def test_uniform_draws(self, golden_rng):
        k = int(golden_rng["path_key"])
        got = list(oracle.uniforms_at(k, 0, 16)) + list(oracle.uniforms_at(k, 1000, 8))
        assert got == golden_rng["draws"]

    def test_inverse_normal_bitwise(self, golden_rng):
        got = oracle.inverse_normal_cdf(np.array(golden_rng["ndtri_u"]))
        np.testing.assert_array_equal(got, np.array(golden_rng["ndtri_x"]))

    def test_inverse_normal_accuracy(self):
        # reference pin tests/test_rng.py:94-96
        from scipy.special import ndtri
        u = np.linspace(1e-9, 1 - 1e-9, 20001)
        assert np.max(np.abs(oracle.inverse_normal_cdf(u) - ndtri(u))) < 1e-9


class TestReplayPinned:
    def test_golden_bitwise(self, golden_replay):
        for name, c in golden_replay.items():
            got = oracle.discretised_batch(_p(c["params"]), c["s0"], c["T"], c["n_steps"],
                                           c["milstein"], c["path_lo"], c["path_hi"],
                                           c["key_run"], c["uniforms"], c["avg"])
            np.testing.assert_array_equal(got, c["out"], err_msg=name)

    @pytest.mark.skipif(oracle.ref_core() is None, reason="oracle/_ref not built")
    def test_against_reference_kernel(self, bench_params):
        core = oracle.ref_core()
        kr = oracle.derive_key(oracle.root_key(1234), 5)
        for mil in (False, True):
            for avg in (np.array([100]), np.arange(1, 101), np.array([7, 50, 99])):
                a = core.discretised_batch(bench_params, 100.0, 1.5, 100, mil, 333, 1357, kr, None, avg)
                b = oracle.discretised_batch(bench_params, 100.0, 1.5, 100, mil, 333, 1357, kr, None, avg)
                np.testing.assert_array_equal(a, b)


def _cfg(c):
    kw = dict(c["config"])
    return SimConfig(**kw)


class TestEnginePinned:
    """The oracle's engine restatement reproduces the reference engine's
    per-run values exactly (same kernel bits, same summation order)."""

    def test_per_run_values(self, golden_engine):
        for name, c in golden_engine.items():
            if c["config"]["scheme"] == "exact":
                continue  # the C oracle restates the discretised path only
            p, spec, cfg = _p(c["params"]), spec_from(c["spec"]), _cfg(c)
            runs = oengine.per_run_values(p, spec, cfg, False, "port", workers=4)
            assert list(runs[:, 0]) == c["price"], name
            if "greeks_delta" in c:
                g = oengine.per_run_values(p, spec, cfg, True, "port", workers=4)
                assert list(g[:, 0]) == c["greeks_price"], name
                assert list(g[:, 1]) == c["greeks_delta"], name
                assert list(g[:, 2]) == c["greeks_rho"], name

    def test_crn_fd_columns_match_reference_fd(self, golden_engine):
        """Columns delta_fd / rho_fd / vega of the oracle's per-path Greeks are
        the reference's own CRN finite differences (test_products.py:101-137)."""
        for name, c in golden_engine.items():
            if "fd_delta" not in c or c["config"]["scheme"] == "exact":
                continue
            p, spec, cfg = _p(c["params"]), spec_from(c["spec"]), _cfg(c)
            b = c["bumps"]
            s = oengine.greeks_sums(p, spec, cfg, (b["h_spot"], b["v0_up"], b["v0_dn"], b["h_r"]),
                                    workers=4)
            N = cfg.n_paths
            for col, key in ((5, "fd_delta"), (6, "fd_rho"), (4, "fd_vega")):
                got = s[:, 2 * col] / N
                np.testing.assert_allclose(got, c[key], rtol=1e-9, atol=1e-9, err_msg=f"{name} {key}")
            np.testing.assert_allclose(s[:, 0] / N, c["price"], rtol=1e-13, err_msg=name)
            np.testing.assert_allclose(s[:, 2] / N, c["greeks_delta"], rtol=1e-13, err_msg=name)
            np.testing.assert_allclose(s[:, 4] / N, c["greeks_rho"], rtol=1e-13, err_msg=name)


class TestOracleProperties:
    def test_gamma_is_fd_of_pathwise_delta(self, bench_params, euro_call):
        kr = oracle.derive_key(oracle.root_key(3), 0)
        q = oracle.greeks_paths(bench_params, euro_call, 32, True, 0, 2000, kr, None,
                                np.array([32]), (0.5, 0.0404, 0.0396, 1e-4))
        # away from K the bumped pathwise deltas agree to rounding; only paths
        # whose terminal price lies within h of K carry a real gamma
        nz = np.abs(q[:, 3]) > 0.1
        assert 0 < nz.sum() < 200
        assert np.all(q[:, 0] >= 0)

    def test_price_only_zero_greeks(self, bench_params, euro_call):
        kr = oracle.derive_key(oracle.root_key(3), 0)
        q = oracle.greeks_paths(bench_params, euro_call, 8, True, 0, 64, kr, None,
                                np.array([8]), (0.5, 0.0404, 0.0396, 1e-4), want_greeks=False)
        assert np.all(q[:, 1:] == 0)


class TestStatsGolden:
    def test_stats_fixture_sane(self, golden_stats):
        e = golden_stats["euro"]
        # SURVEY 8c numbers for the same seed/size
        assert e["price"][0] == pytest.approx(9.26375, abs=1e-4)
        assert e["delta"][0] == pytest.approx(0.65616, abs=1e-4)
        a = golden_stats["asian_daily"]
        assert a["price"][0] == pytest.approx(5.25426, abs=1e-4)
        assert golden_stats["bk_exact_euro"]["price"][1] > 0
