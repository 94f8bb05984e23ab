"""Pin the semi-analytic oracle to the paper's reference values before using
it to check the GPU (reference tests/test_acceptance.py:22-25)."""

import pytest

from oracle.semi_analytic import call_greeks


def test_paper_table_values(params):
    g = call_greeks(100.0, 100.0, 1.0, params.r, params.kappa, params.theta, params.sigma,
                    params.rho, params.v0)
    assert g["price"] == pytest.approx(6.8061, abs=5e-5)
    assert g["delta"] == pytest.approx(0.6958, abs=5e-5)
    assert g["rho"] == pytest.approx(62.7752, abs=5e-5)


def test_black_scholes_limit():
    # sigma -> 0 with v0 = theta: constant variance, Black-Scholes price
    import math
    from scipy.special import ndtr
    g = call_greeks(100.0, 95.0, 0.5, 0.02, 1.0, 0.04, 1e-4, 0.0, 0.04)
    sq = math.sqrt(0.04 * 0.5)
    d1 = (math.log(100 / 95) + 0.02 * 0.5 + 0.5 * sq * sq) / sq
    bs = 100 * ndtr(d1) - 95 * math.exp(-0.01) * ndtr(d1 - sq)
    assert g["price"] == pytest.approx(bs, rel=1e-6)
    assert g["delta"] == pytest.approx(ndtr(d1), rel=1e-6)
