"""The drop-in's ``products`` module (reference ``products.py:23-51``): the
scalar payoff / pathwise-Greek formulas, on the reference's own known
answers (``tests/test_products.py:22-65``) -- host arithmetic, no device."""

import math

import pytest

from paper_2309_10477_b200 import OptionSpec, UnsupportedProduct
from paper_2309_10477_b200.model import PathObservables
from paper_2309_10477_b200.products import pathwise_delta, pathwise_rho, payoff

R = 0.0319
EURO = OptionSpec("european", "call", 100.0, 1.0, 100.0)
ASIAN = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=(0.25, 0.5, 0.75, 1.0))
PUT = OptionSpec("european", "put", 100.0, 1.0, 100.0)


def obs(s_T=100.0, avg=None, tw=None):
    return PathObservables(s_T=s_T, avg=s_T if avg is None else avg, tw_sum=s_T if tw is None else tw)


def test_payoffs():
    assert payoff(EURO, obs(110.0)) == 10.0
    assert payoff(ASIAN, obs(120.0, avg=95.0)) == 0.0
    assert payoff(PUT, obs(90.0)) == 10.0
    assert payoff(EURO, obs(100.0)) == 0.0


def test_pathwise_formulas():
    assert pathwise_delta(EURO, obs(110.0), R) == pytest.approx(math.exp(-R) * 1.10)
    assert pathwise_delta(EURO, obs(90.0), R) == 0.0
    assert pathwise_delta(EURO, obs(100.0), R) == 0.0
    assert pathwise_rho(EURO, obs(150.0), R) == pytest.approx(math.exp(-R) * 100.0)
    assert pathwise_rho(EURO, obs(50.0), R) == 0.0
    o = obs(120.0, avg=105.0, tw=80.0)
    assert pathwise_rho(ASIAN, o, R) == pytest.approx(math.exp(-R) * (80.0 - 1.0 * (105.0 - 100.0)))
    assert pathwise_delta(ASIAN, o, R) == pytest.approx(math.exp(-R) * 1.05)


def test_put_greeks_unsupported():
    with pytest.raises(UnsupportedProduct):
        pathwise_delta(PUT, obs(90.0), R)
    with pytest.raises(UnsupportedProduct):
        pathwise_rho(PUT, obs(90.0), R)
