"""The reference's ``products`` module (``hestonmc/products.py:23-51``):
payoff and pathwise Greek estimators of ONE path, the scalar form of the
per-path epilogue the kernels evaluate in bulk (``greeks_epilogue``,
csrc/hmc_device.cuh; reference ``engine._per_path_stats``,
``engine.py:47-68``).  Greeks are derived for calls only; the indicator at
equality contributes 0.
"""

from __future__ import annotations

import math

from .errors import UnsupportedProduct
from .model import OptionSpec, PathObservables


def _underlying(spec: OptionSpec, obs: PathObservables) -> float:
    return obs.avg if spec.is_asian else obs.s_T


def payoff(spec: OptionSpec, obs: PathObservables) -> float:
    """Undiscounted payoff."""
    a = _underlying(spec, obs)
    intrinsic = a - spec.strike if spec.right == "call" else spec.strike - a
    return max(intrinsic, 0.0)


def _call_only(spec: OptionSpec) -> None:
    if spec.right != "call":
        raise UnsupportedProduct("pathwise Greeks are derived for calls only")


def pathwise_delta(spec: OptionSpec, obs: PathObservables, r: float) -> float:
    """e^{-rT} (A / S0) 1{A > K}, A = S_T or the fixing average."""
    _call_only(spec)
    a = _underlying(spec, obs)
    return math.exp(-r * spec.maturity) * a / spec.spot if a > spec.strike else 0.0


def pathwise_rho(spec: OptionSpec, obs: PathObservables, r: float) -> float:
    """d(discounted payoff)/dr: European e^{-rT} K T 1{S_T > K}; Asian
    e^{-rT} ((1/N) sum S_i t_i - T (A - K)) 1{A > K}."""
    _call_only(spec)
    a = _underlying(spec, obs)
    if a <= spec.strike:
        return 0.0
    disc = math.exp(-r * spec.maturity)
    if spec.is_asian:
        return disc * (obs.tw_sum - spec.maturity * (a - spec.strike))
    return disc * spec.strike * spec.maturity
