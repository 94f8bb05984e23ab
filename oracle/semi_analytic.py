"""Heston semi-analytic European call and Greeks -- TEST ORACLE ONLY.

Not part of the reference package (which has no closed form); used as the
independent check SURVEY.md section 8(c) and the north star ask for:
European GPU prices/Greeks must agree with it within 3 SE.

Characteristic function of ln S_T in the "little Heston trap" form
(Albrecher, Mayer, Schoutens, Tistaert 2007), which stays on the principal
branch of the complex logarithm:

    d = sqrt((rho s i u - kappa)^2 + s^2 (i u + u^2))
    g = (kappa - rho s i u - d) / (kappa - rho s i u + d)
    C = kappa theta / s^2 [(kappa - rho s i u - d) T - 2 ln((1 - g e^{-dT}) / (1 - g))]
    D = (kappa - rho s i u - d) / s^2 (1 - e^{-dT}) / (1 - g e^{-dT})
    phi(u) = exp(i u (ln S0 + r T) + C + D v0)

Call = S0 P1 - K e^{-rT} P2 with the Gil-Pelaez probabilities P1, P2.
Pinned by tests/test_semi_analytic.py against the paper's reference values
(tests/test_acceptance.py:22-25 of the reference: 6.8061, 0.6958, 62.7752).
"""

from __future__ import annotations

import math

import numpy as np
from scipy.integrate import quad


def _cf(u, S0, T, r, kappa, theta, sigma, rho, v0):
    iu = 1j * u
    b = kappa - rho * sigma * iu
    d = np.sqrt(b * b + sigma * sigma * (iu + u * u))
    g = (b - d) / (b + d)
    e = np.exp(-d * T)
    C = kappa * theta / sigma ** 2 * ((b - d) * T - 2.0 * np.log((1.0 - g * e) / (1.0 - g)))
    D = (b - d) / sigma ** 2 * (1.0 - e) / (1.0 - g * e)
    return np.exp(iu * (math.log(S0) + r * T) + C + D * v0)


def probabilities(S0, K, T, r, kappa, theta, sigma, rho, v0):
    args = (S0, T, r, kappa, theta, sigma, rho, v0)
    lnK = math.log(K)
    fwd = S0 * math.exp(r * T)  # phi(-i)

    def p1(u):
        return (np.exp(-1j * u * lnK) * _cf(u - 1j, *args) / (1j * u * fwd)).real

    def p2(u):
        return (np.exp(-1j * u * lnK) * _cf(u, *args) / (1j * u)).real

    opts = dict(limit=500, epsabs=1e-12, epsrel=1e-12)
    P1 = 0.5 + quad(p1, 1e-12, 200.0, **opts)[0] / math.pi
    P2 = 0.5 + quad(p2, 1e-12, 200.0, **opts)[0] / math.pi
    return P1, P2


def call_price(S0, K, T, r, kappa, theta, sigma, rho, v0) -> float:
    P1, P2 = probabilities(S0, K, T, r, kappa, theta, sigma, rho, v0)
    return S0 * P1 - K * math.exp(-r * T) * P2


def call_greeks(S0, K, T, r, kappa, theta, sigma, rho, v0) -> dict:
    """price, delta = P1, rho = K T e^{-rT} P2, gamma and vega (dC/dv0) by
    central differences of the (1e-12-accurate) semi-analytic price."""
    P1, P2 = probabilities(S0, K, T, r, kappa, theta, sigma, rho, v0)
    price = S0 * P1 - K * math.exp(-r * T) * P2
    hs = 1e-2 * S0
    up = call_price(S0 + hs, K, T, r, kappa, theta, sigma, rho, v0)
    dn = call_price(S0 - hs, K, T, r, kappa, theta, sigma, rho, v0)
    hv = 1e-3 * max(v0, 1e-4)
    vu = call_price(S0, K, T, r, kappa, theta, sigma, rho, v0 + hv)
    vd = call_price(S0, K, T, r, kappa, theta, sigma, rho, v0 - hv)
    return {"price": price, "delta": P1, "rho": K * T * math.exp(-r * T) * P2,
            "gamma": (up - 2.0 * price + dn) / hs ** 2, "vega": (vu - vd) / (2.0 * hv)}
