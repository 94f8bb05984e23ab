"""The reference's ``bessel`` module (``hestonmc/bessel.py``) for the drop-in.

The modified Bessel function of the first kind of complex argument, in the
normalised power-series form the exact scheme uses (``_core.pyx:143-159``):
``I_nu(z) = (z/2)^nu / Gamma(nu+1) * sum_k t_k``, ``t_0 = 1``,
``t_{k+1} = t_k (z^2/4) / ((k+1)(nu+k+1))``, at most 400 terms, relative
tolerance 1e-12, ``|z| > 50`` rejected (BesselNonConvergence) -- evaluated
on the device by the exact kernel's own series (``hmc_bessel_f64``,
``csrc/hmc_exact.cu`` ``bessel_series``), elementwise.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .rng import _device

_DP = ctypes.POINTER(ctypes.c_double)


def _call(mode: int, nu: float, z, aux=None) -> np.ndarray:
    z = np.ascontiguousarray(np.asarray(z, dtype=np.complex128).reshape(-1))
    out = np.empty_like(z)
    a = None if aux is None else np.ascontiguousarray(aux, dtype=np.float64)
    _lib.check(_lib.lib().hmc_bessel_f64(
        mode, float(nu), z.ctypes.data_as(_DP), None if a is None else a.ctypes.data_as(_DP), z.size,
        out.ctypes.data_as(_DP), _device()))
    return out


def bessel_i_series(nu: float, z: complex) -> complex:
    """The normalised series sum (the factor multiplying (z/2)^nu /
    Gamma(nu+1)); works for z = 0."""
    return complex(_call(_lib.HMC_BESSEL_SERIES, nu, [z])[0])


def bessel_i(nu: float, z: complex) -> complex:
    """I_nu(z) for complex z, nu > -1 (z = 0: the limits 0, 1 / Gamma(1), inf)."""
    return complex(_call(_lib.HMC_BESSEL_I, nu, [z])[0])


def bessel_i_ratio(nu: float, coeff_num: complex, coeff_den: float, w: float,
                   log_coeff_ratio: complex | None = None) -> complex:
    """I_nu(w coeff_num) / I_nu(w coeff_den) with the (z/2)^nu prefactors
    cancelled analytically (w = 0 gives the ratio of the limits exactly);
    ``log_coeff_ratio`` is the continuous logarithm of coeff_num / coeff_den
    where its phase winds past pi (default: the principal log)."""
    lr = (math.nan, 0.0) if log_coeff_ratio is None else (log_coeff_ratio.real, log_coeff_ratio.imag)
    aux = np.array([[float(coeff_den), float(w), lr[0], lr[1]]])
    return complex(_call(_lib.HMC_BESSEL_RATIO, nu, [coeff_num], aux)[0])


def bessel_i_series_vec(nu: float, z: np.ndarray) -> np.ndarray:
    """``bessel_i_series`` over an array of complex arguments (any |z| > 50
    raises BesselNonConvergence)."""
    z = np.asarray(z, dtype=np.complex128)
    return _call(_lib.HMC_BESSEL_SERIES, nu, z).reshape(z.shape)
