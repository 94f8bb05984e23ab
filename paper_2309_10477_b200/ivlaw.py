"""The reference's ``ivlaw`` module (``hestonmc/ivlaw.py``) for the drop-in.

The conditional law of the integrated variance over one step given both
variance endpoints -- the Broadie-Kaya characteristic function Phi (Bessel
series of complex argument), its moments from Phi at a small frequency,
the trapezoid-quadrature CDF
``F(x) = h x / pi + 2/pi sum_j sin(j h x) / j Re Phi(j h)`` truncated by the
tail criterion, and inverse-transform sampling by second-order Newton with a
bisection fallback.  Every evaluation runs on the device through the exact
kernel's own routines (``hmc_ivlaw_phi_f64`` / ``hmc_ivlaw_eval_f64``,
``csrc/hmc_exact.cu`` ``phi_node`` / ``iv_law`` / ``iv_nodes`` /
``sample_iv``), so the law here is the one the GPU exact scheme samples
from; the constants are the reference's (period mean + 12 std, tail 1e-7 for
3 nodes, at most 20000 nodes, Newton tolerance 1e-7, degenerate below a
relative spread of 1e-5).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import InvalidParams
from .model import HestonParams
from .rng import _device

_DP = ctypes.POINTER(ctypes.c_double)
_DEGENERATE_REL_STD = 1e-5


def _model(p: HestonParams) -> _lib.Model:
    return _lib.Model(p.kappa, p.theta, p.sigma, p.rho, p.r, p.v0)


def _characteristic_fn_vec(params: HestonParams, v_u: float, v_t: float, dt: float,
                           a: np.ndarray) -> np.ndarray:
    """Phi over an array of frequencies."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
    out = np.empty(a.size, dtype=np.complex128)
    _lib.check(_lib.lib().hmc_ivlaw_phi_f64(ctypes.byref(_model(params)), float(v_u), float(v_t), float(dt),
                                            a.ctypes.data_as(_DP), a.size, out.ctypes.data_as(_DP), _device()))
    return out


def characteristic_fn_raw(params: HestonParams, v_u: float, v_t: float, dt: float, a: float) -> complex:
    """Phi(a) for one real frequency a >= 0 (Phi(0) = 1 exactly)."""
    if a == 0.0:
        return 1.0 + 0.0j
    return complex(_characteristic_fn_vec(params, v_u, v_t, dt, np.array([a]))[0])


@dataclass
class IntegratedVarianceLaw:
    """F(x) = Pr(int_u^t V_s ds <= x | v_u, v_t) over a step of length dt."""

    params: HestonParams
    v_u: float
    v_t: float
    dt: float
    h: float = field(init=False)
    mean: float = field(init=False)
    std: float = field(init=False)

    def __post_init__(self):
        if self.params.kappa <= 0.0 or self.params.sigma <= 0.0:
            raise InvalidParams("kappa and sigma must be strictly positive")
        if self.dt <= 0.0:
            raise InvalidParams(f"dt must be > 0, got {self.dt}")
        info = np.empty(4)
        self._eval(_lib.HMC_IVLAW_INFO, np.empty(0), info)
        self.mean, self.std, self.h = float(info[0]), float(info[1]), float(info[2])

    def _eval(self, mode: int, x: np.ndarray, info: np.ndarray | None = None) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        out = np.empty(x.size)
        info = np.empty(4) if info is None else info
        _lib.check(_lib.lib().hmc_ivlaw_eval_f64(
            ctypes.byref(_model(self.params)), float(self.v_u), float(self.v_t), float(self.dt), mode,
            x.ctypes.data_as(_DP), x.size, out.ctypes.data_as(_DP), info.ctypes.data_as(_DP), _device()))
        return out

    def characteristic_fn(self, a: float) -> complex:
        """Phi(a); Phi(0) = 1 exactly."""
        return characteristic_fn_raw(self.params, self.v_u, self.v_t, self.dt, a)

    @property
    def is_degenerate(self) -> bool:
        return self.std < _DEGENERATE_REL_STD * self.mean

    @property
    def is_point_mass(self) -> bool:
        """Vanishing vol-of-vol: the law is the deterministic mean-path integral."""
        return self.params.sigma < 1e-4 * self.params.kappa

    def cdf_raw(self, x: float) -> float:
        """Unclamped trapezoid CDF (0 for x <= 0)."""
        return float(self._eval(_lib.HMC_IVLAW_CDF_RAW, np.array([x]))[0])

    def cdf(self, x: float) -> float:
        """F(x) clamped to [0, 1]; a step (point mass) or a Gaussian
        (degenerate spread) in the degenerate regimes."""
        return float(self._eval(_lib.HMC_IVLAW_CDF, np.array([x]))[0])

    def inverse_cdf(self, u: float) -> float:
        """F^{-1}(u), |F(result) - u| < 1e-6 (u clamped to [1e-12, 1 - 1e-12])."""
        return float(self._eval(_lib.HMC_IVLAW_INVERSE, np.array([u]))[0])
