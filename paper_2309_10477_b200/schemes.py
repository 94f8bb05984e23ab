"""The reference's ``schemes`` module (``hestonmc/schemes.py``): one-path,
step-at-a-time Euler / Milstein full-truncation simulation driven by a
caller's uniform stream -- the scalar specification the engine's kernels
implement in bulk.

Every step runs on the device through the same fp64 step and quantile code
as the replay kernels (``hmc_steps_f64``: ``_core.pyx:399-404``,
``schemes.py:33-61``); ``simulate_path`` draws the path's 2 * n_steps
uniforms from the stream in the reference's order (asset, variance per step)
and runs the whole path as one device call of the reference backend kernel
(``hmc_discretised_batch_f64`` with supplied uniforms).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib, rng
from .errors import InvalidParams, ValidationError
from .model import GridSpec, HestonParams, PathObservables, averaging_indices

_DP = ctypes.POINTER(ctypes.c_double)
SCHEMES = ("euler", "milstein")


@dataclass(frozen=True)
class PathState:
    s: float
    v: float
    t: float


def _model(p: HestonParams) -> _lib.Model:
    return _lib.Model(p.kappa, p.theta, p.sigma, p.rho, p.r, p.v0)


def _step(stream, params: HestonParams, state: PathState, dt: float, milstein: bool) -> PathState:
    if not dt > 0.0:
        raise InvalidParams(f"dt must be > 0, got {dt}")
    u = np.array([stream.next_uniform(), stream.next_uniform()])   # (asset, variance)
    s, v = np.array([state.s]), np.array([state.v])
    s_out, v_out = np.empty(1), np.empty(1)
    _lib.check(_lib.lib().hmc_steps_f64(
        ctypes.byref(_model(params)), int(milstein), float(dt), s.ctypes.data_as(_DP),
        v.ctypes.data_as(_DP), u.ctypes.data_as(_DP), 1, s_out.ctypes.data_as(_DP),
        v_out.ctypes.data_as(_DP), rng._device()))
    return PathState(s=float(s_out[0]), v=float(v_out[0]), t=state.t + dt)


def euler_step(stream, params: HestonParams, state: PathState, dt: float) -> PathState:
    """Full-truncation Euler step (log-Euler asset); two draws from ``stream``."""
    return _step(stream, params, state, dt, milstein=False)


def milstein_step(stream, params: HestonParams, state: PathState, dt: float) -> PathState:
    """Euler plus the variance correction sigma^2 dt (Z2^2 - 1) / 4."""
    return _step(stream, params, state, dt, milstein=True)


def simulate_path(stream, params: HestonParams, grid: GridSpec, scheme: str, s0: float,
                  averaging_times: tuple[float, ...] = ()) -> PathObservables:
    """One path from (s0, v0) on ``grid``: terminal price, the average over
    the averaging dates (European: the single date T) and the time-weighted
    average."""
    if scheme not in SCHEMES:
        raise ValidationError(f"unknown discretisation scheme {scheme!r}")
    idx = sorted(set(averaging_indices(grid, averaging_times))) if averaging_times else [grid.n_steps]
    u = np.array([stream.next_uniform() for _ in range(2 * grid.n_steps)]).reshape(1, -1)
    avg = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty((1, 3))
    _lib.check(_lib.lib().hmc_discretised_batch_f64(
        ctypes.byref(_model(params)), float(s0), float(grid.maturity), int(grid.n_steps),
        int(scheme == "milstein"), 0, 1, 0, u.ctypes.data_as(_DP),
        avg.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), avg.size, out.ctypes.data_as(_DP),
        rng._device()))
    return PathObservables(s_T=float(out[0, 0]), avg=float(out[0, 1]), tw_sum=float(out[0, 2]))
