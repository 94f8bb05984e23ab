"""The reference backend-module protocol, served by the GPU.

A drop-in for ``hestonmc._core`` / ``hestonmc._batch_py`` behind the
reference's plugin seam (``backend.py:28-41``): a module exposing
``BACKEND_NAME`` and ``discretised_batch`` / ``exact_batch`` with the
reference signatures.  The reference engine can be driven through it
unchanged, e.g. ``monkeypatch.setattr(engine, "get_backend", lambda:
cuda_backend)`` (the swap ``tests/test_backends.py:63-71`` uses).

``exact_batch`` runs the reference's Broadie-Kaya scheme (same stream, same
algorithm) on the GPU in fp64.

``discretised_batch`` is the fp64 replay kernel: the reference's SplitMix64
stream (or the caller's uniforms), its Acklam+Halley inverse normal and its
operation order, one path per GPU thread; per-path outputs match the
reference to ~1e-15 relative (gate 1e-12).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

BACKEND_NAME = "cuda"


def _device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return int(torch.cuda.current_device())
    except ImportError:  # pragma: no cover - torch is part of the image
        pass
    return 0


def discretised_batch(params, s0: float, T: float, n_steps: int, milstein: bool,
                      path_lo: int, path_hi: int, key_run: int, uniforms,
                      avg_indices) -> np.ndarray:
    """Euler/Milstein paths for [path_lo, path_hi): (n, 3) float64
    [s_T, avg, tw_sum] (reference ``_core.pyx:354-412``)."""
    n = int(path_hi) - int(path_lo)
    out = np.empty((max(n, 0), 3))
    avg = np.ascontiguousarray(avg_indices, dtype=np.int64)
    u = None
    if uniforms is not None:
        u = np.ascontiguousarray(uniforms, dtype=np.float64)
        if u.shape[0] < n or u.shape[1] < 2 * n_steps:
            raise ValueError("uniforms must be at least (path_hi - path_lo, 2 * n_steps)")
        if u.shape[1] != 2 * n_steps:
            u = np.ascontiguousarray(u[:, : 2 * n_steps])
    m = _lib.Model(params.kappa, params.theta, params.sigma, params.rho, params.r, params.v0)
    pd = ctypes.POINTER(ctypes.c_double)
    rc = _lib.lib().hmc_discretised_batch_f64(
        ctypes.byref(m), float(s0), float(T), int(n_steps), int(bool(milstein)),
        int(path_lo), int(path_hi), int(key_run) & (2**64 - 1),
        None if u is None else u.ctypes.data_as(pd),
        avg.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), avg.size,
        out.ctypes.data_as(pd), _device())
    _lib.check(rc)
    return out


def exact_batch(params, s0: float, step_times, avg_flags, path_lo: int, path_hi: int,
                key_run: int, uniforms) -> np.ndarray:
    """Broadie-Kaya exact paths stepping through ``step_times`` (reference
    ``_core.pyx:415-521``), fp64 on the GPU with the reference's stream and
    algorithm: (n, 3) float64 [s_T, avg, tw_sum].  Numerical failures raise
    the reference's exceptions (BesselNonConvergence, ...)."""
    times = np.ascontiguousarray(step_times, dtype=np.float64)
    flags = np.ascontiguousarray(avg_flags, dtype=np.int64)
    n_steps = times.size - 1
    if flags.size != n_steps:
        raise ValueError("avg_flags needs one flag per step")
    n = int(path_hi) - int(path_lo)
    out = np.empty((max(n, 0), 3))
    u = None
    if uniforms is not None:
        u = np.ascontiguousarray(uniforms, dtype=np.float64)
        if u.shape[0] < n or u.shape[1] < 3 * n_steps:
            raise ValueError("uniforms must be at least (path_hi - path_lo, 3 * n_steps)")
        if u.shape[1] != 3 * n_steps:
            u = np.ascontiguousarray(u[:, : 3 * n_steps])
    m = _lib.Model(params.kappa, params.theta, params.sigma, params.rho, params.r, params.v0)
    pd = ctypes.POINTER(ctypes.c_double)
    rc = _lib.lib().hmc_exact_batch_f64(
        ctypes.byref(m), float(s0), times.ctypes.data_as(pd), n_steps,
        flags.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(path_lo), int(path_hi),
        int(key_run) & (2**64 - 1), None if u is None else u.ctypes.data_as(pd),
        out.ctypes.data_as(pd), _device())
    _lib.check(rc)
    return out


def exact_runs(params, s0: float, step_times, avg_flags, path_lo: int, path_hi: int, key_runs,
               uniforms, sobol=None) -> np.ndarray:
    """``exact_batch`` for several runs in one launch: run r uses
    ``key_runs[r]``; ``uniforms`` is None or (n_runs, n, 3*n_steps).
    ``sobol = (directions [30, 3*n_steps], scramble, n_paths)`` generates the
    Sobol points on the device instead (same points as the host's
    ``sobol.points``).  Returns (n_runs, n, 3) -- each run's rows equal
    ``exact_batch``'s."""
    times = np.ascontiguousarray(step_times, dtype=np.float64)
    flags = np.ascontiguousarray(avg_flags, dtype=np.int64)
    n_steps = times.size - 1
    if flags.size != n_steps:
        raise ValueError("avg_flags needs one flag per step")
    keys = np.ascontiguousarray([int(k) & (2**64 - 1) for k in key_runs], dtype=np.uint64)
    n = int(path_hi) - int(path_lo)
    out = np.empty((keys.size, max(n, 0), 3))
    u = None
    if uniforms is not None:
        u = np.ascontiguousarray(uniforms, dtype=np.float64)
        if u.shape != (keys.size, n, 3 * n_steps):
            raise ValueError("uniforms must be (n_runs, path_hi - path_lo, 3 * n_steps)")
    v, scramble, n_total = None, 0, 0
    if sobol is not None:
        v = np.ascontiguousarray(sobol[0], dtype=np.uint32)
        if v.shape != (30, 3 * n_steps):
            raise ValueError("sobol directions must be (30, 3 * n_steps)")
        scramble, n_total = int(bool(sobol[1])), int(sobol[2])
    m = _lib.Model(params.kappa, params.theta, params.sigma, params.rho, params.r, params.v0)
    pd = ctypes.POINTER(ctypes.c_double)
    rc = _lib.lib().hmc_exact_runs_f64(
        ctypes.byref(m), float(s0), times.ctypes.data_as(pd), n_steps,
        flags.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(path_lo), int(path_hi),
        keys.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), keys.size,
        None if u is None else u.ctypes.data_as(pd),
        None if v is None else v.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), scramble, n_total,
        out.ctypes.data_as(pd), _device())
    _lib.check(rc)
    return out
