"""Sobol direction numbers for the on-device Gray-code generator.

Same point set as the reference's ``rng.sobol_points``
(``rng.py:143-152`` -> ``scipy.stats.qmc.Sobol(d, scramble=False)``, 30-bit,
Joe-Kuo D(6) numbers): the table is built by the native
``hmc_sobol_init_directions`` from scipy's shipped
``_sobol_direction_numbers.npz`` (the data file the reference's generator
reads), and point n is ``x_d(n) = 2^-30 XOR_{b in gray(n)} v[b][d]`` --
random access, so every GPU thread computes its own point with no
sequential recurrence and no HBM point buffer.
"""

from __future__ import annotations

import ctypes
import functools
import os

import numpy as np

from . import _lib

BITS = 30
MAXDIM = 21201


@functools.lru_cache(maxsize=4)
def _joe_kuo() -> tuple[np.ndarray, np.ndarray]:
    import scipy.stats  # data file location only
    path = os.path.join(os.path.dirname(scipy.stats.__file__), "_sobol_direction_numbers.npz")
    with np.load(path) as z:
        return (np.ascontiguousarray(z["poly"], dtype=np.int64),
                np.ascontiguousarray(z["vinit"], dtype=np.int64))


@functools.lru_cache(maxsize=16)
def directions(dim: int) -> np.ndarray:
    """uint32 array [30, dim]: v[b, d] (read-only, cached)."""
    if not (1 <= dim <= MAXDIM):
        raise ValueError(f"sobol dimension must be in [1, {MAXDIM}], got {dim}")
    poly, vinit = _joe_kuo()
    out = np.empty((BITS, dim), dtype=np.uint32)
    rc = _lib.lib().hmc_sobol_init_directions(
        poly.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        vinit.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), dim,
        out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
    _lib.check(rc)
    out.setflags(write=False)
    return out


def _mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def digital_shifts(key_run: int, dim: int) -> np.ndarray:
    """Per-dimension 30-bit random digital shifts of one run -- the same
    values as the kernels' ``sobol_shift`` (csrc/hmc_device.cuh)."""
    d = np.arange(1, dim + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key_run & (2**64 - 1)) ^ (d * np.uint64(0x9E3779B97F4A7C15))
    return _mix64(z) >> np.uint64(34)


def points(dim: int, start: int, count: int, key_run: int | None = None) -> np.ndarray:
    """Host evaluation of rows start..start+count-1 (float64, as scipy's
    ``random``) from the same table the kernels use.  With ``key_run`` the
    run's digital shifts are applied and cell midpoints returned (the
    randomised-QMC points of ``SimConfig(sobol_scramble=True)``)."""
    v = directions(dim).astype(np.uint64)
    n = np.arange(start, start + count, dtype=np.uint64)
    g = n ^ (n >> np.uint64(1))
    x = np.zeros((count, dim), dtype=np.uint64)
    for b in range(BITS):
        on = ((g >> np.uint64(b)) & np.uint64(1)).astype(bool)
        x[on] ^= v[b]
    if key_run is None:
        return x.astype(np.float64) * 2.0 ** -BITS
    x ^= digital_shifts(key_run, dim)[None, :]
    return (x.astype(np.float64) + 0.5) * 2.0 ** -BITS
