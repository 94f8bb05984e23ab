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


def points(dim: int, start: int, count: int) -> np.ndarray:
    """Host evaluation of rows start..start+count-1 (float64, as scipy's
    ``random``) from the same table the kernels use -- for checks."""
    v = directions(dim).astype(np.uint64)
    n = np.arange(start, start + count, dtype=np.uint64)
    g = n ^ (n >> np.uint64(1))
    x = np.zeros((count, dim), dtype=np.uint64)
    for b in range(BITS):
        on = ((g >> np.uint64(b)) & np.uint64(1)).astype(bool)
        x[on] ^= v[b]
    return x.astype(np.float64) * 2.0 ** -BITS
