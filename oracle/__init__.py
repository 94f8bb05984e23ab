"""CPU oracle for the Heston Milstein Greeks path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline.  The product (``paper_2309_10477_b200``) never imports
it and has no CPU fallback.

Two checkers live here:

* ``hmc_oracle.c`` (built to ``_build/libhmc_oracle.so``): a plain-C
  restatement of the reference kernel (``_core.pyx:53-109,354-412``) plus the
  reference's CRN finite-difference method for Gamma/Vega/FD-Rho
  (``tests/test_products.py:101-137``).
* ``_ref/_core*.so``: the reference's OWN compiled kernel, built by
  ``oracle/Makefile`` from ``/root/reference/pkg/src/hestonmc/_core.c``.

Parity pin: ``tests/test_oracle.py`` checks the C restatement bit-for-bit
against golden vectors the reference produced (``tests/golden/``) and, when
``_ref`` is present, against the reference kernel directly.
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libhmc_oracle.so")

#: per-path quantity columns shared with the product's Greeks kernel
QUANTITIES = ("price", "delta", "rho", "gamma", "vega", "delta_fd", "rho_fd")


class _Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("kappa", "theta", "sigma", "rho", "r", "v0")]


class _Product(ctypes.Structure):
    _fields_ = [("is_asian", ctypes.c_int), ("is_call", ctypes.c_int),
                ("strike", ctypes.c_double), ("maturity", ctypes.c_double),
                ("spot", ctypes.c_double)]


class _Bumps(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("h_spot", "v0_up", "v0_dn", "h_r")]


_lib = None


def build() -> None:
    """Compile the C restatement (and the reference's _core when the
    reference tree is present) via oracle/Makefile."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = ctypes.CDLL(ORACLE_SO)
        u64, i64, dbl, i32 = (ctypes.c_uint64, ctypes.c_int64, ctypes.c_double,
                              ctypes.c_int)
        pd = ctypes.POINTER(ctypes.c_double)
        pi64 = ctypes.POINTER(ctypes.c_int64)
        L.hmo_mix64.restype = u64
        L.hmo_mix64.argtypes = [u64]
        L.hmo_root_key.restype = u64
        L.hmo_root_key.argtypes = [u64]
        L.hmo_derive.restype = u64
        L.hmo_derive.argtypes = [u64, u64]
        L.hmo_uniform_at.restype = dbl
        L.hmo_uniform_at.argtypes = [u64, u64]
        L.hmo_uniforms_vec.restype = None
        L.hmo_uniforms_vec.argtypes = [u64, u64, i64, pd]
        L.hmo_ndtri.restype = dbl
        L.hmo_ndtri.argtypes = [dbl]
        L.hmo_ndtri_vec.restype = None
        L.hmo_ndtri_vec.argtypes = [pd, pd, i64]
        L.hmo_discretised_batch.restype = i32
        L.hmo_discretised_batch.argtypes = [
            ctypes.POINTER(_Params), dbl, dbl, i32, i32, i64, i64, u64, pd,
            pi64, i64, pd]
        L.hmo_greeks_paths.restype = i32
        L.hmo_greeks_paths.argtypes = [
            ctypes.POINTER(_Params), ctypes.POINTER(_Product), i32, i32, i64,
            i64, u64, pd, pi64, i64, ctypes.POINTER(_Bumps), i32, pd]
        _lib = L
    return _lib


def _pd(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _params(p) -> _Params:
    return _Params(p.kappa, p.theta, p.sigma, p.rho, p.r, p.v0)


# ---- RNG restatement --------------------------------------------------------

def mix64(z: int) -> int:
    return int(lib().hmo_mix64(z))


def root_key(seed: int) -> int:
    return int(lib().hmo_root_key(seed & (2**64 - 1)))


def derive_key(parent: int, index: int) -> int:
    return int(lib().hmo_derive(parent, index))


def uniforms_at(key: int, start: int, count: int) -> np.ndarray:
    out = np.empty(count)
    lib().hmo_uniforms_vec(key, start, count, _pd(out))
    return out


def inverse_normal_cdf(u) -> np.ndarray:
    u = np.ascontiguousarray(np.atleast_1d(np.asarray(u, dtype=np.float64)))
    out = np.empty_like(u)
    lib().hmo_ndtri_vec(_pd(u), _pd(out), u.size)
    return out


# ---- path kernel restatement ---------------------------------------------

def discretised_batch(params, s0, T, n_steps, milstein, path_lo, path_hi,
                      key_run, uniforms, avg_indices) -> np.ndarray:
    """Same signature and output as the reference backend call
    (_core.pyx:354-412): (n, 3) float64 [s_T, avg, tw_sum]."""
    n = path_hi - path_lo
    out = np.empty((n, 3))
    avg = np.ascontiguousarray(avg_indices, dtype=np.int64)
    u = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.float64)
    p = _params(params)
    rc = lib().hmo_discretised_batch(
        ctypes.byref(p), float(s0), float(T), int(n_steps), int(bool(milstein)),
        int(path_lo), int(path_hi), int(key_run) & (2**64 - 1), _pd(u),
        avg.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), avg.size, _pd(out))
    assert rc == 0
    return out


def greeks_paths(params, spec, n_steps, milstein, path_lo, path_hi, key_run,
                 uniforms, avg_indices, bumps, want_greeks=True) -> np.ndarray:
    """(n, 7) per-path [price, delta, rho, gamma, vega, delta_fd, rho_fd] by
    the reference's method: pathwise Delta/Rho (engine.py:47-68) and CRN
    re-simulation of bumped inputs (test_products.py:101-137).

    ``bumps`` is (h_spot, v0_up, v0_dn, h_r) in absolute units."""
    n = path_hi - path_lo
    out = np.empty((n, 7))
    avg = np.ascontiguousarray(avg_indices, dtype=np.int64)
    u = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.float64)
    p = _params(params)
    pr = _Product(int(spec.is_asian), int(spec.right == "call"), spec.strike,
                  spec.maturity, spec.spot)
    b = _Bumps(*[float(x) for x in bumps])
    rc = lib().hmo_greeks_paths(
        ctypes.byref(p), ctypes.byref(pr), int(n_steps), int(bool(milstein)),
        int(path_lo), int(path_hi), int(key_run) & (2**64 - 1), _pd(u),
        avg.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), avg.size,
        ctypes.byref(b), int(bool(want_greeks)), _pd(out))
    assert rc == 0
    return out


def greeks_paths_z(params, spec, n_steps, milstein, normals, avg_indices, bumps,
                   want_greeks=True) -> np.ndarray:
    """``greeks_paths`` driven by given step normals ``(n, 2*n_steps)``
    ``[z1, z2]`` (z2 already correlated) instead of uniforms -- for samplers
    that build the normals differently (``oracle.bridge``)."""
    z = np.ascontiguousarray(normals, dtype=np.float64)
    n = z.shape[0]
    out = np.empty((n, 7))
    avg = np.ascontiguousarray(avg_indices, dtype=np.int64)
    pr = _Product(int(spec.is_asian), int(spec.right == "call"), spec.strike,
                  spec.maturity, spec.spot)
    b = _Bumps(*[float(x) for x in bumps])
    rc = lib().hmo_greeks_paths_z(
        ctypes.byref(_params(params)), ctypes.byref(pr), int(n_steps), int(bool(milstein)), n,
        _pd(z), avg.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), avg.size, ctypes.byref(b),
        int(bool(want_greeks)), _pd(out))
    assert rc == 0
    return out


# ---- the reference's own compiled kernel (oracle/_ref) -------------------

_ref_core = None


def ref_core():
    """The reference's compiled ``_core`` module built by oracle/Makefile
    from the reference tree, or None when it was never built here."""
    global _ref_core
    if _ref_core is None:
        hits = glob.glob(os.path.join(HERE, "_ref", "_core*.so"))
        if not hits:
            return None
        spec = importlib.util.spec_from_file_location("hestonmc._core", hits[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _ref_core = mod
    return _ref_core
