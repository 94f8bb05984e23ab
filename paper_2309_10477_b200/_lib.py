"""ctypes binding of libhmc.so (include/hmc.h).

The binding is the whole Python->CUDA boundary: plain structs and pointers,
no torch types.  ctypes releases the GIL for the duration of every call, like
the reference kernel's ``with nogil`` block (``_core.pyx:383``).

A missing library raises :class:`DeviceError` -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (BesselNonConvergence, DeviceError, QuadratureNonConvergence,
                     RootNotBracketed, UnsupportedProduct, ValidationError)

LIB_PATH = os.environ.get("HMC_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libhmc.so")

# mirrors of include/hmc.h
HMC_ABI_VERSION = 2
HMC_TILE = 128
HMC_CHUNK_TILES = 128
HMC_CHUNK = HMC_TILE * HMC_CHUNK_TILES
HMC_NQ = 7
HMC_NW = 2 * HMC_NQ
QUANTITIES = ("price", "delta", "rho", "gamma", "vega", "delta_fd", "rho_fd")

HMC_OK, HMC_E_INVALID, HMC_E_CUDA, HMC_E_NODEVICE, HMC_E_UNSUPPORTED = 0, -1, -2, -3, -4
HMC_E_BESSEL, HMC_E_QUAD, HMC_E_ROOT = -5, -6, -7
STYLE = {"european": 0, "asian_arithmetic": 1}
RIGHT = {"call": 0, "put": 1}
SCHEME = {"euler": 1, "milstein": 2}
SAMPLER = {"pseudo": 0, "sobol": 1}
PRECISION = {"fp32": 0, "fp64": 1}

#: every symbol include/hmc.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "hmc_abi_version", "hmc_last_error", "hmc_device_count",
    "hmc_chunks_in_slice", "hmc_workspace_bytes", "hmc_greeks_chunks",
    "hmc_reduce_chunks", "hmc_greeks", "hmc_greeks_multi", "hmc_discretised_batch_f64",
    "hmc_sobol_init_directions", "hmc_root_key", "hmc_derive_key", "hmc_philox_check",
    "hmc_sobol_quantile_check", "hmc_box_muller_check", "hmc_fp32_paths_check",
    "hmc_surface_acc_words", "hmc_surface_workspace_bytes", "hmc_surface_partials",
    "hmc_surface_finalize", "hmc_surface", "hmc_exact_batch_f64", "hmc_exact_runs_f64",
    "hmc_exact_greeks_chunks", "hmc_slice_chunks", "hmc_comm_unique_id", "hmc_comm_init",
    "hmc_comm_destroy", "hmc_comm_gather_chunks", "hmc_comm_allreduce_sum",
    "hmc_uniforms_f64", "hmc_ndtri_f64", "hmc_steps_f64", "hmc_gamma_f64",
    "hmc_bessel_f64", "hmc_ivlaw_phi_f64", "hmc_ivlaw_eval_f64", "hmc_exact_step_f64",
)
HMC_BESSEL_SERIES, HMC_BESSEL_I, HMC_BESSEL_RATIO = 0, 1, 2
HMC_IVLAW_INFO, HMC_IVLAW_CDF_RAW, HMC_IVLAW_CDF, HMC_IVLAW_INVERSE = 0, 1, 2, 3
HMC_COMM_ID_BYTES = 128
HMC_DTYPE_I64, HMC_DTYPE_F64 = 0, 1
HMC_SURF_MAX_STRIKES = 128
HMC_SURF_MAX_MATS = 32
HMC_BRIDGE_MAX_SEGMENTS = 64
HMC_SURF_VALS = 23


class Model(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("kappa", "theta", "sigma", "rho", "r", "v0")]


class Product(ctypes.Structure):
    _fields_ = [("style", ctypes.c_int32), ("right", ctypes.c_int32),
                ("strike", ctypes.c_double), ("maturity", ctypes.c_double),
                ("spot", ctypes.c_double),
                ("avg_idx", ctypes.POINTER(ctypes.c_int64)), ("n_avg", ctypes.c_int64)]


class Sim(ctypes.Structure):
    _fields_ = [("scheme", ctypes.c_int32), ("sampler", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("want_greeks", ctypes.c_int32),
                ("n_steps", ctypes.c_int32), ("n_runs", ctypes.c_int32),
                ("n_paths", ctypes.c_int64), ("path_lo", ctypes.c_int64),
                ("path_hi", ctypes.c_int64), ("seed", ctypes.c_uint64),
                ("h_spot", ctypes.c_double), ("v0_up", ctypes.c_double),
                ("v0_dn", ctypes.c_double), ("h_r", ctypes.c_double),
                ("sobol_v", ctypes.POINTER(ctypes.c_uint32)),
                ("sobol_v_on_device", ctypes.c_int32), ("sobol_scramble", ctypes.c_int32),
                ("sobol_bridge", ctypes.c_int32)]


class SurfaceSpec(ctypes.Structure):
    _fields_ = [("spot", ctypes.c_double), ("dt", ctypes.c_double),
                ("strikes", ctypes.POINTER(ctypes.c_double)), ("n_strikes", ctypes.c_int32),
                ("n_mats", ctypes.c_int32), ("mat_idx", ctypes.POINTER(ctypes.c_int64))]


_lib = None
_lock = threading.Lock()


def _declare(L: ctypes.CDLL) -> None:
    i32, i64, u64, dbl, vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                              ctypes.c_double, ctypes.c_void_p)
    pd = ctypes.POINTER(ctypes.c_double)
    pM, pP, pS = ctypes.POINTER(Model), ctypes.POINTER(Product), ctypes.POINTER(Sim)
    sig = {
        "hmc_abi_version": (ctypes.c_int, []),
        "hmc_last_error": (ctypes.c_char_p, []),
        "hmc_device_count": (ctypes.c_int, [ctypes.POINTER(i32)]),
        "hmc_chunks_in_slice": (i64, [pS]),
        "hmc_workspace_bytes": (i64, [pS]),
        "hmc_greeks_chunks": (ctypes.c_int, [pM, pP, pS, vp, vp, vp]),
        "hmc_reduce_chunks": (ctypes.c_int, [vp, i32, i64, vp, vp]),
        "hmc_greeks": (ctypes.c_int, [pM, pP, pS, pd, i32]),
        "hmc_greeks_multi": (ctypes.c_int, [pM, pP, pS, pd, ctypes.POINTER(i32), i32]),
        "hmc_discretised_batch_f64": (ctypes.c_int, [pM, dbl, dbl, i32, i32, i64, i64, u64,
                                                     pd, ctypes.POINTER(i64), i64, pd, i32]),
        "hmc_sobol_init_directions": (ctypes.c_int, [ctypes.POINTER(i64), ctypes.POINTER(i64),
                                                     i32, ctypes.POINTER(ctypes.c_uint32)]),
        "hmc_fp32_paths_check": (ctypes.c_int, [pM, pP, pS, ctypes.POINTER(ctypes.c_float), i64, pd, i32]),
        "hmc_box_muller_check": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint32), i32,
                                                ctypes.POINTER(ctypes.c_float), i32]),
        "hmc_sobol_quantile_check": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint32), i32, i32,
                                                    ctypes.POINTER(ctypes.c_float), i32]),
        "hmc_philox_check": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint32), i32,
                                             ctypes.POINTER(ctypes.c_uint32), i32]),
        "hmc_surface_acc_words": (i64, [ctypes.POINTER(SurfaceSpec), i32]),
        "hmc_surface_workspace_bytes": (i64, [ctypes.POINTER(SurfaceSpec), pS]),
        "hmc_surface_partials": (ctypes.c_int, [pM, ctypes.POINTER(SurfaceSpec), pS, vp, vp, vp]),
        "hmc_surface_finalize": (ctypes.c_int, [pM, ctypes.POINTER(SurfaceSpec), pS,
                                                ctypes.POINTER(i64), pd]),
        "hmc_surface": (ctypes.c_int, [pM, ctypes.POINTER(SurfaceSpec), pS, pd, i32]),
        "hmc_exact_batch_f64": (ctypes.c_int, [pM, dbl, pd, i32, ctypes.POINTER(i64), i64, i64, u64,
                                               pd, pd, i32]),
        "hmc_exact_greeks_chunks": (ctypes.c_int, [pM, pP, pS, pd, i32, ctypes.POINTER(i64), vp, vp]),
        "hmc_exact_runs_f64": (ctypes.c_int, [pM, dbl, pd, i32, ctypes.POINTER(i64), i64, i64,
                                              ctypes.POINTER(u64), i32, pd,
                                              ctypes.POINTER(ctypes.c_uint32), i32, i64, pd, i32]),
        "hmc_slice_chunks": (ctypes.c_int, [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "hmc_comm_unique_id": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint8)]),
        "hmc_comm_init": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint8), i32, i32, i32,
                                         ctypes.POINTER(vp)]),
        "hmc_comm_destroy": (ctypes.c_int, [vp]),
        "hmc_comm_gather_chunks": (ctypes.c_int, [vp, vp, i32, i64, vp, vp]),
        "hmc_comm_allreduce_sum": (ctypes.c_int, [vp, vp, i64, i32, vp]),
        "hmc_uniforms_f64": (ctypes.c_int, [ctypes.POINTER(u64), i64, ctypes.POINTER(u64), i64, pd, i32]),
        "hmc_ndtri_f64": (ctypes.c_int, [pd, i64, pd, i32]),
        "hmc_gamma_f64": (ctypes.c_int, [ctypes.POINTER(u64), ctypes.POINTER(u64), i64, dbl, dbl, pd,
                                         ctypes.POINTER(u64), i32]),
        "hmc_steps_f64": (ctypes.c_int, [pM, i32, dbl, pd, pd, pd, i64, pd, pd, i32]),
        "hmc_bessel_f64": (ctypes.c_int, [i32, dbl, pd, pd, i64, pd, i32]),
        "hmc_ivlaw_phi_f64": (ctypes.c_int, [pM, dbl, dbl, dbl, pd, i64, pd, i32]),
        "hmc_ivlaw_eval_f64": (ctypes.c_int, [pM, dbl, dbl, dbl, i32, pd, i64, pd, pd, i32]),
        "hmc_exact_step_f64": (ctypes.c_int, [pM, i32, dbl, dbl, dbl, pd, i64, pd, i32]),
        "hmc_root_key": (u64, [u64]),
        "hmc_derive_key": (u64, [u64, u64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> ctypes.CDLL:
    """The loaded native library; DeviceError if it was never built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise DeviceError(
                        f"native library missing: {LIB_PATH} "
                        "(build it with `python -m paper_2309_10477_b200._build`); "
                        "the engine has no CPU fallback")
                L = ctypes.CDLL(LIB_PATH)
                _declare(L)
                if L.hmc_abi_version() != HMC_ABI_VERSION:
                    raise DeviceError("libhmc.so ABI version mismatch; rebuild it")
                _lib = L
    return _lib


def check(rc: int) -> None:
    """Map an HMC_E* return code to the engine's exception classes."""
    if rc == HMC_OK:
        return
    msg = lib().hmc_last_error().decode(errors="replace")
    if rc == HMC_E_INVALID:
        raise ValidationError(msg)
    if rc == HMC_E_UNSUPPORTED:
        raise UnsupportedProduct(msg)
    if rc == HMC_E_BESSEL:
        raise BesselNonConvergence(msg)
    if rc == HMC_E_QUAD:
        raise QuadratureNonConvergence(msg)
    if rc == HMC_E_ROOT:
        raise RootNotBracketed(msg)
    raise DeviceError(f"libhmc error {rc}: {msg}")


def device_count() -> int:
    n = ctypes.c_int32(0)
    rc = lib().hmc_device_count(ctypes.byref(n))
    return int(n.value) if rc == HMC_OK else 0
