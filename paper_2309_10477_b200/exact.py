"""Broadie-Kaya exact scheme behind the engine API.

``SimConfig(scheme="exact")`` -- the reference's DEFAULT scheme -- runs the
reference's exact simulation (``_core.pyx:415-521``) on the GPU
(``csrc/hmc_exact.cu``: same stream, same algorithm, fp64; per-path
observables match the reference to ~1e-15) with the reference engine's step
layout (``engine.py:32-37``: one step per averaging interval for Asians,
one [0, T] step for Europeans) and its per-path estimators
(``engine.py:47-68``).

Everything after the simulation also stays on the device
(``hmc_exact_greeks_chunks``): the estimators are reduced per 16384-path
chunk exactly like the discretised kernels' partials, so the exact scheme
shares the chunk exchange across GPUs and the fixed-shape run reduction
(bit-identical for any GPU count).  Per-run values agree with the reference
engine's 4096-path job sums + ``math.fsum`` to ~1e-15 relative (the
summation order differs; the golden tests hold them to 1e-12).

Greeks beyond the reference's pathwise Delta/Rho: the S0 and r bumps are
exact rescalings of the simulated path (ln S starts at ln S0 and accumulates
r dt, so S_k(r +- h) = S_k e^{+-h t_k}); the v0 bumps re-run the exact
kernel on the same streams (common random numbers) -- the reference's own
finite-difference method (tests/test_products.py:101-137).

The module also carries the reference's scalar exact-step API
(``hestonmc/exact.py``: ``nccs_coefficients``, ``variance_transition``,
``ExactStepResult``, ``exact_step``), drawing from the caller's streams in
the reference's order and evaluating the step on the device with the exact
kernel's arithmetic (``hmc_exact_step_f64``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib, parallel, rng, sobol
from .errors import InvalidParams
from .model import HestonParams, OptionSpec, SimConfig


# ---- the reference's scalar exact step (exact.py) ----------------------------

def nccs_coefficients(params: HestonParams, dt: float, v_u: float) -> tuple[float, float]:
    """(scale c, noncentrality lambda) of v_t = c chi'2_d(lambda) (exact.py:22-33)."""
    if dt <= 0.0:
        raise InvalidParams(f"dt must be > 0, got {dt}")
    kappa, sigma = params.kappa, params.sigma
    ek = math.exp(-kappa * dt)
    return (sigma * sigma * (1.0 - ek) / (4.0 * kappa),
            4.0 * kappa * ek * v_u / (sigma * sigma * (1.0 - ek)))


def _device_step(params: HestonParams, full: bool, s_u: float, v_u: float, dt: float,
                 draws: list[float]) -> np.ndarray:
    d = np.ascontiguousarray(draws, dtype=np.float64)
    out = np.empty(3)
    dp = ctypes.POINTER(ctypes.c_double)
    m = _lib.Model(params.kappa, params.theta, params.sigma, params.rho, params.r, params.v0)
    _lib.check(_lib.lib().hmc_exact_step_f64(ctypes.byref(m), int(full), float(s_u), float(v_u), float(dt),
                                             d.ctypes.data_as(dp), 1, out.ctypes.data_as(dp), rng._device()))
    return out


def variance_transition(stream, params: HestonParams, v_u: float, dt: float, gamma_stream=None) -> float:
    """v_t given v_u from the scaled non-central chi-squared law: one normal
    from ``stream``, the Gamma part from ``gamma_stream`` (default ``stream``)."""
    _, lam = nccs_coefficients(params, dt, v_u)
    p = rng.NccsParams(dof=params.dof, noncentrality=lam)
    z = rng.sample_normal(stream)
    g = rng.sample_gamma(gamma_stream if gamma_stream is not None else stream, 0.5 * (p.dof - 1.0), 2.0)
    return float(_device_step(params, False, 1.0, v_u, dt, [z, g, 0.5, 0.0])[1])


@dataclass(frozen=True)
class ExactStepResult:
    s_t: float
    v_t: float
    integrated_variance: float


def exact_step(stream, params: HestonParams, s_u: float, v_u: float, dt: float,
               gamma_stream=None) -> ExactStepResult:
    """One exact transition of (S, V) over [u, u + dt]: variance transition,
    integrated variance by CDF inversion, int sqrt(V) dW2 from the endpoints,
    Gaussian ln S_t -- three logical draws from ``stream`` in the reference's
    order (normal, inversion uniform, normal), the Gamma from its substream."""
    if s_u <= 0.0:
        raise InvalidParams(f"s_u must be > 0, got {s_u}")
    _, lam = nccs_coefficients(params, dt, v_u)
    p = rng.NccsParams(dof=params.dof, noncentrality=lam)
    z1 = rng.sample_normal(stream)
    g = rng.sample_gamma(gamma_stream if gamma_stream is not None else stream, 0.5 * (p.dof - 1.0), 2.0)
    u_iv = stream.next_uniform()
    z3 = rng.sample_normal(stream)
    s_t, v_t, iv = _device_step(params, True, s_u, v_u, dt, [z1, g, u_iv, z3])
    return ExactStepResult(s_t=float(s_t), v_t=float(v_t), integrated_variance=float(iv))



def exact_step_times(spec: OptionSpec) -> np.ndarray:
    """reference ``engine.py:32-37``"""
    if spec.is_asian:
        return np.concatenate([[0.0], np.asarray(spec.averaging_times, dtype=np.float64)])
    return np.array([0.0, spec.maturity])


def execute(params: HestonParams, spec: OptionSpec, config: SimConfig, want_greeks: bool,
            bumps, group=None) -> np.ndarray:
    """[n_runs, 14] {sum, sum of squares} per quantity over all paths (every
    rank returns the same, gathered in path order)."""
    import torch
    from .errors import DeviceError
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible; the engine has no CPU fallback")
    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    times = exact_step_times(spec)
    n_steps = times.size - 1
    flags = np.ones(n_steps, dtype=np.int64)  # every step end is a fixing (European: T)
    rank, world = parallel.world_info(group)
    sl = parallel.shard(config.n_paths, rank, world)
    h_spot, v_up, v_dn, h_r = bumps
    model = _lib.Model(params.kappa, params.theta, params.sigma, params.rho, params.r, params.v0)
    unused_idx = np.zeros(1, dtype=np.int64)   # the exact path takes step_times / flags instead
    product = _lib.Product(_lib.STYLE[spec.style], _lib.RIGHT[spec.right], spec.strike, spec.maturity,
                           spec.spot, unused_idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 1)
    sim = _lib.Sim(scheme=_lib.SCHEME["milstein"], sampler=_lib.SAMPLER[config.sampler], precision=1,
                   want_greeks=int(want_greeks), n_steps=n_steps, n_runs=config.n_runs,
                   n_paths=config.n_paths, path_lo=sl.path_lo, path_hi=sl.path_hi,
                   seed=config.seed & (2**64 - 1), h_spot=h_spot, v0_up=v_up, v0_dn=v_dn, h_r=h_r,
                   sobol_scramble=int(bool(config.sobol_scramble)))
    directions = None
    if config.sampler == "sobol":               # engine.py:97-101, points made on the device
        directions = np.ascontiguousarray(sobol.directions(3 * n_steps))
        sim.sobol_v = directions.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
        sim.sobol_v_on_device = 0
    local = torch.empty((config.n_runs, sl.n_chunks, _lib.HMC_NW), dtype=torch.float64, device=dev)
    if sl.n_paths > 0:
        _lib.check(L.hmc_exact_greeks_chunks(
            ctypes.byref(model), ctypes.byref(product), ctypes.byref(sim),
            times.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n_steps,
            flags.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.c_void_p(local.data_ptr()),
            ctypes.c_void_p(stream.cuda_stream)))
    full = parallel.gather_chunks(local, config.n_paths, group)
    out = torch.empty((config.n_runs, _lib.HMC_NW), dtype=torch.float64, device=dev)
    _lib.check(L.hmc_reduce_chunks(ctypes.c_void_p(full.data_ptr()), config.n_runs, full.shape[1],
                                   ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))
    del directions
    return out.cpu().numpy()
