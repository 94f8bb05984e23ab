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

Greeks beyond the reference's pathwise Delta/Rho: the S0 bump (and the r
bump of a European) is an exact rescaling of the simulated path (ln S
starts at ln S0 and accumulates r dt); the v0 bumps and the Asian r bumps
re-run the exact kernel on the same streams (common random numbers) -- the
reference's own finite-difference method (tests/test_products.py:101-137).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib, parallel, sobol
from .model import HestonParams, OptionSpec, SimConfig


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
