"""Strike x maturity surfaces (BASELINE config 5).

``surface(params, strikes, maturities, config, spot)`` prices European and
daily-average Asian calls on a strike grid at several maturities of ONE
time grid, with the full Greeks set, from a single set of simulated paths
(common random numbers across every strike, maturity and style).  The
payoff epilogue is a histogram of the underlying over strike buckets
(``csrc/hmc_surface.cu``): O(log K) work per path and maturity, int64
fixed-point accumulation, so results are bit-identical for any grid size or
number of GPUs.

Each (strike, maturity) estimate is the same estimator the single-product
engine computes for ``OptionSpec(strike=K, maturity=T_m)`` with
``n_steps = T_m / dt`` and, for the Asian, daily fixings on that grid
(tests/test_gpu_surface.py checks this equality).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, parallel, sobol
from .errors import DeviceError, UnsupportedProduct, ValidationError
from .model import GridSpec, HestonParams, OptionSpec, SimConfig

STYLES = ("european", "asian_arithmetic")


@dataclass
class SurfaceResult:
    strikes: np.ndarray
    maturities: np.ndarray
    #: estimate[style][quantity] -> (n_maturities, n_strikes)
    estimate: dict = field(default_factory=dict)
    #: SD of the per-run estimates (ddof=1, reference convention), 0 for 1 run
    std_error: dict = field(default_factory=dict)
    #: per-path standard error of ``estimate``
    path_std_error: dict = field(default_factory=dict)
    wall_ms: float = 0.0
    n_paths: int = 0
    n_runs: int = 0


def _grid(maturities, config: SimConfig) -> tuple[float, list[int]]:
    mats = [float(t) for t in maturities]
    if not mats or any(b <= a for a, b in zip(mats[:-1], mats[1:])) or mats[0] <= 0:
        raise ValidationError("maturities must be positive and strictly increasing")
    grid = GridSpec(maturity=mats[-1], n_steps=config.n_steps)
    return grid.dt, [grid.index_of(t) for t in mats]


class SurfaceJob:
    def __init__(self, params: HestonParams, strikes, maturities, config: SimConfig,
                 spot: float = 100.0):
        if config.scheme == "exact":
            raise UnsupportedProduct("surfaces run on the euler / milstein schemes")
        if config.precision != "fp32":
            raise UnsupportedProduct("surfaces run on the fp32 path (pseudo or Sobol)")
        if config.sobol_bridge:
            raise UnsupportedProduct("surfaces take time-ordered Sobol dimensions (no Brownian bridge)")
        self.strikes = np.ascontiguousarray(strikes, dtype=np.float64)
        if not (1 <= self.strikes.size <= _lib.HMC_SURF_MAX_STRIKES):
            raise ValidationError(f"need 1..{_lib.HMC_SURF_MAX_STRIKES} strikes")
        if not (np.all(self.strikes > 0) and np.all(np.diff(self.strikes) > 0)):
            raise ValidationError("strikes must be positive and strictly increasing")
        if len(maturities) > _lib.HMC_SURF_MAX_MATS:
            raise ValidationError(f"need at most {_lib.HMC_SURF_MAX_MATS} maturities")
        dt, idx = _grid(maturities, config)
        self.maturities = np.array([float(t) for t in maturities])
        self.mat_idx = np.ascontiguousarray(idx, dtype=np.int64)
        OptionSpec("european", "call", float(self.strikes[0]), float(self.maturities[-1]), spot)
        self.spec = _lib.SurfaceSpec(
            spot, dt, self.strikes.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            self.strikes.size, self.mat_idx.size,
            self.mat_idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
        hv = config.bump_v0 * (params.v0 if params.v0 > 0.0 else params.theta)
        self.model = _lib.Model(params.kappa, params.theta, params.sigma, params.rho, params.r,
                                params.v0)
        self.sim = _lib.Sim(
            scheme=_lib.SCHEME[config.scheme], sampler=_lib.SAMPLER[config.sampler], precision=0,
            want_greeks=1, sobol_scramble=int(bool(config.sobol_scramble)),
            n_steps=config.n_steps, n_runs=config.n_runs, n_paths=config.n_paths, path_lo=0,
            path_hi=config.n_paths, seed=config.seed & (2**64 - 1), h_spot=config.bump_spot * spot,
            v0_up=params.v0 + hv, v0_dn=max(params.v0 - hv, 0.0), h_r=config.bump_r)
        self.config = config
        self._directions = None
        if config.sampler == "sobol":   # the single-product engine's points (engine.py:97-101)
            self._directions = np.ascontiguousarray(sobol.directions(2 * config.n_steps))
            self.sim.sobol_v = self._directions.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
            self.sim.sobol_v_on_device = 0

    def run_device(self, group=None) -> np.ndarray:
        """Accumulate this rank's slice, all-reduce the int64 histograms,
        finalize on the host -> [run][style][mat][strike][HMC_NW]."""
        import torch
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device visible; the engine has no CPU fallback")
        L = _lib.lib()
        dev = torch.device("cuda", torch.cuda.current_device())
        stream = torch.cuda.current_stream(dev)
        rank, world = parallel.world_info(group)
        sl = parallel.shard(self.config.n_paths, rank, world)
        words = int(L.hmc_surface_acc_words(ctypes.byref(self.spec), self.config.n_runs))
        acc = torch.zeros(words, dtype=torch.int64, device=dev)
        if sl.n_paths > 0:
            self.sim.path_lo, self.sim.path_hi = sl.path_lo, sl.path_hi
            work = torch.empty(int(L.hmc_surface_workspace_bytes(ctypes.byref(self.spec),
                                                                 ctypes.byref(self.sim))),
                               dtype=torch.uint8, device=dev)
            _lib.check(L.hmc_surface_partials(ctypes.byref(self.model), ctypes.byref(self.spec),
                                              ctypes.byref(self.sim), ctypes.c_void_p(acc.data_ptr()),
                                              ctypes.c_void_p(work.data_ptr()),
                                              ctypes.c_void_p(stream.cuda_stream)))
        parallel.allreduce_sum(acc, group)  # exact: integers
        h_acc = acc.cpu().numpy()
        n_m, n_k = self.mat_idx.size, self.strikes.size
        out = np.zeros((self.config.n_runs, 2, n_m, n_k, _lib.HMC_NW))
        _lib.check(L.hmc_surface_finalize(ctypes.byref(self.model), ctypes.byref(self.spec),
                                          ctypes.byref(self.sim),
                                          h_acc.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out


def summarise(job: SurfaceJob, sums: np.ndarray, wall_ms: float) -> SurfaceResult:
    cfg = job.config
    N, R = cfg.n_paths, cfg.n_runs
    M = N * R
    res = SurfaceResult(strikes=job.strikes.copy(), maturities=job.maturities.copy(),
                        wall_ms=wall_ms, n_paths=N, n_runs=R)
    s1, s2 = sums[..., 0::2], sums[..., 1::2]          # (R, style, mat, strike, quantity)
    runs = s1 / N
    est = runs.mean(axis=0)
    sd = runs.std(axis=0, ddof=1) if R > 1 else np.zeros_like(est)
    tot, tot2 = s1.sum(axis=0), s2.sum(axis=0)
    pse = np.sqrt(np.maximum(tot2 - tot * tot / M, 0.0) / max(M - 1, 1) / M)
    for si, style in enumerate(STYLES):
        res.estimate[style] = {n: est[si, ..., q] for q, n in enumerate(_lib.QUANTITIES)}
        res.std_error[style] = {n: sd[si, ..., q] for q, n in enumerate(_lib.QUANTITIES)}
        res.path_std_error[style] = {n: pse[si, ..., q] for q, n in enumerate(_lib.QUANTITIES)}
    return res


def surface(params: HestonParams, strikes, maturities, config: SimConfig, spot: float = 100.0,
            group=None) -> SurfaceResult:
    """Full-Greeks European + Asian call surfaces from one set of paths."""
    job = SurfaceJob(params, strikes, maturities, config, spot)
    t0 = time.perf_counter()
    sums = job.run_device(group)
    return summarise(job, sums, (time.perf_counter() - t0) * 1000.0 / config.n_runs)
