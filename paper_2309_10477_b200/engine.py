"""GPU Monte Carlo engine: the reference's ``price`` / ``greeks`` /
``run_experiment`` entry points (``hestonmc/engine.py:163-186``) on B200.

Same parameters, same return structure.  What changes underneath:

* reference: per run, 4096-path jobs on a thread pool, each calling the
  Cython kernel for (s_T, avg, tw_sum) per path, numpy per-path statistics,
  ``math.fsum`` of chunk sums (``engine.py:71-116``);
* here: ONE fused kernel launch covers all runs x paths of this rank, keeps
  path state in registers, evaluates price, pathwise Delta/Rho and the CRN
  bumps (S0, v0, r) in the same thread, and reduces per-path values to fp64
  sums and sums of squares in a fixed order; chunk partials are all-gathered
  across GPUs (NCCL) and reduced in global path order.

Determinism: results are a pure function of (seed, inputs) and bit-identical
across repeated calls and across GPU counts.

There is no CPU fallback: without the native library or a CUDA device the
engine raises :class:`DeviceError`.
"""

from __future__ import annotations

import ctypes
import math
import time

import numpy as np

from . import _lib, parallel, sobol
# the reference engine resolves its per-chunk kernel module here
# (engine.py:146); the fused GPU engine never calls a per-chunk kernel, the
# name stays for source compatibility (reference tests monkeypatch it)
from .backend import get_backend  # noqa: F401
from .errors import DeviceError, UnsupportedProduct
from .model import GridSpec, HestonParams, McSummary, OptionSpec, SimConfig, fixing_index_array

_QNAMES = _lib.QUANTITIES


def sobol_dimension(spec: OptionSpec, config: SimConfig) -> int:
    """QMC dimension (reference ``engine.py:40-44``): 2 per discretised step,
    3 per exact step."""
    if config.scheme == "exact":
        n = len(spec.averaging_times) if spec.is_asian else 1
        return 3 * n
    return 2 * config.n_steps


def _validate(spec: OptionSpec, config: SimConfig, want_greeks: bool) -> list[int]:
    """Reference checks (``engine.py:119-125``) plus the GPU scope; returns
    the fixing-date grid indices."""
    if want_greeks and spec.right != "call":
        raise UnsupportedProduct("pathwise Greeks are derived for calls only")
    if config.scheme == "exact":
        return []
    grid = GridSpec(maturity=spec.maturity, n_steps=config.n_steps)
    if spec.is_asian:
        return fixing_index_array(grid, spec.averaging_times)
    return np.array([config.n_steps], dtype=np.int64)


def bump_sizes(params: HestonParams, spec: OptionSpec, config: SimConfig) -> tuple[float, float, float, float]:
    """(h_spot, v0_up, v0_dn, h_r) in absolute units.  v0 bumps are relative
    (``bump_v0 * v0``; ``bump_v0 * theta`` when v0 == 0) and the down
    trajectory is floored at v = 0 (one-sided difference there)."""
    hv = config.bump_v0 * (params.v0 if params.v0 > 0.0 else params.theta)
    return (config.bump_spot * spec.spot, params.v0 + hv, max(params.v0 - hv, 0.0),
            config.bump_r)


_DIRECTIONS_ON_DEVICE: dict = {}


def _device_directions(host: np.ndarray, dev):
    """Sobol direction numbers on the device, uploaded once per (dimension,
    device): the table of a dimension is a fixed function of it
    (sobol.directions), so repeated QMC calls skip the 60 KB upload.  At
    most one tensor per (dimension, device) is kept."""
    import torch
    key = (int(host.shape[-1]), dev.index)
    hit = _DIRECTIONS_ON_DEVICE.get(key)
    if hit is None or hit.shape != host.shape:
        hit = torch.from_numpy(np.array(host)).to(dev)
        _DIRECTIONS_ON_DEVICE[key] = hit
    return hit


class Job:
    """ctypes image of one (params, spec, config) request."""

    def __init__(self, params: HestonParams, spec: OptionSpec, config: SimConfig,
                 want_greeks: bool):
        self.avg_idx = np.ascontiguousarray(_validate(spec, config, want_greeks), dtype=np.int64)
        self.model = _lib.Model(params.kappa, params.theta, params.sigma, params.rho,
                                params.r, params.v0)
        self.product = _lib.Product(
            _lib.STYLE[spec.style], _lib.RIGHT[spec.right], spec.strike, spec.maturity,
            spec.spot, self.avg_idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            self.avg_idx.size)
        h_spot, v_up, v_dn, h_r = bump_sizes(params, spec, config)
        self.sim = _lib.Sim(
            scheme=_lib.SCHEME[config.scheme], sampler=_lib.SAMPLER[config.sampler],
            precision=_lib.PRECISION[config.precision], want_greeks=int(want_greeks),
            n_steps=config.n_steps, n_runs=config.n_runs, n_paths=config.n_paths,
            path_lo=0, path_hi=config.n_paths, seed=config.seed & (2**64 - 1),
            h_spot=h_spot, v0_up=v_up, v0_dn=v_dn, h_r=h_r,
            sobol_scramble=int(bool(config.sobol_scramble)), sobol_bridge=config.sobol_bridge)
        self.sobol_host = None
        if config.sampler == "sobol":
            blocks = 1 if config.sobol_scramble else config.n_runs
            if 1 + blocks * config.n_paths > 2 ** sobol.BITS:
                raise UnsupportedProduct("sobol index range exceeds the 2^30-point sequence")
            self.sobol_host = sobol.directions(sobol_dimension(spec, config))
        self.n_runs = config.n_runs
        self.n_paths = config.n_paths
        self.want_greeks = want_greeks

    # -- device execution ------------------------------------------------
    def run_device(self, group=None):
        """Simulate this rank's slice, exchange chunk partials, reduce.
        Returns a host float64 array [n_runs, HMC_NW] (identical on all
        ranks).  Uses torch only for device buffers, the current stream and
        the process group."""
        import torch
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device visible; the engine has no CPU fallback")
        L = _lib.lib()
        dev = torch.device("cuda", torch.cuda.current_device())
        stream = torch.cuda.current_stream(dev)
        rank, world = parallel.world_info(group)
        sl = parallel.shard(self.n_paths, rank, world)
        keep = []
        if self.sobol_host is not None:
            v = _device_directions(self.sobol_host, dev)
            keep.append(v)
            self.sim.sobol_v = ctypes.cast(ctypes.c_void_p(v.data_ptr()), ctypes.POINTER(ctypes.c_uint32))
            self.sim.sobol_v_on_device = 1
        # every chunk of the slice is written by hmc_greeks_chunks
        local = torch.empty((self.n_runs, sl.n_chunks, _lib.HMC_NW), dtype=torch.float64, device=dev)
        if sl.n_paths > 0:
            self.sim.path_lo, self.sim.path_hi = sl.path_lo, sl.path_hi
            work = torch.empty(int(L.hmc_workspace_bytes(ctypes.byref(self.sim))),
                               dtype=torch.uint8, device=dev)
            _lib.check(L.hmc_greeks_chunks(ctypes.byref(self.model), ctypes.byref(self.product),
                                           ctypes.byref(self.sim), ctypes.c_void_p(local.data_ptr()),
                                           ctypes.c_void_p(work.data_ptr()),
                                           ctypes.c_void_p(stream.cuda_stream)))
            keep.append(work)
        full = parallel.gather_chunks(local, self.n_paths, group)
        out = torch.empty((self.n_runs, _lib.HMC_NW), dtype=torch.float64, device=dev)
        _lib.check(L.hmc_reduce_chunks(ctypes.c_void_p(full.data_ptr()), self.n_runs,
                                       full.shape[1], ctypes.c_void_p(out.data_ptr()),
                                       ctypes.c_void_p(stream.cuda_stream)))
        host = out.cpu().numpy()  # synchronises the stream
        del keep
        return host


def summarise(config: SimConfig, sums: np.ndarray, wall_ms: float,
              names=_QNAMES) -> dict[str, McSummary]:
    """Reference ``_summaries`` (``engine.py:128-139``) plus per-path SE.
    ``sums`` is [n_runs, HMC_NW] = {sum, sum of squares} per quantity."""
    N, R = config.n_paths, config.n_runs
    M = R * N
    if R == 1 and N > 1:
        # one run: the same values without the numpy reductions on 1-element
        # rows (np.mean of one value is that value; the run-level SD is 0)
        row = sums[0].tolist()
        out = {}
        for q, name in enumerate(names):
            s, ss = row[2 * q], row[2 * q + 1]
            v = s / N
            var = max(ss - s * s / M, 0.0) / (M - 1)
            out[name] = McSummary(estimate=v, std_error=0.0, per_run_values=[v], wall_ms=wall_ms,
                                  n_paths=N, n_runs=1, path_std_error=math.sqrt(var / M))
        return out
    # one row per quantity, contiguous: the row reductions are exactly the
    # reference's 1-D np.mean / np.std per quantity (engine.py:133-135)
    runs = np.ascontiguousarray(sums[:, 0::2].T) / N
    est = np.mean(runs, axis=1)
    sd = np.std(runs, axis=1, ddof=1) if R > 1 else np.zeros(len(names))
    s, ss = sums[:, 0::2].sum(axis=0), sums[:, 1::2].sum(axis=0)
    var = np.maximum(ss - s * s / M, 0.0) / (M - 1) if M > 1 else np.zeros(len(names))
    pse = np.sqrt(var / M)
    runs_l, est_l, sd_l, pse_l = runs.tolist(), est.tolist(), sd.tolist(), pse.tolist()
    return {name: McSummary(estimate=est_l[q], std_error=sd_l[q], per_run_values=runs_l[q],
                            wall_ms=wall_ms, n_paths=N, n_runs=R, path_std_error=pse_l[q])
            for q, name in enumerate(names)}


def _execute(params: HestonParams, spec: OptionSpec, config: SimConfig,
             want_greeks: bool, group=None) -> dict[str, McSummary]:
    t0 = time.perf_counter()
    if config.scheme == "exact":
        from . import exact
        _validate(spec, config, want_greeks)
        sums = exact.execute(params, spec, config, want_greeks,
                             bump_sizes(params, spec, config), group)
    else:
        sums = Job(params, spec, config, want_greeks).run_device(group)
    wall = (time.perf_counter() - t0) * 1000.0 / config.n_runs
    res = summarise(config, sums, wall)
    if not want_greeks:
        return {k: res[k] for k in ("price", "delta", "rho")}
    return res


def price(params: HestonParams, spec: OptionSpec, config: SimConfig) -> McSummary:
    """Discounted-payoff estimate: per-run path average, summarised over runs."""
    return _execute(params, spec, config, want_greeks=False)["price"]


def greeks(params: HestonParams, spec: OptionSpec, config: SimConfig) -> dict[str, McSummary]:
    """Price, pathwise Delta and Rho (reference keys) plus Gamma, Vega and the
    FD cross-checks delta_fd / rho_fd, all from ONE fused pass."""
    return _execute(params, spec, config, want_greeks=True)


def run_experiment(grid: list[SimConfig], params: HestonParams, spec: OptionSpec,
                   want_greeks: bool = False) -> list[dict]:
    """One row per configuration (reference ``engine.py:175-186``)."""
    rows = []
    for config in grid:
        res = _execute(params, spec, config, want_greeks)
        rows.append({"scheme": config.scheme, "sampler": config.sampler,
                     "paths": config.n_paths, "steps": config.n_steps,
                     "runs": config.n_runs, "summaries": res})
    return rows


def warm_up() -> None:
    """Create the CUDA context, load ``libhmc.so`` and launch one tiny job,
    so a fresh process (the CLI) does not book that one-time start-up as the
    ``wall_ms`` of its first timed run.  No-op without a CUDA device (the
    real call then raises :class:`DeviceError`)."""
    import torch
    if not torch.cuda.is_available():
        return
    from .model import BENCH_PARAMS
    price(HestonParams(**BENCH_PARAMS), OptionSpec("european", "call", 100.0, 1.0, 100.0),
          SimConfig(scheme="milstein", n_paths=128, n_steps=3, n_runs=1))
