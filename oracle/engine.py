"""CPU restatement of the reference engine orchestration -- TEST
INFRASTRUCTURE / CPU BASELINE ONLY.

Follows ``hestonmc/engine.py:71-160`` step for step: per run the key
``derive_key(root_key(seed), run)`` (``:96``), the Sobol block starting at
``1 + run * n_paths`` (``:97-101``), 4096-path jobs (``:27,102-103``) on a
thread pool (``:147``), per-path statistics (``:47-68``) summed per job with
numpy's pairwise sum (``:110``) and combined with ``math.fsum`` in job order
(``:116``).  The per-path kernel is either the reference's own compiled
``_core`` (``oracle/_ref``, kind "reference") or the C restatement
(``oracle/hmc_oracle.c``, kind "port").

``greeks_sums`` extends it to the seven Greeks quantities with per-path sums
of squares (for standard errors), using the reference's CRN re-simulation
method for the bumped quantities.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import QUANTITIES, discretised_batch, greeks_paths, ref_core

CHUNK = 4096  # engine.py:27


def _kernel(kind: str):
    if kind == "reference":
        core = ref_core()
        if core is None:
            raise RuntimeError("oracle/_ref not built (make -C oracle on the build host)")
        return core.discretised_batch
    return discretised_batch


def avg_indices(spec, n_steps: int) -> np.ndarray:
    if spec.is_asian:
        return np.array([round(t * n_steps / spec.maturity) for t in spec.averaging_times],
                        dtype=np.int64)
    return np.array([n_steps], dtype=np.int64)


def per_path_stats(spec, obs: np.ndarray, r: float, want_greeks: bool) -> np.ndarray:
    """engine._per_path_stats (engine.py:47-68)."""
    disc = math.exp(-r * spec.maturity)
    s = obs[:, 1] if spec.is_asian else obs[:, 0]
    out = np.zeros((obs.shape[0], 3))
    if spec.right == "call":
        out[:, 0] = disc * np.maximum(s - spec.strike, 0.0)
    else:
        out[:, 0] = disc * np.maximum(spec.strike - s, 0.0)
    if want_greeks:
        itm = s > spec.strike
        out[:, 1] = np.where(itm, disc * s / spec.spot, 0.0)
        if spec.is_asian:
            out[:, 2] = np.where(itm, disc * (obs[:, 2] - spec.maturity * (s - spec.strike)), 0.0)
        else:
            out[:, 2] = np.where(itm, disc * spec.strike * spec.maturity, 0.0)
    return out


def _sobol_block(dim: int, start: int, count: int) -> np.ndarray:
    from scipy.stats import qmc  # rng.sobol_points (rng.py:143-152)
    eng = qmc.Sobol(d=dim, scramble=False)
    if start > 0:
        eng.fast_forward(start)
    return eng.random(count)


def run_sums(params, spec, config, run: int, pool, want_greeks: bool, kind: str) -> list[float]:
    """engine._run_sums (engine.py:93-116)."""
    from . import derive_key, root_key
    kernel = _kernel(kind)
    key_run = derive_key(root_key(config.seed), run)
    uniforms = None
    if config.sampler == "sobol":
        uniforms = _sobol_block(2 * config.n_steps, 1 + run * config.n_paths, config.n_paths)
    avg = avg_indices(spec, config.n_steps)
    bounds = list(range(0, config.n_paths, CHUNK)) + [config.n_paths]
    jobs = [(lo, hi) for lo, hi in zip(bounds, bounds[1:]) if hi > lo]

    def work(job):
        lo, hi = job
        u = None if uniforms is None else uniforms[lo:hi]
        obs = kernel(params, spec.spot, spec.maturity, config.n_steps,
                     config.scheme == "milstein", lo, hi, key_run, u, avg)
        return per_path_stats(spec, obs, params.r, want_greeks).sum(axis=0)

    partials = list(pool.map(work, jobs)) if pool is not None else [work(j) for j in jobs]
    return [math.fsum(p[k] for p in partials) for k in range(3)]


def per_run_values(params, spec, config, want_greeks: bool, kind: str = "port",
                   workers: int = 1) -> np.ndarray:
    """[n_runs, 3] per-run estimates of (price, delta, rho), engine.py:151-156."""
    pool = ThreadPoolExecutor(workers) if workers > 1 else None
    try:
        runs = np.empty((config.n_runs, 3))
        for run in range(config.n_runs):
            sums = run_sums(params, spec, config, run, pool, want_greeks, kind)
            runs[run] = [s / config.n_paths for s in sums]
    finally:
        if pool is not None:
            pool.shutdown()
    return runs


def greeks_sums(params, spec, config, bumps, want_greeks: bool = True, workers: int = 1,
                path_range: tuple[int, int] | None = None) -> np.ndarray:
    """[n_runs, 14] {sum, sum of squares} of the seven per-path quantities
    (``oracle.QUANTITIES``) over paths [lo, hi) (default all), computed by the
    C restatement with CRN re-simulation of every bump."""
    from . import derive_key, root_key
    lo_all, hi_all = path_range or (0, config.n_paths)
    avg = avg_indices(spec, config.n_steps)
    out = np.zeros((config.n_runs, 2 * len(QUANTITIES)))
    pool = ThreadPoolExecutor(workers) if workers > 1 else None
    try:
        for run in range(config.n_runs):
            key_run = derive_key(root_key(config.seed), run)
            uniforms = None
            if config.sampler == "sobol":
                uniforms = _sobol_block(2 * config.n_steps, 1 + run * config.n_paths + lo_all,
                                        hi_all - lo_all)
            bounds = list(range(lo_all, hi_all, CHUNK)) + [hi_all]
            jobs = [(lo, hi) for lo, hi in zip(bounds, bounds[1:]) if hi > lo]

            def work(job):
                lo, hi = job
                u = None if uniforms is None else uniforms[lo - lo_all:hi - lo_all]
                q = greeks_paths(params, spec, config.n_steps, config.scheme == "milstein",
                                 lo, hi, key_run, u, avg, bumps, want_greeks)
                return np.concatenate([q.sum(axis=0), (q * q).sum(axis=0)])
            parts = list(pool.map(work, jobs)) if pool is not None else [work(j) for j in jobs]
            tot = np.array([math.fsum(p[k] for p in parts) for k in range(2 * len(QUANTITIES))])
            nq = len(QUANTITIES)
            out[run, 0::2] = tot[:nq]
            out[run, 1::2] = tot[nq:]
    finally:
        if pool is not None:
            pool.shutdown()
    return out
