"""Broadie-Kaya exact scheme behind the engine API.

``SimConfig(scheme="exact")`` -- the reference's DEFAULT scheme -- runs the
reference's exact simulation (``_core.pyx:415-521``) on the GPU
(``csrc/hmc_exact.cu``: same stream, same algorithm, fp64; per-path
observables match the reference to ~1e-15) and then follows the
reference engine's own per-run procedure (``engine.py:71-116``): step
endpoints from ``exact_step_times`` (one step per averaging interval for
Asians, one [0, T] step for Europeans), 4096-path jobs, numpy pairwise job
sums and an exactly rounded ``math.fsum`` across jobs -- so per-run values
reproduce the reference engine's.

Greeks beyond the reference's pathwise Delta/Rho: the S0 bump (and the r
bump of a European) is an exact rescaling of the simulated path (ln S
starts at ln S0 and accumulates r dt); the v0 bumps and the Asian r bumps
re-run the exact kernel on the same streams (common random numbers) -- the
reference's own finite-difference method (tests/test_products.py:101-137).
"""

from __future__ import annotations

import math

import numpy as np

from . import cuda_backend, parallel, sobol
from .model import HestonParams, OptionSpec, SimConfig

CHUNK = 4096  # reference engine.py:27


def exact_step_times(spec: OptionSpec) -> np.ndarray:
    """reference ``engine.py:32-37``"""
    if spec.is_asian:
        return np.concatenate([[0.0], np.asarray(spec.averaging_times, dtype=np.float64)])
    return np.array([0.0, spec.maturity])


def _per_path(spec: OptionSpec, params: HestonParams, obs, obs_u, obs_d, obs_rp, obs_rm, bumps,
              want_greeks: bool) -> np.ndarray:
    """(n, 7) per-path [price, delta, rho, gamma, vega, delta_fd, rho_fd];
    columns 0-2 are the reference's _per_path_stats (engine.py:47-68)."""
    T, K, S0, r = spec.maturity, spec.strike, spec.spot, params.r
    disc = math.exp(-r * T)
    A = obs[:, 1] if spec.is_asian else obs[:, 0]
    q = np.zeros((obs.shape[0], 7))
    q[:, 0] = disc * np.maximum(A - K, 0.0) if spec.right == "call" else disc * np.maximum(K - A, 0.0)
    if not want_greeks:
        return q
    itm = A > K
    q[:, 1] = np.where(itm, disc * A / S0, 0.0)
    q[:, 2] = np.where(itm, disc * (obs[:, 2] - T * (A - K)), 0.0) if spec.is_asian \
        else np.where(itm, disc * K * T, 0.0)
    h_spot, v_up, v_dn, h_r = bumps
    pay = lambda x, d: d * np.maximum(x - K, 0.0)  # noqa: E731
    up, dn = A * ((S0 + h_spot) / S0), A * ((S0 - h_spot) / S0)
    q[:, 3] = ((up > K).astype(float) - (dn > K)) * (disc * A / S0) / (2 * h_spot)
    q[:, 5] = (pay(up, disc) - pay(dn, disc)) / (2 * h_spot)
    Au = obs_u[:, 1] if spec.is_asian else obs_u[:, 0]
    Ad = obs_d[:, 1] if spec.is_asian else obs_d[:, 0]
    q[:, 4] = (pay(Au, disc) - pay(Ad, disc)) / (v_up - v_dn)
    # r +- h: European S_T scales by e^{+-h T} exactly; the Asian average
    # comes from the r-bumped re-simulations (same streams)
    if spec.is_asian:
        Rp, Rm = obs_rp[:, 1], obs_rm[:, 1]
    else:
        Rp, Rm = A * math.exp(h_r * T), A * math.exp(-h_r * T)
    q[:, 6] = (pay(Rp, math.exp(-(r + h_r) * T)) - pay(Rm, math.exp(-(r - h_r) * T))) / (2 * h_r)
    return q


def execute(params: HestonParams, spec: OptionSpec, config: SimConfig, want_greeks: bool,
            bumps, group=None) -> np.ndarray:
    """[n_runs, 14] {sum, sum of squares} per quantity; this rank's
    reference-chunk partials are all-gathered so every rank returns the
    same, reference-ordered sums."""
    times = exact_step_times(spec)
    n_steps = times.size - 1
    flags = np.ones(n_steps, dtype=np.int64) if spec.is_asian else np.array([1], dtype=np.int64)
    rank, world = parallel.world_info(group)
    sl = parallel.shard(config.n_paths, rank, world)
    bounds = list(range(0, config.n_paths, CHUNK)) + [config.n_paths]
    jobs = [(lo, hi) for lo, hi in zip(bounds, bounds[1:]) if sl.path_lo <= lo < sl.path_hi]
    p_up = HestonParams(params.kappa, params.theta, params.sigma, params.rho, params.r, bumps[1])
    p_dn = HestonParams(params.kappa, params.theta, params.sigma, params.rho, params.r, bumps[2])
    p_rp = HestonParams(params.kappa, params.theta, params.sigma, params.rho, params.r + bumps[3],
                        params.v0)
    p_rm = HestonParams(params.kappa, params.theta, params.sigma, params.rho, params.r - bumps[3],
                        params.v0)
    from . import _lib
    key_root = _lib.lib().hmc_root_key(config.seed & (2**64 - 1))
    out = np.zeros((config.n_runs, 14))
    variants = [params]
    if want_greeks:
        variants += [p_up, p_dn] + ([p_rp, p_rm] if spec.is_asian else [])
    # runs go to the GPU in batches (one launch per model variant and batch);
    # a batch is bounded so the host buffers stay ~<= 256 MB
    per_run_bytes = max(sl.n_paths, 1) * 8 * 3 * len(variants)
    batch = max(1, min(config.n_runs, (256 << 20) // per_run_bytes))
    # Sobol points (engine.py:97-101) are generated on the device from the
    # direction numbers -- the same points as sobol.points on the host
    sob = None
    if config.sampler == "sobol":
        sob = (sobol.directions(3 * n_steps), bool(config.sobol_scramble), config.n_paths)
    for r0 in range(0, config.n_runs, batch):
        runs = range(r0, min(config.n_runs, r0 + batch))
        key_runs = [_lib.lib().hmc_derive_key(key_root, run) for run in runs]
        obs = [None] * len(variants)
        if sl.n_paths > 0:
            obs = [cuda_backend.exact_runs(v, spec.spot, times, flags, sl.path_lo, sl.path_hi,
                                           key_runs, None, sobol=sob) for v in variants]
        for b, run in enumerate(runs):
            partials = np.zeros((len(jobs), 14))
            if sl.n_paths > 0:
                o = [x[b] for x in obs]
                base = o[0]
                obs_u, obs_d = (o[1], o[2]) if want_greeks else (base, base)
                obs_rp, obs_rm = (o[3], o[4]) if want_greeks and spec.is_asian else (base, base)
                q = _per_path(spec, params, base, obs_u, obs_d, obs_rp, obs_rm, bumps, want_greeks)
                for i, (lo, hi) in enumerate(jobs):
                    blk = q[lo - sl.path_lo:hi - sl.path_lo]
                    partials[i, 0::2] = blk.sum(axis=0)          # numpy pairwise, engine.py:110
                    partials[i, 1::2] = (blk * blk).sum(axis=0)
            if world > 1:
                partials = _gather_rows(partials, config.n_paths, group)
            for c in range(14):
                out[run, c] = math.fsum(partials[:, c])           # engine.py:116
    return out


def _gather_rows(local: np.ndarray, n_paths: int, group) -> np.ndarray:
    import torch
    import torch.distributed as dist
    # NCCL exchanges device tensors; a gloo group (CPU tests) host tensors
    dev = (torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl"
           else torch.device("cpu"))
    world = dist.get_world_size(group)
    counts = []
    for r in range(world):
        s = parallel.shard(n_paths, r, world)
        counts.append(len([lo for lo in range(0, n_paths, CHUNK) if s.path_lo <= lo < s.path_hi]))
    width = max(counts)
    send = torch.zeros((width, 14), dtype=torch.float64, device=dev)
    send[: local.shape[0]] = torch.from_numpy(local).to(dev)
    recv = torch.empty((world * width, 14), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    recv = recv.view(world, width, 14).cpu().numpy()
    return np.concatenate([recv[r, : counts[r]] for r in range(world)])
