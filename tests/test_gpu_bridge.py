"""Sobol Brownian-bridge ordering on the GPU (SimConfig.sobol_bridge).

* fp64: per-run Greeks equal the CPU restatement (oracle/bridge.py + the C
  oracle driven by the bridge normals) to ~1e-10 -- same points, same
  construction, same path arithmetic;
* fp32: the production kernel agrees with fp64 to fp32 accuracy (a wrong
  dimension, node or segment would move estimates by O(SE));
* statistics: unbiased, and a much smaller randomised-QMC spread than
  time-ordered Sobol at the same cost.
"""

import math

import numpy as np
import pytest

import oracle
from oracle import bridge
from oracle.semi_analytic import call_price
from paper_2309_10477_b200 import OptionSpec, SimConfig, daily_fixings, engine, greeks, price, sobol

pytestmark = pytest.mark.gpu

QN = ("price", "delta", "rho", "gamma", "vega", "delta_fd", "rho_fd")


def _oracle_runs(params, spec, cfg):
    avg = engine._validate(spec, cfg, True)
    n_sim = int(avg[-1])
    dt = spec.maturity / cfg.n_steps
    bumps = engine.bump_sizes(params, spec, cfg)
    out = np.zeros((cfg.n_runs, 7))
    for run in range(cfg.n_runs):
        key_run = oracle.derive_key(oracle.root_key(cfg.seed), run)
        if cfg.sobol_scramble:
            U = sobol.points(2 * cfg.n_steps, 1, cfg.n_paths, key_run=key_run)
        else:
            U = sobol.points(2 * cfg.n_steps, 1 + run * cfg.n_paths, cfg.n_paths)
        z = bridge.step_normals(U, cfg.sobol_bridge, n_sim, cfg.n_steps, dt, params.rho)
        q = oracle.greeks_paths_z(params, spec, cfg.n_steps, cfg.scheme == "milstein", z, avg, bumps)
        out[run] = q.mean(axis=0)
    return out


@pytest.mark.parametrize("style,n_steps,S,n_paths,scramble", [
    ("asian", 64, 16, 3000, False), ("asian", 40, 5, 2048, True),
    ("european", 64, 64, 1500, False), ("european", 33, 1, 777, True)])
def test_fp64_bridge_matches_oracle(bench_params, style, n_steps, S, n_paths, scramble):
    spec = (OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                       averaging_times=daily_fixings(1.0, n_steps)) if style == "asian"
            else OptionSpec("european", "call", 100.0, 1.0, 100.0))
    cfg = SimConfig(scheme="milstein", sampler="sobol", sobol_highdim_ack=True, n_paths=n_paths,
                    n_steps=n_steps, n_runs=2, seed=23, sobol_scramble=scramble, sobol_bridge=S,
                    precision="fp64")
    g = greeks(bench_params, spec, cfg)
    ref = _oracle_runs(bench_params, spec, cfg)
    for i, q in enumerate(QN):
        np.testing.assert_allclose(g[q].per_run_values, ref[:, i], rtol=1e-9, atol=1e-9, err_msg=q)


@pytest.mark.parametrize("n_paths,n_steps,S,scramble", [(4096, 252, 16, False), (5000, 100, 7, True),
                                                        (2048, 64, 64, True)])
def test_fp32_bridge_matches_fp64_bridge(bench_params, n_paths, n_steps, S, scramble):
    spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                      averaging_times=daily_fixings(1.0, n_steps))
    kw = dict(scheme="milstein", sampler="sobol", sobol_highdim_ack=True, n_paths=n_paths,
              n_steps=n_steps, n_runs=2, seed=31, sobol_scramble=scramble, sobol_bridge=S)
    a = greeks(bench_params, spec, SimConfig(**kw))
    b = greeks(bench_params, spec, SimConfig(precision="fp64", **kw))
    for q in ("price", "delta", "rho", "vega", "delta_fd", "rho_fd"):
        np.testing.assert_allclose(a[q].per_run_values, b[q].per_run_values, rtol=5e-5, atol=1e-6,
                                   err_msg=q)
    np.testing.assert_allclose(a["gamma"].per_run_values, b["gamma"].per_run_values, rtol=5e-3)
    # the European kernel variant (one fixing) as well
    e = OptionSpec("european", "call", 100.0, 1.0, 100.0)
    a = greeks(bench_params, e, SimConfig(**kw))
    b = greeks(bench_params, e, SimConfig(precision="fp64", **kw))
    np.testing.assert_allclose(a["price"].per_run_values, b["price"].per_run_values, rtol=3e-5)


def test_bridge_unbiased_and_tighter(bench_params):
    """Randomised QMC with bridge ordering: unbiased against the plain-MC
    estimate of the same discretisation, and a run spread well below
    time-ordered Sobol (the point of the ordering)."""
    e = OptionSpec("european", "call", 100.0, 1.0, 100.0)
    a = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 64))
    base = dict(scheme="milstein", sampler="sobol", sobol_highdim_ack=True, sobol_scramble=True,
                n_paths=2**14, n_steps=64, n_runs=32, seed=7)
    est = {}
    for spec in (e, a):
        br = price(bench_params, spec, SimConfig(sobol_bridge=16, **base))
        tord = price(bench_params, spec, SimConfig(**base))
        mc = price(bench_params, spec, SimConfig(scheme="milstein", n_paths=2**21, n_steps=64, n_runs=8,
                                                 seed=8))
        se_b = br.std_error / math.sqrt(br.n_runs)
        se_m = mc.std_error / math.sqrt(mc.n_runs)
        assert abs(br.estimate - mc.estimate) <= 4 * math.hypot(se_b, se_m), (spec.style, br.estimate,
                                                                            mc.estimate)
        assert br.std_error < 0.6 * tord.std_error, (spec.style, br.std_error, tord.std_error)
        est[spec.style] = br.estimate
    ref = call_price(100.0, 100.0, 1.0, bench_params.r, bench_params.kappa, bench_params.theta,
                     bench_params.sigma, bench_params.rho, bench_params.v0)
    assert abs(est["european"] - ref) < 0.05   # 64-step Milstein bias is a few cents at most
