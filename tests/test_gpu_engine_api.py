"""The reference engine's API-level tests (reference tests/test_engine.py:
46-117) on the GPU engine: Sobol acknowledgement and run blocks, summary
conventions, run_experiment rows."""

import numpy as np
import pytest

from paper_2309_10477_b200 import (ConfigInvalid, OptionSpec, SimConfig, UnsupportedProduct, greeks, price,
                                   run_experiment)
from paper_2309_10477_b200 import engine

pytestmark = pytest.mark.gpu


def cfg(**kw):
    base = dict(scheme="milstein", sampler="pseudo", n_paths=8192, n_steps=32, n_runs=3, seed=42)
    base.update(kw)
    return SimConfig(**base)


def test_sobol_discretised_needs_ack(params, euro_call):
    with pytest.raises(ConfigInvalid):
        cfg(sampler="sobol")
    s = price(params, euro_call, cfg(sampler="sobol", sobol_highdim_ack=True, n_paths=512, n_steps=8))
    assert s.estimate > 0.0


def test_sobol_dimension_accounting(params, euro_call, asian_call):
    assert engine.sobol_dimension(euro_call, cfg(scheme="exact")) == 3
    assert engine.sobol_dimension(asian_call, cfg(scheme="exact")) == 12
    assert engine.sobol_dimension(euro_call, cfg(sampler="sobol", sobol_highdim_ack=True, n_steps=16)) == 32


@pytest.mark.parametrize("scheme,steps", [("exact", 1), ("milstein", 16)])
def test_sobol_runs_use_distinct_blocks(params, euro_call, scheme, steps):
    s = price(params, euro_call, cfg(scheme=scheme, sampler="sobol", sobol_highdim_ack=True, n_paths=256,
                                     n_steps=steps, n_runs=4))
    assert len(set(s.per_run_values)) == 4


def test_summary_echoes_config(params, euro_call):
    s = price(params, euro_call, cfg(n_runs=5))
    assert s.n_runs == 5 and s.n_paths == 8192
    assert len(s.per_run_values) == 5
    assert s.estimate == pytest.approx(np.mean(s.per_run_values))
    assert s.std_error == pytest.approx(np.std(s.per_run_values, ddof=1))
    assert s.wall_ms > 0.0


def test_put_greeks_rejected(params):
    put = OptionSpec(style="european", right="put", strike=100.0, maturity=1.0, spot=100.0)
    with pytest.raises(UnsupportedProduct):
        greeks(params, put, cfg())


def test_run_experiment_empty_grid(params, euro_call):
    assert run_experiment([], params, euro_call) == []


def test_run_experiment_rows_echo_configs(params, euro_call):
    rows = run_experiment([cfg(n_paths=1000, n_runs=2), cfg(n_paths=2000, n_runs=2)], params, euro_call)
    assert [r["paths"] for r in rows] == [1000, 2000]
    assert all("price" in r["summaries"] for r in rows)


def test_run_experiment_paths_sweep_shrinks_spread(params, euro_call):
    rows = run_experiment([cfg(n_paths=n, n_steps=64, n_runs=20) for n in (2000, 32000)], params, euro_call)
    assert rows[1]["summaries"]["price"].std_error < rows[0]["summaries"]["price"].std_error


def test_run_experiment_greeks_rows(params, euro_call):
    rows = run_experiment([cfg(n_paths=4096)], params, euro_call, want_greeks=True)
    assert {"price", "delta", "rho", "gamma", "vega"} <= set(rows[0]["summaries"])


def test_schemes_agree_as_vol_of_vol_vanishes(euro_call):
    """reference tests/test_schemes.py:80-88: the Milstein correction is
    O(sigma^2), so on the same normals Euler and Milstein coincide as
    sigma -> 0 (fp32 path state: to ~1e-6 relative)."""
    from paper_2309_10477_b200 import DEFAULT_PARAMS, HestonParams
    p = HestonParams(**dict(DEFAULT_PARAMS, sigma=1e-6))
    e = price(p, euro_call, cfg(scheme="euler", n_paths=20_000, n_steps=64))
    m = price(p, euro_call, cfg(scheme="milstein", n_paths=20_000, n_steps=64))
    np.testing.assert_allclose(e.per_run_values, m.per_run_values, rtol=1e-5)


def test_variance_truncation_under_stress(euro_call):
    """reference tests/test_schemes.py:70-78: far outside the Feller
    condition the truncated variance keeps every path finite (fp32 kernel,
    Euler and Milstein, full Greeks)."""
    from paper_2309_10477_b200 import HestonParams
    p = HestonParams(kappa=0.5, theta=0.09, sigma=2.0, rho=-0.9, r=0.02, v0=0.09)
    for scheme in ("euler", "milstein"):
        g = greeks(p, euro_call, cfg(scheme=scheme, n_paths=20_000, n_steps=64))
        for q, s in g.items():
            assert np.all(np.isfinite(s.per_run_values)), (scheme, q)
        assert g["price"].estimate > 0.0
