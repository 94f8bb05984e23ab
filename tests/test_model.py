"""Drop-in types: same validation contract as the reference's dataclasses
(reference tests/test_products.py:68-82, tests/test_engine.py:109-120,
tests/test_schemes.py:159-169)."""

import pytest

from paper_2309_10477_b200 import (ConfigInvalid, GridSpec, HestonParams, InvalidParams,
                                   OptionSpec, SimConfig, UnsupportedProduct, ValidationError,
                                   averaging_indices, daily_fixings, engine, sobol_dimension)


class TestHestonParams:
    @pytest.mark.parametrize("field", ["kappa", "theta", "sigma"])
    def test_positive(self, field):
        kw = dict(kappa=1.0, theta=0.04, sigma=0.3, rho=0.0, r=0.0, v0=0.04)
        kw[field] = 0.0
        with pytest.raises(InvalidParams):
            HestonParams(**kw)

    def test_rho_and_v0(self):
        with pytest.raises(InvalidParams):
            HestonParams(1.0, 0.04, 0.3, 1.5, 0.0, 0.04)
        with pytest.raises(InvalidParams):
            HestonParams(1.0, 0.04, 0.3, 0.0, 0.0, -1e-9)
        assert HestonParams(2.0, 0.04, 0.3, -0.7, 0.03, 0.04).dof == pytest.approx(3.5555555)


class TestOptionSpec:
    def test_asian_needs_dates(self):
        with pytest.raises(ValidationError):
            OptionSpec(style="asian_arithmetic", right="call", strike=100.0, maturity=1.0, spot=100.0)

    def test_dates_must_increase(self):
        with pytest.raises(ValidationError):
            OptionSpec(style="asian_arithmetic", right="call", strike=100.0, maturity=1.0,
                       spot=100.0, averaging_times=(0.5, 0.25))

    def test_dates_within_maturity(self):
        with pytest.raises(ValidationError):
            OptionSpec(style="asian_arithmetic", right="call", strike=100.0, maturity=1.0,
                       spot=100.0, averaging_times=(0.5, 1.5))

    def test_european_rejects_dates(self):
        with pytest.raises(ValidationError):
            OptionSpec(style="european", right="call", strike=100.0, maturity=1.0, spot=100.0,
                       averaging_times=(0.5,))

    def test_bad_style_right(self):
        with pytest.raises(ValidationError):
            OptionSpec(style="bermudan", right="call", strike=1.0, maturity=1.0, spot=1.0)
        with pytest.raises(ValidationError):
            OptionSpec(style="european", right="straddle", strike=1.0, maturity=1.0, spot=1.0)


class TestGrid:
    def test_index_of(self):
        g = GridSpec(maturity=1.0, n_steps=252)
        assert averaging_indices(g, daily_fixings(1.0, 252)) == list(range(1, 253))
        with pytest.raises(ValidationError):
            g.index_of(0.3001)
        with pytest.raises(ValidationError):
            GridSpec(maturity=1.0, n_steps=0)


class TestSimConfig:
    def test_sobol_discretised_needs_ack(self):
        with pytest.raises(ConfigInvalid):
            SimConfig(scheme="milstein", sampler="sobol")
        SimConfig(scheme="milstein", sampler="sobol", sobol_highdim_ack=True)

    @pytest.mark.parametrize("kw", [dict(scheme="heun"), dict(sampler="halton"), dict(n_paths=0),
                                    dict(n_steps=0), dict(n_runs=0), dict(max_parallelism=0),
                                    dict(max_parallelism="many"), dict(precision="fp16"),
                                    dict(bump_v0=0.0)])
    def test_rejected(self, kw):
        with pytest.raises(ConfigInvalid):
            SimConfig(**kw)

    def test_defaults_match_reference(self):
        c = SimConfig()
        assert (c.scheme, c.sampler, c.n_paths, c.n_steps, c.n_runs, c.seed) == \
            ("exact", "pseudo", 2048, 128, 30, 0)
        assert c.precision == "fp32"

    def test_sobol_dimension_accounting(self, euro_call, asian_call):
        # reference tests/test_engine.py:54-59
        assert sobol_dimension(euro_call, SimConfig(scheme="exact")) == 3
        assert sobol_dimension(asian_call, SimConfig(scheme="exact")) == 12
        assert sobol_dimension(euro_call, SimConfig(scheme="milstein", sampler="sobol",
                                                    sobol_highdim_ack=True, n_steps=16)) == 32


class TestEngineValidation:
    """Host-side checks that run before any device work."""

    def test_put_greeks_rejected(self, params):
        put = OptionSpec(style="european", right="put", strike=100.0, maturity=1.0, spot=100.0)
        with pytest.raises(UnsupportedProduct):
            engine.greeks(params, put, SimConfig(scheme="milstein"))


    def test_off_grid_asian_date_rejected(self, params):
        spec = OptionSpec(style="asian_arithmetic", right="call", strike=100.0, maturity=1.0,
                          spot=100.0, averaging_times=(0.3,))
        with pytest.raises(ValidationError):
            engine.price(params, spec, SimConfig(scheme="milstein", n_steps=16))

    def test_bump_sizes(self, params, euro_call):
        h, up, dn, hr = engine.bump_sizes(params, euro_call, SimConfig())
        assert h == pytest.approx(0.5) and hr == 1e-4
        assert up - params.v0 == pytest.approx(0.01 * params.v0)
        assert params.v0 - dn == pytest.approx(0.01 * params.v0)
        p0 = HestonParams(params.kappa, params.theta, params.sigma, params.rho, params.r, 0.0)
        _, up, dn, _ = engine.bump_sizes(p0, euro_call, SimConfig())
        assert dn == 0.0 and up > 0.0


class TestSurfaceValidation:
    """Rejected on the host before any device work."""

    def test_bad_grids(self, params):
        from paper_2309_10477_b200 import surface
        cfg = SimConfig(scheme="milstein", n_steps=64, n_paths=1024, n_runs=1)
        with pytest.raises(ValidationError):
            surface(params, [100.0, 90.0], [0.5, 1.0], cfg)
        with pytest.raises(ValidationError):
            surface(params, [90.0, 100.0], [0.3, 1.0], cfg)      # off the dt = 1/64 grid
        with pytest.raises(ValidationError):
            surface(params, list(range(1, 200)), [1.0], cfg)     # > 128 strikes
        with pytest.raises(UnsupportedProduct):
            surface(params, [100.0], [1.0], SimConfig(scheme="exact", n_steps=1))
        with pytest.raises(UnsupportedProduct):
            surface(params, [100.0], [1.0], SimConfig(scheme="milstein", precision="fp64"))
