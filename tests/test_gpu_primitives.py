"""The drop-in's rng / schemes modules on the device primitives, against
vectors the reference itself produced (tests/golden/make_golden.py):

* ``uniform_at`` / ``uniforms_at`` (``hmc_uniforms_f64``): bit-identical to
  the reference's SplitMix64 draws (integer work);
* ``inverse_normal_cdf`` (``hmc_ndtri_f64``): the reference's Acklam + Halley
  values to 1e-15 relative (CUDA's erfc/exp vs glibc's, last ulp);
* ``gamma_batch`` / ``sample_gamma`` (``hmc_gamma_f64``): the reference's
  Marsaglia-Tsang draws to 1e-13 relative, and the stream left at the same
  position;
* ``euler_step`` / ``milstein_step`` (``hmc_steps_f64``): the reference's
  scalar steps to 1e-13 relative, truncation at v = 0 exact;
* ``simulate_path``: equal to the reference backend kernel on the same draws.
"""

import math

import numpy as np
import pytest

from conftest import load_json
from paper_2309_10477_b200 import rng, schemes
from paper_2309_10477_b200.errors import BesselNonConvergence, InvalidParams
from paper_2309_10477_b200.model import GridSpec, HestonParams, BENCH_PARAMS

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def test_keys_and_draws_bit_exact(golden_rng):
    for seed, k in golden_rng["keys"].items():
        rk = rng.root_key(int(seed))
        assert str(rk) == k["root"]
        assert [str(rng.derive_key(rk, i)) for i in (0, 1, 2, 1000, 2**40)] == k["derived"]
    key = int(golden_rng["path_key"])
    draws = [rng.uniform_at(key, i) for i in range(16)] + list(rng.uniforms_at(key, 1000, 8))
    assert draws == golden_rng["draws"]
    # vector forms agree with the scalar form
    keys = rng.derive_keys(np.uint64(rng.root_key(3)), np.arange(50, dtype=np.uint64))
    assert [str(k) for k in keys] == [str(rng.derive_key(rng.root_key(3), i)) for i in range(50)]
    ctr = np.arange(50, dtype=np.uint64) % 7
    assert rng._uniform_keys(keys, ctr).tolist() == [rng.uniform_at(int(k), int(c)) for k, c in zip(keys, ctr)]
    assert rng.mix64(12345) == rng.root_key(12345 ^ 0x8CB92BA72F3D8DD7)


def test_inverse_normal_matches_reference(golden_rng):
    got = rng.inverse_normal_cdf(np.array(golden_rng["ndtri_u"]))
    want = np.array(golden_rng["ndtri_x"])
    assert _rel(got, want) <= 1e-15
    assert rng.inverse_normal_cdf(0.5) == 0.0
    assert isinstance(rng.inverse_normal_cdf(0.3), float)


def test_gamma_matches_reference():
    g = load_json("primitive_cases.json")
    keys = np.array([int(k) for k in g["gamma_keys"]], dtype=np.uint64)
    for tag, want in g["gamma"].items():
        shape, scale = (float(x) for x in tag.split("_"))
        assert _rel(rng.gamma_batch(keys, shape, scale), want) <= 1e-13, tag
    m = g["gamma_mid_stream"]
    st = rng.UniformStream(seed=m["seed"], stream_index=m["stream_index"])
    for _ in range(m["skip"]):
        st.next_uniform()
    assert _rel(rng.sample_gamma(st, 0.634, 2.0), m["value"]) <= 1e-13
    assert st.next_uniform() == m["next_draw"]       # same number of draws consumed


def test_steps_match_reference():
    g = load_json("primitive_cases.json")
    for c in g["steps"]:
        p = HestonParams(**c["params"])
        for name, fn in (("euler", schemes.euler_step), ("milstein", schemes.milstein_step)):
            class _Fixed(rng.UniformStream):
                def __init__(self, values):
                    super().__init__(kind="pseudo", seed=0)
                    self._v, self._i = list(values), 0

                def next_uniform(self):
                    u = self._v[self._i]
                    self._i += 1
                    return u
            out = fn(_Fixed(c["u"]), p, schemes.PathState(c["s"], c["v"], 0.0), c["dt"])
            s_want, v_want = c[name]
            assert _rel(out.s, s_want) <= 1e-13, (name, c)
            if v_want == 0.0:
                assert out.v == 0.0
            else:
                assert _rel(out.v, v_want) <= 1e-13, (name, c)
            assert out.t == c["dt"]


@pytest.mark.parametrize("scheme", ["euler", "milstein"])
def test_simulate_path_equals_backend_on_same_draws(scheme):
    from paper_2309_10477_b200 import cuda_backend
    p = HestonParams(**BENCH_PARAMS)
    grid = GridSpec(maturity=1.0, n_steps=32)
    dates = (0.25, 0.5, 0.75, 1.0)
    obs = schemes.simulate_path(rng.UniformStream(seed=4, stream_index=9), p, grid, scheme, 100.0, dates)
    u = rng.uniforms_at(rng.stream_key(4, 9), 0, 64).reshape(1, 64)
    ref = cuda_backend.discretised_batch(p, 100.0, 1.0, 32, scheme == "milstein", 0, 1, 0, u,
                                         np.array([8, 16, 24, 32]))
    assert (obs.s_T, obs.avg, obs.tw_sum) == tuple(ref[0])
    # stepping by hand gives the same terminal value
    st, state = rng.UniformStream(seed=4, stream_index=9), schemes.PathState(100.0, p.v0, 0.0)
    step = schemes.milstein_step if scheme == "milstein" else schemes.euler_step
    for _ in range(32):
        state = step(st, p, state, grid.dt)
    assert math.isclose(state.s, obs.s_T, rel_tol=1e-14)


# ---------------------------------------------------------------------------
# The exact scheme's host modules on the device (bessel / ivlaw / exact):
# the same routines the exact kernel runs (csrc/hmc_exact.cu), checked here
# against scipy and against the exact kernel itself.  The reference's own
# test_bessel / test_ivlaw / test_exact modules also run unmodified in
# tests/test_gpu_reference_suite.py.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("nu", [-0.3658, 0.0, 1.5])
def test_bessel_i_matches_scipy(nu):
    from scipy.special import iv
    from paper_2309_10477_b200 import bessel
    for z in (0.05, 1.0, 7.5, 30.0, 49.0):
        ours = bessel.bessel_i(nu, complex(z, 0.0))
        assert abs(ours.imag) <= 1e-10 * abs(iv(nu, z))
        assert _rel(ours.real, float(iv(nu, z))) <= 1e-10
    with pytest.raises(BesselNonConvergence):
        bessel.bessel_i_series(nu, 50.5 + 0j)
    vec = bessel.bessel_i_series_vec(nu, np.array([0.1 + 0.2j, 3 - 4j, 20 + 1j]))
    for z, v in zip((0.1 + 0.2j, 3 - 4j, 20 + 1j), vec):
        assert v == bessel.bessel_i_series(nu, z)


def test_ivlaw_round_trip_and_exact_kernel_draw():
    """inverse_cdf(u) satisfies |F(x) - u| < 1e-6, and it is the value the
    exact kernel draws for the same (v_u, v_t, dt, u): one exact step on
    given draws (hmc_exact_step_f64) reports the same integrated variance."""
    from paper_2309_10477_b200 import exact, ivlaw
    p = HestonParams(**BENCH_PARAMS)
    law = ivlaw.IntegratedVarianceLaw(p, 0.04, 0.03, 0.25)
    assert law.mean > 0.0 and law.std > 0.0 and not law.is_degenerate
    for u in (1e-6, 0.02, 0.5, 0.98, 1 - 1e-6):
        x = law.inverse_cdf(u)
        assert abs(law.cdf_raw(x) - u) < 1e-6
    # the step's v_t is c (g + (z1 + sqrt(lambda))^2); choose draws giving v_t = 0.03
    c, lam = exact.nccs_coefficients(p, 0.25, 0.04)
    g = 0.03 / c - (0.3 + math.sqrt(lam)) ** 2
    out = exact._device_step(p, True, 100.0, 0.04, 0.25, [0.3, g, 0.37, -0.2])
    assert _rel(out[1], 0.03) <= 1e-14
    law2 = ivlaw.IntegratedVarianceLaw(p, 0.04, out[1], 0.25)
    assert _rel(out[2], law2.inverse_cdf(0.37)) <= 1e-14


def test_exact_step_draw_budget():
    from paper_2309_10477_b200 import exact
    p = HestonParams(**BENCH_PARAMS)
    main, gam = rng.UniformStream(seed=5), rng.UniformStream(seed=5, stream_index=1)
    res = exact.exact_step(main, p, 100.0, 0.04, 0.5, gamma_stream=gam)
    assert main._counter == 3 and gam._counter > 0
    assert res.s_t > 0.0 and res.v_t >= 0.0 and res.integrated_variance > 0.0
    with pytest.raises(InvalidParams):
        exact.exact_step(rng.UniformStream(seed=5), p, 0.0, 0.04, 0.5)
