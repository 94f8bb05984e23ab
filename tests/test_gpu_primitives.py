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
