"""GPU engine parity: the drop-in ``price`` / ``greeks`` / ``run_experiment``.

* fp64 replay precision: per-run values equal the reference engine's
  (golden, produced by the reference) to 1e-12 relative for price / Delta /
  Rho and to 1e-9 for the CRN finite differences (FD quotients amplify
  last-ulp differences by 1/h).
* fp32 production precision (Philox): independent-RNG estimates agree with
  the reference's within 3 combined standard errors (north star, check (b)),
  and European prices/Greeks with the Heston semi-analytic values and the
  Broadie-Kaya exact baseline (check (c)).
"""

import ctypes
import math

import numpy as np
import pytest

import oracle
from oracle import engine as oe
from oracle.semi_analytic import call_greeks
from conftest import spec_from
from paper_2309_10477_b200 import (BENCH_PARAMS, HestonParams, OptionSpec, SimConfig,
                                   UnsupportedProduct, daily_fixings, engine, greeks, price,
                                   run_experiment)

pytestmark = pytest.mark.gpu

QN = ("price", "delta", "rho", "gamma", "vega", "delta_fd", "rho_fd")


def _close_se(a, a_se, b, b_se, k=3.0, floor=0.0):
    return abs(a - b) <= k * math.hypot(a_se, b_se) + floor


class TestReplayPrecisionMatchesReferenceEngine:
    def test_per_run_values(self, golden_engine):
        for name, c in golden_engine.items():
            p, spec = HestonParams(**c["params"]), spec_from(c["spec"])
            cfg = SimConfig(precision="fp64", **c["config"])
            s = price(p, spec, cfg)
            np.testing.assert_allclose(s.per_run_values, c["price"], rtol=1e-12, err_msg=name)
            if "greeks_delta" not in c:
                continue
            b = c["bumps"]
            cfg = SimConfig(precision="fp64", bump_spot=b["h_spot"] / spec.spot,
                            bump_v0=(b["v0_up"] - p.v0) / p.v0, bump_r=b["h_r"], **c["config"])
            g = greeks(p, spec, cfg)
            np.testing.assert_allclose(g["price"].per_run_values, c["greeks_price"], rtol=1e-12)
            np.testing.assert_allclose(g["delta"].per_run_values, c["greeks_delta"], rtol=1e-12)
            np.testing.assert_allclose(g["rho"].per_run_values, c["greeks_rho"], rtol=1e-12)
            np.testing.assert_allclose(g["delta_fd"].per_run_values, c["fd_delta"], rtol=1e-9, atol=1e-10)
            np.testing.assert_allclose(g["rho_fd"].per_run_values, c["fd_rho"], rtol=1e-9, atol=1e-8)
            np.testing.assert_allclose(g["vega"].per_run_values, c["fd_vega"], rtol=1e-9, atol=1e-8)

    def test_gamma_vs_oracle_fd(self, bench_params, euro_call):
        cfg = SimConfig(scheme="milstein", n_paths=20000, n_steps=32, n_runs=2, seed=5,
                        precision="fp64")
        g = greeks(bench_params, euro_call, cfg)
        bumps = engine.bump_sizes(bench_params, euro_call, cfg)
        s = oe.greeks_sums(bench_params, euro_call, cfg, bumps, workers=8)
        for q, name in enumerate(QN):
            np.testing.assert_allclose(g[name].per_run_values, s[:, 2 * q] / cfg.n_paths,
                                       rtol=1e-9, atol=1e-9, err_msg=name)


class TestProductionPrecision:
    def test_full_size_vs_reference_statistics(self, golden_stats):
        """BASELINE params, 252 steps: fp32 Philox GPU at 2^22 paths vs the
        reference's 2^20-path per-path statistics (same discretisation,
        independent RNG) -- all seven quantities within 3 combined SE."""
        p = HestonParams(**golden_stats["params"])
        b = golden_stats["bumps"]
        specs = {
            "euro": OptionSpec("european", "call", 100.0, 1.0, 100.0),
            "asian_daily": OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                                      averaging_times=daily_fixings(1.0, 252)),
        }
        cfg = SimConfig(scheme="milstein", n_paths=2**22, n_steps=252, n_runs=1, seed=7,
                        bump_spot=b["h_spot"] / 100.0, bump_v0=(b["v0_up"] - p.v0) / p.v0,
                        bump_r=b["h_r"])
        for name, spec in specs.items():
            g = greeks(p, spec, cfg)
            for q in QN:
                ref, ref_se = golden_stats[name][q]
                assert _close_se(g[q].estimate, g[q].path_std_error, ref, ref_se), \
                    (name, q, g[q].estimate, g[q].path_std_error, ref, ref_se)

    def test_european_vs_semi_analytic(self):
        """Pooled over seeds 1-4 at 2^22 paths each (2^24 paths, 252 steps)."""
        p = HestonParams(**BENCH_PARAMS)
        spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
        gs = [greeks(p, spec, SimConfig(scheme="milstein", n_paths=2**22, n_steps=252, n_runs=1,
                                         seed=seed)) for seed in (1, 2, 3, 4)]
        sa = call_greeks(100.0, 100.0, 1.0, p.r, p.kappa, p.theta, p.sigma, p.rho, p.v0)
        for q in ("price", "delta", "rho", "gamma", "vega"):
            est = sum(g[q].estimate for g in gs) / 4
            se = math.sqrt(sum(g[q].path_std_error ** 2 for g in gs)) / 4
            # FD gamma/vega carry an O(h^2) bump bias and a small time-step bias: 4 SE
            k = 3.0 if q in ("price", "delta", "rho") else 4.0
            assert _close_se(est, se, sa[q], 0.0, k=k), (q, est, se, sa[q])

    def test_fp32_unbiased_vs_fp64_replay(self, bench_params, euro_call):
        """2^28 paths x 64 steps: the fp32 Philox path and the fp64 replay of
        the reference stream estimate the same discretised expectation."""
        res = {}
        for prec in ("fp32", "fp64"):
            res[prec] = price(bench_params, euro_call, SimConfig(
                scheme="milstein", n_paths=2**24, n_steps=64, n_runs=16, seed=123, precision=prec))
        a, b = res["fp32"], res["fp64"]
        assert _close_se(a.estimate, a.path_std_error, b.estimate, b.path_std_error), \
            (a.estimate, b.estimate)

    def test_headline_full_greeks_fp32_vs_fp64_replay(self, bench_params):
        """The headline configuration (Asian, 252 daily fixings) at 2^26 paths:
        all seven fp32 production estimates agree with the fp64 replay of the
        reference's own stream and arithmetic within 3 combined SE -- no fp32
        bias at the size of ~0.03 % of the price (independent streams, same
        discretised expectation)."""
        from paper_2309_10477_b200 import daily_fixings
        spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 252))
        res = {prec: greeks(bench_params, spec, SimConfig(scheme="milstein", n_paths=2**24, n_steps=252,
                                                         n_runs=4, seed=77, precision=prec))
               for prec in ("fp32", "fp64")}
        for q in QN:
            a, b = res["fp32"][q], res["fp64"][q]
            assert _close_se(a.estimate, a.path_std_error, b.estimate, b.path_std_error), (q, a.estimate, b.estimate)

    def test_european_vs_broadie_kaya(self, golden_stats):
        p = HestonParams(**golden_stats["params"])
        spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
        s = price(p, spec, SimConfig(scheme="milstein", n_paths=2**22, n_steps=252, n_runs=1, seed=3))
        bk, bk_se = golden_stats["bk_exact_euro"]["price"]
        assert _close_se(s.estimate, s.path_std_error, bk, bk_se)

    def test_paper_acceptance_values(self, params, euro_call, asian_call):
        """Reference acceptance criteria 3-5 (tests/test_acceptance.py:67-132)
        on the production path: Milstein 32k x 128 x 30 runs."""
        cfg = SimConfig(scheme="milstein", n_paths=32000, n_steps=128, n_runs=30, seed=42)
        g = greeks(params, euro_call, cfg)
        assert abs(g["price"].estimate - 6.8061) <= 0.15
        assert abs(g["delta"].estimate - 0.6958) <= 3 * g["delta"].std_error
        assert abs(g["rho"].estimate - 62.7752) <= 3 * g["rho"].std_error
        a = price(params, asian_call, cfg)
        assert abs(a.estimate - 4.3840) <= 0.15

    def test_timestep_plateau(self, params, euro_call):
        grid = [SimConfig(scheme="milstein", n_paths=32000, n_steps=n, n_runs=30, seed=42)
                for n in (32, 64, 128, 256)]
        rows = run_experiment(grid, params, euro_call)
        sums = {r["steps"]: r["summaries"]["price"] for r in rows}
        for a in sums:
            for b in sums:
                if a < b:
                    assert abs(sums[a].estimate - sums[b].estimate) <= \
                        3 * max(sums[a].std_error, sums[b].std_error)

    def test_black_scholes_limit(self, euro_call):
        # reference criterion 8 (tests/test_acceptance.py:196-212)
        from scipy.special import ndtr
        p = HestonParams(kappa=6.21, theta=0.019, sigma=1e-6, rho=-0.7, r=0.0319, v0=0.010201)
        tv = p.theta + (p.v0 - p.theta) * (1.0 - math.exp(-p.kappa)) / p.kappa
        sq = math.sqrt(tv)
        d1 = (math.log(1.0) + p.r + 0.5 * tv) / sq
        bs = 100 * ndtr(d1) - 100 * math.exp(-p.r) * ndtr(d1 - sq)
        for scheme in ("euler", "milstein"):
            s = price(p, euro_call, SimConfig(scheme=scheme, n_paths=100_000, n_steps=128,
                                               n_runs=10, seed=42))
            assert abs(s.estimate - bs) <= 3 * s.std_error, (scheme, s.estimate, bs)

    def test_put_call_parity(self, bench_params):
        call = OptionSpec("european", "call", 105.0, 1.0, 100.0)
        put = OptionSpec("european", "put", 105.0, 1.0, 100.0)
        cfg = SimConfig(scheme="milstein", n_paths=8000, n_steps=64, n_runs=10, seed=77)
        c, pt = price(bench_params, call, cfg), price(bench_params, put, cfg)
        diffs = np.array(c.per_run_values) - np.array(pt.per_run_values)
        target = 100.0 - 105.0 * math.exp(-bench_params.r)
        se = diffs.std(ddof=1) / math.sqrt(len(diffs))
        assert abs(diffs.mean() - target) < 3.0 * max(se, 1e-12)

    @pytest.mark.parametrize("spec_name", ["euro_call", "asian_call"])
    def test_pathwise_vs_fd_in_one_pass(self, params, spec_name, request):
        """delta vs delta_fd and rho vs rho_fd from the same fused pass
        (reference tests/test_products.py:101-125, CRN)."""
        spec = request.getfixturevalue(spec_name)
        g = greeks(params, spec, SimConfig(scheme="milstein", n_paths=8000, n_steps=64, n_runs=10,
                                           seed=77))
        for pw, fd, floor in (("delta", "delta_fd", 1e-4), ("rho", "rho_fd", 1e-2)):
            diff = np.array(g[pw].per_run_values) - np.array(g[fd].per_run_values)
            se = diff.std(ddof=1) / math.sqrt(len(diff))
            assert abs(diff.mean()) < 3.0 * max(se, floor), (pw, diff.mean(), se)

    def test_delta_to_discounted_forward_as_strike_vanishes(self, params):
        spec = OptionSpec("european", "call", 1e-6, 1.0, 100.0)
        g = greeks(params, spec, SimConfig(scheme="milstein", n_paths=20000, n_steps=64, n_runs=10,
                                           seed=42))
        d = g["delta"]
        assert abs(d.estimate - 1.0) < 3.0 * d.std_error / math.sqrt(d.n_runs)


class TestEngineContract:
    def test_deterministic_repeat(self, params, euro_call):
        cfg = SimConfig(scheme="milstein", n_paths=50000, n_steps=64, n_runs=3, seed=42)
        a, b = greeks(params, euro_call, cfg), greeks(params, euro_call, cfg)
        for q in QN:
            assert a[q].per_run_values == b[q].per_run_values

    def test_single_pass_greeks_match_price(self, params, euro_call, asian_call):
        # reference tests/test_engine.py:39-42
        for spec in (euro_call, asian_call):
            for prec in ("fp32", "fp64"):
                cfg = SimConfig(scheme="milstein", n_paths=8192, n_steps=32, n_runs=3, seed=42,
                                precision=prec)
                assert greeks(params, spec, cfg)["price"].per_run_values == \
                    price(params, spec, cfg).per_run_values

    def test_split_slices_bit_identical(self, bench_params):
        """Two chunk-aligned slices reduced together == the whole job: the
        property that makes multi-GPU results identical to 1-GPU results."""
        import torch
        from paper_2309_10477_b200 import _lib, parallel
        spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                          averaging_times=daily_fixings(1.0, 64))
        cfg = SimConfig(scheme="milstein", n_paths=5 * 16384 + 1000, n_steps=64, n_runs=2, seed=9)
        whole = engine.Job(bench_params, spec, cfg, True).run_device()
        L = _lib.lib()
        parts = []
        for rank in range(3):
            sl = parallel.shard(cfg.n_paths, rank, 3)
            job = engine.Job(bench_params, spec, cfg, True)
            job.sim.path_lo, job.sim.path_hi = sl.path_lo, sl.path_hi
            loc = torch.zeros((cfg.n_runs, sl.n_chunks, _lib.HMC_NW), dtype=torch.float64, device="cuda")
            work = torch.empty(L.hmc_workspace_bytes(ctypes.byref(job.sim)), dtype=torch.uint8, device="cuda")
            _lib.check(L.hmc_greeks_chunks(ctypes.byref(job.model), ctypes.byref(job.product),
                                           ctypes.byref(job.sim), ctypes.c_void_p(loc.data_ptr()),
                                           ctypes.c_void_p(work.data_ptr()), None))
            parts.append(loc)
        full = torch.cat(parts, dim=1).contiguous()
        out = torch.empty((cfg.n_runs, _lib.HMC_NW), dtype=torch.float64, device="cuda")
        _lib.check(L.hmc_reduce_chunks(ctypes.c_void_p(full.data_ptr()), cfg.n_runs, full.shape[1],
                                       ctypes.c_void_p(out.data_ptr()), None))
        np.testing.assert_array_equal(out.cpu().numpy(), whole)

    def test_c_abi_one_call_matches_engine(self, bench_params, euro_call):
        from paper_2309_10477_b200 import _lib
        cfg = SimConfig(scheme="milstein", n_paths=40000, n_steps=63, n_runs=2, seed=4)
        job = engine.Job(bench_params, euro_call, cfg, True)
        host = np.zeros((cfg.n_runs, _lib.HMC_NW))
        _lib.check(_lib.lib().hmc_greeks(ctypes.byref(job.model), ctypes.byref(job.product),
                                         ctypes.byref(job.sim),
                                         host.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 0))
        np.testing.assert_array_equal(host, job.run_device())

    def test_summary_fields(self, params, euro_call):
        s = price(params, euro_call, SimConfig(scheme="milstein", n_paths=8192, n_steps=32, n_runs=5,
                                               seed=42))
        assert s.n_runs == 5 and s.n_paths == 8192 and len(s.per_run_values) == 5
        assert s.estimate == pytest.approx(np.mean(s.per_run_values))
        assert s.std_error == pytest.approx(np.std(s.per_run_values, ddof=1))
        assert s.wall_ms > 0.0 and s.path_std_error > 0.0

    def test_se_scaling(self, params, euro_call):
        small = price(params, euro_call, SimConfig(scheme="milstein", n_paths=2000, n_steps=64,
                                                   n_runs=30, seed=21))
        large = price(params, euro_call, SimConfig(scheme="milstein", n_paths=8000, n_steps=64,
                                                   n_runs=30, seed=21))
        assert 0.35 < large.std_error / small.std_error < 0.65

    @pytest.mark.parametrize("n_paths,n_steps", [(1, 1), (2, 3), (127, 5), (129, 7),
                                                 (16385, 2), (100_000, 1)])
    def test_ragged_sizes_vs_fp64(self, bench_params, n_paths, n_steps):
        """Partial tiles / chunks and odd step counts (Philox tail): fp32
        agrees with the fp64 replay within 3 SE."""
        spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
        a = price(bench_params, spec, SimConfig(scheme="milstein", n_paths=n_paths, n_steps=n_steps,
                                                 n_runs=1, seed=1))
        b = price(bench_params, spec, SimConfig(scheme="milstein", n_paths=n_paths, n_steps=n_steps,
                                                 n_runs=1, seed=1, precision="fp64"))
        assert np.isfinite(a.estimate)
        if n_paths > 1000:
            assert _close_se(a.estimate, a.path_std_error, b.estimate, b.path_std_error)

    @pytest.mark.parametrize("over", [dict(v0=0.0), dict(rho=1.0), dict(rho=-1.0),
                                      dict(sigma=2.0, theta=0.01)])
    def test_edge_params_vs_oracle(self, over):
        p = HestonParams(**{**BENCH_PARAMS, **over})
        spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                          averaging_times=daily_fixings(1.0, 32))
        cfg = SimConfig(scheme="milstein", n_paths=2**17, n_steps=32, n_runs=1, seed=2)
        g = greeks(p, spec, cfg)
        s = oe.greeks_sums(p, spec, SimConfig(scheme="milstein", n_paths=2**15, n_steps=32, n_runs=1,
                                              seed=3), engine.bump_sizes(p, spec, cfg), workers=8)
        M = 2**15
        for q, name in enumerate(QN):
            mean = s[0, 2 * q] / M
            se = math.sqrt(max(s[0, 2 * q + 1] / M - mean * mean, 0.0) / (M - 1))
            assert np.isfinite(g[name].estimate)
            assert _close_se(g[name].estimate, g[name].path_std_error, mean, se, k=4.0, floor=1e-6), \
                (over, name, g[name].estimate, mean, se)


class TestSobol:
    def test_fp32_sobol_vs_reference_engine(self, golden_engine):
        c = golden_engine["paper_asian_sobol"]
        p, spec = HestonParams(**c["params"]), spec_from(c["spec"])
        cfg = SimConfig(**c["config"])
        g = greeks(p, spec, cfg)
        ref = np.array(c["greeks_price"])
        assert abs(g["price"].estimate - ref.mean()) < 0.05
        # fp32 and the reference consume the same Sobol points; only the
        # inverse normal and arithmetic precision differ
        np.testing.assert_allclose(g["price"].per_run_values, ref, rtol=2e-4)

    @pytest.mark.parametrize("n_paths,n_steps,scramble", [(1000, 16, False), (70001, 130, False),
                                                          (4096, 252, False), (3333, 65, True)])
    def test_fp32_sobol_matches_fp64_sobol(self, bench_params, n_paths, n_steps, scramble):
        """The shared-memory Gray-code generator of the fp32 kernel feeds the
        same points (and digital shifts) as the fp64 per-coordinate path:
        per-run Asian Greeks agree to fp32 accuracy (a wrong coordinate
        would move them by O(SE) ~ 1e-3)."""
        spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                          averaging_times=daily_fixings(1.0, n_steps))
        kw = dict(scheme="milstein", sampler="sobol", sobol_highdim_ack=True, n_paths=n_paths,
                  n_steps=n_steps, n_runs=3, seed=17, sobol_scramble=scramble)
        a = greeks(bench_params, spec, SimConfig(**kw))
        b = greeks(bench_params, spec, SimConfig(precision="fp64", **kw))
        # same points: every estimator to fp32 accuracy (FD Greeks included,
        # via the cancellation-free epilogue); Gamma is an indicator
        # difference, so one path flipping at a band edge moves it by O(1/N)
        for q in ("price", "delta", "rho", "vega", "delta_fd", "rho_fd"):
            np.testing.assert_allclose(a[q].per_run_values, b[q].per_run_values, rtol=3e-5, atol=1e-6,
                                       err_msg=q)
        np.testing.assert_allclose(a["gamma"].per_run_values, b["gamma"].per_run_values, rtol=5e-3,
                                   err_msg="gamma")

    def test_scrambled_sobol_finite_at_scale(self, bench_params):
        """Shifted coordinates can be exactly 0 (x == shift): the quantile
        must stay finite (2^21 points x 504 dimensions hits such cells)."""
        spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                          averaging_times=daily_fixings(1.0, 252))
        for prec in ("fp32", "fp64"):
            g = greeks(bench_params, spec, SimConfig(
                scheme="milstein", sampler="sobol", sobol_highdim_ack=True, sobol_scramble=True,
                n_paths=2**21, n_steps=252, n_runs=2, seed=2024, precision=prec))
            for q in QN:
                assert all(np.isfinite(g[q].per_run_values)), (prec, q)
            assert abs(g["price"].estimate - 5.238) < 0.02

    def test_scrambled_sobol_unbiased(self, bench_params):
        spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
        q = price(bench_params, spec, SimConfig(scheme="milstein", sampler="sobol", sobol_highdim_ack=True,
                                                 sobol_scramble=True, n_paths=2**16, n_steps=64,
                                                 n_runs=32, seed=5))
        ps = price(bench_params, spec, SimConfig(scheme="milstein", n_paths=2**20, n_steps=64, n_runs=8,
                                                 seed=5))
        se_q = q.std_error / math.sqrt(q.n_runs)
        se_p = ps.std_error / math.sqrt(ps.n_runs)
        assert _close_se(q.estimate, se_q, ps.estimate, se_p, k=4.0)
        # the randomised-QMC spread is below the plain-MC spread at equal paths
        mc = price(bench_params, spec, SimConfig(scheme="milstein", n_paths=2**16, n_steps=64,
                                                 n_runs=32, seed=6))
        assert q.std_error < mc.std_error

    def test_sobol_index_range_limit(self, params, euro_call):
        cfg = SimConfig(scheme="milstein", sampler="sobol", sobol_highdim_ack=True, n_paths=2**29,
                        n_steps=4, n_runs=3)
        with pytest.raises(UnsupportedProduct):
            price(params, euro_call, cfg)


class TestSobolQuantile:
    """The fp32 kernels' Sobol quantile (hmc_path32.cuh sobol_normal_u,
    Giles' erfinv on min(u, 1-u)) against scipy's ndtri on the exact 30-bit
    coordinates, both point conventions, including the extreme cells (the
    scrambled upper half uses 1 - u = (2^30 - x - 1/2) 2^-30) and the centre."""

    @pytest.mark.parametrize("scrambled", [0, 1])
    def test_against_ndtri(self, scrambled):
        from scipy.special import ndtri
        from paper_2309_10477_b200 import _lib
        rng = np.random.default_rng(11)
        lo = 0 if scrambled else 1
        x = np.concatenate([rng.integers(lo, 2**30, 400_000), np.arange(lo, lo + 2000),
                            2**30 - 1 - np.arange(2000), 2**29 + np.arange(-2000, 2000)]).astype(np.uint32)
        out = np.empty(x.size, dtype=np.float32)
        _lib.check(_lib.lib().hmc_sobol_quantile_check(
            x.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), x.size, scrambled,
            out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), 0))
        u = (x.astype(np.float64) + 0.5 * scrambled) * 2.0 ** -30
        ref = ndtri(u)
        err = np.abs(out.astype(np.float64) - ref) / np.maximum(1.0, np.abs(ref))
        # a few fp32 ulps of z everywhere, including the extreme cells
        assert err.max() < 1e-6, (err.max(), u[err.argmax()])
        # monotone in u (ties allowed at fp32 resolution)
        order = np.argsort(u, kind="stable")
        assert np.all(np.diff(out[order]) >= -1e-6)


class TestBoxMuller:
    """The production normals: hmc_box_muller_check runs the kernels'
    tri_unpack + box_muller_f on given Philox blocks."""

    @staticmethod
    def _device(words):
        from paper_2309_10477_b200 import _lib
        w = np.ascontiguousarray(words, dtype=np.uint32)
        out = np.empty((w.shape[0], 6), dtype=np.float32)
        _lib.check(_lib.lib().hmc_box_muller_check(w.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                                   w.shape[0], out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                                   0))
        return out.astype(np.float64)

    @staticmethod
    def _restated(w):
        """The documented bit layout (hmc_path32.cuh tri_unpack) in fp64."""
        w = w.astype(np.uint64)
        m32 = np.uint64(0xFFFFFFFF)
        f = lambda bits: (bits.astype(np.uint32).view(np.float32)).astype(np.float64)  # noqa: E731
        one = np.uint64(0x3F800000)
        fr = [f((w[:, k] >> np.uint64(9)) + one) for k in range(3)]
        fa = [f(((w[:, 3] >> np.uint64(9)) & np.uint64(0x007FFFF0)) | one),
              f((((w[:, 3] << np.uint64(10)) & m32) & np.uint64(0x007FFC00))
                | (((w[:, 0] << np.uint64(1)) & m32) & np.uint64(0x000003F0)) | one),
              f((((w[:, 1] << np.uint64(14)) & m32) & np.uint64(0x007FC000))
                | (((w[:, 2] << np.uint64(5)) & m32) & np.uint64(0x00003FE0)) | one)]
        out = np.empty((w.shape[0], 6))
        for k in range(3):
            r = np.sqrt(-2.0 * np.log(2.0 - fr[k]))
            th = 2.0 * np.pi * fa[k] - 3.0 * np.pi
            out[:, 2 * k], out[:, 2 * k + 1] = r * np.cos(th), r * np.sin(th)
        return out

    def test_bit_layout_known_answers(self):
        rng = np.random.default_rng(5)
        w = rng.integers(0, 2**32, size=(200_000, 4), dtype=np.uint64).astype(np.uint32)
        w[:4] = [[0, 0, 0, 0], [0xFFFFFFFF] * 4, [0x80000000, 1, 0x7FFFFFFF, 0xFFFF0000],
                 [0x00000200, 0x00000200, 0x00000200, 0x00001000]]
        got, ref = self._device(w), self._restated(w)
        err = np.abs(got - ref) / np.maximum(1.0, np.abs(ref))
        # MUFU.LG2's absolute error near 1 dominates the radius when u1 -> 1
        # (R = sqrt(-2 ln u1) < 0.01, probability ~5e-5 per draw): absolute
        # error there up to ~2e-4 in z; a few fp32 ulps everywhere else
        r2 = ref[:, 0::2] ** 2 + ref[:, 1::2] ** 2
        small = np.repeat(r2 < 1e-4, 2, axis=1)
        assert err[~small].max() < 5e-6, err[~small].max()
        assert np.abs(got - ref)[small].max(initial=0.0) < 3e-4

    def test_production_stream_is_standard_normal(self):
        """Philox4x32-10 blocks on production counters (step triple, path,
        key_run) through the device transform: 6e6 normals with N(0, 1)
        moments, no correlation within a block, KS against the normal CDF."""
        import oracle
        from scipy import stats
        from paper_2309_10477_b200 import _lib
        n = 1_000_000
        key = oracle.derive_key(oracle.root_key(42), 0)
        ctr = np.zeros((n, 4), dtype=np.uint32)
        ctr[:, 0] = np.arange(n) % 84
        ctr[:, 1] = np.arange(n) // 84
        ctr[:, 2], ctr[:, 3] = key & 0xFFFFFFFF, key >> 32
        words = np.empty_like(ctr)
        _lib.check(_lib.lib().hmc_philox_check(ctr.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), n,
                                               words.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), 0))
        z = self._device(words)
        flat = z.ravel()
        m = flat.size
        assert abs(flat.mean()) < 5 / math.sqrt(m)
        assert abs(flat.var() - 1.0) < 5 * math.sqrt(2.0 / m)
        assert abs(stats.skew(flat)) < 5 * math.sqrt(6.0 / m)
        assert abs(stats.kurtosis(flat)) < 5 * math.sqrt(24.0 / m)
        c = np.corrcoef(z.T)
        assert np.max(np.abs(c - np.eye(6))) < 5 / math.sqrt(n)
        assert stats.kstest(flat[:2_000_000], "norm").pvalue > 1e-4


class TestFp32PathsKnownAnswer:
    """The production fp32 step arithmetic (regrouped Milstein update, r-free
    log2 price ratio, fixing-weight table, CRN trajectories, fp32 epilogue)
    against the fp64 oracle (the reference's operation order, CRN
    re-simulation of every bump) on IDENTICAL normals -- RNG-free parity of
    the kernel math, path by path."""

    @pytest.mark.parametrize("style,n_steps,dates", [("european", 252, None), ("asian", 252, "daily"),
                                                     ("asian", 64, (0.25, 0.5, 0.75, 1.0))])
    def test_against_oracle(self, bench_params, style, n_steps, dates):
        from paper_2309_10477_b200 import _lib
        if style == "european":
            spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
        else:
            at = daily_fixings(1.0, n_steps) if dates == "daily" else dates
            spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=at)
        cfg = SimConfig(scheme="milstein", n_paths=4096, n_steps=n_steps, n_runs=1, seed=1)
        job = engine.Job(bench_params, spec, cfg, True)
        n, n_sim = 4096, int(job.avg_idx[-1])
        rng = np.random.default_rng(17)
        z = rng.standard_normal((n, n_sim, 2)).astype(np.float32)
        got = np.empty((n, 7))
        _lib.check(_lib.lib().hmc_fp32_paths_check(
            ctypes.byref(job.model), ctypes.byref(job.product), ctypes.byref(job.sim),
            z.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), n, got.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            0))
        p = bench_params
        zz = np.zeros((n, 2 * n_steps))
        z1 = z[:, :, 0].astype(np.float64)
        zz[:, 0:2 * n_sim:2] = z1
        zz[:, 1:2 * n_sim:2] = p.rho * z1 + math.sqrt(1 - p.rho ** 2) * z[:, :, 1].astype(np.float64)
        ref = oracle.greeks_paths_z(p, spec, n_steps, True, zz, job.avg_idx,
                                    engine.bump_sizes(p, spec, cfg))
        # per path: price within fp32 accumulation error of A (~1e-6 relative)
        assert np.max(np.abs(got[:, 0] - ref[:, 0])) < 2e-3
        # pathwise Delta / Rho, away from the strike where the indicator can flip
        far = np.abs(ref[:, 0]) > 0.05
        for c in (1, 2):
            np.testing.assert_allclose(got[far, c], ref[far, c], rtol=1e-4, atol=1e-4)
        # the cancellation-free FD forms: FD Delta / FD Rho means to 2e-5
        for c in (5, 6):
            assert abs(got[:, c].mean() - ref[:, c].mean()) <= 2e-5 * abs(ref[:, c].mean()), c
        # every estimator's mean (what the engine reports) agrees closely
        for c in range(7):
            assert abs(got[:, c].mean() - ref[:, c].mean()) <= 2e-4 * max(1.0, abs(ref[:, c].mean())) + \
                3 * ref[:, c].std() / math.sqrt(n) * 0.05, (c, got[:, c].mean(), ref[:, c].mean())


@pytest.mark.parametrize("over,scheme", [(dict(v0=0.0), "milstein"), (dict(rho=1.0), "milstein"),
                                         (dict(rho=-1.0), "milstein"), (dict(sigma=2.0, theta=0.01), "milstein"),
                                         (dict(kappa=0.05, sigma=0.9), "milstein"), ({}, "euler"),
                                         (dict(sigma=2.0, theta=0.01), "euler")])
def test_fp32_paths_known_answer_edge_params(over, scheme):
    """Same normals, edge regimes (v0 = 0 one-sided bump, perfect
    correlation, frequent truncation at v = 0, slow mean reversion): the
    fp32 arithmetic stays within fp32 accuracy of the fp64 oracle."""
    from paper_2309_10477_b200 import _lib
    p = HestonParams(**{**BENCH_PARAMS, **over})
    spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 64))
    cfg = SimConfig(scheme=scheme, n_paths=8192, n_steps=64, n_runs=1, seed=1)
    job = engine.Job(p, spec, cfg, True)
    n = 8192
    z = np.random.default_rng(23).standard_normal((n, 64, 2)).astype(np.float32)
    got = np.empty((n, 7))
    _lib.check(_lib.lib().hmc_fp32_paths_check(
        ctypes.byref(job.model), ctypes.byref(job.product), ctypes.byref(job.sim),
        z.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), n, got.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 0))
    zz = np.zeros((n, 128))
    zz[:, 0::2] = z[:, :, 0]
    zz[:, 1::2] = p.rho * z[:, :, 0].astype(np.float64) + math.sqrt(max(1 - p.rho ** 2, 0.0)) * z[:, :, 1]
    ref = oracle.greeks_paths_z(p, spec, 64, scheme == "milstein", zz, job.avg_idx,
                                engine.bump_sizes(p, spec, cfg))
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got[:, 0] - ref[:, 0])) < 2e-3
    for c in range(7):
        if c == 3:   # Gamma: indicator difference, compare at O(1/N)
            assert abs(got[:, c].mean() - ref[:, c].mean()) <= 2.0 / n * np.abs(ref[:, 1]).max() / 0.5 + 1e-6
            continue
        assert abs(got[:, c].mean() - ref[:, c].mean()) <= 1e-4 * max(1.0, abs(ref[:, c].mean())), \
            (over, c, got[:, c].mean(), ref[:, c].mean())


def test_path_standard_error_is_calibrated(bench_params):
    """The per-path standard error (from fp64 sums of squares) predicts the
    spread of independent estimates: 24 seeds x 2^18 paths, Asian daily
    fixings, all seven estimators (SD ratio within the chi-square band)."""
    spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 64))
    est = {q: [] for q in QN}
    se = {q: [] for q in QN}
    for seed in range(100, 124):
        g = greeks(bench_params, spec, SimConfig(scheme="milstein", n_paths=2**18, n_steps=64, n_runs=1,
                                                 seed=seed))
        for q in QN:
            est[q].append(g[q].estimate)
            se[q].append(g[q].path_std_error)
    for q in QN:
        ratio = np.std(est[q], ddof=1) / np.mean(se[q])
        assert 0.6 < ratio < 1.45, (q, ratio)


class TestManyRuns:
    """Runs map to gridDim.y; beyond 65 535 they go out in launch batches
    with a run offset (KernelArgs.run0).  The reference engine has no run
    limit (engine.py:151); its per-run values are checked at the batch
    boundary against the oracle's restatement of ``_run_sums``."""

    def test_runs_past_grid_y_limit(self, bench_params, euro_call):
        cfg = SimConfig(scheme="milstein", n_paths=32, n_steps=4, n_runs=65537, seed=3,
                        precision="fp64")
        s = price(bench_params, euro_call, cfg)
        assert len(s.per_run_values) == 65537
        for run in (0, 65534, 65535, 65536):
            want = oe.run_sums(bench_params, euro_call, cfg, run, None, False, "port")[0] / cfg.n_paths
            assert math.isclose(s.per_run_values[run], want, rel_tol=1e-12), run
        # fp32 production path: the batch boundary changes nothing either
        f = greeks(bench_params, euro_call, SimConfig(scheme="milstein", n_paths=32, n_steps=4,
                                                       n_runs=65537, seed=3))
        g = greeks(bench_params, euro_call, SimConfig(scheme="milstein", n_paths=32, n_steps=4,
                                                       n_runs=3, seed=3))
        assert f["vega"].per_run_values[:3] == g["vega"].per_run_values
        assert len(set(f["price"].per_run_values[65530:])) == 7
