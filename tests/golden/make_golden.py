"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (the reference tree is not on the GPU box):

    make -C oracle                      # builds oracle/_ref/_core*.so
    python tests/golden/make_golden.py [--stats]

The reference package is imported from /root/reference/pkg/src with its
compiled kernel (the oracle/_ref build of the reference's own _core.c)
registered as ``hestonmc._core``, i.e. exactly the reference's default
"compiled" backend.  Nothing here is product code.

Outputs
  replay_cases.npz     per-path (s_T, avg, tw_sum) of discretised_batch
  engine_cases.json    engine.price / engine.greeks per-run values, plus the
                       reference's CRN finite differences on bumped inputs
  rng_cases.json       key derivation, uniform draws, inverse normal
  sobol_points.npz     rng.sobol_points rows
  primitive_cases.json rng.gamma_batch / sample_gamma, schemes.euler_step /
                       milstein_step on fixed inputs
  stats_golden.json    (--stats) large-N reference statistics with per-path
                       SE: Milstein Euro/Asian price, Delta, Rho, FD Gamma,
                       FD Vega, FD Rho at BASELINE params, and the
                       Broadie-Kaya exact European price
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"


def load_reference():
    sys.path.insert(0, ROOT)
    import oracle
    core = oracle.ref_core()
    if core is None:
        raise SystemExit("build the reference kernel first: make -C oracle")
    sys.modules["hestonmc._core"] = core
    sys.path.insert(0, REF_SRC)
    import hestonmc
    from hestonmc import backend
    assert backend.BACKEND_NAME == "compiled", backend.BACKEND_NAME
    return hestonmc, core


BENCH = dict(kappa=2.0, theta=0.04, sigma=0.3, rho=-0.7, r=0.03, v0=0.04)


def replay_cases(hm, core):
    from hestonmc.model import DEFAULT_PARAMS, HestonParams
    from hestonmc.rng import derive_key, root_key, sobol_points
    rng = np.random.default_rng(20230918)
    kr = lambda seed, run=0: int(derive_key(root_key(seed), run))  # noqa: E731
    daily = np.arange(1, 253, dtype=np.int64)
    cases = {
        # name: (params, s0, T, n_steps, milstein, lo, hi, key_run, uniforms, avg)
        "paper_mil_32": (DEFAULT_PARAMS, 100.0, 1.0, 32, True, 0, 256, kr(42), None,
                         np.array([8, 16, 24, 32])),
        "paper_eul_32": (DEFAULT_PARAMS, 100.0, 1.0, 32, False, 0, 256, kr(42), None,
                         np.array([8, 16, 24, 32])),
        "bench_euro_252": (BENCH, 100.0, 1.0, 252, True, 1000, 1512, kr(42), None,
                           np.array([252])),
        "bench_asian_daily": (BENCH, 100.0, 1.0, 252, True, 0, 256, kr(7, 3), None, daily),
        "bench_euler_daily": (BENCH, 90.0, 2.0, 252, False, 4096, 4352, kr(7, 1), None, daily),
        "stress_trunc": (dict(kappa=2.0, theta=0.01, sigma=2.0, rho=-0.5, r=0.0, v0=1e-6),
                         100.0, 1.0, 128, True, 0, 256, kr(99), None, np.array([128])),
        "rho_plus_one": ({**BENCH, "rho": 1.0}, 100.0, 1.0, 16, True, 0, 128, kr(5), None,
                         np.array([16])),
        "rho_minus_one": ({**BENCH, "rho": -1.0}, 100.0, 1.0, 16, True, 0, 128, kr(5), None,
                          np.array([16])),
        "one_step": (BENCH, 100.0, 1.0, 1, True, 0, 128, kr(1), None, np.array([1])),
        "v0_zero": ({**BENCH, "v0": 0.0}, 100.0, 0.5, 64, True, 0, 128, kr(3), None,
                    np.array([16, 32, 64])),
    }
    u = rng.random((128, 64))
    u[0, :4] = [0.0, 1.0 - 1e-17, 1e-310, 0.5]   # clamp paths of ndtri
    u[1, :4] = [0.02425, 0.97575, 0.0242499, 0.9757501]  # branch edges
    cases["uniforms_random"] = (BENCH, 100.0, 1.0, 32, True, 0, 128, kr(42), u,
                                np.array([8, 16, 24, 32]))
    s = sobol_points(2 * 16, 1, 256)
    cases["uniforms_sobol"] = (DEFAULT_PARAMS, 100.0, 1.0, 16, True, 0, 256, kr(42), s,
                               np.array([16]))
    out = {}
    meta = {}
    for name, (p, s0, T, n, mil, lo, hi, k, uu, avg) in cases.items():
        hp = HestonParams(**p)
        res = core.discretised_batch(hp, s0, T, n, mil, lo, hi, k, uu, avg.astype(np.int64))
        out[f"{name}__out"] = res
        out[f"{name}__avg"] = avg.astype(np.int64)
        if uu is not None:
            out[f"{name}__uniforms"] = uu
        meta[name] = dict(params=p, s0=s0, T=T, n_steps=n, milstein=mil, path_lo=lo,
                          path_hi=hi, key_run=str(k), has_uniforms=uu is not None)
    out["__meta__"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "replay_cases.npz"), **out)
    print(f"replay_cases.npz: {len(cases)} cases")


def exact_cases(hm, core):
    """Reference exact_batch (Broadie-Kaya) outputs (_core.pyx:415-521)."""
    from hestonmc.model import DEFAULT_PARAMS, HestonParams
    from hestonmc.rng import derive_key, root_key, sobol_points
    kr = lambda seed, run=0: int(derive_key(root_key(seed), run))  # noqa: E731
    cases = {
        "paper_euro_1": (DEFAULT_PARAMS, 100.0, [0.0, 1.0], [1], 0, 96, kr(42), None),
        "paper_asian_4": (DEFAULT_PARAMS, 100.0, [0.0, 0.25, 0.5, 0.75, 1.0], [1, 1, 1, 1], 5, 69,
                          kr(7, 2), None),
        "bench_euro_1": (BENCH, 100.0, [0.0, 1.0], [1], 1000, 1064, kr(3), None),
        "bench_half_2": (BENCH, 95.0, [0.0, 0.25, 0.5], [0, 1], 0, 64, kr(11), None),
        "paper_sobol_1": (DEFAULT_PARAMS, 100.0, [0.0, 1.0], [1], 0, 64, kr(42),
                          sobol_points(3, 1, 64)),
    }
    out, meta = {}, {}
    for name, (p, s0, times, flags, lo, hi, k, uu) in cases.items():
        res = core.exact_batch(HestonParams(**p), s0, np.array(times), np.array(flags, dtype=np.int64),
                               lo, hi, k, uu)
        out[f"{name}__out"] = res
        if uu is not None:
            out[f"{name}__uniforms"] = uu
        meta[name] = dict(params=p, s0=s0, times=times, flags=flags, path_lo=lo, path_hi=hi,
                          key_run=str(k), has_uniforms=uu is not None)
    out["__meta__"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "exact_cases.npz"), **out)
    print(f"exact_cases.npz: {len(cases)} cases")


def _bump_spot(spec, h):
    from hestonmc.model import OptionSpec
    return OptionSpec(style=spec.style, right=spec.right, strike=spec.strike,
                      maturity=spec.maturity, spot=spec.spot + h,
                      averaging_times=spec.averaging_times)


def _bump(params, **kw):
    from hestonmc.model import HestonParams
    d = dict(kappa=params.kappa, theta=params.theta, sigma=params.sigma, rho=params.rho,
             r=params.r, v0=params.v0)
    for k, v in kw.items():
        d[k] = d[k] + v
    return HestonParams(**d)


def engine_cases(hm):
    from hestonmc import engine
    from hestonmc.model import DEFAULT_PARAMS, HestonParams, OptionSpec, SimConfig
    paper = HestonParams(**DEFAULT_PARAMS)
    bench = HestonParams(**BENCH)
    euro = OptionSpec(style="european", right="call", strike=100.0, maturity=1.0, spot=100.0)
    asian4 = OptionSpec(style="asian_arithmetic", right="call", strike=100.0, maturity=1.0,
                        spot=100.0, averaging_times=(0.25, 0.5, 0.75, 1.0))
    daily = OptionSpec(style="asian_arithmetic", right="call", strike=100.0, maturity=1.0,
                       spot=100.0, averaging_times=tuple(k / 64 for k in range(1, 65)))
    put = OptionSpec(style="european", right="put", strike=95.0, maturity=1.0, spot=100.0)
    cases = [
        ("paper_euro_mil", paper, euro, dict(scheme="milstein", n_paths=8192, n_steps=32, n_runs=3, seed=42)),
        ("paper_asian_mil", paper, asian4, dict(scheme="milstein", n_paths=5000, n_steps=32, n_runs=2, seed=42)),
        ("bench_euro_euler", bench, euro, dict(scheme="euler", n_paths=20000, n_steps=64, n_runs=2, seed=7)),
        ("bench_daily_mil", bench, daily, dict(scheme="milstein", n_paths=4096, n_steps=64, n_runs=1, seed=11)),
        ("paper_euro_sobol", paper, euro, dict(scheme="milstein", sampler="sobol", sobol_highdim_ack=True,
                                               n_paths=512, n_steps=8, n_runs=2, seed=3)),
        ("paper_asian_sobol", paper, asian4, dict(scheme="milstein", sampler="sobol", sobol_highdim_ack=True,
                                                  n_paths=1000, n_steps=16, n_runs=3, seed=3)),
        ("bench_put_price", bench, put, dict(scheme="milstein", n_paths=3000, n_steps=32, n_runs=2, seed=5)),
        # Broadie-Kaya exact scheme (the reference's default), cf. tests/test_backends.py:63-71
        ("paper_euro_exact_sobol", paper, euro, dict(scheme="exact", sampler="sobol", n_paths=256,
                                                     n_steps=1, n_runs=2, seed=3)),
        ("paper_euro_exact", paper, euro, dict(scheme="exact", n_paths=5000, n_steps=1, n_runs=2, seed=42)),
        ("paper_asian_exact", paper, asian4, dict(scheme="exact", sampler="sobol", n_paths=700,
                                                  n_steps=4, n_runs=2, seed=42)),
    ]
    h_s, h_r, h_v = 0.005, 1e-4, 0.01
    out = {}
    for name, p, spec, kw in cases:
        cfg = SimConfig(**kw)
        row = {"config": kw, "params": dict(kappa=p.kappa, theta=p.theta, sigma=p.sigma, rho=p.rho,
                                            r=p.r, v0=p.v0),
               "spec": dict(style=spec.style, right=spec.right, strike=spec.strike,
                            maturity=spec.maturity, spot=spec.spot,
                            averaging_times=list(spec.averaging_times))}
        row["price"] = engine.price(p, spec, cfg).per_run_values
        if spec.right == "call":
            g = engine.greeks(p, spec, cfg)
            for k in ("price", "delta", "rho"):
                row[f"greeks_{k}"] = g[k].per_run_values
            # the reference's own CRN finite differences (test_products.py:101-137)
            h = h_s * spec.spot
            up = engine.price(p, _bump_spot(spec, +h), cfg).per_run_values
            dn = engine.price(p, _bump_spot(spec, -h), cfg).per_run_values
            row["fd_delta"] = [(a - b) / (2 * h) for a, b in zip(up, dn)]
            up = engine.price(_bump(p, r=+h_r), spec, cfg).per_run_values
            dn = engine.price(_bump(p, r=-h_r), spec, cfg).per_run_values
            row["fd_rho"] = [(a - b) / (2 * h_r) for a, b in zip(up, dn)]
            hv = h_v * p.v0
            up = engine.price(_bump(p, v0=+hv), spec, cfg).per_run_values
            dn = engine.price(_bump(p, v0=-hv), spec, cfg).per_run_values
            row["fd_vega"] = [(a - b) / (2 * hv) for a, b in zip(up, dn)]
            row["bumps"] = dict(h_spot=h, h_r=h_r, v0_up=p.v0 + hv, v0_dn=p.v0 - hv)
        out[name] = row
    with open(os.path.join(HERE, "engine_cases.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(f"engine_cases.json: {len(out)} cases")


def rng_cases(hm):
    from hestonmc.rng import derive_key, inverse_normal_cdf, root_key, uniform_at, uniforms_at
    keys = {}
    for seed in (0, 1, 42, 2**63 + 5):
        rk = root_key(seed)
        keys[str(seed)] = {"root": str(rk), "derived": [str(derive_key(rk, i)) for i in (0, 1, 2, 1000, 2**40)]}
    k = derive_key(derive_key(derive_key(root_key(42), 0), 17), 0)
    draws = [uniform_at(k, i) for i in range(16)] + list(uniforms_at(k, 1000, 8))
    us = [1e-300, 1e-20, 1e-9, 0.001, 0.02425, 0.024249999, 0.1, 0.3, 0.5, 0.7, 0.97575,
          0.975750001, 0.999, 1 - 1e-9, 1 - 1e-16, 0.0, 1.0]
    out = {"keys": keys, "path_key": str(k), "draws": draws,
           "ndtri_u": us, "ndtri_x": [float(x) for x in inverse_normal_cdf(np.array(us))]}
    with open(os.path.join(HERE, "rng_cases.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("rng_cases.json")


def primitive_cases(hm):
    """Reference rng.gamma_batch / sample_gamma and schemes.euler_step /
    milstein_step on fixed inputs (the drop-in's device primitives
    hmc_gamma_f64 / hmc_steps_f64 are checked against these)."""
    from hestonmc.model import DEFAULT_PARAMS, HestonParams
    from hestonmc.rng import UniformStream, gamma_batch, sample_gamma, stream_key
    from hestonmc.schemes import PathState, euler_step, milstein_step
    keys = [stream_key(41, i) for i in range(64)]
    gam = {}
    for shape, scale in ((0.634, 2.0), (2.0, 2.0), (0.05, 1.0), (7.5, 0.5)):
        gam[f"{shape}_{scale}"] = [float(x) for x in gamma_batch(np.array(keys, dtype=np.uint64), shape, scale)]
    # scalar sampler from a stream that already consumed 3 draws
    st = UniformStream(seed=5, stream_index=2)
    for _ in range(3):
        st.next_uniform()
    g_mid = sample_gamma(st, 0.634, 2.0)
    after = st.next_uniform()

    class _Fixed(UniformStream):
        def __init__(self, values):
            super().__init__(kind="pseudo", seed=0)
            self._v, self._i = list(values), 0

        def next_uniform(self):
            u = self._v[self._i % len(self._v)]
            self._i += 1
            return u

    rng = np.random.default_rng(7)
    steps = []
    for pset in (DEFAULT_PARAMS, BENCH, {**BENCH, "rho": 1.0}, {**BENCH, "theta": 0.001, "sigma": 1.5}):
        p = HestonParams(**pset)
        for _ in range(8):
            s0, v0 = float(rng.uniform(50, 150)), float(rng.choice([0.0, rng.uniform(0, 0.2)]))
            u = [float(x) for x in rng.random(2)]
            dt = float(rng.choice([1 / 252, 0.125, 0.5]))
            e = euler_step(_Fixed(u), p, PathState(s0, v0, 0.0), dt)
            m = milstein_step(_Fixed(u), p, PathState(s0, v0, 0.0), dt)
            steps.append({"params": pset, "s": s0, "v": v0, "u": u, "dt": dt,
                          "euler": [e.s, e.v], "milstein": [m.s, m.v]})
    out = {"gamma_keys": [str(k) for k in keys], "gamma": gam,
           "gamma_mid_stream": {"seed": 5, "stream_index": 2, "skip": 3, "value": g_mid, "next_draw": after},
           "steps": steps}
    with open(os.path.join(HERE, "primitive_cases.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("primitive_cases.json")


def sobol_cases(hm):
    from hestonmc.rng import sobol_points
    out = {"d504_0": sobol_points(504, 0, 64), "d504_far": sobol_points(504, 3 * 2**20 + 1, 64),
           "d2_1": sobol_points(2, 1, 1024)}
    np.savez_compressed(os.path.join(HERE, "sobol_points.npz"), **out)
    print("sobol_points.npz")


def _per_path(spec, obs, r, S0):
    """engine._per_path_stats restated for arrays of observables."""
    disc = math.exp(-r * spec.maturity)
    s = obs[:, 1] if spec.is_asian else obs[:, 0]
    price = disc * np.maximum(s - spec.strike, 0.0)
    itm = s > spec.strike
    delta = np.where(itm, disc * s / S0, 0.0)
    if spec.is_asian:
        rho = np.where(itm, disc * (obs[:, 2] - spec.maturity * (s - spec.strike)), 0.0)
    else:
        rho = np.where(itm, disc * spec.strike * spec.maturity, 0.0)
    return price, delta, rho


def stats_golden(hm, core, n_paths=2**20, seed=42, workers=None):
    """Per-path reference statistics at BASELINE params."""
    from hestonmc.model import HestonParams, OptionSpec
    from hestonmc.rng import derive_key, root_key
    workers = workers or os.cpu_count()
    p = HestonParams(**BENCH)
    n_steps, T = 252, 1.0
    kr = int(derive_key(root_key(seed), 0))
    specs = {
        "euro": OptionSpec(style="european", right="call", strike=100.0, maturity=T, spot=100.0),
        "asian_daily": OptionSpec(style="asian_arithmetic", right="call", strike=100.0, maturity=T,
                                  spot=100.0, averaging_times=tuple(k / 252 for k in range(1, 253))),
    }
    h_s, h_r, h_v = 0.5, 1e-4, 0.01 * p.v0
    res = {"params": BENCH, "n_paths": n_paths, "n_steps": n_steps, "seed": seed,
           "bumps": dict(h_spot=h_s, h_r=h_r, v0_up=p.v0 + h_v, v0_dn=p.v0 - h_v),
           "workers": workers, "cpu_count": os.cpu_count()}
    chunk = 4096
    jobs = [(lo, min(lo + chunk, n_paths)) for lo in range(0, n_paths, chunk)]
    with ThreadPoolExecutor(workers) as pool:
        for name, spec in specs.items():
            avg = np.arange(1, 253, dtype=np.int64) if spec.is_asian else np.array([252], dtype=np.int64)

            def sim(prm, s0):
                parts = pool.map(lambda j: core.discretised_batch(prm, s0, T, n_steps, True, j[0], j[1],
                                                                  kr, None, avg), jobs)
                return np.concatenate(list(parts))
            t0 = time.time()
            base = sim(p, 100.0)
            t_base = time.time() - t0
            price, delta, rho = _per_path(spec, base, p.r, 100.0)
            su, sd = sim(p, 100.0 + h_s), sim(p, 100.0 - h_s)
            _, du, _ = _per_path(spec, su, p.r, 100.0 + h_s)
            _, dd, _ = _per_path(spec, sd, p.r, 100.0 - h_s)
            gamma = (du - dd) / (2 * h_s)
            pu, _, _ = _per_path(spec, su, p.r, 100.0 + h_s)
            pd_, _, _ = _per_path(spec, sd, p.r, 100.0 - h_s)
            delta_fd = (pu - pd_) / (2 * h_s)
            vu = sim(_bump(p, v0=+h_v), 100.0)
            vd = sim(_bump(p, v0=-h_v), 100.0)
            vega = (_per_path(spec, vu, p.r, 100.0)[0] - _per_path(spec, vd, p.r, 100.0)[0]) / (2 * h_v)
            ru = sim(_bump(p, r=+h_r), 100.0)
            rd = sim(_bump(p, r=-h_r), 100.0)
            rho_fd = (_per_path(spec, ru, p.r + h_r, 100.0)[0] -
                      _per_path(spec, rd, p.r - h_r, 100.0)[0]) / (2 * h_r)
            row = {}
            for qn, arr in (("price", price), ("delta", delta), ("rho", rho), ("gamma", gamma),
                            ("vega", vega), ("delta_fd", delta_fd), ("rho_fd", rho_fd)):
                row[qn] = [float(arr.mean()), float(arr.std(ddof=1) / math.sqrt(arr.size))]
            row["base_pass_seconds"] = t_base
            res[name] = row
            print(name, {k: v for k, v in row.items()}, flush=True)
        # Broadie-Kaya exact European (1 step), pseudo sampler
        n_bk = 2**15
        times = np.array([0.0, T])
        flags = np.array([1], dtype=np.int64)
        kr_bk = int(derive_key(root_key(seed + 1), 0))
        jobs_bk = [(lo, min(lo + 1024, n_bk)) for lo in range(0, n_bk, 1024)]
        t0 = time.time()
        obs = np.concatenate(list(pool.map(
            lambda j: core.exact_batch(p, 100.0, times, flags, j[0], j[1], kr_bk, None), jobs_bk)))
        price = math.exp(-p.r * T) * np.maximum(obs[:, 0] - 100.0, 0.0)
        res["bk_exact_euro"] = {"price": [float(price.mean()), float(price.std(ddof=1) / math.sqrt(n_bk))],
                                "n_paths": n_bk, "seconds": time.time() - t0}
        print("bk", res["bk_exact_euro"], flush=True)
    with open(os.path.join(HERE, "stats_golden.json"), "w") as f:
        json.dump(res, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stats", action="store_true")
    ap.add_argument("--only", default=None, help="one fixture group, e.g. primitives")
    args = ap.parse_args()
    hm, core = load_reference()
    if args.only == "primitives":
        primitive_cases(hm)
        return
    replay_cases(hm, core)
    engine_cases(hm)
    rng_cases(hm)
    sobol_cases(hm)
    primitive_cases(hm)
    exact_cases(hm, core)
    if args.stats:
        stats_golden(hm, core)


if __name__ == "__main__":
    main()
