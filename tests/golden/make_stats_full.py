"""Reference statistics AT THE BENCH SIZES, produced by the reference itself.

Test infrastructure (run in the build container; the reference tree is not on
the GPU box):

    make -C oracle                                # oracle/_ref/_core*.so
    python tests/golden/make_stats_full.py [c3] [c2] [c5]

Every number comes from the reference's own compiled kernel
(``_core.discretised_batch``, ``_core.pyx:354-412``, built from the
reference's ``_core.c`` by ``oracle/Makefile``) on the reference's own key
stream ``derive_key(root_key(seed), 0)`` (``engine.py:96``), with the
reference's per-path statistics (``engine._per_path_stats``,
``engine.py:47-68``) and the reference's CRN finite-difference method for the
quantities it does not compute (``tests/test_products.py:101-137``):

* price, Delta, Rho       pathwise, base paths
* Gamma                   (Delta(S0+h) - Delta(S0-h)) / 2h, re-simulated
* Vega                    (price(v0+h) - price(v0-h)) / 2h, re-simulated
* delta_fd, rho_fd        (price(x+h) - price(x-h)) / 2h, re-simulated

Per-path sums and sums of squares are accumulated per 2^20-path block in
fp64 and combined with ``math.fsum``, so each quantity carries its per-path
standard error.  Outputs (``tests/golden/``):

* ``stats_c3_2p24.json``  BASELINE config 3: Asian call, 252 daily fixings,
  2^24 paths x 252 steps, seed 42 -- the bench job itself.
* ``stats_c2_2p22.json``  BASELINE config 2: European call, 2^22 x 252.
* ``stats_c5_points.json`` BASELINE config 5 sample points: European and
  daily-Asian calls at maturities 0.5 and 2.0 on the surface's dt = 1/252
  grid, strikes {70, 85, 100, 115, 133}, 2^21 paths per maturity.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import BENCH, _bump, load_reference  # noqa: E402

QN = ("price", "delta", "rho", "gamma", "vega", "delta_fd", "rho_fd")
BLOCK = 2 ** 20
CHUNK = 4096      # engine.py:27


def _stats(K, T, s0, r, is_asian, obs):
    """engine._per_path_stats for a call: (price, delta, rho) per path."""
    disc = math.exp(-r * T)
    a = obs[:, 1] if is_asian else obs[:, 0]
    itm = a > K
    price = disc * np.maximum(a - K, 0.0)
    delta = np.where(itm, disc * a / s0, 0.0)
    if is_asian:
        rho = np.where(itm, disc * (obs[:, 2] - T * (a - K)), 0.0)
    else:
        rho = np.where(itm, disc * K * T, 0.0)
    return price, delta, rho


def run(core, pool, p, n_paths, n_steps, T, seed, products, h_rel_spot=0.005, h_r=1e-4,
        h_rel_v0=0.01, s0=100.0, log=""):
    """products: list of (name, K, is_asian).  Asian = average over every
    grid step 1..n_steps (daily fixings on the grid), European = s_T; both
    come out of ONE discretised_batch call (columns 0 and 1)."""
    from hestonmc.rng import derive_key, root_key
    kr = int(derive_key(root_key(seed), 0))
    avg = np.arange(1, n_steps + 1, dtype=np.int64)
    hs, hv = h_rel_spot * s0, h_rel_v0 * p.v0
    variants = {"base": (p, s0), "s_up": (p, s0 + hs), "s_dn": (p, s0 - hs),
                "v_up": (_bump(p, v0=+hv), s0), "v_dn": (_bump(p, v0=-hv), s0),
                "r_up": (_bump(p, r=+h_r), s0), "r_dn": (_bump(p, r=-h_r), s0)}
    acc = {name: {q: ([], []) for q in QN} for name, _, _ in products}
    t_start = time.time()
    for lo in range(0, n_paths, BLOCK):
        hi = min(lo + BLOCK, n_paths)
        jobs = [(a, min(a + CHUNK, hi)) for a in range(lo, hi, CHUNK)]
        obs = {}
        for vn, (pp, ss) in variants.items():
            parts = pool.map(lambda j, pp=pp, ss=ss: core.discretised_batch(
                pp, ss, T, n_steps, True, j[0], j[1], kr, None, avg), jobs)
            obs[vn] = np.concatenate(list(parts))
        for name, K, asian in products:
            price, delta, rho = _stats(K, T, s0, p.r, asian, obs["base"])
            pu, du, _ = _stats(K, T, s0 + hs, p.r, asian, obs["s_up"])
            pd_, dd, _ = _stats(K, T, s0 - hs, p.r, asian, obs["s_dn"])
            vu = _stats(K, T, s0, p.r, asian, obs["v_up"])[0]
            vd = _stats(K, T, s0, p.r, asian, obs["v_dn"])[0]
            ru = _stats(K, T, s0, p.r + h_r, asian, obs["r_up"])[0]
            rd = _stats(K, T, s0, p.r - h_r, asian, obs["r_dn"])[0]
            per = {"price": price, "delta": delta, "rho": rho, "gamma": (du - dd) / (2 * hs),
                   "vega": (vu - vd) / (2 * hv), "delta_fd": (pu - pd_) / (2 * hs),
                   "rho_fd": (ru - rd) / (2 * h_r)}
            for q, x in per.items():
                acc[name][q][0].append(float(x.sum()))
                acc[name][q][1].append(float((x * x).sum()))
        print(f"{log} block {lo // BLOCK + 1}/{(n_paths + BLOCK - 1) // BLOCK} "
              f"{time.time() - t_start:.0f}s", flush=True)
    out = {}
    for name, K, asian in products:
        row = {"strike": K, "maturity": T, "style": "asian_arithmetic" if asian else "european"}
        for q in QN:
            s, ss = math.fsum(acc[name][q][0]), math.fsum(acc[name][q][1])
            mean = s / n_paths
            var = max(ss - s * s / n_paths, 0.0) / (n_paths - 1)
            row[q] = [mean, math.sqrt(var / n_paths)]
        out[name] = row
    meta = {"params": BENCH, "n_paths": n_paths, "n_steps": n_steps, "maturity": T, "seed": seed,
            "spot": s0, "bumps": {"h_spot": hs, "h_r": h_r, "v0_up": p.v0 + hv, "v0_dn": p.v0 - hv},
            "workers": os.cpu_count(), "seconds": time.time() - t_start,
            "kernel": "reference _core.discretised_batch (oracle/_ref), milstein"}
    return out, meta


def main(which):
    hm, core = load_reference()
    from hestonmc.model import HestonParams
    p = HestonParams(**BENCH)
    with ThreadPoolExecutor(os.cpu_count()) as pool:
        if "c2" in which:
            res, meta = run(core, pool, p, 2 ** 22, 252, 1.0, 42, [("euro", 100.0, False)], log="c2")
            with open(os.path.join(HERE, "stats_c2_2p22.json"), "w") as f:
                json.dump({"meta": meta, **res}, f, indent=1)
        if "c5" in which:
            pts = {}
            metas = {}
            strikes = (70.0, 85.0, 100.0, 115.0, 133.0)
            for T in (0.5, 2.0):
                n = int(round(252 * T))
                prods = [(f"{style}_T{T}_K{K:g}", K, style == "asian")
                         for style in ("euro", "asian") for K in strikes]
                res, meta = run(core, pool, p, 2 ** 21, n, T, 42, prods, log=f"c5 T={T}")
                pts.update(res)
                metas[str(T)] = meta
            with open(os.path.join(HERE, "stats_c5_points.json"), "w") as f:
                json.dump({"meta": metas, "points": pts}, f, indent=1)
        if "c3" in which:
            res, meta = run(core, pool, p, 2 ** 24, 252, 1.0, 42, [("asian_daily", 100.0, True)],
                            log="c3")
            with open(os.path.join(HERE, "stats_c3_2p24.json"), "w") as f:
                json.dump({"meta": meta, **res}, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c5", "c3"])
