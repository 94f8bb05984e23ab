"""CPU check of the surface epilogue algebra (hmc_surface_finalize, host C++):
histograms built in numpy exactly as the kernel bins them (same buckets,
same fixed-point rounding) must reproduce brute-force per-strike sums and
sums of squares of every estimator computed path by path in fp64."""

import ctypes
import math

import numpy as np
import pytest

from paper_2309_10477_b200 import _lib

LIN, QUAD, BAND = 1024.0, 4.0, 1048576.0  # hmc_launch.h kSurf*Scale
ROWS = 23


def _bucket(K, x):
    return np.searchsorted(K, x, side="left")  # #{K_j < x}


def _fix(x, scale):
    return np.rint(np.asarray(x, dtype=np.float64) * scale).astype(np.int64)


def _hist(K, obs, d, eps, dv):
    """Replicates surface_update for one (style, maturity)."""
    nK = K.size
    nb = nK + 1
    H = np.zeros((ROWS, nb), dtype=np.int64)
    A, Au, Ad, Rp, Rm, w, al = (obs[k] for k in ("A", "Au", "Ad", "Rp", "Rm", "w", "al"))
    def add(row, c, v, scale):
        np.add.at(H[row], c, _fix(v, scale))
    cu, c1, cd = _bucket(K, A * (1 + eps)), _bucket(K, A), _bucket(K, A * (1 - eps))
    add(0, cu, A, LIN); add(1, cu, A * A, QUAD)
    np.add.at(H[2], c1, 1); add(3, c1, A, LIN); add(4, c1, A * A, QUAD); add(5, c1, w, LIN); add(6, c1, w * w, QUAD)
    np.add.at(H[7], cd, 1); add(8, cd, A, LIN); add(9, cd, A * A, QUAD)
    cvu, cvd = _bucket(K, Au), _bucket(K, Ad)
    g = d * (Au - Ad) / dv
    cmin = np.minimum(cvu, cvd)
    add(10, cmin, g, LIN); add(11, cmin, g * g, QUAD)
    cp, cm = _bucket(K, Rp), _bucket(K, Rm)
    np.add.at(H[12], cm, 1); add(13, cm, al, LIN); add(14, cm, al * al, QUAD)
    for row, lo, hi, x in ((15, cd, cu, A * (1 + eps)), (17, cvd, cvu, Au), (19, cvu, cvd, Ad),
                           (21, cm, cp, Rp)):
        for p in range(A.size):
            for j in range(lo[p], hi[p]):
                e = x[p] - K[j]
                H[row, j] += _fix(e, BAND)
                H[row + 1, j] += _fix(e * e, BAND)
    return H


def test_finalize_matches_brute_force():
    rng = np.random.default_rng(5)
    S0, r, T, h, hr = 100.0, 0.03, 1.0, 0.5, 1e-4
    v0, vu, vd = 0.04, 0.0404, 0.0396
    eps, dv = h / S0, vu - vd
    K = np.array([80.0, 90.0, 95.0, 99.5, 100.0, 100.2, 105.0, 120.0])
    n = 4000
    A = 100.0 * np.exp(0.2 * rng.standard_normal(n))
    Au = A * np.exp(0.004 * rng.standard_normal(n))
    Ad = A * np.exp(0.004 * rng.standard_normal(n))
    d, dp, dm = math.exp(-r * T), math.exp(-(r + hr) * T), math.exp(-(r - hr) * T)
    D = A * 0.5 * T * hr
    Rp, Rm = A + D, A - D
    tw = 0.5 * T * A * (1 + 0.01 * rng.standard_normal(n))
    w = tw - T * A
    al = (dp * Rp - dm * Rm) / (2 * hr)
    obs = dict(A=A, Au=Au, Ad=Ad, Rp=Rp, Rm=Rm, w=w, al=al)
    H = _hist(K, obs, d, eps, dv)

    # call hmc_surface_finalize with one run, one style pair (european slot = asian slot = H)
    mats = np.array([252], dtype=np.int64)
    spec = _lib.SurfaceSpec(S0, T / 252, K.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), K.size, 1,
                            mats.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    sim = _lib.Sim(scheme=2, sampler=0, precision=0, want_greeks=1, n_steps=252, n_runs=1, n_paths=n,
                   path_lo=0, path_hi=n, seed=1, h_spot=h, v0_up=vu, v0_dn=vd, h_r=hr)
    model = _lib.Model(2.0, 0.04, 0.3, -0.7, r, v0)
    acc = np.ascontiguousarray(np.stack([H, H]).reshape(-1))
    out = np.zeros((1, 2, 1, K.size, _lib.HMC_NW))
    _lib.check(_lib.lib().hmc_surface_finalize(
        ctypes.byref(model), ctypes.byref(spec), ctypes.byref(sim),
        acc.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    got = out[0, 0, 0]

    pos = lambda x: np.maximum(x, 0.0)  # noqa: E731
    for j, k in enumerate(K):
        q = {
            "price": d * pos(A - k),
            "delta": np.where(A > k, d * A / S0, 0.0),
            "rho": np.where(A > k, d * (w + T * k), 0.0),
            "gamma": d * A / S0 * ((A * (1 + eps) > k).astype(float) - (A * (1 - eps) > k)) / (2 * h),
            "vega": d * (pos(Au - k) - pos(Ad - k)) / dv,
            "delta_fd": d * (pos(A * (1 + eps) - k) - pos(A * (1 - eps) - k)) / (2 * h),
            "rho_fd": (dp * pos(Rp - k) - dm * pos(Rm - k)) / (2 * hr),
        }
        for qi, name in enumerate(_lib.QUANTITIES):
            s1, s2 = q[name].sum(), (q[name] ** 2).sum()
            assert got[j, 2 * qi] == pytest.approx(s1, rel=2e-5, abs=2e-3), (k, name)
            assert got[j, 2 * qi + 1] == pytest.approx(s2, rel=2e-3, abs=5.0), (k, name)
