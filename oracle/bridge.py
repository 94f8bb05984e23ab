"""Sobol Brownian-bridge ordering -- CPU restatement, TEST INFRASTRUCTURE ONLY.

No reference counterpart: the reference feeds Sobol dimension pair k-1 to
step k (``engine.py:97-101``, ``_core.pyx:391-398``) and its paper calls
plain high-dimensional QMC "unsatisfactory" (``PAPER.md:495``); SURVEY
8f-2 lists bridge ordering as the follow-up.  This module states the
construction the product's kernels implement (``SimConfig.sobol_bridge``)
in plain numpy so tests can check them:

* skeleton points j = 0..S at steps b_j = floor(j n / S), point 0 = origin;
* level order: the horizon first, then the midpoint (floor) of every
  interval of the previous level, left to right; node i takes dimension
  pair i and sets W(b_m) = W(b_l) + a (W(b_r) - W(b_l)) + sd z with
  a = (t_m - t_l) / (t_r - t_l), sd^2 = (t_m - t_l)(t_r - t_m) / (t_r - t_l);
* then steps k = 1..n in time order; step k of segment j draws
  dW = (W(b_j) - W_{k-1}) / (b_j - k + 1) + sqrt(dt (b_j - k) / (b_j - k + 1)) z
  from the next unused pair (none at k = b_j, where dW = W(b_j) - W_{k-1}).

Both Brownian motions (asset, variance) share the ordering: pair
(2i, 2i+1) feeds (B1, B2); z1 = dB1 / sqrt(dt), z2 = rho z1 +
sqrt(1 - rho^2) dB2 / sqrt(dt) (the reference's correlation, _core.pyx:397-398).
"""

from __future__ import annotations

import math

import numpy as np

from . import inverse_normal_cdf


def skeleton(S: int, n: int) -> tuple[list[int], list[tuple[int, int, int]]]:
    """(segment-end steps b_0..b_S, level-order nodes (m, l, r))."""
    b = [j * n // S for j in range(S + 1)]
    nodes = [(S, 0, 0)]
    level = [(0, S)]
    while level:
        nxt = []
        for lo, hi in level:
            if hi - lo < 2:
                continue
            m = (lo + hi) // 2
            nodes.append((m, lo, hi))
            nxt += [(lo, m), (m, hi)]
        level = nxt
    return b, nodes


def construct(Z: np.ndarray, S: int, n: int, dt: float) -> np.ndarray:
    """Brownian values W[..., k] at steps k = 0..n of one motion from standard
    normals Z[..., i] in bridge-consumption order (i = 0..n-1)."""
    b, nodes = skeleton(S, n)
    t = [bj * dt for bj in b]
    sk = np.zeros(Z.shape[:-1] + (S + 1,))
    for i, (m, lo, hi) in enumerate(nodes):
        if i == 0:
            sk[..., m] = math.sqrt(t[S]) * Z[..., 0]
            continue
        a = (t[m] - t[lo]) / (t[hi] - t[lo])
        sd = math.sqrt((t[m] - t[lo]) * (t[hi] - t[m]) / (t[hi] - t[lo]))
        sk[..., m] = sk[..., lo] + a * (sk[..., hi] - sk[..., lo]) + sd * Z[..., i]
    W = np.zeros(Z.shape[:-1] + (n + 1,))
    pc = S
    j = 1
    for k in range(1, n + 1):
        while k > b[j]:
            j += 1
        if k == b[j]:
            W[..., k] = sk[..., j]
            continue
        left = b[j] - k
        W[..., k] = (W[..., k - 1] + (sk[..., j] - W[..., k - 1]) / (left + 1)
                     + math.sqrt(dt * left / (left + 1)) * Z[..., pc])
        pc += 1
    return W


def step_normals(U: np.ndarray, S: int, n_sim: int, n_steps: int, dt: float, rho: float) -> np.ndarray:
    """(N, 2*n_steps) step normals [z1, z2] (z2 correlated) from Sobol points
    U (N, >= 2*n_sim) under bridge ordering over the first n_sim steps;
    steps beyond n_sim (never observed) get zeros."""
    Z = inverse_normal_cdf(np.ascontiguousarray(U[:, :2 * n_sim]).ravel()).reshape(U.shape[0], n_sim, 2)
    W1 = construct(Z[:, :, 0], S, n_sim, dt)
    W2 = construct(Z[:, :, 1], S, n_sim, dt)
    isq = 1.0 / math.sqrt(dt)
    z1 = np.diff(W1, axis=1) * isq
    z2 = rho * z1 + math.sqrt(1.0 - rho * rho) * (np.diff(W2, axis=1) * isq)
    out = np.zeros((U.shape[0], 2 * n_steps))
    out[:, 0:2 * n_sim:2] = z1
    out[:, 1:2 * n_sim:2] = z2
    return out


def covariance_matrix(S: int, n: int, dt: float) -> np.ndarray:
    """Cov(W(t_k), W(t_l)), k, l = 1..n, implied by the construction (it is
    linear in Z, so Cov = A A^T with A = dW/dZ) -- equals min(t_k, t_l) for
    a correct bridge."""
    A = construct(np.eye(n), S, n, dt)[:, 1:].T   # rows: W(t_k), columns: Z_i
    return A @ A.T
