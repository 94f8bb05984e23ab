"""The reference's ``rng`` module (``hestonmc/rng.py``) for the drop-in.

Same names, same streams, same values -- served by libhmc:

* keys: ``root_key`` / ``derive_key`` / ``stream_key`` are the C ABI's
  ``hmc_root_key`` / ``hmc_derive_key`` (SplitMix64 finaliser, salts of
  ``rng.py:25-52``); ``derive_keys`` is their vectorised form;
* draws: ``uniform_at`` / ``uniforms_at`` / ``_uniform_keys`` run the device
  function the fp64 replay kernels draw with (``hmc_uniforms_f64``,
  ``rng.py:63-74,356-361``): draw i of key k is
  ``(mix64(k + (i+1) * GOLDEN) >> 11) * 2^-53``;
* ``inverse_normal_cdf`` is the device Acklam + Halley quantile of the
  replay kernels (``hmc_ndtri_f64``, ``rng.py:95-132``);
* ``sobol_points`` evaluates the unscrambled Gray-code Sobol rows from the
  direction table the kernels use (``sobol.points``), bit-identical to the
  reference's ``scipy.stats.qmc.Sobol`` (``rng.py:143-152``).

``UniformStream`` / ``sample_normal`` / ``correlated_pair`` keep the
reference's draw order (``rng.py:155-235``); pseudo streams fetch their draws
from the device 4096 at a time.

The Gamma / non-central chi-squared samplers of the exact scheme
(``rng.py:238-343``) are the exact kernel's device sampler
(``hmc_gamma_f64``, ``csrc/hmc_exact.cu`` ``sample_gamma_from``): same draws,
same Marsaglia-Tsang rejection loop as ``_core.pyx:116-136``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib, sobol
from .errors import DofOutOfRange, UnsupportedProduct, ValidationError

_MASK = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_ROOT_SALT = 0x8CB92BA72F3D8DD7
_INDEX_SALT = 0xD1B54A32D192ED03

PURPOSE_MAIN = 0
PURPOSE_GAMMA = 1
#: Sobol points reserved per stream_index block of a sobol UniformStream
SOBOL_BLOCK = 1 << 20

_U64P = ctypes.POINTER(ctypes.c_uint64)
_DP = ctypes.POINTER(ctypes.c_double)


def _device() -> int:
    import torch
    return torch.cuda.current_device() if torch.cuda.is_available() else 0


# ---- keys --------------------------------------------------------------------

def mix64(z: int) -> int:
    """SplitMix64 finaliser (Stafford 13): root_key's core with the salt undone."""
    return int(_lib.lib().hmc_root_key((int(z) & _MASK) ^ _ROOT_SALT))


def root_key(seed: int) -> int:
    return int(_lib.lib().hmc_root_key(int(seed) & _MASK))


def derive_key(parent: int, index: int) -> int:
    return int(_lib.lib().hmc_derive_key(int(parent) & _MASK, int(index) & _MASK))


def stream_key(seed: int, *indices: int) -> int:
    """Key of the substream (seed, i0, i1, ...), e.g. (run, path, purpose)."""
    k = root_key(seed)
    for ix in indices:
        k = derive_key(k, ix)
    return k


def mix64_vec(z) -> np.ndarray:
    return sobol._mix64(np.asarray(z, dtype=np.uint64))


def derive_keys(parent, indices) -> np.ndarray:
    """``derive_key`` over broadcast arrays of parents and indices."""
    parent = np.asarray(parent, dtype=np.uint64)
    with np.errstate(over="ignore"):
        salted = np.asarray(indices, dtype=np.uint64) + np.uint64(_INDEX_SALT)
    return mix64_vec(parent ^ mix64_vec(salted))


# ---- draws (device) -----------------------------------------------------------

def _draws(keys: np.ndarray, draws: np.ndarray) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1)
    draws = np.ascontiguousarray(draws, dtype=np.uint64).reshape(-1)
    out = np.empty(draws.size)
    _lib.check(_lib.lib().hmc_uniforms_f64(keys.ctypes.data_as(_U64P), keys.size,
                                           draws.ctypes.data_as(_U64P), draws.size,
                                           out.ctypes.data_as(_DP), _device()))
    return out


def uniform_at(key: int, i: int) -> float:
    """Draw i of the stream with the given key, in [0, 1)."""
    return float(_draws(np.array([int(key) & _MASK]), np.array([int(i) & _MASK]))[0])


def uniforms_at(key: int, start: int, count: int) -> np.ndarray:
    """Draws start .. start+count-1 of one stream."""
    idx = np.arange(start, start + count, dtype=np.uint64)
    return _draws(np.array([int(key) & _MASK], dtype=np.uint64), idx)


def _uniform_keys(keys, counters) -> np.ndarray:
    """uniform_at(keys[i], counters[i]) for aligned arrays."""
    keys = np.asarray(keys, dtype=np.uint64)
    counters = np.asarray(counters, dtype=np.uint64)
    keys, counters = np.broadcast_arrays(keys, counters)
    return _draws(keys, counters).reshape(keys.shape)


def inverse_normal_cdf(u):
    """Standard-normal quantile elementwise (Acklam + one Halley step, inputs
    clamped to [1e-300, 1 - 1e-16]); a scalar in gives a float out."""
    a = np.asarray(u, dtype=np.float64)
    flat = np.ascontiguousarray(a.reshape(-1))
    out = np.empty_like(flat)
    _lib.check(_lib.lib().hmc_ndtri_f64(flat.ctypes.data_as(_DP), flat.size,
                                        out.ctypes.data_as(_DP), _device()))
    return float(out[0]) if a.ndim == 0 else out.reshape(a.shape)


def sobol_points(dimension: int, start: int, count: int) -> np.ndarray:
    """Rows start .. start+count-1 of the unscrambled Sobol sequence (row 0
    is the all-zeros point)."""
    if count <= 0:
        return np.zeros((0, dimension))
    return sobol.points(dimension, start, count)


# ---- streams -----------------------------------------------------------------

@dataclass
class UniformStream:
    """Single-owner stream of uniforms in [0, 1) (reference ``rng.py:155-215``).

    kind "pseudo": counter stream of key stream_key(seed, stream_index);
    kind "sobol": coordinates of successive points of the given dimension,
    block stream_index of 2^20 points, the all-zeros point skipped.
    """

    kind: str = "pseudo"
    seed: int = 0
    dimension: int = 1
    stream_index: int = 0
    _key: int = field(init=False, default=0)
    _fetched: int = field(init=False, default=0, repr=False)   # draws (pseudo) / points (sobol) fetched
    _buffer: np.ndarray | None = field(init=False, default=None, repr=False)
    _buf_pos: int = field(init=False, default=0, repr=False)

    _CHUNK = 4096

    def __post_init__(self):
        if self.kind not in ("pseudo", "sobol"):
            raise ValidationError(f"unknown stream kind {self.kind!r}")
        if self.dimension < 1:
            raise ValidationError("dimension must be >= 1")
        if self.stream_index < 0:
            raise ValidationError("stream_index must be >= 0")
        self._key = stream_key(self.seed, self.stream_index)

    @property
    def _counter(self) -> int:
        """The reference's counter (rng.py:171-207): draws consumed so far
        for a pseudo stream (its draws are fetched from the device in
        blocks, consumed one at a time), points fetched for a sobol one."""
        return self._position() if self.kind == "pseudo" else self._fetched

    def _refill(self):
        if self.kind == "pseudo":
            self._buffer = uniforms_at(self._key, self._fetched, self._CHUNK)
        else:
            start = 1 + self.stream_index * SOBOL_BLOCK + self._fetched
            self._buffer = sobol_points(self.dimension, start, self._CHUNK).reshape(-1)
        self._fetched += self._CHUNK
        self._buf_pos = 0

    def next_uniform(self) -> float:
        """Next draw; for sobol, the next coordinate of the current point."""
        if self._buffer is None or self._buf_pos >= self._buffer.size:
            self._refill()
        u = float(self._buffer[self._buf_pos])
        self._buf_pos += 1
        return u

    def _position(self) -> int:
        """Index of the next draw (pseudo streams)."""
        pending = 0 if self._buffer is None else self._buffer.size - self._buf_pos
        return self._fetched - pending

    def _skip(self, n: int) -> None:
        """Consume n draws (pseudo streams)."""
        pos = self._position() + n
        self._buffer, self._buf_pos, self._fetched = None, 0, pos

    def next_point(self) -> np.ndarray:
        return np.array([self.next_uniform() for _ in range(self.dimension)])

    def spawn(self, stream_index: int) -> "UniformStream":
        return UniformStream(kind=self.kind, seed=self.seed, dimension=self.dimension,
                             stream_index=stream_index)


def sample_normal(stream: UniformStream) -> float:
    """One standard normal by inversion of one draw."""
    return inverse_normal_cdf(stream.next_uniform())


def correlated_pair(stream: UniformStream, rho: float) -> tuple[float, float]:
    """(Z1, Z2), Z2 = rho Z1 + sqrt(1 - rho^2) Zb; exactly two draws."""
    if not (-1.0 <= rho <= 1.0):
        raise ValidationError(f"rho must lie in [-1, 1], got {rho}")
    za = sample_normal(stream)
    zb = sample_normal(stream)
    return za, rho * za + float(np.sqrt(1.0 - rho * rho)) * zb


# ---- Gamma / non-central chi-squared (the exact scheme's samplers) ---------

def _gamma(keys: np.ndarray, start: np.ndarray, shape: float, scale: float):
    if not (shape > 0.0):
        raise ValidationError(f"gamma shape must be > 0, got {shape}")
    if not (scale > 0.0):
        raise ValidationError(f"gamma scale must be > 0, got {scale}")
    keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1)
    start = np.ascontiguousarray(start, dtype=np.uint64).reshape(-1)
    out = np.empty(keys.size)
    used = np.empty(keys.size, dtype=np.uint64)
    _lib.check(_lib.lib().hmc_gamma_f64(keys.ctypes.data_as(_U64P), start.ctypes.data_as(_U64P), keys.size,
                                        float(shape), float(scale), out.ctypes.data_as(_DP),
                                        used.ctypes.data_as(_U64P), _device()))
    return out, used


def gamma_batch(keys, shape: float, scale: float = 1.0) -> np.ndarray:
    """One Gamma(shape, scale) draw per key (Marsaglia-Tsang from draw 0 of
    each key's stream; shape < 1 boosted by U^(1/shape)) -- the exact
    kernel's device sampler."""
    keys = np.asarray(keys, dtype=np.uint64)
    out, _ = _gamma(keys, np.zeros(keys.size, dtype=np.uint64), shape, scale)
    return out.reshape(keys.shape)


def sample_gamma(stream: UniformStream, shape: float, scale: float = 1.0) -> float:
    """Gamma(shape, scale) from the stream's next draws (same draws and value
    as the reference's scalar sampler); pseudo streams only -- a rejection
    loop cannot consume QMC coordinates."""
    if not (shape > 0.0):
        raise ValidationError(f"gamma shape must be > 0, got {shape}")
    if not (scale > 0.0):
        raise ValidationError(f"gamma scale must be > 0, got {scale}")
    if type(stream) is not UniformStream or stream.kind != "pseudo":
        raise UnsupportedProduct("sample_gamma draws from a pseudo UniformStream's own counter stream")
    out, used = _gamma(np.array([stream._key], dtype=np.uint64),
                       np.array([stream._position()], dtype=np.uint64), shape, scale)
    stream._skip(int(used[0]))
    return float(out[0])


@dataclass(frozen=True)
class NccsParams:
    """Non-central chi-squared parameters (dof > 1, noncentrality >= 0)."""

    dof: float
    noncentrality: float

    def __post_init__(self):
        if not (self.dof > 1.0):
            raise DofOutOfRange(f"non-central chi-squared sampling needs dof > 1, got {self.dof}")
        if self.noncentrality < 0.0:
            raise ValidationError(f"noncentrality must be >= 0, got {self.noncentrality}")


def sample_nccs(stream: UniformStream, p: NccsParams, gamma_stream: UniformStream | None = None) -> float:
    """chi2_{dof-1} + (Z + sqrt(lambda))^2: one normal from ``stream``, the
    Gamma((dof-1)/2, 2) from ``gamma_stream`` (default: ``stream``)."""
    z = sample_normal(stream)
    g = sample_gamma(gamma_stream if gamma_stream is not None else stream, 0.5 * (p.dof - 1.0), 2.0)
    shifted = z + float(np.sqrt(p.noncentrality))
    return g + shifted * shifted
