"""The C ABI library loads and exports what include/hmc.h declares; host-side
logic of the library that needs no GPU (CPU only)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2309_10477_b200 import _lib, sobol
from conftest import ROOT


def _header_functions():
    src = open(os.path.join(ROOT, "include", "hmc.h")).read()
    return sorted(set(re.findall(r"\b(hmc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _header_functions()
    assert declared, "no declarations parsed"
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name


def test_abi_version_and_constants():
    L = _lib.lib()
    assert L.hmc_abi_version() == _lib.HMC_ABI_VERSION
    src = open(os.path.join(ROOT, "include", "hmc.h")).read()
    assert re.search(r"#define HMC_TILE 128\b", src)
    assert re.search(r"#define HMC_CHUNK_TILES 128\b", src)
    assert re.search(r"#define HMC_NQ 7\b", src)
    assert _lib.HMC_CHUNK == 16384


def test_key_derivation_matches_reference(golden_rng):
    L = _lib.lib()
    for seed, row in golden_rng["keys"].items():
        rk = L.hmc_root_key(int(seed))
        assert rk == int(row["root"])
        got = [L.hmc_derive_key(rk, i) for i in (0, 1, 2, 1000, 2**40)]
        assert got == [int(x) for x in row["derived"]]


def test_sobol_directions_bit_identical_to_scipy(golden_sobol):
    for key, start in (("d504_0", 0), ("d504_far", 3 * 2**20 + 1)):
        ref = golden_sobol[key]
        np.testing.assert_array_equal(sobol.points(504, start, ref.shape[0]), ref)
    ref = golden_sobol["d2_1"]
    np.testing.assert_array_equal(sobol.points(2, 1, ref.shape[0]), ref)
    # first points of dimension one (reference tests/test_rng.py:55-57)
    assert sobol.points(1, 1, 4)[:, 0].tolist() == [0.5, 0.75, 0.25, 0.375]


def _job(**over):
    m = _lib.Model(2.0, 0.04, 0.3, -0.7, 0.03, 0.04)
    avg = np.array([over.pop("n_steps_avg", 252)], dtype=np.int64)
    pr = _lib.Product(over.pop("style", 0), over.pop("right", 0), 100.0, 1.0, 100.0,
                      avg.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), avg.size)
    kw = dict(scheme=2, sampler=0, precision=0, want_greeks=1, n_steps=252, n_runs=1,
              n_paths=2**20, path_lo=0, path_hi=2**20, seed=42, h_spot=0.5, v0_up=0.0404,
              v0_dn=0.0396, h_r=1e-4)
    kw.update(over)
    return m, pr, _lib.Sim(**kw), avg


def test_slice_geometry():
    L = _lib.lib()
    _, _, sim, _ = _job(n_paths=100000, path_lo=16384, path_hi=100000, n_runs=3)
    assert L.hmc_chunks_in_slice(ctypes.byref(sim)) == -(-(100000 - 16384) // 16384)
    tiles = -(-(100000 - 16384) // 128)
    assert L.hmc_workspace_bytes(ctypes.byref(sim)) >= 3 * tiles * 14 * 8


@pytest.mark.parametrize("over,code", [
    (dict(right=1), _lib.HMC_E_UNSUPPORTED),          # put Greeks (engine.py:120-121)
    (dict(scheme=0), _lib.HMC_E_UNSUPPORTED),         # exact scheme: hmc_exact_batch_f64
    (dict(path_lo=5), _lib.HMC_E_INVALID),            # slices are chunk aligned
    (dict(path_hi=2**20 + 1), _lib.HMC_E_INVALID),
    (dict(n_steps_avg=251), _lib.HMC_E_INVALID),      # european fixes at n_steps
    (dict(v0_dn=0.05), _lib.HMC_E_INVALID),
    (dict(sampler=1), _lib.HMC_E_INVALID),            # sobol without directions
    (dict(n_runs=0), _lib.HMC_E_INVALID),
])
def test_argument_validation_before_any_device_work(over, code):
    """Validation runs on the host before any CUDA call, so it is testable
    without a GPU and the error contract maps to the engine's exceptions."""
    L = _lib.lib()
    m, pr, sim, _keep = _job(**over)
    buf = ctypes.create_string_buffer(64)
    rc = L.hmc_greeks_chunks(ctypes.byref(m), ctypes.byref(pr), ctypes.byref(sim), buf, buf, None)
    assert rc == code
    assert L.hmc_last_error()


def test_error_mapping():
    from paper_2309_10477_b200.errors import DeviceError, UnsupportedProduct, ValidationError
    L = _lib.lib()
    m, pr, sim, _keep = _job(right=1)
    rc = L.hmc_greeks_chunks(ctypes.byref(m), ctypes.byref(pr), ctypes.byref(sim), None, None, None)
    with pytest.raises(UnsupportedProduct):
        _lib.check(rc)
    m, pr, sim, _keep = _job(path_lo=3)
    rc = L.hmc_greeks_chunks(ctypes.byref(m), ctypes.byref(pr), ctypes.byref(sim), None, None, None)
    with pytest.raises(ValidationError):
        _lib.check(rc)
    with pytest.raises(DeviceError):
        _lib.check(_lib.HMC_E_CUDA)


def test_no_cpu_fallback_without_device():
    """On a host without a GPU the engine fails loudly instead of computing
    on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2309_10477_b200 import DeviceError, HestonParams, OptionSpec, SimConfig, price
    p = HestonParams(2.0, 0.04, 0.3, -0.7, 0.03, 0.04)
    spec = OptionSpec("european", "call", 100.0, 1.0, 100.0)
    with pytest.raises(DeviceError):
        price(p, spec, SimConfig(scheme="milstein", n_paths=1024, n_steps=8, n_runs=1))
    from paper_2309_10477_b200 import cuda_backend
    with pytest.raises(DeviceError):
        cuda_backend.discretised_batch(p, 100.0, 1.0, 8, True, 0, 16, 1, None, np.array([8]))


def test_host_digital_shifts_match_device_derivation():
    """sobol.digital_shifts restates csrc sobol_shift: mix64(key ^ (d+1) GOLDEN) >> 34."""
    import oracle
    key = 0x0123456789ABCDEF
    got = sobol.digital_shifts(key, 6)
    for d in range(6):
        want = oracle.mix64(key ^ (((d + 1) * 0x9E3779B97F4A7C15) & (2**64 - 1))) >> 34
        assert int(got[d]) == want
    pts = sobol.points(4, 1, 8, key_run=key)
    assert np.all((pts > 0) & (pts < 1))


def test_greeks_multi_validates_before_device_work():
    L = _lib.lib()
    m, pr, sim, _keep = _job()
    out = np.zeros(_lib.HMC_NW)
    pd = ctypes.POINTER(ctypes.c_double)
    devs = (ctypes.c_int32 * 2)(0, 0)
    assert L.hmc_greeks_multi(ctypes.byref(m), ctypes.byref(pr), ctypes.byref(sim),
                              out.ctypes.data_as(pd), None, 2) == _lib.HMC_E_INVALID
    assert L.hmc_greeks_multi(ctypes.byref(m), ctypes.byref(pr), ctypes.byref(sim),
                              out.ctypes.data_as(pd), devs, 0) == _lib.HMC_E_INVALID
    m, pr, sim, _keep = _job(right=1)
    assert L.hmc_greeks_multi(ctypes.byref(m), ctypes.byref(pr), ctypes.byref(sim),
                              out.ctypes.data_as(pd), devs, 2) == _lib.HMC_E_UNSUPPORTED


@pytest.mark.parametrize("over,code", [(dict(right=1), _lib.HMC_E_UNSUPPORTED), (dict(path_lo=5), _lib.HMC_E_INVALID),
                                       (dict(sampler=1), _lib.HMC_E_INVALID), (dict(h_r=0.0), _lib.HMC_E_INVALID)])
def test_exact_greeks_chunks_validates_on_host(over, code):
    L = _lib.lib()
    right = over.pop("right", 0)
    m = _lib.Model(2.0, 0.04, 0.3, -0.7, 0.03, 0.04)
    idx = np.zeros(1, dtype=np.int64)
    pr = _lib.Product(0, right, 100.0, 1.0, 100.0, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 1)
    kw = dict(scheme=2, sampler=0, precision=1, want_greeks=1, n_steps=1, n_runs=1, n_paths=4096, path_lo=0,
              path_hi=4096, seed=1, h_spot=0.5, v0_up=0.0404, v0_dn=0.0396, h_r=1e-4)
    kw.update(over)
    sim = _lib.Sim(**kw)
    t = np.array([0.0, 1.0])
    f = np.ones(1, dtype=np.int64)
    buf = ctypes.create_string_buffer(64)
    rc = L.hmc_exact_greeks_chunks(ctypes.byref(m), ctypes.byref(pr), ctypes.byref(sim),
                                   t.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 1,
                                   f.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), buf, None)
    assert rc == code
