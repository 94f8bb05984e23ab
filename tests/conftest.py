"""Shared fixtures.  GPU tests carry ``@pytest.mark.gpu``; everything else runs
on a CPU-only host (``pytest -m "not gpu"``)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2309_10477_b200.model import (BENCH_PARAMS, DEFAULT_PARAMS,  # noqa: E402
                                         HestonParams, OptionSpec)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libhmc.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def params() -> HestonParams:
    """Paper Table-1 parameters (reference tests/conftest.py:8-11)."""
    return HestonParams(**DEFAULT_PARAMS)


@pytest.fixture(scope="session")
def bench_params() -> HestonParams:
    return HestonParams(**BENCH_PARAMS)


@pytest.fixture(scope="session")
def euro_call() -> OptionSpec:
    return OptionSpec(style="european", right="call", strike=100.0, maturity=1.0, spot=100.0)


@pytest.fixture(scope="session")
def asian_call() -> OptionSpec:
    return OptionSpec(style="asian_arithmetic", right="call", strike=100.0, maturity=1.0,
                      spot=100.0, averaging_times=(0.25, 0.5, 0.75, 1.0))


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def replay_cases():
    z = np.load(os.path.join(GOLDEN, "replay_cases.npz"))
    meta = json.loads(bytes(z["__meta__"]).decode())
    cases = {}
    for name, m in meta.items():
        c = dict(m)
        c["out"] = z[f"{name}__out"]
        c["avg"] = z[f"{name}__avg"]
        c["uniforms"] = z[f"{name}__uniforms"] if m["has_uniforms"] else None
        c["key_run"] = int(m["key_run"])
        cases[name] = c
    return cases


@pytest.fixture(scope="session")
def golden_replay():
    return replay_cases()


@pytest.fixture(scope="session")
def golden_engine():
    return load_json("engine_cases.json")


@pytest.fixture(scope="session")
def golden_rng():
    return load_json("rng_cases.json")


@pytest.fixture(scope="session")
def golden_stats():
    path = os.path.join(GOLDEN, "stats_golden.json")
    if not os.path.exists(path):
        pytest.skip("stats_golden.json not generated")
    return load_json("stats_golden.json")


@pytest.fixture(scope="session")
def golden_sobol():
    return dict(np.load(os.path.join(GOLDEN, "sobol_points.npz")))


def spec_from(d) -> OptionSpec:
    return OptionSpec(style=d["style"], right=d["right"], strike=d["strike"],
                      maturity=d["maturity"], spot=d["spot"],
                      averaging_times=tuple(d.get("averaging_times", ())))
