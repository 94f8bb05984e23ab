"""bench.py's JSON-line contract on the CPU: the reference arm runs and
prints the required keys, non-zero ranks stay silent, and the B200 arm
fails loudly (no CPU fallback) when no GPU is visible."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

import oracle


def _run(args, **env):
    e = dict(os.environ, **env)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, env=e, cwd=ROOT, timeout=600)


@pytest.mark.skipif(oracle.ref_core() is None, reason="oracle/_ref (reference kernel) not built")
def test_reference_arm_line():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], HMC_BENCH_REF_PATHS="4096")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"]


def test_reference_arm_silent_on_other_ranks():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], RANK="1", WORLD_SIZE="2")
    assert r.returncode == 0
    assert r.stdout.strip() == ""


def test_b200_arm_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    r = _run(["--steps", "1", "--warmup", "3"])
    assert r.returncode != 0
    assert '"value"' not in r.stdout


@pytest.mark.skipif(oracle.ref_core() is None, reason="oracle/_ref (reference kernel) not built")
def test_json_line_owns_stdout_under_torchrun():
    """Under torch.distributed.run (LOCAL_RANK set) file descriptor 1 is
    handed to stderr, so banners written straight to fd 1 (NCCL prints its
    version there) cannot precede the JSON line."""
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], HMC_BENCH_REF_PATHS="4096",
             LOCAL_RANK="0", RANK="0", WORLD_SIZE="1")
    assert r.returncode == 0, r.stderr[-2000:]
    out = r.stdout.splitlines()
    assert len(out) == 1 and json.loads(out[0])["impl"] == "reference"


def test_committed_b200_line_has_the_contract_keys():
    """The B200 arm's last measured line (profiles/r01_bench_line.json, from
    `python bench.py` on a B200) carries every key the bench contract and the
    tier's measurement rules ask for, with self-consistent values."""
    d = json.load(open(os.path.join(ROOT, "profiles", "r01_bench_line.json")))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["warmup"] >= 3 and d["n_gpus"] == 1 and d["config"]["workload"]
    r = d["roofline"]
    assert 0.0 < r["frac"] <= 1.0 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    assert r["traffic"] is None or r["traffic"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["gpu_launches"] > 0
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
