"""The reference's OWN test modules, unmodified, against the drop-in on the GPU.

``make -C oracle`` copies ``/root/reference/pkg/tests`` into the git-ignored
``oracle/_ref/tests`` (it travels to the GPU box like the reference kernel
build); ``oracle/refsuite_shim.py`` aliases ``hestonmc`` to the package
before collection.  Every test of the modules (engine, products,
acceptance, backends, cli, schemes, rng) runs; the outcome must match the
ledger below exactly: every test not listed passes, and each listed test
fails for the stated design reason (INTEGRATION.md §4 carries the same list).
Since round 2 that includes the exact scheme's host modules (``test_bessel``,
``test_ivlaw``, ``test_exact``: Bessel series, integrated-variance law,
scalar exact step), served by the exact kernel's device routines.
"""

import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "oracle", "_ref", "tests")
MODULES = ("test_engine.py", "test_products.py", "test_acceptance.py", "test_backends.py",
           "test_cli.py", "test_schemes.py", "test_rng.py", "test_bessel.py", "test_ivlaw.py",
           "test_exact.py")

pytestmark = pytest.mark.gpu

#: reference tests that fail against the drop-in BY DESIGN -> reason
EXPECTED_FAILURES = {
    "test_backends.py::TestKernelAgreement::test_backend_names":
        "the drop-in's only backend is the GPU one (BACKEND_NAME 'cuda'); get_backend('python') "
        "returns it too -- there is deliberately no CPU backend",
    "test_backends.py::TestEngineAgreement::test_env_var_forces_fallback":
        "HESTONMC_PURE_PYTHON cannot force a CPU fallback: there is none (and the subprocess "
        "imports `hestonmc`, which is only an alias inside the shimmed test process)",
    "test_engine.py::TestStatistics::test_se_scaling_one_over_sqrt_n":
        "statistical test with a ~5 % false-failure rate at an arbitrary seed (40-seed sweep, "
        "profiles/r02_se_scaling_seed_sweep.txt: 5 % for the fp32 Philox stream AND for the "
        "reference's own stream); at seed 42 the fp32 stream's ratio is 0.785 (bound 0.65); the "
        "same test on the reference's stream (precision='fp64', the replay path) gives 0.559 and passes",
}


def _run_suite(tmp_path):
    if not os.path.isdir(SUITE):
        pytest.skip("oracle/_ref/tests missing (make -C oracle where /root/reference exists)")
    xml = tmp_path / "ref_suite.xml"
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    cmd = [sys.executable, "-m", "pytest", "-p", "oracle.refsuite_shim", "-q", "-p", "no:cacheprovider",
           f"--junitxml={xml}", *MODULES]
    r = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=3000)
    outcomes = {}
    for case in ET.parse(xml).getroot().iter("testcase"):
        mod = case.get("classname", "").split(".")
        name = f"{mod[0]}.py::" + "::".join(mod[1:] + [case.get("name")])
        name = name.replace(".py::::", ".py::")
        if case.find("failure") is not None or case.find("error") is not None:
            el = case.find("failure") if case.find("failure") is not None else case.find("error")
            outcomes[name] = ("failed", (el.get("message") or "")[:300])
        elif case.find("skipped") is not None:
            outcomes[name] = ("skipped", (case.find("skipped").get("message") or "")[:300])
        else:
            outcomes[name] = ("passed", "")
    return r, outcomes


def test_reference_suite_unmodified(tmp_path):
    r, outcomes = _run_suite(tmp_path)
    counts = {k: sum(1 for o, _ in outcomes.values() if o == k) for k in ("passed", "failed", "skipped")}
    failed = {n: m for n, (o, m) in outcomes.items() if o == "failed"}
    report = {"modules": MODULES, "counts": counts, "failed": failed,
              "skipped": {n: m for n, (o, m) in outcomes.items() if o == "skipped"},
              "expected_failures": EXPECTED_FAILURES, "tail": r.stdout[-4000:]}
    out = os.environ.get("REF_SUITE_REPORT")
    if out:
        with open(out, "w") as f:
            json.dump(report, f, indent=1)
    print(json.dumps(counts))
    assert counts["passed"] > 0, r.stdout[-3000:] + r.stderr[-3000:]
    unexpected = sorted(set(failed) - set(EXPECTED_FAILURES))
    assert not unexpected, {n: failed[n] for n in unexpected}
    now_passing = sorted(n for n in EXPECTED_FAILURES if outcomes.get(n, ("missing",))[0] != "failed")
    assert not now_passing, f"ledger out of date: {now_passing}"
