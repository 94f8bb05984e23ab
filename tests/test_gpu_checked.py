"""The bounds-checked build (HMC_DEBUG_BOUNDS=1: a device assert on every
data- or table-dependent index -- Sobol tables, surface histograms and strike
buckets, bridge skeletons, exact-scheme node caches, step tables, tile
writes) runs every kernel on small and ragged shapes without tripping a
check and with finite results (tools/checked_suite.py).  compute-sanitizer
is closed on this GPU pool; this is its stand-in."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2309_10477_b200", "_variants", "libhmc_checked.so")

pytestmark = pytest.mark.gpu


def test_checked_build_runs_every_kernel_clean():
    if not os.path.exists(CHECKED):
        sys.path.insert(0, ROOT)
        from paper_2309_10477_b200 import _build
        _build.build_checked()
    env = dict(os.environ, HMC_LIB_PATH=CHECKED)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_suite.py")], env=env,
                       capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    assert "checked suite ok" in r.stdout, r.stdout[-2000:]
    assert "Assertion" not in r.stderr, r.stderr[-4000:]


def test_checks_are_compiled_into_the_checked_build_only():
    """The asserts exist in the checked library and nowhere in the product."""
    import shutil
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    prod = os.path.join(ROOT, "paper_2309_10477_b200", "libhmc.so")
    n = {}
    for name, lib in (("checked", CHECKED), ("product", prod)):
        elf = subprocess.run([tool, "-elf", lib], capture_output=True, text=True).stdout
        n[name] = elf.count("__assertfail")
    assert n["checked"] > 100 and n["product"] == 0, n
