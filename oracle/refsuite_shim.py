"""pytest plugin: run the reference's UNMODIFIED test modules against the
drop-in -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    python -m pytest -p oracle.refsuite_shim oracle/_ref/tests ...

(``make -C oracle`` copies the reference's ``pkg/tests`` into the git-ignored
``oracle/_ref/tests``; tests/test_gpu_reference_suite.py drives this.)

Before collection, ``hestonmc`` and its submodules are aliased to
``paper_2309_10477_b200`` (the reference tests import ``hestonmc.engine``,
``.model``, ``.errors``, ``.rng``, ``.products``, ``.schemes``,
``.backend``, ``.cli``, and the exact scheme's ``.bessel``, ``.ivlaw``,
``.exact``).  The reference's two kernel modules are mapped as
the reference's backend seam would see them on this machine:
``hestonmc._core`` (the compiled backend) -> the drop-in's GPU backend
``cuda_backend``, ``hestonmc._batch_py`` (the other backend of the
cross-backend tests) -> ``oracle.ref_batch``, the reference's own compiled
kernel.
"""

from __future__ import annotations

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_2309_10477_b200 as _pkg  # noqa: E402

_SUBMODULES = ("engine", "model", "errors", "rng", "products", "schemes", "backend", "cli", "bessel", "ivlaw",
               "exact")

sys.modules["hestonmc"] = _pkg
for _name in _SUBMODULES:
    sys.modules[f"hestonmc.{_name}"] = importlib.import_module(f"paper_2309_10477_b200.{_name}")
sys.modules["hestonmc._core"] = importlib.import_module("paper_2309_10477_b200.cuda_backend")
sys.modules["hestonmc._batch_py"] = importlib.import_module("oracle.ref_batch")
_pkg._core = sys.modules["hestonmc._core"]
_pkg._batch_py = sys.modules["hestonmc._batch_py"]
