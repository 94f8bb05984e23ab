"""The reference's own compiled kernel as a backend-protocol module --
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

When the reference's unmodified test modules run against the drop-in
(tests/test_gpu_reference_suite.py, oracle/refsuite_shim.py), the drop-in's
GPU backend stands in for ``hestonmc._core`` and this module for
``hestonmc._batch_py``: the reference's cross-backend tests
(``tests/test_backends.py:26-60``) then compare the GPU kernels with the
reference's compiled ``_core`` (``oracle/_ref``, built from the reference's
``_core.c``) at the reference's own tolerance.
"""

from __future__ import annotations

from . import ref_core

BACKEND_NAME = "reference-core"


def _core():
    core = ref_core()
    if core is None:
        raise RuntimeError("oracle/_ref not built (make -C oracle on the build host)")
    return core


def discretised_batch(*args, **kwargs):
    return _core().discretised_batch(*args, **kwargs)


def exact_batch(*args, **kwargs):
    return _core().exact_batch(*args, **kwargs)
