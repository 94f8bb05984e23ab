"""Backend selection (reference ``backend.py:14-41``).

The only backend is the CUDA one: ``get_backend()`` / ``get_backend("cuda")``
return :mod:`cuda_backend`.  The reference's names ``"compiled"`` and
``"python"`` are accepted for source compatibility and map to the same GPU
module -- there is deliberately no CPU backend to fall back to.
"""

from __future__ import annotations

from . import cuda_backend

BACKEND_NAME: str = cuda_backend.BACKEND_NAME
HAVE_COMPILED = True


def get_backend(name: str | None = None):
    """Module implementing ``discretised_batch`` / ``exact_batch``."""
    if name in (None, "cuda", "compiled", "python"):
        return cuda_backend
    raise ValueError(f"unknown backend {name!r}")
