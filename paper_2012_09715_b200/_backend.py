"""Kernel-plugin selector (mirrors approxrv/_backend.py:1-42).

The reference chooses between its compiled Cython module and a numpy
fallback.  Here there is exactly one backend -- the sm_100a CUDA kernels --
and no fallback: if libarv_b200.so cannot be loaded, importing this package
fails.  ``APPROXRV_BACKEND`` is honoured only to reject requests for a CPU
backend loudly.
"""

from __future__ import annotations

import os

from . import _kernels as kernels

_choice = os.environ.get("APPROXRV_BACKEND", "auto").lower()
if _choice == "python":
    raise ImportError("APPROXRV_BACKEND=python: approxrv-b200 has no CPU backend (sm_100a CUDA only)")


def backend_name() -> str:
    """'cuda-sm100a' -- the only backend."""
    return "cuda-sm100a"


def get_kernels(name: str | None = None):
    """Return the kernel module ('active', 'compiled' or 'cuda')."""
    if name in (None, "active", "compiled", "cuda", "cuda-sm100a"):
        return kernels
    raise ValueError(f"unknown backend {name!r} (only the CUDA backend exists)")
