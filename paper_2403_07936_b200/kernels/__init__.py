"""Stencil kernel backend -- the reference's plugin point (kernels/__init__.py:11-49).

The reference selects ``cython`` or ``numpy`` via ``MGSR_BACKEND``; this
package provides the ``cuda`` backend (sm_100a, libmgsr_b200.so) and nothing
else: ``MGSR_BACKEND`` may be ``auto`` or ``cuda``; any other value raises,
and a missing library or GPU raises at call time (no CPU fallback).

``gs_sweeps(p, f, h2, sweeps)`` mutates ``p`` in place and ``laplacian``
returns a new array, exactly like the reference backends; both accept host
numpy arrays (staged through the device) or CUDA float64 tensors.
"""

from __future__ import annotations

import os

import numpy as np

from .. import _lib

__all__ = ["active_backend", "gs_sweeps", "laplacian", "HAVE_CUDA"]

_choice = os.environ.get("MGSR_BACKEND", "auto").lower()
if _choice not in ("auto", "cuda"):
    raise ValueError(f"MGSR_BACKEND must be auto or cuda, got {_choice!r}")

HAVE_CUDA = os.path.exists(_lib.LIB_PATH)


def active_backend() -> str:
    """Name of the backend in use: always ``cuda``."""
    return "cuda"


def _is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch")


def gs_sweeps(p, f, h2: float, sweeps: int) -> None:
    """In-place red-black Gauss-Seidel with mean subtraction (_stencil.pyx:12-45)."""
    n = p.shape[0]
    if n % 2 != 0:
        raise ValueError(f"red-black coloring needs an even side, got {n}")
    if tuple(f.shape) != tuple(p.shape):
        raise ValueError("p and f shapes differ")
    from .. import ops
    if _is_tensor(p):
        ops.gs_sweeps_(p, f, float(h2), int(sweeps))
        return
    from .._device import to_dev, to_host
    dp, df = to_dev(p), to_dev(f)
    ops.gs_sweeps_(dp, df, float(h2), int(sweeps))
    p[...] = to_host(dp)


def laplacian(p, inv_h2: float):
    """Periodic 5-point Laplacian (nb - 4p) * inv_h2 (_stencil.pyx:48-63)."""
    from .. import ops
    if _is_tensor(p):
        return ops.laplacian(p, float(inv_h2))
    from .._device import to_dev, to_host
    return to_host(ops.laplacian(to_dev(np.asarray(p)), float(inv_h2)))
