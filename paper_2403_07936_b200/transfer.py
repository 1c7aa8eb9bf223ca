"""Grid transfer operators between multigrid levels (mirrors ``mgsr.transfer``,
transfer.py:16-74): injection restriction and separable periodic Keys
(a = -1/2) cubic-convolution prolongation, evaluated by CUDA kernels."""

from __future__ import annotations

from . import ops
from ._device import to_dev, to_host
from .grid import Grid

__all__ = ["PROLONG_RATIOS", "restrict", "spline_prolong"]

PROLONG_RATIOS = (2, 4, 8, 16)


def _check_power_of_two(s: int) -> None:
    if s < 2 or (s & (s - 1)) != 0:
        raise ValueError(f"transfer ratio must be a power of two >= 2, got {s}")


def restrict(fine: Grid, s: int, subtract_mean: bool = True) -> Grid:
    """coarse[i, j] = fine[s i, s j], mean-subtracted by default (transfer.py:27-39)."""
    _check_power_of_two(s)
    if fine.n % s != 0:
        raise ValueError(f"fine side {fine.n} is not divisible by ratio {s}")
    return Grid(to_host(ops.restrict(to_dev(fine.data), int(s), bool(subtract_mean))))


def spline_prolong(coarse: Grid, s: int) -> Grid:
    """Separable periodic cubic interpolation onto an s-times finer grid (transfer.py:64-74)."""
    _check_power_of_two(s)
    if s not in PROLONG_RATIOS:
        raise ValueError(f"prolongation ratio must be one of {PROLONG_RATIOS}, got {s}")
    return Grid(to_host(ops.spline_prolong(to_dev(coarse.data), int(s))))
