"""paper_2403_07936_b200 -- B200-native (sm_100a) V-cycle hot path of the
arXiv 2403.07936 hybrid multigrid / super-resolution Poisson solver.

Drop-in for the reference package ``mgsr``'s hot path: ``kernels`` (the
stencil backend plugin), ``smoother``, ``transfer``, ``srmodel`` and
``solver`` keep the reference names, arguments and errors; the compute runs
in ``libmgsr_b200.so`` (hand-written CUDA for sm_100a, C ABI in
``include/mgsr_b200.h``), exposed as ``torch.ops.mgsr.*`` custom ops.
"""

__version__ = "0.1.0"

from . import grid, kernels, smoother, solver, srmodel, transfer  # noqa: E402,F401
