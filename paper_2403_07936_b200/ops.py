"""PyTorch custom ops (``torch.ops.mgsr.*``) over the C ABI.

Each op takes CUDA float64 tensors, launches on the current torch stream and
calls straight into libmgsr_b200.so; there is no CPU implementation.
"""

from __future__ import annotations

import torch

from . import _lib

_ws_cache: dict[int, torch.Tensor] = {}


def workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    """Per-device scratch buffer, grown on demand (caller-owned memory for the C ABI)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    buf = _ws_cache.get(idx)
    if buf is None or buf.numel() < nbytes:
        buf = torch.zeros(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=device)
        _ws_cache[idx] = buf
    return buf


def _check_t(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous CUDA float64 tensor")


def _st() -> int:
    return torch.cuda.current_stream().cuda_stream


@torch.library.custom_op("mgsr::gs_sweeps_", mutates_args=("p",))
def gs_sweeps_(p: torch.Tensor, f: torch.Tensor, h2: float, sweeps: int) -> None:
    """In-place red-black Gauss-Seidel (kernels.gs_sweeps, _stencil.pyx:12-45)."""
    _check_t(p, "p"); _check_t(f, "f")
    lib = _lib.load()
    n = p.shape[0]
    nb = lib.mgsr_workspace_bytes(n)
    ws = workspace(nb, p.device)
    _lib.check(lib.mgsr_gs_sweeps(p.data_ptr(), f.data_ptr(), n, float(h2), int(sweeps), ws.data_ptr(), nb, _st()))


@torch.library.custom_op("mgsr::laplacian", mutates_args=())
def laplacian(p: torch.Tensor, inv_h2: float) -> torch.Tensor:
    """Periodic 5-point Laplacian (kernels.laplacian, _stencil.pyx:48-63)."""
    _check_t(p, "p")
    out = torch.empty_like(p)
    _lib.check(_lib.load().mgsr_laplacian(p.data_ptr(), out.data_ptr(), p.shape[0], float(inv_h2), _st()))
    return out


@torch.library.custom_op("mgsr::residual", mutates_args=())
def residual(p: torch.Tensor, f: torch.Tensor) -> torch.Tensor:
    """Mean-subtracted r = f - L p (smoother.residual, smoother.py:52-57)."""
    _check_t(p, "p"); _check_t(f, "f")
    lib = _lib.load()
    n = p.shape[0]
    nb = lib.mgsr_workspace_bytes(n)
    ws = workspace(nb, p.device)
    out = torch.empty_like(p)
    _lib.check(lib.mgsr_residual(p.data_ptr(), f.data_ptr(), out.data_ptr(), n, ws.data_ptr(), nb, _st()))
    return out


@torch.library.custom_op("mgsr::restrict", mutates_args=())
def restrict(fine: torch.Tensor, s: int, subtract_mean: bool) -> torch.Tensor:
    """Injection restriction (transfer.restrict, transfer.py:27-39)."""
    _check_t(fine, "fine")
    lib = _lib.load()
    n = fine.shape[0]
    nc = n // s if s > 0 and n % s == 0 else 1
    out = torch.empty((nc, nc), dtype=torch.float64, device=fine.device)
    nb = lib.mgsr_workspace_bytes(n)
    ws = workspace(nb, fine.device)
    _lib.check(lib.mgsr_restrict(fine.data_ptr(), out.data_ptr(), n, int(s), int(bool(subtract_mean)),
                                 ws.data_ptr(), nb, _st()))
    return out


@torch.library.custom_op("mgsr::spline_prolong", mutates_args=())
def spline_prolong(c: torch.Tensor, s: int) -> torch.Tensor:
    """Separable periodic Keys interpolation (transfer.spline_prolong, transfer.py:64-74)."""
    _check_t(c, "coarse")
    nc = c.shape[0]
    out = torch.empty((nc * max(s, 1), nc * max(s, 1)), dtype=torch.float64, device=c.device)
    _lib.check(_lib.load().mgsr_spline_prolong(c.data_ptr(), nc, int(s), out.data_ptr(), _st()))
    return out


@torch.library.custom_op("mgsr::sr_prolong", mutates_args=())
def sr_prolong(c: torch.Tensor, gen: int, s: int, p_min: float, p_max: float, precision: int) -> torch.Tensor:
    """Windowed SR prolongation (srmodel.sr_prolong, srmodel.py:470-487)."""
    _check_t(c, "coarse")
    lib = _lib.load()
    nc = c.shape[0]
    out = torch.empty((nc * s, nc * s), dtype=torch.float64, device=c.device)
    nb = lib.mgsr_sr_workspace_bytes(nc, int(s))
    ws = workspace(nb, c.device)
    _lib.check(lib.mgsr_sr_prolong(gen, c.data_ptr(), nc, int(s), float(p_min), float(p_max), int(precision),
                                   out.data_ptr(), ws.data_ptr(), nb, _st()))
    return out


@torch.library.custom_op("mgsr::generator_forward", mutates_args=())
def generator_forward(x: torch.Tensor, gen: int) -> torch.Tensor:
    """Generator on a batch (N,3,h,h) -> (N,3,2h,2h) (srmodel._forward_batch, srmodel.py:330-344)."""
    _check_t(x, "x")
    n, _, h, _ = x.shape
    y = torch.empty((n, 3, 2 * h, 2 * h), dtype=torch.float64, device=x.device)
    _lib.check(_lib.load().mgsr_generator_forward(gen, x.data_ptr(), n, h, y.data_ptr(), _st()))
    return y


@torch.library.custom_op("mgsr::vcycle_", mutates_args=("p", "stats"))
def vcycle_(p: torch.Tensor, f: torch.Tensor, plan: int, use_sr: int, stats: torch.Tensor) -> None:
    """One graph-launched V-cycle + logging pass (solver.v_cycle + solver.py:312-313)."""
    _check_t(p, "p"); _check_t(f, "f"); _check_t(stats, "stats")
    _lib.check(_lib.load().mgsr_plan_vcycle(plan, p.data_ptr(), f.data_ptr(), int(use_sr), stats.data_ptr(), _st()))


# Fake (meta) kernels: output shapes and dtypes for tracing / FakeTensor propagation (no compute, no library).
@gs_sweeps_.register_fake
def _(p, f, h2, sweeps):
    return None


@laplacian.register_fake
def _(p, inv_h2):
    return torch.empty_like(p)


@residual.register_fake
def _(p, f):
    return torch.empty_like(p)


@restrict.register_fake
def _(fine, s, subtract_mean):
    n = fine.shape[0]
    nc = n // s if s > 0 and n % s == 0 else 1
    return fine.new_empty((nc, nc))


@spline_prolong.register_fake
def _(c, s):
    return c.new_empty((c.shape[0] * max(s, 1), c.shape[0] * max(s, 1)))


@sr_prolong.register_fake
def _(c, gen, s, p_min, p_max, precision):
    return c.new_empty((c.shape[0] * s, c.shape[0] * s))


@generator_forward.register_fake
def _(x, gen):
    return x.new_empty((x.shape[0], 3, 2 * x.shape[2], 2 * x.shape[3]))


@vcycle_.register_fake
def _(p, f, plan, use_sr, stats):
    return None
