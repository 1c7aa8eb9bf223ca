"""Host <-> device staging for the reference-shaped (host Grid) API."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def to_dev(a: np.ndarray):
    torch = _lib.require_cuda()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda", non_blocking=False)


def to_host(t) -> np.ndarray:
    return t.detach().to("cpu").numpy()


def rms_diff(a: np.ndarray, b: np.ndarray | None) -> float:
    torch = _lib.require_cuda()
    from .ops import workspace
    lib = _lib.load()
    da = to_dev(a)
    db = to_dev(b) if b is not None else None
    nb = lib.mgsr_workspace_bytes(da.shape[0])
    ws = workspace(nb, da.device)
    out = ctypes.c_double(0.0)
    _lib.check(lib.mgsr_rms_diff(da.data_ptr(), db.data_ptr() if db is not None else None, da.numel(),
                                 ctypes.byref(out), ws.data_ptr(), nb, torch.cuda.current_stream().cuda_stream))
    return float(out.value)
