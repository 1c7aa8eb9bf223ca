"""ctypes binding of the C ABI in include/mgsr_b200.h (libmgsr_b200.so).

The library is loaded lazily; any compute call without it (or without a CUDA
device) raises -- there is no CPU fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MGSR_LIB") or os.path.join(HERE, "libmgsr_b200.so")

_PROFILER_ENV = ("MGSR_NO_GRAPH", "CUDA_INJECTION64_PATH", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE",
                 "NV_TPS_LAUNCH_TOKEN", "NV_COMPUTE_PROFILER_PERFWORKS_DIR")


def graphs_disabled() -> bool:
    """Same rule as plan.cu: MGSR_NO_GRAPH=1, or an injected profiler (Nsight Compute fails the first
    kernel launched into a stream capture), makes the plan issue its kernel sequence eagerly; the
    device-resident solve loop (graph conditional nodes) is then replaced by the per-cycle loop."""
    return any(os.environ.get(k) for k in _PROFILER_ENV)


MGSR_OK = 0
MGSR_E_CUDA = -8
PREC = {"fp32": 0, "bf16": 1, "fp16": 2, "mixed": 3}


def precision(p: str | None) -> str:
    """Generator precision of an operator call: an explicit argument wins, else ``MGSR_PRECISION``, else
    "mixed": the tcgen05 tensor-core generator with fp16 operands, except the first pass of a two-pass
    ratio (x8, x16), which runs on the fp32 CUDA cores because the second pass amplifies its rounding
    ~25x.  "fp16" / "bf16": tensor cores for every pass; "fp32": the exact CUDA-core mode."""
    import os
    p = p if p is not None else os.environ.get("MGSR_PRECISION", "mixed")
    if p not in PREC:
        raise ValueError(f"precision must be one of {sorted(PREC)}, got {p!r}")
    return p

_lock = threading.Lock()
_lib = None

c_double_p = ctypes.POINTER(ctypes.c_double)
vp = ctypes.c_void_p
i64, i32, u32, f64, sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_double, ctypes.c_size_t


class PlanConfig(ctypes.Structure):
    _fields_ = [("n", i64), ("n_step", i32), ("r_min", i32), ("n_smooth", i32), ("coarse_sweeps", i32),
                ("p_min", f64), ("p_max", f64), ("precision", i32), ("sr_level_mask", u32)]


# name -> (restype, argtypes); mirrors include/mgsr_b200.h one to one
SIGNATURES = {
    "mgsr_last_error": (ctypes.c_char_p, []),
    "mgsr_version": (ctypes.c_char_p, []),
    "mgsr_workspace_bytes": (sz, [i64]),
    "mgsr_gs_sweeps": (ctypes.c_int, [vp, vp, i64, f64, i32, vp, sz, vp]),
    "mgsr_laplacian": (ctypes.c_int, [vp, vp, i64, f64, vp]),
    "mgsr_residual": (ctypes.c_int, [vp, vp, vp, i64, vp, sz, vp]),
    "mgsr_restrict": (ctypes.c_int, [vp, vp, i64, i32, i32, vp, sz, vp]),
    "mgsr_spline_prolong": (ctypes.c_int, [vp, i64, i32, vp, vp]),
    "mgsr_rms_diff": (ctypes.c_int, [vp, vp, i64, c_double_p, vp, sz, vp]),
    "mgsr_generator_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), i32, i32, f64,
                                             ctypes.POINTER(ctypes.c_void_p)]),
    "mgsr_generator_destroy": (ctypes.c_int, [vp]),
    "mgsr_generator_forward": (ctypes.c_int, [vp, vp, i64, i64, vp, vp]),
    "mgsr_sr_workspace_bytes": (sz, [i64, i32]),
    "mgsr_sr_prolong": (ctypes.c_int, [vp, vp, i64, i32, f64, f64, i32, vp, vp, sz, vp]),
    "mgsr_plan_create": (ctypes.c_int, [ctypes.POINTER(PlanConfig), vp, ctypes.POINTER(ctypes.c_void_p)]),
    "mgsr_plan_destroy": (ctypes.c_int, [vp]),
    "mgsr_plan_levels": (i32, [vp, ctypes.POINTER(i64)]),
    "mgsr_plan_vcycle": (ctypes.c_int, [vp, vp, vp, i32, vp, vp]),
    "mgsr_plan_solve": (ctypes.c_int, [vp, vp, vp, i32, i32, f64, f64, i32, i32, i32, vp, vp, vp]),
    "mgsr_plan_solve_batch": (ctypes.c_int, [vp, i32, vp, vp, i32, i32, f64, f64, i32, i32, i32, vp, vp, vp]),
    "mgsr_plan_timing_enable": (ctypes.c_int, [vp, i32]),
    "mgsr_plan_timing_read": (ctypes.c_int, [vp, c_double_p, ctypes.POINTER(i32)]),
    "mgsr_plan_kernel_nodes": (i32, [vp, i32]),
    "mgsr_initial_iterate_workspace_bytes": (sz, [i64]),
    "mgsr_initial_iterate": (ctypes.c_int, [vp, i64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.c_uint64, f64, f64, vp, sz, vp]),
}


class MgsrError(ValueError):
    """Error reported by the CUDA library (ValueError, like the reference's checks)."""


class MgsrCudaError(RuntimeError):
    """CUDA runtime failure inside the library."""


def load(path: str = LIB_PATH):
    """Load the shared library and bind every exported symbol (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"mgsr_b200 CUDA library not found at {path}; build it with "
                "`python -m paper_2403_07936_b200.build` (there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == MGSR_OK:
        return
    msg = load().mgsr_last_error().decode(errors="replace")
    if rc == MGSR_E_CUDA:
        raise MgsrCudaError(msg)
    raise MgsrError(msg)


def require_cuda():
    """Return torch with a usable CUDA device or raise loudly."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2403_07936_b200 requires a CUDA (sm_100a) device; there is no CPU fallback")
    load()
    return torch


def stream_ptr(torch_mod=None) -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream
