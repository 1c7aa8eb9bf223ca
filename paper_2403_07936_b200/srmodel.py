"""Windowed super-resolution prolongation with the SRGAN-style generator.

Mirrors ``mgsr.srmodel`` (srmodel.py:25-487).  Weights are host tensors in
the MGSR1 format (same names, shapes, validation and typed errors); inference
runs on the GPU:

* ``precision="mixed"`` (the default; ``MGSR_PRECISION`` overrides it) -- the tcgen05 tensor-core
  megakernel (fp16 operands, fp32 accumulation in TMEM) for ratio-2 passes on 6x6 windows and
  ratio-4 passes (two applications: full 12x12x3 first output, 12x12 windows of 3 channels
  second), except the first pass of a two-pass ratio (x8 = x4 + x2, x16 = x4 + x4), which runs on
  the fp32 CUDA cores: the second pass re-normalises it logarithmically and amplifies its operand
  rounding ~25x (fp16 throughout: ~5e-2 relL2 at x16; mixed: ~2e-3);
* ``precision="fp16"`` / ``"bf16"`` -- the tensor cores for every pass;
* ``precision="fp32"`` -- CUDA-core fp32 generator (the exact mode: <= 1e-5 of the reference's
  fp64; any window side).
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib, ops
from ._device import to_dev, to_host
from .grid import Grid, NormBounds

__all__ = [
    "GeneratorWeights", "WeightsError", "WeightsMagicError", "WeightsShapeError", "WeightsTruncatedError",
    "WeightsVersionError", "WindowGeometry", "WINDOW", "expected_tensor_shapes", "generator_forward",
    "load_weights", "make_nearest_neighbor_weights", "random_weights", "save_weights", "sr_prolong",
    "stitch_plan", "window_positions",
]

_MAGIC = b"MGSR"
_VERSION = 1
_CHANNELS = 3
_FEATURES = 64
_TANH_SCALE_NAME = "tail.tanh_scale"


class WeightsError(ValueError):
    """Base class for MGSR1 weight-file problems (srmodel.py:52-53)."""


class WeightsMagicError(WeightsError):
    """File does not start with the MGSR magic."""


class WeightsVersionError(WeightsError):
    """Unsupported format version."""


class WeightsShapeError(WeightsError):
    """Tensor set or tensor shapes do not match the architecture."""


class WeightsTruncatedError(WeightsError):
    """File ends before the declared payload."""


@dataclass(frozen=True)
class WindowGeometry:
    """Sliding-window layout of the SR prolongation (srmodel.py:72-87)."""

    n_s: int = 6
    stride: int = 2
    central_lo: int = 2
    central_hi: int = 4

    @property
    def n_l(self) -> int:
        return self.n_s * 4


WINDOW = WindowGeometry()


def expected_tensor_shapes(num_residual_blocks: int) -> dict[str, tuple[int, ...]]:
    """Canonical names/shapes for B residual blocks, in creation order (srmodel.py:90-114)."""
    if num_residual_blocks < 1:
        raise ValueError(f"need >= 1 residual block, got {num_residual_blocks}")
    c, f = _CHANNELS, _FEATURES
    shapes: dict[str, tuple[int, ...]] = {"head.conv.weight": (f, c, 9, 9), "head.prelu.alpha": (f,)}
    for i in range(num_residual_blocks):
        shapes[f"res{i}.conv1.weight"] = (f, f, 3, 3)
        for st in ("gamma", "beta", "mean", "var"):
            shapes[f"res{i}.bn1.{st}"] = (f,)
        shapes[f"res{i}.prelu.alpha"] = (f,)
        shapes[f"res{i}.conv2.weight"] = (f, f, 3, 3)
        for st in ("gamma", "beta", "mean", "var"):
            shapes[f"res{i}.bn2.{st}"] = (f,)
    shapes["post.conv.weight"] = (f, f, 3, 3)
    for st in ("gamma", "beta", "mean", "var"):
        shapes[f"post.bn.{st}"] = (f,)
    shapes["up.conv.weight"] = (f * 4, f, 3, 3)
    shapes["up.prelu.alpha"] = (f,)
    shapes["tail.conv.weight"] = (c, f, 9, 9)
    shapes["tail.conv.bias"] = (c,)
    return shapes


@dataclass
class GeneratorWeights:
    """Named tensors + architecture metadata (srmodel.py:117-162).  The device
    copy (an ``mgsr_gen`` handle) is built lazily and cached."""

    tensors: dict
    num_residual_blocks: int
    upscale_per_pass: int = 2
    tanh_scale: float = 1.0

    def __post_init__(self):
        self.tensors = {k: np.ascontiguousarray(np.asarray(v, dtype=np.float64)) for k, v in self.tensors.items()}
        self._handle = None
        self.validate()

    def validate(self) -> None:
        if self.upscale_per_pass != 2:
            raise WeightsShapeError(f"upscale per pass must be 2, got {self.upscale_per_pass}")
        expected = expected_tensor_shapes(self.num_residual_blocks)
        missing = sorted(expected.keys() - self.tensors.keys())
        if missing:
            raise WeightsShapeError(f"missing tensors: {missing}")
        extra = sorted(self.tensors.keys() - expected.keys())
        if extra:
            raise WeightsShapeError(f"unexpected tensors: {extra}")
        for name, shape in expected.items():
            if self.tensors[name].shape != shape:
                raise WeightsShapeError(f"tensor {name}: expected shape {shape}, got {self.tensors[name].shape}")
        for name, arr in self.tensors.items():
            if name.endswith(".var") and np.any(arr <= 0.0):
                raise WeightsShapeError(f"tensor {name}: variances must be > 0")
        if not (self.tanh_scale >= 1.0):
            raise WeightsShapeError(f"tanh scale must be >= 1, got {self.tanh_scale}")

    # -- device handle -------------------------------------------------------
    def device_handle(self) -> int:
        """mgsr_gen* built from the f32 tensors in expected_tensor_shapes order."""
        if self._handle is None:
            _lib.require_cuda()
            lib = _lib.load()
            names = list(expected_tensor_shapes(self.num_residual_blocks))
            arrs = [np.ascontiguousarray(self.tensors[k], dtype=np.float32) for k in names]
            ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
            out = ctypes.c_void_p()
            _lib.check(lib.mgsr_generator_create(ptrs, len(arrs), self.num_residual_blocks,
                                                 float(self.tanh_scale), ctypes.byref(out)))
            self._handle = out.value
            self._keep = arrs
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h:
            try:
                _lib.load().mgsr_generator_destroy(h)
            except Exception:
                pass


def save_weights(w: GeneratorWeights, path) -> None:
    """MGSR1 writer: magic, <IIII version/upscale/B/count, then per tensor
    (u32 name len, UTF-8 name, u8 dtype 0 = f32, u8 ndim, dims, f32 LE data);
    names sorted, tanh scale record appended only when != 1 (srmodel.py:165-194)."""
    names = sorted(w.tensors)
    extras = [] if w.tanh_scale == 1.0 else [_TANH_SCALE_NAME]
    with open(path, "wb") as fh:
        fh.write(_MAGIC + struct.pack("<IIII", _VERSION, w.upscale_per_pass, w.num_residual_blocks,
                                      len(names) + len(extras)))
        for name in names + extras:
            arr = np.asarray(w.tensors[name]) if name in w.tensors else np.asarray(np.float64(w.tanh_scale))
            raw = name.encode("utf-8")
            fh.write(struct.pack("<I", len(raw)) + raw + struct.pack("<BB", 0, arr.ndim))
            fh.write(struct.pack(f"<{arr.ndim}I", *arr.shape))
            fh.write(arr.astype("<f4").tobytes(order="C"))


def load_weights(path) -> GeneratorWeights:
    """Read and validate an MGSR1 file (srmodel.py:197-248)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    pos = 0

    def take(count: int) -> bytes:
        nonlocal pos
        if pos + count > len(blob):
            raise WeightsTruncatedError(f"need {pos + count} bytes, file has {len(blob)}")
        out = blob[pos:pos + count]
        pos += count
        return out

    magic = take(4)
    if magic != _MAGIC:
        raise WeightsMagicError(f"bad magic {magic!r}, expected {_MAGIC!r}")
    version, upscale, blocks, count = struct.unpack("<IIII", take(16))
    if version != _VERSION:
        raise WeightsVersionError(f"unsupported version {version}")
    tensors: dict[str, np.ndarray] = {}
    for _ in range(count):
        (nlen,) = struct.unpack("<I", take(4))
        name = take(nlen).decode("utf-8")
        dtype, ndim = struct.unpack("<BB", take(2))
        if dtype != 0:
            raise WeightsShapeError(f"tensor {name}: unsupported dtype {dtype}")
        dims = struct.unpack(f"<{ndim}I", take(4 * ndim)) if ndim else ()
        size = int(np.prod(dims, dtype=np.int64)) if ndim else 1
        raw = take(4 * size)
        if name in tensors:
            raise WeightsShapeError(f"duplicate tensor {name}")
        tensors[name] = np.frombuffer(raw, dtype="<f4").reshape(dims).astype(np.float64)
    if pos != len(blob):
        raise WeightsShapeError(f"trailing bytes after {count} tensors")
    tanh_scale = 1.0
    if _TANH_SCALE_NAME in tensors:
        scale = tensors.pop(_TANH_SCALE_NAME)
        if scale.shape != ():
            raise WeightsShapeError(f"{_TANH_SCALE_NAME} must be a scalar")
        tanh_scale = float(scale)
    return GeneratorWeights(tensors=tensors, num_residual_blocks=blocks, upscale_per_pass=upscale,
                            tanh_scale=tanh_scale)


def make_nearest_neighbor_weights(num_residual_blocks: int = 1) -> GeneratorWeights:
    """Weights making the generator an exact x2 nearest-neighbour upsampler (srmodel.py:361-387)."""
    t = {k: np.zeros(s) for k, s in expected_tensor_shapes(num_residual_blocks).items()}
    for k in t:
        if k.endswith(".var") or k.endswith("prelu.alpha"):
            t[k][:] = 1.0
    for c in range(_CHANNELS):
        t["head.conv.weight"][c, c, 4, 4] = 1.0
        t["tail.conv.weight"][c, c, 4, 4] = 1.0
    for c in range(_FEATURES):
        for di in range(2):
            for dj in range(2):
                t["up.conv.weight"][c * 4 + di * 2 + dj, c, 1, 1] = 1.0
    return GeneratorWeights(tensors=t, num_residual_blocks=num_residual_blocks, tanh_scale=1e6)


def random_weights(num_residual_blocks: int, seed: int) -> GeneratorWeights:
    """He-normal conv weights, identity BN statistics, PReLU 0.25 (srmodel.py:390-407)."""
    rng = np.random.default_rng(seed)
    t: dict[str, np.ndarray] = {}
    for name, shape in expected_tensor_shapes(num_residual_blocks).items():
        if name.endswith(("conv.weight", "conv1.weight", "conv2.weight")):
            t[name] = rng.normal(0.0, np.sqrt(2.0 / (shape[1] * shape[2] * shape[3])), shape)
        elif name.endswith((".gamma", ".var")):
            t[name] = np.ones(shape)
        elif name.endswith("prelu.alpha"):
            t[name] = np.full(shape, 0.25)
        else:
            t[name] = np.zeros(shape)
    return GeneratorWeights(tensors=t, num_residual_blocks=num_residual_blocks)


def generator_forward(w: GeneratorWeights, x: np.ndarray) -> np.ndarray:
    """Generator on one (3, n, n) input -> (3, 2n, 2n) (srmodel.py:347-354); fp32 CUDA cores."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 3 or x.shape[0] != _CHANNELS:
        raise ValueError(f"input must have shape (3, n, n), got {x.shape}")
    if x.shape[1] < WINDOW.n_s or x.shape[1] != x.shape[2]:
        raise ValueError(f"input must be square with side >= {WINDOW.n_s}")
    return to_host(ops.generator_forward(to_dev(x[None]), w.device_handle()))[0]


def window_positions(n_coarse: int) -> list[int]:
    """Window corners 0, 2, ..., n_coarse - 6 (srmodel.py:414-420)."""
    if n_coarse < WINDOW.n_s:
        raise ValueError(f"coarse side must be >= {WINDOW.n_s}, got {n_coarse}")
    if n_coarse % 2 != 0:
        raise ValueError(f"coarse side must be even, got {n_coarse}")
    return list(range(0, n_coarse - WINDOW.n_s + 1, WINDOW.stride))


def stitch_plan(n_coarse: int) -> list[tuple[int, int, slice, slice]]:
    """Windows and the coarse-cell band each contributes (srmodel.py:423-440)."""
    pos = window_positions(n_coarse)
    last = pos[-1]
    plan = []
    for i_w in pos:
        lo_i = 0 if i_w == 0 else WINDOW.central_lo
        hi_i = WINDOW.n_s if i_w == last else WINDOW.central_hi
        for j_w in pos:
            lo_j = 0 if j_w == 0 else WINDOW.central_lo
            hi_j = WINDOW.n_s if j_w == last else WINDOW.central_hi
            plan.append((i_w, j_w, slice(lo_i, hi_i), slice(lo_j, hi_j)))
    return plan


_PASS_PLAN = {2: (1,), 4: (2,), 8: (2, 1), 16: (2, 2)}


def sr_prolong(coarse: Grid, w: GeneratorWeights, b: NormBounds, s: int, precision: str | None = None) -> Grid:
    """SR prolongation by s in {2, 4, 8, 16} (srmodel.py:470-487), on the GPU."""
    precision = _lib.precision(precision)
    if s not in _PASS_PLAN:
        raise ValueError(f"unsupported SR ratio {s}; expected one of {sorted(_PASS_PLAN)}")
    window_positions(coarse.n)
    out = ops.sr_prolong(to_dev(coarse.data), w.device_handle(), int(s), float(b.p_min), float(b.p_max),
                         _lib.PREC[precision])
    return Grid(to_host(out))
