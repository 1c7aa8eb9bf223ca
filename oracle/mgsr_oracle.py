"""CPU oracle for the mgsr V-cycle hot path -- TEST INFRASTRUCTURE ONLY.

This module is a from-scratch NumPy restatement of the reference algorithm
(arXiv 2403.07936 reference package ``mgsr``).  It exists so that the tests,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` leg can check
the CUDA path; the product package (``paper_2403_07936_b200``) never imports
it.  Every function cites the reference file:line it restates (paths relative
to ``/root/reference/pkg/src/mgsr``).

Parity is PINNED: ``tests/golden/`` holds vectors produced by importing the
reference itself (script ``tests/golden/make_golden.py``), and
``tests/test_oracle.py`` checks this restatement against them.  When
``oracle/_ref`` (the reference compiled from its own sources by
``oracle/build_ref.py``) is present, the tests also compare against it live.

Deliberate deviations (all measured <= 6e-16 relative by the survey):
* ``spline_prolong`` uses the separable banded 4-tap form instead of the
  dense ``op @ c @ op.T`` sandwich (transfer.py:64-74).
* the C twin of ``gs_sweeps`` (``oracle/stencil.c``) follows the Cython
  backend's sequential mean; the NumPy form here follows numpy_backend.py.
"""

from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# stencil kernels  (kernels/_stencil.pyx:12-63, kernels/numpy_backend.py:33-56)

_HERE = os.path.dirname(os.path.abspath(__file__))
_clib = None


def _load_c():
    """The gcc-built C twin of the stencil loops (oracle/stencil.c)."""
    global _clib
    if _clib is None:
        path = os.path.join(_HERE, "libmgsr_oracle.so")
        if not os.path.exists(path):
            return None
        lib = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_gs_sweeps.argtypes = [dp, dp, ctypes.c_long, ctypes.c_double, ctypes.c_int]
        lib.oracle_gs_sweeps.restype = None
        lib.oracle_laplacian.argtypes = [dp, dp, ctypes.c_long, ctypes.c_double]
        lib.oracle_laplacian.restype = None
        _clib = lib
    return _clib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _neighbor_sum(p: np.ndarray) -> np.ndarray:
    # ((up + down) + left) + right, exactly the reference's association order
    # (_stencil.pyx:36, numpy_backend.py:26-29)
    return ((np.roll(p, 1, 0) + np.roll(p, -1, 0)) + np.roll(p, 1, 1)) + np.roll(p, -1, 1)


def gs_sweeps(p: np.ndarray, f: np.ndarray, h2: float, sweeps: int, use_c: bool = True) -> None:
    """In-place red-black Gauss-Seidel, red = (i+j) even first, then black,
    each sweep followed by subtraction of the grid mean.
    Reference: _stencil.pyx:12-45 (numpy twin numpy_backend.py:33-51)."""
    n = p.shape[0]
    if n % 2 != 0:
        raise ValueError(f"red-black coloring needs an even side, got {n}")
    if f.shape != p.shape:
        raise ValueError("p and f shapes differ")
    lib = _load_c() if use_c else None
    if lib is not None and p.flags.c_contiguous and p.dtype == np.float64:
        fc = np.ascontiguousarray(f, dtype=np.float64)
        lib.oracle_gs_sweeps(_ptr(p), _ptr(fc), n, float(h2), int(sweeps))
        return
    idx = np.add.outer(np.arange(n), np.arange(n))
    red = (idx % 2) == 0
    h2f = h2 * f
    for _ in range(sweeps):
        for mask in (red, ~red):
            upd = (_neighbor_sum(p) - h2f) * 0.25
            p[mask] = upd[mask]
        p -= p.mean()


def laplacian(p: np.ndarray, inv_h2: float) -> np.ndarray:
    """Periodic 5-point Laplacian (nb - 4p) * inv_h2. Reference: _stencil.pyx:48-63."""
    return (_neighbor_sum(p) - 4.0 * p) * inv_h2


# ---------------------------------------------------------------------------
# fields (grid.py:36-114)

def diff_norm(a: np.ndarray, b: np.ndarray) -> float:
    """RMS difference (grid.py:74-78)."""
    return float(np.sqrt(np.mean((a - b) ** 2)))


def rms(a: np.ndarray) -> float:
    """Grid.rms (grid.py:70-71)."""
    return float(np.sqrt(np.mean(a ** 2)))


@dataclass(frozen=True)
class Bounds:
    """NormBounds (grid.py:81-100): defaults p_min 1e-10, p_max 1e-3."""
    p_min: float = 1e-10
    p_max: float = 1e-3

    @property
    def log_lo(self) -> float:
        return float(np.log10(self.p_min))

    @property
    def log_span(self) -> float:
        return float(np.log10(self.p_max) - np.log10(self.p_min))


def normalize(p: np.ndarray, b: Bounds) -> np.ndarray:
    """q = clip((log10|p| - log_lo)/span, 0, 1) * sign(p) (grid.py:103-109)."""
    with np.errstate(divide="ignore"):
        t = (np.log10(np.abs(p)) - b.log_lo) / b.log_span
    return np.clip(t, 0.0, 1.0) * np.sign(p)


def denormalize(q: np.ndarray, signs: np.ndarray, b: Bounds) -> np.ndarray:
    """p = sign * 10**(log_lo + |q| span) (grid.py:112-114)."""
    return signs * 10.0 ** (b.log_lo + np.abs(q) * b.log_span)


# ---------------------------------------------------------------------------
# smoother (smoother.py:22-75)

def check_rhs(f: np.ndarray) -> None:
    """PoissonProblem mean-free check (smoother.py:28-34)."""
    mean = abs(float(f.mean()))
    if mean > 1e-12 * max(rms(f), 1e-300):
        raise ValueError(f"RHS mean {mean:.3e} is not zero within 1e-12 * RMS; mean-free f required")


def residual(p: np.ndarray, f: np.ndarray) -> np.ndarray:
    """r = f - L p, then minus its mean (smoother.py:52-57)."""
    n = p.shape[0]
    h = 2.0 * np.pi / n
    r = f - laplacian(p, 1.0 / (h * h))
    return r - r.mean()


def gauss_seidel(p: np.ndarray, f: np.ndarray, sweeps: int) -> np.ndarray:
    """Copying wrapper around gs_sweeps (smoother.py:60-75)."""
    if sweeps < 0:
        raise ValueError(f"sweep count must be >= 0, got {sweeps}")
    out = p.copy()
    if sweeps:
        n = p.shape[0]
        h = 2.0 * np.pi / n
        gs_sweeps(out, f, h * h, sweeps)
    return out


# ---------------------------------------------------------------------------
# transfer (transfer.py:19-74)

PROLONG_RATIOS = (2, 4, 8, 16)


def restrict(fine: np.ndarray, s: int, subtract_mean: bool = True) -> np.ndarray:
    """Injection coarse = fine[::s, ::s] (minus its mean) (transfer.py:27-39)."""
    if s < 2 or (s & (s - 1)) != 0:
        raise ValueError(f"transfer ratio must be a power of two >= 2, got {s}")
    if fine.shape[0] % s != 0:
        raise ValueError(f"fine side {fine.shape[0]} is not divisible by ratio {s}")
    c = fine[::s, ::s].copy()
    if subtract_mean:
        c -= c.mean()
    return c


def keys_weight(d):
    """Keys cubic convolution, a = -1/2 (transfer.py:42-47)."""
    d = np.abs(d)
    near = (1.5 * d - 2.5) * d * d + 1.0
    far = ((-0.5 * d + 2.5) * d - 4.0) * d + 2.0
    return np.where(d <= 1.0, near, np.where(d < 2.0, far, 0.0))


def prolong_taps(s: int) -> np.ndarray:
    """Per-phase 4-tap weights w[phase, offset+1] for offsets -1..2
    (the non-zero band of _prolong_matrix, transfer.py:50-61)."""
    t = np.arange(s) / s
    return np.stack([keys_weight(t - o) for o in (-1, 0, 1, 2)], axis=1)


def _prolong_1d(c: np.ndarray, s: int, axis: int) -> np.ndarray:
    n = c.shape[axis]
    w = prolong_taps(s)
    base = np.arange(n * s) // s
    phase = np.arange(n * s) % s
    out = 0.0
    for k, o in enumerate((-1, 0, 1, 2)):
        idx = (base + o) % n
        wk = w[phase, k]
        if axis == 0:
            out = out + wk[:, None] * c[idx, :]
        else:
            out = out + wk[None, :] * c[:, idx]
    return out


def spline_prolong(c: np.ndarray, s: int) -> np.ndarray:
    """Separable periodic cubic-convolution interpolation (transfer.py:64-74),
    evaluated as the banded 4-tap form of op @ c @ op.T."""
    if s < 2 or (s & (s - 1)) != 0:
        raise ValueError(f"transfer ratio must be a power of two >= 2, got {s}")
    if s not in PROLONG_RATIOS:
        raise ValueError(f"prolongation ratio must be one of {PROLONG_RATIOS}, got {s}")
    return _prolong_1d(_prolong_1d(c, s, 0), s, 1)


# ---------------------------------------------------------------------------
# generator (srmodel.py:45-407)

CHANNELS, FEATURES = 3, 64
N_S, STRIDE, C_LO, C_HI = 6, 2, 2, 4          # WindowGeometry (srmodel.py:72-87)


def tensor_shapes(blocks: int) -> dict:
    """expected_tensor_shapes (srmodel.py:90-114)."""
    c, f = CHANNELS, FEATURES
    s = {"head.conv.weight": (f, c, 9, 9), "head.prelu.alpha": (f,)}
    for i in range(blocks):
        s[f"res{i}.conv1.weight"] = (f, f, 3, 3)
        for st in ("gamma", "beta", "mean", "var"):
            s[f"res{i}.bn1.{st}"] = (f,)
        s[f"res{i}.prelu.alpha"] = (f,)
        s[f"res{i}.conv2.weight"] = (f, f, 3, 3)
        for st in ("gamma", "beta", "mean", "var"):
            s[f"res{i}.bn2.{st}"] = (f,)
    s["post.conv.weight"] = (f, f, 3, 3)
    for st in ("gamma", "beta", "mean", "var"):
        s[f"post.bn.{st}"] = (f,)
    s["up.conv.weight"] = (4 * f, f, 3, 3)
    s["up.prelu.alpha"] = (f,)
    s["tail.conv.weight"] = (c, f, 9, 9)
    s["tail.conv.bias"] = (c,)
    return s


@dataclass
class Weights:
    tensors: dict
    blocks: int
    tanh_scale: float = 1.0


def read_mgsr1(path) -> Weights:
    """MGSR1 reader (srmodel.py:197-248): magic, <IIII version/upscale/B/count,
    then (u32 len, name, u8 dtype=0, u8 ndim, ndim*u32, f32 data)."""
    blob = open(path, "rb").read()
    if blob[:4] != b"MGSR":
        raise ValueError("bad magic")
    version, upscale, blocks, count = struct.unpack_from("<IIII", blob, 4)
    pos = 20
    t = {}
    for _ in range(count):
        (ln,) = struct.unpack_from("<I", blob, pos); pos += 4
        name = blob[pos:pos + ln].decode(); pos += ln
        dtype, ndim = struct.unpack_from("<BB", blob, pos); pos += 2
        dims = struct.unpack_from(f"<{ndim}I", blob, pos) if ndim else (); pos += 4 * ndim
        size = int(np.prod(dims)) if ndim else 1
        t[name] = np.frombuffer(blob, "<f4", size, pos).reshape(dims).astype(np.float64); pos += 4 * size
    scale = float(t.pop("tail.tanh_scale")) if "tail.tanh_scale" in t else 1.0
    return Weights(t, blocks, scale)


def write_mgsr1(w: Weights, path) -> None:
    """MGSR1 writer (srmodel.py:165-194): sorted names, tanh scale last if != 1."""
    names = sorted(w.tensors)
    extra = [] if w.tanh_scale == 1.0 else ["tail.tanh_scale"]
    with open(path, "wb") as fh:
        fh.write(b"MGSR" + struct.pack("<IIII", 1, 2, w.blocks, len(names) + len(extra)))
        for name in names + extra:
            arr = np.asarray(w.tensors[name] if name in w.tensors else np.float64(w.tanh_scale))
            raw = name.encode()
            fh.write(struct.pack("<I", len(raw)) + raw + struct.pack("<BB", 0, arr.ndim))
            fh.write(struct.pack(f"<{arr.ndim}I", *arr.shape))
            fh.write(arr.astype("<f4").tobytes(order="C"))


def random_weights(blocks: int, seed: int) -> Weights:
    """He-normal init with identity BN statistics (srmodel.py:390-407); the
    draw order follows expected_tensor_shapes' insertion order."""
    rng = np.random.default_rng(seed)
    t = {}
    for name, shape in tensor_shapes(blocks).items():
        if name.endswith(("conv.weight", "conv1.weight", "conv2.weight")):
            t[name] = rng.normal(0.0, np.sqrt(2.0 / (shape[1] * shape[2] * shape[3])), shape)
        elif name.endswith((".gamma", ".var")):
            t[name] = np.ones(shape)
        elif name.endswith("prelu.alpha"):
            t[name] = np.full(shape, 0.25)
        else:
            t[name] = np.zeros(shape)
    return Weights(t, blocks)


def nn_weights(blocks: int = 1) -> Weights:
    """Exact x2 nearest-neighbour upsampler (srmodel.py:361-387)."""
    t = {k: np.zeros(s) for k, s in tensor_shapes(blocks).items()}
    for k in t:
        if k.endswith(".var") or k.endswith("prelu.alpha"):
            t[k][:] = 1.0
    for c in range(CHANNELS):
        t["head.conv.weight"][c, c, 4, 4] = 1.0
        t["tail.conv.weight"][c, c, 4, 4] = 1.0
    for c in range(FEATURES):
        for di in range(2):
            for dj in range(2):
                t["up.conv.weight"][c * 4 + di * 2 + dj, c, 1, 1] = 1.0
    return Weights(t, blocks, 1e6)


def quantize_f32(w: Weights) -> Weights:
    """What a MGSR1 round trip does to the values (f32 storage, srmodel.py:189, 233)."""
    return Weights({k: v.astype(np.float32).astype(np.float64) for k, v in w.tensors.items()},
                   w.blocks, float(np.float32(w.tanh_scale)))


def conv2d(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Same-size correlation with replicate padding (srmodel.py:285-305), im2col form."""
    n, c, hh, ww = x.shape
    o, _, kh, kw = w.shape
    xp = np.pad(x, ((0, 0), (0, 0), (kh // 2, kh // 2), (kw // 2, kw // 2)), mode="edge")
    out = np.zeros((n, hh, ww, o))
    wm = w.transpose(2, 3, 1, 0)  # (kh, kw, c, o)
    xt = xp.transpose(0, 2, 3, 1)  # (n, H, W, c)
    for dy in range(kh):
        for dx in range(kw):
            out += xt[:, dy:dy + hh, dx:dx + ww, :] @ wm[dy, dx]
    return out.transpose(0, 3, 1, 2)


def _prelu(x, a):
    return np.where(x > 0.0, x, a[None, :, None, None] * x)


def _bn(x, t, pre):
    g, b, m, v = (t[f"{pre}.{s}"][None, :, None, None] for s in ("gamma", "beta", "mean", "var"))
    return g * (x - m) / np.sqrt(v + 1e-5) + b


def pixel_shuffle(x: np.ndarray, r: int = 2) -> np.ndarray:
    """(N, C r r, H, W) -> (N, C, H r, W r), channel c*r*r + i*r + j -> offset (i, j)
    (srmodel.py:321-327)."""
    nb, crr, h, w = x.shape
    c = crr // (r * r)
    return x.reshape(nb, c, r, r, h, w).transpose(0, 1, 4, 2, 5, 3).reshape(nb, c, h * r, w * r)


def forward_batch(w: Weights, x: np.ndarray, chunk: int = 512) -> np.ndarray:
    """Generator (N,3,n,n) -> (N,3,2n,2n) (srmodel.py:330-344)."""
    if x.shape[0] > chunk:
        return np.concatenate([forward_batch(w, x[i:i + chunk], chunk)
                               for i in range(0, x.shape[0], chunk)], axis=0)
    t = w.tensors
    y = _prelu(conv2d(x, t["head.conv.weight"]), t["head.prelu.alpha"])
    skip = y
    for i in range(w.blocks):
        z = _prelu(_bn(conv2d(y, t[f"res{i}.conv1.weight"]), t, f"res{i}.bn1"), t[f"res{i}.prelu.alpha"])
        y = y + _bn(conv2d(z, t[f"res{i}.conv2.weight"]), t, f"res{i}.bn2")
    y = _bn(conv2d(y, t["post.conv.weight"]), t, "post.bn") + skip
    y = _prelu(pixel_shuffle(conv2d(y, t["up.conv.weight"])), t["up.prelu.alpha"])
    y = conv2d(y, t["tail.conv.weight"]) + t["tail.conv.bias"][None, :, None, None]
    s = w.tanh_scale
    return s * np.tanh(y / s)


def window_positions(n: int) -> list:
    """Corners 0, 2, ..., n-6 (srmodel.py:414-420)."""
    if n < N_S:
        raise ValueError(f"coarse side must be >= {N_S}, got {n}")
    if n % 2:
        raise ValueError(f"coarse side must be even, got {n}")
    return list(range(0, n - N_S + 1, STRIDE))


def stitch_plan(n: int) -> list:
    """(i_w, j_w, lo_i, hi_i, lo_j, hi_j) bands tiling [0,n)^2 once (srmodel.py:423-440)."""
    pos = window_positions(n)
    last = pos[-1]
    plan = []
    for iw in pos:
        lo_i, hi_i = (0 if iw == 0 else C_LO), (N_S if iw == last else C_HI)
        for jw in pos:
            lo_j, hi_j = (0 if jw == 0 else C_LO), (N_S if jw == last else C_HI)
            plan.append((iw, jw, lo_i, hi_i, lo_j, hi_j))
    return plan


def sr_pass(q: np.ndarray, w: Weights, applications: int, sample=None) -> np.ndarray:
    """Gather 6x6 windows, apply the generator, channel-mean, stitch (srmodel.py:443-463).
    ``sample`` (list of plan indices) restricts the pass to those windows; the
    returned fine grid is then NaN outside their bands (window-sampled parity)."""
    n = q.shape[0]
    plan = stitch_plan(n)
    ks = range(len(plan)) if sample is None else sample
    wins = np.empty((len(ks), CHANNELS, N_S, N_S))
    for a, k in enumerate(ks):
        iw, jw = plan[k][:2]
        wins[a] = q[iw:iw + N_S, jw:jw + N_S]
    out = wins
    for _ in range(applications):
        out = forward_batch(w, out)
    merged = out.mean(axis=1)
    sc = 2 ** applications
    fine = np.full((n * sc, n * sc), np.nan)
    for a, k in enumerate(ks):
        iw, jw, li, hi, lj, hj = plan[k]
        fine[(iw + li) * sc:(iw + hi) * sc, (jw + lj) * sc:(jw + hj) * sc] = \
            merged[a, li * sc:hi * sc, lj * sc:hj * sc]
    return fine


PASS_PLAN = {2: (1,), 4: (2,), 8: (2, 1), 16: (2, 2)}   # srmodel.py:467


def sr_prolong(c: np.ndarray, w: Weights, b: Bounds, s: int) -> np.ndarray:
    """Normalise -> windowed generator -> denormalise with the output signs ->
    mean-subtract, per pass (srmodel.py:470-487)."""
    if s not in PASS_PLAN:
        raise ValueError(f"unsupported SR ratio {s}; expected one of {sorted(PASS_PLAN)}")
    data = c
    for apps in PASS_PLAN[s]:
        q = normalize(data, b)
        qf = sr_pass(q, w, apps)
        data = denormalize(qf, np.sign(qf), b)
        data = data - data.mean()
    return data


# ---------------------------------------------------------------------------
# V-cycle driver (solver.py:39-330)

@dataclass(frozen=True)
class Config:
    """RunConfig (solver.py:39-97) -- the fields on the hot path."""
    N_iter: int = 300
    r_min: int = 12
    N_smooth_pre: int = 10
    N_smooth: int = 20
    N_step: int = 4
    N_GAN: float = 1.0
    S_thres: float = 1e-10
    tol: float = 1e-10
    mode: str = "spline"
    p_min: float = 1e-10
    p_max: float = 1e-3
    seed: int = 0
    coarse_sweeps: int = 10

    @property
    def bounds(self) -> Bounds:
        return Bounds(self.p_min, self.p_max)


def level_sides(n: int, n_step: int, r_min: int) -> list:
    """Ladder fine -> coarse, /2**n_step per level, clamped at r_min (solver.py:100-119)."""
    if n <= r_min:
        raise ValueError(f"fine side {n} must exceed r_min {r_min}")
    sides = [n]
    while sides[-1] > r_min:
        nxt = max(r_min, sides[-1] // 2 ** n_step)
        ratio = sides[-1] / nxt
        if nxt * int(ratio) != sides[-1] or int(ratio) not in PROLONG_RATIOS:
            raise ValueError(f"no valid ladder from {n} to r_min {r_min} with step 2^{n_step}")
        sides.append(nxt)
    return sides


def schedule_operator(it: int, n_gan: float, latched: bool) -> str:
    """N_GAN cadence with latch (solver.py:122-144)."""
    if n_gan < 1.0:
        cadence, first, second = max(1, round(1.0 / n_gan)), "spline", "sr"
    else:
        cadence, first, second = max(1, round(n_gan)), "sr", "spline"
    if latched:
        return second
    if n_gan == 1.0:
        return "sr" if it % 2 == 1 else "spline"
    return first if it % cadence != 0 else second


def v_cycle(p: np.ndarray, f: np.ndarray, cfg: Config, operator: str, weights=None,
            level_ops=None) -> np.ndarray:
    """One V-cycle (solver.py:158-197).  ``level_ops`` (optional list, index =
    coarse level l >= 1 of the prolongation into level l-1) overrides the
    operator per level -- the SURVEY §8(c) per-level GAN-mask wrapper."""
    sides = level_sides(p.shape[0], cfg.N_step, cfg.r_min)

    def prolong(c, s, level):
        op = operator if level_ops is None else level_ops[level]
        if op == "spline":
            return spline_prolong(c, s)
        if weights is None:
            raise ValueError("SR prolongation requires generator weights")
        return sr_prolong(c, weights, cfg.bounds, s)

    def restricted(r, s):
        return 0.5 * restrict(r, s)

    def correction(rhs, level):
        check_rhs(rhs)
        z = np.zeros_like(rhs)
        if level == len(sides) - 1:
            return gauss_seidel(z, rhs, cfg.coarse_sweeps)
        delta = gauss_seidel(z, rhs, cfg.N_smooth)
        r = residual(delta, rhs)
        s = sides[level] // sides[level + 1]
        c = correction(restricted(r, s), level + 1)
        return delta + prolong(c, s, level + 1)

    smoothed = gauss_seidel(p, f, cfg.N_smooth)
    r = residual(smoothed, f)
    s0 = sides[0] // sides[1]
    delta = correction(restricted(r, s0), 1)
    out = smoothed + prolong(delta, s0, 1)
    return out - out.mean()


@dataclass
class Record:
    iteration: int
    diff_norm: float
    residual_norm: float
    operator: str
    switch_latched: bool


@dataclass
class Log:
    records: list = field(default_factory=list)

    @property
    def iterations(self) -> int:
        return len(self.records)


def initial_iterate(n: int, cfg: Config) -> np.ndarray:
    """Seeded start U(-p_max, p_max), mean-subtracted (solver.py:298-300)."""
    rng = np.random.default_rng(cfg.seed)
    start = rng.uniform(-cfg.p_max, cfg.p_max, size=(n, n))
    return start - start.mean()


def solve(f: np.ndarray, cfg: Config, weights=None, level_ops=None):
    """V-cycles until diff_norm < tol (solver.py:280-330)."""
    check_rhs(f)
    level_sides(f.shape[0], cfg.N_step, cfg.r_min)
    p = gauss_seidel(initial_iterate(f.shape[0], cfg), f, cfg.N_smooth_pre)
    log = Log()
    latched = False
    for it in range(1, cfg.N_iter + 1):
        op = schedule_operator(it, cfg.N_GAN, latched) if cfg.mode == "hybrid" else cfg.mode
        lops = None
        if level_ops is not None:
            lops = [op if x == "sr" else x for x in level_ops]
        new_p = v_cycle(p, f, cfg, op, weights, lops)
        d = diff_norm(new_p, p)
        r_rms = rms(residual(new_p, f))
        log.records.append(Record(it, d, r_rms, op, latched))
        if not latched and d <= cfg.S_thres:
            latched = True
        p = new_p
        if d < cfg.tol:
            break
    return p, log


# ---------------------------------------------------------------------------
# seeded synthetic inputs (SURVEY §8(d) config mapping; shared with the GPU runs)

def sine_modes_rhs(n: int, seed: int = 0, modes: int = 16) -> np.ndarray:
    """Config 1/2 RHS: 16 seeded sine modes, k in 1..8, a ~ N(0,1)|k|^-5/3."""
    rng = np.random.default_rng(seed)
    x = 2.0 * np.pi * np.arange(n) / n
    f = np.zeros((n, n))
    for _ in range(modes):
        kx, ky = rng.integers(1, 9, size=2)
        a = rng.standard_normal() * float(kx * kx + ky * ky) ** (-5.0 / 6.0)
        f += a * np.outer(np.sin(ky * x), np.sin(kx * x))
    return f - f.mean()


def grf_blobs_rhs(n: int, seed: int = 0, kmin: float = 4.0, kmax: float = None,
                  blobs: int = 32) -> np.ndarray:
    """Config 3/4/5 RHS: Gaussian random field with |f^(k)|^2 ~ |k|^-8/3 on
    kmin <= |k| <= kmax (shell spectrum ~ k^-5/3) plus 32 periodic Gaussian blobs."""
    rng = np.random.default_rng(seed)
    kmax = kmax if kmax is not None else n / 4
    fr = np.fft.fftfreq(n, d=1.0 / n)
    kx, ky = np.meshgrid(fr, fr, indexing="xy")
    k = np.hypot(kx, ky)
    amp = np.where((k >= kmin) & (k <= kmax), np.maximum(k, 1.0) ** (-4.0 / 3.0), 0.0)
    phase = rng.uniform(0.0, 2.0 * np.pi, size=(n, n))
    f = np.real(np.fft.ifft2(amp * np.exp(1j * phase)))
    f /= max(rms(f), 1e-300)
    x = 2.0 * np.pi * np.arange(n) / n
    for _ in range(blobs):
        cx, cy = rng.uniform(0.0, 2.0 * np.pi, size=2)
        sig = rng.uniform(0.005, 0.05) * 2.0 * np.pi
        a = rng.uniform(1.0, 10.0) * (1.0 if rng.random() < 0.5 else -1.0)
        dx = (x - cx + np.pi) % (2.0 * np.pi) - np.pi
        dy = (x - cy + np.pi) % (2.0 * np.pi) - np.pi
        f += a * np.outer(np.exp(-dy ** 2 / (2 * sig ** 2)), np.exp(-dx ** 2 / (2 * sig ** 2)))
    return f - f.mean()


def spectral_solution(f: np.ndarray) -> np.ndarray:
    """Exact-discrete FFT solution (datagen.py:56-75, discrete=True)."""
    n = f.shape[0]
    h = 2.0 * np.pi / n
    fr = np.fft.fftfreq(n, d=1.0 / n)
    kx, ky = np.meshgrid(fr, fr, indexing="xy")
    lam = -(4.0 / h ** 2) * (np.sin(kx * h / 2.0) ** 2 + np.sin(ky * h / 2.0) ** 2)
    lam[0, 0] = 1.0
    ph = np.fft.fft2(f) / lam
    ph[0, 0] = 0.0
    p = np.real(np.fft.ifft2(ph))
    return p - p.mean()


def scale_to_p_rms(f: np.ndarray, p_rms: float = 1e-4) -> np.ndarray:
    """Scale a RHS so the discrete solution has RMS p_rms (in-band for the SR map)."""
    return f * (p_rms / rms(spectral_solution(f)))
