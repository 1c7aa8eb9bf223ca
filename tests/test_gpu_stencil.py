"""GPU parity: fp64 stencil kernels through the C ABI vs the oracle / golden vectors.

Bar (north_star): stencil, restriction and spline results agree within 1e-12
relative in fp64.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def random_problem(n, seed):
    rng = np.random.default_rng(seed)
    p = rng.standard_normal((n, n)); p -= p.mean()
    f = rng.standard_normal((n, n)); f -= f.mean()
    return p, f, (2.0 * np.pi / n) ** 2


@pytest.mark.parametrize("n", [8, 16, 64])
def test_gs_golden(cuda, golden, n):
    from paper_2403_07936_b200 import kernels
    p = golden[f"gs{n}_p"].copy()
    kernels.gs_sweeps(p, golden[f"gs{n}_f"], (2 * np.pi / n) ** 2, 3)
    assert rel(p, golden[f"gs{n}_out"]) < 1e-13


@pytest.mark.parametrize("n,sweeps", [(96, 3), (128, 2), (130, 3), (200, 1), (256, 5), (512, 9), (1000, 4),
                                      (1024, 2), (2048, 4), (4096, 1), (4096, 2)])
def test_gs_large_vs_oracle(cuda, orc, n, sweeps):
    """Register-blocked TMA tiles (n >= 128, incl. ragged n: shifted edge tiles), half-sweep (n = 96) paths
    vs the C oracle."""
    from paper_2403_07936_b200 import kernels
    p, f, h2 = random_problem(n, n)
    exp = p.copy(); orc.gs_sweeps(exp, f, h2, sweeps)
    got = p.copy(); kernels.gs_sweeps(got, f, h2, sweeps)
    assert rel(got, exp) < 1e-12


def test_gs_device_tensor_in_place_and_deterministic(cuda):
    from paper_2403_07936_b200 import kernels
    p, f, h2 = random_problem(512, 4)
    a = cuda.from_numpy(p).cuda(); b = a.clone(); df = cuda.from_numpy(f).cuda()
    kernels.gs_sweeps(a, df, h2, 5)
    kernels.gs_sweeps(b, df, h2, 5)
    assert cuda.equal(a, b)
    assert abs(float(a.mean())) < 1e-15 * float(a.abs().max()) * 512


def test_gs_zero_sweeps_noop_and_odd_side(cuda):
    from paper_2403_07936_b200 import kernels
    p, f, h2 = random_problem(8, 2)
    before = p.copy()
    kernels.gs_sweeps(p, f, h2, 0)
    assert np.array_equal(p, before)
    q, g, h2 = random_problem(7, 3)
    with pytest.raises(ValueError, match="even side"):
        kernels.gs_sweeps(q, g, h2, 1)


@pytest.mark.parametrize("n", [16, 256])
def test_last_updated_color_has_zero_residual(cuda, n):
    """Update-order pin (reference tests/test_kernels.py:107-121)."""
    from paper_2403_07936_b200 import kernels
    p, f, h2 = random_problem(n, 5)
    kernels.gs_sweeps(p, f, h2, 1)
    r = f - kernels.laplacian(p, 1.0 / h2)
    parity = np.add.outer(np.arange(n), np.arange(n)) % 2
    scale = np.abs(f).max() / h2
    assert np.abs(r[parity == 1]).max() < 1e-12 * scale
    assert np.abs(r[parity == 0]).max() > 1e-6 * scale


def test_laplacian(cuda, golden, orc):
    from paper_2403_07936_b200 import kernels
    out = kernels.laplacian(golden["lap9_p"], 1.0 / (2 * np.pi / 9) ** 2)
    assert np.abs(out - golden["lap9_out"]).max() < 1e-12
    c = np.full((12, 12), 0.375)
    assert np.all(kernels.laplacian(c, 1.0 / (2 * np.pi / 12) ** 2) == 0.0)
    p, _, h2 = random_problem(1024, 9)
    assert rel(kernels.laplacian(p, 1 / h2), orc.laplacian(p, 1 / h2)) < 1e-14


def test_residual_restrict_spline_golden(cuda, golden):
    from paper_2403_07936_b200 import smoother, transfer
    from paper_2403_07936_b200.grid import Grid
    r = smoother.residual(Grid(golden["res_p"]), smoother.PoissonProblem(Grid(golden["res_f"])))
    assert rel(r.data, golden["res_out"]) < 1e-13
    assert rel(transfer.restrict(Grid(golden["res_p"]), 2).data, golden["restrict_out"]) < 1e-14
    raw = transfer.restrict(Grid(golden["res_p"]), 4, subtract_mean=False).data
    assert np.array_equal(raw, golden["restrict4_raw"])
    for s in (2, 4, 8, 16):
        out = transfer.spline_prolong(Grid(golden[f"spline{s}_c"]), s).data
        assert rel(out, golden[f"spline{s}_out"]) < 1e-13


@pytest.mark.parametrize("nc,s", [(1024, 2), (2048, 2), (256, 4), (128, 16)])
def test_spline_large_vs_oracle(cuda, orc, nc, s):
    from paper_2403_07936_b200 import transfer
    from paper_2403_07936_b200.grid import Grid
    c = np.random.default_rng(nc + s).standard_normal((nc, nc))
    assert rel(transfer.spline_prolong(Grid(c), s).data, orc.spline_prolong(c, s)) < 1e-12


def test_transfer_errors(cuda):
    from paper_2403_07936_b200 import transfer
    from paper_2403_07936_b200.grid import Grid
    g = Grid(np.zeros((12, 12)))
    with pytest.raises(ValueError, match="power of two"):
        transfer.restrict(g, 3)
    with pytest.raises(ValueError, match="not divisible"):
        transfer.restrict(g, 8)
    with pytest.raises(ValueError, match="must be one of"):
        transfer.spline_prolong(g, 32)


def test_restrict_prolong_is_identity(cuda):
    from paper_2403_07936_b200 import transfer
    from paper_2403_07936_b200.grid import Grid
    c = np.random.default_rng(1).standard_normal((64, 64))
    for s in (2, 4, 8, 16):
        back = transfer.restrict(transfer.spline_prolong(Grid(c), s), s, subtract_mean=False).data
        assert np.abs(back - c).max() < 1e-13


def test_diff_norm(cuda):
    from paper_2403_07936_b200.grid import Grid, diff_norm
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal((300, 300)), rng.standard_normal((300, 300))
    assert abs(diff_norm(Grid(a), Grid(b)) - np.sqrt(np.mean((a - b) ** 2))) < 1e-14


@pytest.mark.parametrize("n,sweeps", [(2, 3), (4, 1), (6, 2), (10, 5), (32, 7), (66, 2)])
def test_gs_tiny_and_odd_multiple_sides_vs_oracle(cuda, orc, n, sweeps):
    """Smallest sides (single-CTA kernel, n <= 64, every sweep's exact mean) and a side just above it
    (66: the generic half-sweep path) against the C oracle."""
    from paper_2403_07936_b200 import kernels
    p, f, h2 = random_problem(n, 40 + n)
    exp = p.copy(); orc.gs_sweeps(exp, f, h2, sweeps)
    got = p.copy(); kernels.gs_sweeps(got, f, h2, sweeps)
    assert rel(got, exp) < 1e-12


@pytest.mark.parametrize("nc,s", [(2, 2), (3, 4), (5, 8), (2, 16), (6, 2)])
def test_spline_tiny_coarse_grids_vs_oracle(cuda, orc, nc, s):
    """Coarse sides below the 4-tap stencil width: the periodic wrap folds taps onto the same cells."""
    from paper_2403_07936_b200 import transfer
    from paper_2403_07936_b200.grid import Grid
    c = np.random.default_rng(nc * 31 + s).standard_normal((nc, nc))
    assert rel(transfer.spline_prolong(Grid(c), s).data, orc.spline_prolong(c, s)) < 1e-12


@pytest.mark.parametrize("n,s", [(4, 2), (32, 16), (48, 4)])
def test_restrict_edge_sizes_vs_oracle(cuda, orc, n, s):
    from paper_2403_07936_b200 import transfer
    from paper_2403_07936_b200.grid import Grid
    x = np.random.default_rng(n + s).standard_normal((n, n))
    assert rel(transfer.restrict(Grid(x), s).data, orc.restrict(x, s)) < 1e-13
    assert np.array_equal(transfer.restrict(Grid(x), s, subtract_mean=False).data, orc.restrict(x, s, False))


def test_c_abi_binding_as_documented(cuda, orc):
    """The reference-side ctypes stub of INTEGRATION.md §3, verbatim in shape: raw device pointers,
    the workspace size from mgsr_workspace_bytes, ValueError from mgsr_last_error -- no torch ops."""
    import ctypes
    from paper_2403_07936_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    lib.mgsr_last_error.restype = ctypes.c_char_p
    lib.mgsr_workspace_bytes.restype = ctypes.c_size_t
    lib.mgsr_workspace_bytes.argtypes = [ctypes.c_int64]
    lib.mgsr_gs_sweeps.restype = ctypes.c_int
    lib.mgsr_gs_sweeps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                   ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]

    def check(rc):
        if rc != 0:
            raise ValueError(lib.mgsr_last_error().decode())

    n, sweeps = 256, 3
    p, f, h2 = random_problem(n, 77)
    dp, df = cuda.from_numpy(p.copy()).cuda(), cuda.from_numpy(f).cuda()
    nb = lib.mgsr_workspace_bytes(n)
    ws = cuda.empty(nb, dtype=cuda.uint8, device="cuda")
    check(lib.mgsr_gs_sweeps(dp.data_ptr(), df.data_ptr(), n, h2, sweeps, ws.data_ptr(), nb, None))
    exp = p.copy(); orc.gs_sweeps(exp, f, h2, sweeps)
    assert rel(dp.cpu().numpy(), exp) < 1e-12
    with pytest.raises(ValueError, match="even side"):
        check(lib.mgsr_gs_sweeps(dp.data_ptr(), df.data_ptr(), 255, h2, 1, ws.data_ptr(), nb, None))
