"""GPU parity: spectral tooling (cuFFT via torch.fft) against golden vectors the reference
produced (tests/golden/make_spectral_golden.py): power_spectrum (grid.py:148-171),
solve_poisson_spectral (datagen.py:56-75), turbulent_source (datagen.py:88-161),
single_mode_field (datagen.py:34-49).  Bar: FFT rounding, <= 1e-12 relative to the field max.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def sg():
    return np.load(os.path.join(HERE, "golden", "spectral.npz"))


@pytest.mark.parametrize("n", [32, 48])
def test_power_spectrum_golden(cuda, sg, n):
    from paper_2403_07936_b200 import spectral
    from paper_2403_07936_b200.grid import Grid
    x = sg[f"ps{n}_in"]
    s = spectral.power_spectrum(Grid(x))
    assert np.array_equal(s.k, np.arange(n // 2 + 1))
    assert rel(s.power, sg[f"ps{n}_power"]) < 1e-12
    assert rel(spectral.power_spectrum(Grid(x), peak_normalize=True).power, sg[f"ps{n}_power_peak"]) < 1e-12
    # Parseval: the unnormalised total is n^2 * sum(p^2)
    assert abs(s.power.sum() - n * n * np.sum(x ** 2)) < 1e-10 * s.power.sum()


@pytest.mark.parametrize("n", [32, 48])
def test_solve_poisson_spectral_golden(cuda, sg, n):
    from paper_2403_07936_b200 import spectral
    from paper_2403_07936_b200.grid import Grid
    f = sg[f"sp{n}_f"]
    assert rel(spectral.solve_poisson_spectral(Grid(f)).data, sg[f"sp{n}_cont"]) < 1e-12
    assert rel(spectral.solve_poisson_spectral(Grid(f), discrete=True).data, sg[f"sp{n}_disc"]) < 1e-12


def test_discrete_spectral_solution_is_a_fixed_point_of_the_stencil(cuda):
    """The discrete-symbol solve is the exact solution of the 5-point system the V-cycle
    solves: its device residual vanishes."""
    from paper_2403_07936_b200 import datagen, smoother, spectral
    from paper_2403_07936_b200.grid import Grid
    f = datagen.grf_blobs_rhs(256, seed=2, kmax=64.0)
    p = spectral.solve_poisson_spectral(Grid(f), discrete=True)
    r = smoother.residual(p, smoother.PoissonProblem(Grid(f))).data
    assert np.abs(r).max() < 1e-9 * np.abs(f).max()


@pytest.mark.parametrize("n,kp,seed,prms", [(32, 4, 3, None), (64, 8, 11, 1e-4)])
def test_turbulent_source_golden(cuda, sg, n, kp, seed, prms):
    from paper_2403_07936_b200 import spectral
    f, flow, p = spectral.turbulent_source(n, kp, seed, p_rms=prms)
    tag = f"turb{n}"
    assert rel(f.data, sg[tag + "_f"]) < 1e-12
    assert rel(flow.u.data, sg[tag + "_u"]) < 1e-12
    assert rel(flow.v.data, sg[tag + "_v"]) < 1e-12
    assert rel(p.data, sg[tag + "_p"]) < 1e-12
    assert flow.k_peak == kp and flow.seed == seed


def test_single_mode_and_errors(cuda, sg):
    from paper_2403_07936_b200 import spectral
    from paper_2403_07936_b200.grid import Grid
    p, f = spectral.single_mode_field(16, 3)
    assert rel(p.data, sg["mode16_p"]) < 1e-14 and rel(f.data, sg["mode16_f"]) < 1e-14
    with pytest.raises(ValueError, match="mode number"):
        spectral.single_mode_field(16, 8)
    with pytest.raises(ValueError, match="k_peak"):
        spectral.turbulent_source(32, 9, 0)
    with pytest.raises(ValueError, match="p_rms"):
        spectral.turbulent_source(32, 4, 0, p_rms=-1.0)
    with pytest.raises(ValueError, match="n >= 4"):
        spectral.power_spectrum(Grid(np.zeros((2, 2))))


def test_power_spectrum_zero_field_and_peak_normalize(cuda):
    from paper_2403_07936_b200 import spectral
    from paper_2403_07936_b200.grid import Grid
    z = spectral.power_spectrum(Grid(np.zeros((16, 16))), peak_normalize=True)
    assert np.array_equal(z.power, np.zeros(9))   # a zero field stays all-zero (grid.py:165-169)
    x = np.random.default_rng(5).standard_normal((32, 32))
    s = spectral.power_spectrum(Grid(x), peak_normalize=True).power
    assert s.max() == 1.0
