"""Spectral tooling on the GPU: the reference's FFT-based helpers,
evaluated with cuFFT (through torch.fft) on the device instead of numpy's pocketfft.

- ``power_spectrum``          grid.py:148-171   radial |FFT|^2 bins (Parseval-exact total)
- ``solve_poisson_spectral``  datagen.py:56-75  mean-free spectral Poisson solve (continuous or
                                                 the 5-point stencil's exact discrete symbol)
- ``turbulent_source``        datagen.py:88-161 pseudo-spectral turbulent source + its oracle
- ``single_mode_field``       datagen.py:34-49  analytic cos(kx) + cos(ky) pair

Same arguments, return types and ``ValueError`` texts as the reference.  The seeded noise of
``turbulent_source`` is drawn on the host with the reference's generator
(``default_rng(seed).standard_normal``) so the fields are the reference's; every transform runs
on the device.  Results agree with the reference to FFT rounding (<= 1e-12 relative; the
parity tests hold golden vectors the reference produced, tests/golden/spectral.npz).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .grid import Grid

__all__ = ["FlowField", "Spectrum", "power_spectrum", "single_mode_field", "solve_poisson_spectral",
           "turbulent_source"]


@dataclass(frozen=True)
class Spectrum:
    """Radially binned Fourier power: ``power[i]`` at integer radius ``k[i]`` (grid.py:140-146)."""

    k: np.ndarray
    power: np.ndarray


@dataclass(frozen=True)
class FlowField:
    """Divergence-free velocity field that generated a turbulent source (datagen.py:78-85)."""

    u: Grid
    v: Grid
    k_peak: int
    seed: int


def _dev(a):
    torch = _lib.require_cuda()
    if isinstance(a, Grid):
        a = a.data
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64)
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")


def _wavenumbers(n: int):
    """(kx, ky) = meshgrid(fftfreq(n, 1/n)) with indexing "xy" (datagen.py:52-54)."""
    torch = _lib.require_cuda()
    fr = torch.fft.fftfreq(n, d=1.0 / n, dtype=torch.float64, device="cuda")
    ky, kx = torch.meshgrid(fr, fr, indexing="ij")
    return kx, ky


def power_spectrum(p, peak_normalize: bool = False) -> Spectrum:
    """Radial power spectrum of a periodic field (grid.py:148-171): |FFT|^2 summed over annuli
    of integer radius rint(hypot(kx, ky)), radii beyond n/2 folded into the last bin."""
    torch = _lib.require_cuda()
    d = _dev(p)
    n = d.shape[0]
    if n < 4:
        raise ValueError(f"power spectrum needs n >= 4, got {n}")
    p2 = torch.fft.fft2(d).abs() ** 2
    kx, ky = _wavenumbers(n)
    radius = torch.round(torch.hypot(kx, ky)).to(torch.int64).clamp_(max=n // 2)
    power = torch.zeros(n // 2 + 1, dtype=torch.float64, device="cuda")
    power.index_add_(0, radius.reshape(-1), p2.reshape(-1))
    if peak_normalize:
        peak = power.max()
        if float(peak) > 0.0:
            power = power / peak
    return Spectrum(k=np.arange(n // 2 + 1), power=power.cpu().numpy())


def solve_poisson_spectral(f, discrete: bool = False) -> Grid:
    """Mean-free Poisson solution by FFT (datagen.py:56-75): lambda = -|k|^2, or with
    ``discrete`` the 5-point eigenvalues -(4/h^2)(sin^2(kx h/2) + sin^2(ky h/2))."""
    torch = _lib.require_cuda()
    d = _dev(f)
    n = d.shape[0]
    kx, ky = _wavenumbers(n)
    if discrete:
        h = 2.0 * np.pi / n
        lam = -(4.0 / h ** 2) * (torch.sin(kx * h / 2.0) ** 2 + torch.sin(ky * h / 2.0) ** 2)
    else:
        lam = -(kx ** 2 + ky ** 2)
    lam[0, 0] = 1.0
    phat = torch.fft.fft2(d) / lam
    phat[0, 0] = 0.0
    p = torch.fft.ifft2(phat).real
    return Grid((p - p.mean()).cpu().numpy())


def single_mode_field(n: int, k: int) -> tuple[Grid, Grid]:
    """Analytic pair p = cos(kx) + cos(ky), f = laplace(p) = -k^2 p (datagen.py:34-49)."""
    torch = _lib.require_cuda()
    if not (1 <= k < n / 2):
        raise ValueError(f"mode number must satisfy 1 <= k < n/2, got k={k}, n={n}")
    x = 2.0 * np.pi * torch.arange(n, dtype=torch.float64, device="cuda") / n
    mode = torch.cos(k * x)
    p = mode[:, None] + mode[None, :]
    p = p - p.mean()
    f = -(k ** 2) * p
    f = f - f.mean()
    return Grid(p.cpu().numpy()), Grid(f.cpu().numpy())


def turbulent_source(n: int, k_peak: int, seed: int, p_rms: float | None = None
                     ) -> tuple[Grid, FlowField, Grid]:
    """Pseudo-spectral turbulent Poisson source with its spectral oracle (datagen.py:88-161):
    random-phase streamfunction |psi^(k)| ~ k exp(-(k/k_peak)^2), u = d psi/dy, v = -d psi/dx
    at unit RMS speed, f = -div((u . grad) u) with 2/3-rule dealiasing, p^ = -f^/|k|^2;
    ``p_rms`` rescales the problem so the oracle has that RMS.  Returns (f, flow, p_oracle)."""
    torch = _lib.require_cuda()
    if not (2 <= k_peak <= n / 4):
        raise ValueError(f"need 2 <= k_peak <= n/4, got k_peak={k_peak}, n={n}")
    noise = np.random.default_rng(seed).standard_normal((n, n))   # the reference's seeded stream
    kx, ky = _wavenumbers(n)
    k2 = kx ** 2 + ky ** 2
    kr = torch.sqrt(k2)
    noise_hat = torch.fft.fft2(_dev(noise))
    mag = noise_hat.abs()
    mag[mag == 0.0] = 1.0
    phases = noise_hat / mag
    psi_hat = kr * torch.exp(-((kr / k_peak) ** 2)) * phases
    psi_hat[0, 0] = 0.0
    u_hat = 1j * ky * psi_hat
    v_hat = -1j * kx * psi_hat
    u = torch.fft.ifft2(u_hat).real
    v = torch.fft.ifft2(v_hat).real
    vel_rms = torch.sqrt(torch.mean(u ** 2 + v ** 2))
    u, v = u / vel_rms, v / vel_rms
    u_hat, v_hat = u_hat / vel_rms, v_hat / vel_rms
    ux = torch.fft.ifft2(1j * kx * u_hat).real
    uy = torch.fft.ifft2(1j * ky * u_hat).real
    vx = torch.fft.ifft2(1j * kx * v_hat).real
    vy = torch.fft.ifft2(1j * ky * v_hat).real
    adv_x = u * ux + v * uy
    adv_y = u * vx + v * vy
    kmax = n // 2
    dealias = (kx.abs() <= (2.0 / 3.0) * kmax) & (ky.abs() <= (2.0 / 3.0) * kmax)
    f_hat = -(1j * kx * torch.fft.fft2(adv_x) + 1j * ky * torch.fft.fft2(adv_y))
    f_hat = f_hat * dealias
    f_hat[0, 0] = 0.0
    lam = k2.clone()
    lam[0, 0] = 1.0
    p_hat = -f_hat / lam
    p_hat[0, 0] = 0.0
    f = torch.fft.ifft2(f_hat).real
    f = f - f.mean()
    p = torch.fft.ifft2(p_hat).real
    p = p - p.mean()
    if p_rms is not None:
        if p_rms <= 0.0:
            raise ValueError(f"p_rms must be > 0, got {p_rms}")
        scale = p_rms / torch.sqrt(torch.mean(p ** 2))
        f, p = f * scale, p * scale
        u, v = u * torch.sqrt(scale), v * torch.sqrt(scale)
    flow = FlowField(u=Grid(u.cpu().numpy()), v=Grid(v.cpu().numpy()), k_peak=k_peak, seed=seed)
    return Grid(f.cpu().numpy()), flow, Grid(p.cpu().numpy())
