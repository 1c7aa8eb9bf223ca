"""Seeded synthetic right-hand sides for the BASELINE configs.

Host NumPy generators shared by the GPU runs (bench.py) and, through the
oracle's identical restatement, by the CPU baseline, so both sides see the
same inputs.  The paper's Navier-Stokes fields are not available; these
stand in with the shapes, spectra and magnitudes BASELINE.json names.
"""

from __future__ import annotations

import numpy as np

__all__ = ["grf_blobs_rhs", "scale_to_p_rms", "sine_modes_rhs", "spectral_solution"]


def sine_modes_rhs(n: int, seed: int = 0, modes: int = 16) -> np.ndarray:
    """Configs 1/2: 16 seeded sine modes, wavenumbers 1..8, amplitude N(0,1)|k|^-5/3."""
    rng = np.random.default_rng(seed)
    x = 2.0 * np.pi * np.arange(n) / n
    f = np.zeros((n, n))
    for _ in range(modes):
        kx, ky = rng.integers(1, 9, size=2)
        a = rng.standard_normal() * float(kx * kx + ky * ky) ** (-5.0 / 6.0)
        f += a * np.outer(np.sin(ky * x), np.sin(kx * x))
    return f - f.mean()


def grf_blobs_rhs(n: int, seed: int = 0, kmin: float = 4.0, kmax: float | None = None,
                  blobs: int = 32) -> np.ndarray:
    """Configs 3-5: Gaussian random field, |f^(k)|^2 ~ |k|^-8/3 on kmin <= |k| <= kmax
    (shell spectrum ~ k^-5/3), plus 32 periodic Gaussian blobs (sigma U[0.005, 0.05]
    of the domain, amplitude +-U(1, 10)), mean-subtracted."""
    rng = np.random.default_rng(seed)
    kmax = kmax if kmax is not None else n / 4
    fr = np.fft.fftfreq(n, d=1.0 / n)
    kx, ky = np.meshgrid(fr, fr, indexing="xy")
    k = np.hypot(kx, ky)
    amp = np.where((k >= kmin) & (k <= kmax), np.maximum(k, 1.0) ** (-4.0 / 3.0), 0.0)
    phase = rng.uniform(0.0, 2.0 * np.pi, size=(n, n))
    f = np.real(np.fft.ifft2(amp * np.exp(1j * phase)))
    f /= max(float(np.sqrt(np.mean(f ** 2))), 1e-300)
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
    """Exact solution of the discrete periodic 5-point system by FFT."""
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
    """Scale f so the discrete solution has RMS p_rms, inside the SR map's band [1e-10, 1e-3]."""
    p = spectral_solution(f)
    return f * (p_rms / max(float(np.sqrt(np.mean(p ** 2))), 1e-300))
