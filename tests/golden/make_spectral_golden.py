"""Golden vectors for the spectral tooling (paper_2403_07936_b200.spectral), produced by the
REFERENCE's own functions (grid.power_spectrum, datagen.solve_poisson_spectral,
datagen.turbulent_source, datagen.single_mode_field).  Run in the build container:

    python tests/golden/make_spectral_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_reference  # noqa: E402


def main() -> None:
    load_reference()
    from mgsr import datagen
    from mgsr.grid import Grid, power_spectrum

    g: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(77)
    for n in (32, 48):
        x = rng.standard_normal((n, n))
        g[f"ps{n}_in"] = x
        g[f"ps{n}_power"] = power_spectrum(Grid(x)).power
        g[f"ps{n}_power_peak"] = power_spectrum(Grid(x), peak_normalize=True).power
        f = x - x.mean()
        g[f"sp{n}_f"] = f
        g[f"sp{n}_cont"] = datagen.solve_poisson_spectral(Grid(f), discrete=False).data
        g[f"sp{n}_disc"] = datagen.solve_poisson_spectral(Grid(f), discrete=True).data
    for n, kp, seed, prms in ((32, 4, 3, None), (64, 8, 11, 1e-4)):
        f, flow, p = datagen.turbulent_source(n, kp, seed, p_rms=prms)
        tag = f"turb{n}"
        g[tag + "_f"], g[tag + "_u"], g[tag + "_v"], g[tag + "_p"] = f.data, flow.u.data, flow.v.data, p.data
    p, f = datagen.single_mode_field(16, 3)
    g["mode16_p"], g["mode16_f"] = p.data, f.data
    np.savez_compressed(os.path.join(HERE, "spectral.npz"), **g)
    print(f"wrote {len(g)} arrays to tests/golden/spectral.npz")


if __name__ == "__main__":
    main()
