"""Spectral tooling timing (GPU, cuFFT via torch.fft) next to the reference's numpy
implementation (oracle/_ref) on the host cores.  Not collected by pytest.

    python tests/spectral_timing.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2403_07936_b200 import spectral  # noqa: E402
from paper_2403_07936_b200.grid import Grid  # noqa: E402


def best(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    import oracle
    ref = oracle.import_ref()
    rows = []
    for n in (1024, 4096):
        x = np.random.default_rng(0).standard_normal((n, n))
        g = Grid(x - x.mean())
        cases = {
            "power_spectrum": (lambda: spectral.power_spectrum(g), None),
            "solve_poisson_spectral(discrete)": (lambda: spectral.solve_poisson_spectral(g, discrete=True), None),
            "turbulent_source(k_peak=n/16)": (lambda: spectral.turbulent_source(n, n // 16, 0), None),
        }
        if ref is not None:
            from mgsr import datagen as rdg
            from mgsr.grid import Grid as RGrid, power_spectrum as rps
            rg = RGrid(x - x.mean())
            cases["power_spectrum"] = (cases["power_spectrum"][0], lambda: rps(rg))
            cases["solve_poisson_spectral(discrete)"] = (cases["solve_poisson_spectral(discrete)"][0],
                                                         lambda: rdg.solve_poisson_spectral(rg, discrete=True))
            cases["turbulent_source(k_peak=n/16)"] = (cases["turbulent_source(k_peak=n/16)"][0],
                                                      lambda: rdg.turbulent_source(n, n // 16, 0))
        for name, (mine, theirs) in cases.items():
            mine()
            row = {"n": n, "op": name, "gpu_ms_incl_host_io": 1e3 * best(mine)}
            if theirs is not None:
                row["reference_cpu_ms"] = 1e3 * best(theirs, 1)
            rows.append(row)
            print(json.dumps(row), flush=True)
    if out:
        json.dump({"note": "wall clock per call incl. host<->device copies of the Grid arguments/results; "
                           "reference = numpy/pocketfft on the host cores (oracle/_ref)", "rows": rows},
                  open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
