"""BASELINE config 3 (hybrid) reference fixture, produced by running the REFERENCE itself.

    python tests/golden/make_config3_golden.py          # build container, ~15-30 min on 8 cores

1024^2 periodic grid (8 levels... N_step=1, r_min=8 gives 1024 -> 8), RHS = seeded GRF k^-5/3 on
4 <= |k| <= 256 plus 32 blobs (oracle.grf_blobs_rhs(1024, seed=0, kmax=256)), scaled so the
discrete solution has p_rms = 1e-4 (inside the SR normalisation band), latched hybrid schedule
(N_GAN = 1, S_thres = 5e-4), N_smooth = 2, tol 1e-10, generator = artifacts/trained_b8.mgsr (the
reference's MGSR1 loader).  The reference's ``solver.solve`` applies the SR operator at every level
of an SR cycle (solver.py:147-197), so this is its own hybrid path end to end.

Writes tests/golden/config3_hybrid.npz: per-iteration diff_norm / residual_norm, the operator and
latch sequences, and a 64x64 subsample + checksums of the converged field (the full 1024^2 field
would be 8 MB).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from make_golden import load_reference  # noqa: E402


def main() -> None:
    load_reference()
    from mgsr import kernels, smoother, solver, srmodel
    from mgsr.grid import Grid
    from oracle import mgsr_oracle as orc

    n = 1024
    f = orc.scale_to_p_rms(orc.grf_blobs_rhs(n, seed=0, kmax=256.0), 1e-4)
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b8.mgsr"))
    cfg = solver.RunConfig(N_step=1, r_min=8, N_smooth=2, mode="hybrid", N_GAN=1.0, S_thres=5e-4)
    t0 = time.time()
    p, log = solver.solve(smoother.PoissonProblem(Grid(f)), cfg, w)
    wall = time.time() - t0
    hist = np.array([[r.diff_norm, r.residual_norm] for r in log.records])
    out = {
        "f_checksum": np.array([f.sum(), np.abs(f).sum(), (f * f).sum()]),
        "log": hist,
        "p_sub": p.data[::16, ::16].copy(),
        "p_checksum": np.array([p.data.sum(), np.abs(p.data).sum(), (p.data * p.data).sum()]),
    }
    np.savez_compressed(os.path.join(HERE, "config3_hybrid.npz"), **out)
    meta = {"backend": kernels.active_backend(), "operators": [r.operator for r in log.records],
            "latched": [bool(r.switch_latched) for r in log.records], "iterations": len(log.records),
            "wall_s": wall, "weights": "artifacts/trained_b8.mgsr",
            "config": dict(n=n, N_step=1, r_min=8, N_smooth=2, mode="hybrid", N_GAN=1.0, S_thres=5e-4,
                           rhs="orc.scale_to_p_rms(orc.grf_blobs_rhs(1024, seed=0, kmax=256.0), 1e-4)")}
    with open(os.path.join(HERE, "config3_hybrid_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
