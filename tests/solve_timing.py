"""Solve-loop timing (GPU): BASELINE configs 1-3 (periodic mapping) through
solver.solve with the single-launch device loop (resident=True) and the per-cycle host loop
(resident=False), next to the compiled reference (oracle/_ref) on the host cores where it is
importable.  Not collected by pytest.

    python tests/solve_timing.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2403_07936_b200 import datagen, solver, srmodel  # noqa: E402
from paper_2403_07936_b200.grid import Grid  # noqa: E402
from paper_2403_07936_b200.smoother import PoissonProblem  # noqa: E402


def gpu_solve(f, cfg, w, resident, reps, prec):
    solver.solve(PoissonProblem(Grid(f)), cfg, w, resident=resident, precision=prec)   # plan + graph capture
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        p, log = solver.solve(PoissonProblem(Grid(f)), cfg, w, resident=resident, precision=prec)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), log


def ref_solve(f, cfg_kw, weights_path):
    try:
        import oracle
        ref = oracle.import_ref()
    except Exception:
        ref = None
    if ref is None:
        return None
    from mgsr import smoother, solver as rsolver, srmodel as rsr
    from mgsr.grid import Grid as RGrid
    w = rsr.load_weights(weights_path) if weights_path else None
    cfg = rsolver.RunConfig(**cfg_kw)
    t0 = time.perf_counter()
    _, log = rsolver.solve(smoother.PoissonProblem(RGrid(f)), cfg, w)
    return time.perf_counter() - t0, len(log.records)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    wpath = os.path.join(ROOT, "artifacts", "trained_b8.mgsr")
    w = srmodel.load_weights(wpath)
    rows = []
    cases = [
        ("config1 65^2 spline", 64, dict(mode="spline"), datagen.sine_modes_rhs(64, 0), None),
        ("config2 257^2 hybrid (trained B=8)", 256, dict(mode="hybrid", N_GAN=1.0, S_thres=5e-4),
         datagen.scale_to_p_rms(datagen.sine_modes_rhs(256, 0), 1e-4), w),
        ("config3 1025^2 spline", 1024, dict(mode="spline"), datagen.grf_blobs_rhs(1024, seed=0, kmax=256.0), None),
        ("config3 1025^2 hybrid (trained B=8)", 1024, dict(mode="hybrid", N_GAN=1.0, S_thres=5e-4),
         datagen.scale_to_p_rms(datagen.grf_blobs_rhs(1024, seed=0, kmax=256.0), 1e-4), w),
    ]
    cases = [c + ("fp32",) for c in cases] + [
        (c[0] + " fp16 tensor cores", c[1], c[2], c[3], c[4], "fp16") for c in cases if c[4] is not None]
    for name, n, kw, f, ww, prec in cases:
        cfg_kw = dict(N_step=1, r_min=8, N_smooth=2, **kw)
        cfg = solver.RunConfig(**cfg_kw)
        t_res, log = gpu_solve(f, cfg, ww, True, 5, prec)
        t_host, log_h = gpu_solve(f, cfg, ww, False, 5, prec)
        row = {"case": name, "n": n, "precision": prec, "iterations": log.iterations,
               "operators": "".join("G" if r.operator == "sr" else "s" for r in log.records),
               "final_diff": log.records[-1].diff_norm, "final_residual": log.records[-1].residual_norm,
               "gpu_resident_ms": 1e3 * t_res, "gpu_host_loop_ms": 1e3 * t_host,
               "host_loop_iterations": log_h.iterations}
        if prec == "fp32" and (n <= 256 or kw["mode"] == "spline"):
            r = ref_solve(f, cfg_kw, wpath if ww is not None else None)
            if r is not None:
                row["reference_cpu_ms"], row["reference_iterations"] = 1e3 * r[0], r[1]
        rows.append(row)
        print(json.dumps(row), flush=True)
    if out:
        json.dump({"note": "median of 5 solves, wall clock incl. host->device RHS copy and the result readback; "
                           "reference = oracle/_ref (compiled reference) on the host cores",
                   "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
