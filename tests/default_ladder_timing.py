"""V-cycle timing with the reference's default RunConfig (N_step=4, r_min=12, N_smooth=20): ladders
[3072, 192, 12] and [192, 12], spline vs SR prolongation (ratio 16 = two ratio-4 passes per SR level),
fp16 tensor cores and the fp32 CUDA-core generator.  CUDA events over graph-replayed cycles (the
plan's captured graph per operator).  Not collected by pytest.

    python tests/default_ladder_timing.py [out.json]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_07936_b200 import datagen, solver, srmodel  # noqa: E402


def main():
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b8.mgsr"))
    cfg = solver.RunConfig(N_step=4, r_min=12, N_smooth=20)
    rows = []
    for n, runs in [(192, [("spline", "fp16"), ("sr", "fp16"), ("sr", "mixed"), ("sr", "fp32")]),
                    (3072, [("spline", "fp16"), ("sr", "fp16"), ("sr", "mixed"), ("sr", "fp32")])]:
        f = torch.from_numpy(datagen.scale_to_p_rms(datagen.grf_blobs_rhs(n, seed=0, kmax=n / 8), 1e-4)).cuda()
        for op, pr in runs:
            plan = solver.VCyclePlan(n, cfg, w, precision=pr)
            p = torch.zeros((n, n), dtype=torch.float64, device="cuda")
            reps = 3 if (pr == "fp32" and op == "sr" and n > 1000) else 10
            plan.cycle(p, f, op)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                plan.cycle(p, f, op)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            rows.append({"n": n, "ladder": plan.sides, "operator": op, "precision": pr if op == "sr" else "fp64",
                         "ms_per_cycle": ms, "cycles_per_s": 1000.0 / ms})
            print(json.dumps(rows[-1]), flush=True)
            del plan
    if len(sys.argv) > 1:
        json.dump(rows, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
