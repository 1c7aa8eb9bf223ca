"""BASELINE config 5 (GPU): 16 independent 2048^2 right-hand sides (seeded k^-5/3
random fields, config-3 generator), latched hybrid solves run concurrently with
solver.solve_batch, for smoothing sweeps nu in {1, 2, 4} and SR at the {1, 2, 3}
finest prolongations (per-level GAN mask).  Reports V-cycles to diff < 1e-10 per RHS
and wall time per solve, for the batched solve (all loops in lockstep in one graph
launch, one generator launch per SR level across the batch) next to one resident
solve per RHS on its own stream, and checks that both give identical results.
Not collected by pytest.

    python tests/config5_timing.py [out.json] [batch] [n]
    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 tests/config5_timing.py ...
        (RHS sharded round-robin over the ranks, one GPU each: solver.solve_batch_distributed)
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


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    run = (lambda ps, cfg, w, **kw: solver.solve_batch_distributed(ps, cfg, w, **kw)) if world > 1 else \
        (lambda ps, cfg, w, **kw: solver.solve_batch(ps, cfg, w, **kw))
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b8.mgsr"))
    probs = [PoissonProblem(Grid(datagen.scale_to_p_rms(datagen.grf_blobs_rhs(n, seed=s, kmax=256.0), 1e-4)))
             for s in range(batch)]
    rows = []
    for nu in (1, 2, 4):
        for gl in (1, 2, 3):
            cfg = solver.RunConfig(N_step=1, r_min=8, N_smooth=nu, mode="hybrid", N_GAN=1.0, S_thres=5e-4,
                                   N_iter=100)
            walls, outs = {}, {}
            for batched in (True, False):
                run(probs, cfg, w, precision="fp16", sr_levels=gl, batched=batched)   # plans, graphs (not timed)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                outs[batched] = run(probs, cfg, w, precision="fp16", sr_levels=gl, batched=batched)
                walls[batched] = time.perf_counter() - t0   # includes the gather: every rank holds all results
            res, wall = outs[True], walls[True]
            same = all(np.array_equal(a[0].data, b[0].data) and a[1].iterations == b[1].iterations
                       for a, b in zip(outs[True], outs[False]))
            its = [log.iterations for _, log in res]
            conv = [log.converged(1e-10) for _, log in res]
            sr_cycles = [sum(r.operator == "sr" for r in log.records) for _, log in res]
            row = {"nu": nu, "gan_levels": gl, "batch": batch, "n": n,
                   "iterations_mean": float(np.mean(its)), "iterations_min": int(min(its)),
                   "iterations_max": int(max(its)), "all_converged": bool(all(conv)),
                   "sr_cycles_mean": float(np.mean(sr_cycles)),
                   "wall_s_batch": wall, "wall_ms_per_solve": 1e3 * wall / batch,
                   "wall_ms_per_solve_streams": 1e3 * walls[False] / batch, "batched_equals_streams": bool(same)}
            row["ranks"] = world
            rows.append(row)
            if rank == 0:
                print(json.dumps(row), flush=True)
    if out and rank == 0:
        json.dump({"note": "fp16 tensor-core generator (trained B=8 fixture), latched hybrid N_GAN=1, S_thres=5e-4, "
                           "tol 1e-10; wall clock of the whole batch incl. host->device RHS copies and result "
                           "readback; wall_ms_per_solve: the batched solve (solve_batch(batched=True): one graph launch for the "
                           "whole batch, one generator launch per SR level across the RHS); wall_ms_per_solve_streams: one "
                           "resident solve per RHS, each on its own stream",
                   "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
