"""Worker for tests/test_host.py::test_solve_batch_distributed_gloo_world2 (one rank, gloo, CPU):
the sharding and gathering of solver.solve_batch_distributed with a stand-in per-rank solve."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch.distributed as dist

    from paper_2403_07936_b200 import solver
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem

    dist.init_process_group("gloo")
    rank = dist.get_rank()
    probs = [PoissonProblem(Grid(np.full((4, 4), float(i)) - float(i))) for i in range(5)]
    tag = {id(pr): i for i, pr in enumerate(probs)}   # identify the RHS in the stand-in solve
    seen = []

    def fake_solve(ps):
        out = []
        for pr in ps:
            seen.append(tag[id(pr)])
            log = solver.ConvergenceLog()
            log.records.append(solver.IterationRecord(1, float(tag[id(pr)]), 0.0, "spline", False, float(rank)))
            out.append((Grid(np.full((4, 4), float(tag[id(pr)]))), log))
        return out

    res = solver.solve_batch_distributed(probs, solver.RunConfig(), solve_fn=fake_solve)
    dist.barrier()
    out = {"rank": rank, "seen": seen, "order": [float(g.data[0, 0]) for g, _ in res],
           "solved_by": [log.records[0].wall_ms for _, log in res]}
    with open(os.path.join(sys.argv[1], f"shard{rank}.json"), "w") as fh:
        json.dump(out, fh)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
