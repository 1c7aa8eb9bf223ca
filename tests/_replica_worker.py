"""Worker for tests/test_host.py::test_replicas_gloo_world2 (one rank, gloo, CPU).

Exercises bench.py's multi-rank host logic: max-over-ranks timing, whole-job
value of independent replicas, per-rank seeds (distinct inputs), barrier."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import bench

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    dev = torch.device("cpu")
    ms_local = 100.0 + 50.0 * rank           # rank 1 is the slow one
    ms = bench.reduce_max(ms_local, dist, dev)
    val = bench.replica_value(10, ms, world)
    f, p = bench.make_inputs(64, bench.replica_seed(rank), "gan")
    digest = torch.tensor([float(np.abs(f).sum())], dtype=torch.float64)
    allv = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allv, digest)
    dist.barrier()
    out = {"rank": rank, "ms": ms, "value": val, "digests": [float(t.item()) for t in allv],
           "f_mean": float(f.mean())}
    with open(os.path.join(sys.argv[1], f"rank{rank}.json"), "w") as fh:
        json.dump(out, fh)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
