"""Generator pass time vs depth (GPU): the finest bench pass (n_c = 2048, fp16) for B = 1, 2, 4, 8, 12, 16 residual
blocks, to split the per-body-layer cost (slope) from the head / up / tail / stitch cost (intercept).  Not collected
by pytest.   python tests/gen_depth_timing.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07936_b200 import _lib, ops, srmodel  # noqa: E402

nc = 2048
rng = np.random.default_rng(0)
c = torch.from_numpy((10.0 ** rng.uniform(-7, -3.5, (nc, nc))) * np.where(rng.random((nc, nc)) < 0.5, -1, 1)).cuda()
rows = []
for B in (1, 2, 4, 8, 12, 16):
    w = srmodel.random_weights(B, 0)
    f = lambda: ops.sr_prolong(c, w.device_handle(), 2, 1e-10, 1e-3, _lib.PREC["fp16"])  # noqa: E731
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    rows.append((B, 2 * B + 1, min(ts)))
    print(B, 2 * B + 1, f"{min(ts):.2f} ms", flush=True)
L = np.array([r[1] for r in rows], float); T = np.array([r[2] for r in rows])
k, b0 = np.polyfit(L, T, 1)
print(f"per body layer {k:.3f} ms, intercept {b0:.3f} ms")
