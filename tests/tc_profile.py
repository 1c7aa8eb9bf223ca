"""Profiling driver (GPU): one SR pass (fp16 operands by default, argv[3] = bf16/fp16; argv[4] = ratio, default 2) at coarse
side nc (default 2048 = the finest 4096^2 prolongation).  Not collected by pytest.  Used as
    ncu --set full -k regex:k_gen_tc -s 1 -c 1 python tests/tc_profile.py
(the per-role event trace of one window group is tests/tc_trace.py)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07936_b200 import ops, srmodel, _lib  # noqa: E402

nc = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prec = sys.argv[3] if len(sys.argv) > 3 else "fp16"
ratio = int(sys.argv[4]) if len(sys.argv) > 4 else 2
w = srmodel.random_weights(8, 0)
rng = np.random.default_rng(0)
c = torch.from_numpy((10.0 ** rng.uniform(-7, -3.5, (nc, nc))) * np.where(rng.random((nc, nc)) < 0.5, -1, 1)).cuda()
for _ in range(reps):
    out = ops.sr_prolong(c, w.device_handle(), ratio, 1e-10, 1e-3, _lib.PREC[prec])
torch.cuda.synchronize()
print("ok", float(out.abs().max()))
