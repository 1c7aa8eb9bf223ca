"""Profiling driver (GPU): one bf16 SR pass at coarse side nc (default 2048 = the
finest 4096^2 prolongation).  Not collected by pytest.  Used as
    ncu --set full -k regex:k_gen_tc -s 1 -c 1 python tests/tc_profile.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07936_b200 import ops, srmodel, _lib  # noqa: E402

nc = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = srmodel.random_weights(8, 0)
rng = np.random.default_rng(0)
c = torch.from_numpy((10.0 ** rng.uniform(-7, -3.5, (nc, nc))) * np.where(rng.random((nc, nc)) < 0.5, -1, 1)).cuda()
for _ in range(reps):
    out = ops.sr_prolong(c, w.device_handle(), 2, 1e-10, 1e-3, _lib.PREC["bf16"])
torch.cuda.synchronize()
print("ok", float(out.abs().max()))

if len(sys.argv) > 3 and sys.argv[3] == "prof":
    import ctypes
    lib = _lib.load()
    lib.mgsr_debug_tc_prof.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p]
    prof = torch.zeros(48, dtype=torch.int64, device="cuda")
    fine = torch.empty((2 * nc, 2 * nc), dtype=torch.float64, device="cuda")
    _lib.check(lib.mgsr_debug_tc_prof(w.device_handle(), c.data_ptr(), nc, fine.data_ptr(), prof.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    p = prof.cpu().numpy().astype(float) / 148
    ng = ((nc // 2 - 2) ** 2 + 5) // 6 / 148
    print(f"per-CTA cycles: MMA total {p[2]:.3e}  wait act_ready {p[0]:.3e} ({100*p[0]/p[2]:.1f}%)  "
          f"wait weights {p[1]:.3e} ({100*p[1]/p[2]:.1f}%)  | epi wait acc {p[3]:.3e} ({100*p[3]/p[2]:.1f}%)  "
          f"up+tail phase {p[4]:.3e} ({100*p[4]/p[2]:.1f}%)  head phase {p[5]:.3e} ({100*p[5]/p[2]:.1f}%)\n"
          f"  MMA phases: head {100*p[40]/p[2]:.1f}%  body {100*p[41]/p[2]:.1f}%  up {100*p[42]/p[2]:.1f}%"
          f"  (per group cycles: head {p[40]/ng:.0f} body {p[41]/ng:.0f} up {p[42]/ng:.0f})")
    for nm, o in (("drain warp", 0), ("tail warp", 8)):
        print(f"  epilogue {nm} per group: q {p[20+o]/ng:.0f}  i2c {p[21+o]/ng:.0f}  head-epi {p[22+o]/ng:.0f}  "
              f"body {p[23+o]/ng:.0f}  up {p[4+o]/ng:.0f}  end-barrier {p[24+o]/ng:.0f}")
