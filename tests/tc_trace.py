"""Bring-up tool (GPU): event trace of one steady-state window group of CTA 0 in
the tensor-core generator (k_gen_tc), for the critical-path analysis.  Not
collected by pytest.

    python tests/tc_trace.py [nc] [fp16|bf16] [out.json]
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07936_b200 import _lib, srmodel  # noqa: E402

NAMES = {1: "P.fill", 2: "M.act_ready", 3: "M.issued", 4: "M.weights", 5: "M.i2c_full",
         6: "E.acc_full", 7: "E.arrive", 8: "D.acc_full", 9: "D.ubuf_free", 10: "D.ubuf_full",
         11: "E.group_start/q", 12: "E.i2c_built", 13: "Z.full", 14: "Z.stored", 15: "E.end",
         16: "M.tail_issue", 17: "E.acc_loaded"}
ROLES = ["producer", "mma", "epi_w2", "epi_w10"]


def main():
    nc = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    f16 = 1 if (len(sys.argv) <= 2 or sys.argv[2] == "fp16") else 0
    out = sys.argv[3] if len(sys.argv) > 3 else None
    lib = _lib.load()
    lib.mgsr_debug_tc_prof.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]
    w = srmodel.random_weights(8, 0)
    rng = np.random.default_rng(0)
    c = torch.from_numpy((10.0 ** rng.uniform(-7, -3.5, (nc, nc))) * np.where(rng.random((nc, nc)) < 0.5, -1, 1)).cuda()
    fine = torch.empty((2 * nc, 2 * nc), dtype=torch.float64, device="cuda")
    tr = torch.zeros(4 * 4096, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        tr.zero_()
        _lib.check(lib.mgsr_debug_tc_prof(w.device_handle(), c.data_ptr(), nc, fine.data_ptr(), tr.data_ptr(), f16, st))
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.int64).reshape(4, 2048, 2)
    ev = []
    for r in range(4):
        for i in range(2048):
            idn, clk = int(t[r, i, 0]), int(t[r, i, 1])
            if idn == 0 and clk == 0:
                break
            ev.append((clk, ROLES[r], idn // 1000, (idn % 1000) // 10, idn % 10))
    ev.sort()
    t0 = ev[0][0]
    rows = [(c - t0, r, NAMES.get(k, str(k)), a, b) for c, r, k, a, b in ev]
    for row in rows:
        print(f"{row[0]:8d}  {row[1]:9s} {row[2]:16s} a={row[3]:3d} t={row[4]}")
    if out:
        json.dump(rows, open(out, "w"))


if __name__ == "__main__":
    main()
