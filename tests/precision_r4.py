"""GPU bring-up: multi-pass (ratio 4/8/16) SR-prolongation field error of the tensor-core path
against the fp64 CPU oracle, next to the oracle run with fp16-rounded conv operands (the error the
operand format alone costs).  Not collected by pytest."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import mgsr_oracle as orc  # noqa: E402
from paper_2403_07936_b200 import srmodel  # noqa: E402
from paper_2403_07936_b200.grid import Grid, NormBounds  # noqa: E402
import test_gpu_generator as tg  # noqa: E402

f16 = lambda a: a.astype(np.float16).astype(np.float64)  # noqa: E731
base_conv = orc.conv2d
emulate = "--emulate" in sys.argv
weights = {"trained_b8": tg._trained(8), "trained_b4": tg._trained(4), "he_b1": srmodel.random_weights(1, 3),
           "he_b8": srmodel.random_weights(8, 0)}
for wn, w in weights.items():
    ow = orc.quantize_f32(tg._oracle_weights(orc, w))
    for s, nc in [(4, 12), (4, 40), (8, 16), (8, 40), (16, 12), (16, 24)]:
        c = tg._fields(max(nc, 16))["smooth"][:nc, :nc]
        c = c - c.mean()
        orc.conv2d = base_conv
        ref = orc.sr_prolong(c, ow, orc.Bounds(), s)
        row = []
        for pr in ("fp16", "fp32"):
            got = srmodel.sr_prolong(Grid(c), w, NormBounds(), s, precision=pr).data
            row.append(f"{pr} {np.linalg.norm(got - ref) / np.linalg.norm(ref):.2e}")
        if emulate:
            orc.conv2d = lambda x, w_: base_conv(f16(x), f16(w_))
            emu = orc.sr_prolong(c, ow, orc.Bounds(), s)
            row.append(f"fp16-emulated {np.linalg.norm(emu - ref) / np.linalg.norm(ref):.2e}")
        print(f"{wn:11s} s={s:2d} nc={nc:3d} " + "  ".join(row), flush=True)
