"""fp32 CUDA-core generator timing (the exact mode, and MIXED's first pass of x8 / x16): ops.sr_prolong on
device tensors, CUDA events, best of 3 after a warm-up, with the algorithmic TFLOP/s of the generator
applications (2 x MACs per window: 61.34 MFLOP per 6x6 application, 245.35 per 12x12).  Not collected by pytest.

    python tests/f32_gen_timing.py [out.json]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2403_07936_b200 import _lib, datagen, ops  # noqa: E402
import test_gpu_generator as tg  # noqa: E402
from sr_pass_timing import timed  # noqa: E402


def main():
    w = tg._trained(8)
    rows = []
    for s, nc, pr in [(2, 256, "fp32"), (2, 1024, "fp32"), (4, 192, "fp32"), (4, 384, "fp32"), (16, 192, "mixed"),
                      (8, 384, "mixed"), (16, 12, "mixed")]:
        f = datagen.scale_to_p_rms(datagen.grf_blobs_rhs(nc, seed=5, kmax=nc / 8), 1e-4)
        c = torch.from_numpy(datagen.spectral_solution(f)).cuda()
        ms = timed(lambda: ops.sr_prolong(c, w.device_handle(), s, 1e-10, 1e-3, _lib.PREC[pr]))
        nw = (nc // 2 - 2) ** 2
        flop = nw * (61.34e6 if s == 2 else 61.34e6 + 245.35e6)   # the fp32 pass only
        rows.append({"ratio": s, "n_c": nc, "precision": pr, "ms": ms, "windows_first_pass": nw,
                     "fp32_pass_tflops_if_all_time": flop / ms / 1e9})
        print(json.dumps(rows[-1]), flush=True)
    if len(sys.argv) > 1:
        json.dump(rows, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
