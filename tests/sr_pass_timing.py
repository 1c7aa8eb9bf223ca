"""SR-prolongation timing by ratio and precision through ops.sr_prolong on device-resident tensors
(CUDA events, best of 3 after a warm-up; includes the per-call workspace and the normalise / mean
launches).  Windows = (n_c / 2 - 2)^2 per pass.  Not collected by pytest.

    python tests/sr_pass_timing.py [out.json]
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


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    w = tg._trained(8)
    rows = []
    for s, nc, precs in [(2, 2048, ("fp16",)), (4, 768, ("fp16", "fp32")), (4, 1024, ("fp16",)),
                         (16, 12, ("fp16", "mixed", "fp32")), (16, 192, ("fp16", "mixed", "fp32")), (8, 384, ("fp16", "mixed"))]:
        f = datagen.scale_to_p_rms(datagen.grf_blobs_rhs(nc, seed=5, kmax=nc / 8), 1e-4)
        c = torch.from_numpy(datagen.spectral_solution(f)).cuda()
        for pr in precs:
            ms = timed(lambda: ops.sr_prolong(c, w.device_handle(), s, 1e-10, 1e-3, _lib.PREC[pr]))
            nw = (nc // 2 - 2) ** 2
            rows.append({"ratio": s, "n_c": nc, "precision": pr, "ms": ms, "windows_first_pass": nw})
            print(json.dumps(rows[-1]), flush=True)
    if len(sys.argv) > 1:
        json.dump(rows, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
