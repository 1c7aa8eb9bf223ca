"""The reference's own kernel benchmark (``mgsr bench``, cli.py:277-311) for the cuda plugin:
ms per GS sweep and per laplacian at the reference's sizes (96, 192, 384) and larger ones, through
``kernels.gs_sweeps`` / ``kernels.laplacian`` with host numpy arrays (the plugin level of
INTEGRATION.md: a host->device->host round trip per call) and with device-resident tensors,
next to the reference's compiled Cython backend (oracle/_ref) on the host cores.  Not collected
by pytest.

    python tests/kernel_bench.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2403_07936_b200 import kernels  # noqa: E402


def best(fn, repeats=3):
    ts = []
    for _ in range(repeats):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    import oracle
    ref = oracle.import_ref()
    sweeps = 20
    rows = []
    for n in (96, 192, 384, 1024, 4096):
        rng = np.random.default_rng(0)
        f = rng.standard_normal((n, n))
        f -= f.mean()
        h2 = (2.0 * np.pi / n) ** 2
        p = np.zeros((n, n))
        row = {"n": n, "sweeps": sweeps}
        row["cuda_host_ms_per_sweep"] = 1e3 * best(lambda: kernels.gs_sweeps(p, f, h2, sweeps)) / sweeps
        row["cuda_host_ms_laplacian"] = 1e3 * best(lambda: kernels.laplacian(p, 1.0 / h2))
        dp, df = torch.from_numpy(p).cuda(), torch.from_numpy(f).cuda()
        row["cuda_device_ms_per_sweep"] = 1e3 * best(lambda: kernels.gs_sweeps(dp, df, h2, sweeps)) / sweeps
        row["cuda_device_ms_laplacian"] = 1e3 * best(lambda: kernels.laplacian(dp, 1.0 / h2))
        if ref is not None and n <= 1024:
            from mgsr.kernels import _stencil
            q = np.zeros((n, n))
            row["cython_ms_per_sweep"] = 1e3 * best(lambda: _stencil.gs_sweeps(q, f, h2, sweeps), 1) / sweeps
            row["cython_ms_laplacian"] = 1e3 * best(lambda: _stencil.laplacian(q, 1.0 / h2), 1)
        rows.append(row)
        print(json.dumps(row), flush=True)
    if out:
        json.dump({"note": "reference `mgsr bench` table for the cuda plugin; host = numpy arrays staged per call, "
                           "device = CUDA tensors; cython = the reference's compiled backend (oracle/_ref), one core",
                   "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
