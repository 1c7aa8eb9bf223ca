"""GPU bring-up: SR-prolongation field error of the tensor-core paths vs the fp32 path
for several weights / precisions / inputs.  Not collected by pytest."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_07936_b200 import datagen, srmodel  # noqa: E402
from paper_2403_07936_b200.grid import Grid, NormBounds  # noqa: E402

nc = int(sys.argv[1]) if len(sys.argv) > 1 else 128
rng = np.random.default_rng(0)
noise = (10.0 ** rng.uniform(-7, -3.5, (nc, nc))) * np.where(rng.random((nc, nc)) < 0.5, -1, 1)
# smooth correction-like field: discrete solution of a GRF RHS, p_rms 1e-5, mean-free
f = datagen.scale_to_p_rms(datagen.grf_blobs_rhs(nc, seed=3, kmax=nc / 8), 1e-5)
smooth = datagen.spectral_solution(f)
weights = {"he_init_b8": srmodel.random_weights(8, 0),
           "trained_b8": srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b8.mgsr")),
           "trained_b4": srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b4.mgsr"))}
for wn, w in weights.items():
    for inn, c in (("noise", noise), ("smooth", smooth)):
        ref = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp32").data
        row = []
        for pr in ("bf16", "fp16"):
            got = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision=pr).data
            row.append(f"{pr} {np.linalg.norm(got - ref) / np.linalg.norm(ref):.2e}")
        print(f"{wn:12s} {inn:7s} " + "  ".join(row), flush=True)
