"""Regenerate the reference trainer's parity fixtures for the committed trained weights, by running
the REFERENCE's own pipeline (pkg/artifacts/trained/PROVENANCE.md:11-19) in the build container:

    python tests/golden/make_trainer_fixtures.py

1. ``mgsr datagen --kind windows --n 192 --fields 200 --count 1000 --k-peak 8 --p-rms 1e-4 --seed 42``
   (the reference CLI, in-process) -> /tmp MGWP corpus;
2. ``mgsr-train fixtures --weights artifacts/trained_b{4,8}.mgsr --data <corpus> --count 10 --seed 0
   --include-zero`` (the reference trainer's torch fp32 generator, eval mode) -> /tmp fixture blobs;
3. the ten (3,6,6) inputs and (3,12,12) outputs per weight file -> tests/golden/trainer_fixtures.npz.

The fixtures are recorded from the weight files themselves, so they pin this repo's generator to the
reference TRAINER's implementation (torch), independently of the reference solver's NumPy one.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)



def main() -> None:
    # the reference's pure-Python tree (its CLI is not part of the Cythonized oracle/_ref build)
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, "/root/reference/pkg/trainer/src")
    from mgsr import cli as ref_cli
    from mgsr_trainer import cli as tr_cli
    tmp = tempfile.mkdtemp()
    corpus = os.path.join(tmp, "pairs.mgwp")
    assert ref_cli.main(["datagen", "--kind", "windows", "--n", "192", "--fields", "200", "--count", "1000",
                         "--k-peak", "8", "--p-rms", "1e-4", "--seed", "42", "--out", corpus]) == 0
    out = {}
    for b in (4, 8):
        wpath = os.path.join(ROOT, "artifacts", f"trained_b{b}.mgsr")
        fdir = os.path.join(tmp, f"fx{b}")
        assert tr_cli.main(["fixtures", "--weights", wpath, "--data", corpus, "--out-dir", fdir, "--count", "10",
                            "--seed", "0", "--include-zero"]) == 0
        man = json.load(open(os.path.join(fdir, "manifest.json")))
        ins = [np.fromfile(os.path.join(fdir, p["input"]), dtype="<f4").reshape(man["input_shape"]) for p in man["pairs"]]
        outs = [np.fromfile(os.path.join(fdir, p["output"]), dtype="<f4").reshape(man["output_shape"])
                for p in man["pairs"]]
        out[f"b{b}_inputs"], out[f"b{b}_outputs"] = np.stack(ins), np.stack(outs)
    np.savez_compressed(os.path.join(HERE, "trainer_fixtures.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
