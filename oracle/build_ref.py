"""Recipe: compile the REFERENCE package from its own sources into oracle/_ref.

TEST INFRASTRUCTURE ONLY.  The reference (``/root/reference/pkg/src/mgsr``)
is ~2k lines of Python/NumPy plus one Cython file.  Cython compiles every one
of those modules, exactly as they lie under /root/reference, into CPython
extension modules; the outputs (``oracle/_ref/mgsr/**.so``) are the only
files written.  No reference source is copied into the repository: the
generated C goes to a scratch directory under /tmp and ``oracle/_ref`` is
git-ignored (but not gpurun-ignored), so the real reference travels to the
GPU box as a binary and serves as the CPU baseline (``kind: "reference"``)
and as a live parity checker there.

The stencil module is built with the reference's own flags
(pkg/setup.py:32-42: ``-O3 -ffp-contract=off``).

Usage:  python oracle/build_ref.py   (no-op when /root/reference is absent)
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile

REF = "/root/reference/pkg/src/mgsr"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
MODULES = ["__init__", "grid", "smoother", "transfer", "srmodel", "solver", "datagen",
           "kernels/__init__", "kernels/numpy_backend"]


def built() -> bool:
    return os.path.isdir(os.path.join(OUT, "mgsr")) and any(
        f.startswith("solver") and f.endswith(".so") for f in os.listdir(os.path.join(OUT, "mgsr")))


def main(force: bool = False) -> int:
    if not os.path.isdir(REF):
        print("build_ref: /root/reference absent; keeping prebuilt oracle/_ref if any")
        return 0
    if built() and not force:
        print("build_ref: oracle/_ref already built")
        return 0
    import numpy as np
    from Cython.Build import cythonize
    from setuptools import Extension, setup

    exts = []
    for m in MODULES:
        exts.append(Extension("mgsr." + m.replace("/", "."), [f"{REF}/{m}.py"]))
    exts.append(Extension("mgsr.kernels._stencil", [f"{REF}/kernels/_stencil.pyx"],
                          include_dirs=[np.get_include()],
                          extra_compile_args=["-O3", "-ffp-contract=off"]))
    scratch = tempfile.mkdtemp(prefix="mgsr_ref_build_")
    try:
        setup(ext_modules=cythonize(exts, build_dir=os.path.join(scratch, "c"), language_level=3,
                                    quiet=True, nthreads=os.cpu_count() or 1),
              script_args=["build_ext", "--build-lib", OUT, "--build-temp",
                           os.path.join(scratch, "o"), "--parallel", str(os.cpu_count() or 1)])
    finally:
        shutil.rmtree(scratch, ignore_errors=True)
    print(f"build_ref: reference compiled into {OUT}")
    return 0


if __name__ == "__main__":
    sys.exit(main(force="--force" in sys.argv))
