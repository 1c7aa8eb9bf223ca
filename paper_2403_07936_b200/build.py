"""Build the in-tree CUDA library ``libmgsr_b200.so`` for sm_100a.

    python -m paper_2403_07936_b200.build      (or __graft_entry__.build())

Each .cu compiles to an object with nvcc (-gencode arch=compute_100a,code=sm_100a,
-lineinfo); the fp64 stencil objects additionally use --fmad=false so that
every product/sum rounds like the reference's -ffp-contract=off loops.  The
objects link into one shared library next to this file (git-ignored; it
travels to the GPU box with the snapshot).
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libmgsr_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{ROOT}/include", f"-I{CSRC}"]
SOURCES = {
    "stencil.cu": ["--fmad=false"],
    "plan.cu": ["--fmad=false"],
    "rng.cu": ["--fmad=false"],
    "generator_simt.cu": [],
    "generator_tc.cu": ["-maxrregcount=112"],
}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or cand == "nvcc"):
            return cand
    return "nvcc"


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "mgsr_b200.h"))
    jobs = []
    for src, extra in SOURCES.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        if _stale(o, [s] + headers):
            jobs.append([nvcc(), *ARCH, *COMMON, *extra, "-c", s, "-o", o])
    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(OBJ, s.replace(".cu", ".o")) for s in SOURCES]
    if _stale(LIB, objs):
        run([nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-lcuda"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
