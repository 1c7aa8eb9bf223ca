"""Build a variant of libmgsr_b200.so with extra nvcc flags for generator_tc.cu (e.g. -DMGSR_EXP_X=1),
linked with this tree's other objects, for same-box A/B runs (MGSR_LIB=<path> python bench.py).
Not collected by pytest.

    python tests/ab_variant.py exp/libB.so -DMGSR_EXP_X=1              (generator_tc.cu)
    python tests/ab_variant.py exp/libB.so --src stencil.cu -DMGSR_EXP_Y=1
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_07936_b200 import build as b  # noqa: E402


def main():
    out, flags = sys.argv[1], sys.argv[2:]
    src = "generator_tc.cu"
    if flags[:1] == ["--src"]:
        src, flags = flags[1], flags[2:]
    b.build()
    obj = out + "." + src.replace(".cu", ".o")
    subprocess.run([b.nvcc(), *b.ARCH, *b.COMMON, *b.SOURCES[src], *flags, "-c",
                    os.path.join(b.CSRC, src), "-o", obj], check=True)
    objs = [obj if s == src else os.path.join(b.OBJ, s.replace(".cu", ".o")) for s in b.SOURCES]
    subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", out, *objs, "-lcudart", "-lcuda"], check=True)


if __name__ == "__main__":
    main()
