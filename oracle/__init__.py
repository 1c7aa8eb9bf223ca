"""CPU oracle for parity checking -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2403_07936_b200`` never does.

* ``mgsr_oracle``  -- NumPy restatement of the reference hot path.
* ``stencil.c``    -- gcc-built C twin of the reference stencil loops.
* ``build_ref.py`` -- compiles the reference itself into ``oracle/_ref``.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def build_c() -> None:
    """Compile stencil.c -> libmgsr_oracle.so (reference flags: -O3 -ffp-contract=off)."""
    src = os.path.join(HERE, "stencil.c")
    out = os.path.join(HERE, "libmgsr_oracle.so")
    if os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return
    subprocess.check_call(["gcc", "-O3", "-ffp-contract=off", "-shared", "-fPIC", src, "-o", out])


def import_ref():
    """Import the compiled reference package from oracle/_ref (or None)."""
    if not os.path.isdir(os.path.join(REF_DIR, "mgsr")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import mgsr  # noqa: F401
        import mgsr.solver  # noqa: F401
        import mgsr.srmodel  # noqa: F401
        return sys.modules["mgsr"]
    except ImportError:
        return None
