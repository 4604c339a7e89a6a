"""Parity of the two-level 3D kernels in a mode fixed per process by the
environment: TVS_J3D=cpasync (K4b, the cp.async-staged kernel K4c falls back
to when a block cannot be a tensor map) or TVS_J3D_FRAME=32 / 64 (K4c's frame
height; 32 by default).  Run by
tests/test_gpu_parity.py::test_jacobi3d_modes; exits non-zero on any
mismatch."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import cref  # noqa: E402  (test infrastructure only)
from paper_2010_04868_b200 import Grid  # noqa: E402
from paper_2010_04868_b200.catalog import get  # noqa: E402
from paper_2010_04868_b200.kernels._common import execute  # noqa: E402
import dataclasses  # noqa: E402

assert os.environ.get("TVS_J3D") == "cpasync" or os.environ.get("TVS_J3D_FRAME") in ("32", "64")
bad = 0
for kernel in ("heat3d", "jac3d27p"):
    for ext in ((1, 1, 1), (2, 30, 62), (70, 31, 63), (65, 61, 125), (131, 29, 200), (9, 63, 62), (20, 130, 70)):
        g = Grid.random(ext, seed=sum(ext), boundary=0.375)
        spec = dataclasses.replace(get(kernel).spec, boundary=g.boundary)
        want = cref.scalar_reference(spec, g, 7)
        for depth in (0, 2):
            got = execute(spec, g, 7, depth=depth, fma="never")
            ok = np.array_equal(got.interior, want.interior)
            bad += not ok
            print(f"{'ok  ' if ok else 'FAIL'} {kernel} {ext} depth={depth}")
sys.exit(1 if bad else 0)
