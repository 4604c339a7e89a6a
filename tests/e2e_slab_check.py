"""3D Jacobi drop-in parity through tvs_run's pipelined slab path for one
slab thickness (TVS_E2E_SLAB, read once per process; 0 = single-stream path).
Run by tests/test_gpu_parity.py::test_jacobi3d_pipelined_e2e_slabs; exits
non-zero on any mismatch."""
import dataclasses
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import cref  # noqa: E402  (test infrastructure only)
from paper_2010_04868_b200 import Grid, config  # noqa: E402
from paper_2010_04868_b200.catalog import get  # noqa: E402
from paper_2010_04868_b200.kernels._common import execute  # noqa: E402

# (planes, rows, cols, steps, depth): >= 4 slabs, ragged last slab, odd T
# (last pass a single step), total shift beyond one slab, depth 1
CASES = [(130, 20, 30, 13, 0), (96, 33, 65, 40, 0), (64, 17, 9, 1, 0), (80, 31, 63, 9, 1)]
bad = 0
for kernel in ("heat3d", "jac3d27p"):
    for planes, rows, cols, steps, depth in CASES:
        g = Grid.random((planes, rows, cols), seed=planes + rows + steps, boundary=0.25)
        spec = dataclasses.replace(get(kernel).spec, boundary=g.boundary)
        with config.using(depth=depth, fma="never"):
            got = execute(spec, g, steps)  # the drop-in's path: tvs_run on host buffers
        want = cref.scalar_reference(spec, g, steps, threads=8)
        ok = np.array_equal(got.interior, want.interior) and np.all(got.data[: got.offset] == g.boundary)
        bad += not ok
        print(f"{'ok  ' if ok else 'FAIL'} {kernel} {planes}x{rows}x{cols} T={steps} depth={depth}")
sys.exit(1 if bad else 0)
