"""2D Jacobi drop-in parity through tvs_run's pipelined host path for one
band size (TVS_E2E_BANDS, read once per process; 0 = single-stream path).
Run by tests/test_gpu_parity.py::test_jacobi2d_pipelined_e2e_bands; exits
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

# (rows, cols, steps, depth): >= 4 bands, ragged last band, bands shifted by the
# levels of every pass (skewed pipeline),
# T not a multiple of the depth, 1-step runs, both P regimes (D <= 4, D 5..8)
CASES = [(4100, 130, 19, 0), (4096, 333, 8, 0), (5000, 64, 1, 0), (9000, 50, 33, 5), (4608, 97, 12, 3),
         (4096, 40, 700, 0)]  # total band shift (700 rows) beyond one band: empty / clipped bands
bad = 0
for kernel in ("heat2d", "jac2d9p"):
    for rows, cols, steps, depth in CASES:
        g = Grid.random((rows, cols), seed=rows + cols + steps, boundary=0.25)
        spec = dataclasses.replace(get(kernel).spec, boundary=g.boundary)
        with config.using(depth=depth):
            got = execute(spec, g, steps)  # the drop-in's path: tvs_run on host buffers
        want = cref.scalar_reference(spec, g, steps, order="lexicographic", threads=8)
        ok = np.array_equal(got.interior, want.interior) and np.all(got.data[: got.offset] == g.boundary)
        bad += not ok
        print(f"{'ok  ' if ok else 'FAIL'} {kernel} {rows}x{cols} T={steps} depth={depth}")
sys.exit(1 if bad else 0)
