"""2D Gauss-Seidel drop-in parity through tvs_run's pipelined path (row-band
uploads / downloads overlapping the pipeline kernel through stream memory
operations) for one band size (TVS_E2E_BANDS; 0 = plain path).  Run by
tests/test_gpu_parity.py::test_gs2d_pipelined_e2e_bands; exits non-zero on
any mismatch."""
import dataclasses
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import cref  # noqa: E402  (test infrastructure only)
from paper_2010_04868_b200 import Grid  # noqa: E402
from paper_2010_04868_b200.catalog import get  # noqa: E402
from paper_2010_04868_b200.kernels._common import execute  # noqa: E402

# (rows, cols, sweeps): narrow (cluster hand-off) and wide grids, ragged last
# band, 1 sweep, a full 128-sweep pass, and 130 sweeps (two passes: plain path)
CASES = [(1100, 300, 37), (4096, 500, 100), (2048, 64, 1), (1300, 2100, 128), (1500, 100, 130)]
bad = 0
for kernel in ("gs2d9p", "gs2d"):
    for rows, cols, steps in CASES:
        g = Grid.random((rows, cols), seed=rows + cols + steps, boundary=0.125)
        spec = dataclasses.replace(get(kernel).spec, boundary=g.boundary)
        got = execute(spec, g, steps)
        want = cref.scalar_reference(spec, g, steps, order="lexicographic")
        ok = np.array_equal(got.interior, want.interior) and np.all(got.data[: got.offset] == g.boundary)
        bad += not ok
        print(f"{'ok  ' if ok else 'FAIL'} {kernel} {rows}x{cols} T={steps}")
sys.exit(1 if bad else 0)
