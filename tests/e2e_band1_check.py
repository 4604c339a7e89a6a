"""1D Jacobi drop-in parity through tvs_run's pipelined band path for one
band length (TVS_E2E_BAND1; 0 = plain path).  Run by
tests/test_gpu_parity.py::test_jacobi1d_pipelined_e2e_bands; exits non-zero
on any mismatch."""
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

# (n, steps, depth): ragged last band, T not a multiple of the depth, total
# shift beyond several bands, 1 step, shallow blocks
CASES = [(5000, 300, 0), (20000, 1000, 0), (8192, 1, 0), (12345, 65, 0), (9000, 77, 7)]
bad = 0
for kernel in ("heat1d", "gs1d_w343"):
    for n, steps, depth in CASES:
        g = Grid.random((n,), seed=n + steps, boundary=0.25)
        spec = dataclasses.replace(get(kernel).spec, boundary=g.boundary, dependence_kind="jacobi")
        with config.using(depth=depth, fma="never"):
            got = execute(spec, g, steps)
        want = cref.scalar_reference(spec, g, steps, threads=8)
        ok = np.array_equal(got.interior, want.interior) and np.all(got.data[: got.offset] == g.boundary)
        bad += not ok
        print(f"{'ok  ' if ok else 'FAIL'} {kernel} n={n} T={steps} depth={depth}")
sys.exit(1 if bad else 0)
