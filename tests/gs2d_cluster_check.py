"""GS-2D pipeline parity for one cluster size (set TVS_GS2D_CLUSTER before the
library loads; the size is read once per process).  Run by
tests/test_gpu_parity.py::test_gs2d_pipeline_cluster_sizes; prints one line
per case and exits non-zero on any mismatch."""
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

# (rows, cols, sweeps): rows set the number of blocks (ceil((rows + 127) / 4))
CASES = [(5, 7, 1), (40, 37, 5), (97, 64, 100), (130, 9, 128), (61, 300, 129), (257, 33, 17), (9, 1000, 3),
         (700, 40000, 1)]  # more blocks than resident and c_end > 148 * 256: global-ring sizing
bad = 0
for kernel in ("gs2d9p", "gs2d"):
    for rows, cols, steps in CASES:
        if kernel == "gs2d" and rows * cols > 10 ** 6:
            continue
        g = Grid.random((rows, cols), seed=rows * 7 + cols + steps, boundary=0.5 if rows % 2 else -0.25)
        spec = dataclasses.replace(get(kernel).spec, boundary=g.boundary)
        got = execute(spec, g, steps)
        want = cref.scalar_reference(spec, g, steps, order="lexicographic")
        ok = np.array_equal(got.interior, want.interior)
        bad += not ok
        print(f"{'ok  ' if ok else 'FAIL'} {kernel} {rows}x{cols} T={steps}")
sys.exit(1 if bad else 0)
