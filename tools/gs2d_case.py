"""One GS-2D pipeline parity case: python tools/gs2d_case.py ROWS COLS T [kernel]"""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cref  # noqa: E402  (checker)
from paper_2010_04868_b200 import Grid  # noqa: E402
from paper_2010_04868_b200.catalog import get  # noqa: E402
from paper_2010_04868_b200.kernels._common import execute  # noqa: E402

rows, cols, steps = (int(x) for x in sys.argv[1:4])
kernel = sys.argv[4] if len(sys.argv) > 4 else "gs2d9p"
g = Grid.random((rows, cols), seed=rows * 7 + cols + steps, boundary=0.5)
spec = dataclasses.replace(get(kernel).spec, boundary=g.boundary)
got = execute(spec, g, steps).interior
want = cref.scalar_reference(spec, g, steps, order="lexicographic").interior
bad = np.argwhere(got != want)
print(f"{kernel} {rows}x{cols} T={steps}: {'ok' if len(bad) == 0 else f'FAIL {len(bad)} cells, first {bad[0].tolist()}, rows {sorted(set(bad[:, 0].tolist()))[:12]}'}")
