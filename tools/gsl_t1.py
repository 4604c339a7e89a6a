import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import cref
from paper_2010_04868_b200 import Grid
from paper_2010_04868_b200.catalog import get
from paper_2010_04868_b200.kernels._common import execute
spec = get("gs2d9p").spec
for rows, cols, T in [(300, 64, 1), (1000, 64, 1), (1300, 64, 1), (1400, 64, 1), (2048, 64, 1), (2048, 64, 2), (2048, 64, 5), (2048, 200, 1), (1300, 64, 33), (3000, 64, 40)]:
    g = Grid.random((rows, cols), seed=rows + cols + T)
    got = execute(spec, g, T).interior
    want = cref.scalar_reference(spec, g, T, order="lexicographic").interior
    bad = np.where((got != want).any(1))[0]
    print(rows, cols, T, "ok" if bad.size == 0 else f"bad rows {bad[:8].tolist()} n={bad.size}", flush=True)
