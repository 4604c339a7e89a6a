"""Repeat-run stress for the pipelined kernels (races show up as run-to-run
differences): K6v3 both orders, K4c, K2 on mid-size grids, N repeats each,
every result compared bit for bit with the first and the first with the C
oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import cref
from paper_2010_04868_b200 import Grid
from paper_2010_04868_b200.catalog import get
from paper_2010_04868_b200.kernels._common import execute

N = int(sys.argv[1]) if len(sys.argv) > 1 else 12
bad = 0
cases = (("gs2d9p", (1500, 2100), 100, {"order": "lexicographic"}), ("gs2d9p", (1200, 1700), 100, {"order": "reference"}),
         ("gs2d9p", (3000, 700), 37, {"order": "lexicographic"}), ("gs2d", (900, 1300), 64, {"order": "reference"}),
         ("jac3d27p", (150, 130, 200), 8, {}), ("heat1d", (300001,), 333, {}))
for kernel, ext, steps, kw in cases:
    g = Grid.random(ext, seed=7)
    spec = get(kernel).spec
    t0 = time.time()
    want = cref.scalar_reference(spec, g, steps, **kw).interior
    first = execute(spec, g, steps, **kw).interior
    ok = np.array_equal(first, want)
    diffs = 0
    for _ in range(N - 1):
        diffs += not np.array_equal(execute(spec, g, steps, **kw).interior, first)
    bad += (not ok) + diffs
    print("ok  " if ok and not diffs else "FAIL", kernel, ext, steps, kw, "oracle", ok, "run-to-run diffs", diffs, f"{time.time()-t0:.1f}s", flush=True)
sys.exit(1 if bad else 0)
