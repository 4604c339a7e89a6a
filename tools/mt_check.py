"""Concurrent drop-in calls from a thread pool: results vs the single-thread run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from concurrent.futures import ThreadPoolExecutor
import numpy as np
from paper_2010_04868_b200 import Grid, _native
from paper_2010_04868_b200.kernels import jacobi2d_temporal, jacobi3d_temporal

cases = [("3d pipelined", jacobi3d_temporal, (192, 160, 200), "jac3d27p"),
         ("3d plain", jacobi3d_temporal, (100, 60, 70), "jac3d27p"),
         ("2d pipelined", jacobi2d_temporal, (1200, 300), "heat2d")]
for name, fn, ext, k in cases:
    g = Grid.random(ext, seed=3)
    want = fn(g, 2, kernel=k).interior.copy()
    def work(_):
        got = fn(g, 2, kernel=k).interior
        return bool(np.array_equal(got, want)), float(np.max(np.abs(got - want)))
    for workers in (1, 2, 8):
        with ThreadPoolExecutor(max_workers=workers) as pool:
            res = list(pool.map(work, range(8)))
        print(name, "workers", workers, "ok", sum(r[0] for r in res), "/ 8", "maxdiff", max(r[1] for r in res), flush=True)
