"""Small K6v3 / K4c / K2 cases for compute-sanitizer (memcheck, racecheck):
    compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import cref
from paper_2010_04868_b200 import Grid
from paper_2010_04868_b200.catalog import get
from paper_2010_04868_b200.kernels._common import execute

bad = 0
for kernel, ext, steps, kw in (("gs2d9p", (40, 70), 9, {"order": "lexicographic"}), ("gs2d9p", (33, 50), 6, {"order": "reference"}),
                               ("jac3d27p", (12, 40, 70), 4, {}), ("heat1d", (5000,), 70, {})):
    g = Grid.random(ext, seed=3)
    spec = get(kernel).spec
    got = execute(spec, g, steps, **kw).interior
    want = cref.scalar_reference(spec, g, steps, **kw).interior
    ok = np.array_equal(got, want)
    bad += not ok
    print("ok  " if ok else "FAIL", kernel, ext, steps, kw, flush=True)
sys.exit(1 if bad else 0)
