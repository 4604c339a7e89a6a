"""GS-2D lane kernel (K6v2) quick check: parity vs the C oracle (both
orders, box and star) over shapes / sweep counts, then config-4 timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import cref
from paper_2010_04868_b200 import Grid, _native, config
from paper_2010_04868_b200.catalog import get
from paper_2010_04868_b200.kernels._common import execute

bad = 0
for kernel in ("gs2d9p", "gs2d"):
    spec = get(kernel).spec
    for ext, T in (((40, 50), 1), ((37, 61), 5), ((100, 33), 31), ((64, 300), 32), ((50, 70), 33),
                   ((300, 129), 64), ((20, 1000), 100), ((3, 5), 7), ((1, 9), 3), ((200, 200), 100)):
        g = Grid.random(ext, seed=T + ext[0], boundary=0.25 if T % 2 else 0.0)
        for order in ("lexicographic", "reference"):
            got = execute(spec, g, T, order=order).interior
            want = cref.scalar_reference(spec, g, T, order=order).interior
            ok = np.array_equal(got, want)
            bad += not ok
            if not ok:
                rows = np.where((got != want).any(1))[0]
                print("MISMATCH", kernel, ext, T, order, "rows", rows[:10].tolist(), flush=True)
print("parity failures:", bad, flush=True)
import bench
cfg = bench.CONFIGS[4]
for order in ("lexicographic", "reference"):
    t, l = bench.device_time(cfg, 3, 3, order=order)
    print(order, "config 4 ms", [round(x, 2) for x in t], "GSt/s", round(8192 * 8192 * 100 / (np.mean(t) * 1e-3) / 1e9, 1),
          "launches", l, flush=True)
