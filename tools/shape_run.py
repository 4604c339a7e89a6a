"""Device-resident timing of one stencil on an arbitrary shape:
    python tools/shape_run.py gs2d9p 8192 2048 --T 100"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04868_b200 import _native, config  # noqa: E402
from paper_2010_04868_b200.catalog import get  # noqa: E402
from paper_2010_04868_b200.grid import Grid  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("kernel")
ap.add_argument("ext", type=int, nargs="+")
ap.add_argument("--T", type=int, default=10)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--depth", type=int, default=0)
a = ap.parse_args()
g = Grid.random(tuple(a.ext), seed=1)
plan = _native.Plan(get(a.kernel).spec, tuple(a.ext), config.current().native(depth=a.depth))
plan.upload(g.data, g.offset)
for _ in range(a.reps):
    plan.run(a.T)
    plan.synchronize()
ms = plan.last_ms()
print(f"{a.kernel} {tuple(a.ext)} T={a.T}: {ms:.3f} ms -> {np.prod(a.ext) * a.T / ms / 1e6:.1f} GStencil/s")
plan.close()
