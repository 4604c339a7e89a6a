"""Diagnose sharded 3D mismatches: per-plane error by shard count / steps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import cref
from paper_2010_04868_b200 import Grid, config
from paper_2010_04868_b200.catalog import get
from paper_2010_04868_b200.kernels import jacobi3d_temporal

for kernel, ext in (("jac3d27p", (40, 24, 70)), ("heat3d", (40, 24, 70)), ("jac3d27p", (40, 33, 35))):
    spec = get(kernel).spec
    g = Grid.random(ext, seed=11)
    for steps in (1, 2, 4, 6):
        want = cref.scalar_reference(spec, g, steps).interior
        for n in (2, 3, 4):
            with config.using(emulate_shards=True):
                got = jacobi3d_temporal(g, steps, kernel=kernel, n_gpus=n).interior
            bad = np.where(np.abs(got - want).reshape(ext[0], -1).max(1) > 0)[0]
            print(kernel, ext, "T", steps, "n", n, "bad planes", bad.tolist()[:20], flush=True)
