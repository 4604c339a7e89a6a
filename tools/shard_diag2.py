"""Replay test_sharded_drop_in_bitexact's sequence (for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import cref
from paper_2010_04868_b200 import Grid, config
from paper_2010_04868_b200.catalog import get
from paper_2010_04868_b200.kernels import jacobi2d_temporal, jacobi3d_temporal
cases = [("heat2d", (301, 257), 21), ("jac2d9p", (133, 200), 17), ("heat3d", (41, 33, 35), 7), ("jac3d27p", (40, 24, 70), 6)]
if len(sys.argv) > 1:
    cases = [c for c in cases if c[0] in sys.argv[1:]]
for kernel, ext, steps in cases:
    spec = get(kernel).spec
    g = Grid.random(ext, seed=11)
    want = cref.scalar_reference(spec, g, steps).interior
    fn = jacobi2d_temporal if len(ext) == 2 else jacobi3d_temporal
    for n in (1, 2, 3, 4, 5, 8):
        with config.using(emulate_shards=True):
            got = fn(g, steps, kernel=kernel, n_gpus=n).interior
        bad = np.where(np.abs(got - want).reshape(ext[0], -1).max(1) > 0)[0]
        print(kernel, "n", n, "bad planes", bad.tolist()[:20], flush=True)
