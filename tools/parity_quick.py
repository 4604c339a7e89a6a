"""Quick bit-exact spot check of one kernel family against the C oracle
(for variant libraries selected with TVSTENCIL_LIB)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import cref
from paper_2010_04868_b200 import Grid
from paper_2010_04868_b200.catalog import get
from paper_2010_04868_b200.kernels._common import execute

cases = {"gs2d9p": [((40, 37), 5), ((65, 130), 11), ((300, 257), 100), ((9, 300), 3), ((1000, 700), 130)],
         "gs1d_w343": [((5000,), 257), ((70000,), 140), ((4096,), 1000), ((3001,), 33), ((777,), 70), ((20000,), 95)],
         "heat2d": [((300, 301), 12), ((1000, 999), 48)],
         "heat1d": [((4096,), 100), ((100003,), 1000), ((2 ** 20,), 130)]}
fam = sys.argv[1] if len(sys.argv) > 1 else "gs2d9p"
ok = True
for ext, steps in cases[fam]:
    g = Grid.random(ext, seed=sum(ext) + steps)
    spec = get(fam).spec
    got = execute(spec, g, steps)
    want = cref.scalar_reference(spec, g, steps, order="lexicographic", threads=8)
    same = np.array_equal(got.interior, want.interior)
    ok &= same
    print(fam, ext, steps, "OK" if same else f"MISMATCH max {np.abs(got.interior - want.interior).max()}")
print("PARITY", "PASS" if ok else "FAIL")
