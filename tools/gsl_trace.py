"""GS-2D lane kernel timeline (variant library built with -DGSL_TRACE):
per-CTA start / first iteration / end, loader poll / cp.async waits and
barrier waits, for one config-4 sized run (one pass, T=100)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2010_04868_b200 import _native, config
from paper_2010_04868_b200.catalog import get
cfg = dict(bench.CONFIGS[4])
if len(sys.argv) > 1:
    cfg["extents"] = tuple(int(x) for x in sys.argv[1].split("x"))
t, _ = bench.device_time(cfg, 1, 3)
print("ms", t, flush=True)
lib = _native.lib()
n = (cfg["extents"][0] + 99 + 4) // 5
buf = (C.c_ulonglong * (8 * 8192))()
lib.tvs_gsl_trace(buf, 8192)
a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 8)[:n].astype(np.float64)
t0 = a[:, 0].min()
st, fi, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3
print("ctas", n, "total us", en.max())
for k in (0, 1, 2, 3, 10, 100, 147, 148, 200, 296, 300, 500, 1000, n // 2, n - 1):
    if k < n:
        print(f"cta {k:5d} start {st[k]:9.1f} first {fi[k]:9.1f} end {en[k]:9.1f} life {en[k]-fi[k]:8.1f} us | waitL {a[k,3]/1e6:7.2f} poll {a[k,4]/1e6:7.2f} waitC {a[k,5]/1e6:7.2f} Mcyc")
life = en - fi
print("lifetime us: median", np.median(life), "min", life.min(), "max", life.max())
print("first-iteration lag per CTA (us): median", np.median(np.diff(fi)))
