"""Where the stock drop-in call (pageable Grid in, fresh Grid out) spends its
time on config 3: pageable vs page-locked input / output, allocation."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2010_04868_b200 import Grid, _native
from paper_2010_04868_b200.kernels import jacobi2d_temporal
from paper_2010_04868_b200.catalog import get

cfg = bench.CONFIGS[3]
T = cfg["T"]
g_page = bench.make_grid(cfg)
g_pin = Grid(g_page.extents, 1, pinned=True); np.copyto(g_pin.data, g_page.data)
o_pin = Grid(g_page.extents, 1, pinned=True)
o_page = g_page.copy()  # faulted-in pageable

def tm(label, f, n=3):
    f()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); f(); ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{label:40s} {min(ts):8.1f} ms  (all {[round(x,1) for x in ts]})", flush=True)

tm("result_like (np.empty + frame)", lambda: g_page.result_like())
tm("np.empty + touch (memset)", lambda: np.empty(g_page.data.shape).fill(0))
tm("pinned in, pinned out", lambda: jacobi2d_temporal(g_pin, T, out=o_pin))
tm("pageable in, pinned out", lambda: jacobi2d_temporal(g_page, T, out=o_pin))
tm("pinned in, pageable out (faulted)", lambda: jacobi2d_temporal(g_pin, T, out=o_page))
tm("pageable in, pageable out (faulted)", lambda: jacobi2d_temporal(g_page, T, out=o_page))
tm("stock (pageable in, fresh out)", lambda: jacobi2d_temporal(g_page, T))
