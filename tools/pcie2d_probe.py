"""Strided (Grid layout -> pitched device rows, cudaMemcpy2D) vs contiguous
copies of the config-3 grid, each direction alone and both at once."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04868_b200 import Grid, _native  # noqa: E402

ext = (16384, 16384)
# PINNED=1: Grids on tvs_host_alloc storage; else numpy pages + cudaHostRegister
pinned = os.environ.get("PINNED") == "1"
g = Grid(ext, 1, pinned=pinned)
g.data[...] = 1.0
o = g.alloc_like()
if not pinned:
    _native.host_register(g.data)
    _native.host_register(o.data)
print("pinned" if pinned else "registered")
geo = _native.geometry(2, ext)
n = int(geo.alloc_elems)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
lay = _native.make_layout(g.data, ext, g.offset)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def up(s):
    _native.check(_native.lib().tvs_upload(C.byref(geo), C.c_void_p(d1.data_ptr()), C.byref(lay),
                                           C.c_void_p(g.data.ctypes.data), C.c_void_p(s.cuda_stream)))


def down(s):
    _native.check(_native.lib().tvs_download(C.byref(geo), C.c_void_p(d2.data_ptr()), C.byref(lay),
                                             C.c_void_p(o.data.ctypes.data), C.c_void_p(s.cuda_stream)))


def timed(fn):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


gb = ext[0] * ext[1] * 8 / 1e9
t = timed(lambda: up(s1)); print(f"2D H2D alone {t:.1f} ms {gb / t * 1e3:.1f} GB/s")
t = timed(lambda: down(s2)); print(f"2D D2H alone {t:.1f} ms {gb / t * 1e3:.1f} GB/s")
t = timed(lambda: (up(s1), down(s2))); print(f"2D both {t:.1f} ms")
h1 = torch.from_numpy(g.data.reshape(-1))
h2 = torch.from_numpy(o.data.reshape(-1))
m = ext[0] * (ext[1] + 9)
t = timed(lambda: d1[:m].copy_(h1[:m], non_blocking=True)); print(f"1D H2D alone {t:.1f} ms {m * 8 / 1e9 / t * 1e3:.1f} GB/s")
t = timed(lambda: h2[:m].copy_(d2[:m], non_blocking=True)); print(f"1D D2H alone {t:.1f} ms {m * 8 / 1e9 / t * 1e3:.1f} GB/s")


def both1d():
    with torch.cuda.stream(s1):
        d1[:m].copy_(h1[:m], non_blocking=True)
    with torch.cuda.stream(s2):
        h2[:m].copy_(d2[:m], non_blocking=True)


t = timed(both1d); print(f"1D both {t:.1f} ms")
