"""Where the config-3 drop-in time goes: the band pipeline's copies alone
(no compute; D2H of band b after H2D of band b+1, as in jacobi2d_pipelined)
vs bulk duplex copies vs the real call with TVS_E2E_TRACE timings."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TVS_E2E_TRACE", "1")
from paper_2010_04868_b200 import Grid, _native  # noqa: E402
from paper_2010_04868_b200.catalog import get  # noqa: E402
from paper_2010_04868_b200.kernels._common import execute  # noqa: E402

R, Ccols = 16384, 16384
row = Ccols
n = R * row
h_in = torch.from_numpy(_native.host_empty((n,)))
h_out = torch.from_numpy(_native.host_empty((n,)))
h_in.fill_(1.0)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
up_s = torch.cuda.Stream()
dn_streams = [torch.cuda.Stream() for _ in range(128)]


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def bulk():
    with torch.cuda.stream(up_s):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(dn_streams[0]):
        h_out.copy_(d_b, non_blocking=True)


def pipe(band, per_band_streams, kernel=False):
    nb = R // band
    ev = [torch.cuda.Event() for _ in range(nb)]
    for b in range(nb + 1):
        if b < nb:
            with torch.cuda.stream(up_s):
                sl = slice(b * band * row, (b + 1) * band * row)
                d_a[sl].copy_(h_in[sl], non_blocking=True)
                ev[b].record(up_s)
        d = b - 1
        if d >= 0:
            s = dn_streams[d % len(dn_streams)] if per_band_streams else dn_streams[0]
            s.wait_event(ev[min(d + 1, nb - 1)])
            with torch.cuda.stream(s):
                sl = slice(d * band * row, (d + 1) * band * row)
                if kernel:  # a kernel on the band's rows ahead of its download
                    d_b[sl].mul_(1.0)
                h_out[sl].copy_(d_b[sl], non_blocking=True)


print(f"bulk duplex            {timed(bulk):6.1f} ms", flush=True)
for band in (256,) if os.environ.get("PROBE_SHORT") else (128, 256, 512, 1024):
    print(f"pipe band {band:4d} 1 strm  {timed(lambda: pipe(band, False)):6.1f} ms", flush=True)
    print(f"pipe band {band:4d} per-band {timed(lambda: pipe(band, True)):6.1f} ms", flush=True)
    print(f"pipe band {band:4d} per-band + kernel {timed(lambda: pipe(band, True, True)):6.1f} ms", flush=True)

spec = get("heat2d").spec
g = Grid((R, Ccols), 1, pinned=True)
g.data.fill(0.5)
out = g.alloc_like()
# the copy-only pipeline again, on the Grids' own host storage
h_in = torch.from_numpy(g.data.reshape(-1)[:n])
h_out = torch.from_numpy(out.data.reshape(-1)[:n])
print(f"pipe band  256 per-band on Grid storage {timed(lambda: pipe(256, True)):6.1f} ms", flush=True)
print(f"pipe band  256 per-band + kernel on Grid storage {timed(lambda: pipe(256, True, True)):6.1f} ms", flush=True)
for T in [int(x) for x in os.environ.get("PROBE_T", "8,200").split(",")]:
    for _ in range(3):
        t0 = time.perf_counter()
        execute(spec, g, T, out=out)
        print(f"drop-in T={T}: {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
