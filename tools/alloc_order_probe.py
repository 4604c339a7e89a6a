"""Duplex PCIe rate vs which page-locked buffers are used (allocation order):
four 2 GiB tvs_host_alloc buffers A..D allocated in order, duplex copies
timed on pairs (in, out)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04868_b200 import _native  # noqa: E402

n = 2 * 2 ** 30 // 8
bufs = {}
for k in "ABCD":
    a = _native.host_empty((n,))
    a[...] = 1.0
    bufs[k] = torch.from_numpy(a)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def duplex(hi, ho):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        with torch.cuda.stream(s1):
            d1.copy_(hi, non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def one(h, up):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    (d1.copy_(h, non_blocking=True) if up else h.copy_(d2, non_blocking=True))
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1)


for k in "ABCD":
    print(f"{k}: H2D {one(bufs[k], True):.1f} ms  D2H {one(bufs[k], False):.1f} ms", flush=True)
for pair in ("AB", "CD", "AD", "CB", "BA", "DC"):
    print(f"in {pair[0]} out {pair[1]}: duplex {duplex(bufs[pair[0]], bufs[pair[1]]):.1f} ms", flush=True)
