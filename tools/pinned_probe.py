"""Duplex PCIe rate by host-memory kind (2 GiB each way, both directions at
once on two streams, CUDA events): cudaHostAlloc'd (torch pin_memory) vs
numpy pages registered with cudaHostRegister vs tvs_host_alloc."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04868_b200 import _native  # noqa: E402

n = 2 * 2 ** 30 // 8
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def run(name, h1, h2):
    gb = n * 8 / 1e9
    t_up = timed(lambda: d1.copy_(h1, non_blocking=True))
    t_dn = timed(lambda: h2.copy_(d2, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    t = timed(both)
    print(f"{name:28s} H2D {gb / t_up * 1e3:5.1f} GB/s  D2H {gb / t_dn * 1e3:5.1f} GB/s  both {t:5.1f} ms "
          f"({2 * gb / t * 1e3:5.1f} GB/s)", flush=True)


h1 = torch.ones(n, dtype=torch.float64).pin_memory()
h2 = torch.ones(n, dtype=torch.float64).pin_memory()
run("torch pin_memory", h1, h2)
del h1, h2

a1, a2 = np.ones(n), np.ones(n)
_native.host_register(a1)
_native.host_register(a2)
run("numpy + cudaHostRegister", torch.from_numpy(a1), torch.from_numpy(a2))
_native.host_unregister(a1)
_native.host_unregister(a2)
del a1, a2

if hasattr(_native, "host_array"):
    b1, b2 = _native.host_array(n), _native.host_array(n)
    b1[...] = 1.0
    b2[...] = 1.0
    run("tvs_host_alloc", torch.from_numpy(b1), torch.from_numpy(b2))
