"""LCS kernel timing across shapes (device-resident, CUDA events):
per-step cycles = time x clock / (nb + 128*warps...) diagnostics."""
import ctypes as C
import sys
import os
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04868_b200 import _native  # noqa: E402

for na, nb in [(128, 1 << 20), (1024, 1 << 20), (128 * 148, 1 << 16), (65536, 65536), (65536, 8192)]:
    rng = np.random.default_rng(1)
    a = torch.from_numpy(rng.integers(0, 4, na).astype(np.int32)).cuda()
    b = torch.from_numpy(rng.integers(0, 4, nb).astype(np.int32)).cuda()
    r = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    ts = []
    for i in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        _native.check(_native.lib().tvs_lcs_device(C.c_void_p(a.data_ptr()), na, C.c_void_p(b.data_ptr()), nb,
                                                   C.c_void_p(r.data_ptr()), C.c_void_p(s.cuda_stream)))
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    warps = (na + 127) // 128
    steps = nb + 127 + (warps - 1) * 159
    print(f"na {na} nb {nb}: {ms:.3f} ms  {na * nb / ms / 1e6:.1f} GCells/s  warps {warps}  "
          f"~{ms * 1.9e6 / steps:.0f} cycles per step (model steps {steps})")
