"""PCIe copy ceilings for the e2e leg: pinned H2D alone, D2H alone, both at
once on two streams (2 GiB each, CUDA events)."""
import torch

n = 2 * 2 ** 30 // 8
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
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


gb = n * 8 / 1e9
t = timed(lambda: d1.copy_(h1, non_blocking=True))
print(f"H2D alone: {t:.1f} ms {gb / t * 1e3:.1f} GB/s")
t = timed(lambda: h2.copy_(d2, non_blocking=True))
print(f"D2H alone: {t:.1f} ms {gb / t * 1e3:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


t = timed(both)
print(f"H2D + D2H concurrently: {t:.1f} ms, {2 * gb / t * 1e3:.1f} GB/s combined")
