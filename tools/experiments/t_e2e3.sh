for b in 256 1024; do TVS_E2E_TRACE=1 TVS_E2E_BANDS=$b timeout 300 python bench.py --steps 2 --warmup 3 --no-all --no-cpu 2>&1 | grep "\[e2e\]" | tail -2; done
python - <<'PY'
import numpy as np, torch, time
n = 2 * 1024**3 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); a=time.perf_counter()-t
    t=time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); b=time.perf_counter()-t
print(f"H2D {2/a:.1f} GiB/s  D2H {2/b:.1f} GiB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.float64).pin_memory(); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t=time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); c=time.perf_counter()-t
print(f"concurrent H2D+D2H of 2 GiB each: {c*1e3:.1f} ms")
PY
