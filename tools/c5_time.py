"""Config 5 device time, bit-exact and fma='allow'."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
c = bench.CONFIGS[5]
for fma in (None, "allow"):
    t, l = bench.device_time(c, 2, 3, fma=fma)
    print(fma or "exact", "ms", [round(x, 1) for x in t], "GSt/s", round(1024**3 * 100 / (statistics.mean(t) * 1e-3) / 1e9, 1))
