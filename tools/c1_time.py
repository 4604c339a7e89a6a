"""Config 1 (1D heat) device time."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
c = bench.CONFIGS[1]
t, l = bench.device_time(c, 20, 5)
print("ms", round(statistics.mean(t), 4), "GSt/s", round(2**20 * 1000 / (statistics.mean(t) * 1e-3) / 1e9, 1), "launches", l)
