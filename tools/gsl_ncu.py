"""One config-4 run of the GS-2D lane kernel (for ncu capture)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
t, _ = bench.device_time(bench.CONFIGS[4], 1, 3, order=sys.argv[1] if len(sys.argv) > 1 else "lexicographic")
print("ms", t)
