"""Config 3 device time vs temporal depth (current default arithmetic)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2010_04868_b200 import config
c = bench.CONFIGS[3]
for d in [int(x) for x in sys.argv[1:]] or [6, 7, 8, 9, 10]:
    with config.using(depth=d):
        clk = bench.ClockSampler()
        t, l = bench.device_time(c, 5, 3, sampler=clk)
    print("depth", d, "GSt/s", round(16384**2 * 200 / (statistics.mean(t) * 1e-3) / 1e9, 1), "launches", l, clk.summary().get("sm_mhz"), flush=True)
