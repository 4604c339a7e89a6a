"""Clock / power / throughput probe for one stencil on one shape, device
resident, with nvidia-smi sampled during the run:
    python tools/power_probe.py heat3d27 1024 1024 1024 --T 20 --fma allow --algo naive
Prints one line: GStencil/s, effective GB/s (16 B/update), median SM clock,
median power, throttle reasons."""
import argparse
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04868_b200 import _native, config  # noqa: E402
from paper_2010_04868_b200.catalog import get  # noqa: E402
from paper_2010_04868_b200.grid import Grid  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("kernel")
ap.add_argument("ext", type=int, nargs="+")
ap.add_argument("--T", type=int, default=10)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--depth", type=int, default=0)
ap.add_argument("--fma", default="exact")
ap.add_argument("--algo", default="auto")
a = ap.parse_args()

g = Grid.random(tuple(a.ext), seed=1)
plan = _native.Plan(get(a.kernel).spec, tuple(a.ext), config.current().native(depth=a.depth, fma=a.fma, algo=a.algo))
plan.upload(g.data, g.offset)
plan.run(a.T)
plan.synchronize()

lines = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
th = threading.Thread(target=lambda: [lines.append(l.strip()) for l in proc.stdout], daemon=True)
th.start()
time.sleep(0.3)
lines.clear()
ms = []
for _ in range(a.reps):
    plan.run(a.T)
    plan.synchronize()
    ms.append(plan.last_ms())
proc.terminate()
clk, pw, rs = [], [], set()
for l in lines:
    p = [x.strip() for x in l.split(",")]
    try:
        clk.append(float(p[0]))
        pw.append(float(p[1]))
        rs.add(p[2])
    except (ValueError, IndexError):
        pass
m = statistics.median(ms)
rate = np.prod(a.ext) * a.T / m / 1e6
print(f"{a.kernel} {tuple(a.ext)} T={a.T} fma={a.fma} algo={a.algo} depth={a.depth}: {m:.3f} ms "
      f"{rate:.1f} GSt/s eff {rate * 16:.0f} GB/s launches {plan.last_launches()} "
      f"clk {statistics.median(clk) if clk else None} MHz power {statistics.median(pw) if pw else None} W "
      f"reasons {sorted(rs)} samples {len(clk)}", flush=True)
plan.close()
