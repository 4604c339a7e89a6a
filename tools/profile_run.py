"""One device-resident run of a BASELINE config (or a reduced-T version) for
ncu captures:  python tools/profile_run.py --config 3 --T 16 [--reps 2]"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2010_04868_b200 import _native, config  # noqa: E402
from paper_2010_04868_b200.catalog import get  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--T", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--fma", default="exact")
ap.add_argument("--depth", type=int, default=0)
ap.add_argument("--algo", default="auto")
a = ap.parse_args()
cfg = dict(bench.CONFIGS[a.config])
T = a.T or cfg["T"]
g = bench.make_grid(cfg)
plan = _native.Plan(get(cfg["kernel"]).spec, cfg["extents"], config.current().native(fma=a.fma, depth=a.depth, algo=a.algo))
plan.upload(g.data, g.offset)
for _ in range(a.reps):
    plan.run(T)
    plan.synchronize()
    print(f"config {a.config} T={T}: {plan.last_ms():.3f} ms, {plan.last_launches()} launches, "
          f"{cfg['extents']} -> {__import__('numpy').prod(cfg['extents']) * T / plan.last_ms() / 1e6:.1f} GStencil/s")
plan.close()
