"""Generate tests/golden/acceptance_cells.json from the REAL reference.

The reference's acceptance matrix (tvstencil/verify.py:169-222,
``default_matrix(cells_per_kernel=20)`` as used by test_acceptance.py:32-41)
is recorded cell by cell — kernel, scheme, single_array, size, seed, steps —
together with the FNV-1a-64 checksum of the reference's own result for that
cell (``scalar_reference`` of the seeded Grid, TSTN dump, grid.py:96-133; for
LCS cells the ``lcs_reference`` length).  tests/test_acceptance_gpu.py replays
exactly these cells on the GPU.  Run in the build container:
    python tests/golden/make_acceptance.py
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_reference  # noqa: E402


def main():
    ref = load_reference()
    import importlib

    verify = importlib.import_module("tvstencil_ref.verify")
    baselines = importlib.import_module("tvstencil_ref.baselines")
    catalog = importlib.import_module("tvstencil_ref.catalog")
    grid_mod = importlib.import_module("tvstencil_ref.grid")
    t0 = time.time()
    cells = verify.default_matrix(cells_per_kernel=20)
    out = []
    for c in cells:
        rec = {"kernel": c.kernel, "scheme": c.scheme, "single_array": bool(c.single_array),
               "size": [int(x) for x in c.size], "seed": int(c.seed), "steps": int(c.steps)}
        if c.kernel == "lcs":
            rng = np.random.default_rng(c.seed)
            a = rng.integers(0, 4, size=c.size[0], dtype=np.int32)
            b = rng.integers(0, 4, size=c.size[1], dtype=np.int32)
            rec["lcs"] = int(baselines.lcs_reference(a, b))
        else:
            entry = catalog.get(c.kernel)
            g = grid_mod.Grid.random(c.size, seed=c.seed, element_kind=entry.spec.element_kind, vl=entry.vl)
            want = baselines.scalar_reference(entry.spec, g, c.steps)
            rec["vl"] = int(entry.vl)
            rec["fnv1a64"] = f"{grid_mod.fnv1a64(want.dump_bytes()):016x}"
        out.append(rec)
    meta = {"source": "tvstencil verify.default_matrix(cells_per_kernel=20, master_seed=2024)",
            "cells": out, "seconds": round(time.time() - t0, 1)}
    with open(os.path.join(HERE, "acceptance_cells.json"), "w") as fh:
        json.dump(meta, fh, indent=0)
    print(len(out), "cells", meta["seconds"], "s")


if __name__ == "__main__":
    main()
