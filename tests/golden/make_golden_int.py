"""Golden vectors for the integer kernels (Life-like rules, LCS) straight
from the REAL reference (imported from /root/reference/pkg/src as
``tvstencil_ref``): ``baselines.scalar_reference`` with ``life_plane_update``
(baselines.py:52-66, 110-125) and ``baselines.lcs_reference``
(baselines.py:128-150).

    python tests/golden/make_golden_int.py   # writes reference_int.{json,npz}
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import HERE, load_reference  # noqa: E402

# (name, dim, birth, survive, boundary, extents, steps, seed)
LIFE = [
    ("life", 2, None, None, 0, (64, 64), 10, 1),
    ("life", 2, None, None, 0, (33, 97), 25, 2),
    ("life", 2, None, None, 1, (40, 130), 7, 5),
    ("conway_b3s23", 2, {3}, {2, 3}, 0, (96, 80), 30, 6),
    ("highlife_b36s23", 2, {3, 6}, {2, 3}, 0, (70, 300), 12, 7),
    ("life1d_b1s12", 1, {1}, {1, 2}, 0, (5000,), 9, 8),
    ("life3d_b4s45", 3, {4}, {4, 5}, 0, (20, 24, 40), 5, 9),
]
# (na, nb, alphabet, seed)
LCS = [(0, 7, 4, 1), (7, 0, 4, 2), (1, 1, 2, 3), (31, 33, 4, 4), (32, 32, 2, 5), (33, 31, 26, 6), (100, 257, 4, 7),
       (1000, 999, 4, 8), (64, 5000, 20, 9), (3000, 70, 3, 10), (2048, 2048, 1 << 30, 11)]


def main():
    ref = load_reference()
    base = ref.catalog.get("life").spec
    arrays, life_cases, lcs_cases = {}, [], []
    for idx, (name, dim, birth, survive, bnd, ext, steps, seed) in enumerate(LIFE):
        spec = dataclasses.replace(base, name=name, dim=dim, boundary=bnd,
                                   birth=frozenset(birth) if birth is not None else base.birth,
                                   survive=frozenset(survive) if survive is not None else base.survive)
        grid = ref.grid.Grid.random(ext, seed=seed, boundary=bnd, element_kind="int32")
        out = ref.baselines.scalar_reference(spec, grid, steps)
        key = f"l{idx:02d}"
        arrays[key + "_in"] = np.ascontiguousarray(grid.interior)
        arrays[key + "_out"] = np.ascontiguousarray(out.interior)
        life_cases.append({"key": key, "name": name, "dim": dim, "birth": sorted(spec.birth),
                           "survive": sorted(spec.survive), "boundary": bnd, "extents": list(ext), "steps": steps,
                           "seed": seed})
    for idx, (na, nb, alpha, seed) in enumerate(LCS):
        rng = np.random.default_rng(seed)
        a = rng.integers(0, alpha, na).astype(np.int32)
        b = rng.integers(0, alpha, nb).astype(np.int32)
        key = f"s{idx:02d}"
        arrays[key + "_a"] = a
        arrays[key + "_b"] = b
        lcs_cases.append({"key": key, "na": na, "nb": nb, "alphabet": alpha, "seed": seed,
                          "length": int(ref.baselines.lcs_reference(a, b))})
    np.savez_compressed(os.path.join(HERE, "reference_int.npz"), **arrays)
    with open(os.path.join(HERE, "reference_int.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden_int.py", "reference": "tvstencil 0.1.0 @ /root/reference",
                   "numpy": np.__version__, "life": life_cases, "lcs": lcs_cases}, fh, indent=1)
    print(f"wrote {len(life_cases)} life + {len(lcs_cases)} lcs cases")


if __name__ == "__main__":
    main()
