"""Generate tests/golden/*.npz from the REAL reference package.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports /root/reference/pkg/src/tvstencil under the alias
``tvstencil_ref`` and records, for seeded inputs, the reference's own
``scalar_reference`` output (tvstencil/baselines.py:110-125) — the oracle
of every parity test.  The GPU box never needs /root/reference: the tests
read only these committed fixtures.
"""

from __future__ import annotations

import importlib.util
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "tvstencil_ref", os.path.join(REF_SRC, "tvstencil", "__init__.py"),
        submodule_search_locations=[os.path.join(REF_SRC, "tvstencil")])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["tvstencil_ref"] = mod
    spec.loader.exec_module(mod)
    import importlib as il
    il.import_module("tvstencil_ref.baselines")
    il.import_module("tvstencil_ref.catalog")
    return mod


def config_specs(ref):
    """BASELINE stencils the reference catalog lacks, as reference specs
    (same coefficients as paper_2010_04868_b200.catalog)."""
    import itertools

    SS = ref.model.StencilSpec
    box2 = sorted(itertools.product((-1, 0, 1), repeat=2))
    box3 = sorted(itertools.product((-1, 0, 1), repeat=3))
    w4 = np.random.default_rng(4).uniform(0, 1, 9)
    w4 = w4 / w4.sum()
    w6 = np.random.default_rng(6).uniform(0, 1, 27)
    w6 = w6 / w6.sum()
    return {
        "gs1d_w343": SS("gs1d_w343", 1, 1, "star", "gauss_seidel", coefficients={(-1,): 0.3, (0,): 0.4, (1,): 0.3}),
        "gs2d9p": SS("gs2d9p", 2, 1, "box", "gauss_seidel",
                     coefficients={o: float(w) for o, w in zip(box2, w4)}),
        "jac3d27p": SS("jac3d27p", 3, 1, "box", "jacobi",
                       coefficients={o: float(w) for o, w in zip(box3, w6)}),
    }


# (kernel, extents, steps, seed, boundary)
CASES = [
    ("heat1d", (256,), 8, 42, 0.0),
    ("heat1d", (1000,), 13, 7, 0.0),
    ("heat1d", (1025,), 70, 11, 0.0),
    ("heat1d", (33,), 1, 3, 0.0),
    ("heat1d", (4099,), 129, 5, 0.75),
    ("gs1d", (512,), 8, 8, 0.0),
    ("gs1d", (777,), 37, 9, -0.5),
    ("gs1d_w343", (1024,), 131, 1, 0.0),
    ("gs1d_w343", (130,), 300, 2, 0.0),
    ("heat2d", (32, 20), 4, 1, 0.0),
    ("heat2d", (48, 33), 9, 2, 0.0),
    ("heat2d", (130, 257), 17, 3, 0.25),
    ("jac2d9p", (56, 41), 7, 11, 0.0),
    ("jac2d9p", (67, 129), 12, 12, 1.0),
    ("heat3d", (24, 17, 23), 4, 15, 0.0),
    ("heat3d", (40, 24, 35), 9, 16, 0.5),
    ("jac3d27p", (20, 18, 37), 5, 5, 0.0),
    ("jac3d27p", (33, 9, 40), 3, 6, 0.25),
    ("gs2d", (32, 21), 4, 17, 0.0),
    ("gs2d", (64, 48), 10, 18, 0.0),
    ("gs3d", (24, 18, 15), 4, 20, 0.0),
    ("gs3d", (12, 20, 24), 6, 21, 0.5),
    ("gs2d9p", (40, 37), 5, 3, 0.0),
    ("gs2d9p", (17, 64), 9, 4, 0.0),
]


def main():
    ref = load_reference()
    extra = config_specs(ref)
    manifest = []
    arrays = {}
    for idx, (kernel, ext, steps, seed, bnd) in enumerate(CASES):
        spec = extra[kernel] if kernel in extra else ref.catalog.get(kernel).spec
        if bnd != 0.0:
            import dataclasses

            spec = dataclasses.replace(spec, boundary=bnd)
        grid = ref.grid.Grid.random(ext, seed=seed, boundary=bnd)
        out = ref.baselines.scalar_reference(spec, grid, steps)
        key = f"c{idx:02d}"
        arrays[key + "_in"] = np.ascontiguousarray(grid.interior)
        arrays[key + "_out"] = np.ascontiguousarray(out.interior)
        manifest.append({"key": key, "kernel": kernel, "extents": list(ext), "steps": steps, "seed": seed,
                         "boundary": bnd, "fnv_out": f"{ref.grid.fnv1a64(out.dump_bytes()):016x}"})
    # known answers straight from the reference's own tests
    ka = {}
    g = ref.grid.Grid.from_array(np.arange(1.0, 9.0), halo=1)
    ka["heat1d_1to8"] = ref.baselines.scalar_reference(ref.catalog.get("heat1d").spec, g, 1).interior.tolist()
    g = ref.grid.Grid.from_array(np.ones(3), halo=1)
    ka["gs1d_ones3"] = ref.baselines.scalar_reference(ref.catalog.get("gs1d").spec, g, 1).interior.tolist()
    ka["fnv"] = {"": f"{ref.grid.fnv1a64(b''):016x}", "a": f"{ref.grid.fnv1a64(b'a'):016x}",
                 "foobar": f"{ref.grid.fnv1a64(b'foobar'):016x}"}
    np.savez_compressed(os.path.join(HERE, "reference_cases.npz"), **arrays)
    with open(os.path.join(HERE, "reference_cases.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "tvstencil 0.1.0 @ /root/reference",
                   "numpy": np.__version__, "cases": manifest, "known_answers": ka}, fh, indent=1)
    print(f"wrote {len(manifest)} cases")


if __name__ == "__main__":
    main()
