"""The reference's own acceptance matrix, cell for cell.

tests/golden/acceptance_cells.json (made by tests/golden/make_acceptance.py
from the real reference) lists the 180 cells of
``verify.default_matrix(cells_per_kernel=20)`` (verify.py:169-222, run by
test_acceptance.py:32-41) with the FNV-1a-64 checksum of the reference's own
``scalar_reference`` result (TSTN dump, grid.py:96-133) or LCS length.  The
GPU path (``run_temporal`` / ``lcs_temporal``) must reproduce every checksum:
bit-exact on every cell, halo and pads included.  The CPU test pins the
oracle to the same checksums."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as npo
from paper_2010_04868_b200 import Grid
from paper_2010_04868_b200.catalog import get
from paper_2010_04868_b200.grid import fnv1a64


def _cells():
    with open(os.path.join(GOLDEN, "acceptance_cells.json")) as fh:
        return json.load(fh)["cells"]


def _lcs_inputs(c):
    rng = np.random.default_rng(c["seed"])
    a = rng.integers(0, 4, size=c["size"][0], dtype=np.int32)
    b = rng.integers(0, 4, size=c["size"][1], dtype=np.int32)
    return a, b


def _grid(c):
    entry = get(c["kernel"])
    return Grid.random(tuple(c["size"]), seed=c["seed"], element_kind=entry.spec.element_kind, vl=c["vl"])


def test_oracle_reproduces_reference_acceptance_checksums():
    cells = _cells()
    assert len(cells) == 180
    for c in cells:
        if c["kernel"] == "lcs":
            a, b = _lcs_inputs(c)
            if a.size * b.size <= 400 * 400:  # the NumPy DP is quadratic; the GPU test covers all
                assert npo.lcs_length(a, b) == c["lcs"], c
            continue
        got = npo.scalar_reference(get(c["kernel"]).spec, _grid(c), c["steps"])
        assert f"{fnv1a64(got.dump_bytes()):016x}" == c["fnv1a64"], c


@pytest.mark.gpu
def test_gpu_reproduces_reference_acceptance_matrix(cuda_ready):
    from paper_2010_04868_b200.kernels import KernelVariant, lcs_temporal
    from paper_2010_04868_b200.verify import run_temporal

    bad = []
    for c in _cells():
        if c["kernel"] == "lcs":
            a, b = _lcs_inputs(c)
            if lcs_temporal(a, b) != c["lcs"]:
                bad.append(c)
            continue
        g = _grid(c)
        got = run_temporal(c["kernel"], g, c["steps"], KernelVariant(c["scheme"], c["single_array"]))
        if f"{fnv1a64(got.dump_bytes()):016x}" != c["fnv1a64"]:
            bad.append(c)
    assert not bad, f"{len(bad)} of 180 cells differ, first {bad[0]}"
