"""Shared fixtures.  `-m gpu` tests need a B200 and the built library; the
rest run on CPU (oracle vs golden vectors, host logic, ABI surface)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and libtvstencil.so")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


def load_golden():
    with open(os.path.join(GOLDEN, "reference_cases.json")) as fh:
        meta = json.load(fh)
    arrays = np.load(os.path.join(GOLDEN, "reference_cases.npz"))
    return meta, arrays


def load_golden_int():
    with open(os.path.join(GOLDEN, "reference_int.json")) as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(GOLDEN, "reference_int.npz"))


def life_spec(case):
    """Life-like StencilSpec of a reference_int.json case."""
    import dataclasses

    from paper_2010_04868_b200.catalog import get

    return dataclasses.replace(get("life").spec, name=case["name"], dim=case["dim"], boundary=case["boundary"],
                               birth=frozenset(case["birth"]), survive=frozenset(case["survive"]))


def int_grid(interior, boundary=0):
    from paper_2010_04868_b200 import Grid

    g = Grid(interior.shape, 1, boundary=boundary, element_kind="int32")
    g.set_interior(interior)
    return g


@pytest.fixture(scope="session")
def golden_int():
    return load_golden_int()


@pytest.fixture(scope="session")
def golden():
    return load_golden()


def spec_for(kernel: str, boundary: float = 0.0):
    import dataclasses

    from paper_2010_04868_b200.catalog import get

    spec = get(kernel).spec
    if boundary != spec.boundary:
        spec = dataclasses.replace(spec, boundary=boundary)
    return spec


def grid_from(interior, boundary=0.0):
    from paper_2010_04868_b200 import Grid

    g = Grid(interior.shape, 1, boundary=boundary)
    g.set_interior(interior)
    return g


@pytest.fixture(scope="session")
def cuda_ready():
    """Skip-free guard for gpu tests: fail loudly if the library or device is missing."""
    from paper_2010_04868_b200 import _native

    _native.lib()
    n = _native.device_count()
    assert n > 0, "gpu test without a CUDA device"
    return n
