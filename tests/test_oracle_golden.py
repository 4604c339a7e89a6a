"""The oracle (NumPy + C restatements) pinned against the REAL reference's
outputs (tests/golden, made by tests/golden/make_golden.py) and its
known-answer tests.  CPU only."""

from __future__ import annotations

import dataclasses
import itertools

import numpy as np
import pytest

from conftest import grid_from, spec_for
from oracle import cref
from oracle import oracle as npo
from paper_2010_04868_b200 import Grid, StencilSpec, fnv1a64
from paper_2010_04868_b200.catalog import get


def _cases(golden):
    meta, arrays = golden
    for c in meta["cases"]:
        yield c, arrays[c["key"] + "_in"], arrays[c["key"] + "_out"]


def test_grid_random_reproduces_reference_inputs(golden):
    for c, inp, _ in _cases(golden):
        g = Grid.random(tuple(c["extents"]), seed=c["seed"], boundary=c["boundary"])
        assert np.array_equal(g.interior, inp), c["key"]


def test_numpy_oracle_matches_reference(golden):
    for c, inp, out in _cases(golden):
        spec = spec_for(c["kernel"], c["boundary"])
        got = npo.scalar_reference(spec, grid_from(inp, c["boundary"]), c["steps"], order="reference")
        assert np.array_equal(got.interior, out), c


def test_c_oracle_matches_reference(golden):
    for c, inp, out in _cases(golden):
        spec = spec_for(c["kernel"], c["boundary"])
        got = cref.scalar_reference(spec, grid_from(inp, c["boundary"]), c["steps"], order="reference")
        assert np.array_equal(got.interior, out), c


def test_checksums_match_reference(golden):
    for c, inp, out in _cases(golden):
        g = grid_from(out, c["boundary"])
        assert f"{fnv1a64(g.dump_bytes()):016x}" == c["fnv_out"], c["key"]


def test_known_answers(golden):
    ka = golden[0]["known_answers"]
    g = Grid.from_array(np.arange(1.0, 9.0), halo=1)
    assert npo.scalar_reference(get("heat1d").spec, g, 1).interior.tolist() == ka["heat1d_1to8"]
    assert ka["heat1d_1to8"] == [1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0, 5.75]  # test_baselines.py:17-21
    g = Grid.from_array(np.ones(3), halo=1)
    assert npo.scalar_reference(get("gs1d").spec, g, 1).interior.tolist() == ka["gs1d_ones3"]
    assert ka["gs1d_ones3"] == [0.75, 0.9375, 0.734375]  # test_baselines.py:32-36
    assert cref.scalar_reference(get("gs1d").spec, g, 1).interior.tolist() == ka["gs1d_ones3"]
    for text, want in ka["fnv"].items():
        assert f"{fnv1a64(text.encode()):016x}" == want


def test_fnv_large_buffer_native_path():
    data = np.random.default_rng(0).integers(0, 255, 10000, dtype=np.uint8).tobytes()
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    assert fnv1a64(data) == h


def test_zero_and_constant_fixed_points():
    for name in ("heat1d", "heat2d", "heat3d", "gs1d", "gs2d", "gs3d", "jac3d27p", "gs2d9p"):
        spec = get(name).spec
        g = Grid((12,) * spec.dim, 1)
        for order in ("reference", "lexicographic"):
            assert not npo.scalar_reference(spec, g, 3, order=order).interior.any(), name
            assert not cref.scalar_reference(spec, g, 3, order=order).interior.any(), name


@pytest.mark.parametrize("kernel", ["gs2d", "gs3d"])
def test_lexicographic_equals_reference_for_star(golden, kernel):
    """For star stencils the row-major loop and the reference's anti-diagonal
    order coincide (the reference's own claim, test_baselines.py:39-52) —
    this pins the lexicographic oracle against the reference."""
    for c, inp, out in _cases(golden):
        if c["kernel"] != kernel:
            continue
        spec = spec_for(kernel, c["boundary"])
        g = grid_from(inp, c["boundary"])
        assert np.array_equal(npo.scalar_reference(spec, g, c["steps"], order="lexicographic").interior, out)
        assert np.array_equal(cref.scalar_reference(spec, g, c["steps"], order="lexicographic").interior, out)


def test_reference_loop_test_generalised():
    """test_baselines.py:39-52 restated: one lexicographic sweep by a plain
    loop equals scalar_reference for the 5-point star."""
    spec = get("gs2d").spec
    g = Grid.random((9, 11), seed=5)
    ref = g.copy()
    npo.gs_sweep_loop(spec, ref.data, ref.offset, ref.extents)
    assert np.array_equal(npo.scalar_reference(spec, g, 1).interior, ref.interior)


@pytest.mark.parametrize("kernel,ext,steps", [("gs2d9p", (23, 31), 4), ("gs2d9p", (8, 5), 3),
                                               ("gs3d", (7, 6, 9), 2)])
def test_lexicographic_three_restatements_agree(kernel, ext, steps):
    spec = get(kernel).spec
    g = Grid.random(ext, seed=17)
    loop = g.copy()
    for _ in range(steps):
        npo.gs_sweep_loop(spec, loop.data, loop.offset, loop.extents)
    a = npo.scalar_reference(spec, g, steps, order="lexicographic")
    b = cref.scalar_reference(spec, g, steps, order="lexicographic")
    assert np.array_equal(a.interior, loop.interior)
    assert np.array_equal(b.interior, loop.interior)


def test_box_orders_differ():
    """for the 9-point box the two orders give different
    results (NE read from the previous sweep in the reference order)."""
    spec = get("gs2d9p").spec
    g = Grid.random((16, 16), seed=3)
    a = npo.scalar_reference(spec, g, 2, order="lexicographic")
    b = npo.scalar_reference(spec, g, 2, order="reference")
    assert not np.array_equal(a.interior, b.interior)


def test_c_oracle_threads_deterministic():
    spec = get("jac3d27p").spec
    g = Grid.random((18, 20, 22), seed=4)
    outs = [cref.scalar_reference(spec, g, 3, threads=t).interior.copy() for t in (1, 2, 8)]
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


def test_fma_would_break_bitexactness():
    """Why the kernels default to unfused mul+add: a fused tap changes bits on
    signed data with non-power-of-two weights, but not with
    power-of-two weights (heat1d / heat2d), where the product is exact."""
    import ctypes

    libm = ctypes.CDLL("libm.so.6")
    libm.fma.restype = ctypes.c_double
    libm.fma.argtypes = [ctypes.c_double] * 3
    x = np.random.default_rng(1).uniform(-1, 1, 4096)
    for c0, c1, expect_equal in ((0.3, 0.4, False), (0.25, 0.5, True)):
        unfused = c1 * x[1:] + c0 * x[:-1]
        fused = np.array([libm.fma(c1, b, c0 * a) for a, b in zip(x[:-1], x[1:])])
        assert np.array_equal(unfused, fused) == expect_equal
