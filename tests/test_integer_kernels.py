"""Integer kernels: Life-like rules
(baselines.py:52-66) and LCS (kernels/lcs.py:32, baselines.py:128-150).

CPU: the NumPy oracle and the int32 Grid generator pinned to the REAL
reference's outputs (tests/golden/make_golden_int.py).  GPU: the CUDA
kernels through the drop-in functions / C ABI against the same goldens and
the oracle, bit-exact (integer results)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import int_grid, life_spec
from oracle import oracle as npo
from paper_2010_04868_b200 import Grid
from paper_2010_04868_b200.catalog import get


def test_int_grid_random_reproduces_reference_inputs(golden_int):
    meta, arrays = golden_int
    for c in meta["life"]:
        g = Grid.random(tuple(c["extents"]), seed=c["seed"], boundary=c["boundary"], element_kind="int32")
        assert np.array_equal(g.interior, arrays[c["key"] + "_in"]), c["key"]


def test_oracle_life_matches_reference(golden_int):
    meta, arrays = golden_int
    for c in meta["life"]:
        got = npo.scalar_reference(life_spec(c), int_grid(arrays[c["key"] + "_in"], c["boundary"]), c["steps"])
        assert np.array_equal(got.interior, arrays[c["key"] + "_out"]), c


def test_oracle_lcs_matches_reference(golden_int):
    meta, arrays = golden_int
    for c in meta["lcs"]:
        assert npo.lcs_length(arrays[c["key"] + "_a"], arrays[c["key"] + "_b"]) == c["length"], c


# ---------------------------------------------------------------- GPU ----

@pytest.mark.gpu
def test_life_golden_gpu(cuda_ready, golden_int):
    from paper_2010_04868_b200.kernels._common import execute

    meta, arrays = golden_int
    for c in meta["life"]:
        g = int_grid(arrays[c["key"] + "_in"], c["boundary"])
        got = execute(life_spec(c), g, c["steps"])
        assert np.array_equal(got.interior, arrays[c["key"] + "_out"]), c
        assert np.array_equal(g.interior, arrays[c["key"] + "_in"])  # input untouched
        assert (got.data[0] == c["boundary"]).all()


@pytest.mark.gpu
def test_life_drop_in_dispatch(cuda_ready):
    """run_temporal("life") -> jacobi2d_temporal(kernel="life") as in the
    reference dispatcher (verify.py:60)."""
    from paper_2010_04868_b200.verify import run_temporal

    g = Grid.random((300, 257), seed=4, element_kind="int32")
    want = npo.scalar_reference(get("life").spec, g, 40)
    assert np.array_equal(run_temporal("life", g, 40).interior, want.interior)


@pytest.mark.gpu
@pytest.mark.parametrize("ext", [(1,), (2047,), (2048,), (70001,), (63, 65), (64, 31), (129, 1000), (9, 10, 11),
                                 (3, 65, 40)])
def test_life_tiles_and_wrapping_sums(cuda_ready, ext):
    """Tile edges of the 8-outputs-per-thread layout, and arbitrary int32
    cell values (the neighbour sum wraps mod 2^32 exactly like NumPy)."""
    import dataclasses

    from paper_2010_04868_b200.kernels._common import execute

    rng = np.random.default_rng(len(ext) * 1000 + ext[0])
    spec = dataclasses.replace(get("life").spec, dim=len(ext), boundary=-3, birth=frozenset({0, 3}),
                               survive=frozenset({2, 3, 8}))
    g = Grid(ext, 1, boundary=-3, element_kind="int32")
    vals = rng.integers(0, 2, ext, dtype=np.int32)
    vals[rng.random(ext) < 0.05] = np.int32(2 ** 31 - 1)
    vals[rng.random(ext) < 0.05] = np.int32(-(2 ** 31))
    g.set_interior(vals)
    want = npo.scalar_reference(spec, g, 6)
    assert np.array_equal(execute(spec, g, 6).interior, want.interior)


@pytest.mark.gpu
@pytest.mark.parametrize("ext", [(300, 257), (1000, 130), (70, 2000), (257, 300)])
def test_life_temporal_blocking_depths(cuda_ready, ext):
    """K7b (D levels per pass) for D = 1, 2, 4, 8 and step counts that are
    not multiples of D, against the oracle; a non-zero boundary and a
    non-Conway rule."""
    import dataclasses

    from paper_2010_04868_b200 import config
    from paper_2010_04868_b200.kernels._common import execute

    spec = dataclasses.replace(get("life").spec, boundary=1, birth=frozenset({3, 6}), survive=frozenset({2, 3}))
    g = Grid(ext, 1, boundary=1, element_kind="int32")
    g.set_interior(np.random.default_rng(ext[0]).integers(0, 2, ext, dtype=np.int32))
    want = npo.scalar_reference(spec, g, 23)
    for depth in (1, 2, 4, 8):
        with config.using(depth=depth):
            assert np.array_equal(execute(spec, g, 23).interior, want.interior), depth


@pytest.mark.gpu
def test_lcs_golden_gpu(cuda_ready, golden_int):
    from paper_2010_04868_b200.kernels import lcs_temporal

    meta, arrays = golden_int
    for c in meta["lcs"]:
        assert lcs_temporal(arrays[c["key"] + "_a"], arrays[c["key"] + "_b"]) == c["length"], c


@pytest.mark.gpu
@pytest.mark.parametrize("na,nb,alpha", [(5000, 4000, 4), (777, 12345, 2), (12000, 31, 3), (140000, 40, 4)])
def test_lcs_sizes_gpu(cuda_ready, na, nb, alpha):
    """Many warps in the chain, short and long rows, and (140000 rows) more
    than one pass of kLcsMaxWarps warps."""
    from paper_2010_04868_b200.kernels import lcs_temporal

    rng = np.random.default_rng(na + nb)
    a = rng.integers(0, alpha, na).astype(np.int32)
    b = rng.integers(0, alpha, nb).astype(np.int32)
    assert lcs_temporal(a, b) == npo.lcs_length(a, b)
    assert lcs_temporal(a, a[: nb]) == min(na, nb) if nb <= na else True


@pytest.mark.gpu
def test_integer_acceptance_matrix_gpu(cuda_ready):
    """The reference's acceptance matrix for its integer kernels
    (verify.py:130-222: 20 life cells, 20 lcs cells incl. one 2000x2000)."""
    from paper_2010_04868_b200.verify import default_matrix, equivalence_matrix

    cells = default_matrix(cells_per_kernel=20, master_seed=2024, kernels=["life", "lcs"])
    rep = equivalence_matrix(cells, npo.scalar_reference, lcs_reference=npo.lcs_length)
    assert len(rep.results) == 40 and rep.passed, rep.to_json()


def test_reference_known_lcs_and_life_properties_cpu():
    """Oracle-side known answers the reference tests use (test_lcs.py:11-26,
    test_kernels_nd.py:57-78): identical strings, disjoint alphabets, empty
    inputs; a 2x2 block is a still life under B3/S23; an empty board stays
    empty."""
    import dataclasses

    x = np.arange(50, dtype=np.int32) % 7
    assert npo.lcs_length(x, x) == 50
    assert npo.lcs_length(np.zeros(9, np.int32), np.ones(5, np.int32)) == 0
    assert npo.lcs_length(np.zeros(0, np.int32), x) == 0
    conway = dataclasses.replace(get("life").spec, birth=frozenset({3}), survive=frozenset({2, 3}))
    g = Grid((10, 10), 1, element_kind="int32")
    blk = np.zeros((10, 10), np.int32)
    blk[4:6, 4:6] = 1
    g.set_interior(blk)
    assert np.array_equal(npo.scalar_reference(conway, g, 5).interior, blk)


@pytest.mark.gpu
def test_reference_known_lcs_and_life_properties_gpu(cuda_ready):
    """The same known answers through the GPU drop-ins."""
    import dataclasses

    from paper_2010_04868_b200.kernels import lcs_temporal
    from paper_2010_04868_b200.kernels._common import execute

    x = np.arange(5000, dtype=np.int32) % 7
    assert lcs_temporal(x, x) == 5000
    assert lcs_temporal(np.zeros(900, np.int32), np.ones(700, np.int32)) == 0
    assert lcs_temporal([], x) == 0 and lcs_temporal(x, []) == 0
    for n in range(1, 10):  # short sequences (the reference's scalar path)
        a, b = np.arange(n, dtype=np.int32) % 3, np.arange(n + 2, dtype=np.int32) % 2
        assert lcs_temporal(a, b) == npo.lcs_length(a, b)
    conway = dataclasses.replace(get("life").spec, birth=frozenset({3}), survive=frozenset({2, 3}))
    g = Grid((300, 200), 1, element_kind="int32")
    blk = np.zeros((300, 200), np.int32)
    blk[100:102, 50:52] = 1
    g.set_interior(blk)
    assert np.array_equal(execute(conway, g, 17).interior, blk)
    empty = Grid((300, 200), 1, element_kind="int32")
    assert not execute(get("life").spec, empty, 9).interior.any()
