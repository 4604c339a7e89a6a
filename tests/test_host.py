"""Host-side logic of the drop-in surface (no GPU): Grid, catalog, model,
schedule facts, validation/error parity with the reference."""

from __future__ import annotations

import itertools
import os
import struct
import tempfile

import numpy as np
import pytest

from paper_2010_04868_b200 import (
    Grid,
    SizeError,
    StencilSpec,
    UnsupportedError,
    dependences,
    gs_hyperplane,
    gs_new_taps,
    min_space_stride,
)
from paper_2010_04868_b200.catalog import DEFAULT_CATALOG, get, load_catalog
from paper_2010_04868_b200.kernels import (
    KernelVariant,
    gs1d_temporal,
    gs2d_temporal,
    heat1d_temporal,
    jacobi2d_temporal,
    jacobi3d_temporal,
)
from paper_2010_04868_b200.model import ScheduleParams
from paper_2010_04868_b200.verify import Cell, default_matrix, equivalence_matrix


def test_grid_geometry_matches_reference_layout():
    g = Grid((37,), 1)
    assert g.offset == 4 and g.data.shape == (37 + 4 + 1 + 4,)  # grid.py:35-37
    g = Grid((5, 7), 1, vl=8)
    assert g.offset == 8 and g.data.shape == (5 + 8 + 1 + 8, 7 + 8 + 1 + 8)
    g = Grid((8, 8), 1, boundary=7.5)
    assert g.data[0, 0] == 7.5
    g.interior[...] = 1.0
    g.fill_halo()
    assert g.data[g.offset - 1, g.offset] == 7.5 and np.all(g.interior == 1.0)


def test_grid_dump_load_roundtrip():
    g = Grid.random((17, 9), seed=3)
    raw = g.dump_bytes()
    assert raw[:4] == b"TSTN"
    assert struct.unpack_from("<IBB", raw, 4) == (1, 2, 0)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "g.tstn")
        g.dump(p)
        back = Grid.load(p)
    assert back.extents == g.extents and np.array_equal(back.interior, g.interior)


def test_grid_copy_independent():
    g = Grid.from_array(np.arange(12.0).reshape(3, 4))
    h = g.copy()
    h.interior[0, 0] = -1
    assert g.interior[0, 0] == 0.0


def test_catalog_reference_entries_and_configs():
    for name in ("heat1d", "heat2d", "jac2d9p", "heat3d", "life", "gs1d", "gs2d", "gs3d"):
        assert name in DEFAULT_CATALOG
    assert get("heat1d").spec.coefficients == {(-1,): 0.25, (0,): 0.5, (1,): 0.25}
    w = get("gs2d9p").spec
    assert len(w.offsets()) == 9 and abs(sum(w.coefficients.values()) - 1.0) < 1e-15
    raw = np.random.default_rng(4).uniform(0, 1, 9)
    assert [w.coefficients[o] for o in w.offsets()] == list(raw / raw.sum())
    j = get("jac3d27p").spec
    raw = np.random.default_rng(6).uniform(0, 1, 27)
    assert [j.coefficients[o] for o in j.offsets()] == list(raw / raw.sum())
    assert get("gs1d_w343").spec.coefficients == {(-1,): 0.3, (0,): 0.4, (1,): 0.3}
    with pytest.raises(KeyError):
        get("nope")


def test_load_catalog_json(tmp_path):
    p = tmp_path / "cat.json"
    p.write_text('{"kernels": {"h2": {"dim": 1, "coefficients": {"-1": 0.5, "1": 0.5}, "s": 3}}}')
    table = load_catalog(p)
    assert table["h2"].spec.coefficients == {(-1,): 0.5, (1,): 0.5} and table["h2"].s == 3


def test_dependences_and_min_stride():
    assert min_space_stride(dependences(get("heat1d").spec)) == 2
    assert min_space_stride(dependences(get("gs1d").spec)) == 2  # test_model.py:45-48
    assert min_space_stride(dependences(get("gs2d9p").spec)) == 2
    assert min_space_stride(dependences(get("jac3d27p").spec)) == 2


def _box(dim):
    return {o: 1.0 for o in itertools.product((-1, 0, 1), repeat=dim)}


@pytest.mark.parametrize("dim", [1, 2, 3])
@pytest.mark.parametrize("shape", ["star", "box"])
@pytest.mark.parametrize("order", ["lexicographic", "reference"])
def test_hyperplane_schedule_is_legal(dim, shape, order):
    """Replay check of the GPU wavefront: every tap of every point reads the
    version the sequential sweep would read (new taps: already written this
    sweep; old taps: not yet overwritten), for the (a, tau) the CUDA kernel
    uses.  Brute force over a small box and 3 sweeps."""
    coeffs = _box(dim)
    if shape == "star":
        coeffs = {o: 1.0 for o in coeffs if sum(1 for c in o if c) <= 1}
    spec = StencilSpec("t", dim, 1, shape, "gauss_seidel", coefficients=coeffs)
    a, tau, simul = gs_hyperplane(spec, order)
    new = gs_new_taps(spec, order)
    ext = (5,) * dim
    h = lambda t, x: sum(ai * xi for ai, xi in zip(a, x)) + tau * t
    for t in range(3):
        for x in itertools.product(*[range(e) for e in ext]):
            for off, is_new in zip(spec.offsets(), new):
                y = tuple(xi + oi for xi, oi in zip(x, off))
                if not any(off) or any(c < 0 or c >= 5 for c in y):
                    continue
                write_t = h(t, y) if is_new else h(t - 1, y)  # version we must read
                next_write = h(t + 1, y) if is_new else h(t, y)  # when it gets overwritten
                assert write_t < h(t, x), (off, x)
                assert h(t, x) < next_write or (simul and h(t, x) == next_write), (off, x)
    if shape == "box" and order == "reference" and dim > 1:
        assert simul
    if order == "lexicographic":
        assert not simul


def test_drop_in_errors_match_reference():
    """Error contract (kernels1d.py:79-85, 99-100; kernels_nd.py:62-72):
    raised before any device work, so they run on CPU."""
    with pytest.raises(SizeError):
        heat1d_temporal(Grid((16,), 1), 4)
    with pytest.raises(UnsupportedError):
        heat1d_temporal(Grid((256,), 1), 4, KernelVariant("base", params=ScheduleParams(7, 2, 4)))
    with pytest.raises(UnsupportedError):
        gs1d_temporal(Grid((512,), 1), 4, KernelVariant("base", False))
    with pytest.raises(UnsupportedError):
        jacobi2d_temporal(Grid.random((32, 32), seed=0), 4, KernelVariant("two_stride"))
    with pytest.raises(SizeError):
        jacobi2d_temporal(Grid.random((32,), seed=0), 4)
    with pytest.raises(SizeError):
        jacobi3d_temporal(Grid.random((8, 8), seed=0), 4)
    with pytest.raises(UnsupportedError):
        gs2d_temporal(Grid.random((32, 32), seed=0), 4, KernelVariant("base", False))
    with pytest.raises(ValueError):
        KernelVariant("bogus")
    with pytest.raises(KeyError):
        jacobi2d_temporal(Grid.random((32, 32), seed=0), 4, kernel="nope")

    class CountingBackend:  # the reference's instrumented backend cannot see GPU work
        counters = None

    with pytest.raises(UnsupportedError):
        heat1d_temporal(Grid((256,), 1), 4, None, CountingBackend())


def test_zero_steps_returns_copy_without_device():
    g = Grid.random((300,), seed=1)
    out = heat1d_temporal(g, 0)
    assert out is not g and np.array_equal(out.data, g.data)


def test_equivalence_matrix_harness_fault_injection():
    """verify.py:130-166 semantics with an injected runner and reference."""
    from oracle import oracle as npo

    def runner(kernel, grid, steps, variant=None, backend=None):
        return npo.scalar_reference(get(kernel).spec, grid, steps)

    def corrupted(kernel, grid, steps, variant=None, backend=None):
        out = runner(kernel, grid, steps)
        out.interior[1] += 1e-9
        return out

    cells = [Cell("heat1d", "base", False, (256,), 3, 8), Cell("heat2d", "base", False, (32, 24), 5, 4)]
    rep = equivalence_matrix(cells, npo.scalar_reference, runner=runner)
    assert rep.passed and len(rep.results) == 2
    rep = equivalence_matrix(cells[:1], npo.scalar_reference, runner=corrupted)
    assert not rep.passed and rep.first_divergence == 0
    f = rep.as_dict()["failures"][0]
    assert f["position"] == [1] and f["got_bits"] != f["want_bits"] and f["got_bits"].startswith("0x")
    assert equivalence_matrix([], npo.scalar_reference).passed


def test_default_matrix_classes():
    cells = default_matrix(cells_per_kernel=20)
    kernels = {c.kernel for c in cells}
    assert "life" not in kernels and {"heat1d", "gs2d9p", "jac3d27p"} <= kernels
    for k in kernels:
        sub = [c for c in cells if c.kernel == k]
        e = get(k)
        assert {0, 1, 2, 3} <= {c.steps % e.vl for c in sub}
        assert {0, 1, e.vl - 1} & {c.size[0] % (4 * e.s * e.vl) for c in sub}


def test_cli_parser_and_config(tmp_path):
    from paper_2010_04868_b200.cli import CSV_HEADER, _apply_config, build_parser

    assert CSV_HEADER == "kernel,variant,dim,nx,ny,nz,t,threads,tile,reps,gstencils_per_s,checksum"  # cli.py:39
    cfg = tmp_path / "c.json"
    cfg.write_text('{"t": 7, "nx": 300, "reps": 2}')
    argv = ["--mode", "bench", "--kernel", "heat1d", "--nx", "500", "--config", str(cfg)]
    args = _apply_config(build_parser().parse_args(argv), argv)
    assert args.steps == 7 and args.nx == 500 and args.reps == 2  # explicit flags win


def test_bench_make_rows_exact():
    """bench.make_rows: a rank's slab of the seeded BASELINE grid equals the
    same rows of the full grid (PCG64 advanced past earlier rows), and the
    slab layout puts that row at the right place of the whole-grid layout."""
    import bench

    cfg = dict(bench.CONFIGS[3])
    cfg["extents"] = (37, 29)
    g = bench.make_grid(cfg)
    part, padded, off = bench.make_rows(cfg, 9, 21, pinned=False)
    assert padded == g.data.shape
    assert np.array_equal(part, g.data[off + 9: off + 21])
    lay, ptr = bench._slab_layout(cfg, part, 9, padded, off)
    row_bytes = padded[1] * 8
    assert ptr.value + (off + 9) * row_bytes == part.ctypes.data
    assert tuple(lay.shape[:2]) == padded and lay.offset == off
