"""GPU parity: the CUDA path (through the drop-in functions / C ABI) against
the reference's own outputs (golden) and the oracle, bit-exact."""

from __future__ import annotations

import dataclasses
import os

import numpy as np
import pytest

from conftest import grid_from, spec_for
from oracle import cref
from oracle import oracle as npo
from paper_2010_04868_b200 import Grid, _native, config
from paper_2010_04868_b200.catalog import DEFAULT_CATALOG, get
from paper_2010_04868_b200.kernels import KernelVariant, gs1d_temporal, gs2d_temporal, heat1d_temporal
from paper_2010_04868_b200.kernels._common import execute
from paper_2010_04868_b200.verify import default_matrix, equivalence_matrix, run_temporal

pytestmark = pytest.mark.gpu


def _run(kernel, grid, steps, **kw):
    spec = spec_for(kernel, grid.boundary)
    return execute(spec, grid, steps, **kw)


def test_golden_cases_bitexact(cuda_ready, golden):
    """Every golden vector of the real reference, through the GPU path."""
    meta, arrays = golden
    for c in meta["cases"]:
        g = grid_from(arrays[c["key"] + "_in"], c["boundary"])
        got = _run(c["kernel"], g, c["steps"], order="reference")
        assert np.array_equal(got.interior, arrays[c["key"] + "_out"]), c
        # pads/halo of the result hold the boundary, input untouched
        assert np.array_equal(g.interior, arrays[c["key"] + "_in"])


def test_known_answers_gpu(cuda_ready):
    g = Grid.from_array(np.arange(1.0, 9.0), halo=1)
    # 8 points is below the reference's 1D minimum; run through execute()
    assert _run("heat1d", g, 1).interior.tolist() == [1, 2, 3, 4, 5, 6, 7, 5.75]
    g = Grid.from_array(np.ones(3), halo=1)
    assert _run("gs1d", g, 1).interior.tolist() == [0.75, 0.9375, 0.734375]


def test_equivalence_matrix_gpu(cuda_ready):
    """The reference's acceptance matrix (verify.py:169-222 with
    test_acceptance.py:35's 20 cells per kernel) over every float64 catalog
    kernel, GPU runner vs oracle.  GS in 2D/3D compares against the
    lexicographic oracle (the GPU default order)."""
    cells = default_matrix(cells_per_kernel=20, master_seed=2024)

    def reference(spec, grid, steps):
        return cref.scalar_reference(spec, grid, steps, order="lexicographic", threads=8)

    rep = equivalence_matrix(cells, reference)
    assert rep.passed, rep.to_json()


def test_equivalence_matrix_gpu_reference_order(cuda_ready):
    """The same 20-cell matrix for the Gauss-Seidel kernels in the reference
    oracle's own anti-diagonal order (baselines.py:83-107), GPU runner with
    order="reference" vs the NumPy restatement of scalar_reference."""
    gs = [k for k in ("gs2d", "gs2d9p", "gs3d") if k in DEFAULT_CATALOG]
    cells = default_matrix(cells_per_kernel=20, master_seed=2024, kernels=gs)

    def runner(kernel, grid, steps, variant):
        return run_temporal(kernel, grid, steps, variant, order="reference")

    rep = equivalence_matrix(cells, lambda spec, grid, steps: npo.scalar_reference(spec, grid, steps), runner)
    assert rep.passed, rep.to_json()


@pytest.mark.parametrize("kernel,ext,steps", [
    ("gs2d9p", (40, 37), 5), ("gs2d9p", (65, 130), 11), ("gs2d9p", (9, 300), 3),
    ("gs2d", (33, 64), 7), ("gs3d", (12, 20, 24), 6)])
@pytest.mark.parametrize("order", ["lexicographic", "reference"])
def test_gauss_seidel_orders(cuda_ready, kernel, ext, steps, order):
    g = Grid.random(ext, seed=len(ext) * 100 + steps)
    got = _run(kernel, g, steps, order=order)
    want = cref.scalar_reference(get(kernel).spec, g, steps, order=order)
    assert np.array_equal(got.interior, want.interior)


@pytest.mark.parametrize("n,steps", [(32, 1), (33, 7), (1024, 64), (1025, 65), (4096, 1000), (100000, 129),
                                     (896 * 3, 128), (2 ** 16 + 7, 200)])
def test_heat1d_sizes(cuda_ready, n, steps):
    g = Grid.random((n,), seed=n + steps)
    want = cref.scalar_reference(get("heat1d").spec, g, steps)
    for fma in ("never", "exact"):
        got = _run("heat1d", g, steps, fma=fma)
        assert np.array_equal(got.interior, want.interior), fma


@pytest.mark.parametrize("n,steps", [(32, 1), (35, 3), (127, 130), (128, 129), (129, 300), (5000, 257),
                                     (70000, 140)])
def test_gs1d_pipeline_sizes(cuda_ready, n, steps):
    for kernel in ("gs1d", "gs1d_w343"):
        g = Grid.random((n,), seed=n * 3 + steps, boundary=0.25 if n % 2 else 0.0)
        spec = spec_for(kernel, g.boundary)
        want = cref.scalar_reference(spec, g, steps)
        got = execute(spec, g, steps)
        assert np.array_equal(got.interior, want.interior), (kernel, n, steps)


@pytest.mark.parametrize("n,steps", [(1, 1), (2, 33), (95, 31), (96, 32), (97, 127), (128, 128), (129, 129),
                                     (383, 97), (384, 1), (385, 159), (511, 256), (512, 385), (513, 1000),
                                     (1000, 64 * 4 * 32 + 5), (4099, 100)])
def test_gs1d_chunk_and_writer_lane_edges(cuda_ready, n, steps):
    """Sizes around the 128-position chunk / 512-position ring and sweep counts
    that leave the last block with a partial warp (writer lane (T-1) % 32)."""
    g = Grid.random((n,), seed=7 * n + steps, boundary=0.5 if n % 3 else -1.25)
    spec = spec_for("gs1d_w343", g.boundary)
    want = cref.scalar_reference(spec, g, steps)
    got = execute(spec, g, steps)
    assert np.array_equal(got.interior, want.interior), (n, steps)


def test_gs1d_many_blocks_and_passes(cuda_ready):
    """> 64 blocks of 128 sweeps: exercises multi-launch passes and identity lanes."""
    g = Grid.random((300,), seed=9)
    steps = 64 * 128 + 77
    want = cref.scalar_reference(get("gs1d_w343").spec, g, steps)
    got = _run("gs1d_w343", g, steps)
    assert np.array_equal(got.interior, want.interior)


@pytest.mark.parametrize("kernel", ["heat2d", "jac2d9p"])
@pytest.mark.parametrize("ext", [(64, 64), (257, 130), (9, 1000), (1000, 9), (600, 611)])
def test_jacobi2d_depths(cuda_ready, kernel, ext):
    g = Grid.random(ext, seed=ext[0] + ext[1], boundary=0.5)
    spec = spec_for(kernel, 0.5)
    steps = 19
    want = cref.scalar_reference(spec, g, steps)
    for depth in (0, 1, 2, 3, 5, 8):
        got = execute(spec, g, steps, depth=depth, fma="never")
        assert np.array_equal(got.interior, want.interior), depth
    naive = execute(spec, g, steps, algo="naive", fma="never")
    assert np.array_equal(naive.interior, want.interior)


@pytest.mark.parametrize("kernel", ["heat3d", "jac3d27p"])
@pytest.mark.parametrize("ext", [(20, 18, 37), (65, 17, 33), (130, 40, 9), (3, 70, 70)])
def test_jacobi3d_streaming(cuda_ready, kernel, ext):
    g = Grid.random(ext, seed=sum(ext))
    spec = spec_for(kernel)
    want = cref.scalar_reference(spec, g, 5)
    for algo in ("auto", "naive"):
        got = execute(spec, g, 5, algo=algo, fma="never")
        assert np.array_equal(got.interior, want.interior), algo


@pytest.mark.parametrize("kernel", ["heat3d", "jac3d27p"])
@pytest.mark.parametrize("ext", [(1, 1, 1), (2, 30, 62), (70, 31, 63), (65, 61, 125), (131, 29, 200)])
def test_jacobi3d_two_level_blocking(cuda_ready, kernel, ext):
    """K4c / K4b (two time levels per pass) against the oracle and against K4
    (depth 1) across frame edges (62 x 30 useful per block, 64-plane
    segments), odd step counts (2-level launches + one single step) and both
    FMA contracts."""
    g = Grid.random(ext, seed=sum(ext), boundary=0.375)
    spec = spec_for(kernel, 0.375)
    want = cref.scalar_reference(spec, g, 7)
    for depth in (0, 1, 2, 3):
        got = execute(spec, g, 7, depth=depth, fma="never")
        assert np.array_equal(got.interior, want.interior), depth
    a = execute(spec, g, 6, depth=2, fma="allow")
    b = execute(spec, g, 6, depth=1, fma="allow")
    assert np.array_equal(a.interior, b.interior)


@pytest.mark.parametrize("n", [1, 7, 255, 256, 2047, 2048, 2049, 4096 + 300, 20000])
def test_naive_1d_tiles(cuda_ready, n):
    """Single-step kernel: full 2048-element tiles and ragged tails."""
    g = Grid.random((n,), seed=n, boundary=0.25)
    for kernel in ("heat1d", "gs1d_w343"):
        spec = dataclasses.replace(spec_for(kernel, 0.25), dependence_kind="jacobi")
        want = cref.scalar_reference(spec, g, 7)
        got = execute(spec, g, 7, algo="naive", fma="never")
        assert np.array_equal(got.interior, want.interior), kernel


@pytest.mark.parametrize("ext", [(64, 64, 64), (5, 67, 33), (3, 64, 31)])
def test_naive_generic_taps(cuda_ready, ext):
    """Single-step kernel with a tap count it does not specialise (runtime
    tap loop): a 3D 10-tap stencil and a 2D 4-tap stencil."""
    from paper_2010_04868_b200.model import StencilSpec

    rng = np.random.default_rng(11)
    offs3 = [(-1, 0, 0), (0, -1, 1), (0, 0, -1), (0, 0, 0), (0, 0, 1), (0, 1, -1), (1, -1, -1), (1, 0, 0),
             (1, 1, 0), (1, 1, 1)]
    spec3 = StencilSpec(name="t10", dim=3, radius=1, shape="box", dependence_kind="jacobi",
                        coefficients={o: float(w) for o, w in zip(offs3, rng.uniform(0, 0.2, len(offs3)))})
    g = Grid.random(ext, seed=3)
    want = cref.scalar_reference(spec3, g, 4)
    assert np.array_equal(execute(spec3, g, 4, algo="naive", fma="never").interior, want.interior)
    assert np.array_equal(execute(spec3, g, 4, fma="never").interior, want.interior)
    offs2 = [(-1, 1), (0, -1), (0, 0), (1, 1)]
    spec2 = StencilSpec(name="t4", dim=2, radius=1, shape="box", dependence_kind="jacobi",
                        coefficients={o: float(w) for o, w in zip(offs2, rng.uniform(0, 0.3, 4))})
    g2 = Grid.random(ext[1:], seed=4)
    want2 = cref.scalar_reference(spec2, g2, 5)
    assert np.array_equal(execute(spec2, g2, 5, algo="naive", fma="never").interior, want2.interior)


def test_fma_policies(cuda_ready):
    """exact: power-of-two weights fuse bit-identically; allow: tolerance."""
    g = Grid.random((300, 301), seed=2)
    want = cref.scalar_reference(get("heat2d").spec, g, 12)
    assert np.array_equal(_run("heat2d", g, 12, fma="exact").interior, want.interior)
    # config 5's distribution: uniform[0, 1) (signed data makes pointwise
    # relative error unbounded near zeros, which is why FMA is opt-in)
    g3 = Grid((40, 41, 42), 1)
    g3.set_interior(np.random.default_rng(5).uniform(0.0, 1.0, (40, 41, 42)))
    want3 = cref.scalar_reference(get("jac3d27p").spec, g3, 6)
    got3 = _run("jac3d27p", g3, 6, fma="allow")
    rel = np.abs(got3.interior - want3.interior) / np.maximum(np.abs(want3.interior), 1e-300)
    assert rel.max() <= 1e-12  # BASELINE tolerance
    assert np.array_equal(_run("jac3d27p", g3, 6, fma="exact").interior, want3.interior)


def test_ranged_passes_compose_to_full_pass(cuda_ready):
    """tvs_jacobi_device_rows (the overlapped halo path's interior / edge
    passes): ranged passes covering a slab's owned rows equal one full pass
    there, bit-exact, for 2D depths up to 12 and 3D depths 1-2, on a
    mid-domain slab (ghost rows on both sides)."""
    import ctypes as C

    import torch

    from paper_2010_04868_b200 import halo

    for kernel, ext, depths in (("heat2d", (300, 130), (1, 3, 8, 12)), ("jac2d9p", (200, 70), (2, 5)),
                                ("jac3d27p", (60, 20, 36), (1, 2)), ("heat3d", (50, 17, 40), (2,))):
        spec = get(kernel).spec
        st = _native.make_stencil(spec)
        g = Grid.random(ext, seed=3)
        for k in depths:
            lay = halo.make_layout(ext, 3, 1, max(k, 2))
            n, gh = lay.n_own, lay.ghost
            nel = int(lay.geometry.alloc_elems)
            src = torch.full((nel,), 0.0, dtype=torch.float64, device="cuda")
            view = src.as_strided(tuple(lay.extents), tuple(int(lay.geometry.strides[d]) for d in range(len(ext))),
                                  int(lay.geometry.origin))
            view.copy_(torch.from_numpy(g.interior[lay.r0 - gh: lay.r1 + gh].copy()))
            full = torch.zeros_like(src)
            part = torch.zeros_like(src)
            ex = _native.make_exec(temporal_depth=k)  # the full pass is one launch of k levels too
            stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
            in_dst = C.c_int32(0)
            _native.check(_native.lib().tvs_jacobi_device(C.byref(st), C.byref(lay.geometry), C.c_void_p(src.data_ptr()),
                                                          C.c_void_p(full.data_ptr()), k, C.byref(ex), stream,
                                                          C.byref(in_dst)))
            assert in_dst.value == 1
            for lo, hi in ((gh + k, gh + n - k), (gh, gh + k), (gh + n - k, gh + n)):
                _native.check(_native.lib().tvs_jacobi_device_rows(
                    C.byref(st), C.byref(lay.geometry), C.c_void_p(src.data_ptr()), C.c_void_p(part.data_ptr()), k,
                    C.byref(ex), stream, lo, hi))
            torch.cuda.synchronize()
            s0 = int(lay.geometry.strides[0])
            own = slice((gh + 1) * s0, (gh + n + 1) * s0)
            assert torch.equal(full[own], part[own]), (kernel, k)


def test_concurrent_drop_in_calls(cuda_ready):
    """The reference runs kernels from a ThreadPoolExecutor (tiling.py:365):
    the C ABI is re-entrant (per-thread device context, streams, scratch,
    error string), so concurrent calls of every family — including the
    pipelined 1D/2D/3D Jacobi, the stream-gated 2D Gauss-Seidel path, Life
    and LCS — each return their own oracle result."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as npo
    from paper_2010_04868_b200.kernels import lcs_temporal

    jobs = [("heat2d", (1100, 200), 21), ("jac3d27p", (140, 20, 24), 9), ("gs2d9p", (1100, 150), 17),
            ("heat1d", (1 << 20,), 70), ("gs1d_w343", (3000,), 40), ("life", (300, 260), 13)]

    def one(job):
        kernel, ext, steps = job
        spec = get(kernel).spec
        g = Grid.random(ext, seed=len(ext) + steps, element_kind=spec.element_kind)
        got = execute(spec, g, steps)
        want = (npo.scalar_reference(spec, g, steps) if spec.is_life
                else cref.scalar_reference(spec, g, steps, order="lexicographic", threads=2))
        return np.array_equal(got.interior, want.interior)

    def lcs_job(seed):
        rng = np.random.default_rng(seed)
        a, b = rng.integers(0, 4, 3000, dtype=np.int32), rng.integers(0, 4, 2500, dtype=np.int32)
        return lcs_temporal(a, b) == npo.lcs_length(a, b)

    with ThreadPoolExecutor(max_workers=8) as pool:
        futs = [pool.submit(one, j) for j in jobs * 2] + [pool.submit(lcs_job, s) for s in range(3)]
        results = [f.result() for f in futs]
    assert all(results), results


def test_drop_in_signatures_and_immutability(cuda_ready):
    g = Grid.random((512,), seed=8)
    before = g.data.copy()
    a = heat1d_temporal(g, 8, KernelVariant("two_stride", True))
    b = heat1d_temporal(g, 8, KernelVariant("base", False))
    assert np.array_equal(a.interior, b.interior)
    assert np.array_equal(g.data, before)
    assert np.all(a.data[: a.offset] == 0.0) and np.all(a.data[a.offset + 512:] == 0.0)
    gs = gs1d_temporal(g, 8, KernelVariant("base", True))
    assert np.array_equal(gs.interior, npo.scalar_reference(get("gs1d").spec, g, 8).interior)
    g2 = Grid.random((40, 50), seed=1)
    out = gs2d_temporal(g2, 3, kernel="gs2d9p", order="reference")
    assert np.array_equal(out.interior, npo.scalar_reference(get("gs2d9p").spec, g2, 3).interior)
    r = run_temporal("jac3d27p", Grid.random((20, 20, 20), seed=4), 2)
    assert r.extents == (20, 20, 20)


@pytest.mark.parametrize("kernel,ext,steps", [("heat1d", (300001,), 40), ("heat2d", (1100, 257), 19),
                                                ("gs2d9p", (600, 130), 7), ("heat3d", (70, 33, 40), 5)])
def test_pinned_grids_drop_in(cuda_ready, kernel, ext, steps):
    """Grids on tvs_host_alloc storage (page-locked) through every drop-in
    pipeline: same results as pageable Grids, pinned outputs, halo intact."""
    src = Grid.random(ext, seed=sum(ext) + steps)
    g = Grid(ext, 1, pinned=True)
    np.copyto(g.data, src.data)
    assert g.pinned and g.copy().pinned and g.alloc_like().pinned
    out = g.alloc_like()
    spec = get(kernel).spec
    execute(spec, g, steps, out=out)
    want = cref.scalar_reference(spec, src, steps, order="lexicographic", threads=8)
    assert np.array_equal(out.interior, want.interior)
    assert np.all(out.data[: out.offset] == 0.0)
    assert np.array_equal(g.data, src.data)
    e = _native.host_empty((3, 5), np.int32)
    e[...] = 7
    assert e.shape == (3, 5) and int(e.sum()) == 105


def test_plan_api_accumulates_steps(cuda_ready):
    for kernel, ext in (("heat2d", (200, 333)), ("gs1d_w343", (5000,)), ("gs2d9p", (50, 60)),
                        ("jac3d27p", (30, 20, 40))):
        spec = get(kernel).spec
        g = Grid.random(ext, seed=11)
        plan = _native.Plan(spec, ext, config.current().native())
        plan.upload(g.data, g.offset)
        plan.run(3)
        plan.run(5)
        plan.synchronize()
        out = g.alloc_like()
        plan.download(out.data, out.offset)
        plan.synchronize()
        assert plan.last_launches() >= 1 and plan.last_ms() >= 0.0
        want = cref.scalar_reference(spec, g, 8, order="lexicographic")
        assert np.array_equal(out.interior, want.interior), kernel
        plan.close()


@pytest.mark.parametrize("algo", ["auto", "naive"])
def test_slab_decomposition_emulated_ranks(cuda_ready, algo):
    """The sharded path's device side on one GPU: W emulated ranks, halos
    copied between their buffers (no cross-rank waiting), bit-identical to
    the single-domain result for W in 1..4 and several depths (blocked and
    single-step kernels)."""
    import torch

    from paper_2010_04868_b200 import halo

    for kernel, ext in (("heat2d", (97, 130)), ("jac3d27p", (41, 20, 36))):
        spec = get(kernel).spec
        g = Grid.random(ext, seed=5)
        steps = 13
        want = cref.scalar_reference(spec, g, steps)
        st = _native.make_stencil(spec)
        for world in (1, 2, 3, 4):
            for depth in (1, 4, 8):
                lays = [halo.make_layout(ext, world, r, depth) for r in range(world)]
                bufs = []
                for lay in lays:
                    n = int(lay.geometry.alloc_elems)
                    pair = [torch.full((n,), 0.0, dtype=torch.float64, device="cuda") for _ in range(2)]
                    view = pair[0].as_strided(tuple(lay.extents), tuple(int(lay.geometry.strides[d]) for d in range(len(ext))),
                                              int(lay.geometry.origin))
                    lo, hi = max(lay.r0 - depth, 0), min(lay.r1 + depth, ext[0])
                    view[lo - (lay.r0 - depth): hi - (lay.r0 - depth)] = torch.from_numpy(g.interior[lo:hi].copy()).cuda()
                    bufs.append([pair, 0])
                done = 0
                while done < steps:
                    k = min(depth, steps - done)
                    for r in range(world - 1):  # emulated exchange
                        a, b = lays[r], lays[r + 1]
                        ba, bb = bufs[r][0][bufs[r][1]], bufs[r + 1][0][bufs[r + 1][1]]
                        bb[b.row_slice(0, depth)] = ba[a.row_slice(a.n_own, depth)]
                        ba[a.row_slice(a.n_own + depth, depth)] = bb[b.row_slice(depth, depth)]
                    for r, lay in enumerate(lays):
                        pair, cur = bufs[r]
                        import ctypes as C

                        in_dst = C.c_int32(0)
                        ex = _native.make_exec(temporal_depth=depth, algo=_native.ALGO_NAIVE if algo == "naive" else _native.ALGO_AUTO)
                        _native.check(_native.lib().tvs_jacobi_device(
                            C.byref(st), C.byref(lay.geometry), C.c_void_p(pair[cur].data_ptr()),
                            C.c_void_p(pair[1 - cur].data_ptr()), k, C.byref(ex),
                            C.c_void_p(torch.cuda.current_stream().cuda_stream), C.byref(in_dst)))
                        if in_dst.value:
                            bufs[r][1] = 1 - cur
                    done += k
                torch.cuda.synchronize()
                parts = []
                for r, lay in enumerate(lays):
                    pair, cur = bufs[r]
                    view = pair[cur].as_strided(tuple(lay.extents),
                                                tuple(int(lay.geometry.strides[d]) for d in range(len(ext))),
                                                int(lay.geometry.origin))
                    parts.append(view[depth: depth + lay.n_own].cpu().numpy())
                got = np.concatenate(parts, 0)
                assert np.array_equal(got, want.interior), (kernel, world, depth)


def test_cli_bench_and_verify(cuda_ready, tmp_path):
    """The reference-CLI mirror: CSV row with the reference schema whose FNV
    checksum equals the oracle result's; verify mode passes."""
    from paper_2010_04868_b200 import cli
    from paper_2010_04868_b200.grid import fnv1a64

    csv = tmp_path / "rows.csv"
    assert cli.main(["--mode", "bench", "--kernel", "heat2d", "--nx", "200", "--ny", "150", "--t", "9",
                     "--reps", "2", "--csv", str(csv)]) == 0
    header, row = csv.read_text().strip().splitlines()
    assert header.startswith(cli.CSV_HEADER)
    fields = row.split(",")
    want = cref.scalar_reference(get("heat2d").spec, Grid.random((200, 150), seed=0), 9)
    assert fields[11] == f"{fnv1a64(want.dump_bytes()):016x}"
    assert cli.main(["--mode", "verify", "--kernel", "gs2d9p", "--cells", "3"]) == 0
    assert cli.main(["--mode", "verify", "--kernel", "life", "--cells", "4"]) == 0
    assert cli.main(["--mode", "verify", "--kernel", "lcs", "--cells", "3"]) == 0


def test_cli_tiles_threads_life_lcs(cuda_ready, tmp_path):
    """--tile / --threads route through the tile-schedule executor with the
    same checksum as the unblocked run; life and lcs rows as the reference
    CLI writes them (cli.py:156-240)."""
    from oracle import oracle as npo
    from paper_2010_04868_b200 import cli
    from paper_2010_04868_b200.grid import fnv1a64

    csv = tmp_path / "rows.csv"
    assert cli.main(["--mode", "bench", "--kernel", "heat2d", "--nx", "96", "--ny", "80", "--t", "12",
                     "--tile", "64x32:8", "--threads", "1..2", "--reps", "1", "--csv", str(csv)]) == 0
    assert cli.main(["--mode", "bench", "--kernel", "life", "--nx", "96", "--ny", "80", "--t", "12",
                     "--reps", "1", "--csv", str(csv)]) == 0
    assert cli.main(["--mode", "bench", "--kernel", "lcs", "--nx", "300", "--ny", "200", "--reps", "1",
                     "--csv", str(csv)]) == 0
    assert cli.main(["--mode", "bench", "--kernel", "lcs", "--nx", "300", "--ny", "200", "--reps", "1",
                     "--tile", "64:32", "--csv", str(csv)]) == 0
    rows = [r.split(",") for r in csv.read_text().strip().splitlines()[1:]]
    want = cref.scalar_reference(get("heat2d").spec, Grid.random((96, 80), seed=0), 12)
    assert rows[0][7] == "1" and rows[1][7] == "2" and rows[0][8] == "64x32:8"
    assert rows[0][11] == rows[1][11] == f"{fnv1a64(want.dump_bytes()):016x}"
    wl = npo.scalar_reference(get("life").spec, Grid.random((96, 80), seed=0, element_kind="int32"), 12)
    assert rows[2][11] == f"{fnv1a64(wl.dump_bytes()):016x}"
    rng = np.random.default_rng(0)
    a, b = rng.integers(0, 4, 300, dtype=np.int32), rng.integers(0, 4, 200, dtype=np.int32)
    assert int(rows[3][11], 16) == int(rows[4][11], 16) == npo.lcs_length(a, b)


@pytest.mark.parametrize("mode", [{"TVS_J3D": "cpasync"}, {"TVS_J3D_FRAME": "32"}, {"TVS_J3D_FRAME": "64"}])
def test_jacobi3d_modes(cuda_ready, mode):
    """The two-level 3D kernels in every mode (read once per process): K4b,
    the cp.async-staged kernel K4c (TMA) falls back to when a block cannot be
    a tensor map, and K4c with 64 x 32 (default) and 64 x 64 frames --
    bit-exact against the oracle across frame edges."""
    import subprocess
    import sys

    env = dict(os.environ, **mode)
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "j3d_mode_check.py")],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("cluster", [1, 2, 4, 8])
def test_gs2d_pipeline_cluster_sizes(cuda_ready, cluster):
    """Lexicographic GS-2D pipeline with consecutive blocks handing off through
    distributed shared memory (cluster > 1) or the global ring (cluster 1):
    several clusters, partial last cluster, multi-pass sweeps, narrow grids
    (phantom tail filled by the loader) — bit-exact against the oracle."""
    import subprocess
    import sys

    env = dict(os.environ, TVS_GS2D_CLUSTER=str(cluster))
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "gs2d_cluster_check.py")],
                       env=env, capture_output=True, text=True, timeout=180)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("band", [0, 1024, 1500])
def test_jacobi1d_pipelined_e2e_bands(cuda_ready, band):
    """tvs_run's pipelined 1D Jacobi path (skewed position bands) is
    bit-identical to the oracle; band 0 = the plain path."""
    import subprocess
    import sys

    env = dict(os.environ, TVS_E2E_BAND1=str(band))
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "e2e_band1_check.py")],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("band", [0, 256, 300])
def test_gs2d_pipelined_e2e_bands(cuda_ready, band):
    """tvs_run's overlapped 2D Gauss-Seidel path (uploads gated into the
    running kernel, downloads gated on published blocks) is bit-identical to
    the lexicographic oracle; band 0 = the plain path."""
    import subprocess
    import sys

    env = dict(os.environ, TVS_E2E_BANDS=str(band))
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "e2e_gs2d_check.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("slab", [0, 8, 12, 32])
def test_jacobi3d_pipelined_e2e_slabs(cuda_ready, slab):
    """tvs_run's pipelined 3D Jacobi path (skewed axis-0 slabs on their own
    streams, two levels per pass) is bit-identical to the oracle; slab 0 =
    the single-stream path."""
    import subprocess
    import sys

    env = dict(os.environ, TVS_E2E_SLAB=str(slab))
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "e2e_slab_check.py")],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("band", [0, 300, 512, 777, 1024])
def test_jacobi2d_pipelined_e2e_bands(cuda_ready, band):
    """tvs_run's pipelined 2D Jacobi path (row bands on their own streams,
    uploads / launches / downloads overlapped by events) is bit-identical to
    the oracle for several band sizes; band 0 = the single-stream path."""
    import subprocess
    import sys

    env = dict(os.environ, TVS_E2E_BANDS=str(band))
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "e2e_band_check.py")],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_pipelined_drop_in_repeated_calls(cuda_ready):
    """The pipelined drop-in paths (bands / slabs skewed by each pass's
    levels) reuse the thread's device buffers across calls: every call, one
    pass or many, must read only rows its own passes wrote (regression: the
    last band read rows of the previous band's last pass without waiting
    for it, so a second call could return the first call's values)."""
    from paper_2010_04868_b200.kernels import jacobi2d_temporal, jacobi3d_temporal

    cases = [(jacobi3d_temporal, "jac3d27p", (192, 40, 50), (2, 3, 5)),
             (jacobi2d_temporal, "heat2d", (1100, 90), (3, 8, 21)),
             (heat1d_temporal, "heat1d", (600000,), (5, 64, 130))]
    for fn, kernel, ext, steps_list in cases:
        spec = get(kernel).spec
        for seed, steps in enumerate(steps_list):
            g = Grid.random(ext, seed=seed)
            want = cref.scalar_reference(spec, g, steps).interior
            for rep in range(3):
                got = fn(g, steps, kernel=kernel).interior
                assert np.array_equal(got, want), (kernel, steps, rep)


@pytest.mark.parametrize("order", ["lexicographic", "reference"])
def test_gs2d_lane_ring_slot_reuse(cuda_ready, order):
    """K6v3 hands rows between CTAs through an L2 ring of 320 slots: narrow
    grids (short CTA lifetimes, > 320 CTAs) reuse slots while older CTAs are
    still running.  A consumer may read a reused slot only after its producer
    took it over from the previous consumer (regression: stale cells read as
    valid), through the drop-in (copy overlap) and the plan API."""
    spec = get("gs2d9p").spec
    for rows, cols, steps in [(1300, 64, 1), (2048, 64, 2), (2048, 200, 5), (3000, 64, 40), (1400, 48, 100)]:
        if order == "reference" and steps < 2:
            continue
        g = Grid.random((rows, cols), seed=rows + steps)
        want = cref.scalar_reference(spec, g, steps, order=order).interior
        got = execute(spec, g, steps, order=order).interior  # drop-in (row bands overlap the kernel)
        assert np.array_equal(got, want), (rows, cols, steps, "drop-in")
        plan = _native.Plan(spec, (rows, cols), config.current().native(order=order))
        plan.upload(g.data, g.offset)
        plan.run(steps)
        out = g.alloc_like()
        plan.download(out.data, out.offset)
        plan.close()
        assert np.array_equal(out.interior, want), (rows, cols, steps, "plan")


@pytest.mark.parametrize("order", ["lexicographic", "reference"])
def test_gs2d_lane_capacities(cuda_ready, order):
    """K6v3 packs lr = sweeps-per-pass (rounded up to even) lanes per group
    into warps and picks a lane capacity of 32 / 64 / 102 / 128: sweep counts
    on both sides of every capacity, odd counts (one idle lane), more than
    128 sweeps (balanced passes), grids narrower than a loader block and with
    fewer rows than a CTA's groups -- bit-exact against the oracle."""
    for kernel in ("gs2d9p", "gs2d"):
        spec = get(kernel).spec
        for ext, steps in [((9, 3), 2), ((3, 70), 31), ((40, 33), 33), ((70, 50), 63), ((33, 120), 64),
                           ((50, 40), 65), ((45, 260), 101), ((120, 45), 102), ((60, 60), 103), ((30, 90), 128),
                           ((64, 64), 129), ((40, 70), 200), ((2, 2), 257)]:
            g = Grid.random(ext, seed=ext[0] + steps, boundary=-0.5 if steps % 2 else 0.0)
            sp = spec_for(kernel, g.boundary)
            want = cref.scalar_reference(sp, g, steps, order=order).interior
            got = execute(sp, g, steps, order=order).interior
            assert np.array_equal(got, want), (kernel, ext, steps)


def test_pipelined_kernels_repeat_stable(cuda_ready):
    """Races in the kernels with device-side hand-offs (K6v3's loader /
    compute barriers and L2 ring, K4c's TMA ring) would show as run-to-run
    differences: mid-size grids (several CTA waves), ten runs each, every
    result bit-identical to the first and the first to the oracle."""
    for kernel, ext, steps, kw in (("gs2d9p", (1500, 2100), 100, {"order": "lexicographic"}),
                                   ("gs2d9p", (1200, 1700), 100, {"order": "reference"}),
                                   ("gs2d", (900, 1300), 64, {"order": "reference"}),
                                   ("jac3d27p", (150, 130, 200), 8, {})):
        g = Grid.random(ext, seed=7)
        spec = get(kernel).spec
        want = cref.scalar_reference(spec, g, steps, **kw).interior
        first = execute(spec, g, steps, **kw).interior
        assert np.array_equal(first, want), (kernel, ext)
        for rep in range(9):
            assert np.array_equal(execute(spec, g, steps, **kw).interior, first), (kernel, ext, rep)


def test_staged_pageable_uploads(cuda_ready):
    """Pageable inputs are staged by the library (csrc/hostcopy.cu: host
    thread pool -> page-locked 32 MiB slots -> DMA per slot): 1D, 2D and 3D
    grids larger than several slots, chunks spanning 3D planes, odd row
    widths, results equal to the page-locked path and to the oracle; the
    result Grid comes from the page-locked result pool and keeps the input's
    frame."""
    from paper_2010_04868_b200.kernels import jacobi2d_temporal, jacobi3d_temporal

    cases = [(jacobi3d_temporal, "heat3d", (163, 171, 301), 3), (jacobi2d_temporal, "heat2d", (3001, 2999), 5),
             (heat1d_temporal, "heat1d", (9_000_001,), 4)]
    for fn, kernel, ext, steps in cases:
        spec = get(kernel).spec
        g = Grid.random(ext, seed=len(ext), boundary=0.5)
        assert g.data.nbytes > 2 * (32 << 20)  # several staging slots
        want = cref.scalar_reference(spec, g, steps, threads=8)
        got = fn(g, steps, kernel=kernel)
        assert np.array_equal(got.interior, want.interior), kernel
        for sl in g.frame_slices():
            assert np.array_equal(got.data[sl], g.data[sl]), kernel
        pg = Grid(ext, 1, boundary=0.5, pinned=True)
        np.copyto(pg.data, g.data)
        assert np.array_equal(fn(pg, steps, kernel=kernel).interior, want.interior), kernel


def test_problem_struct_entry_points(cuda_ready):
    """tvs_jacobi / tvs_gauss_seidel (the SURVEY.md §8(b) signatures: one
    tvs_problem for stencil + Grid layout) equal the oracle."""
    import ctypes as C

    lib = _native.lib()
    for kernel, ext, steps in (("heat2d", (130, 97), 9), ("jac3d27p", (20, 33, 41), 3), ("heat1d", (5000,), 40)):
        g = Grid.random(ext, seed=2, boundary=0.25)
        spec = get(kernel).spec
        out = g.copy()
        prob = _native.make_problem(spec, g)
        _native.check(lib.tvs_jacobi(C.byref(prob), g.data.ctypes.data, out.data.ctypes.data, steps,
                                     C.byref(_native.make_exec())))
        assert np.array_equal(out.interior, cref.scalar_reference(spec, g, steps).interior), kernel
    for order, code in (("lexicographic", 0), ("reference", 1)):
        g = Grid.random((90, 70), seed=3)
        spec = get("gs2d9p").spec
        work = g.copy()
        prob = _native.make_problem(spec, g)
        _native.check(lib.tvs_gauss_seidel(C.byref(prob), work.data.ctypes.data, 7, code,
                                           C.byref(_native.make_exec())))
        assert np.array_equal(work.interior, cref.scalar_reference(spec, g, 7, order=order).interior), order
