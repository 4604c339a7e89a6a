"""Sharded Jacobi host logic on CPU: torch.distributed gloo, world size 2/3,
slab split + halo exchange + ghost pinning, with a NumPy stand-in for the
device step.  Must equal the single-domain oracle bit-exactly (the same
invariant the GPU path meets, tests/test_gpu_parity.py)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_04868_b200 import halo


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def numpy_step(spec):
    """k Jacobi steps on one slab in the library's device layout (test
    stand-in for tvs_jacobi_device): unfused taps in sorted order, rows
    outside the global domain pinned to the boundary."""
    offs = spec.offsets()
    cs = [spec.coefficients[o] for o in offs]

    def step(lay, src, dst, k):
        g = lay.geometry
        dim = g.dim
        ext = tuple(int(g.extents[d]) for d in range(dim))
        shape = (ext[0] + 2,) + ((ext[1] + 2,) if dim == 3 else ()) + (int(g.strides[dim - 2]) if dim > 1 else 0,)
        a, b = src.numpy().reshape(shape), dst.numpy().reshape(shape)
        lo = (1,) * (dim - 1) + (32,)
        for _ in range(k):
            def win(arr, o):
                return arr[tuple(slice(l + oo, l + oo + e) for l, oo, e in zip(lo, o, ext))]

            acc = cs[0] * win(a, offs[0])
            for c, o in zip(cs[1:], offs[1:]):
                acc = c * win(a, o) + acc
            rows = np.arange(ext[0]) + int(g.axis0_offset)
            acc[(rows < 0) | (rows >= int(g.axis0_global))] = spec.boundary
            win(b, (0,) * dim)[...] = acc
            a, b = b, a
        return k % 2 == 1

    return step


def numpy_rows(spec):
    """Ranged pass (stand-in for tvs_jacobi_device_rows): k steps writing only
    local rows [lo, hi) of dst.  Rows outside [lo - k, hi + k) are poisoned
    with NaN in the working copy, so a range the k-step cone does not cover
    (or halos used before they land) shows up as NaN in the result."""
    step = numpy_step(spec)

    def rows(lay, src, dst, k, lo, hi):
        g = lay.geometry
        s0 = int(g.strides[0])
        work = src.clone()
        tmp = src.clone()  # pads / memory halo keep the boundary value
        for r in range(-1, int(g.extents[0]) + 1):
            if not lo - k <= r < hi + k:
                work[(r + 1) * s0:(r + 2) * s0] = float("nan")
        res = tmp if step(lay, work, tmp, k) else work
        dst[(lo + 1) * s0:(hi + 1) * s0] = res[(lo + 1) * s0:(hi + 1) * s0]

    return rows


def _worker(rank, world, port, kernel, ext, steps, depth, expect, overlap=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2010_04868_b200.catalog import get

        spec = get(kernel).spec
        full = np.random.default_rng(7).uniform(0, 1, ext)
        sj = halo.ShardedJacobi(spec, ext, dist, depth=depth, device=torch.device("cpu"), step_fn=numpy_step(spec),
                                rows_fn=numpy_rows(spec) if overlap else None, overlap=overlap)
        sj.load_global(full)
        sj.run(steps)
        got = sj.gather().numpy()
        if rank == 0:
            assert got.shape == tuple(ext)
            assert np.array_equal(got, expect), f"world={world} depth={depth}"
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kernel,ext,steps,depth", [("heat2d", (23, 17), 11, 4), ("jac2d9p", (30, 9), 7, 3),
                                                     ("jac3d27p", (13, 6, 7), 5, 2)])
def test_sharded_equals_single_domain(world, kernel, ext, steps, depth, overlap):
    """Blocking exchange, and the overlapped pass (interior rows launched
    while the halos are in flight, edge rows after they land)."""
    from oracle import oracle as npo
    from paper_2010_04868_b200 import Grid
    from paper_2010_04868_b200.catalog import get

    g = Grid(ext, 1)
    g.set_interior(np.random.default_rng(7).uniform(0, 1, ext))
    expect = npo.scalar_reference(get(kernel).spec, g, steps).interior.copy()
    mp.spawn(_worker, args=(world, _free_port(), kernel, ext, steps, depth, expect, overlap), nprocs=world, join=True)


def test_split_rows_balanced():
    for n in (1, 7, 16384):
        for w in (1, 2, 3, 8):
            parts = [halo.split_rows(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_layout_rejects_thin_slabs():
    with pytest.raises(ValueError):
        halo.make_layout((10, 10), world=4, rank=1, ghost=4)
    lay = halo.make_layout((16384, 16384), world=8, rank=3, ghost=8)
    assert lay.r0 == 6144 and lay.extents[0] == 2048 + 16 and lay.geometry.axis0_offset == 6144 - 8
    assert lay.row_slice(0, 1).stop - lay.row_slice(0, 1).start == lay.row_elems
