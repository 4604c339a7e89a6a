"""Parity at BASELINE.json's full sizes through size-independent properties.

1. Light cones.  After T Jacobi steps a point depends only on inputs within
   T cells of it.  After T lexicographic Gauss-Seidel sweeps the first rows
   depend only on the first rows + T: a sweep reads the current sweep only
   from earlier rows (and the row's left part) and the previous sweep at most
   one row further down.  (Not one column to the right: the box stencil's NE
   tap chains current-sweep values rightwards along every earlier row, so 2D
   windows keep the full width.)  So the oracle, run on a window of the
   full-size input with the true Dirichlet boundary on the domain faces the
   window touches, reproduces the full-size GPU result exactly on the part of
   the window farther than T cells from its cut faces.  Bit-exact.
2. Two independent GPU algorithms agree bit-exactly on the whole full-size
   grid: the temporally blocked / pipelined kernels against the single-step
   (Jacobi) and hyperplane-wavefront (Gauss-Seidel) kernels.

Inputs are the BASELINE generators (bench.make_grid: seeds, distributions,
seeded weights)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from oracle import cref
from paper_2010_04868_b200 import Grid, _native, config
from paper_2010_04868_b200.catalog import get

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

pytestmark = pytest.mark.gpu
H = 8  # checked cells per window side


def _gpu_full(cfg, g, out, algo="auto"):
    """Full-size device run of grid ``g`` through the plan API into ``out``."""
    spec = get(cfg["kernel"]).spec
    plan = _native.Plan(spec, cfg["extents"], config.current().native(algo=algo, fma="exact"))
    plan.upload(g.data, g.offset)
    plan.run(cfg["T"])
    plan.download(out.data, out.offset)
    plan.close()
    return out


def _digest(grid):
    """Checksum of checksums: wrapping uint64 sums of the bit patterns of
    every axis-0 slice (exact-match evidence for arrays too large to keep
    twice in host memory)."""
    v = grid.interior.view(np.uint64)
    return v.reshape(v.shape[0], -1).sum(axis=1) if v.ndim > 1 else np.add.reduceat(v, np.arange(0, v.size, 4096))


def _window_oracle(spec, full_in, lo, hi, T):
    """Oracle on input[lo:hi] (per axis) with the grid's boundary outside."""
    sl = tuple(slice(a, b) for a, b in zip(lo, hi))
    w = Grid(tuple(b - a for a, b in zip(lo, hi)), 1, boundary=full_in.boundary)
    w.set_interior(np.ascontiguousarray(full_in.interior[sl]))
    return cref.scalar_reference(spec, w, T, order="lexicographic", threads=16)


def _check(spec, g, out, lo, hi, chk_lo, chk_hi, T):
    """Oracle window [lo, hi) vs the GPU result on [chk_lo, chk_hi)."""
    want = _window_oracle(spec, g, lo, hi, T).interior
    wsl = tuple(slice(c0 - a, c1 - a) for a, c0, c1 in zip(lo, chk_lo, chk_hi))
    gsl = tuple(slice(c0, c1) for c0, c1 in zip(chk_lo, chk_hi))
    assert np.array_equal(out.interior[gsl], want[wsl]), (lo, hi, chk_lo, chk_hi)


def _jacobi_windows(ext, T):
    """(window lo, hi, check lo, hi): every corner and the centre."""
    dim = len(ext)
    wins = []
    for corner in range(2 ** dim):
        lo, hi, clo, chi = [], [], [], []
        for d in range(dim):
            if (corner >> d) & 1:
                lo.append(ext[d] - H - T), hi.append(ext[d]), clo.append(ext[d] - H), chi.append(ext[d])
            else:
                lo.append(0), hi.append(H + T), clo.append(0), chi.append(H)
        wins.append((lo, hi, clo, chi))
    c = [e // 2 for e in ext]
    wins.append(([x - H - T for x in c], [x + H + T for x in c], [x - H for x in c], [x + H for x in c]))
    return wins


@pytest.mark.parametrize("cid", [1, 3, 5])
def test_jacobi_full_size_light_cones_and_single_step_identity(cuda_ready, cid):
    cfg = bench.CONFIGS[cid]
    spec = get(cfg["kernel"]).spec
    T = cfg["T"]
    g = bench.make_grid(cfg)
    out = _gpu_full(cfg, g, g.alloc_like())
    for lo, hi, clo, chi in _jacobi_windows(cfg["extents"], T):
        _check(spec, g, out, lo, hi, clo, chi, T)
    blocked = _digest(out)
    assert np.array_equal(_digest(_gpu_full(cfg, g, out, algo="naive")), blocked)


@pytest.mark.parametrize("cid", [2, 4])
def test_gauss_seidel_full_size_corner_and_wavefront_identity(cuda_ready, cid):
    cfg = bench.CONFIGS[cid]
    spec = get(cfg["kernel"]).spec
    T = cfg["T"]
    g = bench.make_grid(cfg)
    out = _gpu_full(cfg, g, g.alloc_like())
    if cid == 2:
        _check(spec, g, out, [0], [H + T], [0], [H], T)
        _check(spec, g, out, [0], [4096 + T], [0], [4096], T)  # the first 4096 positions
    else:
        w = cfg["extents"][1]
        _check(spec, g, out, [0, 0], [H + T, w], [0, 0], [H, w], T)  # the first H full rows
    pipelined = _digest(out)
    assert np.array_equal(_digest(_gpu_full(cfg, g, out, algo="naive")), pipelined)
