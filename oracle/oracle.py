"""NumPy restatement of the reference CPU stencil path (test infrastructure).

Follows tvstencil/baselines.py of the reference:
* ``jacobi_plane_update``  <- baselines.py:43-49 (whole-plane taps, first a
  multiply, then ``c*v + acc``; NumPy ufuncs round every op separately);
* ``gs_sweep_1d``           <- baselines.py:73-80 (in-place Python loop);
* ``gs_sweep_antidiagonal`` <- baselines.py:83-107 (anti-diagonal groups,
  gather all taps, then scatter);
* ``scalar_reference``      <- baselines.py:110-125 (out of place; Jacobi
  ping-pongs two planes, GS sweeps one copy in place).
* ``life_plane_update``    <- baselines.py:52-66 (int32 neighbour sum, the
  B-then-S ``np.where`` decision tree);
* ``lcs_length``           <- baselines.py:128-150 (full-table quadratic DP
  swept along anti-diagonals).
Added: ``gs_sweep_lexicographic`` (row-major in-place order, the loop of
test_baselines.py:39-52 for any tap set), selected with
``scalar_reference(..., order="lexicographic")``.
"""

from __future__ import annotations

import itertools

import numpy as np


def _window(grid_data, offset, extents, shift):
    return grid_data[tuple(slice(offset + s, offset + s + e) for s, e in zip(shift, extents))]


def jacobi_plane_update(spec, src, dst, offset, extents):
    """One Jacobi step over the whole interior (baselines.py:43-49)."""
    taps = spec.offsets()
    acc = spec.coefficients[taps[0]] * _window(src, offset, extents, taps[0])
    for off in taps[1:]:
        acc = spec.coefficients[off] * _window(src, offset, extents, off) + acc
    _window(dst, offset, extents, (0,) * len(extents))[...] = acc


def life_plane_update(spec, src, dst, offset, extents):
    """One Life-like step over the whole interior (baselines.py:52-66):
    n = int32 sum of the ``offsets()`` neighbours (wrapping), then count in
    birth -> 1, else count in survive (minus birth) -> own state, else 0."""
    taps = spec.offsets()
    n = _window(src, offset, extents, taps[0]) + _window(src, offset, extents, taps[1])
    for off in taps[2:]:
        n = n + _window(src, offset, extents, off)
    alive = _window(src, offset, extents, (0,) * len(extents))
    out = np.zeros_like(alive)
    for b in sorted(spec.birth):
        out = np.where(n == b, np.int32(1), out)
    for sv in sorted(set(spec.survive) - set(spec.birth)):
        out = np.where(n == sv, alive, out)
    _window(dst, offset, extents, (0,) * len(extents))[...] = out


def lcs_length(a, b) -> int:
    """LCS length by the full-table DP along anti-diagonals
    (baselines.py:128-150)."""
    a = np.asarray(a, dtype=np.int32)
    b = np.asarray(b, dtype=np.int32)
    n, m = len(a), len(b)
    if n == 0 or m == 0:
        return 0
    table = np.zeros((n + 1, m + 1), dtype=np.int32)
    for d in range(2, n + m + 1):
        i0, i1 = max(1, d - m), min(n, d - 1)
        if i0 > i1:
            continue
        i = np.arange(i0, i1 + 1)
        j = d - i
        eq = a[i - 1] == b[j - 1]
        table[i, j] = np.where(eq, table[i - 1, j - 1] + np.int32(1), np.maximum(table[i - 1, j], table[i, j - 1]))
    return int(table[n, m])


def gs_sweep_1d(spec, data, offset, n):
    """In-place lexicographic 1D sweep (baselines.py:73-80)."""
    taps = spec.offsets()
    cs = [spec.coefficients[o] for o in taps]
    for x in range(offset, offset + n):
        acc = cs[0] * data[x + taps[0][0]]
        for c, o in zip(cs[1:], taps[1:]):
            acc = c * data[x + o[0]] + acc
        data[x] = acc


def _hyperplane_sweep(spec, data, offset, extents, weights):
    """One in-place sweep that visits points in increasing ``weights . x``
    and, inside a level set, gathers every tap before scattering."""
    taps = spec.offsets()
    cs = [spec.coefficients[o] for o in taps]
    coords = np.indices(extents).reshape(len(extents), -1)
    key = np.tensordot(np.asarray(weights), coords, axes=1)
    order = np.argsort(key, kind="stable")
    key = key[order]
    coords = coords[:, order] + offset
    bounds = np.flatnonzero(np.diff(key)) + 1
    for lo, hi in zip(np.r_[0, bounds], np.r_[bounds, key.size]):
        pts = coords[:, lo:hi]

        def gather(o):
            return data[tuple(pts[d] + o[d] for d in range(len(extents)))]

        acc = cs[0] * gather(taps[0])
        for c, o in zip(cs[1:], taps[1:]):
            acc = c * gather(o) + acc
        data[tuple(pts)] = acc


def gs_sweep_antidiagonal(spec, data, offset, extents):
    """Reference-order sweep (baselines.py:83-107): level sets of the
    coordinate sum, gather then scatter."""
    _hyperplane_sweep(spec, data, offset, extents, [1] * len(extents))


def gs_sweep_lexicographic(spec, data, offset, extents):
    """Row-major in-place sweep, vectorised over the hyperplanes
    ``sum_d 2^(dim-1-d) x_d``: every lexicographically earlier radius-1
    neighbour has a strictly smaller key and every later one a larger key, so
    each level set reads exactly the values the scalar loop would."""
    dim = len(extents)
    _hyperplane_sweep(spec, data, offset, extents, [2 ** (dim - 1 - d) for d in range(dim)])


def gs_sweep_loop(spec, data, offset, extents):
    """Plain nested-loop lexicographic sweep (test_baselines.py:39-52 form);
    tiny grids only — the independent check of the vectorised sweeps."""
    taps = spec.offsets()
    cs = [spec.coefficients[o] for o in taps]
    for x in itertools.product(*[range(e) for e in extents]):
        base = tuple(offset + c for c in x)
        acc = cs[0] * data[tuple(b + o for b, o in zip(base, taps[0]))]
        for c, o in zip(cs[1:], taps[1:]):
            acc = c * data[tuple(b + oo for b, oo in zip(base, o))] + acc
        data[base] = acc


def scalar_reference(spec, grid, steps, order="reference"):
    """Ground truth after ``steps`` updates, out of place (baselines.py:110-125).

    ``order`` only matters for Gauss-Seidel in 2D/3D: ``"reference"`` is the
    reference oracle's anti-diagonal order, ``"lexicographic"`` the row-major
    loop.  Returns a new grid object of the input's class."""
    cur = grid.copy()
    if spec.dependence_kind == "gauss_seidel":
        for _ in range(steps):
            if spec.dim == 1:
                gs_sweep_1d(spec, cur.data, cur.offset, cur.extents[0])
            elif order == "reference":
                gs_sweep_antidiagonal(spec, cur.data, cur.offset, cur.extents)
            elif order == "lexicographic":
                gs_sweep_lexicographic(spec, cur.data, cur.offset, cur.extents)
            else:
                raise ValueError(order)
        return cur
    nxt = grid.alloc_like()
    update = life_plane_update if spec.is_life else jacobi_plane_update
    for _ in range(steps):
        update(spec, cur.data, nxt.data, cur.offset, cur.extents)
        cur, nxt = nxt, cur
    return cur
