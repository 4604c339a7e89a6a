"""Iteration-space tiling and the wave executor (reference ``tiling.py``),
with the waves run on the GPU.

Same API as the reference (``tiling.py:45-148, 252-371``): ``Tile``,
``TileSchedule``, ``SHAPE_BY_KERNEL``, ``build_schedule``, ``coverage_map``,
``check_coverage``, ``check_wave_order``, ``execute_parallel`` and
``lcs_blocked``, with the same size errors.  The schedules follow the
reference's tile shapes:

* ``diamond`` (1D Jacobi): per time band of ``time_height`` steps, a family
  of trapezoids that shrink by one cell per step on each side, then the
  family of growing trapezoids filling the gaps between them;
* ``hybrid`` (2D/3D Jacobi, Life): diamond on axis 0, left-shifting
  parallelograms (slope -1) on the inner axes, chained left to right by
  wave number;
* ``parallelogram`` (Gauss-Seidel): slope -1 on every axis, tile
  (band, k...) in wave (dim + 1) * band + sum(k) — the pipelined wavefront;
* ``rectangle`` (LCS): fixed windows, anti-diagonal waves.

Execution (``execute_parallel``) keeps the reference's full time history
(one padded plane per level, same 3e8-element cap) but in HBM: every wave
is ONE kernel launch in which each CTA runs one tile's time levels (a
barrier between levels; Gauss-Seidel windows are swept by hyperplanes
``h = a.x`` with every lexicographically-earlier neighbour on an earlier
hyperplane).  ``workers`` is accepted for signature parity — all tiles of a
wave already run concurrently as CTAs — so the result is trivially the same
for every worker count.  Gauss-Seidel tiles use the lexicographic in-place
semantics (lexicographically negative offsets read the current sweep),
identical to the reference's tile engine for its star stencils
(``tiling.py:418-447``).
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import _native, config
from .catalog import LCS_PARAMS, get as catalog_get
from .errors import SizeError
from .grid import Grid

SHAPE_BY_KERNEL = {
    "heat1d": "diamond",
    "heat2d": "hybrid",
    "jac2d9p": "hybrid",
    "heat3d": "hybrid",
    "life": "hybrid",
    "gs1d": "parallelogram",
    "gs2d": "parallelogram",
    "gs3d": "parallelogram",
    "lcs": "rectangle",
}

MAX_HISTORY_ELEMS = 3 * 10**8  # reference tiling.py:328


@dataclass(frozen=True)
class Tile:
    """Time range [t0, t1) and per-axis windows moving with the step:
    axis d at time t covers [lo[d] + slope_lo[d]*(t-t0), hi[d] +
    slope_hi[d]*(t-t0)), clipped to the grid."""

    t0: int
    t1: int
    lo: tuple
    hi: tuple
    slope_lo: tuple
    slope_hi: tuple

    def windows(self, t: int, extents) -> list:
        dt = t - self.t0
        out = []
        for d, n in enumerate(extents):
            a = max(self.lo[d] + self.slope_lo[d] * dt, 0)
            b = min(self.hi[d] + self.slope_hi[d] * dt, n)
            out.append((a, max(a, b)))
        return out

    def as_dict(self):
        return {"time": [self.t0, self.t1], "origin": list(self.lo),
                "extents": [h - l for l, h in zip(self.lo, self.hi)],
                "slope_lo": list(self.slope_lo), "slope_hi": list(self.slope_hi)}


@dataclass
class TileSchedule:
    shape: str
    extents: tuple
    steps: int
    space_tile: tuple
    time_height: int
    waves: list = field(default_factory=list)

    def tiles(self):
        for w in self.waves:
            yield from w

    def dump_json(self) -> str:
        return json.dumps({"shape": self.shape, "extents": list(self.extents), "steps": self.steps,
                           "space_tile": list(self.space_tile), "time_height": self.time_height,
                           "waves": [[t.as_dict() for t in w] for w in self.waves]}, indent=1)


def _blocks(n: int, w: int, shifting: bool):
    """Blocks [k*w, (k+1)*w) along one axis; a left-shifting axis needs one
    more block to keep covering the right edge."""
    count = -(-n // w) + (1 if shifting else 0)
    return [(k, k * w, (k + 1) * w) for k in range(count)]


def _product(axes):
    combos = [()]
    for ax in axes:
        combos = [c + (b,) for c in combos for b in ax]
    return combos


def _live(tile: Tile, extents) -> bool:
    return any(all(b > a for a, b in tile.windows(t, extents)) for t in range(tile.t0, tile.t1))


def build_schedule(kernel: str, extents, steps: int, space_tile, time_height: int) -> TileSchedule:
    """Legal tile schedule for one kernel's dependence structure
    (reference tiling.py:116-148, same SizeError conditions)."""
    extents = tuple(int(e) for e in extents)
    space_tile = tuple(int(w) for w in space_tile)
    steps, h = int(steps), int(time_height)
    shape = SHAPE_BY_KERNEL[kernel]
    if kernel == "lcs":
        vl = LCS_PARAMS.vl
    else:
        entry = catalog_get(kernel)
        vl = entry.vl
        if shape in ("diamond", "hybrid") and space_tile[0] < 4 * entry.s * vl:
            raise SizeError(f"vectorized-dimension tile {space_tile[0]} below 4*s*vl = {4 * entry.s * vl}")
    if h <= 0 or h % vl:
        raise SizeError(f"time_height {h} must be a positive multiple of vl={vl}")
    if len(space_tile) != len(extents) or any(w <= 0 for w in space_tile):
        raise SizeError("bad space_tile")
    if shape == "parallelogram" and h > min(space_tile):
        raise SizeError("parallelogram tiling requires time_height <= every space tile")
    if shape == "hybrid" and len(extents) > 1 and h > min(space_tile[1:]):
        raise SizeError("hybrid tiling requires time_height <= inner space tiles")

    sched = TileSchedule(shape, extents, steps, space_tile, h)
    nbands = -(-steps // h)
    waves: dict = {}

    def put(w, tile):
        if _live(tile, extents):
            waves.setdefault(w, []).append(tile)

    if shape in ("diamond", "hybrid"):
        inner = [_blocks(n, w, True) for n, w in zip(extents[1:], space_tile[1:])]
        stride = sum(len(ax) for ax in inner) + 1  # wave slots per family
        wx, nkx = space_tile[0], -(-extents[0] // space_tile[0])
        down = tuple(-1 for _ in inner)
        for b in range(nbands):
            t0, t1 = b * h, min((b + 1) * h, steps)
            for combo in _product(inner):
                k = sum(c[0] for c in combo)
                ilo, ihi = tuple(c[1] for c in combo), tuple(c[2] for c in combo)
                for kx in range(nkx + 1):  # shrinking family
                    put(2 * b * stride + k, Tile(t0, t1, (kx * wx,) + ilo, ((kx + 1) * wx,) + ihi,
                                                 (1,) + down, (-1,) + down))
                for kx in range(-1, nkx + 1):  # growing family, apex at the shared edge
                    c = (kx + 1) * wx
                    put((2 * b + 1) * stride + k, Tile(t0, t1, (c,) + ilo, (c,) + ihi, (-1,) + down, (1,) + down))
    elif shape == "parallelogram":
        axes = [_blocks(n, w, True) for n, w in zip(extents, space_tile)]
        down = tuple(-1 for _ in extents)
        for b in range(nbands):
            t0, t1 = b * h, min((b + 1) * h, steps)
            for combo in _product(axes):
                put((len(extents) + 1) * b + sum(c[0] for c in combo),
                    Tile(t0, t1, tuple(c[1] for c in combo), tuple(c[2] for c in combo), down, down))
    else:  # rectangle
        axes = [_blocks(n, w, False) for n, w in zip(extents, space_tile)]
        flat = tuple(0 for _ in extents)
        for b in range(nbands):
            t0, t1 = b * h, min((b + 1) * h, steps)
            for combo in _product(axes):
                put(b + sum(c[0] for c in combo),
                    Tile(t0, t1, tuple(c[1] for c in combo), tuple(c[2] for c in combo), flat, flat))
    sched.waves = [waves[w] for w in sorted(waves)]
    return sched


# ---- schedule invariants (reference tiling.py:252-325) -------------------

def coverage_map(schedule: TileSchedule):
    """How many tiles compute each (time, point) of the iteration space."""
    counts = np.zeros((schedule.steps,) + schedule.extents, dtype=np.int16)
    for tile in schedule.tiles():
        for t in range(tile.t0, min(tile.t1, schedule.steps)):
            counts[(t,) + tuple(slice(a, b) for a, b in tile.windows(t, schedule.extents))] += 1
    return counts


def check_coverage(schedule: TileSchedule) -> bool:
    """Every point computed exactly once."""
    return bool((coverage_map(schedule) == 1).all())


def check_wave_order(schedule: TileSchedule, deps) -> bool:
    """Every dependence source lies in an earlier wave, or in the same tile
    (ordered by the in-tile sweep).  Exhaustive; test-sized spaces."""
    ext = schedule.extents
    owner = np.full((schedule.steps + 1,) + ext, -1, dtype=np.int64)
    tiles = []
    for w, wave in enumerate(schedule.waves):
        for tile in wave:
            tid = len(tiles)
            tiles.append((tile, w))
            for t in range(tile.t0, min(tile.t1, schedule.steps)):
                owner[(t + 1,) + tuple(slice(a, b) for a, b in tile.windows(t, ext))] = tid
    if (owner[1:] < 0).any():
        return False
    wave_of = np.array([w for _, w in tiles] + [-1], dtype=np.int64)  # index -1 -> initial plane
    for tid, (tile, w) in enumerate(tiles):
        for t in range(tile.t0, min(tile.t1, schedule.steps)):
            win = tile.windows(t, ext)
            if any(b <= a for a, b in win):
                continue
            for d in deps:
                src_t = t + 1 - d.dt
                if src_t < 1:
                    continue  # the initial grid
                sl = []
                for i, (a, b) in enumerate(win):
                    lo, hi = max(a + d.dx[i], 0), min(b + d.dx[i], ext[i])
                    if hi <= lo:
                        break
                    sl.append(slice(lo, hi))
                else:
                    src = owner[(src_t,) + tuple(sl)]
                    sw = wave_of[src]
                    if (sw > w).any() or ((sw == w) & (src != tid)).any():
                        return False
    return True


# ---- GPU execution ---------------------------------------------------------

def _tile_array(schedule: TileSchedule):
    tiles = list(schedule.tiles())
    arr = (_native.TileDesc * max(len(tiles), 1))()
    for i, t in enumerate(tiles):
        arr[i].t0, arr[i].t1 = t.t0, min(t.t1, schedule.steps)
        for d in range(len(schedule.extents)):
            arr[i].lo[d], arr[i].hi[d] = t.lo[d], t.hi[d]
            arr[i].slope_lo[d], arr[i].slope_hi[d] = t.slope_lo[d], t.slope_hi[d]
    starts = [0]
    for w in schedule.waves:
        starts.append(starts[-1] + len(w))
    return arr, (C.c_int64 * len(starts))(*starts), len(schedule.waves)


def execute_parallel(kernel: str, grid: Grid, schedule: TileSchedule, workers: int = 1, variant=None) -> Grid:
    """Run the schedule wave by wave on the GPU (one launch per wave, one
    CTA per tile); bit-identical to the unblocked kernel and independent of
    ``workers`` (reference tiling.py:347-371)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    spec = catalog_get(kernel).spec
    if tuple(grid.extents) != tuple(schedule.extents):
        raise SizeError("grid extents differ from the schedule's")
    total = (schedule.steps + 1) * grid.data.size
    if total > MAX_HISTORY_ELEMS:
        raise SizeError(f"blocked execution would need {total} elements of history; desk scale only")
    out = grid.copy()
    if schedule.steps == 0:
        return out
    tiles, starts, nw = _tile_array(schedule)
    lay = _native.make_layout(grid.data, grid.extents, grid.offset)
    ex = config.current().native()
    if spec.is_life:
        rule = _native.make_life_rule(spec, grid.boundary)
        rc = _native.lib().tvs_tiled_life(C.byref(rule), C.byref(lay), grid.data.ctypes.data, out.data.ctypes.data,
                                          schedule.steps, tiles, starts, nw, C.byref(ex))
    else:
        st = _native.make_stencil(spec, grid.boundary)  # Dirichlet value from the grid (tiling.py:340)
        rc = _native.lib().tvs_tiled_run(C.byref(st), C.byref(lay), grid.data.ctypes.data, out.data.ctypes.data,
                                         schedule.steps, tiles, starts, nw, C.byref(ex))
    _native.check(rc, f"tvs_tiled_run({kernel})")
    out.fill_halo()  # the reference resets the result's halo (tiling.py:370)
    return out


def lcs_blocked(a, b, schedule: TileSchedule, workers: int = 1) -> int:
    """Rectangle-tiled LCS over the full DP table, anti-diagonal waves of
    tiles (reference tiling.py:374-406); time = the A index, space = B."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    a = np.ascontiguousarray(a, dtype=np.int32).ravel()
    b = np.ascontiguousarray(b, dtype=np.int32).ravel()
    if a.size == 0 or b.size == 0:
        return 0
    tiles, starts, nw = _tile_array(schedule)
    n = C.c_int64(0)
    _native.check(_native.lib().tvs_lcs_tiled(a.ctypes.data, a.size, b.ctypes.data, b.size, tiles, starts, nw,
                                              C.byref(config.current().native()), C.byref(n)), "tvs_lcs_tiled")
    return int(n.value)
