"""Stencil problem definitions and the dependence facts the GPU schedules use.

Mirrors the reference's data model (``tvstencil/model.py``): ``StencilSpec``
(``model.py:76-132``) with the same validation and the same ``offsets()``
order — sorted offsets, which fixes the expression tree
``acc = c0*v0; acc = ck*vk + acc`` and hence the float rounding shared by the
oracle and every CUDA kernel; ``dependences`` / ``min_space_stride``
(``model.py:142-193``).

Added for the GPU schedules: ``gs_hyperplane`` — the integer hyperplane
``h = a . x + tau * t`` under which every Gauss-Seidel dependence goes
strictly backwards, for either update order.  The CUDA
wavefront kernels receive (a, tau) and the host verifies them here.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from typing import Mapping

from .errors import IllegalDependence

Offset = tuple[int, ...]


def _lex_negative(dx: Offset) -> bool:
    for c in dx:
        if c:
            return c < 0
    return False


@dataclass(frozen=True)
class Dependence:
    """dt >= 0 time distance and dx = x_source - x_target per space axis."""

    dt: int
    dx: Offset

    def __post_init__(self):
        if self.dt < 0:
            raise ValueError("dt must be >= 0")
        if self.dt == 0 and not _lex_negative(self.dx):
            raise ValueError(f"dt=0 dependence {self.dx} must be lexicographically negative")


@dataclass(frozen=True)
class ScheduleParams:
    """CPU time-lane schedule (s, sl, vl).  Accepted for signature parity
    (``model.py:50-73``); the GPU kernels choose their own lane lag."""

    s: int
    sl: int = 0
    vl: int = 4

    def __post_init__(self):
        if self.s < 1 or self.sl < 0:
            raise ValueError("require s >= 1 and sl >= 0")
        if self.vl not in (1, 4, 8):
            raise ValueError("vl must be 1 (scalar), 4, or 8")

    def lane_offset(self, p: int) -> int:
        off = (self.vl - 1 - p) * self.s
        if p < self.vl // 2:
            off += self.sl
        return off


@dataclass(frozen=True)
class StencilSpec:
    """Update pattern, dependence kind and boundary rule of one stencil."""

    name: str
    dim: int
    radius: int
    shape: str  # "star" | "box"
    dependence_kind: str  # "jacobi" | "gauss_seidel"
    element_kind: str = "float64"
    coefficients: Mapping[Offset, float] = field(default_factory=dict)
    birth: frozenset = frozenset()
    survive: frozenset = frozenset()
    boundary: float = 0.0

    def __post_init__(self):
        if not 1 <= self.dim <= 3:
            raise ValueError("dim must be 1..3")
        if self.radius < 1:
            raise ValueError("radius must be >= 1")
        if self.shape not in ("star", "box"):
            raise ValueError("shape must be star or box")
        if self.dependence_kind not in ("jacobi", "gauss_seidel"):
            raise ValueError("bad dependence_kind")
        if self.element_kind not in ("float64", "int32"):
            raise ValueError("bad element_kind")
        for off in self.coefficients:
            if len(off) != self.dim:
                raise ValueError(f"offset {off} has wrong arity")
            if max(abs(c) for c in off) > self.radius:
                raise ValueError(f"offset {off} exceeds radius {self.radius}")
            if self.shape == "star" and sum(1 for c in off if c) > 1:
                raise ValueError(f"offset {off} not on the star")
        if not (self.birth <= set(range(9)) and self.survive <= set(range(9))):
            raise ValueError("life rule sets must be subsets of 0..8")

    @property
    def is_life(self) -> bool:
        return bool(self.birth or self.survive)

    def offsets(self) -> list[Offset]:
        """Taps in the fixed evaluation order (sorted offsets)."""
        if self.is_life:
            return sorted(o for o in _box(self.dim, self.radius) if any(o))
        return sorted(self.coefficients)


def _box(dim: int, r: int) -> list[Offset]:
    if dim == 1:
        return [(i,) for i in range(-r, r + 1)]
    return [(i,) + rest for i in range(-r, r + 1) for rest in _box(dim - 1, r)]


def dependences(spec: StencilSpec) -> frozenset[Dependence]:
    """Every (dt, dx) pair of the update rule (reference ``model.py:142-160``)."""
    out = set()
    for off in spec.offsets():
        if spec.dependence_kind == "gauss_seidel" and _lex_negative(off):
            out.add(Dependence(0, off))
        else:
            out.add(Dependence(1, off))
    if spec.dependence_kind == "jacobi" and (0,) * spec.dim not in spec.offsets():
        out.add(Dependence(1, (0,) * spec.dim))
    return frozenset(out)


def lcs_dependences() -> frozenset[Dependence]:
    """The LCS recurrence with the A index as time (reference
    ``model.py:163-168``): lcs[x][y] reads lcs[x-1][y], lcs[x-1][y-1] and
    lcs[x][y-1]."""
    return frozenset({Dependence(1, (0,)), Dependence(1, (-1,)), Dependence(0, (-1,))})


def min_space_stride(deps: frozenset[Dependence]) -> int:
    """Smallest integer s > max{dx0/dt : dt >= 1, dx0 > 0}; 1 if none.
    (reference ``model.py:171-193``).  On the GPU this is the minimum lane lag
    of the time-skewed warp pipelines (gs1d: lane k trails lane k-1 by s)."""
    if not deps:
        raise ValueError("empty dependence set")
    best: Fraction | None = None
    for d in deps:
        if d.dt == 0:
            if not _lex_negative(d.dx):
                raise IllegalDependence(f"dt=0 dependence {d.dx} breaks the sweep order")
            continue
        if d.dx[0] > 0:
            slope = Fraction(d.dx[0], d.dt)
            best = slope if best is None or slope > best else best
    return 1 if best is None else int(best) + 1


def gs_new_taps(spec: StencilSpec, order: str = "lexicographic") -> list[bool]:
    """Per tap (in ``offsets()`` order): does the update read the value
    already produced by the *current* sweep?

    * ``lexicographic``: a true row-major in-place loop — lexicographically
      negative offsets are new (``model.py:150-156``; the reference's own
      loop test ``test_baselines.py:39-52``).
    * ``reference``: the reference oracle's anti-diagonal gather-then-scatter
      sweep (``baselines.py:83-107``): an offset is new iff its coordinate sum
      is negative.  Identical to lexicographic for star stencils; for box
      stencils the NE / SW-type taps (sum 0) read the previous sweep.
    """
    if order not in ("lexicographic", "reference"):
        raise ValueError("order must be 'lexicographic' or 'reference'")
    if order == "lexicographic":
        return [_lex_negative(o) for o in spec.offsets()]
    return [sum(o) < 0 for o in spec.offsets()]


def gs_hyperplane(spec: StencilSpec, order: str = "lexicographic"):
    """Integer wavefront ``h = a.x + tau*t`` for the in-place sweep.

    Returns ``(a, tau, simultaneous)``.  Conditions, per tap offset ``o``:

    * new tap (read after the current sweep wrote it): ``0 < -a.o < tau`` —
      the producer is on an earlier hyperplane and the next sweep's overwrite
      of that cell comes later;
    * old tap, ``o != 0``: ``0 <= a.o < tau`` — the reader runs no later than
      the current sweep's overwrite of the cell.  ``a.o == 0`` means reader and
      writer share a hyperplane; such a schedule is only valid with
      gather-then-scatter inside a hyperplane (``simultaneous=True``), which
      is exactly the reference oracle's anti-diagonal semantics
      (``baselines.py:98-107``).

    Lexicographic order always has a conflict-free solution (2D box:
    a=(2,1), tau=4; 3D box: a=(4,2,1), tau=8).  The reference order on a box
    stencil needs the simultaneous form (2D: a=(1,1), tau=3).
    """
    import itertools

    new = gs_new_taps(spec, order)
    offs = spec.offsets()
    best = None
    for a in itertools.product(range(1, 9), repeat=spec.dim):
        for tau in range(1, 40):
            ok, simul = True, False
            for off, is_new in zip(offs, new):
                ao = sum(x * y for x, y in zip(a, off))
                if not any(off):
                    continue
                if is_new:
                    ok = 0 < -ao < tau
                else:
                    ok = 0 <= ao < tau
                    simul = simul or ao == 0
                if not ok:
                    break
            if ok:
                key = (simul, tau, sum(a))
                if best is None or key < best[0]:
                    best = (key, a, tau, simul)
                break
    if best is None:
        raise IllegalDependence(f"no wavefront hyperplane for {spec.name} ({order})")
    return best[1], best[2], best[3]
