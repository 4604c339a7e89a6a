"""Dispatch and the bit-exact equivalence harness.

``run_temporal`` mirrors the reference dispatcher (verify.py:51-68).
``equivalence_matrix`` mirrors verify.py:130-166 (first divergence with
both bit patterns, runner injection for fault-injection tests) but the
expected result comes from an injected ``reference`` callable — the product
package never embeds the CPU oracle; tests pass ``oracle.scalar_reference``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from .catalog import DEFAULT_CATALOG, get as catalog_get
from .grid import Grid
from .kernels import (
    KernelVariant,
    gs1d_temporal,
    gs2d_temporal,
    gs3d_temporal,
    heat1d_temporal,
    jacobi2d_temporal,
    jacobi3d_temporal,
)


def run_temporal(kernel: str, grid: Grid, steps: int, variant: KernelVariant | None = None, backend=None,
                 **opts) -> Grid:
    """Dispatch one named catalog kernel to its drop-in function."""
    if kernel.startswith("gs") and variant is not None and not variant.single_array:
        variant = KernelVariant(variant.scheme, True, variant.params)
    entry = catalog_get(kernel)
    spec = entry.spec
    gauss = spec.dependence_kind == "gauss_seidel"
    if spec.dim == 1:
        fn = gs1d_temporal if gauss else heat1d_temporal
    elif spec.dim == 2:
        fn = gs2d_temporal if gauss else jacobi2d_temporal
    else:
        fn = gs3d_temporal if gauss else jacobi3d_temporal
    return fn(grid, steps, variant, backend, kernel=kernel, **opts)


@dataclass(frozen=True)
class Cell:
    kernel: str
    scheme: str
    single_array: bool
    size: tuple
    seed: int
    steps: int

    def describe(self):
        return (f"{self.kernel}[{self.scheme}{'/1arr' if self.single_array else ''}]"
                f" size={self.size} seed={self.seed} T={self.steps}")


@dataclass
class CellResult:
    cell: Cell
    ok: bool
    position: tuple | None = None
    got_bits: str | None = None
    want_bits: str | None = None


@dataclass
class MatrixReport:
    results: list = field(default_factory=list)
    first_divergence: int | None = None

    @property
    def passed(self) -> bool:
        return self.first_divergence is None

    def as_dict(self):
        return {
            "passed": self.passed,
            "cells": len(self.results),
            "first_divergence": self.first_divergence,
            "failures": [
                {"cell": r.cell.describe(), "position": list(r.position) if r.position is not None else None,
                 "got_bits": r.got_bits, "want_bits": r.want_bits}
                for r in self.results if not r.ok
            ],
        }

    def to_json(self):
        return json.dumps(self.as_dict(), indent=1)


def _bits(value) -> str:
    return f"0x{np.float64(value).view(np.uint64):016x}"


def equivalence_matrix(cells, reference, runner=None, lcs_reference=None) -> MatrixReport:
    """Run every cell through ``runner`` (default: the GPU drop-ins) and
    compare bit-exactly with ``reference(spec, grid, steps)``; ``lcs`` cells
    (reference verify.py:136-145: two seeded 4-letter sequences) compare
    ``lcs_temporal`` with ``lcs_reference(a, b)``."""
    runner = runner or run_temporal
    report = MatrixReport()
    for idx, cell in enumerate(cells):
        if cell.kernel == "lcs":
            from .kernels import lcs_temporal

            if lcs_reference is None:
                raise ValueError("lcs cells need an lcs_reference callable")
            rng = np.random.default_rng(cell.seed)
            a = rng.integers(0, 4, size=cell.size[0], dtype=np.int32)
            b = rng.integers(0, 4, size=cell.size[1], dtype=np.int32)
            got, want = lcs_temporal(a, b), int(lcs_reference(a, b))
            res = CellResult(cell, got == want)
            if not res.ok:
                res.position = ()
                res.got_bits, res.want_bits = f"{got:08x}", f"{want:08x}"
            report.results.append(res)
            if not res.ok and report.first_divergence is None:
                report.first_divergence = idx
            continue
        entry = catalog_get(cell.kernel)
        grid = Grid.random(cell.size, seed=cell.seed, element_kind=entry.spec.element_kind, vl=entry.vl)
        got = runner(cell.kernel, grid, cell.steps, KernelVariant(cell.scheme, cell.single_array))
        want = reference(entry.spec, grid, cell.steps)
        same = got.interior == want.interior
        res = CellResult(cell, bool(same.all()))
        if not res.ok:
            pos = tuple(int(i) for i in np.argwhere(~same)[0])
            res.position = pos
            res.got_bits = _bits(got.interior[pos])
            res.want_bits = _bits(want.interior[pos])
        report.results.append(res)
        if not res.ok and report.first_divergence is None:
            report.first_divergence = idx
    return report


def default_matrix(cells_per_kernel: int = 20, master_seed: int = 2024, kernels=None) -> list:
    """Acceptance matrix in the reference's shape (verify.py:169-222): random
    cells per float64 catalog kernel (or the given ``kernels``, which may
    include ``life`` and ``lcs``) with the size remainder classes
    {0, 1, vl-1} mod 4*s*vl and every steps-mod-vl class."""
    rng = np.random.default_rng(master_seed)
    caps = {1: 4096, 2: 256, 3: 64}
    out = []
    names = kernels or [k for k, e in DEFAULT_CATALOG.items() if e.spec.element_kind == "float64"]
    for kernel in names:
        if kernel == "lcs":  # reference verify.py:184-192: one 2000x2000 cell, the rest below 800
            sizes = [(2000, 2000)] + [(int(rng.integers(1, 800)), int(rng.integers(1, 800)))
                                      for _ in range(cells_per_kernel - 1)]
            out.extend(Cell("lcs", "base", False, size, int(rng.integers(1 << 30)), size[0]) for size in sizes)
            continue
        entry = catalog_get(kernel)
        vl, s, dim = entry.vl, entry.s, entry.spec.dim
        lo = vl * (s + 1) + entry.sl + 1
        cap = caps[dim]
        period = 4 * s * vl
        schemes = ["base", "two_stride"] if dim == 1 else ["base"]
        singles = [False, True] if entry.spec.dependence_kind == "jacobi" else [True]
        for i in range(cells_per_kernel):
            n0 = cap if i == 0 else int(rng.integers(lo, cap + 1))
            if 0 < i < 4:
                n0 = max(lo, (n0 // period) * period) + (0, 1, vl - 1)[i % 3]
            size = (n0,) + tuple(int(rng.integers(max(vl, 8), cap + 1)) for _ in range(dim - 1))
            steps = int(rng.integers(1, 3 * vl + 1))
            if i % (vl + 1) < vl:
                steps = max(1, (steps // vl) * vl + i % (vl + 1))
            out.append(Cell(kernel, schemes[i % len(schemes)], singles[(i // 2) % len(singles)], size,
                            int(rng.integers(1 << 30)), steps))
    return out
