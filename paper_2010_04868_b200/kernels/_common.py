"""Shared body of the drop-in functions: validation parity + native call."""

from __future__ import annotations

from .. import _native, config
from ..errors import UnsupportedError
from ..grid import Grid


def check_backend(backend) -> None:
    """The reference takes a CPU SIMD-emulation backend (vec.py:99, 319).
    An instrumented CountingBackend cannot observe GPU instructions, so it is
    rejected; a plain SimdBackend (or None) is accepted and ignored."""
    if backend is None:
        return
    if hasattr(backend, "counters") or type(backend).__name__ == "CountingBackend":
        raise UnsupportedError("CountingBackend instrumentation is CPU-only; the GPU path has no emulated backend")


def execute(spec, grid: Grid, steps: int, *, order: str = "lexicographic", out: Grid | None = None,
            fma: str | None = None, depth: int | None = None, algo: str | None = None,
            n_gpus: int | None = None) -> Grid:
    """Run ``steps`` updates of ``spec`` on the GPU; never mutates ``grid``."""
    steps = int(steps)
    if steps < 0:
        raise ValueError("steps must be >= 0")
    if spec.is_life:
        if grid.element_kind != "int32":
            raise UnsupportedError(f"{spec.name}: Life rules run on int32 grids")
    elif grid.element_kind != "float64":
        raise UnsupportedError(f"{spec.name}: {grid.element_kind} grids are not on the GPU path")
    if out is None:
        # the reference returns grid.copy() with the interior advanced; only
        # the frame is copied here (the device writes the whole interior)
        out = grid.copy() if steps == 0 else grid.result_like()
    else:
        if out.extents != grid.extents or out.data.shape != grid.data.shape or out.offset != grid.offset:
            raise ValueError("out= grid must have the geometry of the input grid")
        if out is not grid and steps == 0:
            out.data[...] = grid.data
    if steps == 0:
        return out
    ex = config.current().native(order=order, fma=fma, depth=depth, algo=algo, n_gpus=n_gpus)
    if spec.is_life:
        _native.life_run(spec, grid.data, out.data, grid.extents, grid.offset, steps, ex, boundary=grid.boundary)
    else:
        # Dirichlet value from the grid (kernels1d.py:115, kernels_nd.py:90)
        _native.run(spec, grid.data, out.data, grid.extents, grid.offset, steps, ex, boundary=grid.boundary)
    return out
