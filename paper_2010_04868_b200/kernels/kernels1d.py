"""1D drop-ins: heat (3-point Jacobi) and Gauss-Seidel.

Validation mirrors the reference ``_resolve`` (kernels1d.py:72-86) and the
GS in-place rule (kernels1d.py:99-100); the compute is
``jacobi1d_kernel`` (register trapezoid, csrc/jacobi1d.cu) and
``gs1d_kernel`` (time-skewed warp pipeline, csrc/gs1d.cu).

The optional ``kernel=`` keyword (an addition) selects any 1D catalog entry,
e.g. ``gs1d_temporal(g, 1000, kernel="gs1d_w343")`` for BASELINE config 2.
"""

from __future__ import annotations

from ..catalog import get as catalog_get
from ..errors import SizeError, UnsupportedError
from ..grid import Grid
from ..model import ScheduleParams
from . import KernelVariant
from ._common import check_backend, execute


def _resolve(name, grid, variant):
    entry = catalog_get(name)
    spec = entry.spec
    var = variant or KernelVariant()
    params = var.params or entry.params(var.scheme)
    if var.scheme == "two_stride" and params.sl == 0:
        params = ScheduleParams(params.s, entry.sl or 2, params.vl)
    if var.scheme == "base" and params.sl != 0:
        raise UnsupportedError("base scheme requires sl=0")
    if grid.dim != 1 or spec.dim != 1:
        raise SizeError("1D kernel on a non-1D grid")
    nx = grid.extents[0]
    if nx < params.vl * (params.s + 1) + params.sl:
        raise SizeError(f"NX={nx} below the steady-loop minimum for s={params.s}")
    return spec, var


def heat1d_temporal(grid: Grid, steps: int, variant: KernelVariant | None = None, backend=None,
                    kernel: str = "heat1d", **opts) -> Grid:
    spec, _ = _resolve(kernel, grid, variant)
    if spec.dependence_kind != "jacobi":
        raise UnsupportedError(f"{kernel} is not a Jacobi stencil")
    check_backend(backend)
    return execute(spec, grid, steps, **opts)


def gs1d_temporal(grid: Grid, steps: int, variant: KernelVariant | None = None, backend=None,
                  kernel: str = "gs1d", **opts) -> Grid:
    spec, _ = _resolve(kernel, grid, variant)
    if variant is not None and not variant.single_array:
        raise UnsupportedError("Gauss-Seidel runs in place; single_array is implied")
    if spec.dependence_kind != "gauss_seidel":
        raise UnsupportedError(f"{kernel} is not a Gauss-Seidel stencil")
    check_backend(backend)
    return execute(spec, grid, steps, **opts)
