"""2D/3D drop-ins: Jacobi (star / box) and Gauss-Seidel.

Validation mirrors the reference ``_run_nd`` (kernels_nd.py:58-76).  Compute:
``jacobi2d_kernel`` (warp strips, D time levels per HBM pass),
``jacobi3d_kernel`` (2.5D plane streaming), ``gs_wave_kernel`` (hyperplane
wavefront over all sweeps) — csrc/.

Gauss-Seidel takes an added ``order=`` keyword: ``"lexicographic"`` (the
row-major in-place loop; default) or ``"reference"`` (the reference oracle's
anti-diagonal gather/scatter, which differs for box stencils — SURVEY.md
§0.4).  Unlike the reference's ``gs2d_temporal`` (star-only, kernels_nd.py:
306-339), box Gauss-Seidel stencils are supported.
"""

from __future__ import annotations

from ..catalog import get as catalog_get
from ..errors import SizeError, UnsupportedError
from ..grid import Grid
from . import KernelVariant
from ._common import check_backend, execute


def _resolve(kernel, grid, variant, dim, gauss):
    entry = catalog_get(kernel)
    spec = entry.spec
    var = variant or KernelVariant()
    if var.scheme == "two_stride":
        raise UnsupportedError("two_stride is 1D-only")
    params = var.params or entry.params("base")
    if gauss and variant is not None and not variant.single_array:
        raise UnsupportedError("Gauss-Seidel runs in place; single_array is implied")
    if grid.dim != dim or spec.dim != dim:
        raise SizeError(f"{kernel} expects a {spec.dim}D grid")
    if grid.extents[0] < params.vl * (params.s + 1):
        raise SizeError(f"NX={grid.extents[0]} below the steady-loop minimum for s={params.s}")
    if gauss != (spec.dependence_kind == "gauss_seidel"):
        raise UnsupportedError(f"{kernel} is a {spec.dependence_kind} stencil")
    return spec


def jacobi2d_temporal(grid: Grid, steps: int, variant: KernelVariant | None = None, backend=None,
                      kernel: str = "heat2d", **opts) -> Grid:
    spec = _resolve(kernel, grid, variant, 2, False)
    check_backend(backend)
    return execute(spec, grid, steps, **opts)


def jacobi3d_temporal(grid: Grid, steps: int, variant: KernelVariant | None = None, backend=None,
                      kernel: str = "heat3d", **opts) -> Grid:
    spec = _resolve(kernel, grid, variant, 3, False)
    check_backend(backend)
    return execute(spec, grid, steps, **opts)


def gs2d_temporal(grid: Grid, steps: int, variant: KernelVariant | None = None, backend=None,
                  kernel: str = "gs2d", order: str = "lexicographic", **opts) -> Grid:
    spec = _resolve(kernel, grid, variant, 2, True)
    check_backend(backend)
    return execute(spec, grid, steps, order=order, **opts)


def gs3d_temporal(grid: Grid, steps: int, variant: KernelVariant | None = None, backend=None,
                  kernel: str = "gs3d", order: str = "lexicographic", **opts) -> Grid:
    spec = _resolve(kernel, grid, variant, 3, True)
    check_backend(backend)
    return execute(spec, grid, steps, order=order, **opts)
