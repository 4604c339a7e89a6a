"""B200-native drop-in for the stencil-run path of ``tvstencil``
(arXiv 2010.04868, "Temporal Vectorization for Stencils").

``import paper_2010_04868_b200 as tvstencil`` exposes the same names as the
reference package surface (``tvstencil/__init__.py:16-34``) for the hot
path; ``paper_2010_04868_b200.kernels`` holds the drop-in run functions,
whose compute is ``libtvstencil.so`` (hand-written sm_100a CUDA, no CPU
fallback).  The CPU SIMD-emulation layer of the reference (``vec.py``) is
out of scope.
"""

from .errors import AlignmentError, IllegalDependence, NativeError, SizeError, UnsupportedError
from .grid import Grid, fnv1a64
from .model import (
    Dependence,
    ScheduleParams,
    StencilSpec,
    dependences,
    lcs_dependences,
    gs_hyperplane,
    gs_new_taps,
    min_space_stride,
)

__all__ = [
    "AlignmentError",
    "Dependence",
    "Grid",
    "IllegalDependence",
    "NativeError",
    "ScheduleParams",
    "SizeError",
    "StencilSpec",
    "UnsupportedError",
    "dependences",
    "lcs_dependences",
    "fnv1a64",
    "gs_hyperplane",
    "gs_new_taps",
    "min_space_stride",
]

__version__ = "0.1.0"
