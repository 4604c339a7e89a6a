"""ctypes wrapper of the C oracle (TEST INFRASTRUCTURE ONLY, see __init__)."""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")


class Problem(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("ntaps", C.c_int32), ("extents", C.c_int64 * 3), ("shape", C.c_int64 * 3),
        ("offset", C.c_int64), ("offsets", (C.c_int32 * 3) * 27), ("coeffs", C.c_double * 27),
    ]


_lib = None


def build() -> str:
    """Compile liboracle.so (make target; gcc -ffp-contract=off -fopenmp)."""
    subprocess.run(["make", "-s", "-C", os.path.dirname(_HERE), "oracle/liboracle.so"], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        _lib = C.CDLL(_SO)
        _lib.oracle_jacobi.argtypes = [C.POINTER(Problem), C.c_void_p, C.c_void_p, C.c_int64, C.c_int]
        _lib.oracle_gauss_seidel.argtypes = [C.POINTER(Problem), C.c_void_p, C.c_int64, C.c_int, C.c_int]
        _lib.oracle_last_seconds.restype = C.c_double
    return _lib


def _problem(spec, grid) -> Problem:
    p = Problem()
    p.dim = grid.dim
    offs = spec.offsets()
    p.ntaps = len(offs)
    for d in range(3):
        p.extents[d] = grid.extents[d] if d < grid.dim else 1
        p.shape[d] = grid.data.shape[d] if d < grid.dim else 1
    p.offset = grid.offset
    for k, o in enumerate(offs):
        for d in range(3):
            p.offsets[k][d] = o[d] if d < grid.dim else 0
        p.coeffs[k] = float(spec.coefficients[o])
    return p


def scalar_reference(spec, grid, steps, order="reference", threads=0):
    """Same contract as oracle.scalar_reference, in C (Life-like int32 rules
    delegate to the NumPy restatement)."""
    if spec.is_life:
        from . import oracle as _npo

        return _npo.scalar_reference(spec, grid, steps)
    p = _problem(spec, grid)
    out = grid.copy()
    if spec.dependence_kind == "gauss_seidel":
        code = {"lexicographic": 0, "reference": 1}[order]
        rc = lib().oracle_gauss_seidel(C.byref(p), out.data.ctypes.data, int(steps), code, int(threads))
    else:
        src = np.ascontiguousarray(grid.data)
        rc = lib().oracle_jacobi(C.byref(p), src.ctypes.data, out.data.ctypes.data, int(steps), int(threads))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return out


def last_seconds() -> float:
    """Seconds the last scalar_reference call spent in its step / sweep loop
    (allocations and copies excluded): the timed CPU-baseline figure."""
    return float(lib().oracle_last_seconds())
