"""Exception types of the drop-in surface.

Same names and base class as the reference (``tvstencil/errors.py:4-17``) so
``except SizeError`` in caller code keeps working after the switch.  Native
status codes from ``libtvstencil.so`` map onto these in ``_native.py``.
"""


class AlignmentError(ValueError):
    """Index not aligned to the vector length (kept for API parity)."""


class SizeError(ValueError):
    """Grid too small / dimension mismatch for the requested kernel."""


class UnsupportedError(ValueError):
    """Kernel, variant or backend combination the GPU path does not run."""


class IllegalDependence(ValueError):
    """A same-time dependence that no lane lag can legalise."""


class NativeError(RuntimeError):
    """CUDA-side failure reported by libtvstencil.so (status 4/5)."""
