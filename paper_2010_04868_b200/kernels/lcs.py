"""LCS drop-in (reference ``tvstencil/kernels/lcs.py:32``): the length of the
longest common subsequence of two int32 sequences, computed by the time-lane
warp pipeline ``lcs_kernel`` (csrc/integer.cu) through ``tvs_lcs``.

Same signature and result as the reference ``lcs_temporal(a, b,
backend=None) -> int``; an instrumented CountingBackend is rejected like
every other GPU drop-in (no emulated SIMD backend exists on this path)."""

from __future__ import annotations

import numpy as np

from .. import _native, config
from ._common import check_backend


def lcs_temporal(a, b, backend=None) -> int:
    """LCS length of integer sequences ``a`` and ``b``."""
    check_backend(backend)
    a = np.asarray(a, dtype=np.int32).ravel()
    b = np.asarray(b, dtype=np.int32).ravel()
    if a.size == 0 or b.size == 0:
        return 0
    return _native.lcs(a, b, config.current().native())
