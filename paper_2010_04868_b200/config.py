"""Process-wide execution defaults of the GPU path (thread-safe).

The reference functions have no device / precision arguments; these knobs
fill that gap without changing their signatures.  Per-call keyword
arguments (``fma=``, ``depth=``, ``algo=``) override them.
"""

from __future__ import annotations

import threading
from contextlib import contextmanager
from dataclasses import dataclass, replace

from . import _native

_FMA = {"never": _native.FMA_NEVER, "exact": _native.FMA_EXACT, "allow": _native.FMA_ALLOW}
_ALGO = {"auto": _native.ALGO_AUTO, "naive": _native.ALGO_NAIVE, "blocked": _native.ALGO_BLOCKED}
_ORDER = {"lexicographic": _native.GS_LEXICOGRAPHIC, "reference": _native.GS_REFERENCE}


@dataclass(frozen=True)
class ExecConfig:
    device: int = 0
    # "exact": fuse multiply-add only for power-of-two coefficient sets, where
    # the product is exact and the result bit-identical.  The blocked 1D / 2D
    # Jacobi kernels then carry values scaled by 1 / |first coefficient| per
    # level of a temporal block (heat1d 4^64, heat2d 8^8): identical bits
    # unless a value leaves the normal range on the way (|v| beyond ~2^890,
    # or products / rescaled results that are subnormal), DESIGN.md section 1;
    # "never": always separate mul/add, unconditionally the reference's
    # arithmetic; "allow": always fuse (tolerance mode, ~1e-15 relative).
    fma: str = "exact"
    depth: int = 0  # temporal block depth (0 = kernel default)
    algo: str = "auto"
    # GPUs for 2D/3D Jacobi: axis-0 slabs on devices device .. device+n-1
    # (SURVEY.md §8e); 1D and Gauss-Seidel always run on one GPU
    n_gpus: int = 1
    # let the n_gpus shards share devices (round robin): the one-GPU test form
    emulate_shards: bool = False

    def native(self, order: str = "lexicographic", **overrides) -> _native.Exec:
        cfg = replace(self, **{k: v for k, v in overrides.items() if v is not None})
        if cfg.fma not in _FMA:
            raise ValueError(f"fma must be one of {sorted(_FMA)}")
        if cfg.algo not in _ALGO:
            raise ValueError(f"algo must be one of {sorted(_ALGO)}")
        if order not in _ORDER:
            raise ValueError(f"order must be one of {sorted(_ORDER)}")
        if cfg.depth < 0:
            raise ValueError("depth must be >= 0")
        if cfg.n_gpus < 1:
            raise ValueError("n_gpus must be >= 1")
        return _native.make_exec(cfg.device, _FMA[cfg.fma], cfg.depth, _ORDER[order], _ALGO[cfg.algo],
                                 cfg.n_gpus, cfg.emulate_shards)


_local = threading.local()
_global = ExecConfig()


def current() -> ExecConfig:
    return getattr(_local, "cfg", None) or _global


def set_default(**kw) -> ExecConfig:
    global _global
    _global = replace(_global, **kw)
    return _global


@contextmanager
def using(**kw):
    """Temporarily override the execution config for this thread."""
    prev = getattr(_local, "cfg", None)
    _local.cfg = replace(current(), **kw)
    try:
        yield _local.cfg
    finally:
        _local.cfg = prev
