"""ctypes binding to ``libtvstencil.so`` (include/tvstencil.h).

This module is the FFI the drop-in functions use; INTEGRATION.md shows the
same binding as a maintainer would add it to the reference package.  There
is no CPU fallback: if the library is missing, every call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import NativeError, SizeError, UnsupportedError

_LIB_NAME = "libtvstencil.so"
_HERE = os.path.dirname(os.path.abspath(__file__))

TVS_JACOBI, TVS_GAUSS_SEIDEL = 0, 1
FMA_NEVER, FMA_EXACT, FMA_ALLOW = 0, 1, 2
GS_LEXICOGRAPHIC, GS_REFERENCE = 0, 1
ALGO_AUTO, ALGO_NAIVE, ALGO_BLOCKED = 0, 1, 2
EXEC_EMULATE_SHARDS = 1


class Stencil(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("kind", C.c_int32), ("ntaps", C.c_int32), ("radius", C.c_int32),
        ("offsets", (C.c_int32 * 3) * 27), ("coeffs", C.c_double * 27), ("boundary", C.c_double),
    ]


class Layout(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("pad_", C.c_int32), ("extents", C.c_int64 * 3),
        ("shape", C.c_int64 * 3), ("offset", C.c_int64),
    ]


class Exec(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("fma_policy", C.c_int32), ("temporal_depth", C.c_int32),
        ("gs_order", C.c_int32), ("algo", C.c_int32), ("n_gpus", C.c_int32), ("flags", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Geometry(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("pad_", C.c_int32), ("extents", C.c_int64 * 3), ("strides", C.c_int64 * 3),
        ("origin", C.c_int64), ("alloc_elems", C.c_int64), ("axis0_offset", C.c_int64),
        ("axis0_global", C.c_int64),
    ]


class LifeRule(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("ntaps", C.c_int32), ("offsets", (C.c_int32 * 3) * 26),
        ("birth_mask", C.c_int32), ("survive_mask", C.c_int32), ("boundary", C.c_int32), ("pad_", C.c_int32),
    ]


class Problem(C.Structure):
    """tvs_problem (the SURVEY.md §8(b) problem-struct form)."""
    _fields_ = [
        ("dim", C.c_int32), ("ntaps", C.c_int32), ("extents", C.c_int64 * 3), ("radius", C.c_int32),
        ("pad_", C.c_int32), ("boundary", C.c_double), ("offsets", (C.c_int32 * 3) * 27),
        ("coeffs", C.c_double * 27), ("padded_shape", C.c_int64 * 3), ("offset", C.c_int64),
    ]


class ShardHandle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 256)]


class TileDesc(C.Structure):
    _fields_ = [
        ("t0", C.c_int32), ("t1", C.c_int32), ("lo", C.c_int32 * 3), ("hi", C.c_int32 * 3),
        ("slope_lo", C.c_int32 * 3), ("slope_hi", C.c_int32 * 3),
    ]


# exported symbols with their argtypes (checked by tests/test_native_abi.py
# against include/tvstencil.h)
_P = C.c_void_p
_SIGS = {
    "tvs_run": (C.c_int, [C.POINTER(Stencil), C.POINTER(Layout), _P, _P, C.c_int64, C.POINTER(Exec)]),
    "tvs_jacobi": (C.c_int, [C.POINTER(Problem), _P, _P, C.c_int64, C.POINTER(Exec)]),
    "tvs_gauss_seidel": (C.c_int, [C.POINTER(Problem), _P, C.c_int64, C.c_int32, C.POINTER(Exec)]),
    "tvs_plan_create": (C.c_int, [C.POINTER(Stencil), C.c_int32, C.POINTER(C.c_int64), C.POINTER(Exec), C.POINTER(_P)]),
    "tvs_plan_upload": (C.c_int, [_P, C.POINTER(Layout), _P]),
    "tvs_plan_download": (C.c_int, [_P, C.POINTER(Layout), _P]),
    "tvs_plan_run": (C.c_int, [_P, C.c_int64]),
    "tvs_plan_synchronize": (C.c_int, [_P]),
    "tvs_plan_last_ms": (C.c_int, [_P, C.POINTER(C.c_float)]),
    "tvs_plan_last_launches": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "tvs_plan_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "tvs_plan_destroy": (C.c_int, [_P]),
    "tvs_geometry_init": (C.c_int, [C.c_int32, C.POINTER(C.c_int64), C.c_int64, C.c_int64, C.POINTER(Geometry)]),
    "tvs_fill_halo": (C.c_int, [C.POINTER(Geometry), _P, C.c_double, _P]),
    "tvs_jacobi_device": (C.c_int, [C.POINTER(Stencil), C.POINTER(Geometry), _P, _P, C.c_int64, C.POINTER(Exec), _P,
                                    C.POINTER(C.c_int32)]),
    "tvs_jacobi_device_rows": (C.c_int, [C.POINTER(Stencil), C.POINTER(Geometry), _P, _P, C.c_int64, C.POINTER(Exec), _P,
                                         C.c_int64, C.c_int64]),
    "tvs_gauss_seidel_device": (C.c_int, [C.POINTER(Stencil), C.POINTER(Geometry), _P, C.c_int64, C.POINTER(Exec), _P]),
    "tvs_upload": (C.c_int, [C.POINTER(Geometry), _P, C.POINTER(Layout), _P, _P]),
    "tvs_download": (C.c_int, [C.POINTER(Geometry), _P, C.POINTER(Layout), _P, _P]),
    "tvs_last_error": (C.c_char_p, []),
    "tvs_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "tvs_host_register": (C.c_int, [_P, C.c_size_t]),
    "tvs_host_unregister": (C.c_int, [_P]),
    "tvs_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "tvs_host_free": (C.c_int, [_P]),
    "tvs_fnv1a64": (C.c_uint64, [_P, C.c_size_t, C.c_uint64]),
    "tvs_life_run": (C.c_int, [C.POINTER(LifeRule), C.POINTER(Layout), _P, _P, C.c_int64, C.POINTER(Exec)]),
    "tvs_life_device": (C.c_int, [C.POINTER(LifeRule), C.POINTER(Geometry), _P, _P, C.c_int64, C.POINTER(Exec), _P,
                                  C.POINTER(C.c_int32)]),
    "tvs_fill_halo_i32": (C.c_int, [C.POINTER(Geometry), _P, C.c_int32, _P]),
    "tvs_upload_i32": (C.c_int, [C.POINTER(Geometry), _P, C.POINTER(Layout), _P, _P]),
    "tvs_download_i32": (C.c_int, [C.POINTER(Geometry), _P, C.POINTER(Layout), _P, _P]),
    "tvs_lcs": (C.c_int, [_P, C.c_int64, _P, C.c_int64, C.POINTER(Exec), C.POINTER(C.c_int64)]),
    "tvs_lcs_device": (C.c_int, [_P, C.c_int64, _P, C.c_int64, _P, _P]),
    "tvs_tiled_run": (C.c_int, [C.POINTER(Stencil), C.POINTER(Layout), _P, _P, C.c_int64, C.POINTER(TileDesc),
                                C.POINTER(C.c_int64), C.c_int64, C.POINTER(Exec)]),
    "tvs_tiled_life": (C.c_int, [C.POINTER(LifeRule), C.POINTER(Layout), _P, _P, C.c_int64, C.POINTER(TileDesc),
                                 C.POINTER(C.c_int64), C.c_int64, C.POINTER(Exec)]),
    "tvs_lcs_tiled": (C.c_int, [_P, C.c_int64, _P, C.c_int64, C.POINTER(TileDesc), C.POINTER(C.c_int64), C.c_int64,
                                C.POINTER(Exec), C.POINTER(C.c_int64)]),
    "tvs_shard_create": (C.c_int, [C.POINTER(Stencil), C.c_int32, C.POINTER(C.c_int64), C.c_int32, C.c_int32,
                                   C.POINTER(Exec), C.POINTER(_P)]),
    "tvs_shard_info": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                 C.POINTER(C.c_int32)]),
    "tvs_shard_export": (C.c_int, [_P, C.POINTER(ShardHandle)]),
    "tvs_shard_connect": (C.c_int, [_P, C.POINTER(ShardHandle), C.POINTER(ShardHandle)]),
    "tvs_shard_connect_local": (C.c_int, [_P, _P, _P]),
    "tvs_shard_upload": (C.c_int, [_P, C.POINTER(Layout), _P]),
    "tvs_shard_download": (C.c_int, [_P, C.POINTER(Layout), _P]),
    "tvs_shard_run": (C.c_int, [_P, C.c_int64]),
    "tvs_shard_synchronize": (C.c_int, [_P]),
    "tvs_shard_last_ms": (C.c_int, [_P, C.POINTER(C.c_float)]),
    "tvs_shard_last_launches": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "tvs_shard_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "tvs_shard_destroy": (C.c_int, [_P]),
    "tvs_launch_counter": (C.c_int64, []),
    "tvs_release_thread_cache": (C.c_int, []),
    "tvs_version": (C.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return os.environ.get("TVSTENCIL_LIB", os.path.join(_HERE, _LIB_NAME))


def lib():
    """Load libtvstencil.so once; raise loudly if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = library_path()
            if not os.path.exists(path):
                raise ImportError(
                    f"{path} not found: build the CUDA library first "
                    "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
            handle = C.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = lib().tvs_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == 1:
        raise SizeError(text)
    if rc == 2:
        raise UnsupportedError(text)
    if rc == 3:
        raise ValueError(text)
    raise NativeError(text)


def device_count() -> int:
    n = C.c_int32(0)
    lib().tvs_device_count(C.byref(n))
    return int(n.value)


def fnv1a64(view, state: int) -> int:
    buf = np.frombuffer(view, dtype=np.uint8)
    return int(lib().tvs_fnv1a64(buf.ctypes.data, buf.size, C.c_uint64(state)))


def make_stencil(spec, boundary=None) -> Stencil:
    """StencilSpec -> tvs_stencil, taps in ``spec.offsets()`` order.

    ``boundary``: the Dirichlet value of every non-interior cell.  The
    reference kernels take it from the grid, not the spec (kernels1d.py:115,
    kernels_nd.py:90, baselines.py:113-119 read the grid's halo), so the
    drop-ins pass ``grid.boundary``; ``spec.boundary`` is the fallback."""
    st = Stencil()
    offs = spec.offsets()
    if spec.element_kind != "float64" or spec.is_life:
        raise UnsupportedError(f"{spec.name}: only float64 linear stencils run on the GPU path")
    if len(offs) == 0 or len(offs) > 27:
        raise UnsupportedError(f"{spec.name}: needs 1..27 taps")
    st.dim = spec.dim
    st.kind = TVS_GAUSS_SEIDEL if spec.dependence_kind == "gauss_seidel" else TVS_JACOBI
    st.ntaps = len(offs)
    st.radius = spec.radius
    for k, off in enumerate(offs):
        for d in range(3):
            st.offsets[k][d] = off[d] if d < spec.dim else 0
        st.coeffs[k] = float(spec.coefficients[off])
    st.boundary = float(spec.boundary if boundary is None else boundary)
    return st


def make_life_rule(spec, boundary=None) -> LifeRule:
    """Life-like StencilSpec (``is_life``) -> tvs_life_rule, neighbours in
    ``spec.offsets()`` order (model.py: the box minus the centre)."""
    if not spec.is_life:
        raise UnsupportedError(f"{spec.name} is not a Life-like rule")
    offs = spec.offsets()
    if spec.radius != 1 or not 1 <= len(offs) <= 26:
        raise UnsupportedError(f"{spec.name}: only radius-1 Life rules run on the GPU path")
    r = LifeRule()
    r.dim, r.ntaps = spec.dim, len(offs)
    for k, off in enumerate(offs):
        for d in range(3):
            r.offsets[k][d] = off[d] if d < spec.dim else 0
    r.birth_mask = sum(1 << int(v) for v in spec.birth)
    r.survive_mask = sum(1 << int(v) for v in spec.survive)
    r.boundary = int(spec.boundary if boundary is None else boundary)
    return r


def life_run(spec, src: np.ndarray, dst: np.ndarray, extents, offset: int, steps: int, ex: Exec,
             boundary=None) -> None:
    """int32 host Grid data in -> host Grid data out."""
    rule = make_life_rule(spec, boundary)
    for a in (src, dst):
        if a.dtype != np.int32 or not a.flags.c_contiguous:
            raise ValueError("Life grid data must be a C-contiguous int32 array")
    lay = make_layout(src, extents, offset)
    check(lib().tvs_life_run(C.byref(rule), C.byref(lay), src.ctypes.data, dst.ctypes.data, int(steps), C.byref(ex)),
          f"tvs_life_run({spec.name})")


def lcs(a: np.ndarray, b: np.ndarray, ex: Exec) -> int:
    a = np.ascontiguousarray(a, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=np.int32)
    n = C.c_int64(0)
    check(lib().tvs_lcs(a.ctypes.data if a.size else None, a.size, b.ctypes.data if b.size else None, b.size,
                        C.byref(ex), C.byref(n)), "tvs_lcs")
    return int(n.value)


def make_layout(data: np.ndarray, extents, offset: int) -> Layout:
    lay = Layout()
    lay.dim = data.ndim
    for d in range(data.ndim):
        lay.extents[d] = int(extents[d])
        lay.shape[d] = int(data.shape[d])
    for d in range(data.ndim, 3):
        lay.extents[d] = 1
        lay.shape[d] = 1
    lay.offset = int(offset)
    return lay


def make_exec(device=0, fma_policy=FMA_EXACT, temporal_depth=0, gs_order=GS_LEXICOGRAPHIC, algo=ALGO_AUTO,
              n_gpus=1, emulate_shards=False) -> Exec:
    ex = Exec()
    ex.device, ex.fma_policy, ex.temporal_depth = int(device), int(fma_policy), int(temporal_depth)
    ex.gs_order, ex.algo = int(gs_order), int(algo)
    ex.n_gpus = int(n_gpus)
    ex.flags = EXEC_EMULATE_SHARDS if emulate_shards else 0
    return ex


def _host_array(a: np.ndarray) -> np.ndarray:
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise ValueError("grid data must be a C-contiguous float64 array")
    return a


def run(spec, src: np.ndarray, dst: np.ndarray, extents, offset: int, steps: int, ex: Exec,
        boundary=None) -> None:
    """Host Grid data in -> host Grid data out (``src is dst`` allowed)."""
    st = make_stencil(spec, boundary)
    _host_array(src)
    _host_array(dst)
    lay = make_layout(src, extents, offset)
    check(lib().tvs_run(C.byref(st), C.byref(lay), src.ctypes.data, dst.ctypes.data, int(steps), C.byref(ex)),
          f"tvs_run({spec.name})")


def make_problem(spec, grid) -> Problem:
    """StencilSpec + Grid -> tvs_problem (offsets() order, the grid's boundary)."""
    st = make_stencil(spec, grid.boundary)
    p = Problem()
    p.dim, p.ntaps, p.radius, p.boundary = st.dim, st.ntaps, st.radius, st.boundary
    for k in range(st.ntaps):
        for d in range(3):
            p.offsets[k][d] = st.offsets[k][d]
        p.coeffs[k] = st.coeffs[k]
    for d in range(3):
        p.extents[d] = grid.extents[d] if d < grid.dim else 1
        p.padded_shape[d] = grid.data.shape[d] if d < grid.dim else 1
    p.offset = grid.offset
    return p


class Plan:
    """Device-resident run plan (``tvs_plan_*``): upload once, run many,
    time with CUDA events on the plan stream."""

    def __init__(self, spec, extents, ex: Exec):
        self.spec = spec
        self.extents = tuple(int(e) for e in extents)
        self._st = make_stencil(spec)
        self._ex = ex
        ext = (C.c_int64 * 3)(*(list(self.extents) + [1] * (3 - len(self.extents))))
        h = C.c_void_p()
        check(lib().tvs_plan_create(C.byref(self._st), len(self.extents), ext, C.byref(ex), C.byref(h)),
              "tvs_plan_create")
        self._h = h

    def upload(self, data: np.ndarray, offset: int):
        lay = make_layout(_host_array(data), self.extents, offset)
        check(lib().tvs_plan_upload(self._h, C.byref(lay), data.ctypes.data), "tvs_plan_upload")

    def download(self, data: np.ndarray, offset: int):
        lay = make_layout(_host_array(data), self.extents, offset)
        check(lib().tvs_plan_download(self._h, C.byref(lay), data.ctypes.data), "tvs_plan_download")

    def run(self, steps: int):
        check(lib().tvs_plan_run(self._h, int(steps)), "tvs_plan_run")

    def synchronize(self):
        check(lib().tvs_plan_synchronize(self._h), "tvs_plan_synchronize")

    def last_ms(self) -> float:
        ms = C.c_float(0)
        check(lib().tvs_plan_last_ms(self._h, C.byref(ms)), "tvs_plan_last_ms")
        return float(ms.value)

    def last_launches(self) -> int:
        n = C.c_int64(0)
        check(lib().tvs_plan_last_launches(self._h, C.byref(n)), "tvs_plan_last_launches")
        return int(n.value)

    def stream_handle(self) -> int:
        s = C.c_void_p()
        check(lib().tvs_plan_stream(self._h, C.byref(s)), "tvs_plan_stream")
        return int(s.value or 0)

    def close(self):
        if getattr(self, "_h", None):
            lib().tvs_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Shard:
    """One axis-0 slab of a sharded 2D/3D Jacobi grid (``tvs_shard_*``,
    csrc/shard.cu): ``index`` of ``n_shards``, on ``ex.device``.  Neighbours
    are connected in-process (:meth:`connect_local`) or across processes by
    CUDA IPC handles (:meth:`export` / :meth:`connect`); the kernels store
    the neighbour's ghost rows straight into its buffer (fused halo
    exchange over peer memory)."""

    def __init__(self, spec, global_extents, n_shards: int, index: int, ex: Exec, boundary=None):
        self.spec = spec
        self.extents = tuple(int(e) for e in global_extents)
        self._st = make_stencil(spec, boundary)
        ext = (C.c_int64 * 3)(*(list(self.extents) + [1] * (3 - len(self.extents))))
        h = C.c_void_p()
        check(lib().tvs_shard_create(C.byref(self._st), len(self.extents), ext, int(n_shards), int(index),
                                     C.byref(ex), C.byref(h)), "tvs_shard_create")
        self._h = h
        self.index, self.n_shards = int(index), int(n_shards)
        r0, r1, g, dev = C.c_int64(), C.c_int64(), C.c_int32(), C.c_int32()
        check(lib().tvs_shard_info(h, C.byref(r0), C.byref(r1), C.byref(g), C.byref(dev)), "tvs_shard_info")
        self.rows = (int(r0.value), int(r1.value))
        self.ghost, self.device = int(g.value), int(dev.value)

    def export(self) -> bytes:
        hd = ShardHandle()
        check(lib().tvs_shard_export(self._h, C.byref(hd)), "tvs_shard_export")
        return bytes(hd.bytes)

    def connect(self, left: bytes | None, right: bytes | None):
        def mk(b):
            if b is None:
                return None
            hd = ShardHandle()
            C.memmove(hd.bytes, b, len(hd.bytes))
            return C.byref(hd)
        check(lib().tvs_shard_connect(self._h, mk(left), mk(right)), "tvs_shard_connect")

    def connect_local(self, left: "Shard | None", right: "Shard | None"):
        check(lib().tvs_shard_connect_local(self._h, left._h if left else None, right._h if right else None),
              "tvs_shard_connect_local")

    def upload(self, data: np.ndarray, offset: int):
        lay = make_layout(_host_array(data), self.extents, offset)
        check(lib().tvs_shard_upload(self._h, C.byref(lay), data.ctypes.data), "tvs_shard_upload")

    def download(self, data: np.ndarray, offset: int):
        lay = make_layout(_host_array(data), self.extents, offset)
        check(lib().tvs_shard_download(self._h, C.byref(lay), data.ctypes.data), "tvs_shard_download")

    def run(self, steps: int):
        check(lib().tvs_shard_run(self._h, int(steps)), "tvs_shard_run")

    def synchronize(self):
        check(lib().tvs_shard_synchronize(self._h), "tvs_shard_synchronize")

    def last_ms(self) -> float:
        ms = C.c_float(0)
        check(lib().tvs_shard_last_ms(self._h, C.byref(ms)), "tvs_shard_last_ms")
        return float(ms.value)

    def last_launches(self) -> int:
        n = C.c_int64(0)
        check(lib().tvs_shard_last_launches(self._h, C.byref(n)), "tvs_shard_last_launches")
        return int(n.value)

    def stream_handle(self) -> int:
        s = C.c_void_p()
        check(lib().tvs_shard_stream(self._h, C.byref(s)), "tvs_shard_stream")
        return int(s.value or 0)

    def close(self):
        if getattr(self, "_h", None):
            lib().tvs_shard_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def geometry(dim: int, extents, axis0_offset: int = 0, axis0_global: int = 0) -> Geometry:
    g = Geometry()
    ext = (C.c_int64 * 3)(*(list(extents) + [1] * (3 - len(extents))))
    check(lib().tvs_geometry_init(dim, ext, int(axis0_offset), int(axis0_global), C.byref(g)), "tvs_geometry_init")
    return g


def host_register(a: np.ndarray):
    check(lib().tvs_host_register(a.ctypes.data, a.nbytes), "tvs_host_register")


def host_unregister(a: np.ndarray):
    check(lib().tvs_host_unregister(a.ctypes.data), "tvs_host_unregister")


class _HostAlloc:
    """Owner of one tvs_host_alloc block; freed when the last array view of
    it is collected."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        check(lib().tvs_host_alloc(nbytes, C.byref(p)), "tvs_host_alloc")
        self.ptr, self.nbytes = p.value, nbytes
        self._free = lib().tvs_host_free

    def __del__(self):
        if self.ptr:
            self._free(self.ptr)
            self.ptr = None


def host_empty(shape, dtype=np.float64) -> np.ndarray:
    """Uninitialised page-locked (cudaHostAlloc) numpy array."""
    shape = tuple(int(x) for x in np.atleast_1d(shape))
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    owner = _HostAlloc(nbytes)
    raw = (C.c_char * max(nbytes, 1)).from_address(owner.ptr)
    raw._tvs_owner = owner  # the array's base keeps the allocation alive
    return np.frombuffer(raw, dtype=dt, count=int(np.prod(shape))).reshape(shape)


class _HostPool:
    """Caching allocator of page-locked host blocks for result Grids (like a
    framework's caching host allocator): a block returns to the pool when the
    last array view of it is collected and is handed out again to the next
    result of the same size, so the stock drop-in call writes its result by
    DMA into pre-faulted page-locked memory instead of faulting in fresh
    pageable pages (config 3: ~220 ms of page faults, tools/stock_probe.py).
    At most `keep` idle blocks per size are retained."""

    def __init__(self, keep: int = 2):
        self.keep = keep
        self.free: dict[int, list[int]] = {}
        self.lock = threading.Lock()

    def take(self, nbytes: int) -> int:
        with self.lock:
            lst = self.free.get(nbytes)
            if lst:
                return lst.pop()
        p = C.c_void_p()
        check(lib().tvs_host_alloc(nbytes, C.byref(p)), "tvs_host_alloc")
        return p.value

    def give(self, nbytes: int, ptr: int) -> None:
        with self.lock:
            lst = self.free.setdefault(nbytes, [])
            if len(lst) < self.keep:
                lst.append(ptr)
                return
        lib().tvs_host_free(ptr)

    def clear(self) -> None:
        with self.lock:
            blocks = [p for lst in self.free.values() for p in lst]
            self.free.clear()
        for ptr in blocks:
            lib().tvs_host_free(ptr)


_pool = _HostPool()


class _PoolLoan:
    def __init__(self, nbytes: int):
        self.nbytes = nbytes
        self.ptr = _pool.take(nbytes)

    def __del__(self):
        if self.ptr:
            try:
                _pool.give(self.nbytes, self.ptr)
            except Exception:
                pass
            self.ptr = None


def host_pool_empty(shape, dtype=np.float64) -> np.ndarray:
    """Uninitialised page-locked array from the result-buffer pool."""
    shape = tuple(int(x) for x in np.atleast_1d(shape))
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    loan = _PoolLoan(max(nbytes, 1))
    raw = (C.c_char * max(nbytes, 1)).from_address(loan.ptr)
    raw._tvs_owner = loan
    return np.frombuffer(raw, dtype=dt, count=int(np.prod(shape))).reshape(shape)


def clear_host_pool() -> None:
    _pool.clear()


def host_array(n: int) -> np.ndarray:
    """1-D page-locked float64 array of n elements (tools/pinned_probe.py)."""
    return host_empty((n,))


def release_thread_cache() -> None:
    """Free this thread's cached device buffers (see tvs_release_thread_cache)."""
    check(lib().tvs_release_thread_cache(), "tvs_release_thread_cache")


def launch_counter() -> int:
    return int(lib().tvs_launch_counter())
