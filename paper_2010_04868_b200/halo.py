"""Slab decomposition + halo exchange for sharded Jacobi (K7).

The reference has no distributed path; BASELINE configs 3 and 5
shard Jacobi along axis 0 ("rows" / "z-slabs") across the GPUs of one node.
One process per GPU; ``torch.distributed`` (NCCL over NVLink, or gloo on
CPU for tests) moves the halos:

* rank r owns global axis-0 rows [r0, r1) (balanced split) and holds
  ``ghost`` extra rows on each side — its local block is rows
  [r0 - ghost, r1 + ghost) in the library's device layout
  (``tvs_geometry``: axis-0 rows are contiguous slabs of ``strides[0]``
  elements, so a halo is one contiguous slice, no packing);
* every ``ghost`` time steps the ranks swap their outermost ``ghost`` owned
  rows (grouped isend/irecv with rank-1 and rank+1), then advance ``ghost``
  steps with the temporally blocked kernel — the halo width equals the
  temporal block depth, so one exchange per HBM pass;
* rows outside the global domain are pinned to the boundary by the kernel
  (``axis0_offset`` / ``axis0_global``), so edge ranks need no special case.

Every point is computed by the same expression on every rank count, so the
result is bit-identical for any world size (tests/test_halo_cpu.py,
tests/test_gpu_parity.py).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _native


def split_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of n rows: the first n % world ranks get one more."""
    base, extra = divmod(n, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


@dataclass
class SlabLayout:
    rank: int
    world: int
    r0: int
    r1: int
    ghost: int
    extents: tuple  # local extents (axis 0 includes 2*ghost)
    geometry: _native.Geometry

    @property
    def n_own(self) -> int:
        return self.r1 - self.r0

    @property
    def row_elems(self) -> int:
        return int(self.geometry.strides[0])

    def row_slice(self, local_row: int, count: int) -> slice:
        """Flat element range of local axis-0 rows [local_row, local_row+count)
        including their pads (row r lives at [(r+1)*s0, (r+2)*s0))."""
        s0 = self.row_elems
        return slice((local_row + 1) * s0, (local_row + 1 + count) * s0)


def make_layout(global_extents, world: int, rank: int, ghost: int) -> SlabLayout:
    g0 = int(global_extents[0])
    r0, r1 = split_rows(g0, world, rank)
    if world > 1 and r1 - r0 < ghost:
        raise ValueError(f"rank {rank} owns {r1 - r0} rows < ghost depth {ghost}; use fewer ranks or a smaller depth")
    ext = (r1 - r0 + 2 * ghost,) + tuple(int(e) for e in global_extents[1:])
    geo = _native.geometry(len(ext), ext, axis0_offset=r0 - ghost, axis0_global=g0)
    return SlabLayout(rank, world, r0, r1, ghost, ext, geo)


class _StagedRecv:
    """A gloo request on a host copy of a device slice: copies the received
    rows back to the device slice when waited on (gloo moves host tensors
    only; NCCL moves the device rows directly)."""

    def __init__(self, req, host, dev):
        self.req, self.host, self.dev = req, host, dev

    def wait(self):
        self.req.wait()
        if self.dev is not None:
            self.dev.copy_(self.host)


def exchange(lay: SlabLayout, buf, dist, group=None, wait: bool = True):
    """Swap halos: my first `ghost` owned rows -> rank-1's bottom ghosts,
    my last `ghost` owned rows -> rank+1's top ghosts (one grouped batch).
    ``wait=False`` returns the outstanding requests instead of waiting (the
    overlapped pass waits after launching the interior rows).  Device
    buffers on a gloo group are staged through host memory."""
    if lay.world == 1 or lay.ghost == 0:
        return []
    g, n = lay.ghost, lay.n_own
    staged = getattr(buf, "is_cuda", False) and dist.get_backend(group) == "gloo"
    ops, back = [], []

    def send(sl, peer):
        t = buf[sl]
        if staged:
            t = t.cpu()  # synchronous device -> host copy of the rows
        ops.append(dist.P2POp(dist.isend, t, peer, group))
        back.append(None)

    def recv(sl, peer):
        t = buf[sl]
        host = t.cpu() if staged else t
        ops.append(dist.P2POp(dist.irecv, host, peer, group))
        back.append(t if staged else None)

    if lay.rank > 0:
        send(lay.row_slice(g, g), lay.rank - 1)
        recv(lay.row_slice(0, g), lay.rank - 1)
    if lay.rank < lay.world - 1:
        send(lay.row_slice(n, g), lay.rank + 1)
        recv(lay.row_slice(n + g, g), lay.rank + 1)
    reqs = dist.batch_isend_irecv(ops)
    if staged:
        reqs = [_StagedRecv(r, op.tensor, dev) for r, op, dev in zip(reqs, ops, back)]
    if not wait:
        return reqs
    for req in reqs:
        req.wait()
    return []


class ShardedJacobi:
    """Jacobi on this rank's slab; ``step_fn(lay, src, dst, k)`` advances k
    steps src -> dst (default: the CUDA library on torch device tensors)."""

    def __init__(self, spec, global_extents, dist, depth: int = 8, device=None, step_fn=None, group=None,
                 dtype=None, rows_fn=None, overlap: bool = True):
        import torch

        self.spec = spec
        self.dist = dist
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.layout = make_layout(global_extents, world, rank, depth)
        self.depth = depth
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        n = int(self.layout.geometry.alloc_elems)
        self.bufs = [torch.full((n,), float(spec.boundary), dtype=torch.float64, device=self.device)
                     for _ in range(2)]
        self.cur = 0
        self.step_fn = step_fn or self._cuda_step
        # rows_fn(lay, src, dst, k, lo, hi): one k-step pass writing only local
        # axis-0 rows [lo, hi) — lets the halo exchange overlap the interior
        self.rows_fn = rows_fn if rows_fn is not None else (self._cuda_rows if step_fn is None else None)
        self.overlap = overlap
        self._st = _native.make_stencil(spec) if step_fn is None else None
        self.launches = 0

    # -- data movement --------------------------------------------------------
    def load_global(self, interior):
        """Copy this rank's rows (+ ghosts inside the domain) of a global
        interior array (numpy / torch, shape = global extents) into buf."""
        import torch

        lay = self.layout
        lo = max(lay.r0 - lay.ghost, 0)
        hi = min(lay.r1 + lay.ghost, int(self.layout.geometry.axis0_global))
        view = self.interior_view(self.cur)
        src = torch.as_tensor(interior[lo:hi])
        view[lo - (lay.r0 - lay.ghost): hi - (lay.r0 - lay.ghost)] = src.to(view.device)

    def interior_view(self, which=None):
        """Interior of buffer `which` as an (e0, e1[, e2]) strided view."""
        lay = self.layout
        g = lay.geometry
        buf = self.bufs[self.cur if which is None else which]
        dim = g.dim
        sizes = tuple(int(g.extents[d]) for d in range(dim))
        strides = tuple(int(g.strides[d]) for d in range(dim))
        return buf.as_strided(sizes, strides, int(g.origin))

    def owned(self):
        """This rank's owned rows of the current field (view)."""
        lay = self.layout
        return self.interior_view()[lay.ghost: lay.ghost + lay.n_own]

    # -- stepping -------------------------------------------------------------
    def _cuda_step(self, lay, src, dst, k):
        import torch

        ex = _native.make_exec(device=src.device.index or 0)
        in_dst = C.c_int32(0)
        stream = torch.cuda.current_stream(src.device).cuda_stream
        _native.check(_native.lib().tvs_jacobi_device(
            C.byref(self._st), C.byref(lay.geometry), C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
            int(k), C.byref(ex), C.c_void_p(stream), C.byref(in_dst)), "tvs_jacobi_device")
        return bool(in_dst.value)

    def _cuda_rows(self, lay, src, dst, k, lo, hi):
        import torch

        ex = _native.make_exec(device=src.device.index or 0)
        stream = torch.cuda.current_stream(src.device).cuda_stream
        _native.check(_native.lib().tvs_jacobi_device_rows(
            C.byref(self._st), C.byref(lay.geometry), C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
            int(k), C.byref(ex), C.c_void_p(stream), int(lo), int(hi)), "tvs_jacobi_device_rows")

    def _max_pass(self) -> int:
        """Levels one ranged launch can advance (2D kernel depth, 3D two)."""
        return 12 if self.layout.geometry.dim == 2 else 2

    def run(self, steps: int) -> None:
        lay = self.layout
        g, n = lay.ghost, lay.n_own
        done = 0
        while done < steps:
            k = min(self.depth, steps - done)
            src, dst = self.bufs[self.cur], self.bufs[1 - self.cur]
            if self.overlap and self.rows_fn is not None and lay.world > 1 and k <= min(g, self._max_pass()):
                # owned rows are local [g, g+n); rows [g+k, g+n-k) read only
                # owned rows, so they run while the halos are in flight; the
                # k rows at each edge run once the new ghosts have landed.
                # Ghost rows are not recomputed: the next exchange refills them.
                reqs = exchange(lay, src, self.dist, self.group, wait=False)
                if n - 2 * k > 0:
                    self.rows_fn(lay, src, dst, k, g + k, g + n - k)
                for req in reqs:
                    req.wait()
                edges = [(g, g + min(k, n))] + ([(g + max(n - k, k), g + n)] if n > k else [])
                for lo, hi in edges:
                    self.rows_fn(lay, src, dst, k, lo, hi)
                self.cur = 1 - self.cur
            else:
                exchange(lay, src, self.dist, self.group)
                in_dst = self.step_fn(lay, src, dst, k)
                if in_dst:
                    self.cur = 1 - self.cur
            done += k

    def gather(self):
        """All owned rows on every rank -> global interior (torch, CPU)."""
        import torch

        own = self.owned().contiguous().cpu()
        if self.layout.world == 1:
            return own
        sizes = [None] * self.layout.world
        self.dist.all_gather_object(sizes, tuple(own.shape), group=self.group)
        parts = [torch.empty(s, dtype=own.dtype) for s in sizes]
        # gloo/nccl all_gather needs equal shapes: pad to the max row count
        mx = max(s[0] for s in sizes)
        pad = torch.zeros((mx,) + tuple(own.shape[1:]), dtype=own.dtype)
        pad[: own.shape[0]] = own
        if self.bufs[0].is_cuda:
            pad = pad.to(self.bufs[0].device)
        bucket = [torch.empty_like(pad) for _ in sizes]
        self.dist.all_gather(bucket, pad, group=self.group)
        for i, s in enumerate(sizes):
            parts[i] = bucket[i][: s[0]].cpu()
        return torch.cat(parts, 0)
