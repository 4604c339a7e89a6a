"""Sharded Jacobi (csrc/shard.cu) on the GPU.

The product path: ``jacobi2d_temporal(grid, T, n_gpus=N)`` /
``jacobi3d_temporal`` split axis 0 into N slabs whose kernels store the
neighbour's ghost rows straight into its buffer (peer memory) and order
their passes by pass counters and stream waits.  This box has one GPU, so
the N shards share it (``emulate_shards``): the same kernels, mirror stores,
counters and waits as on N devices, with peer pointers that happen to be
local.  Every result must equal the unsharded oracle bit for bit.

The multi-process form (one process per GPU, CUDA IPC handles exchanged over
torch.distributed) is driven with 2 processes on the one GPU; and the
NCCL/gloo ``halo.ShardedJacobi`` path with CUDA steps (gloo staging the
halos through host memory, so no kernel waits on another process).
"""

from __future__ import annotations

import os
import signal
import subprocess
import sys
import textwrap

import numpy as np
import pytest

from oracle import cref
from paper_2010_04868_b200 import Grid, _native, config
from paper_2010_04868_b200.catalog import get
from paper_2010_04868_b200.kernels import jacobi2d_temporal, jacobi3d_temporal

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kernel,ext,steps", [
    ("heat2d", (301, 257), 21),     # 5-point star, depth 8, uneven slabs
    ("jac2d9p", (133, 200), 17),    # 9-point box
    ("heat3d", (41, 33, 35), 7),    # 7-point star, 2 levels per pass, odd T
    ("jac3d27p", (40, 24, 70), 6),  # 27-point box
])
def test_sharded_drop_in_bitexact(cuda_ready, kernel, ext, steps):
    spec = get(kernel).spec
    g = Grid.random(ext, seed=11)
    want = cref.scalar_reference(spec, g, steps)
    fn = jacobi2d_temporal if len(ext) == 2 else jacobi3d_temporal
    with config.using(emulate_shards=True):
        for n in (1, 2, 3, 4, 5, 8):
            got = fn(g, steps, kernel=kernel, n_gpus=n)
            assert np.array_equal(got.interior, want.interior), (kernel, n)
            assert np.array_equal(g.interior, Grid.random(ext, seed=11).interior)  # input untouched


@pytest.mark.parametrize("depth", [1, 2, 3, 5, 12])
def test_sharded_depths(cuda_ready, depth):
    """Ghost width = temporal depth for every depth the 2D kernel has."""
    spec = get("heat2d").spec
    g = Grid.random((260, 130), seed=3, boundary=0.5)
    want = cref.scalar_reference(spec, g, 29)
    with config.using(emulate_shards=True, depth=depth):
        for n in (2, 7):
            got = jacobi2d_temporal(g, 29, n_gpus=n)
            assert np.array_equal(got.interior, want.interior), (depth, n)


def test_sharded_fma_allow_matches_unsharded(cuda_ready):
    """fma='allow' (tolerance mode): sharded == unsharded bit for bit, and
    within 1e-12 of the oracle."""
    spec = get("jac3d27p").spec
    g = Grid((36, 30, 40), 1)
    g.set_interior(np.random.default_rng(9).uniform(0.0, 1.0, g.extents))  # config 5's distribution
    one = jacobi3d_temporal(g, 8, kernel="jac3d27p", fma="allow")
    want = cref.scalar_reference(spec, g, 8)
    assert np.max(np.abs(one.interior - want.interior) / np.maximum(np.abs(want.interior), 1e-300)) <= 1e-12
    with config.using(emulate_shards=True, fma="allow"):
        for n in (2, 4):
            got = jacobi3d_temporal(g, 8, kernel="jac3d27p", n_gpus=n)
            assert np.array_equal(got.interior, one.interior), n


def test_sharded_plan_repeated_runs(cuda_ready):
    """Device-resident plan with n_gpus: pass counters continue across runs
    (run(7) + run(6) == 13 steps), and a fresh upload restarts cleanly."""
    spec = get("heat2d").spec
    ext = (200, 96)
    g = Grid.random(ext, seed=4)
    ex = config.ExecConfig(n_gpus=4, emulate_shards=True).native()
    plan = _native.Plan(spec, ext, ex)
    out = g.alloc_like()
    for rep in range(2):
        plan.upload(g.data, g.offset)
        plan.run(7)
        plan.run(6)
        plan.synchronize()
        plan.download(out.data, out.offset)
        assert np.array_equal(out.interior, cref.scalar_reference(spec, g, 13).interior), rep
        assert plan.last_launches() > 0 and plan.last_ms() >= 0.0
    plan.close()


def test_sharded_grid_too_small_and_too_many_gpus(cuda_ready):
    g = Grid.random((20, 40), seed=1)
    from paper_2010_04868_b200.errors import SizeError

    with config.using(emulate_shards=True):
        with pytest.raises(SizeError):  # 20 rows over 8 shards < depth 8 rows each
            jacobi2d_temporal(g, 3, n_gpus=8)
    with pytest.raises(ValueError):  # more GPUs than the box has, without emulation
        jacobi2d_temporal(g, 3, n_gpus=_native.device_count() + 1)


def test_sharded_gauss_seidel_runs_on_one_gpu(cuda_ready):
    """Gauss-Seidel is single-GPU (north_star): n_gpus is accepted and ignored."""
    from paper_2010_04868_b200.kernels import gs2d_temporal

    spec = get("gs2d9p").spec
    g = Grid.random((64, 80), seed=2)
    got = gs2d_temporal(g, 5, kernel="gs2d9p", n_gpus=4)
    want = cref.scalar_reference(spec, g, 5, order="lexicographic")
    assert np.array_equal(got.interior, want.interior)


def _run_ranks(script: str, world: int, timeout: float = 240.0):
    """Run `script` as `world` processes (RANK/WORLD_SIZE/MASTER_* set) in
    their own process group; kill the group on timeout."""
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), PYTHONPATH=ROOT)
        procs.append(subprocess.Popen([sys.executable, "-c", textwrap.dedent(script)], env=env, cwd=ROOT,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, start_new_session=True))
    outs = []
    try:
        for p in procs:
            out, _ = p.communicate(timeout=timeout)
            outs.append(out.decode(errors="replace"))
    except subprocess.TimeoutExpired:
        for p in procs:
            try:
                os.killpg(p.pid, signal.SIGKILL)
            except ProcessLookupError:
                pass
        raise
    for p, out in zip(procs, outs):
        assert p.returncode == 0, out[-3000:]
    return outs


IPC_SCRIPT = """
import os, sys
import numpy as np
import torch.distributed as dist
from paper_2010_04868_b200 import Grid, _native
from paper_2010_04868_b200.catalog import get
from oracle import cref
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
for kernel, ext, steps in (("heat2d", (150, 200), 19), ("jac3d27p", (30, 20, 40), 5)):
    spec = get(kernel).spec
    g = Grid.random(ext, seed=8)
    sh = _native.Shard(spec, ext, world, rank, _native.make_exec(device=0))
    hs = [None] * world
    dist.all_gather_object(hs, sh.export())
    sh.connect(hs[rank - 1] if rank > 0 else None, hs[rank + 1] if rank + 1 < world else None)
    sh.upload(g.data, g.offset)
    sh.synchronize()
    dist.barrier()
    sh.run(steps)
    sh.synchronize()
    dist.barrier()  # neighbours' last mirror stores landed
    out = g.alloc_like()
    sh.download(out.data, out.offset)
    sh.synchronize()
    r0, r1 = sh.rows
    parts = [None] * world
    dist.all_gather_object(parts, (r0, r1, out.interior[r0:r1].copy()))
    if rank == 0:
        full = np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])], 0)
        want = cref.scalar_reference(spec, g, steps)
        assert np.array_equal(full, want.interior), kernel
        print("ok", kernel)
    dist.barrier()
    sh.close()
dist.destroy_process_group()
"""


def test_sharded_ipc_two_processes(cuda_ready):
    """One process per shard: CUDA IPC handles exchanged with
    torch.distributed, fused mirror stores into the other process's buffers,
    pass counters across processes (both on this box's one GPU)."""
    outs = _run_ranks(IPC_SCRIPT, 2)
    assert "ok heat2d" in outs[0] and "ok jac3d27p" in outs[0]


HALO_SCRIPT = """
import os
import numpy as np
import torch, torch.distributed as dist
from paper_2010_04868_b200 import Grid, halo
from paper_2010_04868_b200.catalog import get
from oracle import cref
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
torch.cuda.set_device(0)
for kernel, ext, steps, depth in (("heat2d", (120, 150), 17, 8), ("jac3d27p", (24, 18, 30), 5, 2)):
    for overlap in (True, False):
        spec = get(kernel).spec
        g = Grid.random(ext, seed=6)
        sj = halo.ShardedJacobi(spec, ext, dist, depth=depth, device=torch.device("cuda", 0), overlap=overlap)
        sj.load_global(g.interior)
        sj.run(steps)
        torch.cuda.synchronize()
        full = sj.gather()
        if rank == 0:
            want = cref.scalar_reference(spec, g, steps)
            assert np.array_equal(full.numpy(), want.interior), (kernel, overlap)
            print("ok", kernel, overlap)
dist.destroy_process_group()
"""


def test_halo_sharded_jacobi_cuda_steps(cuda_ready):
    """halo.ShardedJacobi.run() with the CUDA kernels (overlapped interior /
    edge passes and the plain form), 2 ranks on gloo."""
    outs = _run_ranks(HALO_SCRIPT, 2)
    assert outs[0].count("ok ") == 4


def test_thread_cache_release_bounds_hbm(cuda_ready):
    """tvs_run keeps per-thread device buffers between calls; 8 pool workers
    (the reference's ThreadPool pattern, tiling.py:363-367) each release
    theirs with tvs_release_thread_cache, and device memory returns to the
    baseline (cached buffers were never released)."""
    from concurrent.futures import ThreadPoolExecutor

    import torch

    torch.cuda.init()
    g = Grid.random((192, 160, 200), seed=3)
    want = jacobi3d_temporal(g, 2, kernel="jac3d27p").interior
    _native.release_thread_cache()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()

    def work(_):
        got = jacobi3d_temporal(g, 2, kernel="jac3d27p").interior
        held = torch.cuda.mem_get_info()[0]
        _native.release_thread_cache()
        return np.array_equal(got, want), held

    with ThreadPoolExecutor(max_workers=8) as pool:
        res = list(pool.map(work, range(8)))
    assert all(ok for ok, _ in res)
    assert min(h for _, h in res) < free0 - 100 * 2 ** 20  # the buffers were really cached while in use
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free1 > free0 - 64 * 2 ** 20, (free0, free1)
