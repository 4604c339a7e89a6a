"""Command-line harness mirroring the reference CLI (tvstencil/cli.py:73-286).

    python -m paper_2010_04868_b200.cli --mode bench --kernel heat2d --nx 16384 --ny 16384 --t 200 --reps 5
    python -m paper_2010_04868_b200.cli --mode verify --kernel all --cells 20

Same flags, JSON ``--config`` defaults (explicit flags win), metric
(GStencil/s = interior points x T / median seconds / 1e9, cli.py:228-231),
median of ``--reps`` after one warm-up, and CSV schema
``kernel,variant,dim,nx,ny,nz,t,threads,tile,reps,gstencils_per_s,checksum``
(cli.py:39) with the FNV-1a checksum of the final grid's TSTN dump — so a
GPU row and a reference CPU row of the same run carry the same checksum.
Appended columns: ``backend,device_ms,depth``.  ``--tile WxH[xD]:T`` and
``--threads a[..b]`` select the tile-schedule executor (tiling.py: one GPU
launch per wave, one CTA per tile) as in the reference (cli.py:57-70,
156-170); ``life`` (int32) and ``lcs`` (LCS length of two seeded
sequences, cells = na x nb) are benchmarked like the reference does.

``--mode verify`` runs on the GPU only (the product never embeds the CPU
oracle): the reference's known-answer vectors (test_baselines.py:17-36) and,
for every cell of the reference-shaped acceptance matrix, the temporally
blocked / pipelined kernels against the independent one-step (Jacobi) and
hyperplane-wavefront (Gauss-Seidel) kernels, bit-exact.  Oracle parity
proper lives in tests/.
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
import time

import numpy as np

from . import _native, config
from .catalog import DEFAULT_CATALOG, get as catalog_get
from .grid import Grid, fnv1a64
from .kernels import KernelVariant
from .kernels import lcs_temporal
from .tiling import build_schedule, execute_parallel, lcs_blocked
from .verify import default_matrix, run_temporal

CSV_HEADER = "kernel,variant,dim,nx,ny,nz,t,threads,tile,reps,gstencils_per_s,checksum"
CSV_EXTRA = "backend,device_ms,depth"
DEFAULT_SIZES = {1: (1_000_000,), 2: (512, 512), 3: (64, 64, 64)}
GPU_KERNELS = list(DEFAULT_CATALOG) + ["lcs"]
FP_KERNELS = [k for k, e in DEFAULT_CATALOG.items() if e.spec.element_kind == "float64"]
DEFAULT_TILES = {  # reference cli.py:44-53 (used when --threads > 1 without --tile)
    "heat1d": ((16384,), 128), "heat2d": ((256, 256), 64), "jac2d9p": ((256, 256), 64),
    "heat3d": ((32, 32, 32), 8), "life": ((256, 256), 32), "gs1d": ((2048,), 64), "gs2d": ((128, 128), 32),
    "gs3d": ((32, 32, 32), 32), "lcs": ((4096,), 4096),
}


def _parse_tile(text):
    """'WxHxD:T' -> (space extents, time height) (reference cli.py:57-63)."""
    space, _, t = text.partition(":")
    if not t:
        raise argparse.ArgumentTypeError("tile needs a :T time height")
    return tuple(int(p) for p in space.split("x")), int(t)


def _parse_threads(text):
    if ".." in text:
        lo, hi = text.split("..")
        return list(range(int(lo), int(hi) + 1))
    return [int(text)]


def _fit_tile(tile, extents, entry):
    """Shrink a tile request by powers of two until it fits the grid (the
    reference's rule, cli.py:253-265)."""
    space, height = tile
    space = list(space[: len(extents)]) + [space[-1]] * (len(extents) - len(space))
    floor = 4 * entry.s * entry.vl
    for i, (w, n) in enumerate(zip(space, extents)):
        while w > n and (i > 0 or w // 2 >= floor):
            w //= 2
        space[i] = min(w, n) if i > 0 else w
    while height > entry.vl and height > min(space[1:] or [height]):
        height //= 2
    return tuple(space), max(entry.vl, height // entry.vl * entry.vl)


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="tvstencil-b200", description=__doc__,
                                formatter_class=argparse.RawDescriptionHelpFormatter)
    p.add_argument("--mode", choices=("verify", "bench"), required=True)
    p.add_argument("--kernel", default="all", help=f"one of {GPU_KERNELS} or 'all'")
    p.add_argument("--variant", default="base", choices=("base", "two-stride"))
    p.add_argument("--nx", type=int)
    p.add_argument("--ny", type=int)
    p.add_argument("--nz", type=int)
    p.add_argument("--t", type=int, dest="steps")
    p.add_argument("--tile", type=_parse_tile, help="tile-schedule executor: WxHxD:T (space tile : time height)")
    p.add_argument("--threads", type=_parse_threads, default=None,
                   help="reference worker counts (a or a..b); on the GPU every tile of a wave is a CTA")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--csv", help="append benchmark rows to this file")
    p.add_argument("--dump", help="write the final grid dump (TSTN) here")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--cells", type=int, default=20, help="verify-mode cells per kernel (reference acceptance: 20)")
    p.add_argument("--config", help="JSON file with flag defaults")
    p.add_argument("--order", default="lexicographic", choices=("lexicographic", "reference"),
                   help="Gauss-Seidel update order (2D/3D)")
    p.add_argument("--fma", default="exact", choices=("exact", "never", "allow"))
    p.add_argument("--depth", type=int, default=0, help="temporal block depth (0 = kernel default)")
    return p


def _apply_config(args, argv):
    if not args.config:
        return args
    with open(args.config) as fh:
        cfg = json.load(fh)
    passed = {a.split("=")[0].lstrip("-").replace("-", "_") for a in argv if a.startswith("--")}
    for key, value in cfg.items():
        attr = "steps" if key == "t" else key.replace("-", "_")
        if key in passed or attr in passed or not hasattr(args, attr):
            continue
        if attr == "tile" and isinstance(value, str):
            value = _parse_tile(value)
        if attr == "threads" and isinstance(value, (str, int)):
            value = _parse_threads(str(value))
        setattr(args, attr, value)
    return args


def _kernels(arg):
    if arg == "all":
        return GPU_KERNELS
    if arg not in GPU_KERNELS:
        raise SystemExit(f"unknown or non-GPU kernel {arg!r}; known: {GPU_KERNELS}")
    return [arg]


def _grid_size(args, dim):
    size = list(DEFAULT_SIZES[dim])
    for i, v in enumerate((args.nx, args.ny, args.nz)[:dim]):
        if v:
            size[i] = v
    return tuple(size)


def _timed(fn, reps):
    fn()  # warm-up
    times, out = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        times.append(time.perf_counter() - t0)
    return statistics.median(times), out


def _bench(args) -> int:
    rows = []
    scheme = args.variant.replace("-", "_")
    tile_txt = ("x".join(map(str, args.tile[0])) + f":{args.tile[1]}") if args.tile else ""
    for kernel in _kernels(args.kernel):
        for threads in args.threads or [1]:
            dev_ms = ""
            if kernel == "lcs":
                rng = np.random.default_rng(args.seed)
                na = args.nx or 20000
                nb = args.ny or na
                a = rng.integers(0, 4, na, dtype=np.int32)
                b = rng.integers(0, 4, nb, dtype=np.int32)
                steps, dim, s3 = na, 2, (na, nb, 0)
                if args.tile or threads > 1:
                    tile = args.tile or DEFAULT_TILES["lcs"]
                    sched = build_schedule("lcs", (nb,), na, tile[0], tile[1])
                    med, val = _timed(lambda: lcs_blocked(a, b, sched, workers=threads), args.reps)
                else:
                    med, val = _timed(lambda: lcs_temporal(a, b), args.reps)
                rate = na * nb / med / 1e9
                check = val & 0xFFFFFFFFFFFFFFFF
            else:
                entry = catalog_get(kernel)
                dim = entry.spec.dim
                size = _grid_size(args, dim)
                steps = args.steps or 64
                grid = Grid.random(size, seed=args.seed, element_kind=entry.spec.element_kind, vl=entry.vl)
                gauss = entry.spec.dependence_kind == "gauss_seidel"
                opts = {"order": args.order} if gauss and dim > 1 else {}
                tile = args.tile or (DEFAULT_TILES[kernel] if threads > 1 else None)
                with config.using(fma=args.fma, depth=args.depth):
                    if tile:
                        tile = _fit_tile(tile, grid.extents, entry)
                        sched = build_schedule(kernel, grid.extents, steps, tile[0], tile[1])
                        med, out = _timed(lambda: execute_parallel(kernel, grid, sched, workers=threads), args.reps)
                    else:
                        if entry.spec.element_kind == "float64":
                            # device-resident time (plan API) for the device_ms column
                            plan = _native.Plan(entry.spec, size, config.current().native(order=args.order))
                            plan.upload(grid.data, grid.offset)
                            plan.run(steps)
                            plan.synchronize()
                            dev = []
                            for _ in range(args.reps):
                                plan.upload(grid.data, grid.offset)
                                plan.run(steps)
                                dev.append(plan.last_ms())
                            plan.close()
                            dev_ms = f"{statistics.median(dev):.3f}"
                        var = KernelVariant(scheme, gauss)
                        med, out = _timed(lambda: run_temporal(kernel, grid, steps, var, **opts), args.reps)
                rate = int(np.prod(size)) * steps / med / 1e9
                check = fnv1a64(out.dump_bytes())
                if args.dump:
                    out.dump(args.dump)
                s3 = tuple(size) + (0, 0)
            row = (f"{kernel},{args.variant},{dim},{s3[0]},{s3[1] or ''},{s3[2] or ''},{steps},{threads},{tile_txt},"
                   f"{args.reps},{rate:.6f},{check:016x},cuda-sm100a,{dev_ms},{args.depth}")
            rows.append(row)
            print(row)
    if args.csv:
        try:
            new = not open(args.csv).read(1)
        except OSError:
            new = True
        with open(args.csv, "a") as fh:
            if new:
                fh.write(CSV_HEADER + "," + CSV_EXTRA + "\n")
            fh.write("\n".join(rows) + "\n")
    return 0


_KNOWN = [  # reference test_baselines.py:17-21, 32-36
    ("heat1d", np.arange(1.0, 9.0), [1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0, 5.75]),
    ("gs1d", np.ones(3), [0.75, 0.9375, 0.734375]),
]


def _verify(args) -> int:
    from .kernels._common import execute

    ok = True
    for kernel, values, want in _KNOWN:
        got = execute(catalog_get(kernel).spec, Grid.from_array(values, halo=1), 1).interior.tolist()
        good = got == want
        ok &= good
        print(f"  {'PASS' if good else 'FAIL'} known answer {kernel}: {got}")
    fp_names = [k for k in _kernels(args.kernel) if k in FP_KERNELS]
    cells = default_matrix(cells_per_kernel=args.cells, kernels=fp_names) if fp_names else []
    t0 = time.time()
    bad = 0
    for cell in cells:
        entry = catalog_get(cell.kernel)
        g = Grid.random(cell.size, seed=cell.seed)
        opts = {"order": args.order} if entry.spec.dependence_kind == "gauss_seidel" and entry.spec.dim > 1 else {}
        fast = execute(entry.spec, g, cell.steps, algo="auto", **opts)
        slow = execute(entry.spec, g, cell.steps, algo="naive", **opts)
        if not np.array_equal(fast.interior, slow.interior):
            bad += 1
            pos = tuple(int(i) for i in np.argwhere(fast.interior != slow.interior)[0])
            print(f"  FAIL {cell.describe()} first divergence {pos}")
    ok &= bad == 0
    print(f"equivalence (blocked vs naive, GPU): {len(cells)} cells, {'PASS' if bad == 0 else 'FAIL'} "
          f"({time.time() - t0:.1f}s)")
    # integer kernels: two independent GPU algorithms each (Life: 4 levels per
    # pass vs single steps; LCS: time-lane pipeline vs tiled anti-diagonal waves)
    ints = [k for k in _kernels(args.kernel) if k in ("life", "lcs")]
    if ints:
        t0 = time.time()
        icells = default_matrix(cells_per_kernel=args.cells, kernels=ints)
        ibad = 0
        for cell in icells:
            if cell.kernel == "lcs":
                rng = np.random.default_rng(cell.seed)
                a = rng.integers(0, 4, size=cell.size[0], dtype=np.int32)
                b = rng.integers(0, 4, size=cell.size[1], dtype=np.int32)
                sched = build_schedule("lcs", (len(b),), len(a), (128,), 64)
                same = lcs_temporal(a, b) == lcs_blocked(a, b, sched)
            else:
                spec = catalog_get(cell.kernel).spec
                g = Grid.random(cell.size, seed=cell.seed, element_kind="int32")
                with config.using(depth=4):
                    fast = execute(spec, g, cell.steps)
                with config.using(depth=1):
                    slow = execute(spec, g, cell.steps)
                same = np.array_equal(fast.interior, slow.interior)
            if not same:
                ibad += 1
                print(f"  FAIL {cell.describe()}")
        ok &= ibad == 0
        print(f"equivalence (integer kernels, GPU): {len(icells)} cells, {'PASS' if ibad == 0 else 'FAIL'} "
              f"({time.time() - t0:.1f}s)")
    print("verify:", "PASS" if ok else "FAIL")
    return 0 if ok else 1


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    args = _apply_config(args, sys.argv[1:] if argv is None else argv)
    if args.mode == "verify":
        return _verify(args)
    return _bench(args)


if __name__ == "__main__":
    sys.exit(main())
