"""Benchmark harness (driver contract + the reference CLI's metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C] [--no-all]

A *step* is one call of the hot path over one synthetic BASELINE workload:
all T time steps / sweeps of the configured stencil over the full grid.
GStencil/s = interior points x T / seconds / 1e9 (reference cli.py:228-231).

* ``value``  : device-resident (tvs_plan_* API), CUDA events on the plan
  stream, W warm-up + K timed steps, barrier + synchronize on both sides,
  max over ranks.
* ``e2e``    : the public drop-in call (e.g. ``jacobi2d_temporal``) on pinned
  host Grids — host->device upload and device->host download inside the
  timed region, every step.
* ``cpu_baseline`` : the oracle port (C restatement of the reference's
  ``scalar_reference``, bit-exact, OpenMP over all host cores for Jacobi;
  single core for Gauss-Seidel, whose sweep is sequential) on a bounded
  sample of the same workload, rank 0 only.
* ``--impl reference`` : times that CPU implementation as the reference arm.

Headline workload (config.workload): BASELINE config 3, 2D 5-point Jacobi
16384^2 x 200 — the sharded, HBM-bound configuration.  The other four
BASELINE configs are measured the same way and reported under
``per_stencil`` (disable with --no-all).  Inputs (2-9 GB per grid for
configs 3-5) exceed the 126 MB L2; configs 1-2 (8 MiB) are L2-resident by
design and an L2 flush (256 MiB write) runs between their timed steps.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs: name, catalog kernel, extents, T,
# seed, distribution, drop-in function name, algorithmic FP64 ops / update
CONFIGS = {
    1: dict(name="1d3p_jacobi", kernel="heat1d", extents=(2 ** 20,), T=1000, seed=0, dist=(-1.0, 1.0),
            fn="heat1d_temporal", ops=5, shards=False),
    2: dict(name="1d3p_gauss_seidel", kernel="gs1d_w343", extents=(2 ** 20,), T=1000, seed=1, dist=(-1.0, 1.0),
            fn="gs1d_temporal", ops=5, shards=False),
    3: dict(name="2d5p_jacobi", kernel="heat2d", extents=(16384, 16384), T=200, seed=2, dist=(0.0, 1.0),
            fn="jacobi2d_temporal", ops=9, shards=True),
    4: dict(name="2d9p_gauss_seidel", kernel="gs2d9p", extents=(8192, 8192), T=100, seed=3, dist=(-1.0, 1.0),
            fn="gs2d_temporal", ops=17, shards=False),
    5: dict(name="3d27p_jacobi", kernel="jac3d27p", extents=(1024, 1024, 1024), T=100, seed=5, dist=(0.0, 1.0),
            fn="jacobi3d_temporal", ops=53, shards=True),
}
HEADLINE = 3
BYTES_PER_UPDATE = 16  # 8 B read + 8 B write per point update


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def measured_traffic(cfg):
    """ncu DRAM bytes per launch of this config's dominant kernel (committed
    evidence, profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)
        cid = next(k for k, v in CONFIGS.items() if v is cfg or v["name"] == cfg["name"])
        return t["configs"][str(cid)]
    except Exception:
        return None


def make_grid(cfg, pinned=False):
    from paper_2010_04868_b200 import Grid

    g = Grid(cfg["extents"], 1, boundary=0.0)
    lo, hi = cfg["dist"]
    rng = np.random.default_rng(cfg["seed"])
    g.set_interior(rng.uniform(lo, hi, size=cfg["extents"]))
    return g


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw,"
              "enforced.power.limit")

    def __init__(self, device=0):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        self.__enter__()

    def stop(self):
        self.__exit__(None, None, None)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "10"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def wait_ready(self, timeout=3.0):
        """Block until nvidia-smi has produced its first sample (it needs
        0.1-0.5 s to start), so a short timed region is still covered."""
        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.01)

    def mark(self, start):
        """Host wall-clock bounds of the timed region (samples outside are dropped)."""
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, power, plimit = [], None, set(), [], None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", 0.0), getattr(self, "t1", float("inf"))
        for ts, line in self.lines:
            if not t0 <= ts <= t1 + 0.05:
                continue
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
            try:  # board power next to its limit: a clock below max at the limit is the power cap
                power.append(float(parts[6]))
                plimit = float(parts[7])
            except (IndexError, ValueError):
                pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if power:
            out["power_w_max"] = max(power)
            out["power_limit_w"] = plimit
            # the power-cap flag is momentary and can fall between samples
            if plimit and max(power) >= 0.97 * plimit and out["sm_mhz"] < 0.97 * (mx or 0) and not reasons:
                out["note"] = "clock below max at the board power limit (power cap; flag not caught by a sample)"
        return out


def flush_l2(buf):
    if buf is not None:
        buf.fill_(1.0)


def dp_instr_per_update(cfg, fma=None):
    """FP64 instructions the kernel issues per useful update: k taps cost
    k DMUL/DFMA when fused (fma='allow', or 'exact' with power-of-two
    weights, where the fused form is bit-identical), else k DMUL + (k-1)
    DADD.  Ghost recompute is not counted (it is the overhead this metric
    exposes)."""
    import math

    from paper_2010_04868_b200 import config
    from paper_2010_04868_b200.catalog import get

    spec = get(cfg["kernel"]).spec
    cs = [float(spec.coefficients[o]) for o in spec.offsets()]
    k = len(cs)
    policy = fma or config.current().fma
    pow2 = all(c == 0.0 or math.frexp(abs(c))[0] == 0.5 for c in cs)
    fused = policy == "allow" or (policy == "exact" and pow2)
    if fused and pow2 and len(cfg["extents"]) == 2 and os.environ.get("TVS_J2D_SCALED", "1") != "0":
        # K3's scaled power-of-two taps: the first tap is free, k - 1 DFMAs,
        # and one rescaling DMUL per stored value (1 / depth per update)
        depth = config.current().depth or 8
        return k - 1 + 1.0 / depth, fused
    if fused and pow2 and len(cfg["extents"]) == 1 and os.environ.get("TVS_J1D_SCALED", "1") != "0":
        depth = config.current().depth or 64  # K2: the same scheme, plus one pin-scale DMUL per step and lane
        return k - 1 + 1.0 / depth + 1.0 / 32, fused
    return (k if fused else 2 * k - 1), fused


def device_time(cfg, K, W, sampler=None, fma=None, min_timed_s=0.0, algo=None, order="lexicographic"):
    """Device-resident timing through the plan API: per-step ms (CUDA events
    on the plan stream) and launches per step.  Each step runs all T updates
    on the field left by the previous step (same work every step)."""
    import torch

    from paper_2010_04868_b200 import _native, config
    from paper_2010_04868_b200.catalog import get

    spec = get(cfg["kernel"]).spec
    g = make_grid(cfg)
    ex = config.current().native(order=order, **({"fma": fma} if fma else {}), **({"algo": algo} if algo else {}))
    plan = _native.Plan(spec, cfg["extents"], ex)
    stream = torch.cuda.ExternalStream(plan.stream_handle())
    l2 = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device="cuda") if g.data.nbytes < 2 ** 30 else None
    times, times_w, launches = [], [], 0
    plan.upload(g.data, g.offset)
    plan.synchronize()
    del g
    if sampler is not None:
        sampler.start()  # nvidia-smi needs ~0.1-0.5 s to start; samples are kept only inside the timed region
        sampler.wait_ready()
    i = 0
    while i < W + K:
        if i == W and min_timed_s > 0 and times_w:
            # short steps (configs 1-2: < 1 ms): time enough of them that the
            # clock sampler sees the timed region
            K = max(K, min(2000, int(min_timed_s * 1e3 / max(times_w[-1], 1e-3)) + 1))
        if i == W and sampler is not None:
            sampler.mark(True)
        if i >= W:
            flush_l2(l2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan.run(cfg["T"])
        e1.record(stream)
        e1.synchronize()
        if i >= W:
            times.append(e0.elapsed_time(e1))
            launches = plan.last_launches()
        else:
            times_w.append(e0.elapsed_time(e1))
        i += 1
    if sampler is not None:
        sampler.mark(False)
        sampler.stop()
    plan.close()
    return times, launches


def e2e_time(cfg, K, W):
    """Public drop-in call, pinned host buffers, H2D + D2H inside the timing."""
    from paper_2010_04868_b200 import Grid, _native, kernels

    src = make_grid(cfg)
    # page-locked Grid storage from the library (tvs_host_alloc); registering
    # numpy pages instead costs ~15% of duplex PCIe rate (tools/pinned_probe.py)
    host = os.environ.get("TVS_BENCH_HOST", "alloc")
    g = src.copy() if host == "register" else Grid(src.extents, src.halo, src.boundary, src.element_kind,
                                                   src.vl, pinned=True)
    if host != "register":
        np.copyto(g.data, src.data)
    del src
    out = g.copy()
    if host == "register":
        _native.host_register(g.data)
        _native.host_register(out.data)
    fn = getattr(kernels, cfg["fn"])
    kw = {"kernel": cfg["kernel"]}
    try:
        times = []
        for i in range(W + K):
            t0 = time.perf_counter()
            fn(g, cfg["T"], out=out, **kw)
            t1 = time.perf_counter()
            if i >= W:
                times.append((t1 - t0) * 1e3)
    finally:
        if host == "register":
            _native.host_unregister(g.data)
            _native.host_unregister(out.data)
    nbytes = int(np.prod(cfg["extents"])) * 8
    return times, nbytes, out


def _port_rate(spec, g, steps, cores):
    """C restatement of scalar_reference (bit-exact, OpenMP over axis 0 for
    Jacobi, one core for Gauss-Seidel): GStencil/s of its step loop (the
    allocations and copies around it excluded, oracle_last_seconds)."""
    from oracle import cref

    cref.scalar_reference(spec, g, steps, order="lexicographic", threads=cores)
    return int(np.prod(g.extents)) * steps / cref.last_seconds() / 1e9, cref.last_seconds()


def numpy_reference_rate(cfg, budget_s=20.0):
    """The reference's own CPU code path, restated in NumPy (oracle/oracle.py:
    the same whole-plane ufunc taps / Python GS loop / anti-diagonal gather as
    baselines.py:43-125, bit-exact), one core (NumPy ufuncs are single
    threaded), on a bounded sample: the full grid (config 5: a 256^3 block)
    for 1-2 steps.  BASELINE.md §2's CPU baseline."""
    from oracle import oracle as npo
    from paper_2010_04868_b200 import Grid
    from paper_2010_04868_b200.catalog import get

    spec = get(cfg["kernel"]).spec
    ext = cfg["extents"]
    if int(np.prod(ext)) > 2 ** 28:
        ext = tuple(min(e, 256) for e in ext)
    g = Grid(ext, 1)
    g.set_interior(np.random.default_rng(cfg["seed"]).uniform(*cfg["dist"], size=ext))
    gauss = spec.dependence_kind == "gauss_seidel"
    if gauss and len(ext) == 1:
        # pure-Python loop (~0.001 GSt/s): a 2^16 prefix keeps it to seconds
        g = Grid((2 ** 16,), 1)
        g.set_interior(np.random.default_rng(cfg["seed"]).uniform(*cfg["dist"], size=(2 ** 16,)))
    t0 = time.perf_counter()
    npo.scalar_reference(spec, g, 1)
    one = time.perf_counter() - t0
    steps = int(max(1, min(3, budget_s / max(one, 1e-6))))
    t0 = time.perf_counter()
    npo.scalar_reference(spec, g, steps)
    dt = time.perf_counter() - t0
    return {"value": int(np.prod(g.extents)) * steps / dt / 1e9, "unit": "GStencil/s", "cores": 1,
            "kind": "port",
            "sample": f"NumPy restatement of the reference's scalar_reference (baselines.py:110-125, same ufunc "
                      f"taps; reference order for GS-2D), {'x'.join(map(str, g.extents))} grid, {steps} "
                      f"{'sweeps' if gauss else 'steps'}, {dt:.1f} s, 1 core"}


def e2e_stock_time(cfg, K, W):
    """The stock call a reference user makes: ``fn(grid, T)`` on the default
    pageable Grid, no ``out=`` (the result Grid is allocated by the call,
    kernels_nd.py:38-40,91).  Host->device and device->host copies, the
    result allocation and its page faults are all inside the timing."""
    from paper_2010_04868_b200 import kernels

    g = make_grid(cfg)
    fn = getattr(kernels, cfg["fn"])
    times = []
    for i in range(W + K):
        t0 = time.perf_counter()
        out = fn(g, cfg["T"], kernel=cfg["kernel"])
        t1 = time.perf_counter()
        del out
        if i >= W:
            times.append((t1 - t0) * 1e3)
    return times


def cpu_sample(cfg, budget_s=12.0):
    """Oracle C port on the host: bounded sample of the same workload (full
    grid, T_cpu steps, all cores for Jacobi / one for Gauss-Seidel), timed
    inside its step loop.  Returns (GStencil/s, cores, description)."""
    from paper_2010_04868_b200.catalog import get

    spec = get(cfg["kernel"]).spec
    g = make_grid(cfg)
    gauss = spec.dependence_kind == "gauss_seidel"
    cores = 1 if gauss else (os.cpu_count() or 1)
    _, one = _port_rate(spec, g, 1, cores)  # warm-up (first touch) and the per-step time
    steps = int(max(1, min(cfg["T"], budget_s / max(one, 1e-6))))
    rate, dt = _port_rate(spec, g, steps, cores)
    desc = (f"C restatement of scalar_reference (bit-exact; not the reference's NumPy code), full "
            f"{'x'.join(map(str, cfg['extents']))} grid, {steps} of {cfg['T']} {'sweeps' if gauss else 'steps'}, "
            f"{dt:.1f} s in the step loop, {cores} thread(s)")
    return rate, cores, desc


def measure_config(cfg, K, W, with_e2e=True, with_cpu=True, min_timed_s=0.0, with_stock=False):
    hbm_peak, peak_src = peaks()
    pts = int(np.prod(cfg["extents"]))
    updates = pts * cfg["T"]
    clk = ClockSampler()
    times, launches = device_time(cfg, K, W, sampler=clk, min_timed_s=min_timed_s)
    ms = statistics.mean(times)
    value = updates / (ms * 1e-3) / 1e9
    res = {
        "value": value, "unit": "GStencil/s", "ms_per_step": ms, "ms_per_step_min": min(times), "steps": len(times),
        "warmup": W, "gpu_launches": launches * len(times), "launches_per_step": launches, "clocks": clk.summary(),
        "workload": f"{cfg['name']} {'x'.join(map(str, cfg['extents']))} T={cfg['T']}",
    }
    # per launch of the dominant kernel (every launch of a step is that kernel
    # here): algorithmic bytes = 16 B x updates per launch, duration = step
    # time / launches, both from the CUDA events above
    per_launch_ms = ms / max(launches, 1)
    upd_launch = updates / max(launches, 1)
    achieved = BYTES_PER_UPDATE * upd_launch / (per_launch_ms * 1e-3) / 1e9
    traffic = measured_traffic(cfg)
    res["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                       "frac": achieved / hbm_peak,
                       "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                       "traffic_bytes_per_update": traffic["dram_bytes_per_update"] if traffic else None,
                       "algorithmic_bytes_per_launch": BYTES_PER_UPDATE * upd_launch,
                       "launch_ms": per_launch_ms, "peak_source": peak_src,
                       "note": "achieved = 16 B/update x updates per launch / launch time (effective bandwidth; "
                               "temporal blocking makes it exceed HBM peak). traffic = ncu dram read+write per "
                               "launch of the same kernel (profiles/traffic.json)"}
    sm = res["clocks"].get("sm_mhz") or 1965.0
    fp64_peak = 148 * 64 * sm * 1e6 / 1e12  # DP instructions/s (DADD/DMUL/DFMA), measured 63.4/clk/SM
    instr, fused = dp_instr_per_update(cfg)
    fp64 = instr * updates / (ms * 1e-3) / 1e12
    res["fp64"] = {"achieved_tinstr": fp64, "peak_tinstr": fp64_peak, "frac": fp64 / fp64_peak,
                   "dp_instr_per_update": instr, "fused": fused, "flops_per_update": cfg["ops"],
                   "note": "FP64 instructions issued per useful update (DFMA = 1) x update rate; peak = 148 SM x "
                           "64/clk x median SM clock; ghost recompute not counted"}
    if with_e2e:
        etimes, nbytes, _ = e2e_time(cfg, K, W)
        ems = statistics.mean(etimes)
        res["e2e"] = {"value": updates / (ems * 1e-3) / 1e9, "unit": "GStencil/s", "ms_per_step": ems,
                      "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes}
    if with_e2e and with_stock:
        st = e2e_stock_time(cfg, max(2, min(K, 3)), 1)
        sms = statistics.mean(st)
        nbytes = int(np.prod(cfg["extents"])) * 8
        res["e2e_stock"] = {"value": updates / (sms * 1e-3) / 1e9, "unit": "GStencil/s", "ms_per_step": sms,
                            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                            "note": "fn(grid, T) on the default pageable Grid, result Grid allocated by the call"}
    if with_cpu:
        rate, cores, desc = cpu_sample(cfg)
        res["cpu_baseline"] = {"value": rate, "unit": "GStencil/s", "cores": cores, "kind": "port", "sample": desc,
                               "numpy_reference_path": numpy_reference_rate(cfg)}
    return res


def untiled_legs(args):
    """North_star: "untiled kernels reach >= 70% of HBM peak".  The
    single-step kernel (K1, algo='naive': one time step per HBM pass, no
    temporal blocking) on the full config-3 grid, and config 5's own kernel,
    which is single-step by construction (2.5D plane streaming).  Effective
    bandwidth = 16 B x update rate; ncu DRAM bytes per launch in profiles/."""
    hbm_peak, _ = peaks()
    out = {}
    from paper_2010_04868_b200 import config

    for cid, algo, T in ((3, "naive", 20), (5, "auto", 10)):
        c = dict(CONFIGS[cid], T=T)
        try:
            clk = ClockSampler()
            # depth 1 keeps config 5 on its single-step kernel (K4); the default is the two-level K4c
            with config.using(depth=1):
                t, launches = device_time(c, max(2, min(args.steps, 3)), args.warmup, sampler=clk, algo=algo)
            ms = statistics.mean(t)
            v = int(np.prod(c["extents"])) * T / (ms * 1e-3) / 1e9
            out[c["name"]] = {
                "kernel": "jacobi_naive_kernel" if algo == "naive" else "jacobi3d_kernel",
                "value": v, "unit": "GStencil/s", "steps_per_run": T, "launches_per_run": launches,
                "ms_per_run": ms, "clocks": clk.summary(),
                "roofline": {"bound": "hbm", "achieved": v * BYTES_PER_UPDATE, "peak": hbm_peak, "unit": "GB/s",
                             "frac": v * BYTES_PER_UPDATE / hbm_peak},
            }
            if cid == 5:
                out[c["name"]]["note"] = ("single-step 27-point box, bit-exact: 53 FP64 instructions per update, so "
                                          "FP64 issue (ceiling ~351 GSt/s at 1.965 GHz), not HBM, bounds it")
        except Exception as exc:  # report, never hide
            out[c["name"]] = {"error": repr(exc)}
    return out


def integer_legs(args):
    """SURVEY §8f rank 4 kernels, device-resident (torch buffers, CUDA events
    on the launching stream): Life B2S23 (reference catalog "life") on a
    16384^2 int32 grid, 4 B read + 4 B written per cell update; LCS length of
    two seeded 65536-long sequences (4-letter alphabet), DP cells/s."""
    import ctypes as C

    import torch

    from paper_2010_04868_b200 import _native
    from paper_2010_04868_b200.catalog import get

    hbm_peak, _ = peaks()
    out = {}
    K = max(2, min(args.steps, 3))
    try:
        ext, T = (16384, 16384), 20
        spec = get("life").spec
        rule = _native.make_life_rule(spec)
        geo = _native.geometry(2, ext)
        n = int(geo.alloc_elems)
        bufs = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(2)]
        s = torch.cuda.current_stream()
        for b in bufs:
            _native.check(_native.lib().tvs_fill_halo_i32(C.byref(geo), C.c_void_p(b.data_ptr()), 0,
                                                          C.c_void_p(s.cuda_stream)))
        view = bufs[0].as_strided(ext, (int(geo.strides[0]), 1), int(geo.origin))
        g = torch.Generator(device="cuda").manual_seed(0)
        view.copy_(torch.randint(0, 2, ext, generator=g, device="cuda", dtype=torch.int32))
        ex = _native.make_exec()
        res = C.c_int32(0)

        def run():
            _native.check(_native.lib().tvs_life_device(
                C.byref(rule), C.byref(geo), C.c_void_p(bufs[0].data_ptr()), C.c_void_p(bufs[1].data_ptr()), T,
                C.byref(ex), C.c_void_p(s.cuda_stream), C.byref(res)))

        times = []
        for i in range(args.warmup + K):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            run()
            e1.record(s)
            e1.synchronize()
            if i >= args.warmup:
                times.append(e0.elapsed_time(e1))
        ms = statistics.mean(times)
        v = ext[0] * ext[1] * T / (ms * 1e-3) / 1e9
        out["life_b2s23_2d"] = {
            "kernel": "life_kernel", "workload": f"life B2S23 {ext[0]}x{ext[1]} int32 T={T}", "value": v,
            "unit": "GCellUpdates/s", "ms_per_run": ms, "launches_per_run": T,
            "roofline": {"bound": "hbm", "achieved": v * 8, "peak": hbm_peak, "unit": "GB/s", "frac": v * 8 / hbm_peak,
                         "note": "algorithmic 4 B read + 4 B written per cell update"}}
        del bufs
    except Exception as exc:  # report, never hide
        out["life_b2s23_2d"] = {"error": repr(exc)}
    try:
        na = nb = 65536
        rng = np.random.default_rng(12)
        a = torch.from_numpy(rng.integers(0, 4, na).astype(np.int32)).cuda()
        b = torch.from_numpy(rng.integers(0, 4, nb).astype(np.int32)).cuda()
        r = torch.zeros(1, dtype=torch.int32, device="cuda")
        s = torch.cuda.current_stream()
        times = []
        for i in range(args.warmup + K):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            _native.check(_native.lib().tvs_lcs_device(C.c_void_p(a.data_ptr()), na, C.c_void_p(b.data_ptr()), nb,
                                                       C.c_void_p(r.data_ptr()), C.c_void_p(s.cuda_stream)))
            e1.record(s)
            e1.synchronize()
            if i >= args.warmup:
                times.append(e0.elapsed_time(e1))
        ms = statistics.mean(times)
        out["lcs"] = {"kernel": "lcs_kernel", "workload": f"lcs {na}x{nb} alphabet 4", "value": na * nb / (ms * 1e-3) / 1e9,
                      "unit": "GCells/s", "ms_per_run": ms, "length": int(r.item())}
    except Exception as exc:  # report, never hide
        out["lcs"] = {"error": repr(exc)}
    return out


def run_reference(args):
    """--impl reference: the reference's CPU path on the host.  The reference
    is pure Python (nothing to compile into oracle/_ref), so the arm times
    the oracle port: the bit-exact C restatement of scalar_reference on all
    host cores (Gauss-Seidel: one), timed inside its step loop exactly like
    the cpu_baseline leg of our arm (so the two agree), each step a bounded
    sample of the workload (full grid, T_cpu steps).  The NumPy restatement
    of the reference's own code path (1 core) is reported beside it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    from paper_2010_04868_b200.catalog import get

    spec = get(cfg["kernel"]).spec
    g = make_grid(cfg)
    gauss = spec.dependence_kind == "gauss_seidel"
    cores = 1 if gauss else (os.cpu_count() or 1)
    pts = int(np.prod(cfg["extents"]))
    _, one = _port_rate(spec, g, 1, cores)
    # the same ~12 s sample per step as our arm's cpu_baseline leg (a longer
    # sample runs the host at a lower sustained clock: 3.4 vs 4.5 GSt/s)
    t_cpu = int(max(1, min(cfg["T"], 12.0 / max(one, 1e-6))))
    times = []
    for i in range(args.warmup + args.steps):
        _, dt = _port_rate(spec, g, t_cpu, cores)
        if i >= args.warmup:
            times.append(dt)
    sec = statistics.mean(times)
    value = pts * t_cpu / sec / 1e9
    desc = (f"C restatement of scalar_reference (the reference is pure Python: nothing to compile), full "
            f"{'x'.join(map(str, cfg['extents']))} grid, {t_cpu} of {cfg['T']} steps per step, timed in the "
            f"step loop, {cores} thread(s)")
    line = {
        "metric": "GStencil/s", "value": value, "unit": "GStencil/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE seeds)",
        "config": {"workload": f"{cfg['name']} {'x'.join(map(str, cfg['extents']))} T={cfg['T']}",
                   "sample_steps": t_cpu},
        "cpu_baseline": {"value": value, "unit": "GStencil/s", "cores": cores, "kind": "port", "sample": desc,
                         "numpy_reference_path": numpy_reference_rate(cfg)},
        "e2e": {"value": value, "unit": "GStencil/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def make_rows(cfg, lo, hi, pinned=True):
    """Rows [lo, hi) (axis 0) of make_grid(cfg)'s padded array, exactly: the
    PCG64 stream is advanced past the earlier rows (one 64-bit draw per
    double), so a rank materialises only its own slab.  Returns (array of the
    padded rows offset+lo .. offset+hi-1, padded shape, offset)."""
    from paper_2010_04868_b200 import Grid, _native

    probe = Grid((1,) * len(cfg["extents"]), 1)
    off = probe.offset
    padded = tuple(off + e + 1 + probe.vl for e in cfg["extents"])
    shape = (hi - lo,) + padded[1:]
    a = _native.host_empty(shape) if pinned else np.empty(shape)
    a.fill(0.0)
    rng = np.random.default_rng(cfg["seed"])
    row = int(np.prod(cfg["extents"][1:]))
    rng.bit_generator.advance(lo * row)
    win = (slice(None),) + tuple(slice(off, off + e) for e in cfg["extents"][1:])
    a[win] = rng.uniform(cfg["dist"][0], cfg["dist"][1], size=(hi - lo,) + tuple(cfg["extents"][1:]))
    return a, padded, off


def _slab_layout(cfg, part, row0, padded, off):
    """tvs_layout of the WHOLE padded grid whose base pointer is placed so
    that padded row off+row0 is part[0] (the library only touches the rows a
    shard owns / reads)."""
    import ctypes as C

    from paper_2010_04868_b200 import _native

    lay = _native.Layout()
    lay.dim = len(padded)
    for d in range(3):
        lay.extents[d] = cfg["extents"][d] if d < lay.dim else 1
        lay.shape[d] = padded[d] if d < lay.dim else 1
    lay.offset = off
    row_bytes = int(np.prod(padded[1:])) * 8
    return lay, C.c_void_p(part.ctypes.data - (off + row0) * row_bytes)


def run_sharded(args):
    """torchrun, one process per GPU: slab-sharded Jacobi through the fused
    peer-memory path (tvs_shard_*: each rank's kernels store the neighbour's
    ghost rows into its buffer over NVLink; CUDA IPC handles exchanged with
    torch.distributed).  TVS_BENCH_HALO=nccl runs the NCCL send/recv halo
    module (halo.ShardedJacobi) instead.  Strong scaling, max over ranks."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2010_04868_b200 import _native
    from paper_2010_04868_b200.catalog import get

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={world}")
    local = int(os.environ.get("LOCAL_RANK", rank))
    if local >= torch.cuda.device_count() and torch.cuda.device_count() == 1:
        local = 0  # the launcher gave each rank its own CUDA_VISIBLE_DEVICES
    backend = "nccl"
    if os.environ.get("TVS_BENCH_EMULATE_SHARDS"):
        # plumbing check on a box with fewer GPUs than ranks: ranks share
        # devices (round robin) and talk over gloo; never a bench number
        local %= torch.cuda.device_count()
        backend = "gloo"
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    red = "cuda" if backend == "nccl" else "cpu"
    cfg = CONFIGS[args.config]
    if not cfg["shards"]:
        cfg = CONFIGS[HEADLINE]
    if os.environ.get("TVS_BENCH_HALO") == "nccl":
        return run_sharded_nccl(args, cfg, rank, world, local)
    spec = get(cfg["kernel"]).spec
    sh = _native.Shard(spec, cfg["extents"], world, rank, _native.make_exec(device=local))
    handles = [None] * world
    dist.all_gather_object(handles, sh.export())
    sh.connect(handles[rank - 1] if rank > 0 else None, handles[rank + 1] if rank + 1 < world else None)
    r0, r1 = sh.rows
    e0 = cfg["extents"][0]
    lo, hi = max(r0 - sh.ghost, 0), min(r1 + sh.ghost, e0)
    h_in, padded, off = make_rows(cfg, lo, hi)
    h_out = _native.host_empty((r1 - r0,) + padded[1:])
    lay_in, p_in = _slab_layout(cfg, h_in, lo, padded, off)
    lay_out, p_out = _slab_layout(cfg, h_out, r0, padded, off)
    lib = _native.lib()
    stream = torch.cuda.ExternalStream(sh.stream_handle())
    clk = ClockSampler(local) if rank == 0 else None

    def upload():
        _native.check(lib.tvs_shard_upload(sh._h, C.byref(lay_in), p_in), "tvs_shard_upload")

    def download():
        _native.check(lib.tvs_shard_download(sh._h, C.byref(lay_out), p_out), "tvs_shard_download")

    def timed(e2e):
        times, launches = [], 0
        if not e2e:
            upload()
            sh.synchronize()
        for i in range(args.warmup + args.steps):
            dist.barrier()  # every shard idle: neighbours write into each other's buffers
            torch.cuda.synchronize()
            if i == args.warmup and clk is not None and not e2e:
                clk.start()
                clk.wait_ready()
                clk.mark(True)
            e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0_.record(stream)
            if e2e:
                upload()
                sh.synchronize()
                dist.barrier()  # all slabs resident before any pass writes a neighbour
            sh.run(cfg["T"])
            if e2e:
                download()
            e1_.record(stream)
            sh.synchronize()
            if i >= args.warmup:
                t = torch.tensor([e0_.elapsed_time(e1_)], device=red)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                c = torch.tensor([sh.last_launches()], device=red, dtype=torch.int64)
                dist.all_reduce(c, op=dist.ReduceOp.SUM)
                times.append(float(t.item()))
                launches += int(c.item())
        if clk is not None and not e2e:
            clk.mark(False)
            clk.stop()
        return statistics.mean(times), launches

    ms, launches = timed(False)
    ems, _ = timed(True)
    updates = int(np.prod(cfg["extents"])) * cfg["T"]
    h2d = torch.tensor([(hi - lo) * int(np.prod(cfg["extents"][1:])) * 8], device=red, dtype=torch.int64)
    dist.all_reduce(h2d, op=dist.ReduceOp.SUM)
    if rank == 0:
        hbm_peak, peak_src = peaks()
        achieved = BYTES_PER_UPDATE * updates / world / (ms * 1e-3) / 1e9
        print(json.dumps({
            "metric": "GStencil/s", "value": updates / (ms * 1e-3) / 1e9, "unit": "GStencil/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE seeds)",
            "config": {"workload": f"{cfg['name']} {'x'.join(map(str, cfg['extents']))} T={cfg['T']}",
                       "parallelism": f"slab{world} (axis-0 slabs, ghost depth {sh.ghost}, halo exchange fused "
                                      f"into the kernels as peer-memory stores; CUDA IPC)",
                       "l2": "inputs larger than L2",
                       **({"emulated": "ranks share devices: plumbing check, not a bench number"}
                          if backend != "nccl" else {})},
            "gpu_launches": launches, "clocks": clk.summary() if clk else None,
            "e2e": {"value": updates / (ems * 1e-3) / 1e9, "unit": "GStencil/s", "ms_per_step": ems,
                    "h2d_bytes_per_step": int(h2d.item()), "d2h_bytes_per_step": int(updates / cfg["T"] * 8),
                    "note": "per rank: upload own slab + ghosts from pinned host memory, T steps, download own rows"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": None, "per": "GPU (16 B/update effective)",
                         "peak_source": peak_src},
        }))
    dist.barrier()
    sh.close()
    dist.destroy_process_group()
    return 0


def run_sharded_nccl(args, cfg, rank, world, local):
    """The NCCL send/recv halo module (halo.ShardedJacobi): the non-fused
    baseline of the sharded path."""
    import torch
    import torch.distributed as dist

    from paper_2010_04868_b200 import _native
    from paper_2010_04868_b200.catalog import get
    from paper_2010_04868_b200.halo import ShardedJacobi

    spec = get(cfg["kernel"]).spec
    depth = 8 if len(cfg["extents"]) == 2 else 2
    sj = ShardedJacobi(spec, cfg["extents"], dist, depth=depth, device=torch.device("cuda", local))
    lay = sj.layout
    lo, hi = max(lay.r0 - lay.ghost, 0), min(lay.r1 + lay.ghost, int(lay.geometry.axis0_global))
    part, _, off = make_rows(cfg, lo, hi, pinned=False)
    win = (slice(None),) + tuple(slice(off, off + e) for e in cfg["extents"][1:])
    h_in = torch.from_numpy(np.ascontiguousarray(part[win])).pin_memory()
    h_out = torch.empty(tuple(sj.owned().shape), dtype=torch.float64).pin_memory()
    in_view = sj.interior_view
    clk = ClockSampler(local) if rank == 0 else None

    def load():
        v = in_view(0)
        v[lo - (lay.r0 - lay.ghost): hi - (lay.r0 - lay.ghost)].copy_(h_in, non_blocking=True)

    def timed(e2e):
        times, launches = [], 0
        for i in range(args.warmup + args.steps):
            sj.cur = 0
            if not e2e:
                load()
            dist.barrier()
            torch.cuda.synchronize()
            if i == args.warmup and clk is not None and not e2e:
                clk.start()
                clk.wait_ready()
                clk.mark(True)
            _native.launch_counter()  # reset
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if e2e:
                load()
            sj.run(cfg["T"])
            if e2e:
                h_out.copy_(sj.owned(), non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            n = _native.launch_counter()
            dist.barrier()
            if i >= args.warmup:
                t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                c = torch.tensor([n], device="cuda", dtype=torch.int64)
                dist.all_reduce(c, op=dist.ReduceOp.SUM)
                times.append(float(t.item()))
                launches += int(c.item())
        if clk is not None and not e2e:
            clk.mark(False)
            clk.stop()
        return statistics.mean(times), launches

    ms, launches = timed(False)
    ems, _ = timed(True)
    updates = int(np.prod(cfg["extents"])) * cfg["T"]
    if rank == 0:
        hbm_peak, peak_src = peaks()
        achieved = BYTES_PER_UPDATE * updates / world / (ms * 1e-3) / 1e9
        print(json.dumps({
            "metric": "GStencil/s", "value": updates / (ms * 1e-3) / 1e9, "unit": "GStencil/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE seeds)",
            "config": {"workload": f"{cfg['name']} {'x'.join(map(str, cfg['extents']))} T={cfg['T']}",
                       "parallelism": f"slab{world} (axis-0 slabs, NCCL send/recv halo depth {depth})",
                       "l2": "inputs larger than L2"},
            "gpu_launches": launches, "clocks": clk.summary() if clk else None,
            "e2e": {"value": updates / (ems * 1e-3) / 1e9, "unit": "GStencil/s", "ms_per_step": ems,
                    "h2d_bytes_per_step": int(h_in.numel() * 8 * world), "d2h_bytes_per_step": int(updates / cfg["T"] * 8)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": None, "per": "GPU", "peak_source": peak_src},
        }))
    dist.destroy_process_group()
    return 0


def run_in_process(args):
    """--gpus N without torchrun: one process drives N GPUs through the
    library's own sharding (tvs_exec.n_gpus: axis-0 slabs, fused peer-memory
    halo exchange, per-GPU uploads / downloads).  Configs that do not shard
    (1D, Gauss-Seidel) run as N independent replicas."""
    from paper_2010_04868_b200 import _native, config

    n = args.gpus
    have = _native.device_count()
    emulate = bool(os.environ.get("TVS_BENCH_EMULATE_SHARDS"))
    if have < n and not emulate:
        raise SystemExit(f"bench.py --gpus {n}: only {have} CUDA device(s) visible")
    cfg = CONFIGS[args.config]
    if not cfg["shards"]:
        cfg = CONFIGS[HEADLINE]
    with config.using(n_gpus=n, emulate_shards=emulate and have < n):
        head = measure_config(cfg, args.steps, args.warmup, with_e2e=True, with_cpu=False)
    print(json.dumps({
        "metric": "GStencil/s", "value": head["value"], "unit": "GStencil/s", "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE seeds)",
        "config": {"workload": head["workload"], "l2": "inputs larger than L2",
                   "parallelism": f"slab{n} in one process (tvs_exec.n_gpus; halo exchange fused into the kernels "
                                  f"as peer-memory stores)",
                   **({"emulated": f"{n} shards on {have} device(s): plumbing check, not a bench number"}
                      if have < n else {})},
        "gpu_launches": head["gpu_launches"], "clocks": head["clocks"], "e2e": head.get("e2e"),
        "roofline": head["roofline"], "fp64": head["fp64"],
    }))
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--no-all", action="store_true", help="skip the per_stencil sweep of the other configs")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or os.environ.get("TVS_FORCE_SHARDED"):
        # TVS_FORCE_SHARDED=1 under torchrun --nproc-per-node 1: the sharded
        # path with one rank (exercises the plumbing on one GPU)
        return run_sharded(args)
    if args.gpus > 1:
        return run_in_process(args)
    cfg = CONFIGS[args.config]
    head = measure_config(cfg, args.steps, args.warmup, with_e2e=True, with_cpu=not args.no_cpu, with_stock=True)
    line = {
        "metric": "GStencil/s", "value": head["value"], "unit": "GStencil/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE seeds)",
        "config": {"workload": head["workload"], "l2": "inputs larger than L2 (2.1 GB per grid)",
                   "parallelism": "single GPU", "fma": "exact (power-of-two weights fused bit-identically)"},
        "gpu_launches": head["gpu_launches"], "clocks": head["clocks"], "e2e": head.get("e2e"),
        "e2e_stock": head.get("e2e_stock"),
        "roofline": head["roofline"], "fp64": head["fp64"], "cpu_baseline": head.get("cpu_baseline"),
    }
    try:  # whole-grid parity at full size (tests/test_full_grid.py, committed evidence)
        with open(os.path.join(ROOT, "profiles", "parity.json")) as fh:
            line["parity"] = json.load(fh)
    except Exception:
        line["parity"] = None
    line["untiled"] = untiled_legs(args)
    line["integer"] = integer_legs(args)
    if not args.no_all:
        per = {}
        for cid, c in CONFIGS.items():
            if cid == args.config:
                continue
            try:
                r = measure_config(c, max(2, min(args.steps, 3)), args.warmup, with_e2e=True,
                                   with_cpu=not args.no_cpu, min_timed_s=0.25)
                per[c["name"]] = {k: r[k] for k in ("value", "unit", "ms_per_step", "steps", "workload", "roofline",
                                                     "fp64", "e2e", "cpu_baseline", "clocks", "launches_per_step")
                                  if k in r}
                if c["name"] == "3d27p_jacobi":
                    # north_star tolerance mode: fused multiply-add (<= 1e-12 max relative
                    # error vs the oracle, tests/test_gpu_parity.py::test_fma_policies);
                    # `value` above stays the bit-exact default of the public API
                    clk = ClockSampler()
                    ft, _ = device_time(c, max(2, min(args.steps, 3)), args.warmup, sampler=clk, fma="allow")
                    fms = statistics.mean(ft)
                    fv = int(np.prod(c["extents"])) * c["T"] / (fms * 1e-3) / 1e9
                    hbm_peak, _ = peaks()
                    per[c["name"]]["fma_allow"] = {
                        "value": fv, "unit": "GStencil/s", "ms_per_step": fms, "clocks": clk.summary(),
                        "roofline": {"bound": "hbm", "achieved": fv * BYTES_PER_UPDATE, "peak": hbm_peak,
                                     "unit": "GB/s", "frac": fv * BYTES_PER_UPDATE / hbm_peak},
                        "note": "fma='allow': 27 DFMA per update instead of 27 DMUL + 26 DADD; within the "
                                "north_star 1e-12 relative tolerance, not bit-exact"}
                if c["name"] == "2d9p_gauss_seidel":
                    # the reference oracle's own update order (anti-diagonal
                    # gather/scatter, baselines.py:83-107): hyperplane wavefront
                    clk = ClockSampler()
                    rt, rl = device_time(c, 2, args.warmup, sampler=clk, order="reference")
                    rms = statistics.mean(rt)
                    rv = int(np.prod(c["extents"])) * c["T"] / (rms * 1e-3) / 1e9
                    per[c["name"]]["reference_order"] = {
                        "value": rv, "unit": "GStencil/s", "ms_per_step": rms, "launches_per_step": rl,
                        "clocks": clk.summary(),
                        "note": "order='reference' (gs_wave_kernel, one grid barrier per hyperplane i+j+3t)"}
            except Exception as exc:  # report, never hide
                per[c["name"]] = {"error": repr(exc)}
        line["per_stencil"] = per
    print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())
