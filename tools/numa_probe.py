"""Duplex PCIe rate vs the NUMA node of the page-locked host buffers.

Prints the GPU's PCI NUMA node and local CPUs, then, in fresh processes
pinned to (a) no affinity, (b) the GPU-local CPUs, (c) the other CPUs,
allocates two 2 GiB tvs_host_alloc buffers and times H2D + D2H at once."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gpu_pci():
    out = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", "0"],
                         capture_output=True, text=True).stdout.strip()
    dom, bus, rest = out.split(":")
    return f"{int(dom, 16):04x}:{bus.lower()}:{rest.lower()}"


def parse_list(s):
    cpus = set()
    for part in s.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


def child():
    import torch

    sys.path.insert(0, ROOT)
    from paper_2010_04868_b200 import _native

    n = 2 * 2 ** 30 // 8
    a, b = _native.host_empty((n,)), _native.host_empty((n,))
    a[...] = 1.0
    b[...] = 1.0
    ha, hb = torch.from_numpy(a), torch.from_numpy(b)
    d1 = torch.empty(n, dtype=torch.float64, device="cuda")
    d2 = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        with torch.cuda.stream(s1):
            d1.copy_(ha, non_blocking=True)
        with torch.cuda.stream(s2):
            hb.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{os.environ.get('PROBE_LABEL', '?'):12s} duplex 2 x 2 GiB: {best:.1f} ms", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
        sys.exit(0)
    bus = gpu_pci()
    base = f"/sys/bus/pci/devices/{bus}"
    node = open(f"{base}/numa_node").read().strip() if os.path.exists(f"{base}/numa_node") else "?"
    local = parse_list(open(f"{base}/local_cpulist").read()) if os.path.exists(f"{base}/local_cpulist") else set()
    allc = os.sched_getaffinity(0)
    print(f"GPU {bus}: numa_node {node}, {len(local)} local CPUs of {len(allc)} available", flush=True)
    for label, cpus in (("none", None), ("local", local & allc), ("remote", allc - local)):
        if cpus is not None and not cpus:
            print(f"{label}: no CPUs")
            continue
        env = dict(os.environ, PROBE_LABEL=label)
        pre = (lambda c=cpus: os.sched_setaffinity(0, c)) if cpus else None
        subprocess.run([sys.executable, __file__, "child"], env=env, preexec_fn=pre, timeout=300)
