"""Summarise ncu reports / launch lists into markdown for profiles/.

    python tools/summarize_ncu.py --full gpurun_out/full_c3.ncu-rep ... --launches gpurun_out/launches_c3.csv ...
"""

import argparse
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def stalls(d, n=4):
    items = []
    for k, (v, _) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                items.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    return ", ".join(f"{name} {val:.2f}" for val, name in sorted(items, reverse=True)[:n])


def full_table(paths):
    lines = ["| report | kernel | " + " | ".join(label for _, label in KEYS) + " | top stalls (per issue) |",
             "|---" * (len(KEYS) + 3) + "|"]
    for p in paths:
        d = raw(p)
        name = d.get("Kernel Name", ("?", ""))[0]
        cells = []
        for k, _ in KEYS:
            v, u = d.get(k, ("n/a", ""))
            cells.append(f"{v} {u}".strip())
        lines.append(f"| {p.split('/')[-1]} | `{name[:60]}` | " + " | ".join(cells) + f" | {stalls(d)} |")
    return "\n".join(lines)


def launches_table(path):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    per = {}
    order = []
    for r in rows[start + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"])
        if key not in per:
            per[key] = {}
            order.append(key)
        per[key][d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    agg = {}
    for key in order:
        name = key[1].split("(")[0]
        m = per[key]
        a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += float(m.get("gpu__time_duration.sum", ("0", ""))[0].replace(",", ""))
        for i, k in ((2, "dram__bytes_read.sum"), (3, "dram__bytes_write.sum")):
            v, u = m.get(k, ("0", "byte"))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            a[i] += float(v.replace(",", "")) * scale
    total = sum(a[1] for a in agg.values()) or 1.0
    lines = ["| kernel | launches | total time (ns, cold, serialised) | share | DRAM read (B) | DRAM write (B) |",
             "|---|---|---|---|---|---|"]
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{name}` | {a[0]} | {a[1]:.0f} | {a[1] / total:.1%} | {a[2]:.3e} | {a[3]:.3e} |")
    return "\n".join(lines)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--launches", nargs="*", default=[])
    a = ap.parse_args()
    if a.full:
        print(full_table(a.full))
        print()
    for p in a.launches:
        print(f"#### {p.split('/')[-1]}\n")
        print(launches_table(p))
        print()
