"""Build profiles/traffic.json (DRAM bytes per launch / per update of each
config's dominant kernel) from the ncu launch lists tools/evidence.sh writes:

    python tools/make_traffic.py gpurun_out/launches_c{1..5}.csv > profiles/traffic.json
    python tools/make_traffic.py --full-T gpurun_out/r02_launches_c{1..5}.csv   (round 2: full-T runs)
"""
import csv
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
T_PROFILED = {1: 1000, 2: 1000, 3: 16, 4: 100, 5: 2}  # --T used by tools/evidence.sh
if "--full-T" in sys.argv:  # tools/evidence_r02.sh profiles every config at its full T
    sys.argv.remove("--full-T")
    T_PROFILED = {c: bench.CONFIGS[c]["T"] for c in bench.CONFIGS}
HELPERS = ("fill_halo", "gsl_sentinel", "shard_signal", "shard_fill")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    per = {}
    for r in rows[start + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        m = per.setdefault(d["ID"], {"name": d["Kernel Name"]})
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
        m[d["Metric Name"]] = v
    return list(per.values())


out = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 "--clock-control none (" + ", ".join(os.path.basename(x) for x in sys.argv[1:]) + ")", "configs": {}}
for path in sys.argv[1:]:
    cid = int(re.search(r"c(\d)", os.path.basename(path)).group(1))
    cfg = bench.CONFIGS[cid]
    ls = [x for x in launches(path) if not any(h in x["name"] for h in HELPERS)]
    if not ls:
        continue
    name = ls[0]["name"].split("(")[0].replace("void ", "")
    n = len(ls)
    dram = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in ls) / n
    ns = sum(x.get("gpu__time_duration.sum", 0) for x in ls) / n
    upd = float(1)
    for e in cfg["extents"]:
        upd *= e
    upd *= T_PROFILED[cid] / n
    out["configs"][str(cid)] = {"launches_profiled": n, "dram_bytes_per_launch": dram, "ns_per_launch_cold": ns,
                                "kernel": name, "updates_per_launch": upd, "dram_bytes_per_update": dram / upd,
                                "note": f"{cfg['name']}, T={T_PROFILED[cid]} profiled; per-launch averages"}
print(json.dumps(out, indent=1))
