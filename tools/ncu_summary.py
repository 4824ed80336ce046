"""Summarise ncu captures for profiles/: launch-list shares and full-set metrics.

    python tools/ncu_summary.py launches <launches.csv>
    python tools/ncu_summary.py full <prof.ncu-rep> [--launch-log bytes.json --index i]

`full` prints duration, DRAM bytes (read + write), throughput and occupancy for each
captured kernel; with a launch log (bench.py SPECDEC_BENCH_LAUNCH_LOG) it compares the
captured K2 launch's DRAM traffic with its algorithmic bytes.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "lts__t_bytes.sum", "launch__shared_mem_per_block_dynamic"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9,
         "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-6) * 1e6
            agg[r[ki].split("(")[0]].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"{k:60s} n={len(v):4d} mean={sum(v) / len(v):9.2f}us share={sum(v) / tot * 100:5.1f}%")
    return "\n".join(out)


def full(path, launch_log=None, index=0):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                try:
                    d[w] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    d[w] = r[i]
        d["dram_bytes"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        res.append(d)
    if launch_log:
        lb = json.load(open(launch_log))["realign_bytes_per_launch"][index]
        for d in res:
            if "realign" in d["kernel"]:
                d["algorithmic_bytes"] = lb
                d["traffic_over_algorithmic"] = d["dram_bytes"] / lb if lb else None
                d["achieved_GBps_ncu"] = lb / d["gpu__time_duration.sum"] / 1e9
    return res


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        ll = sys.argv[sys.argv.index("--launch-log") + 1] if "--launch-log" in sys.argv else None
        ix = int(sys.argv[sys.argv.index("--index") + 1]) if "--index" in sys.argv else 0
        print(json.dumps(full(sys.argv[2], ll, ix), indent=1))
