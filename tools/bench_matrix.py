"""SURVEY §8d bench matrix: runs bench.py over the cells and prints one summary line per
cell (plus the raw JSON lines to --jsonl).  Every cell is first checked against the oracle
on its first rounds / epoch (tests/test_gpu_bench_cells.py, one pytest run for all cells)
and its verdict printed with its numbers; each cell's value is the median of --reps timed
repetitions (default 5).

    python tools/bench_matrix.py [--quick] [--reps 5] [--no-oracle] [--jsonl out.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import xml.etree.ElementTree as ET

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ROUND = ["--no-cpu-baseline", "--no-e2e"]
CELLS = (
    # (label, args)
    [(f"Q{B} {m}", ["--B", str(B), "--kv-mode", m]) for B in (1, 2, 4, 8) for m in ("inplace", "pingpong")]
    + [(f"Q8 ctx{c}", ["--ctx", str(c)]) for c in (512, 1024, 2048, 4096)]
    + [(f"Q8 alpha{a}", ["--pattern", "fixed", "--alpha", str(a)]) for a in (0.3, 0.5, 0.8)]
    + [(f"Q8 {p}", ["--pattern", p]) for p in ("all_k", "all_0", "alternating", "one_zero")]
    + [("Q8 anchored", ["--anchor"]), ("Q8 draft-kv", ["--draft-kv"])]
    + [(f"V8 {m}", ["--config", "vicuna", "--kv-mode", m]) for m in ("inplace", "pingpong")]
    + [(f"G8 {m}", ["--config", "glm4", "--kv-mode", m]) for m in ("inplace", "pingpong")]
    + [("T toy", ["--config", "toy"])]
)
POOL = (
    [(f"P N{n} {ln}", ["--config", "pool", "--pool-n", str(n), "--pool-lengths", ln])
     for n in (64, 256, 1024) for ln in ("random", "uniform")]
    + [(f"P N1024 W{w}", ["--config", "pool", "--pool-W", str(w)]) for w in (8, 16, 32)]
    + [("P N1024 min_group 8", ["--config", "pool", "--min-group", "8"]),
       ("P N1024 alg3", ["--config", "pool", "--pool-mode", "alg3"]),
       # the epoch plan: R11's full plan (patience 0) and deferred fallback (R27; default 2)
       ("P N1024 patience 0", ["--config", "pool", "--pool-patience", "0"]),
       ("P N1024 patience 1", ["--config", "pool", "--pool-patience", "1"]),
       ("P N1024 patience 4", ["--config", "pool", "--pool-patience", "4"]),
       ("P N1024 W32 patience 0", ["--config", "pool", "--pool-W", "32", "--pool-patience", "0"]),
       ("P N1024 pipelined fallback", ["--config", "pool", "--pool-pipeline", "1"]),
       ("P N1024 emulated x8 patience 0", ["--config", "pool", "--emulate-ranks", "8", "--pool-patience", "0"]),
       ("P N1024 emulated x8 patience 1", ["--config", "pool", "--emulate-ranks", "8", "--pool-patience", "1"]),
       ("P N1024 dense consumer", ["--config", "pool", "--pool-consumer", "dense"]),
       ("P N1024 slot consumer", ["--config", "pool", "--pool-consumer", "slot"]),
       ("P N1024 serial executor", ["--config", "pool", "--pool-staging", "1"]),
       ("P N1024 emul x8 count bands", ["--config", "pool", "--emulate-ranks", "8", "--shard", "band"])]
    + [(f"P N1024 emulated x{g}", ["--config", "pool", "--emulate-ranks", str(g)]) for g in (2, 4, 8)]
)


def summary(label, d):
    if "emulated" in d:
        e = d["emulated"]
        return (f"{label:26s} {d['value']:10.1f} seq/s predicted (slowest of {e['ranks']} shards, each drained "
                f"alone)  per-rank ms {[round(x, 1) for x in e['per_rank_ms']]}  max/mean "
                f"{e['imbalance_max_over_mean']:.3f}")
    if "pool" in d:
        p = d["pool"]
        return (f"{label:26s} {d['value']:10.1f} seq/s  grouping {p['grouping_rate']:.3f}  "
                f"batches {p['batch_verifications']:6d}  mean_batch {p['mean_batch']:.2f}  "
                f"KV {p['kv_bytes_moved_rank0'] / 1e9:8.1f} GB  K2 {d['roofline']['achieved']:7.1f} GB/s")
    r = d["roofline"]
    k = d["kernels_ms_per_step"]
    return (f"{label:26s} {d['value']:10.1f} rounds/s  {d['ms_per_step'] * 1e3:8.1f} us  "
            f"K2 {r['achieved']:7.1f} GB/s (frac {r['frac']:.3f}, copied {r.get('copied_GBps', 0):7.1f})  "
            f"K1 {k['verify_K1'] * 1e3:5.1f} K3 {k['repad_K3'] * 1e3:5.1f} K2 {k['realign_K2'] * 1e3:7.1f} us")


def oracle_verdicts(quick):
    """Run the per-cell oracle checks once; returns {cell label: "pass" | "FAIL" | "skip"}."""
    xml = os.path.join(tempfile.mkdtemp(), "cells.xml")
    sel = ["-k", "test_round_cell"] if quick else []
    subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_bench_cells.py"), "-q",
                    "-m", "gpu", f"--junitxml={xml}"] + sel, cwd=ROOT, capture_output=True, text=True, timeout=3600)
    res = {}
    for tc in ET.parse(xml).getroot().iter("testcase"):
        name = tc.get("name")
        label = name[name.index("[") + 1:-1] if "[" in name else name
        bad = tc.find("failure") is not None or tc.find("error") is not None
        res[label] = "FAIL" if bad else ("skip" if tc.find("skipped") is not None else "pass")
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="round cells only")
    ap.add_argument("--reps", type=int, default=5, help="timed repetitions per cell (median reported)")
    ap.add_argument("--no-oracle", action="store_true", help="skip the per-cell oracle checks")
    ap.add_argument("--jsonl", default="")
    a = ap.parse_args()
    cells = [(lbl, ROUND + args) for lbl, args in CELLS]
    if not a.quick:
        cells += [(lbl, ["--no-cpu-baseline"] + args) for lbl, args in POOL]
    verdict = {} if a.no_oracle else oracle_verdicts(a.quick)
    out = open(a.jsonl, "w") if a.jsonl else None
    # cell K4: the plan alone (tools/k4bench.py: 50 plans per CUDA graph, best of 5), W in
    # {32, 128, 1024} (+2048); its plans are checked bit-exact against the oracle by
    # tests/test_gpu_pool.py (random pools, the W=2048 window, the fuzz)
    for extra, tag in (([], "K4"), (["--getbatch"], "K4 getbatch")):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "k4bench.py")] + extra, capture_output=True,
                           text=True, timeout=600)
        for ln in r.stdout.strip().splitlines():
            if ln.startswith("{"):
                d = json.loads(ln)
                if out:
                    out.write(json.dumps({"cell": f"{tag} W{d['W']} mg{d['min_group']}", **d}) + "\n")
                print(f"{tag + ' W%d min_group %d' % (d['W'], d['min_group']):26s} {d['us_per_plan']:8.2f} us per "
                      f"plan  batches {d['n_batches']:4d}  (N={d['N']}, B={d['B']})", flush=True)
    for lbl, args in cells:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--reps", str(a.reps)] + args,
                           capture_output=True, text=True, timeout=1800)
        lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
        if r.returncode or not lines:
            print(f"{lbl:26s} FAILED rc={r.returncode} {r.stderr.strip().splitlines()[-1:]}", flush=True)
            continue
        d = json.loads(lines[-1])
        d["oracle_check"] = verdict.get(lbl, "not run")
        if out:
            out.write(json.dumps({"cell": lbl, **d}) + "\n")
        print(f"{summary(lbl, d)}  oracle {d['oracle_check']}", flush=True)


if __name__ == "__main__":
    main()
