"""K4 (specdec_pool_group, or with --getbatch specdec_pool_getbatch) latency: N back-to-back plans captured in one CUDA graph, µs per
plan from CUDA events, for pools of random lengths U[64, 512] (SURVEY §8d cell K4).

    python tools/k4bench.py [--N 1024] [--B 8] [--n 50]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_22876_b200 import _abi  # noqa: E402
from paper_2510_22876_b200.exspec import SequencePool  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--B", type=int, default=8)
    ap.add_argument("--n", type=int, default=50)
    ap.add_argument("--getbatch", action="store_true",
                    help="time specdec_pool_getbatch (Alg. 3's one-batch GetBatch) instead of the full plan")
    a = ap.parse_args()
    dev = torch.device("cuda")
    rng = np.random.default_rng(0)
    out = []
    for Wn in (32, 128, 1024, 2048):
        if Wn > a.N:
            continue
        for mg in (2, a.B):
            sp = SequencePool(a.N, 16, 1, 1, 8, 5, W=Wn, B=a.B, min_group=mg, device=dev)
            lens = rng.integers(64, 513, a.N)
            sp.load(lens, order=np.argsort(lens, kind="stable"))

            fn = _abi.specdec_pool_getbatch if a.getbatch else _abi.specdec_pool_group

            def plan(stream=None):
                fn(sp.len, sp.active, sp.order, sp.W, sp.B, sp.min_group,
                                        sp.window, sp.window_size, sp.batch_of, sp.slot_of,
                                        sp.members, sp.mlen, sp.mpad, sp.mactive, sp.bsize,
                                        sp.bkind, sp.blen, sp.n_batches, sp.counters, stream=stream)
            plan()
            torch.cuda.synchronize()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
                for _ in range(a.n):
                    plan(stream=s)
            torch.cuda.current_stream().wait_stream(s)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e9
            for _ in range(5):
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / a.n * 1e3)
            out.append({"N": a.N, "W": Wn, "B": a.B, "min_group": mg, "getbatch": a.getbatch,
                        "us_per_plan": round(best, 2),
                        "n_batches": int(sp.n_batches.item())})
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
