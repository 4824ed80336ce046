"""Grouping-rate sweep of EXSpec's same-length scheduling (Fig. 6c analog, PAPER.md:650, 700;
SURVEY §8f row f2) on the GPU path (K4 plan + verify + write-back; tiny KV since the rate
depends only on lengths and acceptance).

    python tools/grouping_sweep.py [--n 256] [--max-new 64]

Prints one line per (lengths, B, min_group, W, mode): grouping rate (same-length batches /
all batches), batch verifications, mean batch size, epochs.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_22876_b200.exspec import SequencePool  # noqa: E402
from synth import workloads as W  # noqa: E402


def drain(N, lens, B, mg, Wn, k, V, max_new, mode, dev, seed=0):
    sp = SequencePool(N, int(lens.max()) + max_new + k + 8, 1, 1, 8, k, W=Wn, B=B, min_group=mg,
                      max_new=max_new, device=dev)
    order = np.array(sorted(range(N), key=lambda s: (int(lens[s]), s)), np.int32)
    sp.load(lens, order=order)
    ring = [(W.gen_logits_torch(seed, r, B, k, V, "bf16", dev),
             torch.from_numpy(W.gen_round_truth(seed, r, B, k, V, "alpha").draft).to(dev)) for r in range(16)]
    ctr = [0]

    def inputs(b):
        ctr[0] += 1
        return ring[ctr[0] % 16]
    epochs = ran = same = members = 0
    while True:
        nb, kinds, blens, sizes = sp.plan()
        if nb == 0:
            break
        epochs += 1
        for b in range(1 if mode == "alg3" else nb):     # count the batches that RAN
            lg, d = inputs(b)
            sp.run_batch(b, kinds[b], blens[b], lg, d, V=V)
            ran += 1
            same += int(kinds[b])
            members += int(sizes[b])
    return dict(rate=same / max(1, ran), verifies=ran, mean_bs=members / max(1, ran), epochs=epochs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--max-new", type=int, default=64)
    a = ap.parse_args()
    dev = torch.device("cuda")
    k, V, N = 5, 1024, a.n
    h = W.hash_np(0, W.S_POOL, np.arange(N))
    kinds = {"random U[64,512]": (64 + (h % np.uint64(449)).astype(np.int64)).astype(np.int32),
             "uniform 256 (All-Mean)": np.full(N, 256, np.int32)}
    print(f"# N={N} sequences, max_new={a.max_new}, k={k}, alpha_i~U[0.5,0.9], sort on")
    print("# lengths | B | min_group | W | mode | grouping_rate | batch_verifications | mean_batch | epochs")
    for name, lens in kinds.items():
        for B in (2, 4, 8, 16, 32):
            for mg in sorted({2, B}):
                for Wn, mode in ((N, "epoch"), (4 * B, "epoch"), (4 * B, "alg3")):
                    r = drain(N, lens, B, mg, min(Wn, N), k, V, a.max_new, mode, dev)
                    print(f"{name} | {B} | {mg} | {Wn} | {mode} | {r['rate']:.3f} | {r['verifies']} | "
                          f"{r['mean_bs']:.2f} | {r['epochs']}", flush=True)


if __name__ == "__main__":
    main()
