"""How often does an EXSpec fallback batch re-form with exactly the same members in the next
epoch?  (VERDICT r1 "Next" #3: would keeping a fallback batch's staging resident and
realigning it in place, instead of re-gathering it, save KV traffic?)

Drives the pool workload of `bench.py --config pool` (same lengths, order, logits ring and
drafts, so the same plans) through SequencePool.plan (K4) and specdec_pool_verify on the
GPU -- the KV gathers do not change any plan, so they are skipped -- and records every
epoch's fallback batches.  A fallback batch of epoch e+1 "repeats" when its ordered member
list equals a fallback batch of epoch e; `repeat_gather_bytes` are the bytes such repeats
would not re-gather (2 (len-1) bpt per member, as bench's accounting).

    python tools/pool_repeats.py [--pool-n 1024] [--ranks G]
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

from paper_2510_22876_b200.dist import shard_balanced  # noqa: E402
from paper_2510_22876_b200.exspec import SequencePool  # noqa: E402
from synth import workloads as W  # noqa: E402

RING = 16


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pool-n", type=int, default=1024)
    ap.add_argument("--ranks", type=int, default=1)
    ap.add_argument("--max-new", type=int, default=256)
    a = ap.parse_args()
    dev = torch.device("cuda")
    sh = W.SHAPES["qwen3"]
    k, V, B = sh.k, sh.V, sh.B
    N = a.pool_n
    h = W.hash_np(0, W.S_POOL, np.arange(N))
    lens = (64 + (h % np.uint64(449)).astype(np.int64)).astype(np.int32)
    order = np.array(sorted(range(N), key=lambda s: (int(lens[s]), s)), np.int32)
    shards = shard_balanced(order, a.ranks, np.asarray(lens, np.float64) + a.max_new)
    ring_lg = [W.gen_logits_torch(0, r, B, k, V, sh.logit_dtype, dev) for r in range(RING)]
    ring_dr = [torch.from_numpy(W.gen_round_truth(0, r, B, k, V, "alpha").draft).to(dev) for r in range(RING)]
    out = []
    for g, mine in enumerate(shards):
        n_loc = len(mine)
        cap = ((int(lens.max()) + a.max_new + k + 1) + 15) // 16 * 16
        sp = SequencePool(n_loc, cap, 1, 1, 8, k, W=min(n_loc, 2048), B=B, min_group=2, max_new=a.max_new,
                          device=dev, kv_init=False)
        sp.load(lens[mine], order=np.arange(n_loc))
        prev, i, stats = set(), 0, dict(epochs=0, fallback_batches=0, repeats=0, fallback_members=0,
                                        fallback_gather_bytes=0, repeat_gather_bytes=0)
        while True:
            nb, kinds, blens, sizes = sp.plan()
            if nb == 0:
                break
            mem = sp.members[:nb].cpu().numpy()
            ln = sp.mlen[:nb].cpu().numpy()
            cur = set()
            for b in range(nb):
                if not kinds[b]:
                    t = tuple(int(x) for x in mem[b, :sizes[b]])
                    by = int(2 * (ln[b, :sizes[b]].astype(np.int64) - 1).sum() * sh.bpt)
                    cur.add(t)
                    stats["fallback_batches"] += 1
                    stats["fallback_members"] += int(sizes[b])
                    stats["fallback_gather_bytes"] += by
                    if t in prev:
                        stats["repeats"] += 1
                        stats["repeat_gather_bytes"] += by
                sp.verify_writeback(b, ring_lg[i % RING], ring_dr[i % RING], V)
                i += 1
            prev = cur
            stats["epochs"] += 1
        stats.update(rank=g, seqs=n_loc, batches=i)
        out.append(stats)
        print(json.dumps(stats), flush=True)
    tot = {key: sum(s[key] for s in out) for key in ("fallback_batches", "repeats", "fallback_gather_bytes",
                                                   "repeat_gather_bytes")}
    tot["repeat_share_of_gather_bytes"] = tot["repeat_gather_bytes"] / max(1, tot["fallback_gather_bytes"])
    print(json.dumps({"ranks": a.ranks, "total": tot}))


if __name__ == "__main__":
    main()
