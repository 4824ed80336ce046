"""Kernel micro-benchmarks for K2 (specdec_realign_kv) against a live copy peak.

    python tools/kbench.py [--gb 2.4] [--reps 20]

Reports GB/s (bytes read + written, CUDA events) for:
  copy_      torch out-of-place copy of the same byte count (live peak reference)
  k2_oop     specdec_realign_kv moving every slab to a distinct buffer (pure copy)
  k2_shift   specdec_realign_kv in place, every row shifted by +5 / -5 positions
  k2_mixed   in place, the bench's Qwen3 B=8 shift mix (~65% of rows move)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_22876_b200 import _abi  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--planes", type=int, default=72)
    ap.add_argument("--B", type=int, default=8)
    ap.add_argument("--H", type=int, default=8)
    ap.add_argument("--cap", type=int, default=2304)
    ap.add_argument("--kept", type=int, default=2000)
    ap.add_argument("--seg", action="store_true", help="pass a workspace (segmented slabs)")
    a = ap.parse_args()
    dev = torch.device("cuda")
    P, B, H, cap, D = a.planes, a.B, a.H, a.cap, 128
    kv = torch.randn(P, B, H, cap, D, device=dev).to(torch.bfloat16)
    kv2 = torch.empty_like(kv)
    s = kv.stride()[:3]
    i32 = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)
    res = {}
    nbytes = kv.numel() * 2
    ms = timed(lambda: kv2.copy_(kv), a.reps)
    res["copy_"] = 2 * nbytes / ms / 1e6
    kept = [a.kept] * B
    slab = P * H * a.kept * D * 2

    ws = torch.empty(_abi.specdec_realign_workspace_size(kv.dtype, P, B, H, D, cap), dtype=torch.uint8,
                     device=dev) if a.seg else None

    def k2(src, dst, po, pn, kp):
        _abi.specdec_realign_kv(src, dst, i32(kp), n_planes=P, n_rows=B, H=H, D=D, src_strides=s,
                                dst_strides=s, cap_src=cap, cap_dst=cap, src_col=i32(po), dst_col=i32(pn),
                                ws=ws)

    ms = timed(lambda: k2(kv, kv2, [0] * B, [0] * B, kept), a.reps)
    res["k2_oop"] = 2 * slab * B / ms / 1e6
    state = {"up": True}

    def shift():
        po, pn = ([0] * B, [5] * B) if state["up"] else ([5] * B, [0] * B)
        state["up"] = not state["up"]
        k2(kv, kv, po, pn, kept)
    ms = timed(shift, a.reps)
    res["k2_shift"] = 2 * slab * B / ms / 1e6
    mv = [i for i in range(B) if i % 3 != 2]          # ~2/3 of rows move

    def mixed():
        po = [0] * B
        pn = [5 if i in mv else 0 for i in range(B)]
        if not state["up"]:
            po, pn = pn, po
        state["up"] = not state["up"]
        k2(kv, kv, po, pn, kept)
    ms = timed(mixed, a.reps)
    res["k2_mixed"] = 2 * slab * len(mv) / ms / 1e6
    res["cfg"] = os.environ.get("SPECDEC_REALIGN_CFG", "0") + ("+seg" if a.seg else "")
    print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in res.items()}))


if __name__ == "__main__":
    main()
