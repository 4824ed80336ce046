"""Kernel micro-benchmarks for K2 (specdec_realign_kv) against a live copy peak.

    python tools/kbench.py [--gb 2.4] [--reps 20]

Reports GB/s (bytes read + written, CUDA events) for:
  copy_      torch out-of-place copy of the same byte count (live peak reference)
  k2_oop     specdec_realign_kv moving every slab to a distinct buffer (pure copy)
  k2_shift   specdec_realign_kv in place, every row shifted by +5 / -5 positions
  k2_mixed   in place, the bench's Qwen3 B=8 shift mix (~65% of rows move)
--gather N: the EXSpec pool's fallback gather / scatter geometry (pool of N sequences).
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
    ap.add_argument("--seg", action="store_true", help="SPECDEC_SEGMENTED (in-place segmented slabs)")
    ap.add_argument("--dyn", action="store_true", help="SPECDEC_DYNAMIC (work tickets)")
    ap.add_argument("--gather", type=int, default=0,
                    help="EXSpec pool gather/scatter geometry instead: pool of N sequences")
    a = ap.parse_args()
    if a.gather:
        return gather_bench(a)
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

    ws = torch.zeros(_abi.specdec_realign_workspace_size(kv.dtype, P, B, H, D, cap), dtype=torch.uint8,
                     device=dev) if (a.seg or a.dyn) else None
    kflags = (_abi.SEGMENTED if a.seg else 0) | (_abi.DYNAMIC if a.dyn else 0)

    def k2(src, dst, po, pn, kp):
        _abi.specdec_realign_kv(src, dst, i32(kp), n_planes=P, n_rows=B, H=H, D=D, src_strides=s,
                                dst_strides=s, cap_src=cap, cap_dst=cap, src_col=i32(po), dst_col=i32(pn),
                                ws=ws, flags=kflags)

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


def gather_bench(a):
    """The pool's fallback-batch KV moves (bench.py --config pool): gather B members of a
    pool [N][planes][H][cap][D] into a staging rectangle [planes][B][H][cap][D] right-aligned
    at the batch width, and scatter a+1 rows per member back."""
    import numpy as np
    dev = torch.device("cuda")
    N, P, B, H, cap, D = a.gather, a.planes, a.B, a.H, a.cap, 128
    pool = torch.empty(N, P, H, cap, D, dtype=torch.bfloat16, device=dev)
    stg = torch.empty(P, B, H, cap, D, dtype=torch.bfloat16, device=dev)
    ps, ss = pool.stride(), stg.stride()
    rng = np.random.default_rng(0)
    i32 = lambda v: torch.tensor(np.asarray(v), dtype=torch.int32, device=dev)
    res = {}
    for trial in range(4):
        members = rng.choice(N, B, replace=False)
        lens = rng.integers(64, cap - 16, B)
        L = int(lens.max())
        cnt, pad, mem = i32(lens), i32(L - lens), i32(members)
        acc = i32(rng.integers(0, 6, B))
        moved = torch.zeros(1, dtype=torch.int64, device=dev)

        def gather():
            _abi.specdec_realign_kv(pool, stg, cnt, count_add=-1, n_planes=P, n_rows=B, H=H, D=D,
                                    src_strides=(ps[1], ps[0], ps[2]), dst_strides=ss[:3], cap_src=cap,
                                    cap_dst=cap, dst_col=pad, src_row_map=mem, moved_bytes=moved)

        def scatter():
            _abi.specdec_realign_kv(stg, pool, acc, count_add=1, n_planes=P, n_rows=B, H=H, D=D,
                                    src_strides=ss[:3], dst_strides=(ps[1], ps[0], ps[2]), cap_src=cap,
                                    cap_dst=cap, src_col_add=L - 1, dst_col=cnt, dst_col_add=-1,
                                    dst_row_map=mem, moved_bytes=moved, count_bound=6)
        gb = 2 * int((lens - 1).sum()) * P * H * D * 2
        sb = 2 * int((acc.cpu().numpy() + 1).sum()) * P * H * D * 2
        tg = timed(gather, a.reps)
        ts = timed(scatter, a.reps)
        res[f"t{trial}"] = {"gather_MB": round(gb / 1e6, 1), "gather_us": round(tg * 1e3, 1),
                            "gather_GBps": round(gb / tg / 1e6, 1), "scatter_MB": round(sb / 1e6, 2),
                            "scatter_us": round(ts * 1e3, 1),
                            "both_GBps": round((gb + sb) / (tg + ts) / 1e6, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
