"""K1 (specdec_verify) latency micro-benchmark: N back-to-back launches captured in one CUDA
graph, per-launch time from CUDA events.

    python tools/k1bench.py [--B 8] [--k 5] [--V 151936] [--n 50]

SPECDEC_K1_EXP=1 times the argmax phase alone (no grid-wide arrival / epilogue), =2 an empty
kernel on the same grid (the launch floor), =3 the loads and per-thread max only (no CTA
reduction), =4 up to the CTA maximum (no pass 2), =5 up to pass 2 (no merge), =6 the
grid-wide arrival without the epilogue -- results invalid, for splitting the latency.
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
from synth import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=8)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--V", type=int, default=151936)
    ap.add_argument("--n", type=int, default=50)
    ap.add_argument("--ring", type=int, default=16, help="logits buffers (16 at Qwen3 B=8 > L2)")
    ap.add_argument("--pool", action="store_true",
                    help="specdec_pool_verify (the pool's K1 with the fused write-back) instead")
    a = ap.parse_args()
    dev = torch.device("cuda")
    B, k, V = a.B, a.k, a.V
    ring = [W.gen_logits_torch(0, r, B, k, V, "bf16", dev) for r in range(a.ring)]
    draft = torch.from_numpy(W.gen_round_truth(0, 0, B, k, V, "alpha").draft).to(dev)
    i32, i64, u8 = torch.int32, torch.int64, torch.uint8
    n = torch.full((B,), 100, dtype=i32, device=dev)
    act = torch.ones(B, dtype=u8, device=dev)
    out = [torch.zeros(B, dtype=dt, device=dev) for dt in (i32, i64, i32, u8)]
    plan = [torch.zeros(1, dtype=i32, device=dev)] + [torch.zeros(B, dtype=i32, device=dev) for _ in range(3)]
    ws = torch.zeros((_abi.specdec_verify_workspace_size(B, k) + 7) // 8, dtype=i64, device=dev)

    # pool mode: B member rows of a pool of 4B sequences with room for every launch's tokens
    N, max_new = 4 * B, 1 << 20
    members = torch.arange(B, dtype=i32, device=dev)
    p_len = torch.full((N,), 100, dtype=i32, device=dev)
    p_gen = torch.zeros(N, dtype=i32, device=dev)
    p_act = torch.ones(N, dtype=u8, device=dev)

    def call(lg, stream=None):
        if a.pool:
            _abi.specdec_pool_verify(lg, draft, members, n, act, *out, p_len, p_gen, p_act, ws, max_new=max_new,
                                     stream=stream)
        else:
            _abi.specdec_verify(lg, draft, n, act, *out, plan[0], plan[1], plan[2], plan[3], ws, stream=stream)

    def one(j):
        act.fill_(1)
        call(ring[j % len(ring)])
    for j in range(3):
        one(j)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for j in range(a.n):
            call(ring[j % len(ring)], stream=s)
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
    mb = B * (k + 1) * V * 2 / 1e6
    print(json.dumps({"B": B, "k": k, "V": V, "us_per_launch": round(best, 2), "logits_MB": round(mb, 2),
                      "GBps": round(mb * 1e3 / best, 1), "ring_MB": round(mb * len(ring), 1), "exp": os.environ.get("SPECDEC_K1_EXP", "0"),
                      "split": os.environ.get("SPECDEC_K1_SPLIT", "default"), "pool": a.pool,
                      "pdl": os.environ.get("SPECDEC_PDL", "1")}))


if __name__ == "__main__":
    main()
