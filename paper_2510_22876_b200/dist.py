"""Multi-GPU EXSpec: shard the SequencePool over the GPUs of one box.

The pool partitions into independent units (sequences): every rank groups, verifies
and realigns its own shard with no collective inside an epoch or a round.  The only
exchange is one all-gather of the finished outputs and counters at the end of the run
(NCCL over NVLink on GPUs; gloo in the CPU tests), so scaling is bounded by the shard
imbalance, not by communication.

Sharding: the admission order (ascending prompt length when sorting is on)
is cut into contiguous bands of ~N/G sequences, so each rank's window sees similar
lengths and same-length grouping stays high (0.81 band vs 0.47 strided).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_bands(order, world: int):
    """Contiguous bands of the admission order: rank g gets order[g*N/G : (g+1)*N/G]."""
    order = np.asarray(order)
    N = len(order)
    cuts = [(g * N) // world for g in range(world + 1)]
    return [order[cuts[g]:cuts[g + 1]].copy() for g in range(world)]


def shard_balanced(order, world: int, weights):
    """Contiguous bands of the admission order with equal total weight instead of equal
    counts: band g ends at the first position whose cumulative weight reaches (g+1)/G of
    the total.  With weights = a per-sequence cost estimate (bench.py: prompt length +
    max_new -- KV bytes grow with the length, plus a per-sequence latency share), the
    long-prompt bands get fewer sequences and the slowest rank finishes sooner."""
    order = np.asarray(order)
    w = np.asarray(weights, np.float64)[order]
    cum = np.cumsum(w)
    tot = cum[-1] if len(cum) else 0.0
    cuts = [0] + [int(np.searchsorted(cum, tot * (g + 1) / world - 1e-9) + 1) for g in range(world - 1)] + [len(order)]
    cuts = np.maximum.accumulate(np.minimum(cuts, len(order)))
    return [order[cuts[g]:cuts[g + 1]].copy() for g in range(world)]


def shard_strided(order, world: int):
    order = np.asarray(order)
    return [order[g::world].copy() for g in range(world)]


def gather_results(ids_local, out_local, gen_local, counters_local, N: int, max_new: int,
                   group=None, device=None):
    """All-gather every rank's finished sequences into the global [N, max_new] output
    buffer (ids_local: global sequence ids of this rank's rows) and sum the counters.
    One collective per tensor, at the end of the run."""
    world = dist.get_world_size(group)
    dev = device or torch.device("cpu")
    n_loc = torch.tensor([len(ids_local)], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n_loc, group=group)
    m = int(max(int(s.item()) for s in sizes))
    pad_ids = torch.full((m,), -1, dtype=torch.int64, device=dev)
    pad_ids[:len(ids_local)] = torch.as_tensor(np.asarray(ids_local), dtype=torch.int64, device=dev)
    pad_out = torch.zeros((m, max_new), dtype=torch.int64, device=dev)
    pad_out[:len(ids_local)] = torch.as_tensor(out_local, dtype=torch.int64, device=dev)
    pad_gen = torch.zeros(m, dtype=torch.int64, device=dev)
    pad_gen[:len(ids_local)] = torch.as_tensor(np.asarray(gen_local), dtype=torch.int64, device=dev)
    all_ids = torch.empty((world * m,), dtype=torch.int64, device=dev)
    all_out = torch.empty((world * m, max_new), dtype=torch.int64, device=dev)
    all_gen = torch.empty((world * m,), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(all_ids, pad_ids, group=group)
    dist.all_gather_into_tensor(all_out, pad_out, group=group)
    dist.all_gather_into_tensor(all_gen, pad_gen, group=group)
    cnt = torch.as_tensor(np.asarray(counters_local), dtype=torch.int64, device=dev).clone()
    dist.all_reduce(cnt, group=group)
    ids = all_ids.cpu().numpy()
    keep = ids >= 0
    out = np.zeros((N, max_new), np.int64)
    gen = np.zeros(N, np.int64)
    out[ids[keep]] = all_out.cpu().numpy()[keep]
    gen[ids[keep]] = all_gen.cpu().numpy()[keep]
    return out, gen, cnt.cpu().numpy()
