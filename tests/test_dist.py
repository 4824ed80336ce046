"""N > 1 host path of the sharded EXSpec pool on CPU with gloo, world size 2:
band sharding + the end-of-run all-gather reproduce the single-process result exactly."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.loops import exspec_decode
from oracle.pool import admission_order
from oracle.toy_lm import ToyLM
from paper_2510_22876_b200.dist import gather_results, shard_balanced, shard_bands, shard_strided

MAX_NEW, K, CAP = 10, 3, 64


def _prompts(N, seed=0):
    rng = np.random.default_rng(seed)
    return [list(map(int, rng.integers(2, 32, size=int(l)))) for l in rng.integers(1, 14, N)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, prompts, order, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        T = ToyLM(seed=7)
        mine = shard_bands(order, world)[rank]
        outs, st = exspec_decode(T, T, [prompts[s] for s in mine], K, MAX_NEW, 1, CAP,
                                 W=4, B=2, min_group=2, noise=0.3)
        out_loc = np.zeros((len(mine), MAX_NEW), np.int64)
        gen_loc = np.zeros(len(mine), np.int64)
        for j, o in enumerate(outs):
            out_loc[j, :len(o)] = o
            gen_loc[j] = len(o)
        counters = [st["verify_calls"], st["same_length"], 0, 0, 0, 0, 0, 0]
        out, gen, cnt = gather_results(mine, out_loc, gen_loc, counters, len(prompts), MAX_NEW)
        if rank == 0:
            q.put((out, gen, cnt))
    finally:
        dist.destroy_process_group()


def test_shards_are_partitions():
    order = np.random.default_rng(0).permutation(103)
    for G in (1, 2, 4, 8):
        for fn in (shard_bands, shard_strided):
            parts = fn(order, G)
            assert sorted(np.concatenate(parts).tolist()) == list(range(103))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
    assert list(shard_bands(np.arange(8), 2)[1]) == [4, 5, 6, 7]


def test_gloo_world2_matches_single_process():
    prompts = _prompts(12)
    lens = [len(p) for p in prompts]
    order = admission_order(lens, True)
    T = ToyLM(seed=7)
    ref = [T.greedy_generate(p, MAX_NEW, 1, CAP) for p in prompts]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, prompts, order, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, gen, cnt = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = [list(out[s, :gen[s]]) for s in range(len(prompts))]
    assert got == ref            # sharded EXSpec == per-sequence greedy, token for token
    assert cnt[0] > 0


def test_balanced_bands():
    """Equal-weight contiguous bands: a partition of the admission order, in order, whose
    band weights differ by at most one element's weight."""
    rng = np.random.default_rng(3)
    for N, G in ((1024, 8), (37, 4), (5, 8), (8, 2)):
        w = rng.integers(64, 512, N).astype(np.float64) + 256
        order = np.argsort(w, kind="stable")
        sh = shard_balanced(order, G, w)
        assert len(sh) == G and np.array_equal(np.concatenate(sh), order)
        tot = [w[s].sum() for s in sh if len(s)]
        if N >= G:
            assert max(tot) - min(tot) <= 2 * w.max()
    assert [list(s) for s in shard_balanced(np.arange(4), 2, [1, 1, 1, 3])] == [[0, 1, 2], [3]]


@pytest.mark.gpu
def test_nccl_gather_results_world1():
    """The NCCL path of the end-of-run exchange (CUDA tensors, all_gather_into_tensor,
    all_reduce) and bench's max-over-ranks, in a one-rank NCCL group on the one GPU: the
    gathered outputs equal the local ones."""
    import torch
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        ids = np.array([3, 0, 2], np.int64)
        out_loc = np.arange(3 * 5, dtype=np.int64).reshape(3, 5)
        gen_loc = np.array([5, 1, 3], np.int64)
        out, gen, cnt = gather_results(ids, out_loc, gen_loc, [7, 1, 0, 0, 0, 0, 0, 0], 4, 5, device=dev)
        assert np.array_equal(out[ids], out_loc) and np.array_equal(gen[ids], gen_loc) and gen[1] == 0
        assert list(cnt[:2]) == [7, 1]
        assert bench.max_over_ranks(3.5, dev, 2) == 3.5          # the NCCL all_reduce(MAX) path
        assert bench.coll_device(dev) == dev
    finally:
        dist.destroy_process_group()
