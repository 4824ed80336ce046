"""The sharded EXSpec pool on the CUDA path: two ranks -- gloo, both on cuda:0
(the GPU box has one GPU) -- each drain their band of the pool through libspecdec.so with
the toy LM, then the end-of-run all-gather (dist.gather_results) assembles the outputs.
Every sequence's output must equal per-sequence greedy decoding and the 1-rank
libspecdec run, token for token (the sharded GPU pool's gathered outputs were
never compared with a 1-rank run)."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.test_dist import _free_port

pytestmark = pytest.mark.gpu

N, K, MAX_NEW, WN, B, MG = 14, 3, 12, 7, 3, 2


def _worker(rank, world, port, q):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pool import admission_order
        from oracle.toy_lm import ToyLM
        from paper_2510_22876_b200.dist import gather_results, shard_bands
        from tests.test_gpu_toylm import D, H, LAYERS, V, _exspec_gpu, _prompts
        cuda = torch.device("cuda:0")
        T = ToyLM(V, LAYERS, H, D, seed=7)
        prompts = _prompts(N, seed=91)
        order = admission_order([len(p) for p in prompts], True)
        mine = shard_bands(order, world)[rank]
        outs, _, status = _exspec_gpu(cuda, T, [prompts[s] for s in mine], K, MAX_NEW, min(WN, len(mine)),
                                      min(B, len(mine)), MG)
        out_loc = np.zeros((len(mine), MAX_NEW), np.int64)
        gen_loc = np.zeros(len(mine), np.int64)
        for j, o in enumerate(outs):
            out_loc[j, :len(o)] = o
            gen_loc[j] = len(o)
        out, gen, cnt = gather_results(mine, out_loc, gen_loc, [status, 0, 0, 0, 0, 0, 0, 0], N, MAX_NEW)
        if rank == 0:
            q.put(([list(out[s, :gen[s]]) for s in range(N)], int(cnt[0])))
    finally:
        dist.destroy_process_group()


def test_sharded_gpu_pool_equals_one_rank_and_greedy(cuda):
    from oracle.toy_lm import ToyLM
    from tests.test_gpu_toylm import D, H, LAYERS, V, _exspec_gpu, _prompts
    T = ToyLM(V, LAYERS, H, D, seed=7)
    prompts = _prompts(N, seed=91)
    ref = [T.greedy_generate(p, MAX_NEW, 1, 64) for p in prompts]
    one, _, st = _exspec_gpu(cuda, T, prompts, K, MAX_NEW, WN, B, MG)
    assert one == ref and st == 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    two, status_sum = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert two == one == ref and status_sum == 0
