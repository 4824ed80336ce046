"""GPU-side brute force (SURVEY §4 tier 2):

  * K1 -> K3 -> K2 over EVERY content-length vector n in {1..k+1}^B and EVERY accept vector
    a in {0..k}^B, for B <= 3 and k <= 4 (22,100 rounds), through the native round driver:
    accept, bonus, emit, kept, L', n', p', tokens', masks, positions and the whole KV
    buffer of every case against oracle.verify / oracle.align;
  * K4 over EVERY window of W <= 6 sequences with lengths in {1, 2, 3}, every batch size
    B <= W and every min_group in 1..B+1: the whole plan and its counters against
    oracle.pool.form_batches.

The rounds are enqueued back to back with their results copied into history buffers on
the device; the comparison runs once at the end."""
import itertools

import numpy as np
import pytest
import torch

from oracle import align as OA
from oracle import pool as OP
from oracle import verify as OV
from paper_2510_22876_b200.eqspec import EqSpecBatch
from tests.test_gpu_pool import _check_plan, _plan_gpu

pytestmark = pytest.mark.gpu

V, D = 16, 8


def _cases(B, k):
    return [(n, a) for n in itertools.product(range(1, k + 2), repeat=B)
            for a in itertools.product(range(0, k + 1), repeat=B)]


@pytest.mark.parametrize("B,k", [(1, 1), (1, 4), (2, 1), (2, 2), (2, 3), (2, 4), (3, 1), (3, 2), (3, 3), (3, 4)])
def test_round_brute_force(cuda, B, k):
    cases = _cases(B, k)
    C = len(cases)
    assert C == (k + 1) ** (2 * B)
    cap = 2 * (k + 1) + k + 4
    rng = np.random.default_rng(B * 10 + k)
    # per-case inputs, built on the host and uploaded once
    tok = np.zeros((C, B, cap), np.int64)
    nn = np.zeros((C, B), np.int32)
    pd = np.zeros((C, B), np.int32)
    lg = np.zeros((C, B, k + 1, V), np.float32)
    dr = np.zeros((C, B, k), np.int64)
    for c, (n, a) in enumerate(cases):
        n = np.array(n, np.int32)
        L = int(n.max())
        nn[c], pd[c] = n, L - n
        for i in range(B):
            tok[c, i, L - n[i]:L] = rng.integers(2, V, n[i])
            tgt = rng.integers(0, V, k + 1)
            lg[c, i, np.arange(k + 1), tgt] = 1.0                       # planted argmax per slot
            d = rng.integers(0, V, k)
            d[:a[i]] = tgt[:a[i]]                                       # accepted prefix
            if a[i] < k:
                d[a[i]] = (tgt[a[i]] + 1 + rng.integers(V - 1)) % V     # first mismatch
            dr[c, i] = d
    # initial KV: every (plane, row, column) entry tagged with its identity
    kv0 = np.zeros((2, B, 1, cap, D), np.int16)
    pl, i_, _, col, d_ = np.indices(kv0.shape)
    kv0[:] = ((pl * 4 + i_) * 64 + col) * 8 + d_
    dev = lambda x: torch.from_numpy(x).to(cuda)
    tok_d, nn_d, pd_d, lg_d, dr_d = dev(tok), dev(nn), dev(pd), dev(lg), dev(dr)
    kv0_d = dev(kv0).view(torch.bfloat16)
    bt = EqSpecBatch(B, k, cap, 1, 1, D, "bf16", cuda)
    bt.V = V
    i32, i64 = torch.int32, torch.int64
    h = dict(accept=torch.zeros((C, B), dtype=i32, device=cuda), bonus=torch.zeros((C, B), dtype=i64, device=cuda),
             emit=torch.zeros((C, B), dtype=i32, device=cuda), kept=torch.zeros((C, B), dtype=i32, device=cuda),
             L=torch.zeros((C, 1), dtype=i32, device=cuda), n=torch.zeros((C, B), dtype=i32, device=cuda),
             pad=torch.zeros((C, B), dtype=i32, device=cuda), tok=torch.zeros((C, B, cap), dtype=i64, device=cuda),
             mask=torch.zeros((C, B, cap + k), dtype=i64, device=cuda),
             pos=torch.zeros((C, B, cap + k), dtype=i64, device=cuda),
             kv=torch.zeros((C,) + kv0.shape, dtype=torch.int16, device=cuda))
    for c in range(C):
        bt.cur = 0
        bt.tok[0].copy_(tok_d[c])
        bt.n[0].copy_(nn_d[c])
        bt.pad[0].copy_(pd_d[c])
        bt.active.fill_(1)
        bt.kv.copy_(kv0_d)
        bt.mask.fill_(-1)
        bt.pos.fill_(-1)
        bt.step(lg_d[c], dr_d[c], V=V)                  # native driver: K1 -> K3 -> K2
        for key, src in (("accept", bt._accept[0]), ("bonus", bt._bonus[0]), ("emit", bt._emit[0]),
                         ("kept", bt.kept), ("L", bt.plan_L), ("n", bt.n[1]), ("pad", bt.pad[1]),
                         ("tok", bt.tok[1]), ("mask", bt.mask), ("pos", bt.pos), ("kv", bt.kv.view(torch.int16))):
            h[key][c].copy_(src)
    torch.cuda.synchronize()
    g = {key: t.cpu().numpy() for key, t in h.items()}
    assert int(bt.status.item()) == 0
    ones = np.ones(B, np.uint8)
    for c, (n, a) in enumerate(cases):
        n = np.array(n, np.int32)
        L = int(n.max())
        bits = lg[c]
        v = OV.batch_verify(bits, "fp32", dr[c], n, L - n, ones)
        assert list(v["accept"]) == list(a), c                 # the construction's intent
        for key in ("accept", "bonus", "emit", "kept"):
            assert np.array_equal(g[key][c], v[key]), (c, key)
        Ln = v["L_new"]
        assert g["L"][c, 0] == Ln and np.array_equal(g["n"][c], v["n_new"]) and np.array_equal(g["pad"][c], v["pad_new"])
        tok_n, mask_n, pos_n = OA.repad_tokens(tok[c], cap, k, L - n, L, v)
        assert np.array_equal(g["tok"][c][:, :Ln], tok_n[:, :Ln]), c
        assert np.array_equal(g["mask"][c][:, :Ln + k], mask_n) and np.array_equal(g["pos"][c][:, :Ln + k], pos_n), c
        kv_o = OA.realign_kv_inplace(kv0.copy(), L - n, v["pad_new"], v["kept"]) if B > 1 else kv0
        assert np.array_equal(g["kv"][c], kv_o), (c, n, a)


def test_pool_group_brute_force(cuda):
    """K4 on every window of W <= 6 sequences with lengths in {1, 2, 3}, every B <= W and
    every min_group in 1..B+1 (above B too)."""
    cnt = 0
    for Wn in range(1, 7):
        for lens in itertools.product((1, 2, 3), repeat=Wn):
            lens = list(lens)
            order = list(range(Wn))
            for B in range(1, Wn + 1):
                for mg in range(1, B + 2):
                    g = _plan_gpu(cuda, lens, [1] * Wn, order, Wn, B, mg)
                    _check_plan(g, OP.form_batches(lens, [1] * Wn, order, Wn, B, mg), lens, B)
                    cnt += 1
    assert cnt > 10_000


def test_pool_getbatch_brute_force(cuda):
    """Alg. 3's one-batch GetBatch on every window of W <= 6 sequences with lengths in
    {1, 2, 3}, every B <= W and every min_group in 1..B+1: batch 0 == the oracle plan's."""
    from tests.test_gpu_pool import _check_getbatch, _getbatch_gpu
    cnt = 0
    for Wn in range(1, 7):
        for lens in itertools.product((1, 2, 3), repeat=Wn):
            lens = list(lens)
            order = list(range(Wn))
            for B in range(1, Wn + 1):
                for mg in range(1, B + 2):
                    g = _getbatch_gpu(cuda, lens, [1] * Wn, order, Wn, B, mg)
                    _check_getbatch(g, OP.form_batches(lens, [1] * Wn, order, Wn, B, mg), lens, B)
                    cnt += 1
    assert cnt > 10_000


def test_pool_group_deferred_brute_force(cuda):
    """The deferred-fallback plan (R27) on every window of W <= 6 sequences with lengths in
    {1, 2, 3}, every B <= W, min_group in {1, 2, B}, patience 1 and 2, seeded waits in
    {0, 1, 2}: plan, deferred members and updated waits == the oracle's."""
    from tests.test_gpu_pool import _check_deferred, _plan_gpu_deferred
    cnt = 0
    for Wn in range(1, 7):
        for lens in itertools.product((1, 2, 3), repeat=Wn):
            lens = list(lens)
            order = list(range(Wn))
            rng = np.random.default_rng(sum(l * 3 ** i for i, l in enumerate(lens)) + 7 * Wn)
            for B in range(1, Wn + 1):
                for mg in sorted({1, 2, B}):
                    for patience in (1, 2):
                        wait = rng.integers(0, 3, Wn).astype(np.int64)
                        g = _plan_gpu_deferred(cuda, lens, [1] * Wn, order, Wn, B, mg, wait, patience)
                        o_wait = wait.copy()
                        o = OP.form_batches_deferred(lens, [1] * Wn, order, Wn, B, mg, o_wait, patience)
                        _check_deferred(g, o, lens, B, o_wait)
                        cnt += 1
    assert cnt > 10_000
