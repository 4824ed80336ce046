"""Every cell of tools/bench_matrix.py checked against the oracle on its first rounds
(SURVEY §8(d) bench matrix: "every cell also runs the bit-exact oracle comparison on its
first rounds").

Each round cell builds bench.py's own RoundBench from the cell's command-line arguments
(shape, B, context, accept pattern, in-place / ping-pong KV, anchored origin, draft KV) and
replays its first rounds from the bench's captured per-round graphs.  After every round:
accept, bonus, emit, finished, kept, L', n', p', tokens', masks and positions are compared
element by element with oracle.verify / oracle.align, and so are sampled KV slabs --
whole (plane, row, head) slabs of the target cache (and of the draft cache), every byte,
both buffers in ping-pong mode, physical columns with the anchored origin -- modelled with
the K2 contract (destination ranges move, nothing else changes; oracle.align.copy_rows).

Each pool cell builds the bench's pool (N, prompt lengths, window, min_group, Alg. 3 mode,
consumer, executor) and runs its first epoch (or Alg. 3 iterations) through the native
executor exactly as bench.run_pool does; the plan, every integer of the pool state and
the untouched KV prefix of sampled sequences are compared with the oracle's Alg. 3.

tools/bench_matrix.py runs this file first and prints each cell's verdict next to its
numbers.
"""
import os
import sys

import numpy as np
import pytest
import torch

import bench
from oracle import align as OA
from oracle import pool as OP
from oracle import verify as OV
from synth import workloads as W
from tests.gpu_helpers import torch_to_bits

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import bench_matrix  # noqa: E402

pytestmark = pytest.mark.gpu

N_SAMPLES = 24


class SlabModel:
    """Sampled (plane, row, head) slabs of one KV cache ([planes, B, H, cap_phys, D]
    buffers, one or two), kept as host copies and advanced with the oracle's row move."""

    def __init__(self, bufs, seed, gen_bufs, rng, B):
        self.bufs = bufs                           # the device buffers ([0] or [0, 1])
        P, _, H, capp, D = bufs[0].shape
        self.keys = sorted({(int(rng.integers(P)), int(rng.integers(B)), int(rng.integers(H)))
                            for _ in range(N_SAMPLES)})   # distinct slabs (small shapes repeat)
        per = capp * D
        self.host = []
        for bi in range(len(bufs)):
            d = {}
            for (pl, i, h) in self.keys:
                if bi in gen_bufs:                  # filled by the bench from the generator
                    off = ((pl * B + i) * H + h) * per
                    d[(pl, i, h)] = W.gen_kv_bits_np(seed, per, offset=off).reshape(capp, D)
                else:                               # allocated zero, never filled
                    d[(pl, i, h)] = np.zeros((capp, D), np.uint16)
            self.host.append(d)

    def move(self, src_b, dst_b, src_col, dst_col, count):
        """K2 contract on every sampled slab: dst[dcol + c] = src[scol + c], c < count."""
        for (pl, i, h) in self.keys:
            s = self.host[src_b][(pl, i, h)]
            d = self.host[dst_b][(pl, i, h)]
            c = int(count[i])
            rows_s = s[None, None, None]            # [1, 1, 1, cap, D] logical rows view
            rows_d = d[None, None, None]
            OA.copy_rows(rows_s, rows_d, [c], src_col=[int(src_col[i])], dst_col=[int(dst_col[i])])

    def compare(self, tag):
        for bi, buf in enumerate(self.bufs):
            for (pl, i, h) in self.keys:
                got = torch_to_bits(buf[pl, i, h])
                assert np.array_equal(got, self.host[bi][(pl, i, h)]), (tag, bi, pl, i, h)


def _round_cell(cuda, cli, rounds=3):
    args = bench.parse(cli)
    sh = bench.shape_for(args)
    total = args.warmup + args.steps + 2
    rb = bench.RoundBench(sh, args, cuda, total)
    bt, k = rb.bt, sh.k
    bt.V = sh.V
    bt.capture(list(zip(rb.logits, rb.drafts)), V=sh.V)      # the bench's per-round graphs
    rb.reset()
    torch.cuda.synchronize()
    rng = np.random.default_rng(11)
    two = bt.kv_mode == "pingpong"
    tgt = SlabModel(bt._kvbuf, args.seed, {0}, rng, sh.B)
    drf = SlabModel(bt._dkvbuf, args.seed + 1, {0}, rng, sh.B) if bt._dkvbuf is not None else None
    tok, n = rb.tokens.copy(), rb.lengths.astype(np.int32)
    L = int(n.max())
    pad = (L - n).astype(np.int32)
    act = np.ones(sh.B, np.uint8)
    base = bt.anchor_slack
    bits = [W.gen_logits_np(args.seed, j, sh.B, k, sh.V, sh.logit_dtype) for j in range(min(rounds, bench.RING))]
    for r in range(rounds):
        j = r % bench.RING
        parity = bt.cur
        bt.replay(j)
        v = OV.batch_verify(bits[j], sh.logit_dtype, rb.truth[j].draft, n, pad, act)
        tok_n, mask_n, pos_n = OA.repad_tokens(tok, rb.cap, k, pad, L, v)
        src_b, dst_b = (parity, 1 - parity) if two else (0, 0)
        if bt.anchor is not None:
            base, col_old, col_new = OA.anchor_plan(pad, v["pad_new"], v["kept"], v["finished"], v["accept"], L,
                                                    v["L_new"], base, bt.cap_phys, k)
        else:
            col_old, col_new = pad, v["pad_new"]
        if sh.B > 1 or bt.anchor is not None or two:     # B = 1 in place: K2 is not launched (no move)
            tgt.move(src_b, dst_b, col_old, col_new, v["kept"])
            if drf is not None:
                drf.move(src_b, dst_b, col_old, col_new, v["kept_draft"])
        torch.cuda.synchronize()
        tag = f"{cli} round {r}"
        for key, g in (("accept", bt._accept[parity]), ("bonus", bt._bonus[parity]), ("emit", bt._emit[parity]),
                       ("finished", bt._finished[parity]), ("kept", bt.kept)):
            assert np.array_equal(g.cpu().numpy(), v[key]), (tag, key)
        if drf is not None:
            assert np.array_equal(bt.kept_draft.cpu().numpy(), v["kept_draft"]), tag
        Ln = v["L_new"]
        c = bt.cur
        assert int(bt.plan_L.item()) == Ln, tag
        assert np.array_equal(bt.n[c].cpu().numpy(), v["n_new"]), tag
        assert np.array_equal(bt.pad[c].cpu().numpy(), v["pad_new"]), tag
        assert np.array_equal(bt.tok[c][:, :Ln].cpu().numpy(), tok_n[:, :Ln]), tag
        assert np.array_equal(bt.mask[:, :Ln + k].cpu().numpy(), mask_n), tag
        assert np.array_equal(bt.pos[:, :Ln + k].cpu().numpy(), pos_n), tag
        if bt.anchor is not None:
            assert bt.base() == base, tag
        assert int(bt.status.item()) == 0, tag
        tgt.compare(tag)
        if drf is not None:
            drf.compare(tag + " (draft KV)")
        tok, n, pad, L = tok_n, v["n_new"], v["pad_new"], Ln
        act = (v["finished"] == 0).astype(np.uint8)


ROUND_CELLS = [(lbl, cli) for lbl, cli in bench_matrix.CELLS]


@pytest.mark.parametrize("label,cli", ROUND_CELLS, ids=[c[0] for c in ROUND_CELLS])
def test_round_cell(cuda, label, cli):
    _round_cell(cuda, cli)
    torch.cuda.empty_cache()


# ----------------------------------------------------------------------------- pool cells
def _pool_cell(cuda, cli, seqs_checked=16):
    from paper_2510_22876_b200.exspec import SequencePool
    args = bench.parse(cli)
    if args.emulate_ranks > 1:        # one shard of the emulation: rank 0 of G, as run_pool
        world, rank = args.emulate_ranks, 0
    else:
        world, rank = 1, 0
    sh = W.SHAPES["qwen3"]
    k, V, B = sh.k, sh.V, sh.B
    lens, order = bench.pool_workload(args)
    from paper_2510_22876_b200.dist import shard_balanced, shard_bands, shard_strided
    if args.shard == "balanced":
        shards = shard_balanced(order, world, np.asarray(lens, np.float64) + args.shard_c * args.max_new)
    else:
        shards = (shard_bands if args.shard == "band" else shard_strided)(order, world)
    mine = shards[rank]
    n_loc = len(mine)
    cap = ((int(lens.max()) + args.max_new + k + 1) + 15) // 16 * 16
    Wn = min(args.pool_W or n_loc, 2048, n_loc)
    Bp = min(B, Wn)
    sp = SequencePool(n_loc, cap, sh.layers, sh.H, sh.D, k, W=Wn, B=Bp, min_group=args.min_group,
                      max_new=args.max_new, device=cuda, kv_init=False,
                      dense_consumer=args.pool_consumer == "dense",
                      n_staging=args.pool_staging if args.pool_exec == "native" else 1,
                      patience=args.pool_patience,
                      pipeline=bool(args.pool_pipeline) and args.pool_mode == "epoch")
    local_lens = lens[mine]
    local_order = np.arange(n_loc)
    seed = args.seed
    sp.load(local_lens, order=local_order)
    per = sp.kv[0].numel()
    rng = np.random.default_rng(5)
    checked = sorted(set(int(x) for x in rng.integers(0, n_loc, seqs_checked)))
    for s in checked:                 # known bytes in the sampled slots only
        sp.kv[s].copy_(W.gen_kv_torch(seed + s, sp.kv[s].shape, sp.kv.dtype, cuda))
    before = {s: torch_to_bits(sp.kv[s][:, :, :int(local_lens[s]) - 1]) for s in checked}
    ring_lg = [W.gen_logits_torch(seed, r, Bp, k, V, sh.logit_dtype, cuda) for r in range(bench.RING)]
    truth = [W.gen_round_truth(seed, r, Bp, k, V, args.pattern, alpha=args.alpha) for r in range(bench.RING)]
    ring_dr = [torch.from_numpy(t.draft).to(cuda) for t in truth]
    bits = [W.gen_logits_np(seed, r, Bp, k, V, sh.logit_dtype) for r in range(bench.RING)]
    assert args.pool_exec == "native"
    sp.native(list(zip(ring_lg, ring_dr)), V=V, logit_dtype=ring_lg[0].dtype)
    o_len, o_gen, o_act = local_lens.astype(np.int64), np.zeros(n_loc, np.int64), np.ones(n_loc, np.uint8)
    o_tok, o_out = np.zeros((n_loc, cap), np.int64), np.zeros((n_loc, args.max_new), np.int64)
    sp.tokens.zero_()
    ring_pos = 0

    def oracle_batch(mem, b_len, j):
        nbat, act = np.ones(Bp, np.int32), np.zeros(Bp, np.uint8)
        nbat[:len(mem)] = o_len[mem]
        act[:len(mem)] = 1
        budget = np.array([args.max_new - o_gen[s] for s in mem] + [1] * (Bp - len(mem)))
        v = OV.batch_verify(bits[j], sh.logit_dtype, truth[j].draft, nbat, b_len - nbat, act, -1, budget)
        OP.writeback(o_len, o_gen, o_act, o_tok, o_out, mem, v["E"], v["finished"])

    if args.pool_mode == "alg3":
        iters = 24
        sp.alg3_native(iters)
        for it in range(iters):
            plan = OP.form_batches(o_len, o_act, local_order, Wn, Bp, args.min_group)
            if not plan["batches"]:
                break
            oracle_batch(plan["batches"][0], plan["blen"][0], (ring_pos + it) % bench.RING)
    else:
        # with deferred fallback (R27) the waits matter from the second epoch on: 4 epochs;
        # pipelined fallback (R28): the last plan's mixed members sit the next plan out
        o_wait = np.zeros(n_loc, np.int64)
        inflight = []
        for _ in range(4 if args.pool_patience > 0 or sp.pipeline else 1):
            plan = OP.form_batches_deferred(o_len, OP.pipeline_window_active(o_act, inflight), local_order, Wn,
                                            Bp, args.min_group, o_wait, args.pool_patience)
            inflight = OP.mixed_members(plan) if sp.pipeline else []
            ran = sp.epoch_native()[0]
            assert ran == len(plan["batches"])
            for b, mem in enumerate(plan["batches"]):
                oracle_batch(mem, plan["blen"][b], (ring_pos + b) % bench.RING)
            ring_pos += ran
        assert np.array_equal(sp.wait.cpu().numpy(), o_wait)
    torch.cuda.synchronize()
    tag = str(cli)
    assert np.array_equal(sp.len.cpu().numpy(), o_len), tag
    assert np.array_equal(sp.gen.cpu().numpy(), o_gen), tag
    assert np.array_equal(sp.active.cpu().numpy(), o_act), tag
    tg, og = sp.tokens.cpu().numpy(), sp.out_buf.cpu().numpy()
    for s in range(n_loc):
        lo = int(local_lens[s])
        assert np.array_equal(tg[s, lo:o_len[s]], o_tok[s, lo:o_len[s]]), (tag, s)
        assert np.array_equal(og[s, :o_gen[s]], o_out[s, :o_gen[s]]), (tag, s)
    for s in checked:                 # the KV a sequence had before is never disturbed
        lo = int(local_lens[s]) - 1
        assert np.array_equal(torch_to_bits(sp.kv[s][:, :, :lo]), before[s]), (tag, s)
    assert int(sp.status.item()) == 0, tag


POOL_CELLS = [(lbl, cli) for lbl, cli in bench_matrix.POOL]


@pytest.mark.parametrize("label,cli", POOL_CELLS, ids=[c[0] for c in POOL_CELLS])
def test_pool_cell(cuda, label, cli):
    _pool_cell(cuda, cli)
    torch.cuda.empty_cache()
