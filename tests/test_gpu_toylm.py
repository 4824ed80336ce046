"""End-to-end equivalence on the CUDA path (BASELINE.json north_star):
the toy LM (oracle side, CPU, fp64, bf16 KV) supplies logits and KV; every step of the hot
path -- verify, repad/positions/masks, KV realign, pool plan, gather/scatter, write-back --
runs in libspecdec.so.  Batched speculative output must equal per-sequence greedy output
token for token, which only holds if positions, masks and every realigned KV row are
right (SPEC.md:169 alignment soundness)."""
import numpy as np
import pytest
import torch

from oracle.align import build_batch, mask_pos_row
from oracle.loops import draft_cached
from oracle.toy_lm import ToyLM
from paper_2510_22876_b200.eqspec import EqSpecBatch
from paper_2510_22876_b200.exspec import SequencePool

pytestmark = pytest.mark.gpu

V, LAYERS, H, D = 32, 2, 2, 8


def _bits(t):
    return t.detach().cpu().view(torch.int16).numpy().view(np.uint16)


def _to_dev(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(dev).view(torch.bfloat16)


def _prompts(n, seed):
    rng = np.random.default_rng(seed)
    return [list(map(int, rng.integers(2, V, size=int(l)))) for l in rng.integers(1, 15, n)]


def _eqspec_gpu(cuda, T, prompts, k, max_new, eos, noise, cap=64, fault=None, drafter=None,
                draft_log=None, anchor_slack=0, kv_mode="inplace"):
    """EqSpec with the toy LM on the host and K1/K3/K2 in libspecdec.so.  `fault` injects
    one of the paper's §2 failure classes at a module seam.  With a
    `drafter`, the draft model keeps its own KV cache on the GPU, realigned by K2 with
    K1's kept_draft (f1); its proposals are logged next to recompute-mode proposals."""
    B = len(prompts)
    tokens, pad, L = build_batch(prompts, cap)
    bt = EqSpecBatch(B, k, cap, LAYERS, H, D, "bf16", cuda, max_new=max_new, eos_id=eos,
                     draft=None if drafter is None else (LAYERS, H, D), anchor_slack=anchor_slack,
                     kv_mode=kv_mode)
    bt.load(tokens, [len(p) for p in prompts])
    if fault is not None:
        bt.native_round = False    # the faults patch the Python-side calls of the round
    if fault == "skip_kv_realign":             # DSD error (iii): KV not realigned
        bt.realign = lambda stream=None: None
    if fault == "bonus_from_draft":            # DSD error (i): bonus from the draft
        orig = bt.verify

        def verify(logits, draft, stream=None):
            orig(logits, draft, stream)
            a = bt.accept.long().clamp(max=draft.shape[1] - 1)
            bt.bonus.copy_(torch.gather(draft, 1, a[:, None])[:, 0])
        bt.verify = verify
    stale = None
    first = True
    rounds = 0
    for _ in range(128):
        if not bt.active.any().item():
            break
        act = bt.active.cpu().numpy()
        tok = bt.tokens.cpu().numpy()
        pad_c = bt.pad_cur.cpu().numpy()
        L = int((bt.pad_cur + bt.n_cur).max().item())
        if first:
            mask = np.stack([mask_pos_row(int(p), L + k)[0] for p in pad_c])
            pos = np.stack([mask_pos_row(int(p), L + k)[1] for p in pad_c])
        else:                                    # K3's outputs drive the forward
            mask = bt.mask[:, :L + k].cpu().numpy()
            pos = bt.pos[:, :L + k].cpu().numpy()
        if fault == "stale_position_ids":        # BSP: positions not recomputed
            if stale is not None:
                w = min(pos.shape[1], stale.shape[1])
                pos = pos.copy()
                pos[:, :w] = stale[:, :w]
            stale = pos.copy()
        draft = np.zeros((B, k), np.int64)
        if drafter is None:
            for i in range(B):
                if act[i]:
                    draft[i] = T.propose(list(tok[i, pad_c[i]:L]), k, noise)
        else:
            dview = bt.kv_logical(bt.dkv)
            dcache = _bits(dview).copy()
            dkept = bt.kept_draft.cpu().numpy()
            for i in range(B):
                if act[i]:
                    draft[i] = draft_cached(drafter, tok[i], int(pad_c[i]), L, int(dkept[i]),
                                            dcache[:, i], k, noise)
                    draft_log.append((list(draft[i]), drafter.propose(list(tok[i, pad_c[i]:L]), k, noise)))
            dview.copy_(_to_dev(dcache, cuda))
        kv_view = bt.kv_logical()                # f3: logical columns start at the origin
        cache = _bits(kv_view).copy()
        logits = np.zeros((B, k + 1, V), np.float32)
        for i in range(B):
            if not act[i]:
                continue
            for c in range(0 if first else L - 1, L + k):
                if mask[i, c]:
                    t = int(tok[i, c]) if c < L else int(draft[i, c - L])
                    lg = T.token_forward(t, int(pos[i, c]), c, cache[:, i], mask[i])
                    if c >= L - 1:
                        logits[i, c - L + 1] = lg.astype(np.float32)
        kv_view.copy_(_to_dev(cache, cuda))
        if fault == "rollback_min":
            # rollback: every row is cut to the batch-minimum accept
            # length -- the drafts of longer-accepting rows are made to mismatch at that
            # slot, so K1 accepts min(a) everywhere and the bonus is the target's token there
            pred = logits.argmax(axis=2)
            acc = [next((j for j in range(k) if pred[i, j] != draft[i, j]), k) for i in range(B)]
            m = min(acc[i] for i in range(B) if act[i])
            for i in range(B):
                if act[i] and acc[i] > m:
                    draft[i, m] = (pred[i, m] + 1) % V
        if fault == "skip_unpad" and not first:
            # DSD: "merely repads ... without ever unpadding": the old pads
            # are kept as content, so every active row's content is the whole width L
            a = bt.active.bool()
            bt.n[bt.cur].copy_(torch.where(a, torch.full_like(bt.n[bt.cur], L), bt.n[bt.cur]))
            bt.pad[bt.cur].copy_(torch.where(a, torch.zeros_like(bt.pad[bt.cur]), bt.pad[bt.cur]))
        bt.step(torch.from_numpy(logits).to(cuda), torch.from_numpy(draft).to(cuda), V=V)
        first = False
        rounds += 1
    gen = bt.gen.cpu().numpy()
    out = bt.out_buf.cpu().numpy()
    return [list(out[i, :gen[i]]) for i in range(B)], rounds, int(bt.status.item())


@pytest.mark.parametrize("B,noise,eos,k", [(2, 0.3, 1, 4), (4, 0.0, -1, 4), (5, 0.45, 1, 3), (1, 0.2, 1, 5)])
def test_eqspec_on_gpu_equals_greedy(cuda, B, noise, eos, k):
    T = ToyLM(V, LAYERS, H, D, seed=7)
    prompts = _prompts(B, seed=B * 10 + k)
    ref = [T.greedy_generate(p, 18, eos, 64) for p in prompts]
    out, rounds, status = _eqspec_gpu(cuda, T, prompts, k, 18, eos, noise)
    assert out == ref and status == 0


@pytest.mark.parametrize("B,noise,draft", [(3, 0.3, False), (4, 0.45, True), (1, 0.2, False)])
def test_pingpong_kv_on_gpu_equals_greedy(cuda, B, noise, draft):
    """kv_mode="pingpong": each round's realign writes the other KV buffer, which the next
    forward reads; output == greedy (with the draft cache ping-ponged too)."""
    T = ToyLM(V, LAYERS, H, D, seed=7)
    Dm = ToyLM(V, LAYERS, H, D, seed=8) if draft else None
    prompts = _prompts(B, seed=300 + B)
    ref = [T.greedy_generate(p, 18, 1, 64) for p in prompts]
    log = []
    out, rounds, status = _eqspec_gpu(cuda, T, prompts, 4, 18, 1, noise, drafter=Dm,
                                      draft_log=log if draft else None, kv_mode="pingpong")
    assert out == ref and status == 0
    if draft:
        assert len(log) >= rounds and all(c == r for c, r in log)


@pytest.mark.parametrize("B,noise", [(3, 0.3), (4, 0.0), (2, 0.5)])
def test_draft_kv_realign_on_gpu(cuda, B, noise):
    """f1: the drafter's own KV cache, realigned on the GPU with kept_draft = n + min(a, k-1),
    reproduces recompute-mode proposals every round; output == greedy."""
    T = ToyLM(V, LAYERS, H, D, seed=7)
    Dm = ToyLM(V, LAYERS, H, D, seed=8)
    prompts = _prompts(B, seed=200 + B)
    ref = [T.greedy_generate(p, 18, 1, 64) for p in prompts]
    log = []
    out, rounds, status = _eqspec_gpu(cuda, T, prompts, 4, 18, 1, noise, drafter=Dm, draft_log=log)
    assert out == ref and status == 0
    assert len(log) >= rounds and all(c == r for c, r in log)


CORRUPTING = ("skip_kv_realign", "bonus_from_draft", "stale_position_ids", "skip_unpad")


@pytest.mark.parametrize("seed,B,noise", [(44, 4, 0.35), (45, 6, 0.3), (46, 8, 0.25)])
def test_fault_modes_scored(cuda, seed, B, noise):
    """f4: each §2 failure class injected at
    its seam of the GPU path, scored with exact / partial match (oracle.metrics,
    PAPER.md:658) against per-sequence greedy decoding:
      * control: exact 1.0;
      * skip_kv_realign, bonus_from_draft (DSD i), stale_position_ids (BSP), skip_unpad (DSD
        "merely repads ... without ever unpadding"): exact < 1 -- every fault is caught;
      * rollback_min (rows cut to the batch-minimum accept length): exact 1.0 with strictly
        more rounds -- correct but wasteful;
      * signature separation: bonus_from_draft fails at the first rejection (lowest partial
        match), the stale-position and unrealigned-KV faults decay gradually (higher)."""
    from oracle.metrics import score_equivalence
    T = ToyLM(V, LAYERS, H, D, seed=7)
    k, max_new, cap = 4, 16 if B == 4 else 24, 192
    prompts = _prompts(B, seed=seed)
    ref = [T.greedy_generate(p, max_new, -1, cap) for p in prompts]
    runs = {}
    for f in (None,) + CORRUPTING + ("rollback_min",):
        out, rounds, _ = _eqspec_gpu(cuda, T, prompts, k, max_new, -1, noise, cap=cap, fault=f)
        runs[f] = score_equivalence(out, ref) + (rounds,)
    assert runs[None][:2] == (1.0, 1.0), runs
    for f in CORRUPTING:
        assert runs[f][0] < 1.0, (f, runs)
    assert runs["rollback_min"][:2] == (1.0, 1.0) and runs["rollback_min"][2] > runs[None][2], runs
    assert runs["bonus_from_draft"][1] < min(runs["stale_position_ids"][1], runs["skip_kv_realign"][1]), runs


def _exspec_gpu(cuda, T, prompts, k, max_new, Wn, B, mg, consumer="zero-copy", alg3=False):
    """EXSpec with the toy LM on the host and the pool plan / gather / verify + write-back /
    scatter in libspecdec.so.  Returns (outputs per prompt, kinds seen, final status)."""
    N = len(prompts)
    dense = consumer == "dense"
    lens = np.array([len(p) for p in prompts], np.int32)
    cap = int(lens.max()) + max_new + k + 4
    order = np.array(sorted(range(N), key=lambda s: (lens[s], s)), np.int32)
    tokens = np.zeros((N, cap), np.int64)
    kv = np.zeros((N, 2 * LAYERS, H, cap, D), np.uint16)
    ones = np.ones(cap, np.int64)
    for s, p in enumerate(prompts):
        tokens[s, :len(p)] = p
        for c, t in enumerate(p[:-1]):                    # prefill all but the pending token
            T.token_forward(t, c, c, kv[s], ones)
    sp = SequencePool(N, cap, LAYERS, H, D, k, W=Wn, B=B, min_group=mg, max_new=max_new, eos_id=1,
                      device=cuda, consumer=consumer)
    sp.load(lens, tokens, order, _to_dev(kv, cuda))
    sp.fused = not dense          # the dense case also covers the unfused verify + write-back
    kinds_seen = set()
    for _ in range(400):
        nb, kinds, blens, sizes = sp.plan()
        if nb == 0:
            break
        for b in range(1 if alg3 else nb):
            mem = sp.members[b].cpu().numpy()
            Lb = int(blens[b])
            fallback = sp.moves_kv(kinds[b])
            kinds_seen.add(int(kinds[b]))
            if fallback:
                sp.gather(b)
            ptok = sp.tokens.cpu().numpy()
            plen = sp.len.cpu().numpy()
            src = _bits(sp.staging).copy() if fallback else None
            pool_kv = _bits(sp.kv).copy() if not fallback else None
            logits = np.zeros((B, k + 1, V), np.float32)
            draft = np.zeros((B, k), np.int64)
            for j, s in enumerate(mem):
                if s < 0:
                    continue
                n = int(plen[s])
                Lr = Lb if fallback or kinds[b] else n     # slot consumer: the member's own width
                p = Lr - n
                content = list(ptok[s, :n])
                draft[j] = T.propose(content, k, 0.3)
                mask, pos = mask_pos_row(p, Lr + k)
                if fallback:
                    row = src[:, j]                        # right-aligned staging row
                else:
                    row = pool_kv[s]                       # zero-copy: the pool slot itself
                for c in range(Lr - 1, Lr + k):
                    t = content[-1] if c == Lr - 1 else int(draft[j, c - Lr])
                    lg = T.token_forward(t, int(pos[c]), c, row, mask)
                    logits[j, c - Lr + 1] = lg.astype(np.float32)
            if fallback:
                sp.staging.copy_(_to_dev(src, cuda))
            else:
                sp.kv.copy_(_to_dev(pool_kv, cuda))
            sp.verify_writeback(b, torch.from_numpy(logits).to(cuda), torch.from_numpy(draft).to(cuda), V=V)
            if fallback:
                sp.scatter(b, Lb)
    gen = sp.gen.cpu().numpy()
    out = sp.out_buf.cpu().numpy()
    assert not sp.has_active()
    return [list(out[s, :gen[s]]) for s in range(N)], kinds_seen, int(sp.status.item())


@pytest.mark.parametrize("N,Wn,B,mg,alg3,consumer", [(10, 6, 3, 2, False, "zero-copy"), (8, 8, 4, 4, False, "zero-copy"),
                                                      (7, 7, 1, 2, False, "zero-copy"), (9, 6, 3, 2, True, "zero-copy"),
                                                      (10, 6, 3, 2, False, "dense"), (10, 6, 3, 2, False, "slot"),
                                                      (12, 12, 4, 2, False, "slot")])
def test_exspec_pool_on_gpu_equals_greedy(cuda, N, Wn, B, mg, alg3, consumer):
    """EXSpec on the GPU path; alg3=True runs Alg. 3 as printed (batch 0, then re-plan);
    consumer "dense" gathers / scatters same-length batches too (a dense-rectangle
    consumer), "slot" moves no KV at all: every member's forward reads its own slot at its
    own width (a slot-indexed consumer)."""
    T = ToyLM(V, LAYERS, H, D, seed=7)
    k, max_new = 3, 12
    prompts = _prompts(N, seed=N + B)
    ref = [T.greedy_generate(p, max_new, 1, 64) for p in prompts]
    out, kinds_seen, status = _exspec_gpu(cuda, T, prompts, k, max_new, Wn, B, mg, consumer, alg3)
    assert out == ref and status == 0
    if B > 1:
        assert kinds_seen == {0, 1}           # both lazy (same-length) and fallback batches ran


@pytest.mark.parametrize("B,noise,slack,draft", [(3, 0.3, 48, False), (4, 0.45, 48, True), (2, 0.3, 2, False)])
def test_anchored_origin_on_gpu_equals_greedy(cuda, B, noise, slack, draft):
    """f3: the forward reads the KV through K1's moving origin; output == greedy, with the
    drafter's cache (f1) sharing the same origin when enabled."""
    T = ToyLM(V, LAYERS, H, D, seed=7)
    Dm = ToyLM(V, LAYERS, H, D, seed=8) if draft else None
    prompts = _prompts(B, seed=400 + B)
    ref = [T.greedy_generate(p, 18, 1, 64) for p in prompts]
    log = []
    out, rounds, status = _eqspec_gpu(cuda, T, prompts, 4, 18, 1, noise, drafter=Dm, draft_log=log,
                                      anchor_slack=slack)
    assert out == ref and status == 0
    assert all(c == r for c, r in log)
