"""Pins for oracle/align.py (Alg. 2 Phase 3 + Realign; §3.1):
SPEC worked examples, brute force over tiny batches checked against invariants that do
not restate the formulas (content conservation, right alignment, logical-position
preservation of every KV entry), a torch library cross-check for positions, and the
toy-LM equivalence with per-sequence greedy decoding."""
import itertools

import numpy as np
import pytest
import torch

from oracle import align as A
from oracle import verify as V
from oracle.loops import eqspec_decode
from oracle.toy_lm import ToyLM


def test_build_batch_spec_examples():
    # SPEC.md:127-129
    tok, pad, L = A.build_batch([[2] * 7, [3] * 5, [4] * 6], cap=10)
    assert L == 7 and list(pad) == [0, 2, 1]
    tok, pad, L = A.build_batch([[2] * 4, [3] * 4], cap=8)
    assert list(pad) == [0, 0]
    assert A.mask_pos_row(0, 4)[0].tolist() == [1, 1, 1, 1]
    tok, pad, L = A.build_batch([[5, 6, 7]], cap=4)
    assert L == 3 and list(pad) == [0]


def test_unpad_round_trip():
    seqs = [[2, 3, 4], [5], [6, 7]]
    tok, pad, L = A.build_batch(seqs, cap=6)
    assert A.unpad(tok, pad, L) == seqs


def test_repad_spec_example():
    # ragged lengths [9, 7] -> L = 9, offsets 0 and 2
    plan = V.repad_plan([5, 5], accept=[3, 1], finished=[0, 0])
    assert plan["L_new"] == 9 and list(plan["pad_new"]) == [0, 2]
    plan = V.repad_plan([4, 4], accept=[2, 2], finished=[0, 0])
    assert list(plan["pad_new"]) == [0, 0]              # all equal -> no offsets
    plan = V.repad_plan([6], accept=[1], finished=[0])
    assert list(plan["pad_new"]) == [0]


def test_realign_spec_examples():
    # uniform acceptance -> pure truncation (no shift)
    plan = V.repad_plan([5, 5], [2, 2], [0, 0])
    assert list(plan["pad_new"]) == [0, 0]
    # row A accepts 5, row B accepts 1 (K = 5): B shifted right by 4 relative to A
    n, pad = [6, 6], [0, 0]
    plan = V.repad_plan(n, [5, 1], [0, 0])
    assert plan["pad_new"][1] - plan["pad_new"][0] == 4
    # B = 1 -> simple truncation at kept
    plan = V.repad_plan([7], [3], [0])
    assert plan["pad_new"][0] == 0 and plan["kept"][0] == 10


def _check_round(n, a, fin, k, cap=40, pad_id=0):
    """Run verify-plan + repad + realign on a tiny synthetic batch and check invariants."""
    B = len(n)
    L = max(n)
    pad = np.array([L - x for x in n], np.int32)
    rng = np.random.default_rng(abs(hash((tuple(n), tuple(a)))) % (1 << 32))
    seqs = [list(rng.integers(2, 50, size=x)) for x in n]
    tok, _, _ = A.build_batch(seqs, cap, pad_id)
    E = [list(rng.integers(2, 50, size=ai)) + [int(rng.integers(2, 50))] for ai in a]
    fin = np.asarray(fin, np.uint8)
    plan = V.repad_plan(n, a, fin)
    vres = dict(E=[e if not f else e for e, f in zip(E, fin)], finished=fin, **plan)
    tok2, mask, pos = A.repad_tokens(tok, cap, k, pad, L, vres, pad_id)
    L2 = plan["L_new"]
    alive = fin == 0
    if not alive.any():
        assert L2 == 0
        return
    # right-aligned, minimal: some live row has no pad
    assert min(plan["pad_new"][alive]) == 0
    for i in range(B):
        p2 = plan["pad_new"][i]
        content = list(tok2[i, p2:L2])
        if alive[i]:
            assert content == seqs[i] + E[i]               # conservation
        else:
            assert content == [pad_id]                     # R9 dummy row
        assert all(t == pad_id for t in tok2[i, :p2])
        # mask 0 exactly on pads, positions contiguous from 0
        assert list(mask[i]) == [0] * p2 + [1] * (L2 + k - p2)
        assert list(pos[i]) == [0] * p2 + list(range(L2 + k - p2))
    # library cross-check: pos = clamp(cumsum(mask) - 1, 0)
    tm = torch.from_numpy(mask)
    assert torch.equal(torch.from_numpy(pos), (tm.cumsum(1) - 1).clamp(min=0))
    # KV: encode each entry's (row, logical token index); after realign every kept entry
    # must still sit at its own token index j at column p'_i + j (alignment soundness)
    kv = np.zeros((2, B, 1, cap, 1), np.int64)
    for i in range(B):
        for c in range(cap):
            kv[:, i, 0, c, 0] = 1000 * i + (c - pad[i]) if c >= pad[i] else -1
    kv2, defined = A.realign_kv(kv, pad, plan["pad_new"], plan["kept"])
    for i in range(B):
        if not alive[i]:
            assert not defined[i].any()
            continue
        cols = np.flatnonzero(defined[i])
        assert len(cols) == n[i] + a[i]                    # kept = KV of n-1 old + pending + a
        assert cols[0] == plan["pad_new"][i] and cols[-1] == L2 - 2   # bonus has no KV
        for c in cols:
            assert kv2[0, i, 0, c, 0] == 1000 * i + (c - plan["pad_new"][i])


@pytest.mark.parametrize("B,k", [(1, 4), (2, 3), (3, 2), (2, 4)])
def test_brute_force_plans(B, k):
    """Every accept vector a in {0..k}^B and content lengths n in {1..k+1}^B (SURVEY §4 tier 2)."""
    cnt = 0
    for n in itertools.product(range(1, k + 2), repeat=B):
        for a in itertools.product(range(0, k + 1), repeat=B):
            _check_round(list(n), list(a), [0] * B, k)
            cnt += 1
    assert cnt == (k + 1) ** (2 * B)


def test_finished_rows_brute_force():
    k = 2
    for n in itertools.product(range(1, 4), repeat=3):
        for fin in itertools.product([0, 1], repeat=3):
            _check_round(list(n), [1, 0, 2], list(fin), k)


def test_moved_bytes_and_zero_pad_region():
    pad_old, pad_new, kept = [0, 3, 2], [2, 3, 0], [10, 6, 0]
    assert A.moved_bytes(pad_old, pad_new, kept, bpt=128) == 2 * 10 * 128
    assert A.zero_pad_region(pad_old, pad_new, kept) == [(0, 0, 2)]


def test_copy_rows_gather_scatter():
    src = np.arange(3 * 2 * 1 * 6 * 2).reshape(3, 2, 1, 6, 2)
    dst = np.zeros((2, 2, 1, 8, 2), np.int64)
    A.copy_rows(src, dst, count=[2, 3], src_col=[1, 0], dst_col=[5, 0], src_row=[2, 0])
    assert np.array_equal(dst[0, :, :, 5:7], src[2, :, :, 1:3])
    assert np.array_equal(dst[1, :, :, 0:3], src[0, :, :, 0:3])
    assert dst[0, :, :, :5].sum() == 0


def test_realign_kv_inplace_tracks_token_identity():
    """In-place Realign (the K2 contract): brute force over shifts of both signs, Delta = 0,
    empty rows and overlapping source / destination ranges.  Every entry is tagged with its
    (row, column, plane, head, d) identity; afterwards column p'_i + c holds the entry that
    was at p_i + c, and every other column still holds its own (closed form, no formula of
    the oracle restated)."""
    rng = np.random.default_rng(12)
    for _ in range(300):
        B, P, H, D = int(rng.integers(1, 5)), int(rng.integers(1, 3)), int(rng.integers(1, 3)), 2
        cap = int(rng.integers(8, 40))
        kept = rng.integers(0, cap // 2, B)
        po = np.array([int(rng.integers(0, cap - kept[i] + 1)) for i in range(B)])
        pn = np.array([int(rng.integers(0, cap - kept[i] + 1)) if rng.random() < 0.8 else po[i] for i in range(B)])
        tag = np.zeros((P, B, H, cap, D), np.int64)
        pl, b, h, c, d = np.indices(tag.shape)
        tag[:] = (((pl * 8 + b) * 8 + h) * 64 + c) * 4 + d
        kv = A.realign_kv_inplace(tag.copy(), po, pn, kept)
        for i in range(B):
            for col in range(cap):
                want = col
                if pn[i] <= col < pn[i] + kept[i]:
                    want = col - pn[i] + po[i]
                assert np.array_equal(kv[:, i, :, col], tag[:, i, :, want]), (i, col)
        # the defined region agrees with the fresh-rectangle form
        ref, defined = A.realign_kv(tag, po, pn, kept)
        assert np.array_equal(kv[:, :, :][np.broadcast_to(defined[None, :, None, :, None], kv.shape)],
                              ref[np.broadcast_to(defined[None, :, None, :, None], ref.shape)])


# --------------------------------------------------------------------------- toy-LM equivalence
PROMPTS_SEED = 0


def _prompts(n, lo=1, hi=16, V_=32, seed=PROMPTS_SEED):
    rng = np.random.default_rng(seed)
    return [list(map(int, rng.integers(2, V_, size=int(l)))) for l in rng.integers(lo, hi + 1, size=n)]


@pytest.mark.parametrize("B,noise,drafter_seed,eos", [
    (1, 0.0, None, 1), (2, 0.3, None, 1), (4, 0.0, 8, 1), (4, 0.4, None, -1), (3, 0.15, None, 1)])
def test_eqspec_equals_autoregressive_greedy(B, noise, drafter_seed, eos):
    """Batched speculative output == per-sequence greedy output, token for token
    (BASELINE.json north_star)."""
    T = ToyLM(seed=7)
    Dm = T if drafter_seed is None else ToyLM(seed=drafter_seed)
    prompts = _prompts(B, seed=B)
    ref = [T.greedy_generate(p, 20, eos, 64) for p in prompts]
    out, rounds = eqspec_decode(T, Dm, prompts, 4, 20, eos, 64, noise=noise)
    assert out == ref
    assert rounds >= -(-20 // 5)


def test_equivalence_has_teeth(monkeypatch):
    """Negative controls (§2 failure taxonomy): skipping the KV
    realignment or reusing stale position ids must break equivalence."""
    T = ToyLM(seed=7)
    prompts = _prompts(4, seed=4)
    ref = [T.greedy_generate(p, 16, -1, 64) for p in prompts]
    import oracle.loops as Lp
    orig = Lp.realign_kv
    monkeypatch.setattr(Lp, "realign_kv", lambda kv, po, pn, kept: (kv.copy(), None))
    out, _ = eqspec_decode(T, T, prompts, 4, 16, -1, 64, noise=0.4)
    assert out != ref
    monkeypatch.setattr(Lp, "realign_kv", orig)
    orig_rt = Lp.repad_tokens

    def stale(tokens, cap, k, pad_old, L_old, vres, pad_id=0):
        t, m, p = orig_rt(tokens, cap, k, pad_old, L_old, vres, pad_id)
        return t, m, np.arange(p.shape[1])[None, :].repeat(p.shape[0], 0)  # tensor index as position
    monkeypatch.setattr(Lp, "repad_tokens", stale)
    out, _ = eqspec_decode(T, T, prompts, 4, 16, -1, 64, noise=0.4)
    assert out != ref


def test_alignment_soundness_from_scratch():
    """After each realign, a from-scratch forward of the realigned batch reproduces the
    cached path's logits exactly."""
    T = ToyLM(seed=7)
    prompts = _prompts(3, seed=9)
    k, cap = 3, 64
    trace = []
    import oracle.loops as Lp
    captured = []
    orig = Lp.verify_forward

    def spy(model, tokens, draft, pad, L, k_, cache, active, mask, pos, first):
        lg = orig(model, tokens, draft, pad, L, k_, cache, active, mask, pos, first)
        if not first:
            fresh = np.zeros_like(cache)
            lg2 = orig(model, tokens, draft, pad, L, k_, fresh, active, mask, pos, True)
            captured.append(np.array_equal(lg, lg2))
        return lg
    Lp.verify_forward = spy
    try:
        eqspec_decode(T, T, prompts, k, 14, -1, cap, noise=0.35, trace=trace)
    finally:
        Lp.verify_forward = orig
    assert len(captured) >= 3 and all(captured)
    # the run exercised real shifts in both directions
    shifts = [int(s) for t in trace for s in (t["pad_new"] - t["pad"])]
    assert any(s > 0 for s in shifts) and any(s < 0 for s in shifts)


# --------------------------------------------------------------------------- f1: draft KV realign
def test_kept_draft_rule():
    """n + min(a, k-1): d_k is generated by the draft but never forwarded."""
    plan = V.repad_plan([10, 10, 10], [0, 3, 4], [0, 0, 1], k=4)
    assert list(plan["kept_draft"]) == [10, 13, 0]
    assert list(plan["kept"]) == [10, 13, 0]
    plan = V.repad_plan([7], [4], [0], k=4)
    assert plan["kept_draft"][0] == 7 + 3 and plan["kept"][0] == 11


@pytest.mark.parametrize("noise,B", [(0.0, 3), (0.3, 4), (0.5, 2)])
def test_draft_cache_realign_reproduces_recompute_drafts(noise, B):
    """With its own KV cache realigned by kept_draft every round, the drafter proposes
    exactly what a from-scratch (recompute) drafter proposes -- token for token, every
    round -- and the batched output still equals greedy decoding."""
    T = ToyLM(seed=7)
    Dm = ToyLM(seed=8)
    prompts = _prompts(B, seed=100 + B)
    ref = [T.greedy_generate(p, 18, 1, 64) for p in prompts]
    log = []
    out, _ = eqspec_decode(T, Dm, prompts, 4, 18, 1, 64, noise=noise, draft_cache=True, draft_log=log)
    assert out == ref
    assert len(log) > 5 and all(c == r for c, r in log)
    # a wrong kept rule (keeping d_k's slot as if it had draft KV) is caught
    import oracle.verify as OVm
    orig = OVm.repad_plan

    def wrong(n, accept, finished, k=None):
        p = orig(n, accept, finished, k)
        if k is not None:
            p["kept_draft"] = p["kept"].copy()
        return p
    import oracle.verify
    oracle.verify.repad_plan = wrong
    try:
        log2 = []
        eqspec_decode(T, T, prompts, 4, 18, 1, 64, noise=0.0, draft_cache=True, draft_log=log2)
    finally:
        oracle.verify.repad_plan = orig
    assert any(c != r for c, r in log2)


# --------------------------------------------------------------------------- f3: anchored origin
def _cost(d, pad_old, pad_new, kept, alive):
    return sum(int(kept[i]) for i in range(len(kept)) if alive[i] and kept[i] > 0 and d + pad_new[i] != pad_old[i])


def test_anchor_plan_is_the_brute_force_minimum():
    """The chosen origin moves the fewest KV rows of ALL feasible origins (brute force over
    every shift), never more than the standard alignment (d = 0)."""
    rng = np.random.default_rng(1)
    for _ in range(400):
        B, k = int(rng.integers(1, 7)), int(rng.integers(1, 6))
        n = rng.integers(1, 30, B)
        a = rng.integers(0, k + 1, B)
        fin = (rng.random(B) < 0.2).astype(np.uint8)
        plan = V.repad_plan(n, a, fin)
        L, Ln = int(n.max()), plan["L_new"]
        pad_old = L - n
        # capacity room above L'+k, and an origin anywhere up to 3 columns past the highest
        # one that keeps d = 0 feasible (then only a moving shift -- or the fallback -- fits)
        room = int(rng.integers(0, 12))
        cap_phys = Ln + k + room
        base = int(rng.integers(0, room + 4))
        b2, col_old, col_new = A.anchor_plan(pad_old, plan["pad_new"], plan["kept"], fin, a, L, Ln,
                                             base, cap_phys, k)
        d = b2 - base
        alive = fin == 0
        feas = [x for x in range(-base, cap_phys - base - Ln - k + 1)] if Ln else [0]
        best = min(_cost(x, pad_old, plan["pad_new"], plan["kept"], alive) for x in feas)
        assert _cost(d, pad_old, plan["pad_new"], plan["kept"], alive) == best
        if 0 in feas:
            assert best <= _cost(0, pad_old, plan["pad_new"], plan["kept"], alive)
        assert 0 <= b2 and (Ln == 0 or b2 + Ln + k <= cap_phys)
        assert list(col_old) == list(base + pad_old) and list(col_new) == list(b2 + plan["pad_new"])


def test_anchor_plan_fallback_when_no_candidate_fits():
    """base' + L + k == cap, then L grows by one with a = 0 for the longest row:
    d = 0 and every class shift d = a + 1 - (L' - L) >= 0 overflow the physical buffer; the
    origin must drop to the highest feasible one (every kept row moves) instead of staying."""
    k, cap_phys, base = 2, 20, 5
    n, a = np.array([13, 10]), np.array([0, 2])
    fin = np.zeros(2, np.uint8)
    plan = V.repad_plan(n, a, fin)
    L, Ln = 13, plan["L_new"]
    assert Ln == 14 and base + L + k == cap_phys
    b2, co, cn = A.anchor_plan(L - n, plan["pad_new"], plan["kept"], fin, a, L, Ln, base, cap_phys, k)
    assert b2 == 4 and b2 + Ln + k == cap_phys
    assert list(co) == [5, 8] and list(cn) == [4, 5]
    assert np.all(cn + plan["kept"] <= cap_phys)


def test_anchor_moves_only_the_logical_origin():
    """Physically realigned KV, read through the moved origin, equals Alg. 2's realign."""
    rng = np.random.default_rng(2)
    for _ in range(60):
        B, k, slack = int(rng.integers(1, 6)), 4, 10
        n = rng.integers(2, 20, B)
        a = rng.integers(0, k + 1, B)
        plan = V.repad_plan(n, a, np.zeros(B, np.uint8))
        L, Ln = int(n.max()), plan["L_new"]
        cap = Ln + k + 2
        logical = rng.integers(0, 1 << 15, size=(2, B, 1, cap, 3))
        phys = np.zeros((2, B, 1, cap + slack, 3), np.int64)
        phys[:, :, :, slack:slack + cap] = logical
        b2, co, cn = A.anchor_plan(L - n, plan["pad_new"], plan["kept"], np.zeros(B), a, L, Ln,
                                   slack, cap + slack, k)
        rows = np.moveaxis(phys, 1, 0)
        A.copy_rows(rows, rows, plan["kept"], src_col=co, dst_col=cn)
        ref, defined = A.realign_kv(logical, L - n, plan["pad_new"], plan["kept"])
        view = phys[:, :, :, b2:b2 + cap]
        for i in range(B):
            c = np.flatnonzero(defined[i])
            assert np.array_equal(view[:, i, :, c], ref[:, i, :, c])


@pytest.mark.parametrize("B,noise", [(3, 0.3), (4, 0.45)])
def test_anchored_eqspec_equals_greedy_and_moves_less(B, noise):
    T = ToyLM(seed=7)
    prompts = _prompts(B, seed=300 + B)
    ref = [T.greedy_generate(p, 20, -1, 64) for p in prompts]
    tr = []
    out, _ = eqspec_decode(T, T, prompts, 4, 20, -1, 64, noise=noise, anchor_slack=40, trace=tr)
    assert out == ref
    assert any(t["base"] != 40 for t in tr)       # the origin actually moved
