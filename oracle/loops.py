"""Oracle: Alg. 2 EqSpec and Alg. 3 EXSpec
decode loops driven by the toy LM, and the per-sequence greedy reference.

Test infrastructure only (see oracle/__init__.py).  These loops compose the oracle's
verify / repad / realign / pool functions exactly as the algorithms order them; the
tests require their outputs to equal per-sequence autoregressive greedy decoding
token for token.
"""
from __future__ import annotations

import numpy as np

from .align import (anchor_plan, build_batch, copy_rows, mask_pos_row, realign_kv, repad_tokens,
                    unpad)
from .pool import admission_order, form_batches, form_batches_deferred, mixed_members, pipeline_window_active
from .toy_lm import ToyLM, greedy_fp32
from .verify import batch_verify


def verify_forward(model: ToyLM, tokens, draft, pad, L, k, cache, active, mask, pos, first):
    """BatchVerify's forward (R3): X = S (+) D on the first iteration,
    else [pending token] (+) D.  Writes KV columns and returns the k+1-row logits tail
    [B, k+1, V] as fp32 (the verifier's precision)."""
    B = len(pad)
    logits = np.zeros((B, k + 1, model.V), np.float32)
    lo = 0 if first else L - 1
    for i in range(B):
        if not active[i]:
            continue
        row = cache[:, i]
        for c in range(lo, L + k):
            if mask[i, c] == 0:
                continue
            t = int(tokens[i, c]) if c < L else int(draft[i, c - L])
            lg = model.token_forward(t, int(pos[i, c]), c, row, mask[i])
            if c >= L - 1:
                logits[i, c - (L - 1)] = lg.astype(np.float32)
    return logits


def draft_cached(model: ToyLM, tokens_row, pad: int, L: int, dkept: int, cache_row, k: int,
                 noise: float = 0.0, seed: int = 0):
    """Draft generation with the drafter's own KV cache (f1; Alg. 2 Phase 1, PAPER.md:337-339;
    SPEC.md:217).  Content = tokens_row[pad:L]; the draft cache holds valid KV on
    [pad, pad + dkept).  Forwards the tokens that lack draft KV (1 normally, 2 after a
    full acceptance), then d_1..d_{k-1}; d_k is generated but never forwarded.  The
    proposals (and their noise) equal ToyLM.propose's recompute-mode ones."""
    cap = cache_row.shape[2]
    mask = (np.arange(cap) >= pad).astype(np.int64)
    content = [int(t) for t in tokens_row[pad:L]]
    rng = np.random.default_rng([seed, len(content), int(np.sum(content)) % (1 << 31)])
    logits = None
    for c in range(pad + dkept, L):
        logits = model.token_forward(int(tokens_row[c]), c - pad, c, cache_row, mask)
    props, c = [], L
    for j in range(k):
        t = greedy_fp32(logits)
        if noise > 0 and rng.random() < noise:
            t = (t + 1 + int(rng.integers(model.V - 1))) % model.V
        props.append(t)
        if j < k - 1:
            logits = model.token_forward(t, c - pad, c, cache_row, mask)
            c += 1
    return props


def eqspec_decode(target: ToyLM, drafter: ToyLM, prompts, k, max_new, eos_id, cap,
                  noise=0.0, pad_id=0, trace=None, draft_cache=False, draft_log=None,
                  anchor_slack=0):
    """Alg. 2.  Returns (outputs per prompt, rounds).  With draft_cache=True the drafter
    keeps its own KV cache, realigned every round with kept_draft (f1); draft_log, if a
    list, receives (cached proposals, recompute proposals) per round.  With
    anchor_slack > 0 the target KV lives in a physical buffer of cap + slack columns whose
    logical origin moves by align.anchor_plan (f3); the forward reads the logical view."""
    B = len(prompts)
    tokens, pad, L = build_batch(prompts, cap, pad_id)
    n = np.array([len(p) for p in prompts], np.int32)
    active = np.ones(B, np.uint8)
    gen = np.zeros(B, np.int64)
    out = [[] for _ in range(B)]
    phys = np.zeros((target.n_planes, B, target.H, cap + anchor_slack, target.D), np.uint16)
    base = anchor_slack
    cache = phys[:, :, :, base:base + cap]          # the logical view
    mask = np.stack([mask_pos_row(int(p), L + k)[0] for p in pad])
    pos = np.stack([mask_pos_row(int(p), L + k)[1] for p in pad])
    dcache = np.zeros((drafter.n_planes, B, drafter.H, cap, drafter.D), np.uint16)
    dkept = np.zeros(B, np.int32)
    first, rounds = True, 0
    while active.any():
        assert L + k <= cap, "capacity"
        content = unpad(tokens, pad, L)
        draft = np.full((B, k), pad_id, np.int64)
        for i in range(B):
            if active[i]:
                if draft_cache:
                    draft[i] = draft_cached(drafter, tokens[i], int(pad[i]), L, int(dkept[i]),
                                            dcache[:, i], k, noise)
                else:
                    draft[i] = drafter.propose(content[i], k, noise)
                if draft_log is not None:
                    draft_log.append((list(draft[i]), drafter.propose(content[i], k, noise)))
        logits = verify_forward(target, tokens, draft, pad, L, k, cache, active, mask, pos, first)
        budget = (max_new - gen).astype(np.int64)
        v = batch_verify(logits, "fp32", draft, n, pad, active, eos_id, budget, pad_id)
        for i in range(B):
            out[i] += v["E"][i]
        gen += v["emit"]
        if trace is not None:
            trace.append(dict(L=L, pad=pad.copy(), n=n.copy(), accept=v["accept"].copy(),
                              kept=v["kept"].copy(), pad_new=v["pad_new"].copy()))
        tokens, mask, pos = repad_tokens(tokens, cap, k, pad, L, v, pad_id)
        if anchor_slack:
            base_new, col_old, col_new = anchor_plan(pad, v["pad_new"], v["kept"], v["finished"],
                                                     v["accept"], L, v["L_new"], base,
                                                     cap + anchor_slack, k)
            rows = np.moveaxis(phys, 1, 0)          # [B][planes][H][cap+slack][D] view
            copy_rows(rows, rows, v["kept"], src_col=col_old, dst_col=col_new)
            base = base_new
            cache = phys[:, :, :, base:base + cap]
            if trace is not None:
                trace[-1]["base"] = base
        else:
            cache, _ = realign_kv(cache, pad, v["pad_new"], v["kept"])
        if draft_cache:
            dcache, _ = realign_kv(dcache, pad, v["pad_new"], v["kept_draft"])
            dkept = v["kept_draft"]
        pad, n, L = v["pad_new"], v["n_new"], v["L_new"]
        active = (v["finished"] == 0).astype(np.uint8)
        first = False
        rounds += 1
    return out, rounds


def exspec_decode(target: ToyLM, drafter: ToyLM, prompts, k, max_new, eos_id, cap, W, B,
                  min_group=2, sort_by_length=True, noise=0.0, pad_id=0, sequential=False,
                  patience=0, pipeline=False):
    """Alg. 3 over a SequencePool.  Each epoch plans the whole window (K4 semantics);
    with sequential=True only batch 0 runs per iteration (Alg. 3's one-batch GetBatch);
    patience > 0: the epoch plan defers leftovers (form_batches_deferred, reading R27);
    pipeline: an epoch's mixed batches run beside the next epoch, whose plan excludes their
    members (reading R28; results applied at once -- the batches have disjoint members).
    Returns (outputs, stats)."""
    N = len(prompts)
    lens = np.array([len(p) for p in prompts], np.int32)
    order = admission_order(lens, sort_by_length)
    active = np.ones(N, np.uint8)
    seqs = [list(map(int, p)) for p in prompts]
    gen = np.zeros(N, np.int64)
    out = [[] for _ in range(N)]
    pool_kv = [target.new_row_cache(cap) for _ in range(N)]
    ones = np.ones(cap, np.int64)
    for s in range(N):                      # prefill: KV for all but the pending token
        for c, t in enumerate(seqs[s][:-1]):
            target.token_forward(t, c, c, pool_kv[s], ones)
    stats = dict(verify_calls=0, batches=0, same_length=0, realigned_members=0)
    wait = np.zeros(N, np.int64)
    inflight = []
    while active.any():
        act_plan = pipeline_window_active(active, inflight) if pipeline else active
        if patience > 0:
            plan = form_batches_deferred(lens, act_plan, order, W, B, min_group, wait, patience)
        else:
            plan = form_batches(lens, act_plan, order, W, B, min_group)
        inflight = mixed_members(plan) if pipeline else []
        todo = plan["batches"][:1] if sequential else plan["batches"]
        kinds = plan["kind"][:1] if sequential else plan["kind"]
        for members, kind in zip(todo, kinds):
            Bb = len(members)
            Lb = max(int(lens[s]) for s in members)
            tokens, pad, _ = build_batch([seqs[s] for s in members], cap, pad_id)
            nb = lens[members].astype(np.int32)
            cache = np.zeros((target.n_planes, Bb, target.H, cap, target.D), np.uint16)
            for i, s in enumerate(members):      # same-length: p = 0 (pure stack)
                kv_len = int(lens[s]) - 1
                cache[:, i, :, pad[i]:pad[i] + kv_len] = pool_kv[s][:, :, :kv_len]
            mask = np.stack([mask_pos_row(int(p), Lb + k)[0] for p in pad])
            pos = np.stack([mask_pos_row(int(p), Lb + k)[1] for p in pad])
            draft = np.stack([drafter.propose(seqs[s], k, noise) for s in members]).astype(np.int64)
            act = np.ones(Bb, np.uint8)
            logits = verify_forward(target, tokens, draft, pad, Lb, k, cache, act, mask, pos, False)
            budget = (max_new - gen[members]).astype(np.int64)
            v = batch_verify(logits, "fp32", draft, nb, pad, act, eos_id, budget, pad_id)
            stats["verify_calls"] += 1
            stats["batches"] += 1
            stats["same_length"] += int(kind)
            stats["realigned_members"] += 0 if kind else Bb
            for i, s in enumerate(members):      # Phase 4 write-back
                a, ln = int(v["accept"][i]), int(lens[s])
                pool_kv[s][:, :, ln - 1:ln + a] = cache[:, i, :, Lb - 1:Lb + a]
                seqs[s] += v["E"][i]
                out[s] += v["E"][i]
                lens[s] += int(v["emit"][i])
                gen[s] += int(v["emit"][i])
                if v["finished"][i]:
                    active[s] = 0
    return out, stats
