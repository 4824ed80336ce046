"""Oracle: EXSpec SequencePool scheduling (Alg. 3; §3.2).

Test infrastructure only (see oracle/__init__.py).

Readings: R11 full-partition plan with a min_group parameter; R12 window =
first W active sequences in admission order; R13 grouping key = total token length;
R14 grouping rate = same-length batches / all batches; R27 deferred fallback (an epoch's
leftovers wait up to `patience` epochs for a same-length partner); R28 pipelined fallback
(an epoch's mixed batches run beside the next epoch, whose plan excludes their members).
"""
from __future__ import annotations

import numpy as np


def admission_order(prompt_lens, sort_by_length: bool):
    """InitSequencePool(P), "optionally sort by length": ascending
    prompt length, ties by id; else by id."""
    ids = list(range(len(prompt_lens)))
    if sort_by_length:
        ids.sort(key=lambda s: (int(prompt_lens[s]), s))
    return np.array(ids, np.int32)


def refill_window(active, order, W):
    """RefillWindow(Pool, W): the first W active ids in admission order."""
    return [int(s) for s in order if active[s]][:W]


def form_batches(lens, active, order, W, B, min_group):
    """GetBatch over the whole window: "attempts to form batches
    of identical length", else falls back to unpad-repad.

    Distinct lengths are visited by (-count, length); each length's members (window
    order) yield batches of min(B, remaining) while remaining >= min_group (>= 1 when
    B == 1); leftovers, in window order, are chunked into fallback batches of B.
    Returns dict(window, batches[list of member lists], kind[list: 1 same-length],
    blen, counters)."""
    window = refill_window(active, order, W)
    mg = 1 if B == 1 else min_group
    count = {}
    for s in window:
        count[int(lens[s])] = count.get(int(lens[s]), 0) + 1
    batches, unmatched = [], []
    for length in sorted(count, key=lambda l: (-count[l], l)):
        remaining = [s for s in window if int(lens[s]) == length]
        while len(remaining) >= mg:
            batches.append(remaining[:B])
            remaining = remaining[B:]
        unmatched += remaining
    pos = {s: t for t, s in enumerate(window)}
    unmatched.sort(key=lambda s: pos[s])
    for t in range(0, len(unmatched), B):
        batches.append(unmatched[t:t + B])
    kind = [int(len({int(lens[s]) for s in b}) == 1) for b in batches]
    blen = [max(int(lens[s]) for s in b) for b in batches]
    same_members = sum(len(b) for b, kd in zip(batches, kind) if kd)
    fb_members = sum(len(b) for b, kd in zip(batches, kind) if not kd)
    fb_tokens = sum(int(lens[s]) for b, kd in zip(batches, kind) if not kd for s in b)
    counters = np.array([len(batches), sum(kind), same_members, fb_members, fb_tokens,
                         len(window), len(count), 0], np.int64)
    return dict(window=window, batches=batches, kind=kind, blen=blen, counters=counters,
                deferred=[])


def form_batches_deferred(lens, active, order, W, B, min_group, wait, patience):
    """The epoch plan with deferred fallback (reading R27).  Alg. 3's GetBatch falls back to
    unpad-repad only when no batch of identical length can be formed (PAPER.md:492-494,
    537); an epoch that runs the whole window plan at once would instead send every
    leftover to a fallback batch at once.  Here:

      form_batches' group pass (R11) gives the same-length batches and the leftovers;
      if that pass formed at least one same-length batch and patience > 0:
          a leftover s with wait[s] < patience sits this epoch out (deferred), and only the
          leftovers with wait[s] >= patience, in window order, fill fallback batches of B;
      otherwise the plan is unchanged (every leftover runs);
      wait[s] <- 0 for every planned member, wait[s] + 1 for every deferred one (window
      members only; `wait` is updated in place).

    patience = 0 is form_batches exactly.  counters[7] = deferred members.
    Returns form_batches' dict (batches renumbered: the same-length group batches first,
    then the fallback batches) with `deferred` = the deferred ids in window order."""
    window = refill_window(active, order, W)
    mg = 1 if B == 1 else min_group
    count = {}
    for s in window:
        count[int(lens[s])] = count.get(int(lens[s]), 0) + 1
    # form_batches' group pass: its batches, and the leftovers in window order
    groups, left = [], []
    for length in sorted(count, key=lambda l: (-count[l], l)):
        remaining = [s for s in window if int(lens[s]) == length]
        while len(remaining) >= mg:
            groups.append(remaining[:B])
            remaining = remaining[B:]
        left += remaining
    pos = {s: t for t, s in enumerate(window)}
    left.sort(key=lambda s: pos[s])
    if patience > 0 and len(groups) > 0:
        run_left = [s for s in left if int(wait[s]) >= patience]
        deferred = [s for s in left if int(wait[s]) < patience]
    else:
        run_left, deferred = left, []
    batches = groups + [run_left[t:t + B] for t in range(0, len(run_left), B)]
    for b in batches:
        for s in b:
            wait[s] = 0
    for s in deferred:
        wait[s] += 1
    kind = [int(len({int(lens[s]) for s in b}) == 1) for b in batches]
    blen = [max(int(lens[s]) for s in b) for b in batches]
    same_members = sum(len(b) for b, kd in zip(batches, kind) if kd)
    fb_members = sum(len(b) for b, kd in zip(batches, kind) if not kd)
    fb_tokens = sum(int(lens[s]) for b, kd in zip(batches, kind) if not kd for s in b)
    counters = np.array([len(batches), sum(kind), same_members, fb_members, fb_tokens,
                         len(window), len(count), len(deferred)], np.int64)
    return dict(window=window, batches=batches, kind=kind, blen=blen, counters=counters,
                deferred=deferred)


def pipeline_window_active(active, inflight):
    """Reading R28 (pipelined fallback): the mixed-length (realigned) batches of epoch e run
    beside epoch e+1, so their members sit out epoch e+1's plan -- for exactly one epoch --
    and are planned again from epoch e+2 on.  Returns the `active` array epoch e+1 plans
    with: active and not in epoch e's mixed batches (`inflight`: their ids)."""
    eff = np.array(active, np.uint8, copy=True)
    for s in inflight:
        eff[s] = 0
    return eff


def mixed_members(plan):
    """The members of a plan's mixed-length batches (kind 0): R28's in-flight set."""
    return [s for b, kd in zip(plan["batches"], plan["kind"]) if not kd for s in b]


def writeback(pool_len, pool_gen, pool_active, pool_tokens, out_buf, members, E_rows, finished):
    """Phase 4 write-back: Pool[i] <- Pool[i] (+) A[i] (+) B[i];
    deactivate if complete.  Token lists are appended at the sequence's current
    length; the emitted tokens also go to the per-sequence output buffer."""
    for i, s in enumerate(members):
        if s < 0:
            continue
        E = E_rows[i]
        L0, g0 = int(pool_len[s]), int(pool_gen[s])
        pool_tokens[s, L0:L0 + len(E)] = E
        out_buf[s, g0:g0 + len(E)] = E
        pool_len[s] += len(E)
        pool_gen[s] += len(E)
        if finished[i]:
            pool_active[s] = 0
