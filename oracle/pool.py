"""Oracle: EXSpec SequencePool scheduling (Alg. 3; §3.2).

Test infrastructure only (see oracle/__init__.py).

Readings: R11 full-partition plan with a min_group parameter; R12 window =
first W active sequences in admission order; R13 grouping key = total token length;
R14 grouping rate = same-length batches / all batches.
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
    return dict(window=window, batches=batches, kind=kind, blen=blen, counters=counters)


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
