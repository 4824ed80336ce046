"""Pins for oracle/pool.py (Alg. 3 GetBatch / RefillWindow; §3.2
PAPER.md:532-537): SPEC worked examples, a library cross-check against Python's
sorted(), brute-force partition properties, and toy-LM EXSpec equivalence."""
import itertools

import numpy as np
import pytest

from oracle.loops import exspec_decode
from oracle.pool import admission_order, form_batches, form_batches_deferred, refill_window
from oracle.toy_lm import ToyLM


def test_form_batch_spec_examples():
    # window lengths [5,5,3,5], B=2 -> same-length batch of two length-5 members
    p = form_batches([5, 5, 3, 5], [1] * 4, [0, 1, 2, 3], W=4, B=2, min_group=2)
    assert p["batches"][0] == [0, 1] and p["kind"][0] == 1
    # [5,4,3], B=2 -> no group of size >= 2 -> fallback over [5,4]
    p = form_batches([5, 4, 3], [1] * 3, [0, 1, 2], W=3, B=2, min_group=2)
    assert p["batches"][0] == [0, 1] and p["kind"][0] == 0
    # uniform lengths -> every batch same-length
    p = form_batches([7] * 9, [1] * 9, list(range(9)), W=9, B=4, min_group=2)
    assert all(p["kind"])


def test_form_batch_min_group_above_B():
    """R11 with min_group > B (hand-worked): length 7 has 4 members -> one batch of B=2
    (4 >= 3), then 2 < 3 remain; leftovers 2, 3, 4 in window order -> [2,3] (mixed), [4]."""
    p = form_batches([7, 7, 7, 5, 7], [1] * 5, [0, 1, 2, 3, 4], W=5, B=2, min_group=3)
    assert p["batches"] == [[0, 1], [2, 3], [4]] and p["kind"] == [1, 0, 1]


def test_admission_and_window():
    order = admission_order([5, 2, 9, 2], sort_by_length=True)
    assert list(order) == [1, 3, 0, 2]          # ascending prompt length, ties by id
    assert list(admission_order([5, 2, 9], False)) == [0, 1, 2]
    assert refill_window([1, 0, 1, 1], order, 2) == [3, 0]


def _reference_groups(lens, window, B, mg):
    """Independent formulation: sort the window by the library sort on the key
    (-group count, length, window position); walk it cutting batches.  Returns the
    same-length batches and the leftovers in window order."""
    cnt = {l: sum(1 for s in window if lens[s] == l) for l in {lens[s] for s in window}}
    pos = {s: t for t, s in enumerate(window)}
    srt = sorted(window, key=lambda s: (-cnt[lens[s]], lens[s], pos[s]))
    same, left = [], []
    for l, grp in itertools.groupby(srt, key=lambda s: lens[s]):
        grp = list(grp)
        full = [grp[i:i + B] for i in range(0, len(grp), B)]
        while full and len(full[-1]) < (1 if B == 1 else mg):
            left += full.pop()
        same += full
    return same, sorted(left, key=lambda s: pos[s])


def _reference_plan(lens, window, B, mg):
    same, left = _reference_groups(lens, window, B, mg)
    return same + [left[i:i + B] for i in range(0, len(left), B)]


def test_plan_matches_sorted_library_crosscheck():
    rng = np.random.default_rng(3)
    for _ in range(300):
        N = int(rng.integers(1, 40))
        lens = rng.integers(1, 6, N).tolist()
        active = (rng.random(N) < 0.8).astype(int).tolist()
        order = rng.permutation(N).tolist()
        W = int(rng.integers(1, N + 1))
        B = int(rng.integers(1, 9))
        mg = int(rng.integers(2, max(3, B + 1))) if B > 1 else 2
        mg = min(mg, B) if B > 1 else mg
        p = form_batches(lens, active, order, W, B, mg)
        assert p["batches"] == _reference_plan(lens, p["window"], B, mg)


def test_brute_force_partition_properties():
    """Every window of W <= 6 with lengths in {1,2,3} (SURVEY §4 tier 2)."""
    for W in range(1, 7):
        for lens in itertools.product([1, 2, 3], repeat=W):
            for B, mg in [(1, 2), (2, 2), (3, 2), (4, 4), (8, 2)]:
                p = form_batches(list(lens), [1] * W, list(range(W)), W, B, mg)
                members = [s for b in p["batches"] for s in b]
                assert sorted(members) == list(range(W))                # partition
                for b, kind, bl in zip(p["batches"], p["kind"], p["blen"]):
                    assert 1 <= len(b) <= B
                    assert b == sorted(b)                               # window order
                    assert kind == (len({lens[s] for s in b}) == 1)
                    assert bl == max(lens[s] for s in b)
                c = p["counters"]
                assert c[0] == len(p["batches"]) and c[1] == sum(p["kind"])


def test_grouping_rate_collapses_with_batch_size():
    """grouping rates collapse as batch size grows (random lengths)."""
    rng = np.random.default_rng(5)
    rates = {}
    for B in (2, 8):
        tot_same = tot = 0
        for _ in range(50):
            lens = rng.integers(60, 90, 64).tolist()
            p = form_batches(lens, [1] * 64, list(range(64)), 32, B, B)
            tot_same += p["counters"][1]
            tot += p["counters"][0]
        rates[B] = tot_same / tot
    assert rates[8] < rates[2]


@pytest.mark.parametrize("W,B,mg,seq,noise", [(4, 2, 2, False, 0.3), (6, 3, 2, True, 0.2),
                                            (5, 5, 5, False, 0.0), (1, 1, 2, False, 0.3)])
def test_exspec_equals_autoregressive_greedy(W, B, mg, seq, noise):
    """Scheduling is semantically invisible."""
    T = ToyLM(seed=7)
    rng = np.random.default_rng(W * 10 + B)
    prompts = [list(map(int, rng.integers(2, 32, size=int(l)))) for l in rng.integers(1, 12, 6)]
    ref = [T.greedy_generate(p, 14, 1, 64) for p in prompts]
    out, st = exspec_decode(T, T, prompts, 4, 14, 1, 64, W=W, B=B, min_group=mg,
                            sequential=seq, noise=noise)
    assert out == ref
    assert st["verify_calls"] == st["batches"]


def test_exspec_uniform_lengths_all_same_length():
    """All-Mean analog: uniform prompt lengths and clone
    drafts (uniform acceptance) -> grouping rate 1.0 and no realigned members."""
    T = ToyLM(seed=7)
    rng = np.random.default_rng(1)
    prompts = [list(map(int, rng.integers(2, 32, size=6))) for _ in range(4)]
    out, st = exspec_decode(T, T, prompts, 3, 8, -1, 64, W=4, B=2, min_group=2)
    assert st["same_length"] == st["batches"] and st["realigned_members"] == 0


def test_deferred_patience_zero_is_form_batches():
    """R27 with patience 0 (or an all-stale pool) is R11's plan exactly."""
    rng = np.random.default_rng(11)
    for _ in range(300):
        N = int(rng.integers(1, 40))
        lens = rng.integers(1, 6, N).tolist()
        active = (rng.random(N) < 0.8).astype(int).tolist()
        order = rng.permutation(N).tolist()
        W = int(rng.integers(1, N + 1))
        B = int(rng.integers(1, 9))
        mg = int(rng.integers(1, B + 1))
        p = form_batches(lens, active, order, W, B, mg)
        for patience, w0 in ((0, 0), (3, 3), (2, 7)):
            wait = np.full(N, w0, np.int64)
            q = form_batches_deferred(lens, active, order, W, B, mg, wait, patience)
            assert q["batches"] == p["batches"] and q["kind"] == p["kind"] and q["deferred"] == []
            assert (q["counters"] == p["counters"]).all()
            assert all(wait[s] == 0 for s in p["window"])


def test_deferred_brute_force_properties():
    """Every window of W <= 6 with lengths in {1,2,3}, waits in {0,1,2}, patience 1 and 2:
    planned + deferred partition the window; the group batches are R11's; a leftover is
    deferred iff some group batch exists and its wait is below the patience; the fallback
    batches chunk the rest in window order; the waits update as stated."""
    for W in range(1, 7):
        for lens in itertools.product([1, 2, 3], repeat=W):
            rng = np.random.default_rng(hash(lens) & 0xFFFF)
            for B, mg in [(1, 2), (2, 2), (3, 2), (4, 4), (8, 2)]:
                w0 = rng.integers(0, 3, W)
                for patience in (1, 2):
                    wait = w0.copy()
                    q = form_batches_deferred(list(lens), [1] * W, list(range(W)), W, B, mg, wait, patience)
                    planned = [s for b in q["batches"] for s in b]
                    assert sorted(planned + q["deferred"]) == list(range(W))
                    groups, left = _reference_groups(list(lens), list(range(W)), B, mg)
                    assert q["batches"][:len(groups)] == groups
                    if groups:
                        assert q["deferred"] == [s for s in left if w0[s] < patience]
                        run = [s for s in left if w0[s] >= patience]
                    else:
                        assert q["deferred"] == []
                        run = left
                    assert q["batches"][len(groups):] == [run[t:t + B] for t in range(0, len(run), B)]
                    for s in range(W):
                        assert wait[s] == (w0[s] + 1 if s in q["deferred"] else 0)
                    assert len(q["batches"]) >= 1                      # every epoch makes progress


def test_deferred_drain_bounds_waits_and_finishes():
    """A drain under R27 (planted accepts) ends, and no member is deferred more than
    `patience` epochs in a row."""
    rng = np.random.default_rng(4)
    for patience in (1, 2, 4):
        N, B = 48, 4
        lens = rng.integers(5, 30, N).astype(np.int64)
        gen = np.zeros(N, np.int64)
        act = np.ones(N, np.uint8)
        wait = np.zeros(N, np.int64)
        epochs = 0
        while act.any():
            q = form_batches_deferred(lens, act, list(range(N)), N, B, 2, wait, patience)
            assert q["batches"] and wait.max() <= patience
            for b in q["batches"]:
                for s in b:
                    e = min(int(rng.integers(1, 5)), 24 - int(gen[s]))
                    lens[s] += e
                    gen[s] += e
                    if gen[s] >= 24:
                        act[s] = 0
            epochs += 1
            assert epochs < 10_000


@pytest.mark.parametrize("patience,W,B", [(1, 6, 2), (2, 6, 3), (3, 4, 2)])
def test_exspec_deferred_equals_autoregressive_greedy(patience, W, B):
    """Deferring a sequence changes when it is verified, never what it emits (R27)."""
    T = ToyLM(seed=7)
    rng = np.random.default_rng(patience * 10 + W)
    prompts = [list(map(int, rng.integers(2, 32, size=int(l)))) for l in rng.integers(1, 12, 7)]
    ref = [T.greedy_generate(p, 14, 1, 64) for p in prompts]
    out, st = exspec_decode(T, T, prompts, 4, 14, 1, 64, W=W, B=B, min_group=2, noise=0.3,
                            patience=patience)
    assert out == ref


@pytest.mark.parametrize("patience,W,B", [(0, 6, 2), (2, 6, 3), (1, 7, 2)])
def test_exspec_pipelined_equals_autoregressive_greedy(patience, W, B):
    """R28: running an epoch's mixed batches beside the next epoch (their members out of
    that epoch's plan) changes when a sequence is verified, never what it emits."""
    T = ToyLM(seed=7)
    rng = np.random.default_rng(patience * 100 + W * 10 + B)
    prompts = [list(map(int, rng.integers(2, 32, size=int(l)))) for l in rng.integers(1, 12, 8)]
    ref = [T.greedy_generate(p, 14, 1, 64) for p in prompts]
    out, st = exspec_decode(T, T, prompts, 4, 14, 1, 64, W=W, B=B, min_group=2, noise=0.3,
                            patience=patience, pipeline=True)
    assert out == ref


def test_pipeline_window_excludes_exactly_the_previous_mixed_members():
    """R28 by hand: epoch e's mixed batch [0, 2] (lengths 5, 4) keeps 0 and 2 out of epoch
    e+1's window; the same-length batch [1, 3] does not."""
    from oracle.pool import mixed_members, pipeline_window_active
    plan = form_batches([5, 6, 4, 6], [1] * 4, [0, 1, 2, 3], 4, 2, 2)
    assert plan["batches"] == [[1, 3], [0, 2]] and plan["kind"] == [1, 0]
    assert mixed_members(plan) == [0, 2]
    assert pipeline_window_active([1, 1, 1, 1], mixed_members(plan)).tolist() == [0, 1, 0, 1]
    assert pipeline_window_active([1, 0, 1, 1], []).tolist() == [1, 0, 1, 1]
