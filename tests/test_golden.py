"""The oracle against the hand-worked fixtures in tests/golden/ (each file cites the
passage its values come from; none was produced by oracle/ or by the CUDA path)."""
import json
import os

import numpy as np
import pytest

from oracle import align as A
from oracle import metrics as M
from oracle import pool as P
from oracle import verify as V

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        g = json.load(f)
    assert g.get("cite"), name
    return g


def _f(x):
    return float(x) if not isinstance(x, str) else {"inf": np.inf, "-inf": -np.inf, "nan": np.nan}[x]


def test_golden_argmax():
    for c in load("argmax.json")["cases"]:
        x = np.array([_f(v) for v in c["x"]], np.float64)
        assert V.argmax_first(x) == (c["argmax"], c["nan"]), c


def test_golden_widen():
    for c in load("widen.json")["cases"]:
        bits = np.array([int(c["bits"], 16)], np.uint16)
        got = float(V.widen(bits, c["dtype"])[0])
        want = _f(c["value"])
        assert got == want and np.signbit(got) == np.signbit(want), c


def test_golden_emit():
    for c in load("emit.json")["cases"]:
        E, fin = V.emitted_tokens(np.array(c["draft"]), c["a"], c["bonus"], c["eos"], c["budget"])
        assert (E, fin) == (c["E"], c["finished"]), c
        assert A.append_accepted([c["row"]], [E]) == [c["row_after"]], c


def test_golden_expected_tokens():
    for c in load("expected_tokens.json")["cases"]:
        assert M.expected_tokens_per_iteration(c["alpha"], c["k"]) == pytest.approx(c["value"], rel=1e-12), c


def _round_inputs(g, dtype):
    lg = np.array(g["logits"], np.float64)
    if dtype == "fp32":
        return lg.astype(np.float32)
    if dtype == "fp16":
        return lg.astype(np.float16).view(np.uint16)
    return (lg.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)   # exact values


@pytest.mark.parametrize("dtype", ["fp32", "fp16", "bf16"])
def test_golden_eqspec_round(dtype):
    g = load("eqspec_round.json")
    k, cap, L = g["k"], g["cap"], g["L"]
    B = len(g["n"])
    tok, pad, L0 = A.build_batch(g["content"], cap, g["pad_id"])
    assert L0 == L and pad.tolist() == g["pad"] and tok[:, :L].tolist() == g["tokens_before"]
    kv = (100 * np.arange(B)[:, None] + np.arange(cap)[None, :]).astype(np.int64)
    kv = kv[None, :, None, :, None]                       # [planes=1][B][H=1][cap][D=1]
    for c in g["cases"]:
        v = V.batch_verify(_round_inputs(g, dtype), dtype, np.array(g["draft"]), g["n"], g["pad"],
                           np.ones(B, np.uint8), c["eos_id"],
                           None if c["budget"] is None else np.array(c["budget"]), g["pad_id"])
        for key in ("pred", "accept", "bonus", "emit", "finished", "n_new", "pad_new", "kept", "kept_draft"):
            assert np.asarray(v[key]).tolist() == c[key], (c["name"], key)
        assert v["E"] == c["E"] and v["L_new"] == c["L_new"]
        t, mask, pos = A.repad_tokens(tok, cap, k, np.array(g["pad"]), L, v, g["pad_id"])
        Ln = c["L_new"]
        assert t[:, :Ln].tolist() == c["tokens_after"], c["name"]
        assert mask.tolist() == c["mask"] and pos.tolist() == c["pos"], c["name"]
        kv2, defined = A.realign_kv(kv, np.array(g["pad"]), v["pad_new"], v["kept"])
        want = {int(i): {int(col): val for col, val in row.items()} for i, row in c["kv_after"].items()}
        for i in range(B):
            cols = np.flatnonzero(defined[i]).tolist()
            assert cols == sorted(want.get(i, {})), (c["name"], i)
            assert [int(kv2[0, i, 0, col, 0]) for col in cols] == [want[i][col] for col in cols]


def test_golden_repad_examples():
    g = load("repad_examples.json")
    for c in g["build_batch"]:
        _, pad, L = A.build_batch([[1] * n for n in c["lengths"]], cap=16)
        assert (L, pad.tolist()) == (c["L"], c["pad"]), c
    for c in g["plans"]:
        p = V.repad_plan(c["n"], c["accept"], [0] * len(c["n"]))
        assert (p["L_new"], p["pad_new"].tolist(), p["kept"].tolist()) == (c["L_new"], c["pad_new"], c["kept"]), c


def test_golden_pool_plans():
    for c in load("pool_plans.json")["cases"]:
        r = P.form_batches(np.array(c["lens"]), np.array(c["active"]), np.array(c["order"]),
                           c["W"], c["B"], c["min_group"])
        assert r["window"] == c["window"], c["note"]
        assert r["batches"] == c["batches"], c["note"]
        assert r["kind"] == c["kind"] and r["blen"] == c["blen"], c["note"]
        assert r["counters"].tolist() == c["counters"], c["note"]


def test_golden_pool_deferred():
    """Deferred fallback (R27): hand-worked plans and wait updates (tests/golden/pool_deferred.json)."""
    for c in load("pool_deferred.json")["cases"]:
        wait = np.array(c["wait"], np.int64)
        r = P.form_batches_deferred(np.array(c["lens"]), np.array(c["active"]), np.array(c["order"]),
                                    c["W"], c["B"], c["min_group"], wait, c["patience"])
        assert r["window"] == c["window"], c["note"]
        assert r["batches"] == c["batches"], c["note"]
        assert r["kind"] == c["kind"] and r["blen"] == c["blen"], c["note"]
        assert r["deferred"] == c["deferred"], c["note"]
        assert r["counters"].tolist() == c["counters"], c["note"]
        assert wait.tolist() == c["wait_after"], c["note"]
