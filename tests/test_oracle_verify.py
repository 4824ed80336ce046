"""Pins for oracle/verify.py (Alg. 1 BatchVerify) against values the
paper / SPEC / IEEE-754 / an independent library fix -- never against itself."""
import numpy as np
import pytest
import torch

from oracle import verify as V
from oracle.metrics import expected_tokens_per_iteration
from synth import workloads as W


def f32(vals):
    return np.asarray(vals, np.float32)


# --------------------------------------------------------------------------- widening
def test_widen_ieee_values():
    bf = np.array([0x3F80, 0xC000, 0x7F80, 0xFF80, 0x0001, 0x8000, 0x4049], np.uint16)
    got = V.widen(bf, "bf16")
    assert got[0] == 1.0 and got[1] == -2.0
    assert got[2] == np.inf and got[3] == -np.inf
    assert got[4] == 2.0 ** -133                       # smallest bf16 subnormal
    assert got[5] == 0.0 and np.signbit(got[5])
    assert got[6] == 3.140625
    fp = np.array([0x3C00, 0x0001, 0x7BFF, 0xFC00, 0x0400], np.uint16)
    got = V.widen(fp, "fp16")
    assert list(got) == [1.0, 2.0 ** -24, 65504.0, -np.inf, 2.0 ** -14]
    assert np.isnan(V.widen(np.array([0x7E00], np.uint16), "fp16")[0])
    assert np.isnan(V.widen(np.array([0x7FC0], np.uint16), "bf16")[0])


# --------------------------------------------------------------------------- argmax
@pytest.mark.parametrize("row,expect", [([0.1, 0.9, 0.3], 1), ([0.5, 0.5], 0), ([0.25] * 7, 0)])
def test_argmax_spec_examples(row, expect):
    # the argmax, ties to the lowest token id
    assert V.argmax_first(V.widen(f32(row), "fp32"))[0] == expect


def test_argmax_special_values():
    nan, inf = np.nan, np.inf
    cases = [
        ([1.0, nan, inf, nan], 1, True),        # first NaN wins, NaN above +inf (R4)
        ([-0.0, 0.0, -1.0], 0, False),          # +-0 equal -> lowest index
        ([0.0, -0.0], 0, False),
        ([-inf, -inf], 0, False),               # all -inf -> 0
        ([-inf, 3.0, inf, inf], 2, False),
    ]
    for row, want, isnan in cases:
        got, nan_seen = V.argmax_first(np.asarray(row, np.float64))
        assert (got, nan_seen) == (want, isnan), row


@pytest.mark.parametrize("dtype", ["bf16", "fp16", "fp32"])
def test_argmax_matches_torch_library(dtype):
    """Library cross-check: torch.argmax on CPU (first index on ties, first NaN wins)."""
    rng = np.random.default_rng(11)
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[dtype]
    for trial in range(60):
        V_ = int(rng.integers(1, 300))
        x = torch.from_numpy(rng.integers(-4, 5, V_).astype(np.float32) / 2).to(tdt)
        if trial % 5 == 1:
            x[rng.integers(V_)] = float("nan")
        if trial % 5 == 2:
            x[rng.integers(V_)] = float("inf")
            x[rng.integers(V_)] = -0.0
        if trial % 7 == 3:
            x[:] = -float("inf")
        bits = x.view(torch.int16).numpy().view(np.uint16) if dtype != "fp32" else x.numpy()
        got, _ = V.argmax_first(V.widen(bits, dtype))
        assert got == int(torch.argmax(x.float())), (trial, x)


# --------------------------------------------------------------------------- Alg. 1
def _planted_bits(pred, V_, dtype="fp32"):
    B, K1 = pred.shape
    x = np.zeros((B, K1, V_), np.float32)
    for i in range(B):
        for j in range(K1):
            x[i, j, pred[i, j]] = 1.0
    return W.to_dtype_bits_np(x, dtype)


def test_verify_spec_examples():
    k, V_ = 5, 16
    tgt = np.array([[3, 4, 5, 6, 7, 8]])
    # draft == target continuation -> a = K, bonus = the (K+1)-th greedy token
    r = V.batch_verify(_planted_bits(tgt, V_), "fp32", tgt[:, :k], [4], [0], [1])
    assert r["accept"][0] == k and r["bonus"][0] == 8 and r["emit"][0] == k + 1
    # wrong at position 0 -> a = 0, bonus = the target's next token
    d = tgt[:, :k].copy()
    d[0, 0] = 9
    r = V.batch_verify(_planted_bits(tgt, V_), "fp32", d, [4], [0], [1])
    assert r["accept"][0] == 0 and r["bonus"][0] == 3 and r["E"][0] == [3]
    # first mismatch, not a count of matches: slots after it may match again
    d = tgt[:, :k].copy()
    d[0, 2] = 0
    r = V.batch_verify(_planted_bits(tgt, V_), "fp32", d, [4], [0], [1])
    assert r["accept"][0] == 2 and r["bonus"][0] == 5 and r["E"][0] == [3, 4, 5]


def test_emitted_tokens_spec_append_examples():
    # SPEC.md:145-147
    assert V.emitted_tokens([8, 9, 4], 2, 7, eos_id=1, budget=None) == ([8, 9, 7], False)
    assert V.emitted_tokens([8, 9], 0, 7, eos_id=1, budget=None) == ([7], False)
    assert V.emitted_tokens([8, 1, 5], 2, 7, eos_id=1, budget=None) == ([8, 1], True)
    # budget trim: 3 tokens would be emitted, 2 allowed
    assert V.emitted_tokens([8, 9], 2, 7, eos_id=-1, budget=2) == ([8, 9], True)
    assert V.emitted_tokens([8, 9], 2, 7, eos_id=-1, budget=3) == ([8, 9, 7], True)


def test_inactive_rows():
    tgt = np.array([[3, 4, 5], [3, 4, 5]])
    r = V.batch_verify(_planted_bits(tgt, 8), "fp32", tgt[:, :2], [3, 1], [0, 2], [1, 0], pad_id=0)
    assert r["accept"][1] == 0 and r["bonus"][1] == 0 and r["emit"][1] == 0 and r["finished"][1] == 1
    # the dummy row is excluded from L' and gets p' = L' - 1 (R9)
    assert r["L_new"] == 3 + 2 + 1 and r["pad_new"][1] == r["L_new"] - 1 and r["kept"][1] == 0


@pytest.mark.parametrize("pattern", W.ACCEPT_PATTERNS)
@pytest.mark.parametrize("dtype", ["bf16", "fp16", "fp32"])
def test_verify_recovers_planted_answer(pattern, dtype):
    """The generator planted (argmax, accept) independently of the oracle."""
    B, k, V_ = 6, 5, 777
    for r in range(4):
        rt = W.gen_round_truth(2, r, B, k, V_, pattern, alpha=0.6, tie_rate=2)
        bits = W.gen_logits_np(2, r, B, k, V_, dtype, tie_rate=2)
        res = V.batch_verify(bits, dtype, rt.draft, [10] * B, [0] * B, [1] * B)
        assert np.array_equal(res["pred"], rt.pred)
        assert np.array_equal(res["accept"], rt.accept)
        assert np.array_equal(res["bonus"], rt.pred[np.arange(B), rt.accept])


@pytest.mark.parametrize("alpha", [0.3, 0.5, 0.8])
def test_accept_process_matches_closed_form(alpha):
    """E[accept + 1] = (1 - alpha^(k+1)) / (1 - alpha) -- Monte Carlo through
    the oracle's verify on the generator's Bernoulli(alpha) drafts (>= 10k rounds)."""
    B, k, V_ = 64, 5, 64
    tot, cnt = 0, 0
    for r in range(160):
        rt = W.gen_round_truth(5, r, B, k, V_, "fixed", alpha=alpha)
        bits = W.gen_logits_np(5, r, B, k, V_, "fp32")
        res = V.batch_verify(bits, "fp32", rt.draft, [8] * B, [0] * B, [1] * B)
        tot += int((res["accept"] + 1).sum())
        cnt += B
    assert cnt >= 10_000
    assert abs(tot / cnt / expected_tokens_per_iteration(alpha, k) - 1) < 0.05


def test_closed_form_values():
    # alpha = 0.8, k = 5 -> 3.68928; alpha = 0 -> 1
    assert abs(expected_tokens_per_iteration(0.8, 5) - 3.68928) < 1e-9
    assert expected_tokens_per_iteration(0.0, 5) == 1.0
    assert abs(expected_tokens_per_iteration(0.999999, 5) - 6.0) < 1e-4


def test_nan_logits_flag_and_result():
    x = np.zeros((1, 2, 4), np.float32)
    x[0, 0, 2] = np.nan
    r = V.batch_verify(x, "fp32", [[2]], [1], [0], [1])
    assert r["nan"] and r["pred"][0, 0] == 2 and r["accept"][0] == 1
