"""Oracle: Alg. 1 BatchVerify and the BatchRepad plan.

Test infrastructure only (see oracle/__init__.py).

Readings taken:
  R1  all k drafts match -> a = k (PAPER.md:306's argmax(~matches) is degenerate)
  R2  logits are the k+1-row tail; row j predicts draft slot j; bonus = pred[a]
  R4  NaN ranks above +inf, first NaN wins; +0 == -0 (lowest index)
  R5  ties -> lowest index
  R9  finished rows become dummy length-1 rows (excluded from L')
  R10 EOS inside the emitted span cuts after the first EOS; budget trims
"""
from __future__ import annotations

import numpy as np


# ----------------------------------------------------------------------------- widening
def widen(bits: np.ndarray, dtype: str) -> np.ndarray:
    """Raw logit bits -> float64 values (exact for every supported dtype).

    bf16: the 16 bits are the top half of an IEEE binary32 -> shift left 16.
    fp16: IEEE binary16 decode (numpy float16 is exact IEEE incl. subnormals).
    fp32: as is."""
    if dtype == "bf16":
        return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
    if dtype == "fp16":
        return bits.view(np.float16).astype(np.float64)
    if dtype == "fp32":
        return np.asarray(bits, dtype=np.float32).astype(np.float64)
    raise ValueError(dtype)


def argmax_first(x: np.ndarray) -> tuple[int, bool]:
    """pred = argmax over one vocab row, the definition written out:
    if any NaN -> index of the first NaN (R4); else the first index whose value
    equals the maximum (+0 == -0 under ==, so +-0 ties resolve to the lowest index)."""
    nan = np.isnan(x)
    if nan.any():
        return int(np.flatnonzero(nan)[0]), True
    m = x.max()
    return int(np.flatnonzero(x == m)[0]), False


def argmax_rows(logit_bits: np.ndarray, dtype: str):
    """[B, k+1, V] bits -> pred [B, k+1] int64, nan_seen bool."""
    B, K1, _ = logit_bits.shape
    x = widen(logit_bits, dtype)
    pred = np.zeros((B, K1), dtype=np.int64)
    nan_seen = False
    for i in range(B):
        for j in range(K1):
            pred[i, j], nan = argmax_first(x[i, j])
            nan_seen |= nan
    return pred, nan_seen


# ----------------------------------------------------------------------------- Alg. 1
def accept_and_bonus(pred_row: np.ndarray, draft_row: np.ndarray, k: int) -> tuple[int, int]:
    """matches = (pred = D); J = first mismatch (R1: k if
    none); A = D[:J]; bonus = pred at the first mismatch (R2)."""
    a = k
    for j in range(k):
        if pred_row[j] != draft_row[j]:
            a = j
            break
    return a, int(pred_row[a])


def emitted_tokens(draft_row, a: int, bonus: int, eos_id: int, budget: int | None):
    """E = A[i] ++ [B[i]], cut after the first EOS (R10) and to the
    remaining budget.  Returns (E, finished)."""
    E = [int(t) for t in draft_row[:a]] + [int(bonus)]
    finished = False
    if eos_id >= 0 and eos_id in E:
        E = E[: E.index(eos_id) + 1]
        finished = True
    if budget is not None and len(E) >= max(int(budget), 0):
        E = E[:max(int(budget), 0)]
        finished = True
    return E, finished


def batch_verify(logit_bits, dtype, draft, n, pad, active, eos_id=-1, budget=None, pad_id=0):
    """Full K1 semantics: per-row (accept, bonus, emit, finished) + the BatchRepad plan.

    logit_bits [B, k+1, V]; draft [B, k]; n, pad [B] (content length incl. the pending
    token, left pads); active [B] 0/1; budget [B] remaining new tokens or None.
    Returns a dict of numpy arrays."""
    draft = np.asarray(draft)
    B, k = draft.shape
    pred, _ = argmax_rows(logit_bits, dtype)
    # R4 status: a NaN among the logits of the rows verified this round (a row that is not
    # active is not read at all)
    live = np.asarray(active).astype(bool)
    nan_seen = bool(np.isnan(widen(logit_bits[live], dtype)).any()) if live.any() else False
    accept = np.zeros(B, np.int32)
    bonus = np.full(B, pad_id, np.int64)
    emit = np.zeros(B, np.int32)
    finished = np.zeros(B, np.uint8)
    E_rows = []
    for i in range(B):
        if not active[i]:
            finished[i] = 1
            E_rows.append([])
            continue
        a, b = accept_and_bonus(pred[i], draft[i], k)
        E, fin = emitted_tokens(draft[i], a, b, eos_id, None if budget is None else int(budget[i]))
        accept[i], bonus[i], emit[i], finished[i] = a, b, len(E), int(fin)
        E_rows.append(E)
    plan = repad_plan(n, accept, finished, k)
    return dict(pred=pred, accept=accept, bonus=bonus, emit=emit, finished=finished,
                E=E_rows, nan=nan_seen, **plan)


def repad_plan(n, accept, finished, k=None):
    """BatchRepad plan (§3.1; R6 minimal padding, R9 dummies).

    Still-active rows: n' = n + a + 1 (accepted + bonus), kept = n + a (the bonus has
    no KV yet).  Finished rows: n' = 1, kept = 0.
    L' = max n' over still-active rows (0 if none); p' = L' - n'."""
    n = np.asarray(n, np.int64)
    B = len(n)
    n_new = np.ones(B, np.int64)
    kept = np.zeros(B, np.int64)
    alive = np.asarray(finished) == 0
    n_new[alive] = n[alive] + np.asarray(accept, np.int64)[alive] + 1
    kept[alive] = n[alive] + np.asarray(accept, np.int64)[alive]
    L_new = int(n_new[alive].max()) if alive.any() else 0
    pad_new = np.where(L_new > 0, L_new - n_new, 0)
    out = dict(L_new=L_new, n_new=n_new.astype(np.int32), pad_new=pad_new.astype(np.int32),
               kept=kept.astype(np.int32))
    if k is not None:
        # f1: a draft model that cached its own forwards holds KV for the
        # pending token and d_1..d_{k-1} (d_k is generated, never forwarded),
        # so it keeps the old content plus min(a, k-1) accepted drafts.
        kd = np.zeros(B, np.int64)
        kd[alive] = n[alive] + np.minimum(np.asarray(accept, np.int64)[alive], k - 1)
        out["kept_draft"] = kd.astype(np.int32)
    return out
