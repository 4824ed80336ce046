"""Thread-parallel driver of the oracle, for the CPU baseline timing ("the
same per-element code with a std::thread parallel-for over independent (plane, row, head)
slabs on nproc cores").

Test / measurement infrastructure only (see oracle/__init__.py).  It adds no arithmetic:
the oracle's own functions run unchanged on independent pieces, on `threads` host
threads (numpy releases the GIL inside its loops and copies):

  * Alg. 1 per batch row -- oracle.verify.batch_verify on the row alone (rows are
    independent until the BatchRepad plan), then the plan over all rows
    (oracle.verify.repad_plan);
  * the unpad-append-repad of the tokens (oracle.align.repad_tokens; KB of work, serial);
  * Realign per (plane, row) slab group -- oracle.align.realign_kv_inplace on that slice
    (slabs are independent).

`eqspec_round_parallel` returns exactly what the serial composition returns; pinned by
tests/test_oracle_driver.py.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .align import realign_kv_inplace, repad_tokens
from .verify import batch_verify, repad_plan


def host_threads() -> int:
    """The host cores this process may run on."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover -- non-Linux
        return os.cpu_count() or 1


def batch_verify_parallel(pool, logit_bits, dtype, draft, n, pad, active, eos_id=-1, budget=None, pad_id=0):
    """oracle.verify.batch_verify with its per-row Alg. 1 work spread over threads."""
    draft = np.asarray(draft)
    B, k = draft.shape

    def one(i):
        bud = None if budget is None else np.asarray(budget)[i:i + 1]
        return batch_verify(logit_bits[i:i + 1], dtype, draft[i:i + 1], np.asarray(n)[i:i + 1],
                            np.asarray(pad)[i:i + 1], np.asarray(active)[i:i + 1], eos_id, bud, pad_id)
    rows = list(pool.map(one, range(B)))
    cat = lambda key: np.concatenate([r[key] for r in rows])
    res = dict(pred=cat("pred"), accept=cat("accept"), bonus=cat("bonus"), emit=cat("emit"),
               finished=cat("finished"), E=[r["E"][0] for r in rows], nan=any(r["nan"] for r in rows))
    res.update(repad_plan(n, res["accept"], res["finished"], k))
    return res


def realign_parallel(pool, kv, pad_old, pad_new, kept):
    """oracle.align.realign_kv_inplace on every (plane, row) slice [1, 1, H, cap, D] of kv
    [planes, B, H, cap, D], in place, over threads."""
    P, B = kv.shape[0], kv.shape[1]

    def one(t):
        p, i = divmod(t, B)
        realign_kv_inplace(kv[p:p + 1, i:i + 1], pad_old[i:i + 1], pad_new[i:i + 1], kept[i:i + 1])
    list(pool.map(one, range(P * B)))
    return kv


def eqspec_round_parallel(pool, logit_bits, dtype, draft, tokens, cap, k, n, pad, L, active, kv,
                          eos_id=-1, budget=None, pad_id=0):
    """One EqSpec round (K1 -> K3 -> K2 semantics) through the oracle on `pool`'s threads;
    kv is realigned in place.  Returns (verify result, tokens', mask, pos)."""
    v = batch_verify_parallel(pool, logit_bits, dtype, draft, n, pad, active, eos_id, budget, pad_id)
    tok_n, mask, pos = repad_tokens(tokens, cap, k, pad, L, v, pad_id)
    realign_parallel(pool, kv, pad, v["pad_new"], v["kept"])
    return v, tok_n, mask, pos


def make_pool(threads: int | None = None) -> ThreadPoolExecutor:
    return ThreadPoolExecutor(max_workers=threads or host_threads())
