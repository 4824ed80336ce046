"""Oracle-side toy causal LM (SPEC.md toy_lm).

Test infrastructure only (see oracle/__init__.py).  Used to pin the oracle's
verify / repad / realign composition against per-sequence autoregressive greedy
decoding (the paper's equivalence requirement).

* fp64 arithmetic, every reduction an explicit left-to-right sum, so
  results never depend on batch shape or padding;
* absolute sinusoidal positions looked up by position id: a wrong
  position id changes the output (the BSP failure class);
* K/V are STORED as bf16 bit patterns in a [planes = layers*2, H, cap, D] row cache,
  so a realignment moves real 16-byte bf16 rows (D = 8);
* masked (pad) columns are skipped: they contribute exactly zero weight.
"""
from __future__ import annotations

import numpy as np


def bf16_bits(x64: np.ndarray) -> np.ndarray:
    """fp64 -> fp32 (RNE) -> bf16 (RNE on the fp32 bits); finite inputs only."""
    b = np.asarray(x64, np.float64).astype(np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_value(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def lsum(x: np.ndarray, axis: int = 0) -> np.ndarray:
    """Left-to-right sum (np.cumsum is a sequential accumulate)."""
    if x.shape[axis] == 0:
        return np.zeros(np.delete(x.shape, axis))
    return np.take(np.cumsum(x, axis=axis), -1, axis=axis)


def matvec(x: np.ndarray, W: np.ndarray) -> np.ndarray:
    """x @ W with each output an explicit left-to-right sum over x's index."""
    acc = np.zeros(W.shape[1])
    for j in range(W.shape[0]):
        acc = acc + x[j] * W[j]
    return acc


def rmsnorm(x: np.ndarray) -> np.ndarray:
    return x / np.sqrt(lsum(x * x) / len(x) + 1e-6)


def greedy_fp32(logits64: np.ndarray) -> int:
    """The target's greedy token: argmax of the logits as the verifier sees them (fp32),
    first NaN / lowest index on ties (same decision precision as K1)."""
    x = logits64.astype(np.float32).astype(np.float64)
    nan = np.isnan(x)
    if nan.any():
        return int(np.flatnonzero(nan)[0])
    return int(np.flatnonzero(x == x.max())[0])


class ToyLM:
    LOGIT_SCALE = 1.0
    ATT_SCALE = 1.0

    def __init__(self, V=32, layers=2, H=2, D=8, seed=7, max_pos=512):
        if min(V, layers, H, D) < 1 or V < 4:
            raise ValueError("invalid toy config")
        self.V, self.layers, self.H, self.D = V, layers, H, D
        dm = H * D
        self.dm = dm
        rng = np.random.default_rng(seed)
        self.emb = rng.standard_normal((V, dm))
        self.Wq, self.Wk, self.Wv, self.Wo, self.W1, self.W2 = ([] for _ in range(6))
        for _ in range(layers):
            self.Wq.append(rng.standard_normal((dm, dm)) / np.sqrt(dm))
            self.Wk.append(rng.standard_normal((dm, dm)) / np.sqrt(dm))
            self.Wv.append(rng.standard_normal((dm, dm)) / np.sqrt(dm))
            self.Wo.append(rng.standard_normal((dm, dm)) / np.sqrt(dm))
            self.W1.append(rng.standard_normal((dm, 2 * dm)) / np.sqrt(dm))
            self.W2.append(rng.standard_normal((2 * dm, dm)) / np.sqrt(2 * dm))
        self.Wu = rng.standard_normal((dm, V)) * (self.LOGIT_SCALE / np.sqrt(dm))
        pos = np.arange(max_pos)[:, None]
        i = np.arange(dm)[None, :]
        ang = pos / np.power(10000.0, (2 * (i // 2)) / dm)
        self.pe = np.where(i % 2 == 0, np.sin(ang), np.cos(ang))

    @property
    def n_planes(self):
        return 2 * self.layers

    def new_row_cache(self, cap):
        return np.zeros((self.n_planes, self.H, cap, self.D), np.uint16)

    def token_forward(self, tok: int, pos: int, col: int, cache_row: np.ndarray,
                      mask_row: np.ndarray) -> np.ndarray:
        """One token at cache column `col` with position id `pos`; writes its K/V into
        cache_row[:, :, col] and attends to columns c <= col with mask_row[c] == 1.
        Returns fp64 logits [V]."""
        H, D = self.H, self.D
        x = self.emb[tok] + self.pe[pos]
        for l in range(self.layers):
            hn = rmsnorm(x)
            q = matvec(hn, self.Wq[l]).reshape(H, D)
            cache_row[2 * l, :, col, :] = bf16_bits(matvec(hn, self.Wk[l]).reshape(H, D))
            cache_row[2 * l + 1, :, col, :] = bf16_bits(matvec(hn, self.Wv[l]).reshape(H, D))
            cols = np.flatnonzero(mask_row[:col + 1] == 1)
            att = np.zeros((H, D))
            for h in range(H):
                Kc = bf16_value(cache_row[2 * l, h, cols, :])          # [n, D]
                Vc = bf16_value(cache_row[2 * l + 1, h, cols, :])
                s = lsum(q[h][None, :] * Kc, axis=1) * (self.ATT_SCALE / np.sqrt(D))
                w = np.exp(s - s.max())
                att[h] = lsum(w[:, None] * Vc, axis=0) / lsum(w)
            x = x + matvec(att.reshape(-1), self.Wo[l])
            x = x + matvec(np.maximum(matvec(rmsnorm(x), self.W1[l]), 0.0), self.W2[l])
        return matvec(rmsnorm(x), self.Wu)

    # ------------------------------------------------------------------ references
    def greedy_generate(self, prompt, max_new: int, eos_id: int, cap: int):
        """Per-sequence non-speculative greedy decoding (the equivalence reference,
        SPEC.md:250-257): no padding, positions 0.., one token at a time."""
        cache = self.new_row_cache(cap)
        ones = np.ones(cap, np.int64)
        logits = None
        for c, t in enumerate(prompt):
            logits = self.token_forward(int(t), c, c, cache, ones)
        out, c = [], len(prompt)
        while len(out) < max_new:
            nxt = greedy_fp32(logits)
            out.append(nxt)
            if nxt == eos_id or len(out) == max_new:
                break
            logits = self.token_forward(nxt, c, c, cache, ones)
            c += 1
        return out

    def propose(self, content, k: int, noise: float = 0.0, seed: int = 0):
        """Draft generation in recompute mode: greedy continuation of the
        unpadded content, k tokens; with `noise` each proposal is replaced by another
        token with that probability (deterministic in the sequence state)."""
        cap = len(content) + k + 1
        cache = self.new_row_cache(cap)
        ones = np.ones(cap, np.int64)
        for c, t in enumerate(content):
            logits = self.token_forward(int(t), c, c, cache, ones)
        props, c = [], len(content)
        rng = np.random.default_rng([seed, len(content), int(np.sum(content)) % (1 << 31)])
        for _ in range(k):
            t = greedy_fp32(logits)
            if noise > 0 and rng.random() < noise:
                t = (t + 1 + int(rng.integers(self.V - 1))) % self.V
            props.append(t)
            logits = self.token_forward(t, c, c, cache, ones)
            c += 1
        return props
