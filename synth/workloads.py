"""Seeded synthetic workloads shaped like the paper's model pairs (BASELINE.json configs).

Input construction only.  Nothing here computes what the method computes: the
logits carry *planted* maxima and the drafts are built to agree with them for a
Bernoulli(alpha) number of slots, so the generator knows the intended
(accept, bonus) of every row -- an answer that is independent of both the
oracle and the CUDA path.

Every generator has a numpy form (host) and, where sizes need it, a torch form
(any device) that produces the same bits from the same counter-based hash.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .hashgen import hash_np, hash_torch, uniform_np

PAD_ID = 0
EOS_ID = 1

# hash streams
S_LEN, S_TOK, S_BG, S_TGT, S_TIE, S_ALPHA, S_ACC, S_DRAFT, S_KV, S_POOL, S_NAT = range(1, 12)


@dataclass(frozen=True)
class Shape:
    """One BASELINE.json config (model-pair shape) -- sizes only."""
    name: str
    V: int               # vocab
    layers: int
    H: int               # KV heads
    D: int               # head_dim
    kv_dtype: str        # 'fp16' | 'bf16'
    logit_dtype: str     # 'fp16' | 'bf16' | 'fp32'
    B: int
    k: int
    ctx: int             # context the lengths are drawn around
    len_lo: int          # n_i ~ U[len_lo, len_hi]
    len_hi: int
    cap: int = 0         # KV / token capacity in positions (0 = derive)

    @property
    def n_planes(self) -> int:
        return self.layers * 2

    @property
    def elem(self) -> int:
        return 2

    @property
    def bpt(self) -> int:
        """KV bytes per token per sequence = layers * 2 * H * D * elem."""
        return self.layers * 2 * self.H * self.D * self.elem

    def with_(self, **kw) -> "Shape":
        return replace(self, **kw)


def derive_cap(shape: Shape, rounds: int) -> int:
    """Capacity so that `rounds` rounds fit: widths grow by <= k+1 per round and the
    next forward needs k more columns; rounded up to a multiple of 16."""
    need = shape.len_hi + (rounds + 1) * (shape.k + 1) + shape.k
    return (need + 15) // 16 * 16


SHAPES = {
    # configs[0]: toy: B=2, k=4, vocab 32, 2 layers x 2 KV heads x head_dim 8, max_len 64
    "toy": Shape("toy", 32, 2, 2, 8, "bf16", "fp32", 2, 4, 16, 1, 16, cap=64),
    # configs[1]: Vicuna-7B/68M: vocab 32000, 32 x 32 x 128, fp16, B=8, k=5, ctx 2048
    "vicuna": Shape("vicuna", 32000, 32, 32, 128, "fp16", "fp16", 8, 5, 2048, 1536, 2048),
    # configs[2]: Qwen3-8B/0.6B: vocab 151936, 36 x 8 x 128, bf16, B=1..8, k=5 (ctx 2048, R17)
    "qwen3": Shape("qwen3", 151936, 36, 8, 128, "bf16", "bf16", 8, 5, 2048, 1536, 2048),
    # configs[3]: GLM-4-9B/0.6B: vocab 151552, 40 x 2 x 128, bf16, B=8, k=7, ctx 4096
    "glm4": Shape("glm4", 151552, 40, 2, 128, "bf16", "bf16", 8, 7, 4096, 3584, 4096),
}


# ----------------------------------------------------------------------------- lengths / tokens
def gen_lengths(shape: Shape, seed: int, B: int | None = None) -> np.ndarray:
    B = shape.B if B is None else B
    h = hash_np(seed, S_LEN, np.arange(B))
    span = shape.len_hi - shape.len_lo + 1
    return (shape.len_lo + (h % np.uint64(span)).astype(np.int64)).astype(np.int32)


def gen_content_tokens(seed: int, n_total: int, V: int, stream_offset: int = 0) -> np.ndarray:
    """Content token ids in [2, V) (0 = pad, 1 = eos are reserved)."""
    h = hash_np(seed, S_TOK, np.arange(n_total) + stream_offset)
    return (2 + (h % np.uint64(V - 2)).astype(np.int64)).astype(np.int64)


def left_padded_tokens(lengths: np.ndarray, cap: int, seed: int, V: int) -> np.ndarray:
    """[B, cap] int64: row i has content in [L - n_i, L), pad elsewhere (L = max n)."""
    B = len(lengths)
    L = int(lengths.max())
    out = np.full((B, cap), PAD_ID, dtype=np.int64)
    for i, n in enumerate(lengths):
        out[i, L - n:L] = gen_content_tokens(seed, int(n), V, stream_offset=i * 1_000_003)
    return out


# ----------------------------------------------------------------------------- logits
def _bg_value_from_hash(h: np.ndarray, dtype: str) -> np.ndarray:
    """Background logits in [-4, 4) on a grid exactly representable in `dtype`."""
    if dtype == "bf16":
        q = (h >> np.uint64(56)).astype(np.float32)
        return -4.0 + q / 32.0
    if dtype == "fp16":
        q = (h >> np.uint64(53)).astype(np.float32)
        return -4.0 + q / 256.0
    q = (h >> np.uint64(48)).astype(np.float32)
    return (-4.0 + q / 8192.0).astype(np.float32)


def to_dtype_bits_np(x32: np.ndarray, dtype: str) -> np.ndarray:
    """Exact cast (values are on a representable grid) -> raw bits (uint16 / float32)."""
    x32 = np.ascontiguousarray(x32, dtype=np.float32)
    if dtype == "bf16":
        b = x32.view(np.uint32)
        assert not np.any(b & 0xFFFF), "value not exactly representable in bf16"
        return (b >> 16).astype(np.uint16)
    if dtype == "fp16":
        h = x32.astype(np.float16)
        assert np.array_equal(h.astype(np.float32), x32), "value not exact in fp16"
        return h.view(np.uint16)
    return x32


PLANT = 8.0  # exact in every logit dtype, above the [-4, 4) background


@dataclass
class RoundTruth:
    """What the generator planted for one round (the intended answer)."""
    pred: np.ndarray     # [B, k+1] intended argmax (lowest index among planted maxima)
    accept: np.ndarray   # [B] intended accept length
    draft: np.ndarray    # [B, k] int64


def planted_targets(seed: int, r: int, B: int, k: int, V: int, tie_rate: int = 16):
    """Per (row, slot): the planted max index T, and an optional second planted
    index (tie) -> intended argmax = min of the planted set."""
    idx = (np.arange(B)[:, None] + r * B) * (k + 1) + np.arange(k + 1)[None, :]
    t1 = (hash_np(seed, S_TGT, idx) % np.uint64(V)).astype(np.int64)
    ht = hash_np(seed, S_TIE, idx)
    tie = ((ht & np.uint64(tie_rate - 1)) == 0) if tie_rate > 0 else np.zeros_like(t1, bool)
    t2 = ((ht >> np.uint64(8)) % np.uint64(V)).astype(np.int64)
    tie &= t2 != t1
    t2 = np.where(tie, t2, -1)
    pred = np.where(tie, np.minimum(t1, t2), t1)
    return t1, t2, pred


def gen_logits_np(seed: int, r: int, B: int, k: int, V: int, dtype: str, planted: bool = True,
                  tie_rate: int = 16) -> np.ndarray:
    """Round r's logits tail [B, k+1, V] as raw bits (uint16 for fp16/bf16, float32)."""
    n = B * (k + 1) * V
    h = hash_np(seed, S_BG, np.arange(n, dtype=np.uint64) + np.uint64(r * n))
    x = _bg_value_from_hash(h, dtype).reshape(B, k + 1, V)
    if planted:
        t1, t2, _ = planted_targets(seed, r, B, k, V, tie_rate)
        bi, ji = np.meshgrid(np.arange(B), np.arange(k + 1), indexing="ij")
        x[bi, ji, t1] = PLANT
        m = t2 >= 0
        x[bi[m], ji[m], t2[m]] = PLANT
    return to_dtype_bits_np(x, dtype)


def gen_logits_torch(seed: int, r: int, B: int, k: int, V: int, dtype: str, device,
                     planted: bool = True, tie_rate: int = 16, row_stride: int | None = None):
    """Same bits as gen_logits_np, produced on `device`. Returns a torch tensor of the
    logit dtype, shape [B, k+1, row_stride] (row_stride >= V, tail left zero)."""
    import torch
    n = B * (k + 1) * V
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[dtype]
    rs = V if row_stride is None else row_stride
    out = torch.zeros(B, k + 1, rs, dtype=tdt, device=device)
    idx = torch.arange(n, dtype=torch.int64, device=device) + r * n
    h = hash_torch(seed, S_BG, idx)
    if dtype == "bf16":
        q = ((h >> 56) & 0xFF).to(torch.float32)
        x = -4.0 + q / 32.0
    elif dtype == "fp16":
        q = ((h >> 53) & 0x7FF).to(torch.float32)
        x = -4.0 + q / 256.0
    else:
        q = ((h >> 48) & 0xFFFF).to(torch.float32)
        x = -4.0 + q / 8192.0
    del h, idx
    x = x.view(B, k + 1, V)
    if planted:
        t1, t2, _ = planted_targets(seed, r, B, k, V, tie_rate)
        t1t = torch.from_numpy(t1).to(device)
        x.scatter_(2, t1t.unsqueeze(-1), PLANT)
        m = t2 >= 0
        if m.any():
            bi, ji = np.nonzero(m)
            x[torch.from_numpy(bi).to(device), torch.from_numpy(ji).to(device),
              torch.from_numpy(t2[m]).to(device)] = PLANT
    out[:, :, :V] = x.to(tdt)
    return out


def gen_natural_logits_np(seed: int, r: int, B: int, k: int, V: int, dtype: str) -> np.ndarray:
    """Unplanted logits (natural ties; bf16's 256-value grid makes many) -- raw bits."""
    n = B * (k + 1) * V
    h = hash_np(seed, S_NAT, np.arange(n, dtype=np.uint64) + np.uint64(r * n))
    return to_dtype_bits_np(_bg_value_from_hash(h, dtype).reshape(B, k + 1, V), dtype)


# ----------------------------------------------------------------------------- drafts
ACCEPT_PATTERNS = ("alpha", "fixed", "all_k", "all_0", "alternating", "one_zero")


def gen_round_truth(seed: int, r: int, B: int, k: int, V: int, pattern: str = "alpha",
                    alpha: float = 0.7, tie_rate: int = 16) -> RoundTruth:
    """Drafts for round r that agree with the planted argmax for a Bernoulli(alpha_i)
    number of leading slots (alpha_i ~ U[0.5, 0.9] per row for 'alpha').  After the
    first disagreement, later slots copy the planted argmax with probability 1/2
    (so a "count of matches" reading would differ from "first mismatch")."""
    _, _, pred = planted_targets(seed, r, B, k, V, tie_rate)
    base = (np.arange(B)[:, None] + r * B) * k + np.arange(k)[None, :]
    u = uniform_np(seed, S_ACC, base)
    if pattern == "alpha":
        a_row = 0.5 + 0.4 * uniform_np(seed, S_ALPHA, np.arange(B))
    else:
        a_row = np.full(B, alpha)
    acc_ok = u < a_row[:, None]
    accept = np.where(acc_ok.all(axis=1), k, np.argmin(acc_ok, axis=1)).astype(np.int32)
    if pattern == "all_k":
        accept[:] = k
    elif pattern == "all_0":
        accept[:] = 0
    elif pattern == "alternating":
        accept = np.where(np.arange(B) % 2 == 0, k, 0).astype(np.int32)
    elif pattern == "one_zero":
        accept[:] = k
        accept[0] = 0
    hd = hash_np(seed, S_DRAFT, base)
    wrong = (pred[:, :k] + 1 + (hd % np.uint64(V - 1)).astype(np.int64)) % V  # != pred
    copy_later = ((hd >> np.uint64(40)) & np.uint64(1)) == 1
    j = np.arange(k)[None, :]
    draft = np.where(j < accept[:, None], pred[:, :k],
                     np.where((j > accept[:, None]) & copy_later, pred[:, :k], wrong))
    return RoundTruth(pred=pred, accept=accept, draft=draft.astype(np.int64))


# ----------------------------------------------------------------------------- KV cache
def gen_kv_bits_np(seed: int, n_elems: int, offset: int = 0) -> np.ndarray:
    """n_elems finite 16-bit float patterns (bit 14 cleared: |x| < 2, never inf/NaN)."""
    g0 = offset // 4
    ng = (offset + n_elems + 3) // 4 - g0
    h = hash_np(seed, S_KV, np.arange(ng, dtype=np.uint64) + np.uint64(g0))
    w = h.view(np.uint16)[offset - 4 * g0: offset - 4 * g0 + n_elems]
    return w & np.uint16(0xBFFF)


def gen_kv_torch(seed: int, shape, dtype, device, chunk: int = 1 << 26):
    """Same bits as gen_kv_bits_np over the flattened `shape`, on `device`."""
    import torch
    n = int(np.prod(shape))
    out = torch.empty(n, dtype=torch.int16, device=device)
    for s in range(0, n, chunk * 4):
        e = min(n, s + chunk * 4)
        ng = (e - s + 3) // 4
        idx = torch.arange(ng, dtype=torch.int64, device=device) + s // 4
        w = hash_torch(seed, S_KV, idx).view(torch.int16)[: e - s]
        out[s:e] = w & -16385  # 0xBFFF as int16
    return out.view(dtype).view(*shape)
