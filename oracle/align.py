"""Oracle: unpad-append-repad and KV realignment (Alg. 2 Phase 3, PAPER.md:348-356;
§3.1 invariants PAPER.md:444-447; Fig. 4).

Test infrastructure only (see oracle/__init__.py).

Conventions:
  * a batch row holds n_i content tokens right-aligned at width L (left pads p_i = L - n_i);
    the last content token is "pending": it has no KV entry yet;
  * after the verify forward the KV width is L + k and row i's valid KV is [p_i, L + a_i);
  * after repad row i's kept_i = n_i + a_i entries live at [p'_i, p'_i + kept_i) = [p'_i, L' - 1).
Readings: R7 (pos = 0 on pads), R8 (pad KV is don't-care unless ZERO_PADS), R9 (dummy rows).
"""
from __future__ import annotations

import numpy as np


# ----------------------------------------------------------------------------- tokens
def build_batch(seqs, cap: int, pad_id: int = 0):
    """Batch left padding (Alg. 2 line 1): content right-aligned at
    L = max length; returns tokens [B, cap], pad [B], L."""
    lens = np.array([len(s) for s in seqs], np.int32)
    L = int(lens.max())
    tok = np.full((len(seqs), cap), pad_id, np.int64)
    for i, s in enumerate(seqs):
        tok[i, L - len(s):L] = s
    return tok, (L - lens).astype(np.int32), L


def unpad(tokens, pad, L):
    """S[i] <- Unpad(S[i]): the content columns [p_i, L)."""
    return [list(map(int, tokens[i, pad[i]:L])) for i in range(len(pad))]


def append_accepted(rows, E_rows):
    """S[i] <- S[i] (+) A[i] (+) B[i] -- E already holds A ++ [B], EOS-cut."""
    return [r + list(e) for r, e in zip(rows, E_rows)]


def mask_pos_row(pad_new: int, width: int):
    """Padding-agnostic positions and masks: mask = 1 exactly on content
    columns c >= p'; pos = c - p' there, 0 on pads (R7)."""
    c = np.arange(width)
    mask = (c >= pad_new).astype(np.int64)
    pos = np.where(c >= pad_new, c - pad_new, 0).astype(np.int64)
    return mask, pos


def repad_tokens(tokens, cap, k, pad_old, L_old, vres, pad_id=0):
    """Tokens' / mask / pos after Phase 3.

    vres is batch_verify()'s result (plan included).  Returns (tokens' [B, cap],
    mask [B, L'+k], pos [B, L'+k]); only columns [0, L') of tokens' are defined."""
    B = len(pad_old)
    L_new = vres["L_new"]
    out = np.full((B, cap), pad_id, np.int64)
    mask = np.zeros((B, L_new + k), np.int64)
    pos = np.zeros((B, L_new + k), np.int64)
    if L_new == 0:
        return out, mask, pos
    rows = unpad(tokens, pad_old, L_old)
    rows = append_accepted(rows, vres["E"])
    for i in range(B):
        if vres["finished"][i]:
            content = [pad_id]                         # R9 dummy row
        else:
            content = rows[i]
        assert len(content) == vres["n_new"][i]
        p = int(vres["pad_new"][i])
        out[i, p:L_new] = content
        mask[i], pos[i] = mask_pos_row(p, L_new + k)
    return out, mask, pos


# ----------------------------------------------------------------------------- KV
def realign_kv(kv, pad_old, pad_new, kept):
    """KVCache <- Realign(KVCache, offset) as a fresh rectangle
    (SPEC.md:176 style): KV'[.., i, h, p'_i + c, :] = KV[.., i, h, p_i + c, :] for
    c < kept_i.  kv: [planes, B, H, cap, D] (any dtype; bytes are copied).
    Returns (KV', defined [B, cap] bool): the positions whose value is specified."""
    out = np.zeros_like(kv)
    B, cap = kv.shape[1], kv.shape[3]
    defined = np.zeros((B, cap), bool)
    for i in range(B):
        c = int(kept[i])
        if c <= 0:
            continue
        po, pn = int(pad_old[i]), int(pad_new[i])
        out[:, i, :, pn:pn + c, :] = kv[:, i, :, po:po + c, :]
        defined[i, pn:pn + c] = True
    return out, defined


def zero_pad_region(pad_old, pad_new, kept):
    """ZERO_PADS flag: the old content columns that become pads, [p_i, p'_i) when
    p'_i > p_i (rows with kept_i > 0).  Returns a list of (row, lo, hi)."""
    res = []
    for i in range(len(pad_old)):
        if kept[i] > 0 and pad_new[i] > pad_old[i]:
            res.append((i, int(pad_old[i]), int(pad_new[i])))
    return res


def copy_rows(src, dst, count, src_col=None, dst_col=None, src_row=None, dst_row=None):
    """Generic row-mapped KV move (a3/a5): for every batch row i with count_i > 0 and
    mapped rows >= 0: dst[dst_row_i][:, :, dst_col_i + c] = src[src_row_i][:, :, src_col_i + c]
    for c < count_i.  src/dst are logical [rows][planes][H][cap][D] views.
    dst is modified in place; no other byte of dst changes.  The definition is
    out-of-place: every source is read before it is overwritten.  Without row maps row i
    writes only row i, so reading each row's source block before writing it is enough
    (also when dst is src: the in-place realign); with row maps and aliasing buffers the
    whole source is copied first."""
    if (src_row is not None or dst_row is not None) and np.shares_memory(src, dst):
        src = np.array(src, copy=True)
    for i in range(len(count)):
        c = int(count[i])
        sr = i if src_row is None else int(src_row[i])
        dr = i if dst_row is None else int(dst_row[i])
        if c <= 0 or sr < 0 or dr < 0:
            continue
        sc = 0 if src_col is None else int(src_col[i])
        dc = 0 if dst_col is None else int(dst_col[i])
        block = np.array(src[sr, :, :, sc:sc + c, :], copy=True)
        dst[dr, :, :, dc:dc + c, :] = block
    return dst


def realign_kv_inplace(kv, pad_old, pad_new, kept):
    """Realign in the in-place form K2's contract states (specdec.h): for
    every row i, plane and head, KV[.., i, h, p'_i + c, :] <- KV[.., i, h, p_i + c, :] for
    c < kept_i (the row's source read before it is written), and NO other byte changes --
    so the whole buffer, stale columns included, is defined and comparable.
    kv [planes, B, H, cap, D] is modified in place and returned."""
    rows = np.moveaxis(kv, 1, 0)                 # view [B, planes, H, cap, D]
    copy_rows(rows, rows, kept, src_col=pad_old, dst_col=pad_new)
    return kv


def anchor_plan(pad_old, pad_new, kept, finished, accept, L_old, L_new, base, cap_phys, k):
    """f3 ("anchored-origin realign"; PAPER.md:746 names KV locality as future
    work).  The logical rectangle -- tokens, masks, positions, and the KV of logical
    column c -- is exactly Alg. 2's; only its PHYSICAL origin `base` in the KV buffer may
    move: logical column c lives at physical base + c.  Per round the new origin
    base' = base + d is chosen among d = 0 and the shifts that leave one accept class in
    place, d = (a + 1) - (L' - L), minimising the KV rows that must move (ties: d = 0,
    then larger d), subject to 0 <= base' and base' + L' + k <= cap_phys.  If no candidate
    is feasible (the origin sits too high for the grown width), the feasible shift closest
    to 0 is taken (every kept row moves; none exists only if L' + k > cap_phys).
    Returns (base', physical old columns, physical new columns)."""
    pad_old = np.asarray(pad_old, np.int64)
    pad_new = np.asarray(pad_new, np.int64)
    kept = np.asarray(kept, np.int64)
    alive = np.asarray(finished) == 0
    best_d, best_cost = 0, None
    if L_new > 0:
        cands = sorted({0} | {(a + 1) - (L_new - L_old) for a in range(k + 1)},
                       key=lambda d: (d != 0, -d))
        for d in cands:
            if base + d < 0 or base + d + L_new + k > cap_phys:
                continue
            cost = int(sum(kept[i] for i in range(len(kept))
                           if alive[i] and kept[i] > 0 and d + pad_new[i] != pad_old[i]))
            if best_cost is None or cost < best_cost:
                best_d, best_cost = d, cost
        if best_cost is None:
            lo, hi = -base, cap_phys - L_new - k - base
            if lo <= hi:
                best_d = min(max(0, lo), hi)
    base_new = base + best_d
    return base_new, (base + pad_old).astype(np.int32), (base_new + pad_new).astype(np.int32)


def moved_bytes(pad_old, pad_new, kept, bpt):
    """Algorithmic bytes of an in-place realign: 2 * kept_i * bpt over
    rows whose padding changed (rows with Delta_i = 0 move nothing)."""
    tot = 0
    for i in range(len(kept)):
        if kept[i] > 0 and pad_new[i] != pad_old[i]:
            tot += 2 * int(kept[i]) * bpt
    return tot
