"""Thin ctypes binding of libspecdec.so (include/specdec.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels behind
the C ABI.  Functions keep the C names, take torch CUDA tensors (or None for nullable
pointers) and launch on the current torch stream unless `stream` is given.  A missing
library raises immediately -- there is no fallback of any kind.
"""
from __future__ import annotations

import ctypes
import os

import torch

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libspecdec.so")
_lib = None

OK, ERR_ARG, ERR_SHAPE, ERR_DTYPE, ERR_CAPACITY, ERR_CUDA = 0, -1, -2, -3, -4, -5
ST_NAN, ST_CAPACITY, ST_KEPT, ST_BOUND = 1, 2, 4, 8
ZERO_PADS = 1
OVERLAP_PREV = 2
DYNAMIC = 4
SEGMENTED = 8
DYNAMIC_FORCE = 16
DTYPE = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2}

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U32 = ctypes.c_uint32
_INT = ctypes.c_int

_SIGS = {
    "specdec_version": ([], _INT),
    "specdec_last_cuda_error": ([], ctypes.c_char_p),
    "specdec_verify_workspace_size": ([_I64, _I64], ctypes.c_size_t),
    "specdec_verify_kernels": ([_INT], _INT),
    "specdec_verify": ([_P, _INT, _I64, _I64, _I64, _I64, _P, _P, _P, _I64, _I64, _P, _P, _P,
                        _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P,
                        ctypes.c_size_t, _P], _INT),
    "specdec_batch_init": ([_P, _I64, _P, _P, _P, _P, _I32, _P, _P], _INT),
    "specdec_rebuild_pos_mask": ([_P, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P,
                                  _P, _P, _P, _P, _I64, _P, _P, _I64, _P, _P], _INT),
    "specdec_realign_workspace_size": ([_INT, _I64, _I64, _I64, _I64, _I64], ctypes.c_size_t),
    "specdec_realign_kv": ([_P, _P, _INT, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64,
                            _I64, _I64, _I64, _P, _I32, _P, _I32, _P, _I32, _I32, _P, _P, _U32, _P,
                            ctypes.c_size_t, _P, _P, _P], _INT),
    "specdec_pool_group": ([_P, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P,
                            _P, _P, _P, _P, _P, _P], _INT),
    "specdec_pool_group_deferred": ([_P, _P, _P, _I32, _I32, _I32, _I32, _P, _I32, _P, _P, _P, _P, _P, _P,
                                     _P, _P, _P, _P, _P, _P, _P, _P, _P, _P], _INT),
    "specdec_pool_getbatch": ([_P, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P,
                               _P, _P, _P, _P, _P, _P], _INT),
    "specdec_pool_writeback": ([_P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P,
                                _I64, _P, _P], _INT),
    "specdec_pool_epoch": ([_P, _P, _P, _I32, _P, _P, _P, _P, _P], _INT),
    "specdec_eqspec_round": ([_P, _INT, _P, _P, _P], _INT),
    "specdec_pool_alg3": ([_P, _I32, _P, _P, _P], _INT),
    "specdec_pool_alg3_graph": ([_P, _I32, _P, _P, _I32, _P], _INT),
    "specdec_graph_launch": ([_P, _P], _INT),
    "specdec_graph_destroy": ([_P], _INT),
    "specdec_eqspec_round_host": ([_P, _P, _INT, _INT, _P, _P, _P, _P], _INT),
    "specdec_pool_verify_group": ([_I32, _P, _P, _P, _P, _INT, _I64, _I64, _I64, _P, _P, _P, _I64, _I64,
                                   _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _I64, _P, _P, ctypes.c_size_t,
                                   _P], _INT),
    "specdec_pool_verify": ([_P, _INT, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _I64, _P, _P, _P,
                             _P, _P, _P, _P, _P, _I64, _P, _I64, _P, _P, ctypes.c_size_t, _P], _INT),
}
EXPORTS = tuple(_SIGS)


class PoolDesc(ctypes.Structure):
    """Mirror of `specdec_pool_desc` (include/specdec.h), field for field."""
    _fields_ = [
        ("len", _P), ("gen", _P), ("active", _P), ("order", _P), ("N", _I32),
        ("tokens", _P), ("cap_tok", _I64), ("out_buf", _P), ("max_new", _I64),
        ("kv", _P), ("staging", _P), ("kv_dtype", _INT),
        ("n_planes", _I64), ("H", _I64), ("D", _I64), ("cap", _I64),
        ("window", _P), ("window_size", _P), ("batch_of", _P), ("slot_of", _P), ("members", _P),
        ("mlen", _P), ("mpad", _P), ("mactive", _P), ("bsize", _P), ("bkind", _P), ("blen", _P),
        ("n_batches", _P), ("counters", _P),
        ("accept", _P), ("bonus", _P), ("emit", _P), ("finished", _P), ("n_new", _P),
        ("pad_new", _P), ("kept", _P), ("plan_L", _P),
        ("ws", _P), ("ws_bytes", ctypes.c_size_t), ("status", _P), ("moved", _P),
        ("host_header", _P),
        ("W", _I32), ("B", _I32), ("min_group", _I32),
        ("k", _I64), ("V", _I64), ("logit_stride", _I64), ("eos_id", _I64), ("pad_id", _I64),
        ("logit_dtype", _INT),
        ("logits_ring", _P), ("draft_ring", _P), ("ring_n", _I32), ("ring_pos", _P),
        ("dense_consumer", _I32),
        ("n_staging", _I32), ("staging_ring", _P), ("copy_stream", _P), ("events", _P),
        ("cur_staging", _P), ("accept_ring", _P),
        ("est_gather_GBps", ctypes.c_double), ("est_verify_us", ctypes.c_double),
        ("gather_ws", _P),
        ("verify_group", _I32), ("host_launches", _P),
        ("scatter_stream", _P), ("scatter_events", _P),
        ("wait", _P), ("patience", _I32),
        ("pipeline", _I32), ("fb_epoch", _P), ("plan_epoch", _P), ("ws2", _P), ("ws2_bytes", ctypes.c_size_t),
        ("bonus2", _P), ("emit2", _P), ("finished2", _P), ("pipe_events", _P), ("pipe_host", _P),
    ]


_P2 = _P * 2


class RoundDesc(ctypes.Structure):
    """Mirror of `specdec_round_desc` (include/specdec.h), field for field."""
    _fields_ = [
        ("B", _I64), ("k", _I64), ("V", _I64), ("logit_stride", _I64), ("logit_dtype", _INT),
        ("eos_id", _I64), ("pad_id", _I64),
        ("n", _P2), ("pad", _P2), ("tokens", _P2), ("cap_tok", _I64),
        ("mask", _P), ("pos", _P), ("mp_stride", _I64),
        ("active", _P), ("budget", _P), ("gen", _P), ("out_buf", _P), ("max_new", _I64),
        ("accept", _P2), ("emit", _P2), ("bonus", _P2), ("finished", _P2),
        ("pred", _P), ("kept", _P), ("plan_L", _P), ("kept_draft", _P),
        ("ws", _P), ("ws_bytes", ctypes.c_size_t), ("status", _P), ("moved", _P),
        ("kv", _P2), ("kv_dtype", _INT),
        ("n_planes", _I64), ("H", _I64), ("D", _I64), ("cap_kv", _I64),
        ("s_plane", _I64), ("s_row", _I64), ("s_head", _I64),
        ("dkv", _P2), ("d_planes", _I64), ("d_H", _I64), ("d_D", _I64),
        ("d_s_plane", _I64), ("d_s_row", _I64), ("d_s_head", _I64),
        ("realign_flags", _U32), ("realign_ws", _P), ("realign_ws_bytes", ctypes.c_size_t),
        ("anchor", _P), ("phys_old", _P), ("phys_new", _P),
    ]


HOST_SLOTS = 4
MAX_VERIFY_GROUP = 64   # SPECDEC_MAX_VERIFY_GROUP (include/specdec.h)
_PS = _P * HOST_SLOTS


class HostIO(ctypes.Structure):
    """Mirror of `specdec_host_io` (include/specdec.h)."""
    _fields_ = [("n_slots", _I32), ("d_logits", _PS), ("d_draft", _PS), ("copy_stream", _P),
                ("d2h_stream", _P), ("ev_ready", _PS), ("ev_done", _PS), ("ev_fetched", _P2),
                ("inputs_packed", _I32)]


def specdec_eqspec_round(desc: RoundDesc, parity, logits, draft, stream=None):
    """One EqSpec round (K1 -> K3 -> K2) in the native driver."""
    _check_logits(logits)
    _check(load().specdec_eqspec_round(ctypes.byref(desc), parity, _ptr(logits), _ptr(draft),
                                       _stream(stream)), "specdec_eqspec_round")


_PINNED_OK: set = set()   # (data_ptr, nbytes) of host buffers already checked to be pinned


def specdec_eqspec_round_host(desc: RoundDesc, io: HostIO, parity, slot, h_logits, h_draft,
                              h_emit=None, stream=None):
    """One EqSpec round from pinned HOST logits / drafts (H2D + round + D2H of emit)."""
    ptrs = []
    for t in (h_logits, h_draft, h_emit):
        if t is None:
            ptrs.append(None)
            continue
        key = (t.data_ptr(), t.numel() * t.element_size())
        if key not in _PINNED_OK:    # the pinned check costs a driver query: once per buffer
            if t.is_cuda or not t.is_pinned():
                raise SpecdecError("pinned host tensor expected")
            _PINNED_OK.add(key)
        ptrs.append(key[0])
    # one copy only when the drafts follow the logits inside one allocation (same storage)
    io.inputs_packed = int(h_logits.untyped_storage().data_ptr() == h_draft.untyped_storage().data_ptr()
                           and ptrs[1] == ptrs[0] + h_logits.numel() * h_logits.element_size())
    _check(load().specdec_eqspec_round_host(ctypes.byref(desc), ctypes.byref(io), parity, slot,
                                            ptrs[0], ptrs[1], ptrs[2], _stream(stream)),
           "specdec_eqspec_round_host")


# specdec_forward_fn: (ctx, batch, same_length, width, const void **logits, const int64_t **draft)
FORWARD_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                              ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p))


def specdec_pool_epoch(desc: PoolDesc, max_batches=0, stream=None, forward=None):
    """Native epoch executor; returns (batches run, same-length run, members same, members fallback).
    `forward`: an optional FORWARD_FN (the model's verify forward), else the descriptor's ring."""
    out = [ctypes.c_int32(0) for _ in range(4)]
    _check(load().specdec_pool_epoch(ctypes.byref(desc), forward, None, max_batches,
                                     *[ctypes.byref(o) for o in out], _stream(stream)),
           "specdec_pool_epoch")
    return tuple(o.value for o in out)


def specdec_pool_alg3_graph(desc: PoolDesc, iterations, scratch, exec_counters=None, conditional=False):
    """The Alg. 3 loop of `iterations` iterations as one CUDA graph (conditional: KV moves in
    IF nodes); returns the cudaGraphExec_t handle (an int) for specdec_graph_launch / _destroy."""
    out = ctypes.c_void_p(0)
    _check(load().specdec_pool_alg3_graph(ctypes.byref(desc), iterations, _ptr(scratch), _ptr(exec_counters),
                                          int(conditional), ctypes.byref(out)), "specdec_pool_alg3_graph")
    return out.value


def specdec_graph_launch(graph_exec, stream=None):
    _check(load().specdec_graph_launch(graph_exec, _stream(stream)), "specdec_graph_launch")


def specdec_graph_destroy(graph_exec):
    _check(load().specdec_graph_destroy(graph_exec), "specdec_graph_destroy")


def specdec_pool_alg3(desc: PoolDesc, iterations, scratch, exec_counters=None, stream=None):
    """`iterations` Alg. 3 iterations (plan, batch 0, re-plan) with no host synchronisation."""
    _check(load().specdec_pool_alg3(ctypes.byref(desc), iterations, _ptr(scratch), _ptr(exec_counters),
                                    _stream(stream)), "specdec_pool_alg3")


class SpecdecError(RuntimeError):
    pass


def lib_path() -> str:
    return _LIB_PATH


def load(path: str | None = None):
    """Load libspecdec.so (once).  Raises if it is missing: the product has no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or _LIB_PATH
    if not os.path.exists(p):
        raise SpecdecError(f"{p} not built: run `python -m paper_2510_22876_b200.build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(p)
    for name, (args, res) in _SIGS.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise SpecdecError("device pointer expected (CUDA tensor)")
    return t.data_ptr()


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check(rc: int, name: str):
    if rc != OK:
        msg = {ERR_ARG: "ERR_ARG", ERR_SHAPE: "ERR_SHAPE", ERR_DTYPE: "ERR_DTYPE",
               ERR_CAPACITY: "ERR_CAPACITY", ERR_CUDA: "ERR_CUDA"}.get(rc, str(rc))
        if rc == ERR_CUDA:
            msg += ": " + load().specdec_last_cuda_error().decode()
        raise SpecdecError(f"{name} -> {msg}")


def version() -> int:
    return load().specdec_version()


def specdec_verify_kernels(pool: bool = False) -> int:
    """Kernels one specdec_verify (or specdec_pool_verify) call launches."""
    return load().specdec_verify_kernels(1 if pool else 0)


def specdec_verify_workspace_size(B: int, k: int) -> int:
    return load().specdec_verify_workspace_size(B, k)


def _check_logits(logits):
    """The kernels read row (i, j) at (i * (k+1) + j) * row_stride with unit element stride:
    a view whose batch stride is not (k+1) * row_stride (e.g. logits[:, -(k+1):] of a
    [B, T, V] forward output) would be read wrongly, so it is refused."""
    if logits.dim() != 3 or logits.stride(2) != 1 or logits.stride(0) != logits.shape[1] * logits.stride(1):
        raise SpecdecError(f"logits must be [B, k+1, row_stride] with batch stride (k+1)*row_stride and "
                           f"unit last stride (got shape {tuple(logits.shape)}, strides {logits.stride()}); "
                           "pass .contiguous()")


def specdec_verify(logits, draft, n, active, accept, bonus, emit, finished, plan_L, n_new,
                   pad_new, kept, ws, *, V=None, eos_id=-1, pad_id=0, budget=None, pred=None,
                   kept_draft=None, anchor=None, anchor_cap=0, phys_old=None, phys_new=None,
                   status=None, stream=None):
    """logits [B, k+1, row_stride] (fp32/fp16/bf16); see include/specdec.h."""
    _check_logits(logits)
    B, K1, rs = logits.shape
    _check(load().specdec_verify(
        _ptr(logits), DTYPE[logits.dtype], B, K1 - 1, rs if V is None else V, logits.stride(1),
        _ptr(draft), _ptr(n), _ptr(active), eos_id, pad_id, _ptr(budget), _ptr(accept),
        _ptr(bonus), _ptr(emit), _ptr(finished), _ptr(pred), _ptr(plan_L), _ptr(n_new),
        _ptr(pad_new), _ptr(kept), _ptr(kept_draft), _ptr(anchor), anchor_cap, _ptr(phys_old),
        _ptr(phys_new), _ptr(status), _ptr(ws), ws.numel() * ws.element_size(),
        _stream(stream)), "specdec_verify")


def specdec_batch_init(n, pad, *, L=None, active=None, budget=None, max_new=0, status=None,
                       stream=None):
    _check(load().specdec_batch_init(_ptr(n), n.shape[0], _ptr(pad), _ptr(L), _ptr(active), _ptr(budget),
                                     max_new, _ptr(status), _stream(stream)), "specdec_batch_init")


def specdec_rebuild_pos_mask(tokens_in, tokens_out, k, n_old, pad_old, draft, accept, bonus,
                             emit, finished, plan_L, pad_new, mask, pos, *, pad_id=0,
                             out_buf=None, gen=None, status=None, stream=None):
    B, cap_tok = tokens_in.shape
    _check(load().specdec_rebuild_pos_mask(
        _ptr(tokens_in), _ptr(tokens_out), B, cap_tok, k, pad_id, _ptr(n_old), _ptr(pad_old),
        _ptr(draft), _ptr(accept), _ptr(bonus), _ptr(emit), _ptr(finished), _ptr(plan_L),
        _ptr(pad_new), _ptr(mask), _ptr(pos), mask.stride(0), _ptr(out_buf), _ptr(gen),
        0 if out_buf is None else out_buf.shape[1], _ptr(status), _stream(stream)),
        "specdec_rebuild_pos_mask")


def specdec_realign_workspace_size(dtype, n_planes, n_rows, H, D, cap) -> int:
    return load().specdec_realign_workspace_size(DTYPE[dtype], n_planes, n_rows, H, D, cap)


def specdec_realign_kv(kv_src, kv_dst, count, *, n_planes, n_rows, H, D, src_strides,
                       dst_strides, cap_src, cap_dst, src_col=None, src_col_add=0,
                       dst_col=None, dst_col_add=0, count_add=0, count_bound=0,
                       src_row_map=None, dst_row_map=None, flags=0, ws=None, moved_bytes=None,
                       status=None, stream=None):
    """src/dst_strides = (s_plane, s_row, s_head) in elements; positions are D apart.
    ws: optional workspace tensor of specdec_realign_workspace_size bytes (segmentation).
    count_bound: upper bound on count + count_add (0 = none)."""
    _check(load().specdec_realign_kv(
        _ptr(kv_src), _ptr(kv_dst), DTYPE[kv_src.dtype], n_planes, n_rows, H, D,
        src_strides[0], src_strides[1], src_strides[2], cap_src, dst_strides[0],
        dst_strides[1], dst_strides[2], cap_dst, _ptr(src_col), src_col_add, _ptr(dst_col),
        dst_col_add, _ptr(count), count_add, count_bound, _ptr(src_row_map), _ptr(dst_row_map), flags,
        _ptr(ws), 0 if ws is None else ws.numel() * ws.element_size(),
        _ptr(moved_bytes), _ptr(status), _stream(stream)), "specdec_realign_kv")


def specdec_pool_verify(logits, draft, members, mlen, mactive, accept, bonus, emit, finished,
                        pool_len, pool_gen, pool_active, ws, *, V=None, eos_id=-1, pad_id=0,
                        max_new, pool_tokens=None, out_buf=None, status=None, stream=None):
    """K1 + the pool write-back in one launch (include/specdec.h)."""
    _check_logits(logits)
    B, K1, _ = logits.shape
    _check(load().specdec_pool_verify(
        _ptr(logits), DTYPE[logits.dtype], B, K1 - 1, V or logits.shape[2], logits.stride(1),
        _ptr(draft), _ptr(members), _ptr(mlen), _ptr(mactive), eos_id, pad_id, _ptr(accept),
        _ptr(bonus), _ptr(emit), _ptr(finished), _ptr(pool_len), _ptr(pool_gen),
        _ptr(pool_active), _ptr(pool_tokens), 0 if pool_tokens is None else pool_tokens.shape[1],
        _ptr(out_buf), max_new, _ptr(status), _ptr(ws), ws.numel() * ws.element_size(),
        _stream(stream)), "specdec_pool_verify")


def specdec_pool_verify_group(logits_list, draft_list, offsets, rows, members, mlen, mactive, accept, bonus,
                              emit, finished, pool_len, pool_gen, pool_active, ws, *, V=None, eos_id=-1,
                              pad_id=0, max_new, pool_tokens=None, out_buf=None, status=None, stream=None):
    """specdec_pool_verify over len(logits_list) batches in one launch (include/specdec.h):
    batch g's logits [rows[g]][k+1][V'] and drafts, its member rows at offsets[g] of the
    plan arrays; per-row outputs flat over sum(rows)."""
    G = len(logits_list)
    for lg, r in zip(logits_list, rows):
        _check_logits(lg)
        if lg.shape[0] < r or lg.stride(1) != logits_list[0].stride(1) or lg.dtype != logits_list[0].dtype:
            raise ValueError("grouped logits: rows, row stride and dtype must agree")
    K1 = logits_list[0].shape[1]
    arr = lambda ts: (ctypes.c_void_p * G)(*[t.data_ptr() for t in ts])
    i32 = lambda xs: (ctypes.c_int32 * G)(*[int(x) for x in xs])
    _check(load().specdec_pool_verify_group(
        G, arr(logits_list), arr(draft_list), i32(offsets), i32(rows), DTYPE[logits_list[0].dtype], K1 - 1,
        V or logits_list[0].shape[2], logits_list[0].stride(1), _ptr(members), _ptr(mlen), _ptr(mactive),
        eos_id, pad_id, _ptr(accept), _ptr(bonus), _ptr(emit), _ptr(finished), _ptr(pool_len), _ptr(pool_gen),
        _ptr(pool_active), _ptr(pool_tokens), 0 if pool_tokens is None else pool_tokens.shape[1],
        _ptr(out_buf), max_new, _ptr(status), _ptr(ws), ws.numel() * ws.element_size(),
        _stream(stream)), "specdec_pool_verify_group")


def specdec_pool_group(length, active, order, W, B, min_group, window, window_size, batch_of,
                       slot_of, members, mlen, mpad, mactive, bsize, bkind, blen, n_batches,
                       counters, *, stream=None):
    _check(load().specdec_pool_group(
        _ptr(length), _ptr(active), _ptr(order), length.numel(), W, B, min_group, _ptr(window),
        _ptr(window_size), _ptr(batch_of), _ptr(slot_of), _ptr(members), _ptr(mlen), _ptr(mpad),
        _ptr(mactive), _ptr(bsize), _ptr(bkind), _ptr(blen), _ptr(n_batches), _ptr(counters),
        _stream(stream)), "specdec_pool_group")


def specdec_pool_group_deferred(length, active, order, W, B, min_group, wait, patience, window,
                                window_size, batch_of, slot_of, members, mlen, mpad, mactive, bsize,
                                bkind, blen, n_batches, counters, *, fb_epoch=None, epoch=None, stream=None):
    """The epoch plan with deferred fallback (R27) and, with fb_epoch / epoch, pipelined
    fallback (R28) (include/specdec.h); `wait` (and fb_epoch / epoch) are updated."""
    _check(load().specdec_pool_group_deferred(
        _ptr(length), _ptr(active), _ptr(order), length.numel(), W, B, min_group, _ptr(wait), patience,
        _ptr(fb_epoch), _ptr(epoch), _ptr(window), _ptr(window_size), _ptr(batch_of), _ptr(slot_of), _ptr(members), _ptr(mlen),
        _ptr(mpad), _ptr(mactive), _ptr(bsize), _ptr(bkind), _ptr(blen), _ptr(n_batches),
        _ptr(counters), _stream(stream)), "specdec_pool_group_deferred")


def specdec_pool_getbatch(length, active, order, W, B, min_group, window, window_size, batch_of,
                          slot_of, members, mlen, mpad, mactive, bsize, bkind, blen, n_batches,
                          counters, *, stream=None):
    """Alg. 3's GetBatch: batch 0 of the window plan only (include/specdec.h)."""
    _check(load().specdec_pool_getbatch(
        _ptr(length), _ptr(active), _ptr(order), length.numel(), W, B, min_group, _ptr(window),
        _ptr(window_size), _ptr(batch_of), _ptr(slot_of), _ptr(members), _ptr(mlen), _ptr(mpad),
        _ptr(mactive), _ptr(bsize), _ptr(bkind), _ptr(blen), _ptr(n_batches), _ptr(counters),
        _stream(stream)), "specdec_pool_getbatch")


def specdec_pool_writeback(members, k, draft, accept, bonus, emit, finished, pool_len,
                           pool_gen, pool_active, *, max_new, pool_tokens=None, out_buf=None,
                           status=None, stream=None):
    _check(load().specdec_pool_writeback(
        _ptr(members), members.numel(), k, _ptr(draft), _ptr(accept), _ptr(bonus), _ptr(emit),
        _ptr(finished), _ptr(pool_len), _ptr(pool_gen), _ptr(pool_active), _ptr(pool_tokens),
        0 if pool_tokens is None else pool_tokens.shape[1], _ptr(out_buf), max_new,
        _ptr(status), _stream(stream)), "specdec_pool_writeback")
