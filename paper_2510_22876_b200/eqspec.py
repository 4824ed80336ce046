"""EqSpec batch state and one verification round on device (Alg. 2).

A round is three C-ABI calls on one stream with no host synchronisation:

    specdec_verify            K1  Alg. 1 BatchVerify + the BatchRepad plan (L', p', kept)
    specdec_rebuild_pos_mask  K3  unpad-append-repad of the tokens, positions, masks
    specdec_realign_kv        K2  Realign(KVCache, offset), in place

The small per-row state (n, p, tokens) is double-buffered: round r reads slot r&1 and
writes slot 1-(r&1), which round r+1 reads (the token rebuild is then a pure gather,
spread over many CTAs).  The KV cache -- the only large state -- is realigned in place.
`active` and the remaining `budget` are updated in place by K1.  Everything is
capacity-sized, so the data-dependent width L' never leaves the device,
and a round can be captured once per (parity, input buffer) as a CUDA graph.

Options: `draft=(layers, H, D)` adds the draft model's own KV cache,
realigned with kept_draft (f1); `anchor_slack=S` keeps the KV in a physical buffer of
cap + S columns whose logical origin K1 moves to minimise the rows that must move (f3);
`kv_mode="pingpong"` keeps two KV buffers and realigns out of place from the current into
the other one every round -- rows with Delta = 0 are copied too (the SURVEY §8d ping-pong
cell, the analog of the paper's fresh-tensor realignment).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _abi

TORCH_DT = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}


def pack_inputs_like(logits, draft, device, pin=False):
    """One buffer holding a logits tensor (shape / dtype / strides of `logits`, contiguous)
    followed by a drafts tensor like `draft`: returns the two views.  On the host
    (device='cpu', pin=True) it is pinned memory; specdec_eqspec_round_host then copies a
    step's inputs with one DMA."""
    lg_bytes = logits.numel() * logits.element_size()
    dr_bytes = draft.numel() * draft.element_size()
    buf = torch.empty(lg_bytes + dr_bytes, dtype=torch.uint8, device=device)
    if pin:
        buf = buf.pin_memory()
    lg = buf[:lg_bytes].view(logits.dtype).view(logits.shape)
    dr = buf[lg_bytes:].view(draft.dtype).view(draft.shape)
    return lg, dr


def pack_host_inputs(logits, draft):
    """Pinned host copies of (logits, draft) packed into one buffer (see pack_inputs_like)."""
    lg, dr = pack_inputs_like(logits, draft, "cpu", pin=True)
    lg.copy_(logits)
    dr.copy_(draft)
    return lg, dr


class EqSpecBatch:
    def __init__(self, B, k, cap, layers, H, D, kv_dtype="bf16", device="cuda", max_new=0,
                 eos_id=-1, pad_id=0, with_pred=False, draft=None, anchor_slack=0,
                 kv_mode="inplace"):
        if kv_mode not in ("inplace", "pingpong"):
            raise ValueError(f"kv_mode {kv_mode!r}")
        if kv_mode == "pingpong" and anchor_slack:
            raise ValueError("the anchored origin (f3) is an in-place scheme")
        self.kv_mode = kv_mode
        nbuf = 2 if kv_mode == "pingpong" else 1
        self.cur = 0  # state parity: round r reads slot cur and writes slot 1 - cur
        dev = torch.device(device)
        i32, i64, u8 = torch.int32, torch.int64, torch.uint8
        self.B, self.k, self.cap, self.layers, self.H, self.D = B, k, cap, layers, H, D
        self.n_planes = 2 * layers
        self.eos_id, self.pad_id, self.max_new = eos_id, pad_id, max_new
        self.device = dev
        self.tok = torch.full((2, B, cap), pad_id, dtype=i64, device=dev)
        self.mask = torch.zeros((B, cap + k), dtype=i64, device=dev)
        self.pos = torch.zeros((B, cap + k), dtype=i64, device=dev)
        self.n = torch.zeros((2, B), dtype=i32, device=dev)
        self.pad = torch.zeros((2, B), dtype=i32, device=dev)
        self.active = torch.ones(B, dtype=u8, device=dev)
        self.budget = torch.full((B,), max_new, dtype=i32, device=dev) if max_new else None
        self.gen = torch.zeros(B, dtype=i32, device=dev)
        self.out_buf = torch.zeros((B, max_new), dtype=i64, device=dev) if max_new else None
        # per-round results, one set per state parity: a round's results stay readable
        # (e.g. by an asynchronous D2H on another stream) while the next round runs
        self._accept = torch.zeros((2, B), dtype=i32, device=dev)
        self._bonus = torch.zeros((2, B), dtype=i64, device=dev)
        self._emit = torch.zeros((2, B), dtype=i32, device=dev)
        self._finished = torch.zeros((2, B), dtype=u8, device=dev)
        self._last = 0  # parity of the last launched round
        self.kept = torch.zeros(B, dtype=i32, device=dev)
        self.plan_L = torch.zeros(1, dtype=i32, device=dev)
        self.pred = torch.zeros((B, k + 1), dtype=i64, device=dev) if with_pred else None
        self.status = torch.zeros(1, dtype=i32, device=dev)
        self.moved = torch.zeros(1, dtype=i64, device=dev)
        ws = _abi.specdec_verify_workspace_size(B, k)
        self.ws = torch.zeros((ws + 7) // 8, dtype=i64, device=dev)
        # f3: physical KV columns = logical capacity + slack for the moving origin
        self.anchor_slack = anchor_slack
        self.cap_phys = cap + anchor_slack
        self.anchor = torch.full((1,), anchor_slack, dtype=i32, device=dev) if anchor_slack else None
        self.phys_old = torch.zeros(B, dtype=i32, device=dev) if anchor_slack else None
        self.phys_new = torch.zeros(B, dtype=i32, device=dev) if anchor_slack else None
        # KV buffers: one (in place) or two (ping-pong: the current one is buffer [cur])
        self._kvbuf = [torch.zeros((self.n_planes, B, H, self.cap_phys, D), dtype=TORCH_DT[kv_dtype], device=dev)
                       for _ in range(nbuf)]
        self._dkvbuf = None
        self.kept_draft = None
        if draft is not None:
            dl, dh, dd = draft
            self.d_dims = (2 * dl, dh, dd)
            self._dkvbuf = [torch.zeros((2 * dl, B, dh, self.cap_phys, dd), dtype=TORCH_DT[kv_dtype], device=dev)
                            for _ in range(nbuf)]
            self.kept_draft = torch.zeros(B, dtype=i32, device=dev)
        # K2 workspace: boundary-row slots that let any CTA stream any ~128 KB segment of a
        # slab in place (load balance when few rows move); shared by the target and draft calls
        sizes = [_abi.specdec_realign_workspace_size(self.kv.dtype, self.n_planes, B, H, D, self.cap_phys)]
        if self.dkv is not None:
            sizes.append(_abi.specdec_realign_workspace_size(self.dkv.dtype, *self.d_dims[:1], B,
                                                             *self.d_dims[1:], self.cap_phys))
        self.rws = torch.zeros(max(sizes), dtype=torch.uint8, device=dev)   # header zero (specdec.h)
        self.segment = bool(int(os.environ.get("SPECDEC_SEGMENT", "0")))  # measured: profiles/r01
        # K2 work tickets (SPECDEC_DYNAMIC) from rws's header: +1 % at Qwen3 B=8
        self.dynamic = bool(int(os.environ.get("SPECDEC_DYNAMIC", "1")))
        self.V = None
        self.zero_pads = False
        # K3 on a side stream under K2: a small win for direct launches, a loss inside a
        # CUDA graph (measured: profiles/r01/round_modes.txt), so off by default
        self.fork = False
        # K2 starts under K3 (SPECDEC_OVERLAP_PREV; serial launch order only)
        self.overlap = bool(int(os.environ.get("SPECDEC_OVERLAP", "1")))
        self._graphs = {}
        # launch the round through the native driver (specdec_eqspec_round: one C call for
        # K1 -> K3 -> K2; default) or as the three calls from Python (False); same kernels,
        # same order, same results
        self.native_round = True

    # ----------------------------------------------------------------- state I/O
    def load(self, tokens, lengths, kv=None):
        """tokens [B, cap] left-padded at width L = max(lengths); kv [planes, B, H, cap, D]
        (logical columns; placed at the origin when anchored)."""
        lengths = torch.as_tensor(np.asarray(lengths), dtype=torch.int32)
        self.cur = 0
        self.tok[0].copy_(torch.as_tensor(tokens))
        self.n[0].copy_(lengths)
        # Alg. 2 line 1, the batch left padding: pad = max n - n, every row
        # active, the budget full -- on the device
        _abi.specdec_batch_init(self.n[0], self.pad[0], active=self.active, budget=self.budget,
                                max_new=self.max_new or 0, status=self.status)
        self.gen.zero_()
        if self.kept_draft is not None:
            self.kept_draft.zero_()     # no draft KV yet: the drafter prefills in round 1
        if self.anchor is not None:
            self.anchor.fill_(self.anchor_slack)
        if kv is not None:
            self.kv_logical().copy_(kv)

    def base(self) -> int:
        """Physical column of logical column 0 (host read; 0 unless anchored)."""
        return int(self.anchor.item()) if self.anchor is not None else 0

    def kv_logical(self, kv=None):
        kv = self.kv if kv is None else kv
        b = self.base()
        return kv[:, :, :, b:b + self.cap]

    @property
    def tokens(self):
        return self.tok[self.cur]

    @property
    def n_cur(self):
        return self.n[self.cur]

    @property
    def pad_cur(self):
        return self.pad[self.cur]

    # results of the last launched round (its parity's set)
    @property
    def accept(self):
        return self._accept[self._last]

    @property
    def bonus(self):
        return self._bonus[self._last]

    @property
    def emit(self):
        return self._emit[self._last]

    @property
    def finished(self):
        return self._finished[self._last]

    # the current KV buffers (ping-pong: the one the next round reads)
    @property
    def kv(self):
        return self._kvbuf[self.cur % len(self._kvbuf)]

    @property
    def dkv(self):
        return None if self._dkvbuf is None else self._dkvbuf[self.cur % len(self._dkvbuf)]

    @property
    def kv_strides(self):
        s = self.kv.stride()
        return (s[0], s[1], s[2])

    # ----------------------------------------------------------------- the three calls
    def verify(self, logits, draft, stream=None):
        c, nx = self.cur, 1 - self.cur
        self._last = c
        _abi.specdec_verify(logits, draft, self.n[c], self.active, self.accept, self.bonus,
                            self.emit, self.finished, self.plan_L, self.n[nx], self.pad[nx],
                            self.kept, self.ws, V=self.V or logits.shape[2],
                            eos_id=self.eos_id, pad_id=self.pad_id, budget=self.budget,
                            pred=self.pred, kept_draft=self.kept_draft, anchor=self.anchor,
                            anchor_cap=self.cap_phys, phys_old=self.phys_old,
                            phys_new=self.phys_new, status=self.status, stream=stream)

    def repad(self, draft, stream=None):
        c, nx = self.cur, 1 - self.cur
        _abi.specdec_rebuild_pos_mask(self.tok[c], self.tok[nx], self.k, self.n[c], self.pad[c],
                                      draft, self.accept, self.bonus, self.emit, self.finished,
                                      self.plan_L, self.pad[nx], self.mask, self.pos,
                                      pad_id=self.pad_id, out_buf=self.out_buf,
                                      gen=self.gen if self.out_buf is not None else None,
                                      status=self.status, stream=stream)

    def _realign_one(self, bufs, count, dims, src, dst, stream, overlap=False):
        planes, H, D = dims
        c, nx = self.cur, 1 - self.cur
        kv, kv_dst = (bufs[c], bufs[nx]) if len(bufs) == 2 else (bufs[0], bufs[0])
        s = kv.stride()
        if self.zero_pads and kv_dst is not kv:
            raise ValueError("ZERO_PADS is an in-place option (ping-pong pads are don't-care, R8)")
        flags = (_abi.ZERO_PADS if self.zero_pads else 0) | (_abi.OVERLAP_PREV if overlap else 0) \
            | self._ws_flags()
        _abi.specdec_realign_kv(kv, kv_dst, count, n_planes=planes, n_rows=self.B, H=H, D=D,
                                src_strides=s[:3], dst_strides=s[:3], cap_src=self.cap_phys,
                                cap_dst=self.cap_phys, src_col=src, dst_col=dst,
                                flags=flags, ws=self.rws if self._ws_flags() else None,
                                moved_bytes=self.moved, status=self.status, stream=stream)

    def _ws_flags(self) -> int:
        return (_abi.SEGMENTED if self.segment else 0) | (_abi.DYNAMIC if self.dynamic else 0)

    def realign(self, stream=None):
        c, nx = self.cur, 1 - self.cur
        if self.B == 1 and self.anchor is None and self.kv_mode == "inplace":
            # a single row is always right-aligned at L' = n': p' = p = 0, so Realign is a
            # pure truncation that moves nothing -- no launch at all
            return
        if self.anchor is not None:
            src, dst = self.phys_old, self.phys_new        # f3: physical columns from K1
        else:
            src, dst = self.pad[c], self.pad[nx]
        # serial order K1 -> K3 -> K2: K3 waited on K1, so the first K2 may start under it
        self._realign_one(self._kvbuf, self.kept, (self.n_planes, self.H, self.D), src, dst, stream,
                          overlap=self.overlap and not self.fork)
        if self._dkvbuf is not None:     # f1: the draft model's own cache, same shift, kept_draft
            self._realign_one(self._dkvbuf, self.kept_draft, self.d_dims, src, dst, stream)

    @property
    def kernels_per_round(self) -> int:
        """libspecdec kernels one round launches (K1 = argmax grid + epilogue, K3, K2 per
        cache, + save kernels)."""
        k13 = _abi.specdec_verify_kernels(False) + 1
        if self.B == 1 and self.anchor is None and self.kv_mode == "inplace":
            return k13
        per_cache = 2 if self.segment and self.kv_mode == "inplace" else 1
        return k13 + per_cache * (2 if self.dkv is not None else 1)

    # ----------------------------------------------------------------- native round driver
    def round_desc(self, logits):
        """The `specdec_round_desc` of this batch for logits shaped like `logits`
        [B, k+1, >= V] (specdec_eqspec_round / specdec_eqspec_round_host)."""
        key = (logits.stride(1), logits.dtype, self.V or logits.shape[2])
        if getattr(self, "_rdesc_key", None) == key:
            d = self._rdesc
        else:
            p = lambda t: None if t is None else t.data_ptr()
            two = lambda a, b: (ctypes.c_void_p * 2)(p(a), p(b))
            d = _abi.RoundDesc()
            d.B, d.k, d.V, d.logit_stride = self.B, self.k, key[2], key[0]
            d.logit_dtype = _abi.DTYPE[logits.dtype]
            d.eos_id, d.pad_id = self.eos_id, self.pad_id
            d.n, d.pad, d.tokens = two(self.n[0], self.n[1]), two(self.pad[0], self.pad[1]), two(self.tok[0], self.tok[1])
            d.cap_tok = self.tok.shape[2]
            d.mask, d.pos, d.mp_stride = p(self.mask), p(self.pos), self.mask.stride(0)
            d.active, d.budget = p(self.active), p(self.budget)
            d.gen = p(self.gen) if self.out_buf is not None else None
            d.out_buf, d.max_new = p(self.out_buf), self.max_new
            d.accept = two(self._accept[0], self._accept[1])
            d.emit = two(self._emit[0], self._emit[1])
            d.bonus = two(self._bonus[0], self._bonus[1])
            d.finished = two(self._finished[0], self._finished[1])
            d.pred, d.kept, d.plan_L, d.kept_draft = p(self.pred), p(self.kept), p(self.plan_L), p(self.kept_draft)
            d.ws, d.ws_bytes = p(self.ws), self.ws.numel() * 8
            d.status, d.moved = p(self.status), p(self.moved)
            kb = self._kvbuf
            d.kv = two(kb[0], kb[-1])
            d.kv_dtype = _abi.DTYPE[kb[0].dtype]
            d.n_planes, d.H, d.D, d.cap_kv = self.n_planes, self.H, self.D, self.cap_phys
            d.s_plane, d.s_row, d.s_head = kb[0].stride()[:3]
            if self._dkvbuf is not None:
                db = self._dkvbuf
                d.dkv = two(db[0], db[-1])
                d.d_planes, d.d_H, d.d_D = self.d_dims
                d.d_s_plane, d.d_s_row, d.d_s_head = db[0].stride()[:3]
            d.anchor, d.phys_old, d.phys_new = p(self.anchor), p(self.phys_old), p(self.phys_new)
            self._rdesc, self._rdesc_key = d, key
        d.realign_flags = ((_abi.ZERO_PADS if self.zero_pads else 0)
                           | (_abi.OVERLAP_PREV if self.overlap else 0) | self._ws_flags())
        d.realign_ws = self.rws.data_ptr() if self._ws_flags() else None
        d.realign_ws_bytes = self.rws.numel() if self._ws_flags() else 0
        return d

    def launch_round_native(self, logits, draft, stream=None):
        """The same round through the native driver (one C call, specdec_eqspec_round)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._last = self.cur
        _abi.specdec_eqspec_round(self.round_desc(logits), self.cur, logits, draft, s)

    def host_io(self, like_logits, like_draft, n_slots=3):
        """Device staging (n_slots slots), copy / D2H streams and events for step_host: the
        end-to-end round from pinned host inputs (specdec_eqspec_round_host).  3 slots
        absorb the occasional slow H2D (specdec.h)."""
        io = _abi.HostIO()
        ns = int(n_slots)
        self._io_streams = [torch.cuda.Stream(self.device), torch.cuda.Stream(self.device)]
        self._io_events = [torch.cuda.Event() for _ in range(2 * ns + 2)]
        cur = torch.cuda.current_stream(self.device)
        for e in self._io_events:          # materialise the handles (recorded once, idle)
            e.record(cur)
        # each slot is one device buffer: the logits, then the drafts (one H2D per step when
        # the host inputs are packed the same way, see pack_host_inputs)
        self._io_lg, self._io_dr = zip(*[pack_inputs_like(like_logits, like_draft, self.device)
                                         for _ in range(ns)])
        pad = lambda xs: (ctypes.c_void_p * _abi.HOST_SLOTS)(*(list(xs) + [None] * (_abi.HOST_SLOTS - len(xs))))
        ev = [e.cuda_event for e in self._io_events]
        io.n_slots = ns
        io.d_logits = pad([t.data_ptr() for t in self._io_lg])
        io.d_draft = pad([t.data_ptr() for t in self._io_dr])
        io.copy_stream = self._io_streams[0].cuda_stream
        io.d2h_stream = self._io_streams[1].cuda_stream
        io.ev_ready, io.ev_done = pad(ev[:ns]), pad(ev[ns:2 * ns])
        io.ev_fetched = (ctypes.c_void_p * 2)(ev[2 * ns], ev[2 * ns + 1])
        self._io, self._io_slot, self._io_n = io, 0, ns
        return io

    def step_host(self, h_logits, h_draft, h_emit=None, V=None, zero_pads=False, stream=None):
        """One round from pinned host logits [B, k+1, >= V] / drafts [B, k]: H2D, the round
        and (if h_emit) the D2H of the emitted counts, all enqueued by one C call
        (specdec_eqspec_round_host); alternates the staging slot and flips the parity."""
        self.V, self.zero_pads = V, zero_pads
        if getattr(self, "_io", None) is None:
            self.host_io(h_logits, h_draft)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._last = self.cur
        _abi.specdec_eqspec_round_host(self.round_desc(h_logits), self._io, self.cur, self._io_slot,
                                       h_logits, h_draft, h_emit, s)
        self._io_slot = (self._io_slot + 1) % self._io_n
        self.cur = 1 - self.cur

    def launch_round(self, logits, draft, stream=None):
        """Enqueue K1 -> {K3 || K2} for the current parity (does not flip it).  K3 (tokens,
        masks, positions) and K2 (KV) both depend only on K1's plan and touch disjoint
        memory, so with `fork` K3 runs on a side stream under K2."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if self.native_round and not self.fork:
            self.launch_round_native(logits, draft, s)
            return
        if not self.fork:
            self.verify(logits, draft, s)
            self.repad(draft, s)
            self.realign(s)
            return
        if not hasattr(self, "_side"):
            self._side = torch.cuda.Stream(self.device)
            self._ev_plan, self._ev_rep = torch.cuda.Event(), torch.cuda.Event()
        self.verify(logits, draft, s)
        self._ev_plan.record(s)
        self._side.wait_event(self._ev_plan)
        self.repad(draft, self._side)
        self._ev_rep.record(self._side)
        self.realign(s)
        s.wait_event(self._ev_rep)

    def step(self, logits, draft, V=None, zero_pads=False, stream=None):
        """One EqSpec round on `stream`; flips the state parity."""
        self.V, self.zero_pads = V, zero_pads
        self.launch_round(logits, draft, stream)
        self.cur = 1 - self.cur

    # ----------------------------------------------------------------- CUDA graphs
    def capture(self, inputs, V=None):
        """Capture one graph per (parity, (logits, draft) pair): the round's three kernels
        replay with a single launch.  `inputs` is a list of (logits, draft) tensors whose
        storage must stay alive and fixed."""
        self.V = V
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        saved = self.cur
        with torch.cuda.stream(s):
            for parity in (0, 1):
                for j, (lg, d) in enumerate(inputs):
                    g = torch.cuda.CUDAGraph()
                    self.cur = parity
                    with torch.cuda.graph(g, stream=s):
                        self.launch_round(lg, d, stream=s)
                    self._graphs[(parity, j)] = g
        torch.cuda.current_stream(self.device).wait_stream(s)
        self.cur = saved

    def replay(self, j):
        """One EqSpec round from input pair j via its captured graph; flips the parity."""
        self._graphs[(self.cur, j)].replay()
        self._last = self.cur
        self.cur = 1 - self.cur
