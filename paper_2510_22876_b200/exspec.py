"""EXSpec SequencePool on device (Alg. 3; §3.2).

Sequences live individually in a pool -- tokens, generated output and a left-aligned KV
slab each ([N][planes][H][cap][D], sequence-major) -- in their ragged state.  An epoch:

    specdec_pool_group       K4  RefillWindow + same-length GetBatch plan for the window
    (one small D2H of the plan header: n_batches, kind, width -- the only host sync)
    for every batch of the plan:
        fallback batches only:   specdec_realign_kv gather  (pool -> right-aligned staging)
        [the model's verify forward runs here; synthetic workloads pass a hook]
        specdec_verify           K1  Alg. 1 on the batch rows (no budget: the pool applies it)
        specdec_pool_writeback   Phase 4: Pool[i] (+)= A[i] (+) B[i], deactivate if complete
        fallback batches only:   specdec_realign_kv scatter (the a+1 new KV rows back)

Same-length batches move no KV at all (lazy realignment): the consumer
reads the pool slots directly (zero-copy).  Sharding over GPUs is in dist.py.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _abi
from .eqspec import TORCH_DT


class SequencePool:
    def __init__(self, N, cap, layers, H, D, k, *, kv_dtype="bf16", W=32, B=8, min_group=2,
                 max_new=256, eos_id=-1, pad_id=0, cap_tok=None, device="cuda", kv_init=True,
                 dense_consumer=False, n_staging=1, consumer=None, verify_group=64, scatter_stream=False,
                 patience=0, pipeline=False):
        dev = torch.device(device)
        i32, i64, u8 = torch.int32, torch.int64, torch.uint8
        if B > W:
            raise ValueError("B must be <= W")
        self.N, self.cap, self.layers, self.H, self.D, self.k = N, cap, layers, H, D, k
        self.n_planes = 2 * layers
        self.W, self.B, self.min_group = W, B, min_group
        # deferred fallback (R27): an epoch's leftovers wait up to `patience` epochs for a
        # same-length partner (specdec_pool_group_deferred); 0 = the R11 plan
        if patience < 0:
            raise ValueError("patience must be >= 0")
        self.patience = int(patience)
        # pipelined fallback (R28, native executor only): a plan's mixed batches run on the
        # copy stream beside the next plan, which leaves their members out
        self.pipeline = bool(pipeline)
        self.max_new, self.eos_id, self.pad_id = max_new, eos_id, pad_id
        self.device = dev
        # the consumer of a batch's KV (specdec_pool_desc::dense_consumer): "zero-copy"
        # (mixed batches gathered into the staging, same-length ones on the pool slots),
        # "dense" (every batch gathered) or "slot" (a slot-indexed consumer:
        # no batch moves KV)
        self.consumer = consumer or ("dense" if dense_consumer else "zero-copy")
        if self.consumer not in ("zero-copy", "dense", "slot"):
            raise ValueError(f"consumer {self.consumer!r}")
        self.dense_consumer = self.consumer == "dense"
        if self.pipeline and self.consumer != "zero-copy":
            raise ValueError("pipeline needs the zero-copy consumer")
        # verify + write-back in one launch (specdec_pool_verify); False: the two calls
        self.fused = True
        self.cap_tok = cap_tok or cap
        # pool state
        self.len = torch.zeros(N, dtype=i32, device=dev)
        self.gen = torch.zeros(N, dtype=i32, device=dev)
        self.active = torch.zeros(N, dtype=u8, device=dev)
        self.order = torch.arange(N, dtype=i32, device=dev)
        self.wait = torch.zeros(N, dtype=i32, device=dev)      # R27: epochs sat out
        self.fb_epoch = torch.full((N,), -2, dtype=i32, device=dev)   # R28: plan of the last mixed batch
        self.plan_epoch = torch.zeros(1, dtype=i32, device=dev)       # R28: plans made
        self.tokens = torch.full((N, self.cap_tok), pad_id, dtype=i64, device=dev)
        self.out_buf = torch.zeros((N, max_new), dtype=i64, device=dev)
        alloc = torch.zeros if kv_init else torch.empty
        self.kv = alloc((N, self.n_planes, H, cap, D), dtype=TORCH_DT[kv_dtype], device=dev)
        self.staging = alloc((self.n_planes, B, H, cap, D), dtype=TORCH_DT[kv_dtype], device=dev)
        # native executor only: n_staging >= 2 overlaps the fallback gathers (copy stream,
        # ring of staging buffers) with the same-length batches (specdec_pool_desc)
        self.n_staging = int(n_staging)
        self.scatter_stream = bool(scatter_stream)   # native executor: scatters on a third stream
        self.staging_ring = [self.staging] + [alloc(self.staging.shape, dtype=self.staging.dtype, device=dev)
                                              for _ in range(max(self.n_staging, 1) - 1)]
        # plan (K4 outputs)
        self.window = torch.zeros(W, dtype=i32, device=dev)
        self.window_size = torch.zeros(1, dtype=i32, device=dev)
        self.batch_of = torch.zeros(N, dtype=i32, device=dev)
        self.slot_of = torch.zeros(N, dtype=i32, device=dev)
        # plan rows: 2W batch rows, the pipelined executor alternates between the halves
        # (R28); every other path uses the first W
        self._rows_full = [torch.zeros((2 * W, B), dtype=dt, device=dev) for dt in (i32, i32, i32, u8)]
        self.members, self.mlen, self.mpad, self.mactive = (t[:W] for t in self._rows_full)
        # the plan header arrays share one buffer laid out like the pinned host header
        # (n_batches | bkind in W int32 slots | blen | bsize): one D2H copy per epoch
        self._hdr_dev = torch.zeros(1 + 3 * W, dtype=i32, device=dev)
        self.n_batches = self._hdr_dev[0:1]
        self.bkind = self._hdr_dev[1:1 + W].view(u8)[:W]
        self.blen = self._hdr_dev[1 + W:1 + 2 * W]
        self.bsize = self._hdr_dev[1 + 2 * W:1 + 3 * W]
        self.counters = torch.zeros(8, dtype=i64, device=dev)
        # per-batch verify scratch; the native executor verifies up to `verify_group`
        # same-length batches per launch (specdec_pool_verify_group): rows for all of them
        self.verify_group = max(1, min(int(verify_group), _abi.MAX_VERIFY_GROUP))
        GB = self.verify_group * B
        self.accept = torch.zeros(GB, dtype=i32, device=dev)
        self.bonus = torch.zeros(GB, dtype=i64, device=dev)
        self.emit = torch.zeros(GB, dtype=i32, device=dev)
        self.finished = torch.zeros(GB, dtype=u8, device=dev)
        self.n_new = torch.zeros(B, dtype=i32, device=dev)
        self.pad_new = torch.zeros(B, dtype=i32, device=dev)
        self.kept = torch.zeros(B, dtype=i32, device=dev)
        self.plan_L = torch.zeros(1, dtype=i32, device=dev)
        ws = _abi.specdec_verify_workspace_size(GB, k)
        self.ws = torch.zeros((ws + 7) // 8, dtype=i64, device=dev)
        self.status = torch.zeros(1, dtype=i32, device=dev)
        self.moved = torch.zeros(1, dtype=i64, device=dev)
        self.verify_calls = 0
        self._pinned = torch.zeros(1 + 3 * W, dtype=i32)   # plan header, host side
        if dev.type == "cuda":
            self._pinned = self._pinned.pin_memory()

    # ----------------------------------------------------------------- state
    def load(self, prompts_lens, tokens=None, order=None, kv=None):
        """Admit N sequences: lengths (prompt incl. the pending last token), optional
        tokens [N, cap_tok], admission order (default by id) and KV."""
        self.len.copy_(torch.as_tensor(np.asarray(prompts_lens), dtype=torch.int32))
        self.gen.zero_()
        self.wait.zero_()
        self.fb_epoch.fill_(-2)
        self.plan_epoch.zero_()
        if getattr(self, "_pipe_host", None) is not None:
            self._pipe_host[0] = self._pipe_host[1] = 0
        self.active.fill_(1)
        if order is not None:
            self.order.copy_(torch.as_tensor(np.asarray(order), dtype=torch.int32))
        if tokens is not None:
            self.tokens.copy_(torch.as_tensor(tokens))
        if kv is not None:
            self.kv.copy_(kv)
        self.counters.zero_()
        self.verify_calls = 0
        if getattr(self, "_ring_pos", None) is not None:
            self._ring_pos.value = 0      # the native executor's input ring restarts too

    @property
    def kv_strides(self):
        s = self.kv.stride()          # [N][planes][H][cap][D]
        return (s[1], s[0], s[2])     # (plane, row, head)

    @property
    def staging_strides(self):
        s = self.staging.stride()     # [planes][B][H][cap][D]
        return (s[0], s[1], s[2])

    # ----------------------------------------------------------------- plan
    def plan(self, stream=None):
        """K4 over the window; returns the host copy of the plan header
        (n_batches, kinds, widths, sizes) -- the epoch's single device->host sync."""
        if self.patience > 0:
            _abi.specdec_pool_group_deferred(self.len, self.active, self.order, self.W, self.B, self.min_group,
                                             self.wait, self.patience, self.window, self.window_size,
                                             self.batch_of, self.slot_of, self.members, self.mlen, self.mpad,
                                             self.mactive, self.bsize, self.bkind, self.blen, self.n_batches,
                                             self.counters, stream=stream)
        else:
            _abi.specdec_pool_group(self.len, self.active, self.order, self.W, self.B, self.min_group,
                                    self.window, self.window_size, self.batch_of, self.slot_of,
                                    self.members, self.mlen, self.mpad, self.mactive, self.bsize,
                                    self.bkind, self.blen, self.n_batches, self.counters, stream=stream)
        W = self.W
        hdr = self._pinned
        # the copies are ordered after K4 on the stream it ran on, and that stream is the one
        # synchronised (a non-current `stream` gets no implicit order with torch's stream)
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        with torch.cuda.stream(s):
            hdr[0:1].copy_(self.n_batches, non_blocking=True)
            hdr[1:1 + W].copy_(self.bkind.to(torch.int32), non_blocking=True)
            hdr[1 + W:1 + 2 * W].copy_(self.blen, non_blocking=True)
            hdr[1 + 2 * W:1 + 3 * W].copy_(self.bsize, non_blocking=True)
        s.synchronize()
        nb = int(hdr[0])
        h = hdr.numpy()
        return nb, h[1:1 + nb].copy(), h[1 + W:1 + W + nb].copy(), h[1 + 2 * W:1 + 2 * W + nb].copy()

    # ----------------------------------------------------------------- one batch
    def gather(self, b, stream=None):
        """Fallback batch b: pool slots [0, len-1) -> staging rows right-aligned at the
        batch width (unpad-repad realignment)."""
        _abi.specdec_realign_kv(self.kv, self.staging, self.mlen[b], count_add=-1,
                                n_planes=self.n_planes, n_rows=self.B, H=self.H, D=self.D,
                                src_strides=self.kv_strides, dst_strides=self.staging_strides,
                                cap_src=self.cap, cap_dst=self.cap, dst_col=self.mpad[b],
                                src_row_map=self.members[b], moved_bytes=self.moved,
                                status=self.status, stream=stream)

    def scatter(self, b, blen, stream=None):
        """Write-back Pool.KV[i] <- KV[i]: the a+1 new rows
        staging [L_b-1, L_b+a) -> pool [len-1, len+a)."""
        _abi.specdec_realign_kv(self.staging, self.kv, self.accept, count_add=1, count_bound=self.k + 1,
                                n_planes=self.n_planes, n_rows=self.B, H=self.H, D=self.D,
                                src_strides=self.staging_strides, dst_strides=self.kv_strides,
                                cap_src=self.cap, cap_dst=self.cap, src_col_add=int(blen) - 1,
                                dst_col=self.mlen[b], dst_col_add=-1,
                                dst_row_map=self.members[b], moved_bytes=self.moved,
                                status=self.status, stream=stream)

    def verify(self, b, logits, draft, V=None, stream=None):
        _abi.specdec_verify(logits, draft, self.mlen[b], self.mactive[b], self.accept, self.bonus,
                            self.emit, self.finished, self.plan_L, self.n_new, self.pad_new,
                            self.kept, self.ws, V=V or logits.shape[2], eos_id=self.eos_id,
                            pad_id=self.pad_id, budget=None, status=self.status, stream=stream)
        self.verify_calls += 1

    def writeback(self, b, draft, stream=None):
        _abi.specdec_pool_writeback(self.members[b], self.k, draft, self.accept, self.bonus,
                                    self.emit, self.finished, self.len, self.gen, self.active,
                                    max_new=self.max_new, pool_tokens=self.tokens,
                                    out_buf=self.out_buf, status=self.status, stream=stream)

    def verify_writeback(self, b, logits, draft, V=None, stream=None):
        """Alg. 1 on batch b and the Phase 4 write-back: one fused launch, or the two calls."""
        if not self.fused:
            self.verify(b, logits, draft, V, stream)
            self.writeback(b, draft, stream)
            return
        _abi.specdec_pool_verify(logits, draft, self.members[b], self.mlen[b], self.mactive[b],
                                 self.accept, self.bonus, self.emit, self.finished, self.len,
                                 self.gen, self.active, self.ws, V=V or logits.shape[2],
                                 eos_id=self.eos_id, pad_id=self.pad_id, max_new=self.max_new,
                                 pool_tokens=self.tokens, out_buf=self.out_buf,
                                 status=self.status, stream=stream)
        self.verify_calls += 1

    def moves_kv(self, kind) -> bool:
        """Does a batch of this kind go through the staging (gather / scatter)?"""
        return self.consumer == "dense" or (not kind and self.consumer == "zero-copy")

    def run_batch(self, b, kind, blen, logits, draft, forward=None, V=None, stream=None):
        fallback = self.moves_kv(kind)
        if fallback:
            self.gather(b, stream)
        if forward is not None:
            forward(self, b, not fallback, int(blen))
        self.verify_writeback(b, logits, draft, V, stream)
        if fallback:
            self.scatter(b, blen, stream)

    def epoch(self, inputs, forward=None, V=None, stream=None):
        """Plan the window and run every batch of the plan.  `inputs(i)` returns the
        (logits [B, k+1, V], draft [B, k]) of the epoch's i-th batch.  Returns the plan
        header (n_batches, kinds, widths, sizes)."""
        nb, kinds, blens, sizes = self.plan(stream)
        for b in range(nb):
            lg, d = inputs(b)
            self.run_batch(b, kinds[b], blens[b], lg, d, forward, V, stream)
        return nb, kinds, blens, sizes

    def alg3_step(self, inputs, forward=None, V=None, stream=None):
        """One iteration of Alg. 3 as printed: GetBatch -> draft ->
        verify -> write-back -> RefillWindow, i.e. only batch 0 of the window plan runs
        before the window is re-planned.  Returns False when the
        pool has no active sequence."""
        nb, kinds, blens, sizes = self.plan(stream)
        if nb == 0:
            return False
        lg, d = inputs(0)
        self.run_batch(0, kinds[0], blens[0], lg, d, forward, V, stream)
        return True

    # ----------------------------------------------------------------- native executor
    def native(self, ring, V, logit_dtype=torch.bfloat16, est_gather_GBps=0.0, est_verify_us=0.0):
        """Bind a `specdec_pool_desc` to this pool and an input ring [(logits, draft)] for
        `epoch_native` (the per-batch launch loop in C++, csrc/pool_exec.cu)."""
        p = lambda t: t.data_ptr() if t is not None else None
        d = _abi.PoolDesc()
        for name in ("len", "gen", "active", "order", "tokens", "out_buf", "kv", "staging", "window",
                     "window_size", "batch_of", "slot_of", "members", "mlen", "mpad", "mactive",
                     "bsize", "bkind", "blen", "n_batches", "counters", "accept", "bonus", "emit",
                     "finished", "n_new", "pad_new", "kept", "plan_L", "ws", "status", "moved"):
            setattr(d, name, p(getattr(self, name)))
        d.N, d.cap_tok, d.max_new = self.N, self.tokens.shape[1], self.max_new
        d.kv_dtype = _abi.DTYPE[self.kv.dtype]
        d.n_planes, d.H, d.D, d.cap = self.n_planes, self.H, self.D, self.cap
        d.ws_bytes = self.ws.numel() * 8
        self._hdr = torch.zeros(1 + 3 * self.W, dtype=torch.int32).pin_memory()
        d.host_header = self._hdr.data_ptr()
        d.W, d.B, d.min_group = self.W, self.B, self.min_group
        d.k, d.V, d.eos_id, d.pad_id = self.k, V, self.eos_id, self.pad_id
        d.logit_stride = ring[0][0].stride(1)
        d.logit_dtype = _abi.DTYPE[logit_dtype]
        self._ring = ring                                    # keep the tensors alive
        self._lg_ptrs = (ctypes.c_void_p * len(ring))(*[lg.data_ptr() for lg, _ in ring])
        self._dr_ptrs = (ctypes.c_void_p * len(ring))(*[dr.data_ptr() for _, dr in ring])
        self._ring_pos = ctypes.c_int32(0)
        d.logits_ring = ctypes.cast(self._lg_ptrs, ctypes.c_void_p)
        d.draft_ring = ctypes.cast(self._dr_ptrs, ctypes.c_void_p)
        d.ring_n = len(ring)
        d.ring_pos = ctypes.addressof(self._ring_pos)
        d.dense_consumer = {"zero-copy": 0, "dense": 1, "slot": 2}[self.consumer]
        d.wait, d.patience = self.wait.data_ptr(), self.patience
        # the gathers take K2 work tickets (SPECDEC_DYNAMIC) from a zeroed 128-byte header
        self._gather_ws = torch.zeros(128, dtype=torch.uint8, device=self.device)
        d.gather_ws = self._gather_ws.data_ptr()
        d.verify_group = self.verify_group
        self._launches = ctypes.c_int64(0)      # libspecdec kernels the executor launched
        d.host_launches = ctypes.addressof(self._launches)
        if self.pipeline:
            self._pipe_copy = torch.cuda.Stream(self.device)
            self._pipe_events = [torch.cuda.Event(enable_timing=False) for _ in range(2)]
            for ev in self._pipe_events:
                ev.record(torch.cuda.current_stream(self.device))
            self._pipe_ev_ptrs = (ctypes.c_void_p * 2)(*[ev.cuda_event for ev in self._pipe_events])
            self._pipe_host = (ctypes.c_int64 * 2)(0, 0)
            # the chain runs on one stream: one staging buffer is enough (stream order)
            self._pipe_stg = (ctypes.c_void_p * 1)(self.staging.data_ptr())
            self._pipe_accept = torch.zeros(self.B, dtype=torch.int32, device=self.device)
            ws2 = _abi.specdec_verify_workspace_size(self.B, self.k)
            self._ws2 = torch.zeros((ws2 + 7) // 8, dtype=torch.int64, device=self.device)
            self._bonus2 = torch.zeros(self.B, dtype=torch.int64, device=self.device)
            self._emit2 = torch.zeros(self.B, dtype=torch.int32, device=self.device)
            self._finished2 = torch.zeros(self.B, dtype=torch.uint8, device=self.device)
            d.pipeline = 1
            d.fb_epoch, d.plan_epoch = self.fb_epoch.data_ptr(), self.plan_epoch.data_ptr()
            d.ws2, d.ws2_bytes = self._ws2.data_ptr(), self._ws2.numel() * 8
            d.bonus2, d.emit2, d.finished2 = self._bonus2.data_ptr(), self._emit2.data_ptr(), self._finished2.data_ptr()
            d.pipe_events = ctypes.cast(self._pipe_ev_ptrs, ctypes.c_void_p)
            d.pipe_host = ctypes.addressof(self._pipe_host)
            d.n_staging = 1
            d.staging_ring = ctypes.cast(self._pipe_stg, ctypes.c_void_p)
            d.copy_stream = self._pipe_copy.cuda_stream
            d.accept_ring = self._pipe_accept.data_ptr()
        elif self.n_staging >= 2:
            ns = self.n_staging
            self._copy_stream = torch.cuda.Stream(self.device)
            self._events = [torch.cuda.Event(enable_timing=False) for _ in range(2 * ns)]
            for e in self._events:
                e.record(torch.cuda.current_stream(self.device))   # materialise the handle
            self._stg_ptrs = (ctypes.c_void_p * ns)(*[t.data_ptr() for t in self.staging_ring])
            self._ev_ptrs = (ctypes.c_void_p * (2 * ns))(*[e.cuda_event for e in self._events])
            d.n_staging = ns
            d.staging_ring = ctypes.cast(self._stg_ptrs, ctypes.c_void_p)
            d.copy_stream = self._copy_stream.cuda_stream
            d.events = ctypes.cast(self._ev_ptrs, ctypes.c_void_p)
            self._accept_ring = torch.zeros((ns, self.B), dtype=torch.int32, device=self.device)
            d.accept_ring = self._accept_ring.data_ptr()
            if self.scatter_stream:
                # the scatters on a third stream, beside the gathers
                self._scatter_stream = torch.cuda.Stream(self.device)
                self._sevents = [torch.cuda.Event(enable_timing=False) for _ in range(ns)]
                for ev in self._sevents:
                    ev.record(torch.cuda.current_stream(self.device))
                self._sev_ptrs = (ctypes.c_void_p * ns)(*[ev.cuda_event for ev in self._sevents])
                d.scatter_stream = self._scatter_stream.cuda_stream
                d.scatter_events = ctypes.cast(self._sev_ptrs, ctypes.c_void_p)
            d.est_gather_GBps, d.est_verify_us = float(est_gather_GBps), float(est_verify_us)
        self._desc = d
        return d

    def epoch_native(self, max_batches=0, stream=None, forward=None):
        """One epoch (or, with max_batches=1, one Alg. 3 iteration) in the native executor.
        `forward`: optional _abi.FORWARD_FN called per batch for its (logits, draft).
        pipeline (R28): one plan per call, its mixed batches left running on the copy
        stream; a call returning 0 batches leaves the pool drained and every chain done.
        Returns (batches run, same-length batches run, members same, members fallback)."""
        r = _abi.specdec_pool_epoch(self._desc, max_batches, stream, forward)
        self.verify_calls += r[0]
        return r

    def alg3_native(self, iterations, stream=None):
        """`iterations` iterations of Alg. 3 as printed (plan, batch 0, re-plan) in one C call
        with no host synchronisation (specdec_pool_alg3; after `native`).  Executed-batch
        counters accumulate in self.alg3_exec [batches, same-length, their members,
        fallback members]."""
        if getattr(self, "_alg3_scratch", None) is None:
            self._alg3_scratch = torch.zeros(4 * self.B, dtype=torch.int32, device=self.device)
            self.alg3_exec = torch.zeros(4, dtype=torch.int64, device=self.device)
        _abi.specdec_pool_alg3(self._desc, iterations, self._alg3_scratch, self.alg3_exec, stream)

    def alg3_graph(self, replays, stream=None, conditional=False):
        """`replays` x ring_n iterations of the Alg. 3 device loop from ONE CUDA graph of ring_n
        iterations built by the library (specdec_pool_alg3_graph: the loop's launches with
        their PDL edges; `conditional`: the KV moves in IF nodes instead -- measured slower).
        Call after `native` and one direct `alg3_native` call (which creates the scratch and
        sets the kernels' attributes).  The graph binds the input-ring slots from the ring
        position at build time; ring_n iterations leave it unchanged modulo ring_n, so every
        replay continues the sequence the direct loop takes."""
        if getattr(self, "_alg3_gexec", None) is None:
            self._alg3_gexec = _abi.specdec_pool_alg3_graph(self._desc, len(self._ring), self._alg3_scratch,
                                                            self.alg3_exec, conditional)
        s = stream or torch.cuda.current_stream(self.device)
        for _ in range(replays):
            _abi.specdec_graph_launch(self._alg3_gexec, s)

    def close(self):
        """Release the Alg. 3 graph (if built)."""
        if getattr(self, "_alg3_gexec", None):
            _abi.specdec_graph_destroy(self._alg3_gexec)
            self._alg3_gexec = None

    def has_active(self) -> bool:
        return bool(self.active.any().item())
