/*
 * specdec.h -- C ABI of libspecdec.so: the per-round hot path of batch speculative
 * decoding (EqSpec / EXSpec, arXiv 2510.22876) on NVIDIA B200 (sm_100a).
 *
 * Conventions (all entry points)
 *  - Every compute call is ASYNCHRONOUS on the caller's CUDA stream (`stream`, a
 *    cudaStream_t; NULL = legacy default stream).  It never allocates, never
 *    synchronises the host and never copies device->host.  It is stateless and
 *    thread-safe for disjoint buffers.
 *  - Pointers named `d_*` are DEVICE pointers owned by the caller; they must stay
 *    valid until the stream reaches the call.  Scalars are passed by value.
 *  - Token ids, positions and masks are int64 (HuggingFace layout); lengths, pads,
 *    counts are int32; flags are uint8.
 *  - Return value: SPECDEC_OK (0) or a negative SPECDEC_ERR_* detected on the host
 *    from the arguments alone (nothing is launched on error).  Errors that depend
 *    on device data are OR-ed into the optional device word `d_status` (bits
 *    SPECDEC_ST_*) without any synchronisation; the affected row/item is skipped.
 *
 * Notation (Alg. 1-3): a batch row i holds n_i content tokens
 * right-aligned at width L (left pads p_i = L - n_i); its last content token is
 * "pending" (no KV yet).  The verify forward appends k+1 KV entries,
 * so row i's valid KV after it is [p_i, L + a_i) and kept_i = n_i + a_i.
 */
#ifndef SPECDEC_H_
#define SPECDEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *specdec_stream_t; /* == cudaStream_t */

/* host-detected errors */
#define SPECDEC_OK 0
#define SPECDEC_ERR_ARG (-1)      /* null / misaligned pointer, k outside [1, 31], bad flag, unsupported stride */
#define SPECDEC_ERR_SHAPE (-2)    /* inconsistent sizes (e.g. V < 1, row_stride < V, W < 1) */
#define SPECDEC_ERR_DTYPE (-3)    /* unknown dtype code */
#define SPECDEC_ERR_CAPACITY (-4) /* statically impossible capacity (e.g. cap < k + 2) */
#define SPECDEC_ERR_CUDA (-5)     /* a CUDA launch/runtime error; see specdec_last_cuda_error() */

/* element dtypes */
#define SPECDEC_F32 0
#define SPECDEC_F16 1
#define SPECDEC_BF16 2

/* device status bits (OR-ed into *d_status) */
#define SPECDEC_ST_NAN 1u      /* a NaN logit was seen (the argmax is still defined: first NaN) */
#define SPECDEC_ST_CAPACITY 2u /* a width / buffer bound would be exceeded; the row was skipped */
#define SPECDEC_ST_KEPT 4u     /* a KV row range lies outside [0, cap); the item was skipped */
#define SPECDEC_ST_BOUND 8u    /* a row's count exceeded the caller's count_bound; row skipped */

/* specdec_realign_kv flags */
#define SPECDEC_ZERO_PADS 1u    /* also zero the old content columns that became pads */
#define SPECDEC_OVERLAP_PREV 2u /* start under the previous kernel on the stream (see below) */
#define SPECDEC_DYNAMIC 4u      /* dynamic work tickets from the workspace header (see below) */
#define SPECDEC_SEGMENTED 8u    /* in place: cut slabs into segments (workspace slots) */
#define SPECDEC_DYNAMIC_FORCE 16u /* with SPECDEC_DYNAMIC: tickets even for few units per CTA */

#define SPECDEC_MAX_VERIFY_GROUP 64 /* specdec_pool_verify_group: batches per launch */

/* ------------------------------------------------------------------------------ misc */
int specdec_version(void);                /* ABI version (major*100 + minor) */
const char *specdec_last_cuda_error(void); /* message for the last SPECDEC_ERR_CUDA (thread-local) */

/* Kernels one specdec_verify (pool = 0) or specdec_pool_verify (pool = 1) call launches:
 * 2 for specdec_verify (the argmax grid, then a one-CTA epilogue kernel that builds the
 * plan), 1 for specdec_pool_verify (each batch row's epilogue runs in the last CTA of that
 * row; the pool has no cross-row plan) -- the measured best of each; SPECDEC_K1_SPLIT=E[,P]
 * overrides (0 grid arrival, 1 epilogue kernel, 2 per-row arrival). */
int specdec_verify_kernels(int pool);

/* Bytes of the device workspace specdec_verify needs for (B, k).  The workspace must be
 * zero-filled ONCE when allocated; every completed specdec_verify leaves it zeroed again
 * (self-cleaning), so it can be reused by consecutive calls on one stream. */
size_t specdec_verify_workspace_size(int64_t B, int64_t k);

/* ------------------------------------------------------------------------------ a1
 * specdec_verify -- Alg. 1 BatchVerify fused with the BatchRepad plan
 * (Alg. 2 line "S, offset <- BatchRepad(S)").
 *
 *   pred[i][j] = argmax_v logits[i][j][v]      j = 0..k
 *       ties -> lowest v; NaN ranks above +inf and the first NaN wins; +0 == -0.
 *   a_i = first j < k with pred[i][j] != draft[i][j], else k   (R1)
 *   b_i = pred[i][a_i]                                         (R2)
 *   E_i = draft[i][0:a_i] ++ [b_i], cut after the first eos_id (eos_id >= 0) and to
 *         budget[i] tokens (if d_budget); either cut sets finished_i; emit_i = |E_i|.
 *   Plan (R6, R9): rows still active: n'_i = n_i + a_i + 1,
 *         kept_i = n_i + a_i; finished rows: n'_i = 1, kept_i = 0;
 *         L' = max n' over still-active rows (0 if none); p'_i = L' - n'_i.
 *   Rows with d_active[i] == 0 yield a=0, b=pad_id, emit=0, finished=1.
 *
 * d_logits  [B][k+1][row_stride] of `dtype` (the k+1-row tail of the verify forward;
 *           row j predicts draft slot j, row k the token after d_k).  16-B aligned,
 *           row_stride*sizeof(dtype) % 16 == 0, row_stride >= V.
 * d_draft   [B][k] int64; d_n [B] int32 (content lengths).
 * d_active  [B] uint8, IN/OUT: rows to verify; on completion d_active[i] = !finished_i,
 *           so a fixed-pointer round loop (or CUDA graph) carries it to the next round.
 * d_budget  [B] int32 remaining new-token budget, or NULL (unbounded); IN/OUT: on
 *           completion d_budget[i] = max(budget_i, 0) - emit_i.
 * Outputs: d_accept [B] int32, d_bonus [B] int64, d_emit [B] int32, d_finished [B] uint8,
 *          d_pred [B][k+1] int64 or NULL, d_plan_L [1] int32, d_n_new, d_pad_new,
 *          d_kept [B] int32.
 * d_kept_draft [B] int32 or NULL: the draft model's kept KV count when
 *          it caches its own k forwards (pending token, d_1..d_{k-1}; d_k has no draft KV):
 *          n_i + min(a_i, k-1) for still-active rows, 0 for finished rows.  Realign the
 *          draft cache with the same p -> p' as the target and this count.
 * d_anchor [1] int32 or NULL (anchored origin), IN/OUT: the physical
 *          column of the KV buffer where logical column 0 lives (base).  The logical
 *          plan (tokens, masks, positions, p') is unchanged; the new origin base' = base + d
 *          is chosen among d = 0 and d = (a+1) - (L'-L), a = 0..k, to minimise the KV rows
 *          that move (ties: d = 0, then larger d), subject to 0 <= base' and
 *          base' + L' + k <= anchor_cap (the physical capacity).  Then
 *          d_phys_old[i] = base + (L - n_i) and d_phys_new[i] = base' + p'_i [B] int32 are
 *          the src/dst columns for specdec_realign_kv (L = max n_i, R6).
 * d_ws: workspace of specdec_verify_workspace_size(B, k) bytes (see above).
 * d_status: optional (NULL ok); SPECDEC_ST_NAN.
 */
int specdec_verify(const void *d_logits, int dtype, int64_t B, int64_t k, int64_t V,
                   int64_t row_stride, const int64_t *d_draft, const int32_t *d_n,
                   uint8_t *d_active, int64_t eos_id, int64_t pad_id,
                   int32_t *d_budget, int32_t *d_accept, int64_t *d_bonus,
                   int32_t *d_emit, uint8_t *d_finished, int64_t *d_pred, int32_t *d_plan_L,
                   int32_t *d_n_new, int32_t *d_pad_new, int32_t *d_kept,
                   int32_t *d_kept_draft, int32_t *d_anchor, int64_t anchor_cap,
                   int32_t *d_phys_old, int32_t *d_phys_new, uint32_t *d_status, void *d_ws,
                   size_t ws_bytes, specdec_stream_t stream);

/* ------------------------------------------------------------------------------ a2 (init)
 * specdec_batch_init -- Alg. 2 line 1, S <- Tokenize(P) with "batch left padding"
 * (PAPER.md:334): the batch state an EqSpec loop starts from.
 *
 *   L = max_i n_i (R6: the minimal width; every row is active at admission),
 *   pad_i = L - n_i (content right-aligned at width L),
 *   d_active[i] = 1, d_budget[i] = max_new.
 *
 * d_n [B] int32 content lengths (>= 1; a row with n_i < 1 sets SPECDEC_ST_CAPACITY and
 *   gets pad_i = L).  Outputs: d_pad [B] int32; d_L [1] int32, d_active [B] uint8 and
 *   d_budget [B] int32 are each optional (NULL: not written).  One CTA; no host sync.
 * The caller places the prompt tokens right-aligned in its [B][cap_tok] token buffer
 * (specdec_rebuild_pos_mask derives masks / positions from pad each round).
 * Errors: SPECDEC_ERR_ARG for NULL d_n / d_pad; SPECDEC_ERR_SHAPE for B < 1.
 */
int specdec_batch_init(const int32_t *d_n, int64_t B, int32_t *d_pad, int32_t *d_L,
                       uint8_t *d_active, int32_t *d_budget, int32_t max_new,
                       uint32_t *d_status, specdec_stream_t stream);

/* ------------------------------------------------------------------------------ a2
 * specdec_rebuild_pos_mask -- Alg. 2 Phase 3 unpad-append-repad and
 * the padding-agnostic positions / masks of §3.1, from specdec_verify's
 * outputs, entirely on device (the new width L' is read from d_plan_L).
 *
 *   still-active row i: content' = tokens[i][p_i .. L) ++ draft[i][0:a_i] ++ [b_i]
 *                       written at [p'_i, L'), pad_id on [0, p'_i);
 *   finished row (R9):  content' = [pad_id] at L'-1 (a dummy length-1 row);
 *   for c in [0, L'+k): mask[i][c] = (c >= p'_i); pos[i][c] = c >= p'_i ? c - p'_i : 0 (R7).
 *   If d_out_buf: E_i (the first emit_i tokens of draft[i][0:a_i] ++ [b_i]) is appended
 *   at d_out_buf[i][d_gen[i] ..] and d_gen[i] += emit_i.
 *   If L' == 0 (every row finished) only the out_buf / gen update happens.
 *
 * d_tokens_in / d_tokens_out [B][cap_tok] int64 -- may be the SAME buffer (in place: one CTA
 *   per row walks it in the hazard-free direction) or two buffers (ping-pong: every output
 *   column is an independent gather, spread over many CTAs -- the fast path).
 * d_n_old, d_pad_old [B] int32: the state before this round (L = pad_old + n_old).
 * d_accept, d_bonus, d_emit, d_finished, d_plan_L, d_pad_new: specdec_verify outputs.
 * d_draft [B][k] int64.  d_mask, d_pos [B][mp_stride] int64 (columns [0, L'+k) written).
 * d_out_buf [B][max_new] int64 and d_gen [B] int32, or both NULL.
 * d_status: SPECDEC_ST_CAPACITY if L' > cap_tok, L'+k > mp_stride or gen+emit > max_new.
 */
int specdec_rebuild_pos_mask(const int64_t *d_tokens_in, int64_t *d_tokens_out, int64_t B,
                             int64_t cap_tok, int64_t k, int64_t pad_id,
                             const int32_t *d_n_old, const int32_t *d_pad_old,
                             const int64_t *d_draft, const int32_t *d_accept,
                             const int64_t *d_bonus, const int32_t *d_emit,
                             const uint8_t *d_finished, const int32_t *d_plan_L,
                             const int32_t *d_pad_new, int64_t *d_mask, int64_t *d_pos,
                             int64_t mp_stride, int64_t *d_out_buf, int32_t *d_gen,
                             int64_t max_new, uint32_t *d_status, specdec_stream_t stream);

/* ------------------------------------------------------------------------------ a3 / a5
 * specdec_realign_kv -- KVCache <- Realign(KVCache, offset) (§3.1
 * PAPER.md:447), and the EXSpec pool gather / write-back scatter (Alg. 3 PAPER.md:492,
 * 505), as one row-mapped KV move:
 *
 *   for every batch row r in [0, n_rows) with cnt_r = count[r] + count_add > 0,
 *   srow = src_row_map ? src_row_map[r] : r  (skipped if < 0), drow likewise,
 *   scol = (src_col ? src_col[r] : 0) + src_col_add, dcol likewise,
 *   and every plane (layer x {K,V}) and KV head h:
 *       dst[plane, drow, h, dcol + c, :] = src[plane, srow, h, scol + c, :]   c < cnt_r
 *
 *   and no other byte of dst is written (except the SPECDEC_ZERO_PADS columns): in place,
 *   every column outside a row's destination range keeps its value.
 *
 * EqSpec in place: kv_dst == kv_src, src_col = pad_old, dst_col = pad_new, count = kept.
 * Rows whose source and destination coincide move nothing.  Each (plane, row, head)
 * slab is streamed by one CTA in the hazard-free direction through a TMA bulk-copy
 * (cp.async.bulk) shared-memory ring, so in-place shifts of either sign are exact.
 * In-place calls (kv_dst == kv_src) must not pass row maps.  Distinct src/dst buffers
 * must not overlap.
 *
 * dtype: SPECDEC_F16 / SPECDEC_BF16 / SPECDEC_F32 (only its size matters: bytes are copied).
 * Layout: element (plane, row, head, pos, d) at base + plane*s_plane + row*s_row +
 *   head*s_head + pos*D + d (strides in ELEMENTS; a KV row of D elements is contiguous
 *   and D*elem % 16 == 0; base 16-B aligned; strides*elem multiples of 16).
 * cap_src / cap_dst: position capacity of each buffer (scol+cnt <= cap_src and
 *   dcol+cnt <= cap_dst, else SPECDEC_ST_KEPT and the row is skipped).
 * flags: SPECDEC_ZERO_PADS (in place only): zero [scol, dcol) when dcol > scol.
 *   SPECDEC_OVERLAP_PREV: the caller guarantees that the call enqueued immediately before
 *   on `stream` is a specdec_* kernel launch that itself waited for the producer of this
 *   call's columns / counts / KV (e.g. specdec_rebuild_pos_mask right after
 *   specdec_verify) and that this call does not read what it writes.  The copy then
 *   starts while that kernel runs (programmatic dependent launch) and waits for it only
 *   before exiting, so completion order on the stream is unchanged.  Ignored with
 *   SPECDEC_SEGMENTED in place (the boundary-save kernel must finish first) and with PDL
 *   off.
 *   SPECDEC_DYNAMIC: the streaming CTAs take work units from a ticket counter in the
 *   workspace header instead of a static assignment, so CTAs that stream faster take more
 *   units (measured +1 % at Qwen3 B=8, +1.2 % Vicuna).  Needs d_ws.  With fewer than ~8
 *   units per CTA the static assignment is as balanced and avoids the ticket round trips,
 *   so the library then ignores SPECDEC_DYNAMIC unless SPECDEC_DYNAMIC_FORCE is also set
 *   (tests use it to exercise the ticket path on small problems).
 *   SPECDEC_SEGMENTED (in place): every slab is cut into ~128 KB segments that any CTA can
 *   stream independently: the rows a segment's neighbour overwrites (|dcol - scol| rows,
 *   <= 4 KB) are first copied to a workspace slot by a small kernel on the same stream.
 *   Without it a slab is one unit in place (correct; less balanced when few rows move).
 *   Needs d_ws.  Distinct buffers are always segmented (no slots needed).
 * d_ws / ws_bytes: device workspace (16-B aligned) for SPECDEC_DYNAMIC / SPECDEC_SEGMENTED:
 *   a 128-byte header -- the dynamic-schedule counters (uint32 words 0-1), which must be
 *   ZERO before the first call and are left zero by every call; words 2-3 are diagnostics
 *   that only accumulate (dynamic launches completed, work units streamed by ticket) and
 *   are never read by the library -- then the segment slots.  Size: 128 bytes for
 *   SPECDEC_DYNAMIC alone, specdec_realign_workspace_size(dtype, n_planes, n_rows, H, D,
 *   cap_src) with SPECDEC_SEGMENTED.  Calls that share a workspace must not run
 *   concurrently (stream-ordered calls are fine).  NULL: static assignment, no segments.
 * count_bound: the caller's upper bound on count[r] + count_add over all rows, or 0 for
 *   none (then cap_src).  Tight bounds let the host size the launch: slabs of at most
 *   4 KB (e.g. the pool write-back scatter, a + 1 <= k + 1 rows) are moved by a
 *   register-staged warp-per-slab kernel with every slab in flight at once instead of
 *   the TMA ring.  A row above the bound is skipped and sets SPECDEC_ST_BOUND.
 * d_moved_bytes: optional uint64 accumulator of bytes read + written by this call.
 */
size_t specdec_realign_workspace_size(int dtype, int64_t n_planes, int64_t n_rows, int64_t H,
                                      int64_t D, int64_t cap);
int specdec_realign_kv(const void *d_kv_src, void *d_kv_dst, int dtype, int64_t n_planes,
                       int64_t n_rows, int64_t H, int64_t D, int64_t src_s_plane,
                       int64_t src_s_row, int64_t src_s_head, int64_t cap_src,
                       int64_t dst_s_plane, int64_t dst_s_row, int64_t dst_s_head,
                       int64_t cap_dst, const int32_t *d_src_col, int32_t src_col_add,
                       const int32_t *d_dst_col, int32_t dst_col_add, const int32_t *d_count,
                       int32_t count_add, int32_t count_bound, const int32_t *d_src_row_map,
                       const int32_t *d_dst_row_map, uint32_t flags, void *d_ws,
                       size_t ws_bytes, unsigned long long *d_moved_bytes, uint32_t *d_status,
                       specdec_stream_t stream);

/* ------------------------------------------------------------------------------ a4
 * specdec_pool_group -- EXSpec GetBatch over a sliding window (Alg. 3 PAPER.md:488-494,
 * 508; §3.2; readings R11-R14):
 *
 *   window  = the first W sequence ids s of d_order[0..N) with d_active[s] (RefillWindow);
 *   lengths = d_len[s] (total tokens incl. the pending one; the grouping key, R13);
 *   distinct lengths are visited by (-count, length); each length's members, in window
 *   order, yield same-length batches of min(B, remaining) while remaining >= min_group
 *   (>= 1 when B == 1); leftovers, in window order, form fallback batches of B.
 *   bkind[b] = 1 iff all member lengths of batch b are equal.
 *
 * Outputs (nb_max = W batches at most):
 *   d_window [W], d_window_size [1]; d_batch_of, d_slot_of [N] (-1 if not in the window);
 *   d_members [W][B] sequence ids (-1 = empty slot); per slot: d_mlen [W][B] = len,
 *   d_mpad [W][B] = blen - len, d_mactive [W][B] (1 = real member) -- i.e. each batch's
 *   (n, p, active) arrays for specdec_verify / specdec_realign_kv;
 *   d_bsize, d_bkind, d_blen [W]; d_n_batches [1];
 *   d_counters [8] int64, ACCUMULATED (+=): {batches, same-length batches, members in
 *   same-length batches, members in fallback batches, fallback member tokens, window
 *   size, distinct lengths, deferred members (always 0 here; see _deferred)}.
 * Limits: 1 <= W <= 2048, 1 <= B <= W, 1 <= min_group; d_len values >= 1.
 */
int specdec_pool_group(const int32_t *d_len, const uint8_t *d_active, const int32_t *d_order,
                       int32_t N, int32_t W, int32_t B, int32_t min_group, int32_t *d_window,
                       int32_t *d_window_size, int32_t *d_batch_of, int32_t *d_slot_of,
                       int32_t *d_members, int32_t *d_mlen, int32_t *d_mpad,
                       uint8_t *d_mactive, int32_t *d_bsize, uint8_t *d_bkind,
                       int32_t *d_blen, int32_t *d_n_batches, int64_t *d_counters,
                       specdec_stream_t stream);

/* specdec_pool_group_deferred -- the epoch plan with deferred fallback (reading R27;
 * GetBatch "attempts to form batches of identical length" and falls
 * back to unpad-repad only when it cannot).  specdec_pool_group's plan, except: when its
 * group pass formed at least one same-length batch and patience > 0, a leftover s with
 * d_wait[s] < patience is deferred -- in the window (d_window), in no batch (d_batch_of[s]
 * = d_slot_of[s] = -1) -- and only the leftovers with d_wait[s] >= patience, in window
 * order, fill the fallback batches of B (numbered after the same-length ones).  With no
 * same-length batch every leftover runs, so a non-empty window always plans >= 1 batch.
 * d_wait [N] int32 (caller-owned, zeroed at admission) is updated in place: 0 for every
 * planned member, +1 for every deferred one, untouched outside the window; a member is
 * thus deferred at most `patience` epochs in a row.  d_counters[7] += deferred members.
 * patience == 0 is specdec_pool_group exactly (d_wait may then be NULL; if given, its
 * window entries are zeroed).
 * Pipelined fallback (reading R28; both NULL = off): d_epoch [1] int32 counts the plans
 * made (the call reads e = *d_epoch and stores e + 1); d_fb_epoch [N] int32 (caller-owned,
 * initialised to a value below -1) is the plan that last put each sequence in a
 * mixed-length batch.  A sequence with d_fb_epoch[s] == e - 1 is left out of the window:
 * its mixed batch of the previous plan may still be running (the caller runs mixed
 * batches beside the next plan); the members of this plan's mixed batches get
 * d_fb_epoch[s] = e.  d_len / d_active of an excluded sequence are not used.
 * Errors: as specdec_pool_group; SPECDEC_ERR_ARG for patience < 0, patience > 0 with
 * d_wait NULL, or exactly one of d_fb_epoch / d_epoch NULL.
 */
int specdec_pool_group_deferred(const int32_t *d_len, const uint8_t *d_active, const int32_t *d_order,
                                int32_t N, int32_t W, int32_t B, int32_t min_group, int32_t *d_wait,
                                int32_t patience, int32_t *d_fb_epoch, int32_t *d_epoch,
                                int32_t *d_window, int32_t *d_window_size,
                                int32_t *d_batch_of, int32_t *d_slot_of, int32_t *d_members,
                                int32_t *d_mlen, int32_t *d_mpad, uint8_t *d_mactive, int32_t *d_bsize,
                                uint8_t *d_bkind, int32_t *d_blen, int32_t *d_n_batches,
                                int64_t *d_counters, specdec_stream_t stream);

/* specdec_pool_getbatch -- Alg. 3's GetBatch(Window, B) as printed (ONE batch
 * per iteration): batch 0 of the specdec_pool_group plan, without planning the others.
 * Batch 0 is the first batch of the heaviest length group -- the largest count, ties to
 * the smaller length -- when that count reaches min_group (>= 1 when B == 1): its first
 * min(B, count) members in window order; otherwise the first min(B, |window|) members of
 * the window.  Same arguments as specdec_pool_group; outputs: d_window, d_window_size;
 * batch 0's row of d_members / d_mlen / d_mpad / d_mactive (B entries); d_bsize[0],
 * d_bkind[0], d_blen[0]; d_n_batches = 1 (0 for an empty window); d_batch_of / d_slot_of
 * = 0 / slot for batch 0's members, -1 for every other sequence; d_counters += the
 * counters of that one batch (window size and distinct lengths as specdec_pool_group).
 * Other batch rows are not written.  A window whose lengths span more than 8192 values
 * is planned in full (then batches >= 1 are written too).  specdec_pool_alg3 plans with
 * this call.
 */
int specdec_pool_getbatch(const int32_t *d_len, const uint8_t *d_active, const int32_t *d_order,
                          int32_t N, int32_t W, int32_t B, int32_t min_group, int32_t *d_window,
                          int32_t *d_window_size, int32_t *d_batch_of, int32_t *d_slot_of,
                          int32_t *d_members, int32_t *d_mlen, int32_t *d_mpad,
                          uint8_t *d_mactive, int32_t *d_bsize, uint8_t *d_bkind,
                          int32_t *d_blen, int32_t *d_n_batches, int64_t *d_counters,
                          specdec_stream_t stream);

/* ------------------------------------------------------------------------------ a5
 * specdec_pool_writeback -- Alg. 3 Phase 4: the pool-mode half of
 * the repad step.  For every batch slot r with d_members[r] = s >= 0:
 *   E_r = the first e_r tokens of draft[r][0:a_r] ++ [bonus_r], where
 *         e_r = min(emit_r, max_new - gen_s)  (the per-sequence budget);
 *   pool_tokens[s][len_s .. len_s+e_r) = E_r;  out_buf[s][gen_s .. gen_s+e_r) = E_r;
 *   len_s += e_r; gen_s += e_r;
 *   if finished_r or gen_s == max_new: active_s = 0 (isComplete -> Pool.deactivate).
 * The KV write-back is a specdec_realign_kv scatter (fallback batches only: same-length
 * batches were served zero-copy from the pool).
 * d_pool_tokens [N][cap_tok] int64, d_out_buf [N][max_new] int64 (either may be NULL);
 * max_new >= 1.  Pass d_budget = NULL to specdec_verify in pool mode.
 * d_status: SPECDEC_ST_CAPACITY on overflow (row skipped).
 */
int specdec_pool_writeback(const int32_t *d_members, int64_t B, int64_t k,
                           const int64_t *d_draft, const int32_t *d_accept,
                           const int64_t *d_bonus,
                           const int32_t *d_emit, const uint8_t *d_finished,
                           int32_t *d_pool_len, int32_t *d_pool_gen, uint8_t *d_pool_active,
                           int64_t *d_pool_tokens, int64_t cap_tok, int64_t *d_out_buf,
                           int64_t max_new, uint32_t *d_status, specdec_stream_t stream);

/* ------------------------------------------------------------------------------ a1 + a5
 * specdec_pool_verify -- one EXSpec batch's Alg. 1 BatchVerify with
 * the Alg. 3 Phase 4 write-back fused into its epilogue: exactly
 * specdec_verify(n = d_mlen, active = d_mactive, budget = NULL, no plan outputs) followed
 * by specdec_pool_writeback(d_members, ...), with the write-back inside K1's epilogue (the
 * pool's per-batch path is latency-bound: one dependent kernel fewer per batch).
 * Arguments as in those two calls; d_mlen / d_mactive / d_members are one batch's rows of
 * specdec_pool_group's outputs.  Errors: as specdec_verify (logits / shape / workspace)
 * and specdec_pool_writeback (pool pointers, cap_tok, max_new); SPECDEC_ST_CAPACITY if a
 * pool token row would overflow (that row's write-back is skipped).
 */
int specdec_pool_verify(const void *d_logits, int dtype, int64_t B, int64_t k, int64_t V,
                        int64_t row_stride, const int64_t *d_draft, const int32_t *d_members,
                        const int32_t *d_mlen, uint8_t *d_mactive, int64_t eos_id,
                        int64_t pad_id, int32_t *d_accept, int64_t *d_bonus, int32_t *d_emit,
                        uint8_t *d_finished, int32_t *d_pool_len, int32_t *d_pool_gen,
                        uint8_t *d_pool_active, int64_t *d_pool_tokens, int64_t cap_tok,
                        int64_t *d_out_buf, int64_t max_new, uint32_t *d_status, void *d_ws,
                        size_t ws_bytes, specdec_stream_t stream);

/* specdec_pool_verify_group -- specdec_pool_verify over n_batches (1..SPECDEC_MAX_VERIFY_GROUP) batches of one
 * epoch plan in ONE launch (reading R21: the batches of one plan have disjoint members and
 * are planned from one window state, so verifying them together changes no result; the
 * executor calls each batch's forward first).  Batch g: logits h_logits[g] [h_rows[g]][k+1]
 * [row_stride] and drafts h_draft[g] [h_rows[g]][k] (device pointers held in HOST arrays),
 * member rows d_members / d_mlen / d_mactive [h_offset[g] .. h_offset[g] + h_rows[g]) (the
 * plan arrays, e.g. offset = plan batch index x B).  Per-row outputs d_accept, d_bonus,
 * d_emit, d_finished are flat over the R = sum h_rows rows in group order; d_ws holds
 * specdec_verify_workspace_size(R, k) bytes.  Everything else as specdec_pool_verify.
 * Errors: SPECDEC_ERR_ARG for n_batches outside [1, 16] or a NULL / misaligned pointer;
 * SPECDEC_ERR_SHAPE for h_rows[g] < 1 or the shape errors of specdec_pool_verify.
 */
int specdec_pool_verify_group(int32_t n_batches, const void *const *h_logits,
                              const int64_t *const *h_draft, const int32_t *h_offset,
                              const int32_t *h_rows, int dtype, int64_t k, int64_t V,
                              int64_t row_stride, const int32_t *d_members, const int32_t *d_mlen,
                              uint8_t *d_mactive, int64_t eos_id, int64_t pad_id,
                              int32_t *d_accept, int64_t *d_bonus, int32_t *d_emit,
                              uint8_t *d_finished, int32_t *d_pool_len, int32_t *d_pool_gen,
                              uint8_t *d_pool_active, int64_t *d_pool_tokens, int64_t cap_tok,
                              int64_t *d_out_buf, int64_t max_new, uint32_t *d_status, void *d_ws,
                              size_t ws_bytes, specdec_stream_t stream);

/* ------------------------------------------------------------------------------ a4 + a5
 * specdec_pool_epoch -- native EXSpec epoch executor (Alg. 3): the
 * host-side launch loop of one epoch in C++ instead of one Python call per kernel.
 *   specdec_pool_group over the window; a device->host copy of the plan header (the
 *   epoch's only host synchronisation: ONE copy if n_batches, bkind, blen and bsize are laid
 *   out like host_header in one buffer -- bkind's W bytes in the W int32 slots after
 *   n_batches, then blen, then bsize -- else four); then for each of the first `max_batches` planned
 *   batches (<= 0: all; 1: Alg. 3 as printed -- GetBatch, verify, write-back, re-plan):
 *     fallback batch: specdec_realign_kv gather (pool -> staging, right-aligned);
 *     inputs: `forward(ctx, b, same_length, width, &logits, &draft)` if non-NULL (the
 *       model's verify forward, enqueued on `stream`), else the next (logits, draft) of
 *       the descriptor's input ring;
 *     specdec_verify (no budget; the write-back applies max_new); specdec_pool_writeback;
 *     fallback batch: specdec_realign_kv scatter of the a+1 new KV rows.
 *   With desc->n_staging >= 2 the fallback gathers are overlapped with the same-length
 *   batches (see the descriptor's last fields); results are identical.
 * Errors: SPECDEC_ERR_ARG for a NULL desc / header, W or B < 1, no input ring without a
 * forward callback, or an incomplete overlap configuration (ring, stream or events
 * missing); any error of the calls it makes is returned as is.
 * Host outputs (nullable): batches run, same-length batches run, their members, and
 * the members of the fallback batches run.  All device buffers are caller-owned
 * (paper_2510_22876_b200/exspec.py allocates them); host_header is pinned, 1 + 3W int32.
 */
typedef void (*specdec_forward_fn)(void *ctx, int32_t batch, int32_t same_length /* KV in the pool slots */,
                                   int32_t width, const void **logits, const int64_t **draft);

typedef struct specdec_pool_desc {
    /* pool state */
    int32_t *len, *gen;
    uint8_t *active;
    const int32_t *order;
    int32_t N;
    int64_t *tokens;   /* [N][cap_tok] or NULL */
    int64_t cap_tok;
    int64_t *out_buf;  /* [N][max_new] or NULL */
    int64_t max_new;
    void *kv;          /* [N][n_planes][H][cap][D] */
    void *staging;     /* [n_planes][B][H][cap][D] */
    int kv_dtype;
    int64_t n_planes, H, D, cap;
    /* K4 plan buffers (see specdec_pool_group) */
    int32_t *window, *window_size, *batch_of, *slot_of, *members, *mlen, *mpad;
    uint8_t *mactive;
    int32_t *bsize;
    uint8_t *bkind;
    int32_t *blen, *n_batches;
    int64_t *counters;
    /* specdec_verify scratch, [B] each (plan_L [1]) */
    int32_t *accept;
    int64_t *bonus;
    int32_t *emit;
    uint8_t *finished;
    int32_t *n_new, *pad_new, *kept, *plan_L;
    void *ws;
    size_t ws_bytes;
    uint32_t *status;
    unsigned long long *moved;
    int32_t *host_header; /* pinned host, 1 + 3W int32 */
    int32_t W, B, min_group;
    int64_t k, V, logit_stride, eos_id, pad_id;
    int logit_dtype;
    /* input ring used when forward == NULL: logits [B][k+1][logit_stride], drafts [B][k] */
    const void *const *logits_ring;
    const int64_t *const *draft_ring;
    int32_t ring_n;
    int32_t *ring_pos; /* host, advanced per batch */
    /* The consumer of a batch's KV (the model's verify forward):
     * 0: a dense right-aligned rectangle -- mixed-length batches are gathered into the
     *    staging (realigned) and scattered back; same-length batches run zero-copy on the
     *    pool slots (lazy realignment);
     * 1: a dense rectangle for every batch, same-length ones too ("concatenate directly",
     *    PAPER.md:537);
     * 2: slot-indexed (e.g. a variable-length attention reading each member's KV rows
     *    [0, len-1) in its own slot and appending at column len-1): no batch moves KV
     *    ("slot-indexed zero-copy consumer").
     * The forward callback's `same_length` argument is 1 when the batch's KV is in the pool
     * slots, 0 when it is in the staging. */
    int32_t dense_consumer;
    /* Overlapped fallback gathers (n_staging >= 2; 0 or 1 = off, the serial loop above).
     * The batches of one epoch have disjoint members and are planned from one window
     * state, so the order they run in does not change any result (the input-ring slot of
     * batch b stays ring_pos + b).  With overlap on, every fallback batch's gather runs on
     * `copy_stream` into staging_ring[f % n_staging] (f = its rank among the epoch's
     * fallback batches), and the fallback batches are interleaved with the same-length
     * ones on `stream` by a list schedule on the estimates below (a fallback batch runs
     * as soon as its gather is expected to be complete), so the bandwidth-bound gathers
     * stream under the latency-bound same-length verifies.  The scatters run on
     * `copy_stream` too.  Ordering: the verify of fallback batch f waits for its gather
     * (events[f % n_staging]); its scatter waits for that verify (events[n_staging +
     * f % n_staging]) and reads the batch's accept lengths from accept_ring[f % n_staging];
     * the gather of f + n_staging follows that scatter in copy-stream order; `stream`
     * waits for the copy stream at the end, so the epoch is complete when `stream` is.
     * The caller owns the buffers and the
     * 2 * n_staging events (cudaEvent_t, timing disabled).  staging_ring[0] may be
     * `staging`.  If `cur_staging` is non-NULL the executor stores the staging buffer of
     * a fallback batch there before calling forward() (NULL for same-length batches). */
    int32_t n_staging;
    void *const *staging_ring; /* host array of n_staging device pointers, layout of `staging` */
    specdec_stream_t copy_stream;
    void *const *events;       /* host array of 2 * n_staging cudaEvent_t */
    void **cur_staging;        /* host, nullable */
    int32_t *accept_ring;      /* device [n_staging][B]: accept lengths of the fallback batch in each slot */
    /* scheduling hints for the overlapped order (<= 0: 5500 GB/s, 10 us): the gather rate
     * and the duration of one batch verify; they change the order, never a result */
    double est_gather_GBps, est_verify_us;
    /* optional >= 128-byte zeroed workspace: the fallback gathers take SPECDEC_DYNAMIC
     * work tickets from it (they run one after another on one stream); NULL = static */
    void *gather_ws;
    /* same-length batches verified per launch (specdec_pool_verify_group, <= SPECDEC_MAX_VERIFY_GROUP); <= 1:
     * one specdec_pool_verify per batch.  Runs of same-length batches in the processing
     * order are grouped; forward() is called for every batch of a group before the group's
     * verify, so the buffers it returns must stay valid until then.  Needs `ws` of
     * specdec_verify_workspace_size(verify_group * B, k) bytes (else no grouping) and
     * accept / bonus / emit / finished of verify_group * B entries. */
    int32_t verify_group;
    int64_t *host_launches;    /* host, nullable: += the libspecdec kernels the call launched */
    /* optional third stream for the scatters (n_staging >= 2): scatter f waits for its
     * verify and runs beside the copy stream's gathers (epoch batches have disjoint members,
     * so a scatter and another batch's gather touch disjoint pool rows and staging slots);
     * the gather of f + n_staging waits for scatter f (scatter_events[f % n_staging]).
     * NULL: the scatters run on copy_stream as above.  scatter_events: host array of
     * n_staging cudaEvent_t (timing disabled). */
    specdec_stream_t scatter_stream;
    void *const *scatter_events;
    /* deferred fallback (R27): patience > 0 plans each epoch with
     * specdec_pool_group_deferred on `wait` (device [N] int32, zeroed at admission);
     * 0 = specdec_pool_group.  Alg. 3 as printed (max_batches 1, specdec_pool_alg3) is
     * unaffected: its GetBatch already falls back only when no group qualifies. */
    int32_t *wait;
    int32_t patience;
    /* pipelined fallback (reading R28), pipeline = 1: each call makes ONE plan
     * (specdec_pool_group_deferred with fb_epoch / plan_epoch), verifies its same-length
     * batches on `stream` and runs its mixed-length batches -- gather, verify + write-back,
     * scatter -- on copy_stream into staging_ring[i % n_staging], returning without waiting
     * for them; the next plan leaves their members out, the one after waits for them
     * (pipe_events).  The plan rows alternate between two halves: members / mlen / mpad /
     * mactive must hold 2W batch rows.  Requires forward == NULL, max_batches <= 0,
     * dense_consumer == 0, the packed plan header, n_staging >= 1 with staging_ring and
     * copy_stream, accept_ring.  A call that plans nothing while mixed batches are in flight
     * waits for them and plans again; a call returning 0 batches leaves the pool drained
     * and `stream` after every chain.  Results equal the oracle's R28 drain. */
    int32_t pipeline;
    int32_t *fb_epoch;     /* device [N], initialised below -1 at admission */
    int32_t *plan_epoch;   /* device [1], 0 at admission */
    void *ws2;             /* specdec_verify workspace of the copy stream's verifies */
    size_t ws2_bytes;
    int64_t *bonus2;       /* device [B]: their bonus / emit / finished scratch */
    int32_t *emit2;
    uint8_t *finished2;
    void *const *pipe_events; /* host array of 2 cudaEvent_t (timing disabled) */
    int64_t *pipe_host;    /* host [2]: plans made, mixed batches of the last plan; 0 at admission */
} specdec_pool_desc;

int specdec_pool_epoch(const specdec_pool_desc *d, specdec_forward_fn forward, void *ctx,
                       int32_t max_batches, int32_t *h_ran, int32_t *h_same,
                       int32_t *h_members_same, int32_t *h_members_fallback,
                       specdec_stream_t stream);

/* ------------------------------------------------------------------------------ a1-a3
 * specdec_eqspec_round -- one whole EqSpec round after the verify forward (Alg. 2's loop
 * body): specdec_verify -> specdec_rebuild_pos_mask ->
 * specdec_realign_kv (target cache, then the draft cache if any), enqueued on `stream`
 * with no host synchronisation, exactly the calls paper_2510_22876_b200/eqspec.py makes.
 * The batch state is double-buffered by `parity` p: the round reads n[p], pad[p],
 * tokens[p] and writes n[1-p], pad[1-p], tokens[1-p]; its results go to the result set
 * of parity p (accept[p], ...), so a reader of round r's results (e.g. a D2H on another
 * stream) only has to finish before round r+2.  KV: kv[0] == kv[1] realigns in place;
 * two buffers ping-pong (round p reads kv[p], writes kv[1-p]).  B == 1 in place moves no
 * KV (a single row stays right-aligned): no realign launch (unless the
 * anchored origin (f3) is on: then the realign follows K1's physical columns).
 * Errors: SPECDEC_ERR_ARG for a NULL desc / logits / draft or parity not 0/1; any error of
 * the three calls as is.
 */
typedef struct specdec_round_desc {
    int64_t B, k, V, logit_stride;
    int logit_dtype;
    int64_t eos_id, pad_id;
    /* per-row state, [2] = by parity */
    int32_t *n[2], *pad[2];
    int64_t *tokens[2];        /* [B][cap_tok] each */
    int64_t cap_tok;
    int64_t *mask, *pos;       /* [B][mp_stride] */
    int64_t mp_stride;
    uint8_t *active;           /* [B] in/out */
    int32_t *budget;           /* [B] in/out remaining new tokens, or NULL */
    int32_t *gen;              /* [B], with out_buf, or NULL */
    int64_t *out_buf;          /* [B][max_new] or NULL */
    int64_t max_new;
    /* results, one set per parity */
    int32_t *accept[2], *emit[2];
    int64_t *bonus[2];
    uint8_t *finished[2];
    int64_t *pred;             /* [B][k+1] or NULL */
    int32_t *kept, *plan_L, *kept_draft /* NULL unless a draft cache */;
    void *ws;                  /* specdec_verify workspace */
    size_t ws_bytes;
    uint32_t *status;
    unsigned long long *moved;
    /* target KV [planes][B][H][cap_kv][D] (element strides s_plane, s_row, s_head) */
    void *kv[2];
    int kv_dtype;
    int64_t n_planes, H, D, cap_kv, s_plane, s_row, s_head;
    /* draft-model KV (f1), same layout rules; dkv[0] == NULL: none */
    void *dkv[2];
    int64_t d_planes, d_H, d_D, d_s_plane, d_s_row, d_s_head;
    /* realign: SPECDEC_ZERO_PADS / SPECDEC_OVERLAP_PREV / SPECDEC_DYNAMIC /
     * SPECDEC_SEGMENTED for the target call (the draft call takes all but OVERLAP_PREV);
     * the workspace both calls share, stream-ordered (see specdec_realign_kv) */
    uint32_t realign_flags;
    void *realign_ws;
    size_t realign_ws_bytes;
    /* anchored origin (f3, see specdec_verify): anchor [1] in/out, NULL = off; the realign
     * then moves KV from phys_old to phys_new columns (cap_kv is the physical capacity) */
    int32_t *anchor, *phys_old, *phys_new;
} specdec_round_desc;

int specdec_eqspec_round(const specdec_round_desc *d, int parity, const void *d_logits,
                         const int64_t *d_draft, specdec_stream_t stream);

/* specdec_eqspec_round_host -- the same round from HOST inputs, with the host<->device
 * copies inside the call (the end-to-end path of a caller whose logits live in host
 * memory).  On `io->copy_stream`: wait io->ev_done[slot] (the last round that read
 * staging slot `slot`), copy h_logits [B][k+1][logit_stride] and h_draft [B][k] (pinned
 * host memory, for the copies to be asynchronous) into io->d_logits[slot] /
 * io->d_draft[slot], record io->ev_ready[slot].  On `stream`: wait ev_ready[slot] and
 * io->ev_fetched[parity] (the read-out of the result set this round overwrites), run
 * specdec_eqspec_round, record ev_done[slot].  If h_emit (pinned [B] int32) is non-NULL:
 * on io->d2h_stream wait ev_done[slot], copy emit[parity] -> h_emit, record
 * ev_fetched[parity].  If the caller sets io->inputs_packed (the drafts directly follow
 * the logits in ONE pinned allocation) and the slot's staging is laid out the same way,
 * the inputs go in one copy instead of two.  (Adjacency alone is not enough: two separate
 * pinned allocations can be adjacent, and one copy may not span both.)  Nothing synchronises the host: successive calls with the slot
 * cycling through n_slots and the parity alternating overlap the copies of the next
 * rounds with this one.  With n_slots = 3 the copy of round r starts when round r-3 is
 * done, two rounds ahead of its use, which absorbs the occasional slow H2D (measured at
 * Qwen3 B=8: 280 us median, up to 2 ms; 2 slots 2158 -> 3 slots 2241 rounds/s).  The
 * events are the caller's (cudaEvent_t, timing disabled; a never-recorded event does not
 * block).
 * Errors: as specdec_eqspec_round; SPECDEC_ERR_ARG for a NULL io / host pointer, n_slots
 * outside [2, SPECDEC_HOST_SLOTS] or slot >= n_slots; SPECDEC_ERR_CUDA for a failed copy
 * or event call.
 */
#define SPECDEC_HOST_SLOTS 4
typedef struct specdec_host_io {
    int32_t n_slots;           /* staging slots in use, 2..SPECDEC_HOST_SLOTS; `slot` < n_slots */
    void *d_logits[SPECDEC_HOST_SLOTS];    /* device staging, [B][k+1][logit_stride] each */
    int64_t *d_draft[SPECDEC_HOST_SLOTS];  /* device staging, [B][k] each */
    specdec_stream_t copy_stream, d2h_stream;
    void *ev_ready[SPECDEC_HOST_SLOTS], *ev_done[SPECDEC_HOST_SLOTS];
    void *ev_fetched[2];       /* per result parity */
    int32_t inputs_packed;     /* per call: 1 = h_draft directly follows h_logits in the SAME
                                * pinned allocation (one copy); 0 = two copies */
} specdec_host_io;

int specdec_eqspec_round_host(const specdec_round_desc *d, const specdec_host_io *io,
                              int parity, int slot, const void *h_logits,
                              const int64_t *h_draft, int32_t *h_emit,
                              specdec_stream_t stream);

/* specdec_pool_alg3 -- `iterations` iterations of Alg. 3 as printed:
 * specdec_pool_getbatch over the window (batch 0 of the plan only; d->counters accumulate
 * that batch's counters), then that batch (gather if it is a
 * fallback batch, specdec_pool_verify with the write-back, scatter), then re-plan -- all
 * enqueued on `stream` with NO host synchronisation: the plan kernel's tail writes batch
 * 0 as gated member rows for the gather / verify / scatter (-1 or inactive for the parts
 * that must not run).  Iterations after the pool drains are no-ops;
 * the caller checks `active` between calls.  Inputs come from the descriptor's ring (one
 * slot per iteration); the staging is `staging`; `gather_ws` as in specdec_pool_epoch.
 * d_scratch: device int32 [4 * B] (caller-owned, contents don't-care).
 * d_exec_counters: optional device uint64 [4] accumulating executed batches, same-length
 * batches, their members, fallback members.
 * Errors: SPECDEC_ERR_ARG for a NULL desc / scratch, W or B < 1, B > 1024, no input ring,
 * iterations < 0; any error of the calls it makes as is.
 */
int specdec_pool_alg3(const specdec_pool_desc *d, int32_t iterations, int32_t *d_scratch,
                      unsigned long long *d_exec_counters, specdec_stream_t stream);

/* specdec_pool_alg3_graph -- `iterations` iterations of specdec_pool_alg3's loop built as
 * ONE CUDA graph (instantiated; *graph_exec receives the cudaGraphExec_t).
 *   conditional = 0: the iterations exactly as specdec_pool_alg3 enqueues them (gated
 *     no-op gathers / scatters included), captured with their PDL edges -- the host issues
 *     one graph launch instead of 4 x iterations kernel launches;
 *   conditional = 1: per iteration the GetBatch kernel, the gather in a conditional (IF)
 *     node, the verify with the write-back, the scatter in an IF node; GetBatch sets the
 *     conditions to "batch 0 moves KV" (cudaGraphSetConditional), so a same-length
 *     iteration launches nothing for its KV moves -- but measured slower on B200 (the IF
 *     nodes cost more than the no-op launches they remove, and break the PDL chain):
 *     Alg. 3 pool 3162 (direct) -> 2225 seq/s; kept for the record.
 * With the slot-indexed consumer (dense_consumer = 2) there are no KV launches at all.
 * Input-ring slots are bound
 * at build time: iteration i uses slot (ring_pos + i) % ring_n and *ring_pos advances by
 * `iterations` -- build ring_n iterations and every launch continues the slot sequence.
 * Launch with specdec_graph_launch (any stream), release with specdec_graph_destroy.  The
 * descriptor's buffers and d_scratch / d_exec_counters must outlive the graph.  Results
 * equal specdec_pool_alg3 (tests/test_gpu_pool.py).
 * Errors: as specdec_pool_alg3; SPECDEC_ERR_CUDA if the graph cannot be built.
 */
int specdec_pool_alg3_graph(const specdec_pool_desc *d, int32_t iterations, int32_t *d_scratch,
                            unsigned long long *d_exec_counters, int32_t conditional, void **graph_exec);
int specdec_graph_launch(void *graph_exec, specdec_stream_t stream);
int specdec_graph_destroy(void *graph_exec);

#ifdef __cplusplus
}
#endif
#endif /* SPECDEC_H_ */
