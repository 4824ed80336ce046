// pool_exec.cu -- native EXSpec epoch executor (host C++): the per-batch launch loop of
// Alg. 3 without a Python round trip per kernel.
//
// One call = K4 plan of the window, one small D2H of the plan header (the epoch's only
// host synchronisation), then for every planned batch (or only batch 0: Alg. 3 as printed):
//   fallback batches:  specdec_realign_kv gather (pool -> right-aligned staging)
//   forward callback   (the model's verify forward; may be NULL for synthetic inputs)
//   specdec_pool_verify (Alg. 1 + the Phase 4 write-back in one launch; logits / drafts
//                       from the callback or from the input ring)
//   fallback batches:  specdec_realign_kv scatter (the a+1 new KV rows back to the pool)
// Every launch goes through the same C ABI entry points the Python driver uses.
// With n_staging >= 2 (specdec.h) the fallback batches' gathers and scatters run on a
// copy stream into a ring of staging buffers, interleaved by a list schedule with the
// same-length batches' verifies on the main stream (reading R21: the batches of one plan
// are independent, so their order cannot change a result).
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <vector>

#include "common.cuh"
#include "host_util.h"
#include "pool_gate.h"
#include "specdec.h"

using namespace specdec;

// ---- Pipelined fallback (reading R28; specdec_pool_desc.pipeline): one plan per call, its
// same-length batches verified on `stream` (grouped), its mixed-length batches -- gather,
// verify + write-back, scatter, in plan order -- on the copy stream, left running when the
// call returns.  The next plan leaves their members out (K4's fb_epoch stamp), so it need
// not wait for them; the plan after it waits (pipe_events[parity], recorded after the
// chain) before their members rejoin.  Plans alternate between two halves of the plan
// rows (members / mlen / mpad / mactive are [2W][B]), so a running chain's rows are never
// overwritten by the next plan.  Plan e's rows and pipe_events slot: e % 2 (pipe_host[0]
// = plans made, pipe_host[1] = mixed batches of the last plan).
static int pool_epoch_pipelined(const specdec_pool_desc *d, int32_t *h_ran, int32_t *h_same,
                                int32_t *h_members_same, int32_t *h_members_fallback, specdec_stream_t stream) {
    const int32_t W = d->W, B = d->B;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(d->copy_stream);
    auto pev = [&](int64_t e) { return reinterpret_cast<cudaEvent_t>(d->pipe_events[e & 1]); };
    const int64_t hcd = d->H * d->cap * d->D;
    const int64_t p_plane = hcd, p_row = d->n_planes * hcd, p_head = d->cap * d->D;
    const int64_t s_plane = B * hcd, s_row = hcd, s_head = d->cap * d->D;
    int32_t G = std::min<int32_t>(std::max<int32_t>(d->verify_group, 1), SPECDEC_MAX_VERIFY_GROUP);
    while (G > 1 && specdec_verify_workspace_size(static_cast<int64_t>(G) * B, d->k) > d->ws_bytes) --G;
    const int kv1 = specdec_verify_kernels(1);
    int64_t launches = 0;
    cudaError_t e;
    int rc;
    for (;;) {
        const int64_t ep = d->pipe_host[0];
        const int64_t off = (ep & 1) * static_cast<int64_t>(W) * B;
        int32_t *members = d->members + off, *mlen = d->mlen + off, *mpad = d->mpad + off;
        uint8_t *mactive = d->mactive + off;
        // the chain of plan ep - 2 used these rows and its members rejoin now
        if (ep >= 2 && (e = cudaStreamWaitEvent(s, pev(ep), 0)) != cudaSuccess) return record_cuda_error(e);
        rc = specdec_pool_group_deferred(d->len, d->active, d->order, d->N, W, B, d->min_group, d->wait,
                                         d->patience, d->fb_epoch, d->plan_epoch, d->window, d->window_size,
                                         d->batch_of, d->slot_of, members, mlen, mpad, mactive, d->bsize,
                                         d->bkind, d->blen, d->n_batches, d->counters, stream);
        if (rc) return rc;
        ++launches;
        int32_t *hh = d->host_header;
        e = cudaMemcpyAsync(hh, d->n_batches, (1 + 3 * static_cast<size_t>(W)) * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return record_cuda_error(e);
        d->pipe_host[0] = ep + 1;
        const int32_t nb = hh[0];
        const uint8_t *kinds = reinterpret_cast<const uint8_t *>(hh + 1);
        const int32_t *blens = hh + 1 + W, *sizes = hh + 1 + 2 * W;
        if (nb == 0) {
            const int64_t prev_mixed = d->pipe_host[1];
            d->pipe_host[1] = 0;
            // every active sequence may be in the last plan's mixed batches: let them finish
            // (this call's plan stamped nobody, so the next one plans them), then plan again;
            // with none in flight the pool is drained -- the call ends with the copy stream
            if ((e = cudaEventRecord(pev(ep), cs)) != cudaSuccess || (e = cudaStreamWaitEvent(s, pev(ep), 0)) != cudaSuccess)
                return record_cuda_error(e);
            if (prev_mixed > 0) continue;
            if (d->host_launches) *d->host_launches += launches;
            if (h_ran) *h_ran = 0;
            if (h_same) *h_same = 0;
            if (h_members_same) *h_members_same = 0;
            if (h_members_fallback) *h_members_fallback = 0;
            return SPECDEC_OK;
        }
        const int32_t ring_base = *d->ring_pos;
        auto rows = [&](int32_t b) -> int32_t { return sizes[b] > 0 && sizes[b] < B ? sizes[b] : B; };
        int32_t same = 0, msame = 0, mfb = 0, n_mixed = 0;
        // same-length batches: grouped verifies on `stream`, in plan order
        const void *g_lg[SPECDEC_MAX_VERIFY_GROUP] = {};
        const int64_t *g_dr[SPECDEC_MAX_VERIFY_GROUP] = {};
        int32_t g_off[SPECDEC_MAX_VERIFY_GROUP] = {}, g_rows[SPECDEC_MAX_VERIFY_GROUP] = {};
        int32_t ng = 0;
        auto flush = [&]() -> int {
            if (!ng) return SPECDEC_OK;
            const int r = specdec_pool_verify_group(ng, g_lg, g_dr, g_off, g_rows, d->logit_dtype, d->k, d->V,
                                                    d->logit_stride, members, mlen, mactive, d->eos_id, d->pad_id,
                                                    d->accept, d->bonus, d->emit, d->finished, d->len, d->gen,
                                                    d->active, d->tokens, d->cap_tok, d->out_buf, d->max_new,
                                                    d->status, d->ws, d->ws_bytes, stream);
            launches += kv1;
            ng = 0;
            return r;
        };
        for (int32_t b = 0; b < nb; ++b) {
            const int32_t j = (ring_base + b) % d->ring_n;
            if (kinds[b]) {
                ++same;
                msame += sizes[b];
                g_lg[ng] = d->logits_ring[j];
                g_dr[ng] = d->draft_ring[j];
                g_off[ng] = static_cast<int32_t>(static_cast<int64_t>(b) * B);
                g_rows[ng] = rows(b);
                if (++ng == G && (rc = flush())) return rc;
                continue;
            }
            // a mixed batch: its whole chain on the copy stream (stream order frees the
            // staging buffer and the side verify's scratch for the next one)
            mfb += sizes[b];
            const int64_t o = static_cast<int64_t>(b) * B;
            void *stg = d->staging_ring[n_mixed % d->n_staging];
            ++n_mixed;
            rc = specdec_realign_kv(d->kv, stg, d->kv_dtype, d->n_planes, rows(b), d->H, d->D, p_plane, p_row,
                                    p_head, d->cap, s_plane, s_row, s_head, d->cap, nullptr, 0, mpad + o, 0,
                                    mlen + o, -1, 0, members + o, nullptr, d->gather_ws ? SPECDEC_DYNAMIC : 0u,
                                    d->gather_ws, d->gather_ws ? 128 : 0, d->moved, d->status,
                                    reinterpret_cast<specdec_stream_t>(cs));
            if (rc) return rc;
            rc = specdec_pool_verify(d->logits_ring[j], d->logit_dtype, rows(b), d->k, d->V, d->logit_stride,
                                     d->draft_ring[j], members + o, mlen + o, mactive + o, d->eos_id, d->pad_id,
                                     d->accept_ring, d->bonus2, d->emit2, d->finished2, d->len, d->gen,
                                     d->active, d->tokens, d->cap_tok, d->out_buf, d->max_new, d->status,
                                     d->ws2, d->ws2_bytes, reinterpret_cast<specdec_stream_t>(cs));
            if (rc) return rc;
            rc = specdec_realign_kv(stg, d->kv, d->kv_dtype, d->n_planes, rows(b), d->H, d->D, s_plane, s_row,
                                    s_head, d->cap, p_plane, p_row, p_head, d->cap, nullptr, blens[b] - 1,
                                    mlen + o, -1, d->accept_ring, 1, static_cast<int32_t>(d->k + 1), nullptr,
                                    members + o, 0, nullptr, 0, d->moved, d->status,
                                    reinterpret_cast<specdec_stream_t>(cs));
            if (rc) return rc;
            launches += 2 + kv1;
        }
        if ((rc = flush())) return rc;
        // the chain's completion, waited on by the plan after next (and at the drain's end)
        if ((e = cudaEventRecord(pev(ep), cs)) != cudaSuccess) return record_cuda_error(e);
        d->pipe_host[1] = n_mixed;
        *d->ring_pos = ring_base + nb;
        if (d->host_launches) *d->host_launches += launches;
        if (h_ran) *h_ran = nb;
        if (h_same) *h_same = same;
        if (h_members_same) *h_members_same = msame;
        if (h_members_fallback) *h_members_fallback = mfb;
        return SPECDEC_OK;
    }
}

extern "C" int specdec_pool_epoch(const specdec_pool_desc *d, specdec_forward_fn forward,
                                  void *ctx, int32_t max_batches, int32_t *h_ran,
                                  int32_t *h_same, int32_t *h_members_same,
                                  int32_t *h_members_fallback, specdec_stream_t stream) {
    if (!d || !d->host_header || d->W < 1 || d->B < 1) return SPECDEC_ERR_ARG;
    if (!forward && (!d->logits_ring || !d->draft_ring || d->ring_n < 1 || !d->ring_pos))
        return SPECDEC_ERR_ARG;
    if (d->n_staging >= 2 && (!d->staging_ring || !d->copy_stream || !d->events || !d->accept_ring))
        return SPECDEC_ERR_ARG;
    if (d->n_staging >= 2)
        for (int32_t i = 0; i < d->n_staging; ++i)
            if (!d->staging_ring[i] || !d->events[i] || !d->events[d->n_staging + i] ||
                (d->scatter_stream && (!d->scatter_events || !d->scatter_events[i])))
                return SPECDEC_ERR_ARG;
    if (d->pipeline) {
        // R28: ring inputs, the paper's consumer, a copy stream and its staging ring, the
        // side verify's own workspace / scratch, the events and the host state
        if (forward || max_batches > 0 || d->dense_consumer != 0 || d->n_staging < 1 || !d->staging_ring ||
            !d->copy_stream || !d->fb_epoch || !d->plan_epoch || !d->ws2 || !d->bonus2 || !d->emit2 ||
            !d->finished2 || !d->accept_ring || !d->pipe_events || !d->pipe_events[0] || !d->pipe_events[1] ||
            !d->pipe_host)
            return SPECDEC_ERR_ARG;
        const int32_t W = d->W;  // the packed plan header (one D2H copy)
        if (reinterpret_cast<const char *>(d->bkind) != reinterpret_cast<const char *>(d->n_batches + 1) ||
            d->blen != d->n_batches + 1 + W || d->bsize != d->n_batches + 1 + 2 * W)
            return SPECDEC_ERR_ARG;
        return pool_epoch_pipelined(d, h_ran, h_same, h_members_same, h_members_fallback, stream);
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int32_t W = d->W, B = d->B;
    // the epoch plan: R11's whole-window plan, or with d->patience > 0 the deferred-fallback
    // plan (R27: leftovers wait up to `patience` epochs for a same-length partner)
    int rc = d->patience > 0
        ? specdec_pool_group_deferred(d->len, d->active, d->order, d->N, W, B, d->min_group, d->wait,
                                      d->patience, nullptr, nullptr, d->window, d->window_size, d->batch_of, d->slot_of,
                                      d->members, d->mlen, d->mpad, d->mactive, d->bsize, d->bkind, d->blen,
                                      d->n_batches, d->counters, stream)
        : specdec_pool_group(d->len, d->active, d->order, d->N, W, B, d->min_group, d->window,
                             d->window_size, d->batch_of, d->slot_of, d->members, d->mlen,
                             d->mpad, d->mactive, d->bsize, d->bkind, d->blen, d->n_batches,
                             d->counters, stream);
    if (rc) return rc;
    // plan header -> pinned host: n_batches, kind, width, size (W each)
    int32_t *hh = d->host_header;
    cudaError_t e;
    // one copy when the four device arrays are laid out like host_header in one buffer
    // (n_batches, bkind in the next W int32 slots, blen, bsize), else four
    const bool packed = reinterpret_cast<const char *>(d->bkind) == reinterpret_cast<const char *>(d->n_batches + 1) &&
                        d->blen == d->n_batches + 1 + W && d->bsize == d->n_batches + 1 + 2 * W;
    if (packed) {
        e = cudaMemcpyAsync(hh, d->n_batches, (1 + 3 * static_cast<size_t>(W)) * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, s);
    } else {
        e = cudaMemcpyAsync(hh, d->n_batches, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hh + 1 + W, d->blen, W * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hh + 1 + 2 * W, d->bsize, W * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(reinterpret_cast<uint8_t *>(hh + 1), d->bkind, W, cudaMemcpyDeviceToHost, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return record_cuda_error(e);
    const int32_t nb = hh[0];
    const uint8_t *kinds = reinterpret_cast<const uint8_t *>(hh + 1);
    const int32_t *blens = hh + 1 + W, *sizes = hh + 1 + 2 * W;
    const int32_t run = max_batches > 0 && max_batches < nb ? max_batches : nb;
    // strides in elements: pool [N][planes][H][cap][D], staging [planes][B][H][cap][D]
    const int64_t hcd = d->H * d->cap * d->D;
    const int64_t p_plane = hcd, p_row = d->n_planes * hcd, p_head = d->cap * d->D;
    const int64_t s_plane = B * hcd, s_row = hcd, s_head = d->cap * d->D;
    // Processing order.  Serial: plan order.  Overlapped (n_staging >= 2): the fallback
    // batches are interleaved with the same-length ones, so that while the copy stream
    // gathers fallback f the main stream keeps verifying same-length batches.
    const int32_t NS = d->n_staging >= 2 ? d->n_staging : 0;
    const bool overlap = NS > 0 && run > 1;
    // same-length batches per verify launch (specdec_pool_verify_group), if the workspace
    // holds the grouped rows
    int32_t G = std::min<int32_t>(std::max<int32_t>(d->verify_group, 1), SPECDEC_MAX_VERIFY_GROUP);
    while (G > 1 && specdec_verify_workspace_size(static_cast<int64_t>(G) * B, d->k) > d->ws_bytes) --G;
    int64_t launches = 1;  // K4
    std::vector<int32_t> seq, fb_rank(run, -1);
    std::vector<int32_t> fbs;
    seq.reserve(run);
    for (int32_t b = 0; b < run; ++b)
        if ((kinds[b] == 0 && d->dense_consumer != 2) || d->dense_consumer == 1)
            fb_rank[b] = static_cast<int32_t>(fbs.size()), fbs.push_back(b);
    if (!overlap) {
        for (int32_t b = 0; b < run; ++b) seq.push_back(b);
    } else {
        // List schedule on estimated durations: a fallback batch goes next as soon as its
        // gather is expected to be done, else the next same-length batch; the copy stream
        // runs gathers back to back, the one into staging slot f % NS after the scatter of
        // f - NS (which follows that batch's verify).  Only the order (i.e. the timing)
        // depends on the estimates, never a result.
        const double gbps = d->est_gather_GBps > 0 ? d->est_gather_GBps : 5500.0;
        const double tv = d->est_verify_us > 0 ? d->est_verify_us : 10.0;  // K1 (+ scatter)
        const double row_bytes = static_cast<double>(d->n_planes) * d->H * d->D * dtype_size(d->kv_dtype);
        auto gather_us = [&](int32_t b) {  // read + write of <= size * (width - 1) rows
            return 2.0 * sizes[b] * std::max(blens[b] - 1, 0) * row_bytes / (gbps * 1e3);
        };
        std::vector<int32_t> sames;
        for (int32_t b = 0; b < run; ++b)
            if (fb_rank[b] < 0) sames.push_back(b);
        const size_t nf = fbs.size(), ns = sames.size();
        std::vector<double> g_end(nf, 0.0), s_end(nf, 0.0);
        for (size_t f = 0; f < nf && f < static_cast<size_t>(NS); ++f)
            g_end[f] = (f ? g_end[f - 1] : 0.0) + gather_us(fbs[f]);
        double t = 0.0;
        size_t fi = 0, si = 0;
        while (fi < nf || si < ns) {
            if (fi < nf && (g_end[fi] <= t || si == ns)) {
                t = std::max(t, g_end[fi]) + tv;  // its verify
                s_end[fi] = t;
                // copy stream: ..., gather nx - 1, [verify fi], scatter fi (~ tv), gather nx
                const size_t nx = fi + NS;
                if (nx < nf) g_end[nx] = std::max(g_end[nx - 1], s_end[fi]) + tv + gather_us(fbs[nx]);
                seq.push_back(fbs[fi++]);
            } else {
                t += tv;  // one (grouped) verify
                for (int32_t q = 0; q < G && si < ns; ++q) seq.push_back(sames[si++]);
            }
        }
    }
    cudaStream_t cs = overlap ? reinterpret_cast<cudaStream_t>(d->copy_stream) : nullptr;
    // scatters on their own stream beside the gathers (optional), else on the copy stream
    cudaStream_t ss = overlap && d->scatter_stream ? reinterpret_cast<cudaStream_t>(d->scatter_stream) : cs;
    auto ev = [&](int i) { return reinterpret_cast<cudaEvent_t>(d->events[i]); };
    auto sev = [&](int i) { return reinterpret_cast<cudaEvent_t>(d->scatter_events[i]); };
    auto stg = [&](int32_t b) -> void * {
        return overlap ? d->staging_ring[fb_rank[b] % NS] : d->staging;
    };
    // a batch's members fill its first sizes[b] slots (the rest are -1): every launch of
    // the batch covers those rows only
    auto rows = [&](int32_t b) -> int32_t { return sizes[b] > 0 && sizes[b] < B ? sizes[b] : B; };
    auto gather = [&](int32_t b, cudaStream_t on) {
        const int64_t o = static_cast<int64_t>(b) * B;
        return specdec_realign_kv(d->kv, stg(b), d->kv_dtype, d->n_planes, rows(b), d->H, d->D, p_plane,
                                  p_row, p_head, d->cap, s_plane, s_row, s_head, d->cap, nullptr, 0,
                                  d->mpad + o, 0, d->mlen + o, -1, 0, d->members + o, nullptr,
                                  d->gather_ws ? SPECDEC_DYNAMIC : 0u, d->gather_ws, d->gather_ws ? 128 : 0,
                                  d->moved, d->status,
                                  reinterpret_cast<specdec_stream_t>(on));
    };
    // the first NS gathers: the plan is complete (host sync above) and so is every
    // scatter of the previous epoch, so nothing to wait for
    if (overlap) {
        for (int32_t f = 0; f < NS && f < static_cast<int32_t>(fbs.size()); ++f) {
            if ((rc = gather(fbs[f], cs))) return rc;
            ++launches;
            if ((e = cudaEventRecord(ev(f % NS), cs)) != cudaSuccess) return record_cuda_error(e);
        }
    }
    const int kv1 = specdec_verify_kernels(1);
    // a group of same-length batches: each batch's inputs (forward or ring), one launch
    const void *g_lg[SPECDEC_MAX_VERIFY_GROUP] = {};
    const int64_t *g_dr[SPECDEC_MAX_VERIFY_GROUP] = {};
    int32_t g_off[SPECDEC_MAX_VERIFY_GROUP] = {}, g_rows[SPECDEC_MAX_VERIFY_GROUP] = {};
    int32_t ng = 0;
    auto flush_group = [&]() -> int {
        if (!ng) return SPECDEC_OK;
        const int r = ng == 1
            ? specdec_pool_verify(g_lg[0], d->logit_dtype, g_rows[0], d->k, d->V, d->logit_stride, g_dr[0],
                                  d->members + g_off[0], d->mlen + g_off[0], d->mactive + g_off[0], d->eos_id,
                                  d->pad_id, d->accept, d->bonus, d->emit, d->finished, d->len, d->gen,
                                  d->active, d->tokens, d->cap_tok, d->out_buf, d->max_new, d->status, d->ws,
                                  d->ws_bytes, stream)
            : specdec_pool_verify_group(ng, g_lg, g_dr, g_off, g_rows, d->logit_dtype, d->k, d->V,
                                        d->logit_stride, d->members, d->mlen, d->mactive, d->eos_id,
                                        d->pad_id, d->accept, d->bonus, d->emit, d->finished, d->len,
                                        d->gen, d->active, d->tokens, d->cap_tok, d->out_buf, d->max_new,
                                        d->status, d->ws, d->ws_bytes, stream);
        launches += kv1;
        ng = 0;
        return r;
    };
    const int32_t ring_base = d->ring_pos ? *d->ring_pos : 0;
    int32_t ran = 0, same = 0, msame = 0, mfb = 0;
    for (size_t qi = 0; qi < seq.size(); ++qi) {
        const int32_t b = seq[qi];
        const bool same_len = kinds[b] != 0;
        const bool fallback = fb_rank[b] >= 0;  // moves KV through the staging
        if (fallback && (rc = flush_group())) return rc;
        int32_t *members = d->members + static_cast<int64_t>(b) * B;
        int32_t *mlen = d->mlen + static_cast<int64_t>(b) * B;
        uint8_t *mact = d->mactive + static_cast<int64_t>(b) * B;
        if (fallback) {
            if (overlap) {
                e = cudaStreamWaitEvent(s, ev(fb_rank[b] % NS), 0);
                if (e != cudaSuccess) return record_cuda_error(e);
            } else if ((rc = gather(b, s))) {
                return rc;
            } else {
                ++launches;
            }
        }
        const void *logits;
        const int64_t *draft;
        if (forward) {
            if (d->cur_staging) *d->cur_staging = fallback ? stg(b) : nullptr;
            forward(ctx, b, fallback ? 0 : 1, blens[b], &logits, &draft);
        } else {
            const int32_t j = (ring_base + b) % d->ring_n;  // the plan index picks the slot
            logits = d->logits_ring[j];
            draft = d->draft_ring[j];
        }
        // K1 with the Phase 4 write-back fused into its epilogue; with overlap, a fallback
        // batch's accept lengths go to its staging slot's row of accept_ring, read by its
        // scatter on the copy stream after later batches have reused d->accept
        const int32_t slot = fallback && overlap ? fb_rank[b] % NS : -1;
        int32_t *acc = slot >= 0 ? d->accept_ring + static_cast<int64_t>(slot) * B : d->accept;
        if (!fallback) {
            // joins the open group; launched when the group is full, at the next fallback
            // batch, or at the end of the run of same-length batches
            g_lg[ng] = logits;
            g_dr[ng] = draft;
            g_off[ng] = static_cast<int32_t>(static_cast<int64_t>(b) * B);
            g_rows[ng] = rows(b);
            ++ng;
            const bool next_same = qi + 1 < seq.size() && fb_rank[seq[qi + 1]] < 0;
            if ((ng == G || !next_same) && (rc = flush_group())) return rc;
        } else {
            rc = specdec_pool_verify(logits, d->logit_dtype, rows(b), d->k, d->V, d->logit_stride, draft, members,
                                     mlen, mact, d->eos_id, d->pad_id, acc, d->bonus, d->emit,
                                     d->finished, d->len, d->gen, d->active, d->tokens, d->cap_tok,
                                     d->out_buf, d->max_new, d->status, d->ws, d->ws_bytes, stream);
            if (rc) return rc;
            launches += kv1;
        }
        if (fallback) {
            // scatter of the a+1 new KV rows back to the pool: on `stream` (serial) or on the
            // copy stream after this verify (overlap), where stream order also keeps the
            // next gather into this staging slot behind it
            cudaStream_t on = stream ? reinterpret_cast<cudaStream_t>(stream) : nullptr;
            if (overlap) {
                if ((e = cudaEventRecord(ev(NS + slot), s)) != cudaSuccess ||
                    (e = cudaStreamWaitEvent(ss, ev(NS + slot), 0)) != cudaSuccess)
                    return record_cuda_error(e);
                on = ss;
            }
            rc = specdec_realign_kv(stg(b), d->kv, d->kv_dtype, d->n_planes, rows(b), d->H, d->D,
                                    s_plane, s_row, s_head, d->cap, p_plane, p_row, p_head, d->cap,
                                    nullptr, blens[b] - 1, mlen, -1, acc, 1,
                                    static_cast<int32_t>(d->k + 1),  // a + 1 <= k + 1 rows
                                    nullptr, members, 0, nullptr, 0, d->moved, d->status,
                                    reinterpret_cast<specdec_stream_t>(on));
            if (rc) return rc;
            ++launches;
            const int32_t nxt = fb_rank[b] + NS;  // the gather that reuses this staging buffer
            if (overlap && nxt < static_cast<int32_t>(fbs.size())) {
                if (ss != cs) {  // the scatter (its own stream) first frees the staging slot
                    if ((e = cudaEventRecord(sev(slot), ss)) != cudaSuccess ||
                        (e = cudaStreamWaitEvent(cs, sev(slot), 0)) != cudaSuccess)
                        return record_cuda_error(e);
                }
                if ((rc = gather(fbs[nxt], cs))) return rc;
                ++launches;
                if ((e = cudaEventRecord(ev(nxt % NS), cs)) != cudaSuccess) return record_cuda_error(e);
            }
        }
        if (same_len) {
            ++same;
            msame += sizes[b];
        } else {
            mfb += sizes[b];
        }
        ++ran;
    }
    if (overlap && !fbs.empty()) {
        // the epoch ends on `stream`: it waits for the copy stream's last scatter (events[0]
        // is free again -- every wait on its earlier records has been enqueued), and for the
        // scatter stream's (scatter_events[0] likewise)
        if ((e = cudaEventRecord(ev(0), cs)) != cudaSuccess || (e = cudaStreamWaitEvent(s, ev(0), 0)) != cudaSuccess)
            return record_cuda_error(e);
        if (ss != cs && ((e = cudaEventRecord(sev(0), ss)) != cudaSuccess ||
                         (e = cudaStreamWaitEvent(s, sev(0), 0)) != cudaSuccess))
            return record_cuda_error(e);
    }
    if ((rc = flush_group())) return rc;
    if (!forward && d->ring_pos) *d->ring_pos = ring_base + run;
    if (d->host_launches) *d->host_launches += launches;
    if (h_ran) *h_ran = ran;
    if (h_same) *h_same = same;
    if (h_members_same) *h_members_same = msame;
    if (h_members_fallback) *h_members_fallback = mfb;
    return SPECDEC_OK;
}

// ----------------------------------------------------------------------------- Alg. 3 loop
// Alg. 3 as printed: GetBatch -> verify -> write-back -> RefillWindow,
// one batch per iteration, each iteration re-planning the window -- here without any host
// synchronisation: K4's tail (the gate, pool_gate.h) writes batch 0 as row maps that gate
// the gather / scatter (row map -1 = skip) and the verify (no active row) of a same-length
// or empty plan, so `iterations` iterations are enqueued back to back.  Iterations after the
// pool drains are no-ops.
extern "C" int specdec_pool_alg3(const specdec_pool_desc *d, int32_t iterations, int32_t *d_scratch,
                                 unsigned long long *d_exec_counters, specdec_stream_t stream) {
    if (!d || !d_scratch || d->W < 1 || d->B < 1 || d->B > 1024 || iterations < 0) return SPECDEC_ERR_ARG;
    if (!d->logits_ring || !d->draft_ring || d->ring_n < 1 || !d->ring_pos) return SPECDEC_ERR_ARG;
    const int32_t W = d->W, B = d->B;
    int32_t *g_members = d_scratch, *g_kv = d_scratch + B, *g_scol = d_scratch + 2 * B;
    uint8_t *g_active = reinterpret_cast<uint8_t *>(d_scratch + 3 * B);
    const int64_t hcd = d->H * d->cap * d->D;
    const int64_t p_plane = hcd, p_row = d->n_planes * hcd, p_head = d->cap * d->D;
    const int64_t s_plane = B * hcd, s_row = hcd, s_head = d->cap * d->D;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const uint32_t gflags = d->gather_ws ? SPECDEC_DYNAMIC : 0u;
    // the slot-indexed consumer (dense_consumer == 2) never moves KV: its gather / scatter
    // would be gated no-ops, so they are not launched (SPECDEC_ALG3_NOOP=1 launches them
    // anyway: measures what a gated no-op costs)
    static const int keep_noop = getenv("SPECDEC_ALG3_NOOP") ? atoi(getenv("SPECDEC_ALG3_NOOP")) : 0;
    const bool moves_kv = d->dense_consumer != 2 || keep_noop;
    Alg3Gate gate;
    gate.members = g_members;
    gate.kv = g_kv;
    gate.scol = g_scol;
    gate.active = g_active;
    gate.exec = d_exec_counters;
    gate.dense = d->dense_consumer;
    for (int32_t it = 0; it < iterations; ++it) {
        // Alg. 3's GetBatch: batch 0 of the window plan only (specdec_pool_getbatch)
        int rc = pool_group_launch(d->len, d->active, d->order, d->N, W, B, d->min_group, d->window,
                                   d->window_size, d->batch_of, d->slot_of, d->members, d->mlen, d->mpad,
                                   d->mactive, d->bsize, d->bkind, d->blen, d->n_batches, d->counters, gate,
                                   stream, true);
        if (rc) return rc;
        // fallback batch 0: pool slots [0, len-1) -> staging, right-aligned (rows -1: skipped)
        if (moves_kv)
            rc = specdec_realign_kv(d->kv, d->staging, d->kv_dtype, d->n_planes, B, d->H, d->D, p_plane, p_row,
                                p_head, d->cap, s_plane, s_row, s_head, d->cap, nullptr, 0, d->mpad, 0,
                                d->mlen, -1, 0, g_kv, nullptr, gflags, d->gather_ws, d->gather_ws ? 128 : 0,
                                d->moved, d->status, stream);
        if (rc) return rc;
        const int32_t j = (*d->ring_pos)++ % d->ring_n;
        rc = specdec_pool_verify(d->logits_ring[j], d->logit_dtype, B, d->k, d->V, d->logit_stride,
                                 d->draft_ring[j], g_members, d->mlen, g_active, d->eos_id, d->pad_id,
                                 d->accept, d->bonus, d->emit, d->finished, d->len, d->gen, d->active,
                                 d->tokens, d->cap_tok, d->out_buf, d->max_new, d->status, d->ws,
                                 d->ws_bytes, stream);
        if (rc) return rc;
        // the a+1 new KV rows back to the pool (rows -1: skipped)
        if (moves_kv)
            rc = specdec_realign_kv(d->staging, d->kv, d->kv_dtype, d->n_planes, B, d->H, d->D, s_plane, s_row,
                                s_head, d->cap, p_plane, p_row, p_head, d->cap, g_scol, 0, d->mlen, -1,
                                d->accept, 1, static_cast<int32_t>(d->k + 1), nullptr, g_kv, 0, nullptr, 0,
                                d->moved, d->status, stream);
        if (rc) return rc;
    }
    return SPECDEC_OK;
}

// ----------------------------------------------------------------------------- Alg. 3 graph
// `iterations` iterations of the Alg. 3 device loop as ONE CUDA graph, with the KV moves in
// conditional (IF) nodes: the GetBatch kernel sets the condition to "batch 0 moves KV"
// (cudaGraphSetConditional), so a same-length iteration runs GetBatch and the verify only
// -- no launch at all for its gather and scatter, where specdec_pool_alg3 launches them as
// gated no-ops (~2.3 us each, measured).  The graph is built piece by piece: each run of
// plain launches is stream-captured into it (cudaStreamBeginCaptureToGraph after the
// current frontier), each IF node is added between captures and its body captured from a
// second stream.
using Frontier = std::vector<cudaGraphNode_t>;

static int capture_segment(cudaStream_t s, cudaGraph_t graph, Frontier &deps,
                           const std::function<int(specdec_stream_t)> &launch, const char *what) {
    cudaError_t e = cudaStreamBeginCaptureToGraph(s, graph, deps.empty() ? nullptr : deps.data(), nullptr,
                                                  deps.size(), cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) return annotate_error(record_cuda_error(e), what);
    int rc = launch(reinterpret_cast<specdec_stream_t>(s));
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t *fr = nullptr;
    size_t nfr = 0;
    e = cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &fr, &nfr);
    Frontier next(fr, fr + nfr);
    cudaGraph_t out = nullptr;
    const cudaError_t e2 = cudaStreamEndCapture(s, &out);
    if (rc) return annotate_error(rc, what);
    if (e != cudaSuccess) return annotate_error(record_cuda_error(e), what);
    if (e2 != cudaSuccess) return annotate_error(record_cuda_error(e2), what);
    deps = next;
    return SPECDEC_OK;
}

static int add_if(cudaStream_t bs, cudaGraph_t graph, Frontier &deps, cudaGraphConditionalHandle h,
                  const std::function<int(specdec_stream_t)> &launch, const char *what) {
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    cudaError_t e = cudaGraphAddNode(&node, graph, deps.empty() ? nullptr : deps.data(), deps.size(), &cp);
    if (e != cudaSuccess) return annotate_error(record_cuda_error(e), what);
    Frontier none;
    const int rc = capture_segment(bs, cp.conditional.phGraph_out[0], none, launch, what);
    if (rc) return rc;
    deps.assign(1, node);
    return SPECDEC_OK;
}

extern "C" int specdec_pool_alg3_graph(const specdec_pool_desc *d, int32_t iterations, int32_t *d_scratch,
                                       unsigned long long *d_exec_counters, int32_t conditional,
                                       void **graph_exec) {
    if (!d || !d_scratch || !graph_exec || d->W < 1 || d->B < 1 || d->B > 1024 || iterations < 1)
        return SPECDEC_ERR_ARG;
    if (!d->logits_ring || !d->draft_ring || d->ring_n < 1 || !d->ring_pos) return SPECDEC_ERR_ARG;
    *graph_exec = nullptr;
    const int32_t W = d->W, B = d->B;
    int32_t *g_members = d_scratch, *g_kv = d_scratch + B, *g_scol = d_scratch + 2 * B;
    uint8_t *g_active = reinterpret_cast<uint8_t *>(d_scratch + 3 * B);
    const int64_t hcd = d->H * d->cap * d->D;
    const int64_t p_plane = hcd, p_row = d->n_planes * hcd, p_head = d->cap * d->D;
    const int64_t s_plane = B * hcd, s_row = hcd, s_head = d->cap * d->D;
    const uint32_t gflags = d->gather_ws ? SPECDEC_DYNAMIC : 0u;
    const bool moves_kv = d->dense_consumer != 2;  // the slot-indexed consumer moves no KV
    cudaStream_t s = nullptr, bs = nullptr;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaGraphCreate(&graph, 0);
    int rc = e == cudaSuccess ? SPECDEC_OK : annotate_error(record_cuda_error(e), "graph setup");
    Alg3Gate gate;
    gate.members = g_members;
    gate.kv = g_kv;
    gate.scol = g_scol;
    gate.active = g_active;
    gate.exec = d_exec_counters;
    gate.dense = d->dense_consumer;
    Frontier deps;
    if (!conditional) {
        // plain: the iterations exactly as specdec_pool_alg3 enqueues them (gated no-op KV
        // launches included), captured as one segment with their PDL edges
        if (!rc)
            rc = capture_segment(s, graph, deps, [&](specdec_stream_t on) {
                return specdec_pool_alg3(d, iterations, d_scratch, d_exec_counters, on);
            }, "alg3 loop");
        iterations = 0;
    } else {
        // no programmatic (PDL) edges: the kernels sit between conditional nodes
        pdl_suppress(true);
    }
    for (int32_t it = 0; it < iterations && !rc; ++it) {
        // one conditional handle per IF node (a handle belongs to a single node): the
        // iteration's GetBatch sets both
        cudaGraphConditionalHandle hg = 0, hs = 0;
        if (moves_kv) {
            e = cudaGraphConditionalHandleCreate(&hg, graph, 0, cudaGraphCondAssignDefault);
            if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hs, graph, 0, cudaGraphCondAssignDefault);
            if (e != cudaSuccess) {
                rc = annotate_error(record_cuda_error(e), "conditional handles");
                break;
            }
        }
        gate.cond = hg;
        gate.cond2 = hs;
        rc = capture_segment(s, graph, deps, [&](specdec_stream_t on) {
            return pool_group_launch(d->len, d->active, d->order, d->N, W, B, d->min_group, d->window,
                                     d->window_size, d->batch_of, d->slot_of, d->members, d->mlen, d->mpad,
                                     d->mactive, d->bsize, d->bkind, d->blen, d->n_batches, d->counters, gate, on,
                                     true);
        }, "getbatch");
        if (!rc && moves_kv)
            rc = add_if(bs, graph, deps, hg, [&](specdec_stream_t on) {
                return specdec_realign_kv(d->kv, d->staging, d->kv_dtype, d->n_planes, B, d->H, d->D, p_plane,
                                          p_row, p_head, d->cap, s_plane, s_row, s_head, d->cap, nullptr, 0,
                                          d->mpad, 0, d->mlen, -1, 0, g_kv, nullptr, gflags, d->gather_ws,
                                          d->gather_ws ? 128 : 0, d->moved, d->status, on);
            }, "gather");
        if (rc) break;
        const int32_t j = (*d->ring_pos)++ % d->ring_n;
        rc = capture_segment(s, graph, deps, [&](specdec_stream_t on) {
            return specdec_pool_verify(d->logits_ring[j], d->logit_dtype, B, d->k, d->V, d->logit_stride,
                                       d->draft_ring[j], g_members, d->mlen, g_active, d->eos_id, d->pad_id,
                                       d->accept, d->bonus, d->emit, d->finished, d->len, d->gen, d->active,
                                       d->tokens, d->cap_tok, d->out_buf, d->max_new, d->status, d->ws,
                                       d->ws_bytes, on);
        }, "verify");
        if (!rc && moves_kv)
            rc = add_if(bs, graph, deps, hs, [&](specdec_stream_t on) {
                return specdec_realign_kv(d->staging, d->kv, d->kv_dtype, d->n_planes, B, d->H, d->D, s_plane,
                                          s_row, s_head, d->cap, p_plane, p_row, p_head, d->cap, g_scol, 0,
                                          d->mlen, -1, d->accept, 1, static_cast<int32_t>(d->k + 1), nullptr,
                                          g_kv, 0, nullptr, 0, d->moved, d->status, on);
            }, "scatter");
    }
    if (conditional) pdl_suppress(false);
    cudaGraphExec_t ex = nullptr;
    if (!rc) {
        e = cudaGraphInstantiate(&ex, graph, 0);
        if (e != cudaSuccess) rc = annotate_error(record_cuda_error(e), "instantiate");
    }
    if (graph) cudaGraphDestroy(graph);
    if (bs) cudaStreamDestroy(bs);
    if (s) cudaStreamDestroy(s);
    if (!rc) *graph_exec = ex;
    return rc;
}

extern "C" int specdec_graph_launch(void *graph_exec, specdec_stream_t stream) {
    if (!graph_exec) return SPECDEC_ERR_ARG;
    const cudaError_t e = cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec), reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SPECDEC_OK : record_cuda_error(e);
}

extern "C" int specdec_graph_destroy(void *graph_exec) {
    if (!graph_exec) return SPECDEC_OK;
    const cudaError_t e = cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph_exec));
    return e == cudaSuccess ? SPECDEC_OK : record_cuda_error(e);
}
