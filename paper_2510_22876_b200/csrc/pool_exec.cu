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
#include <cuda_runtime.h>

#include "host_util.h"
#include "specdec.h"

using namespace specdec;

extern "C" int specdec_pool_epoch(const specdec_pool_desc *d, specdec_forward_fn forward,
                                  void *ctx, int32_t max_batches, int32_t *h_ran,
                                  int32_t *h_same, int32_t *h_members_same,
                                  int32_t *h_members_fallback, specdec_stream_t stream) {
    if (!d || !d->host_header || d->W < 1 || d->B < 1) return SPECDEC_ERR_ARG;
    if (!forward && (!d->logits_ring || !d->draft_ring || d->ring_n < 1 || !d->ring_pos))
        return SPECDEC_ERR_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int32_t W = d->W, B = d->B;
    int rc = specdec_pool_group(d->len, d->active, d->order, d->N, W, B, d->min_group, d->window,
                                d->window_size, d->batch_of, d->slot_of, d->members, d->mlen,
                                d->mpad, d->mactive, d->bsize, d->bkind, d->blen, d->n_batches,
                                d->counters, stream);
    if (rc) return rc;
    // plan header -> pinned host: n_batches, kind, width, size (W each)
    int32_t *hh = d->host_header;
    cudaError_t e = cudaMemcpyAsync(hh, d->n_batches, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hh + 1 + W, d->blen, W * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hh + 1 + 2 * W, d->bsize, W * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(reinterpret_cast<uint8_t *>(hh + 1), d->bkind, W, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return record_cuda_error(e);
    const int32_t nb = hh[0];
    const uint8_t *kinds = reinterpret_cast<const uint8_t *>(hh + 1);
    const int32_t *blens = hh + 1 + W, *sizes = hh + 1 + 2 * W;
    const int32_t run = max_batches > 0 && max_batches < nb ? max_batches : nb;
    const int es = dtype_size(d->kv_dtype);
    // strides in elements: pool [N][planes][H][cap][D], staging [planes][B][H][cap][D]
    const int64_t hcd = d->H * d->cap * d->D;
    const int64_t p_plane = hcd, p_row = d->n_planes * hcd, p_head = d->cap * d->D;
    const int64_t s_plane = B * hcd, s_row = hcd, s_head = d->cap * d->D;
    (void)es;
    int32_t ran = 0, same = 0, msame = 0, mfb = 0;
    for (int32_t b = 0; b < run; ++b) {
        const bool same_len = kinds[b] != 0;
        const bool fallback = !same_len || d->dense_consumer;  // moves KV through the staging
        int32_t *members = d->members + static_cast<int64_t>(b) * B;
        int32_t *mlen = d->mlen + static_cast<int64_t>(b) * B;
        int32_t *mpad = d->mpad + static_cast<int64_t>(b) * B;
        uint8_t *mact = d->mactive + static_cast<int64_t>(b) * B;
        if (fallback) {
            rc = specdec_realign_kv(d->kv, d->staging, d->kv_dtype, d->n_planes, B, d->H, d->D,
                                    p_plane, p_row, p_head, d->cap, s_plane, s_row, s_head, d->cap,
                                    nullptr, 0, mpad, 0, mlen, -1, 0, members, nullptr, 0, nullptr, 0,
                                    d->moved, d->status, stream);
            if (rc) return rc;
        }
        const void *logits;
        const int64_t *draft;
        if (forward) {
            forward(ctx, b, fallback ? 0 : 1, blens[b], &logits, &draft);
        } else {
            const int32_t j = (*d->ring_pos)++ % d->ring_n;
            logits = d->logits_ring[j];
            draft = d->draft_ring[j];
        }
        // K1 with the Phase 4 write-back fused into its epilogue
        rc = specdec_pool_verify(logits, d->logit_dtype, B, d->k, d->V, d->logit_stride, draft, members,
                                 mlen, mact, d->eos_id, d->pad_id, d->accept, d->bonus, d->emit,
                                 d->finished, d->len, d->gen, d->active, d->tokens, d->cap_tok,
                                 d->out_buf, d->max_new, d->status, d->ws, d->ws_bytes, stream);
        if (rc) return rc;
        if (fallback) {
            rc = specdec_realign_kv(d->staging, d->kv, d->kv_dtype, d->n_planes, B, d->H, d->D,
                                    s_plane, s_row, s_head, d->cap, p_plane, p_row, p_head, d->cap,
                                    nullptr, blens[b] - 1, mlen, -1, d->accept, 1,
                                    static_cast<int32_t>(d->k + 1),  // a + 1 <= k + 1 rows
                                    nullptr, members, 0, nullptr, 0, d->moved, d->status, stream);
            if (rc) return rc;
        }
        if (same_len) {
            ++same;
            msame += sizes[b];
        } else {
            mfb += sizes[b];
        }
        ++ran;
    }
    if (h_ran) *h_ran = ran;
    if (h_same) *h_same = same;
    if (h_members_same) *h_members_same = msame;
    if (h_members_fallback) *h_members_fallback = mfb;
    return SPECDEC_OK;
}
