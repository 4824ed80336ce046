// round_exec.cu -- native EqSpec round driver (host C++): Alg. 2's loop body after the
// verify forward as one C call, and the same round from host inputs
// with its host<->device copies (the end-to-end path).  Every kernel is launched through
// the same C ABI entry points the Python driver (eqspec.py) uses; nothing here computes.
#include <cuda_runtime.h>

#include "host_util.h"
#include "specdec.h"

using namespace specdec;

extern "C" int specdec_eqspec_round(const specdec_round_desc *d, int parity, const void *d_logits,
                                    const int64_t *d_draft, specdec_stream_t stream) {
    if (!d || !d_logits || !d_draft || (parity != 0 && parity != 1)) return SPECDEC_ERR_ARG;
    const int c = parity, nx = 1 - parity;
    // K1: Alg. 1 + the BatchRepad plan (writes n[nx], pad[nx], kept, plan_L)
    int rc = specdec_verify(d_logits, d->logit_dtype, d->B, d->k, d->V, d->logit_stride, d_draft,
                            d->n[c], d->active, d->eos_id, d->pad_id, d->budget, d->accept[c],
                            d->bonus[c], d->emit[c], d->finished[c], d->pred, d->plan_L, d->n[nx],
                            d->pad[nx], d->kept, d->kept_draft, d->anchor, d->anchor ? d->cap_kv : 0,
                            d->phys_old, d->phys_new,
                            d->status, d->ws, d->ws_bytes, stream);
    if (rc) return rc;
    // K3: tokens' / mask / positions (+ output buffer)
    rc = specdec_rebuild_pos_mask(d->tokens[c], d->tokens[nx], d->B, d->cap_tok, d->k, d->pad_id,
                                  d->n[c], d->pad[c], d_draft, d->accept[c], d->bonus[c], d->emit[c],
                                  d->finished[c], d->plan_L, d->pad[nx], d->mask, d->pos, d->mp_stride,
                                  d->out_buf, d->out_buf ? d->gen : nullptr, d->max_new, d->status,
                                  stream);
    if (rc) return rc;
    // K2: KV[p'_i + c] = KV[p_i + c], c < kept_i (target, then the draft model's cache)
    const bool inplace = d->kv[0] == d->kv[1];
    if (d->B == 1 && inplace && !d->anchor) return SPECDEC_OK;  // one row: p = p' = 0, nothing moves
    // source / destination columns: the pads, or K1's physical columns (anchored origin)
    const int32_t *col_src = d->anchor ? d->phys_old : d->pad[c];
    const int32_t *col_dst = d->anchor ? d->phys_new : d->pad[nx];
    const void *src = d->kv[inplace ? 0 : c];
    void *dst = d->kv[inplace ? 0 : nx];
    const uint32_t flags = d->realign_flags;
    rc = specdec_realign_kv(src, dst, d->kv_dtype, d->n_planes, d->B, d->H, d->D, d->s_plane, d->s_row,
                            d->s_head, d->cap_kv, d->s_plane, d->s_row, d->s_head, d->cap_kv, col_src, 0,
                            col_dst, 0, d->kept, 0, 0, nullptr, nullptr, flags, d->realign_ws,
                            d->realign_ws_bytes, d->moved, d->status, stream);
    if (rc || !d->dkv[0]) return rc;
    if (!d->kept_draft) return SPECDEC_ERR_ARG;
    const bool dinplace = d->dkv[0] == d->dkv[1];
    return specdec_realign_kv(d->dkv[dinplace ? 0 : c], d->dkv[dinplace ? 0 : nx], d->kv_dtype, d->d_planes,
                              d->B, d->d_H, d->d_D, d->d_s_plane, d->d_s_row, d->d_s_head, d->cap_kv,
                              d->d_s_plane, d->d_s_row, d->d_s_head, d->cap_kv, col_src, 0, col_dst, 0,
                              d->kept_draft, 0, 0, nullptr, nullptr,
                              flags & (SPECDEC_ZERO_PADS | SPECDEC_DYNAMIC | SPECDEC_SEGMENTED),
                              d->realign_ws, d->realign_ws_bytes, d->moved, d->status, stream);
}

extern "C" int specdec_eqspec_round_host(const specdec_round_desc *d, const specdec_host_io *io,
                                         int parity, int slot, const void *h_logits,
                                         const int64_t *h_draft, int32_t *h_emit,
                                         specdec_stream_t stream) {
    if (!d || !io || !h_logits || !h_draft || (parity != 0 && parity != 1)) return SPECDEC_ERR_ARG;
    if (io->n_slots < 2 || io->n_slots > SPECDEC_HOST_SLOTS || slot < 0 || slot >= io->n_slots)
        return SPECDEC_ERR_ARG;
    if (!io->d_logits[slot] || !io->d_draft[slot] || !io->copy_stream || !io->ev_ready[slot] ||
        !io->ev_done[slot] || (h_emit && (!io->d2h_stream || !io->ev_fetched[parity])))
        return SPECDEC_ERR_ARG;
    const int es = dtype_size(d->logit_dtype);
    if (es == 0) return SPECDEC_ERR_DTYPE;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaStream_t cp = reinterpret_cast<cudaStream_t>(io->copy_stream);
    auto ev = [](void *e) { return reinterpret_cast<cudaEvent_t>(e); };
    const size_t lg_bytes = static_cast<size_t>(d->B * (d->k + 1) * d->logit_stride) * es;
    const size_t dr_bytes = static_cast<size_t>(d->B * d->k) * sizeof(int64_t);
    cudaError_t e = cudaStreamWaitEvent(cp, ev(io->ev_done[slot]), 0);
    // one DMA when the drafts directly follow the logits on both sides (packed buffers)
    const bool packed = io->inputs_packed &&
                        reinterpret_cast<const char *>(h_draft) == static_cast<const char *>(h_logits) + lg_bytes &&
                        reinterpret_cast<const char *>(io->d_draft[slot]) ==
                            static_cast<const char *>(io->d_logits[slot]) + lg_bytes;
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(io->d_logits[slot], h_logits, packed ? lg_bytes + dr_bytes : lg_bytes,
                            cudaMemcpyHostToDevice, cp);
    if (e == cudaSuccess && !packed)
        e = cudaMemcpyAsync(io->d_draft[slot], h_draft, dr_bytes, cudaMemcpyHostToDevice, cp);
    if (e == cudaSuccess) e = cudaEventRecord(ev(io->ev_ready[slot]), cp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev(io->ev_ready[slot]), 0);
    if (e == cudaSuccess && io->ev_fetched[parity]) e = cudaStreamWaitEvent(s, ev(io->ev_fetched[parity]), 0);
    if (e != cudaSuccess) return record_cuda_error(e);
    int rc = specdec_eqspec_round(d, parity, io->d_logits[slot], io->d_draft[slot], stream);
    if (rc) return rc;
    e = cudaEventRecord(ev(io->ev_done[slot]), s);
    if (e == cudaSuccess && h_emit) {
        cudaStream_t dh = reinterpret_cast<cudaStream_t>(io->d2h_stream);
        e = cudaStreamWaitEvent(dh, ev(io->ev_done[slot]), 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(h_emit, d->emit[parity], static_cast<size_t>(d->B) * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, dh);
        if (e == cudaSuccess) e = cudaEventRecord(ev(io->ev_fetched[parity]), dh);
    }
    return e == cudaSuccess ? SPECDEC_OK : record_cuda_error(e);
}
