// repad.cu -- K3: Alg. 2 Phase 3 unpad-append-repad with the
// padding-agnostic position ids and attention masks of §3.1, and the
// EXSpec pool write-back (Alg. 3 Phase 4).
//
// One CTA per batch row.  The new width L' and pads p' come from device memory
// (specdec_verify's plan), so the round needs no host synchronisation.  The row's old
// content is moved by Delta = p' - p columns in place: the CTA walks the row in the
// hazard-free direction (right shifts high->low, left shifts low->high) one block of
// columns at a time, reading the block into registers before any thread writes it.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "repad_cols.cuh"
#include "host_util.h"

namespace specdec {

constexpr int kRepadThreads = 256;

struct RepadParams {
    const int64_t *tok_in;
    int64_t *tok_out;
    int64_t B, cap_tok, k, pad_id;
    const int32_t *n_old, *pad_old;
    const int64_t *draft;
    const int32_t *accept;
    const int64_t *bonus;
    const int32_t *emit;
    const uint8_t *finished;
    const int32_t *plan_L, *pad_new;
    int64_t *mask, *pos;
    int64_t mp_stride;
    int64_t *out_buf;
    int32_t *gen;
    int64_t max_new;
    uint32_t *status;
};


__global__ void __launch_bounds__(kRepadThreads) repad_kernel(RepadParams p) {
    pdl_wait();
    pdl_launch_dependents();
    const int64_t i = blockIdx.x;
    const int tid = threadIdx.x;
    const int32_t Lnew = *p.plan_L;
    const int32_t a = p.accept[i];
    const int32_t em = p.emit[i];
    const int64_t *d = p.draft + i * p.k;
    const int64_t b = p.bonus[i];

    // output buffer: append E_i (the paper's S[i] <- S[i] (+) A[i] (+) B[i] for the
    // generated part); rows that emitted nothing are untouched.
    if (p.out_buf && em > 0) {
        const int32_t g = p.gen[i];
        if (g + em > p.max_new) {
            if (tid == 0 && p.status) atomicOr(p.status, SPECDEC_ST_CAPACITY);
        } else {
            if (tid < em) p.out_buf[i * p.max_new + g + tid] = emitted_token(d, a, b, tid);
            __syncthreads();
            if (tid == 0) p.gen[i] = g + em;
        }
    }
    if (Lnew <= 0) return;  // every row finished: the batch is done
    if (Lnew > p.cap_tok || Lnew + p.k > p.mp_stride) {
        if (tid == 0 && p.status) atomicOr(p.status, SPECDEC_ST_CAPACITY);
        return;
    }
    const int32_t pn = p.pad_new[i];
    const int64_t *src = p.tok_in + i * p.cap_tok;
    int64_t *dst = p.tok_out + i * p.cap_tok;

    if (p.finished[i]) {
        // R9: a finished row becomes a dummy length-1 row [pad] at L'-1
        for (int c = tid; c < Lnew; c += kRepadThreads) dst[c] = p.pad_id;
    } else {
        const int32_t po = p.pad_old[i];
        const int32_t n = p.n_old[i];
        const int32_t delta = pn - po;
        if (delta != 0 || src != dst) {
            // move old content [po, po+n) -> [pn, pn+n) in the safe direction
            const int nblk = (n + kRepadThreads - 1) / kRepadThreads;
            for (int q = 0; q < nblk; ++q) {
                const int blk = delta > 0 ? nblk - 1 - q : q;
                const int c = blk * kRepadThreads + tid;
                int64_t v = 0;
                if (c < n) v = src[po + c];
                __syncthreads();
                if (c < n) dst[pn + c] = v;
                __syncthreads();
            }
        }
        // append A[i] ++ [B[i]] at [pn+n, L') (Alg. 2 Phase 3)
        if (tid <= a) dst[pn + n + tid] = emitted_token(d, a, b, tid);
        // left pads
        for (int c = tid; c < pn; c += kRepadThreads) dst[c] = p.pad_id;
    }
    // masks exclude pads; positions reset to 0 at the first content token
    int64_t *mrow = p.mask + i * p.mp_stride;
    int64_t *prow = p.pos + i * p.mp_stride;
    const int32_t W = Lnew + static_cast<int32_t>(p.k);
    for (int c = tid; c < W; c += kRepadThreads) {
        const bool content = c >= pn;
        mrow[c] = content ? 1 : 0;
        prow[c] = content ? c - pn : 0;
    }
}

// Out-of-place variant (tokens_out != tokens_in): every output column is an independent
// gather, so a row is spread over many CTAs with no ordering at all.
//   c <  p'            : pad
//   p' <= c < p' + n   : old token at column c - p' + p      (unpad + repad)
//   p' + n <= c < L'   : E[c - p' - n]                        (append A ++ [B])
constexpr int kRepadCols = 1;  // columns per thread: many small CTAs, the kernel is latency-bound
__global__ void __launch_bounds__(kRepadThreads) repad_gather_kernel(RepadParams p) {
    pdl_wait();                // K1's plan is complete and visible
    pdl_launch_dependents();
    const int64_t i = blockIdx.y;
    const int tid = threadIdx.x;
    const int32_t Lnew = *p.plan_L;
    const int32_t a = p.accept[i];
    const int32_t em = p.emit[i];
    const int64_t *d = p.draft + i * p.k;
    const int64_t b = p.bonus[i];
    if (blockIdx.x == 0 && p.out_buf && em > 0) {
        const int32_t g = p.gen[i];
        if (g + em > p.max_new) {
            if (tid == 0 && p.status) atomicOr(p.status, SPECDEC_ST_CAPACITY);
        } else {
            if (tid < em) p.out_buf[i * p.max_new + g + tid] = emitted_token(d, a, b, tid);
            __syncthreads();
            if (tid == 0) p.gen[i] = g + em;
        }
    }
    if (Lnew <= 0) return;
    if (Lnew > p.cap_tok || Lnew + p.k > p.mp_stride) {
        if (blockIdx.x == 0 && tid == 0 && p.status) atomicOr(p.status, SPECDEC_ST_CAPACITY);
        return;
    }
    const int32_t pn = p.pad_new[i];
    const bool fin = p.finished[i] != 0;
    const int32_t po = p.pad_old[i];
    const int32_t n = fin ? 0 : p.n_old[i];
    const int64_t *src = p.tok_in + i * p.cap_tok;
    int64_t *dst = p.tok_out + i * p.cap_tok;
    int64_t *mrow = p.mask + i * p.mp_stride;
    int64_t *prow = p.pos + i * p.mp_stride;
    const int32_t W = Lnew + static_cast<int32_t>(p.k);
    const int c0 = blockIdx.x * (kRepadThreads * kRepadCols) + tid;
#pragma unroll
    for (int u = 0; u < kRepadCols; ++u) {
        const int c = c0 + u * kRepadThreads;
        if (c >= W) break;
        repad_col(c, Lnew, pn, fin, po, n, src, dst, mrow, prow, d, a, b, p.pad_id);
    }
}

// ----------------------------------------------------------------------------- pool write-back
// One CTA per batch slot r; E_r = first emit_r tokens of draft[r][0:a_r] ++ [bonus_r].
__global__ void pool_writeback_kernel(const int32_t *members, int64_t k, const int64_t *draft,
                                      const int32_t *accept, const int64_t *bonus,
                                      const int32_t *emit, const uint8_t *finished,
                                      int32_t *pool_len, int32_t *pool_gen, uint8_t *pool_active,
                                      int64_t *pool_tokens, int64_t cap_tok, int64_t *out_buf,
                                      int64_t max_new, uint32_t *status) {
    pdl_wait();
    pdl_launch_dependents();
    const int64_t r = blockIdx.x;
    const int32_t s = members[r];
    if (s < 0) return;
    const int tid = threadIdx.x;
    const int32_t a = accept[r];
    const int64_t *d = draft + r * k;
    const int64_t b = bonus[r];
    const int32_t len = pool_len[s];
    const int32_t g = pool_gen[s];
    // E_r is already cut after the first EOS by specdec_verify; the per-sequence budget
    // (max_new generated tokens, SPEC.md:354 completion rule) is applied here.
    const int32_t em = min(emit[r], static_cast<int32_t>(max(static_cast<int64_t>(0), max_new - g)));
    const bool fin = finished[r] || g + em >= max_new;
    if (pool_tokens && len + em > cap_tok) {
        if (tid == 0 && status) atomicOr(status, SPECDEC_ST_CAPACITY);
        return;
    }
    if (tid < em) {
        const int64_t t = emitted_token(d, a, b, tid);
        if (pool_tokens) pool_tokens[static_cast<int64_t>(s) * cap_tok + len + tid] = t;
        if (out_buf) out_buf[static_cast<int64_t>(s) * max_new + g + tid] = t;
    }
    if (tid == 0) {
        pool_len[s] = len + em;   // Pool[i] <- Pool[i] (+) A[i] (+) B[i]
        pool_gen[s] = g + em;
        if (fin) pool_active[s] = 0;  // isComplete -> Pool.deactivate(i)
    }
}

}  // namespace specdec

using namespace specdec;

extern "C" int specdec_rebuild_pos_mask(const int64_t *d_tokens_in, int64_t *d_tokens_out,
                                        int64_t B, int64_t cap_tok, int64_t k, int64_t pad_id,
                                        const int32_t *d_n_old, const int32_t *d_pad_old,
                                        const int64_t *d_draft, const int32_t *d_accept,
                                        const int64_t *d_bonus, const int32_t *d_emit,
                                        const uint8_t *d_finished, const int32_t *d_plan_L,
                                        const int32_t *d_pad_new, int64_t *d_mask,
                                        int64_t *d_pos, int64_t mp_stride, int64_t *d_out_buf,
                                        int32_t *d_gen, int64_t max_new, uint32_t *d_status,
                                        specdec_stream_t stream) {
    if (k < 1 || k >= kRepadThreads) return SPECDEC_ERR_ARG;
    if (B < 1 || cap_tok < 1 || mp_stride < 1) return SPECDEC_ERR_SHAPE;
    if (B > 0x7FFFFFFFll) return SPECDEC_ERR_SHAPE;
    if (cap_tok < k + 2 || mp_stride < k + 2) return SPECDEC_ERR_CAPACITY;
    if (!d_tokens_in || !d_tokens_out || !d_n_old || !d_pad_old || !d_draft || !d_accept ||
        !d_bonus || !d_emit || !d_finished || !d_plan_L || !d_pad_new || !d_mask || !d_pos)
        return SPECDEC_ERR_ARG;
    if ((d_out_buf == nullptr) != (d_gen == nullptr)) return SPECDEC_ERR_ARG;
    if (d_out_buf && (max_new < 1 || max_new > 0x7FFFFFFFll)) return SPECDEC_ERR_SHAPE;
    RepadParams p;
    p.tok_in = d_tokens_in; p.tok_out = d_tokens_out;
    p.B = B; p.cap_tok = cap_tok; p.k = k; p.pad_id = pad_id;
    p.n_old = d_n_old; p.pad_old = d_pad_old; p.draft = d_draft; p.accept = d_accept;
    p.bonus = d_bonus; p.emit = d_emit; p.finished = d_finished; p.plan_L = d_plan_L;
    p.pad_new = d_pad_new; p.mask = d_mask; p.pos = d_pos; p.mp_stride = mp_stride;
    p.out_buf = d_out_buf; p.gen = d_gen; p.max_new = max_new; p.status = d_status;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (d_tokens_in == d_tokens_out) {
        // in place: one CTA walks each row in the hazard-free direction
        return launch_k(repad_kernel, dim3(static_cast<unsigned>(B)), dim3(kRepadThreads), 0, s, p);
    }
    if (B > 65535) return SPECDEC_ERR_SHAPE;
    const int64_t cols = std::max(cap_tok, mp_stride);
    const int64_t per = static_cast<int64_t>(kRepadThreads) * kRepadCols;
    dim3 grid(static_cast<unsigned>((cols + per - 1) / per), static_cast<unsigned>(B));
    return launch_k(repad_gather_kernel, grid, dim3(kRepadThreads), 0, s, p);
}

extern "C" int specdec_pool_writeback(const int32_t *d_members, int64_t B, int64_t k,
                                      const int64_t *d_draft, const int32_t *d_accept,
                                      const int64_t *d_bonus, const int32_t *d_emit,
                                      const uint8_t *d_finished, int32_t *d_pool_len,
                                      int32_t *d_pool_gen, uint8_t *d_pool_active,
                                      int64_t *d_pool_tokens, int64_t cap_tok, int64_t *d_out_buf,
                                      int64_t max_new, uint32_t *d_status,
                                      specdec_stream_t stream) {
    if (k < 1 || k >= 1024) return SPECDEC_ERR_ARG;
    if (B < 1 || B > 0x7FFFFFFFll) return SPECDEC_ERR_SHAPE;
    if (!d_members || !d_draft || !d_accept || !d_bonus || !d_emit || !d_finished ||
        !d_pool_len || !d_pool_gen || !d_pool_active)
        return SPECDEC_ERR_ARG;
    if (d_pool_tokens && cap_tok < 1) return SPECDEC_ERR_SHAPE;
    if (max_new < 1) return SPECDEC_ERR_SHAPE;
    const int threads = static_cast<int>((k + 1 + 31) / 32 * 32);
    return launch_k(pool_writeback_kernel, dim3(static_cast<unsigned>(B)), dim3(threads), 0,
                    reinterpret_cast<cudaStream_t>(stream), d_members, k, d_draft, d_accept,
                    d_bonus, d_emit, d_finished, d_pool_len, d_pool_gen, d_pool_active,
                    d_pool_tokens, cap_tok, d_out_buf, max_new, d_status);
}

// ----------------------------------------------------------------------------- batch init
// Alg. 2 line 1: the left-padded batch state -- L = max n (R6), pad = L - n.
__global__ void __launch_bounds__(1024) batch_init_kernel(const int32_t *n, int64_t B, int32_t *pad,
                                                          int32_t *L_out, uint8_t *active,
                                                          int32_t *budget, int32_t max_new,
                                                          uint32_t *status) {
    pdl_wait();
    pdl_launch_dependents();
    __shared__ int s_max[32];
    int m = 0;
    for (int64_t i = threadIdx.x; i < B; i += blockDim.x) m = max(m, n[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = m;
    __syncthreads();
    int L = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) L = max(L, s_max[w]);
    for (int64_t i = threadIdx.x; i < B; i += blockDim.x) {
        const int32_t ni = n[i];
        if (ni < 1 && status) atomicOr(status, SPECDEC_ST_CAPACITY);
        pad[i] = ni >= 1 ? L - ni : L;
        if (active) active[i] = 1;
        if (budget) budget[i] = max_new;
    }
    if (threadIdx.x == 0 && L_out) *L_out = L;
}

extern "C" int specdec_batch_init(const int32_t *d_n, int64_t B, int32_t *d_pad, int32_t *d_L,
                                  uint8_t *d_active, int32_t *d_budget, int32_t max_new,
                                  uint32_t *d_status, specdec_stream_t stream) {
    if (!d_n || !d_pad) return SPECDEC_ERR_ARG;
    if (B < 1) return SPECDEC_ERR_SHAPE;
    return launch_k(batch_init_kernel, dim3(1), dim3(1024), 0, reinterpret_cast<cudaStream_t>(stream), d_n, B,
                    d_pad, d_L, d_active, d_budget, max_new, d_status);
}
