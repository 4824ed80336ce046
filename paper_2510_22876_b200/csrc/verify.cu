// verify.cu -- K1: Alg. 1 BatchVerify fused with the BatchRepad plan
// (§3.1).
//
// One pass over the logits tail [B][k+1][V]: every CTA scans one vocab chunk of one
// (row, slot) with 128-bit streaming loads and reduces it to a packed (key, ~index)
// 64-bit maximum, merged into the row's workspace word with one atomicMax.  The packing
// makes "largest value, then lowest index" a plain unsigned max -- associative and
// commutative -- so the split and the atomic order never change the winner: the argmax
// is bit-exact with lowest-index ties, +0 == -0, and the first-NaN rule (R4, R5).
// The epilogue, one warp per batch row: first-mismatch scan by warp ballot
// (PAPER.md:304-306 with R1), bonus (R2), EOS / budget trim (R10) and the repad plan (L',
// p', kept) -- no host round trip.  It runs in a one-CTA kernel launched right behind the
// argmax grid (programmatic dependent launch: resident before the grid ends, released by
// its completion), which measured faster than a last-CTA-arrival epilogue (the key RED
// plus an acq_rel atomic per CTA): B=1 5.22 -> 4.83 us, pool +5 %.  SPECDEC_K1_SPLIT=0
// selects the arrival design.  The workspace is left zeroed for the next call.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "host_util.h"

namespace specdec {

constexpr int kVerifyThreads = 256;
constexpr int kMaxK = 31;  // k + 1 <= 32: one lane per slot in the epilogue
constexpr int kEpiCache = 1024;  // rows whose n' the epilogue keeps in shared memory
// default completion modes (VerifyParams::split), measured: tools/k1bench.py
constexpr int kSplitEqSpec = 1, kSplitPool = 2;
constexpr int kMaxGroup = SPECDEC_MAX_VERIFY_GROUP;  // specdec_pool_verify_group: batches per launch

struct VerifyParams {
    const void *logits;
    int64_t B, k, V, row_stride, chunk;
    const int64_t *draft;
    const int32_t *n;
    uint8_t *active;
    int64_t eos_id, pad_id;
    int32_t *budget;
    int32_t *accept;
    int64_t *bonus;
    int32_t *emit;
    uint8_t *finished;
    int64_t *pred;
    int32_t *plan_L, *n_new, *pad_new, *kept, *kept_draft;
    int32_t *anchor;          // f3: physical origin (in/out), NULL = off
    int64_t anchor_cap;
    int32_t *phys_old, *phys_new;
    // pool mode (specdec_pool_verify): Alg. 3 Phase 4 write-back fused into the epilogue
    const int32_t *wb_members;  // [B] pool sequence of each row (-1 = empty), NULL = off
    int32_t *wb_len, *wb_gen;
    uint8_t *wb_active;
    int64_t *wb_tokens, wb_cap_tok, *wb_out_buf, wb_max_new;
    int exp;                  // SPECDEC_K1_EXP timing experiments (0 = normal)
    int split;                // completion: 0 grid arrival, 1 epilogue kernel, 2 row arrival
    uint32_t *status;
    unsigned long long *ws_keys;  // [B*(k+1)]
    unsigned int *ws_counter;      // [1] grid / row-finish arrivals
    int32_t *ws_lmax;              // [1] split 2: max n' over the still-active rows
    unsigned int *ws_rowcnt;       // [B] split 2: CTA arrivals per batch row
    unsigned long long *ws_w;      // [k+1] split 2 + f3: kept rows per accept class
    // grouped pool verify (specdec_pool_verify_group): the flat batch rows
    // [g_row0[g], g_row0[g+1]) are batch g of the group -- its own logits and drafts, its
    // member / length / active entries at g_off[g] + (row - g_row0[g]) of the plan arrays
    int ngroup;                    // 0: one batch (flat row = member row)
    int32_t g_row0[kMaxGroup + 1];
    int32_t g_off[kMaxGroup];
    const void *g_logits[kMaxGroup];
    const int64_t *g_draft[kMaxGroup];
};

__device__ __forceinline__ int group_of(const VerifyParams &p, int64_t i) {
    int lo = 0, hi = p.ngroup - 1;  // the last g with g_row0[g] <= i
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p.g_row0[mid] <= i) lo = mid; else hi = mid - 1;
    }
    return lo;
}
// the plan-array index (members / lengths / active) of flat batch row i
__device__ __forceinline__ int64_t src_row(const VerifyParams &p, int64_t i) {
    if (!p.ngroup) return i;
    const int g = group_of(p, i);
    return p.g_off[g] + (i - p.g_row0[g]);
}
// logits row (i, j) = flat logits row `row` = i * (k+1) + j
__device__ __forceinline__ const char *logits_row(const VerifyParams &p, int64_t row, int es) {
    if (!p.ngroup) return static_cast<const char *>(p.logits) + row * p.row_stride * es;
    const int64_t K1 = p.k + 1, i = row / K1;
    const int g = group_of(p, i);
    return static_cast<const char *>(p.g_logits[g]) + ((i - p.g_row0[g]) * K1 + row % K1) * p.row_stride * es;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// ----------------------------------------------------------------------------- epilogue
// The epilogue of one batch row, warp-wide (lane j < k+1 holds slot j's key).  RowPre is
// everything it reads besides the keys -- loaded before the arrival so that no load of
// it sits on the critical path after the last CTA of the row arrives.
struct RowPre {
    uint8_t act;
    int32_t n, bud, sq, len0, gen0;  // sq: pool sequence of the row (pool mode), else -1
    int64_t d;                       // lane t < k: draft[i][t]
    int64_t src;                     // the row's index in the plan arrays (src_row)
};

__device__ __forceinline__ RowPre load_pre(const VerifyParams &p, int64_t i, int lane) {
    RowPre r;
    int64_t di = i;
    const int64_t *draft = p.draft;
    r.src = i;
    if (p.ngroup) {
        const int g = group_of(p, i);
        di = i - p.g_row0[g];
        draft = p.g_draft[g];
        r.src = p.g_off[g] + di;
    }
    r.act = p.active[r.src];
    r.n = p.n[r.src];
    r.d = lane < p.k ? draft[di * p.k + lane] : -1;
    r.bud = p.budget ? p.budget[i] : 0;
    r.sq = p.wb_members ? p.wb_members[r.src] : -1;
    r.len0 = r.sq >= 0 ? p.wb_len[r.sq] : 0;
    r.gen0 = r.sq >= 0 ? p.wb_gen[r.sq] : 0;
    return r;
}

struct RowOut {
    int a, nn, kp;
    bool fin;
};

// Alg. 1 lines 3-9 for row i: first mismatch by warp ballot (R1: all k
// match -> a = k), bonus = pred[a] (R2), E = D[:a] ++ [b] cut after the first EOS and to the
// budget (R10), the row's plan entries (n', kept; R6 / R9), and in pool mode the Phase 4
// write-back.  Writes every per-row output and self-cleans the row's keys.
__device__ __forceinline__ RowOut row_epilogue(const VerifyParams &p, int64_t i, const RowPre &r,
                                               unsigned long long key) {
    const int lane = threadIdx.x & 31;
    const int k = static_cast<int>(p.k);
    const int K1 = k + 1;
    const bool act = r.act != 0;
    int a = 0, m = 0, nn = 1, kp = 0;
    int64_t b = p.pad_id;
    bool fin = true;
    const int64_t pr = (act && lane < K1) ? static_cast<int64_t>(unpack_idx(key)) : -1;
    if (p.pred && lane < K1) p.pred[i * K1 + lane] = pr;
    int64_t tok = -1;
    if (act) {
        // first mismatch; R1: all k match -> a = k
        const unsigned mism = __ballot_sync(0xFFFFFFFFu, lane < k && pr != r.d);
        a = mism ? __ffs(mism) - 1 : k;
        b = __shfl_sync(0xFFFFFFFFu, pr, a);  // bonus = pred at the first mismatch (R2)
        // E = D[:a] ++ [b]: lane t < a holds D[t], lane a holds b; cut after the first EOS
        tok = lane < a ? r.d : b;
        m = a + 1;
        fin = false;
        if (p.eos_id >= 0) {
            const unsigned e = __ballot_sync(0xFFFFFFFFu, lane <= a && tok == p.eos_id);
            if (e) { m = __ffs(e); fin = true; }
        }
        if (p.budget) {  // then to the remaining budget (R10)
            const int bud = max(r.bud, 0);
            if (m >= bud) { m = bud; fin = true; }
            if (lane == 0) p.budget[i] = bud - m;  // in/out
        }
        if (!fin) {
            nn = r.n + a + 1;  // accepted + bonus
            kp = r.n + a;      // the bonus has no KV yet
        }
    }
    if (lane < K1) p.ws_keys[i * K1 + lane] = 0ull;  // self-clean
    if (r.sq >= 0) {
        // Alg. 3 Phase 4, as specdec_pool_writeback: E cut to the
        // sequence's remaining budget, appended to its pool tokens / output, len and gen
        // advanced, deactivated when finished
        const int32_t len = r.len0, g = r.gen0;
        const int32_t em = min(m, static_cast<int32_t>(max(static_cast<int64_t>(0), p.wb_max_new - g)));
        const bool fin2 = fin || g + em >= p.wb_max_new;
        if (p.wb_tokens && len + em > p.wb_cap_tok) {
            if (lane == 0 && p.status) atomicOr(p.status, SPECDEC_ST_CAPACITY);
        } else {
            if (lane < em) {
                if (p.wb_tokens) p.wb_tokens[static_cast<int64_t>(r.sq) * p.wb_cap_tok + len + lane] = tok;
                if (p.wb_out_buf) p.wb_out_buf[static_cast<int64_t>(r.sq) * p.wb_max_new + g + lane] = tok;
            }
            if (lane == 0) {
                p.wb_len[r.sq] = len + em;
                p.wb_gen[r.sq] = g + em;
                if (fin2) p.wb_active[r.sq] = 0;
            }
        }
    }
    if (lane == 0) {
        p.accept[i] = a;
        p.bonus[i] = b;
        p.emit[i] = m;
        p.finished[i] = fin ? 1 : 0;
        p.active[r.src] = fin ? 0 : 1;  // in/out: rows still active after this round
        if (p.n_new) p.n_new[i] = nn;
        if (p.kept) p.kept[i] = kp;
        // f1: a draft model that cached its own k forwards (pending token, d_1..d_{k-1})
        // keeps n + min(a, k-1) entries: d_k never had a draft KV entry
        if (p.kept_draft) p.kept_draft[i] = kp ? r.n + min(a, k - 1) : 0;
    }
    return RowOut{a, nn, kp, fin};
}

// f3 (lane 0): move the physical origin to the shift d that leaves the heaviest accept class
// in place (rows with a = d + (L' - L) - 1 do not move); candidates d = 0 first, then larger
// d; feasible iff 0 <= base + d and base + d + L' + k <= anchor_cap; if none is, the
// feasible shift closest to 0.  w[a] = kept rows of accept class a.  Returns base'.
__device__ __forceinline__ int64_t anchor_choose(const VerifyParams &p, const unsigned long long *w,
                                                 int Lnew, int Lold) {
    const int k = static_cast<int>(p.k);
    const int64_t base = *p.anchor;
    unsigned long long total = 0;
    for (int a = 0; a <= k; ++a) total += w[a];
    auto saved = [&](int64_t d) -> unsigned long long {
        const int64_t a = d + (Lnew - Lold) - 1;
        return (a >= 0 && a <= k) ? w[a] : 0ull;
    };
    auto feasible = [&](int64_t d) { return base + d >= 0 && base + d + Lnew + k <= p.anchor_cap; };
    int64_t best = 0;
    unsigned long long best_cost = ~0ull;
    if (Lnew > 0) {
        if (feasible(0)) best_cost = total - saved(0);
        for (int a = k; a >= 0; --a) {  // larger d first
            const int64_t d = (a + 1) - (Lnew - Lold);
            if (d == 0 || !feasible(d)) continue;
            const unsigned long long c = total - w[a];
            if (c < best_cost) { best_cost = c; best = d; }
        }
        if (best_cost == ~0ull) {
            // no candidate fits (the origin sits too high for the grown width): the
            // feasible shift closest to 0 -- every kept row moves, the bound holds
            const int64_t lo = -base, hi = p.anchor_cap - Lnew - k - base;
            if (lo <= hi) best = min(max(static_cast<int64_t>(0), lo), hi);
        }
    }
    return base + best;
}

// All rows in one CTA (the epilogue kernel behind the argmax grid, or the last CTA of the
// grid-wide arrival): one warp per row, then the BatchRepad plan (L', p', f3 origin).
__device__ void verify_epilogue(const VerifyParams &p) {
    __shared__ int s_red[kVerifyThreads / kWarp];
    __shared__ int s_nmax[kVerifyThreads / kWarp];
    __shared__ unsigned long long s_w[kMaxK + 1];  // f3: kept rows per accept class
    __shared__ int s_base[2];
    __shared__ int32_t s_nn[kEpiCache];  // n' of the first rows (no global re-read below)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int K1 = static_cast<int>(p.k) + 1;
    if (threadIdx.x <= kMaxK) s_w[threadIdx.x] = 0ull;
    __syncthreads();
    int local_max = 0, local_nmax = 0;
    for (int64_t i = warp; i < p.B; i += nwarps) {
        // every load of the row first, independent of each other: one memory round trip
        const unsigned long long key = lane < K1 ? __ldcg(p.ws_keys + i * K1 + lane) : 0ull;
        const RowPre r = load_pre(p, i, lane);
        local_nmax = max(local_nmax, r.n);  // old width L = max n (R6 held last round)
        const RowOut o = row_epilogue(p, i, r, key);
        if (!o.fin) local_max = max(local_max, o.nn);
        if (lane == 0) {
            if (i < kEpiCache) s_nn[i] = o.nn;
            if (p.anchor && o.kp) atomicAdd(&s_w[o.a], static_cast<unsigned long long>(o.kp));
        }
    }
    // L' = max n' over still-active rows (R6 minimal padding)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        local_max = max(local_max, __shfl_xor_sync(0xFFFFFFFFu, local_max, o));
        local_nmax = max(local_nmax, __shfl_xor_sync(0xFFFFFFFFu, local_nmax, o));
    }
    if (lane == 0) {
        s_red[warp] = local_max;
        s_nmax[warp] = local_nmax;
    }
    __syncthreads();
    int Lnew = 0, Lold = 0;
    for (int w = 0; w < nwarps; ++w) {
        Lnew = max(Lnew, s_red[w]);
        Lold = max(Lold, s_nmax[w]);
    }
    if (p.anchor && threadIdx.x == 0) {
        s_base[0] = *p.anchor;
        s_base[1] = static_cast<int>(anchor_choose(p, s_w, Lnew, Lold));
        *p.anchor = s_base[1];
    }
    if (p.anchor) __syncthreads();
    for (int64_t i = threadIdx.x; i < p.B && p.pad_new; i += blockDim.x) {
        const int32_t pn = Lnew > 0 ? Lnew - (i < kEpiCache ? s_nn[i] : p.n_new[i]) : 0;
        p.pad_new[i] = pn;
        if (p.anchor) {
            p.phys_old[i] = s_base[0] + (Lold - p.n[i]);
            p.phys_new[i] = s_base[1] + pn;
        }
    }
    if (threadIdx.x == 0) {
        if (p.plan_L) *p.plan_L = Lnew;
        *p.ws_counter = 0u;  // self-clean
    }
}

// The epilogue kernel (one CTA) behind the argmax grid: griddepcontrol.wait returns once
// every argmax CTA has completed and its key atomicMax is visible.
__global__ void __launch_bounds__(kVerifyThreads) verify_epilogue_kernel(VerifyParams p) {
    pdl_wait();
    pdl_launch_dependents();
    verify_epilogue(p);
}

// split == 0: arrival on the grid-wide counter; the last CTA runs the epilogue.
__device__ __forceinline__ void arrive_and_maybe_finish(const VerifyParams &p, int *s_last) {
    if (p.exp == 1 || p.split == 1) return;  // split: the epilogue kernel follows (EXP=1: probe)
    if (threadIdx.x == 0) {
        // acq_rel: releases this CTA's key atomicMax (same thread, cta_merge) and, in the
        // last CTA, acquires every other CTA's -- no separate sequentially-consistent fences
        const unsigned int total = gridDim.x * gridDim.y;
        unsigned int prev;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.ws_counter) : "memory");
        *s_last = (prev == total - 1);
    }
    __syncthreads();
    if (!*s_last) return;
    if (p.exp == 6) {  // timing experiment only: the arrival, no epilogue (self-clean kept)
        if (threadIdx.x == 0) *p.ws_counter = 0u;
        for (int64_t x = threadIdx.x; x < p.B * (p.k + 1); x += blockDim.x) p.ws_keys[x] = 0ull;
        return;
    }
    verify_epilogue(p);
}

// The plan after every row's epilogue (warp-wide, run by the last row to finish):
// L' = max n' over still-active rows (accumulated in ws_lmax), p'_i = L' - n'_i, the f3
// origin from the accept-class weights in ws_w, plan_L.  Self-cleans the plan words.
__device__ void plan_finalize_warp(const VerifyParams &p) {
    __shared__ unsigned long long s_w[kMaxK + 1];
    __shared__ int s_base[2];
    const int lane = threadIdx.x & 31;
    const int K1 = static_cast<int>(p.k) + 1;
    __syncwarp();
    const int Lnew = __ldcg(p.ws_lmax);
    int Lold = 0;
    for (int64_t t = lane; t < p.B; t += 32) Lold = max(Lold, __ldcg(p.n + t));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Lold = max(Lold, __shfl_xor_sync(0xFFFFFFFFu, Lold, o));
    if (p.anchor) {
        if (lane < K1) {
            s_w[lane] = __ldcg(p.ws_w + lane);
            p.ws_w[lane] = 0ull;  // self-clean
        }
        __syncwarp();
        if (lane == 0) {
            s_base[0] = *p.anchor;
            s_base[1] = static_cast<int>(anchor_choose(p, s_w, Lnew, Lold));
            *p.anchor = s_base[1];
        }
        __syncwarp();
    }
    for (int64_t t = lane; t < p.B; t += 32) {
        const int32_t pn = Lnew > 0 ? Lnew - __ldcg(p.n_new + t) : 0;
        p.pad_new[t] = pn;
        if (p.anchor) {
            p.phys_old[t] = s_base[0] + (Lold - __ldcg(p.n + t));
            p.phys_new[t] = s_base[1] + pn;
        }
    }
    if (lane == 0) {
        *p.plan_L = Lnew;
        *p.ws_lmax = 0;        // self-clean
        *p.ws_counter = 0u;
    }
}

// split == 2: arrival on the batch row's counter ((k+1) x chunks CTAs per row).  The last
// CTA of row i runs that row's epilogue at once (warp 0, with the row inputs prefetched
// before the arrival); in pool mode that is all.  With a plan to build, the row then
// arrives on the grid counter (one arrival per batch row) and the last row writes p', L'.
__device__ __forceinline__ void row_arrive_and_finish(const VerifyParams &p, int64_t i, const RowPre *s_pre,
                                                      int *s_last) {
    const int K1 = static_cast<int>(p.k) + 1;
    if (threadIdx.x == 0) {
        const unsigned int total = static_cast<unsigned int>(K1) * gridDim.x;
        unsigned int prev;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.ws_rowcnt + i) : "memory");
        *s_last = (prev == total - 1);
    }
    __syncthreads();
    if (!*s_last || threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const unsigned long long key = lane < K1 ? __ldcg(p.ws_keys + i * K1 + lane) : 0ull;
    const RowOut o = row_epilogue(p, i, s_pre[lane], key);
    unsigned last = 0;
    if (lane == 0) {
        p.ws_rowcnt[i] = 0u;  // self-clean
        if (p.plan_L) {
            if (!o.fin) atomicMax(p.ws_lmax, o.nn);
            if (p.anchor && o.kp) atomicAdd(p.ws_w + o.a, static_cast<unsigned long long>(o.kp));
            unsigned int prev;
            asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.ws_counter) : "memory");
            last = prev == static_cast<unsigned int>(p.B) - 1;
        }
    }
    if (__shfl_sync(0xFFFFFFFFu, last, 0)) plan_finalize_warp(p);
}

__device__ __forceinline__ void cta_merge(const VerifyParams &p, int64_t row, unsigned long long best,
                                          unsigned long long *s_red) {
    const int tid = threadIdx.x;
    best = warp_max_u64(best);
    if ((tid & 31) == 0) s_red[tid >> 5] = best;
    __syncthreads();
    if (tid < kWarp) {
        unsigned long long v = tid < kVerifyThreads / kWarp ? s_red[tid] : 0ull;
        v = warp_max_u64(v);
        if (tid == 0) {
            atomicMax(p.ws_keys + row, v);
            if ((v >> 32) == 0xFFFFFFFFull && p.status) atomicOr(p.status, SPECDEC_ST_NAN);
        }
    }
}

// After the CTA's merge: the configured completion (epilogue kernel / grid arrival / row
// arrival).  s_pre (shared) holds warp 0's row inputs when p.split == 2.
__device__ __forceinline__ void finish_cta(const VerifyParams &p, int64_t i, const RowPre *s_pre, int *s_last) {
    if (p.split == 2) row_arrive_and_finish(p, i, s_pre, s_last);
    else arrive_and_maybe_finish(p, s_last);
}

// ----------------------------------------------------------------------------- fp32 (toy)
// Per-element keys, strict '>' over ascending indices within a thread.
__global__ void __launch_bounds__(kVerifyThreads) verify_kernel_f32(VerifyParams p) {
    pdl_wait();
    pdl_launch_dependents();
    __shared__ unsigned long long s_red[kVerifyThreads / kWarp];
    __shared__ int s_last;
    __shared__ RowPre s_pre[kWarp];
    const int tid = threadIdx.x;
    const int64_t row = blockIdx.y;
    const int64_t i = row / (p.k + 1);
    if (p.split == 2 && tid < kWarp) s_pre[tid] = load_pre(p, i, tid);
    const bool act = p.active[src_row(p, i)] != 0;
    {
        const char *rowp = logits_row(p, row, 4);
        const int64_t v0 = static_cast<int64_t>(blockIdx.x) * p.chunk;
        const int64_t v1 = min(p.V, v0 + p.chunk);
        const int64_t vec_end = v1 / 4;
        uint32_t bk = 0, bi = 0;
        for (int64_t vb = v0 / 4 + tid; vb < vec_end; vb += kVerifyThreads) {
            const uint4 w = ld_stream_v4(rowp + vb * 16);
            const uint32_t e[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t kk = key32(e[q]);
                if (kk > bk) { bk = kk; bi = static_cast<uint32_t>(vb * 4 + q); }
            }
        }
        for (int64_t v = max(vec_end * 4, v0) + tid; v < v1; v += kVerifyThreads) {
            const uint32_t kk = key32(reinterpret_cast<const uint32_t *>(rowp)[v]);
            if (kk > bk || (kk == bk && static_cast<uint32_t>(v) < bi)) { bk = kk; bi = static_cast<uint32_t>(v); }
        }
        if (act) cta_merge(p, row, bk ? pack_key(bk, bi) : 0ull, s_red);
    }
    finish_cta(p, i, s_pre, &s_last);
}

// ----------------------------------------------------------------------------- fp16 / bf16
// Pass 1 streams the chunk keeping only a packed pair maximum with NaN propagation
// (HMNMX2: one instruction per two logits), reduced over the CTA -> M.  Pass 2 runs only
// in threads whose own maximum has key(M) (usually one): they re-read their elements
// (L2-resident, 14.6 MB << 126 MB) and report the first one whose key equals key(M) --
// keys make +0 == -0 and NaN == NaN, exactly the argmax equality of R4/R5.
template <bool BF16>
struct H16 {
    __device__ static uint32_t max2(uint32_t a, uint32_t b) {
        if constexpr (BF16) {
            __nv_bfloat162 r = __hmax2_nan(*reinterpret_cast<__nv_bfloat162 *>(&a),
                                           *reinterpret_cast<__nv_bfloat162 *>(&b));
            return *reinterpret_cast<uint32_t *>(&r);
        } else {
            __half2 r = __hmax2_nan(*reinterpret_cast<__half2 *>(&a), *reinterpret_cast<__half2 *>(&b));
            return *reinterpret_cast<uint32_t *>(&r);
        }
    }
    // 0xFFFF in each half where a == b (native packed compare, set.eq.u32.{bf16x2,f16x2})
    __device__ static uint32_t eq2(uint32_t a, uint32_t b) {
        if constexpr (BF16)
            return __heq2_mask(*reinterpret_cast<__nv_bfloat162 *>(&a), *reinterpret_cast<__nv_bfloat162 *>(&b));
        else
            return __heq2_mask(*reinterpret_cast<__half2 *>(&a), *reinterpret_cast<__half2 *>(&b));
    }
    __device__ static uint32_t vmax(const uint4 &v) { return max2(max2(v.x, v.y), max2(v.z, v.w)); }
    // the maximum of the two halves, as 16 bits
    __device__ static uint32_t fold(uint32_t m2) { return max2(m2, (m2 >> 16) | (m2 << 16)) & 0xFFFFu; }
    static constexpr uint32_t kExp = BF16 ? 0x7F80u : 0x7C00u;
    static constexpr uint32_t kNegInf2 = BF16 ? 0xFF80FF80u : 0xFC00FC00u;
};

constexpr int kVPT = 8;  // 16-byte vectors per thread, all in flight, kept in registers

template <bool BF16>
__global__ void __launch_bounds__(kVerifyThreads, 4) verify_kernel16(VerifyParams p) {
    pdl_wait();                // the logits' producer (and the previous round) completed
    pdl_launch_dependents();
    if (p.exp == 2) return;    // timing experiment only: the launch floor of this grid
    using T = H16<BF16>;
    __shared__ uint32_t s_c[kVerifyThreads / kWarp];
    __shared__ int s_last;
    __shared__ RowPre s_pre[kWarp];  // split 2: the row's epilogue inputs, per lane of warp 0
    bool act = false;
    const int tid = threadIdx.x;
    const int64_t row = blockIdx.y;
    const int64_t i = row / (p.k + 1);
    {
        // the loads are issued before anything else is read (an inactive row's logits are
        // streamed too -- its CTAs just do not merge): no dependent load ahead of them
        const char *rowp = logits_row(p, row, 2);
        const int64_t v0 = static_cast<int64_t>(blockIdx.x) * p.chunk;
        const int64_t v1 = min(p.V, v0 + p.chunk);
        const int64_t vec0 = v0 / 8, vec_end = v1 / 8;
        // this thread's vectors: vec0 + tid + u*256, u < mine (<= kVPT by the host's chunk)
        const int nvec = static_cast<int>(vec_end - vec0);
        const int mine = nvec > tid ? (nvec - tid + kVerifyThreads - 1) / kVerifyThreads : 0;
        const uint4 *vp = reinterpret_cast<const uint4 *>(rowp) + vec0 + tid;
        uint4 w[kVPT];
#pragma unroll
        for (int u = 0; u < kVPT; ++u)
            w[u] = u < mine ? ld_stream_v4(vp + u * kVerifyThreads)
                            : make_uint4(T::kNegInf2, T::kNegInf2, T::kNegInf2, T::kNegInf2);
        if (p.split == 2 && tid < kWarp) s_pre[tid] = load_pre(p, i, tid);
        act = p.active[src_row(p, i)] != 0;
        // pass 1: the thread's packed maximum (HMNMX2: one instruction per two logits,
        // NaN-propagating)
        uint32_t m2 = T::kNegInf2;
#pragma unroll
        for (int u = 0; u < kVPT; ++u) m2 = T::max2(m2, T::vmax(w[u]));
        const int64_t tail0 = max(vec_end * 8, v0);  // ragged tail (V % 8), scalar
        for (int64_t v = tail0 + tid; v < v1; v += kVerifyThreads) {
            const uint32_t x = reinterpret_cast<const uint16_t *>(rowp)[v];
            m2 = T::max2(m2, x | (x << 16));
        }
        const uint32_t my_m = T::fold(m2);
        if (p.exp == 3) {  // timing experiment only: stream + per-thread max, no CTA reduction
            if (my_m == 0x7FFFu && p.status) atomicOr(p.status, 0x80000000u);
            return;
        }
        // pass 2, per thread (no CTA maximum first): the first of its vectors whose maximum
        // equals my_m, then the first element of that vector that does.  An ordinary
        // maximum (not NaN, not +-0) matches by bits; the special ones by key (+0 == -0,
        // NaN == NaN: the argmax equality of R4/R5).
        const uint32_t kM = key16s(my_m, T::kExp);
        const bool plain = (my_m & 0x7FFFu) != 0 && (my_m & 0x7FFFu) <= T::kExp;
        int ustar = -1;
#pragma unroll
        for (int u = kVPT - 1; u >= 0; --u) {
            const uint32_t fu = T::fold(T::vmax(w[u]));  // recomputed: registers stay <= 64
            if (u < mine && (plain ? fu == my_m : key16s(fu, T::kExp) == kM)) ustar = u;
        }
        if (p.exp == 4) {  // timing experiment only: + the first matching vector
            if (ustar == 100 && p.status) atomicOr(p.status, 0x80000000u);
            return;
        }
        // CTA-local packed candidate: (key << 16) | (0xFFFF - index in the chunk) -- the
        // unsigned max is "largest key, then lowest index" (chunk <= 16384 logits)
        uint32_t cand = 0u;
        if (ustar >= 0) {
            uint4 x = w[0];
#pragma unroll
            for (int u = 1; u < kVPT; ++u)
                if (u == ustar) x = w[u];
            int j;
            if (plain) {
                // one packed compare per word (0xFFFF per equal half), two byte permutes: 8
                // flag bytes, byte j set iff half j equals M; the lowest flag is the first
                const uint32_t mm = my_m | (my_m << 16);
                const uint32_t lo = __byte_perm(T::eq2(x.x, mm), T::eq2(x.y, mm), 0x6420);
                const uint32_t hi = __byte_perm(T::eq2(x.z, mm), T::eq2(x.w, mm), 0x6420);
                j = lo ? (__ffs(lo) - 1) >> 3 : 4 + ((__ffs(hi) - 1) >> 3);
            } else {
                const uint32_t e[4] = {x.x, x.y, x.z, x.w};
                j = 7;
#pragma unroll
                for (int q = 3; q >= 0; --q) {
                    if (key16s(e[q] >> 16, T::kExp) == kM) j = 2 * q + 1;
                    if (key16s(e[q] & 0xFFFFu, T::kExp) == kM) j = 2 * q;
                }
            }
            const int64_t e = (vec0 + tid + static_cast<int64_t>(ustar) * kVerifyThreads) * 8 + j;
            cand = (kM << 16) | (0xFFFFu - static_cast<uint32_t>(e - v0));
        } else {
            for (int64_t v = tail0 + tid; v < v1; v += kVerifyThreads)
                if (key16s(reinterpret_cast<const uint16_t *>(rowp)[v], T::kExp) == kM) {
                    cand = (kM << 16) | (0xFFFFu - static_cast<uint32_t>(v - v0));
                    break;
                }
        }
        if (p.exp == 5) {  // timing experiment only: up to pass 2, no merge
            if (cand == 1u && p.status) atomicOr(p.status, 0x80000000u);
            return;
        }
        // CTA maximum of the candidates (redux.sync), then one 64-bit atomicMax per CTA
        cand = __reduce_max_sync(0xFFFFFFFFu, cand);
        if ((tid & 31) == 0) s_c[tid >> 5] = cand;
        __syncthreads();
        if (tid < kWarp) {
            cand = __reduce_max_sync(0xFFFFFFFFu, tid < kVerifyThreads / kWarp ? s_c[tid] : 0u);
            if (tid == 0 && act && cand) {
                const uint32_t key = cand >> 16;
                atomicMax(p.ws_keys + row, pack_key(key, static_cast<uint32_t>(v0 + (0xFFFFu - (cand & 0xFFFFu)))));
                if (key == 0xFFFFu && p.status) atomicOr(p.status, SPECDEC_ST_NAN);
            }
        }
    }
    finish_cta(p, i, s_pre, &s_last);
}

}  // namespace specdec

using namespace specdec;

// Workspace: keys [B*(k+1)] u64 | grid counter u32, max n' i32, 8 pad | row counters [B]
// u32 (padded to 8) | accept-class weights [k+1] u64.
static size_t ws_rowcnt_off(int64_t B, int64_t k) { return static_cast<size_t>(B * (k + 1)) * 8 + 16; }
static size_t ws_w_off(int64_t B, int64_t k) { return ws_rowcnt_off(B, k) + static_cast<size_t>((B * 4 + 7) / 8 * 8); }

extern "C" size_t specdec_verify_workspace_size(int64_t B, int64_t k) {
    if (B < 1 || k < 1) return 0;
    return ws_w_off(B, k) + static_cast<size_t>(k + 1) * 8;
}

namespace specdec {

static void set_ws(VerifyParams &p, void *d_ws) {
    char *w = static_cast<char *>(d_ws);
    p.ws_keys = reinterpret_cast<unsigned long long *>(w);
    p.ws_counter = reinterpret_cast<unsigned int *>(w + p.B * (p.k + 1) * 8);
    p.ws_lmax = reinterpret_cast<int32_t *>(w + p.B * (p.k + 1) * 8 + 4);
    p.ws_rowcnt = reinterpret_cast<unsigned int *>(w + ws_rowcnt_off(p.B, p.k));
    p.ws_w = reinterpret_cast<unsigned long long *>(w + ws_w_off(p.B, p.k));
}

// Common host path of specdec_verify / specdec_pool_verify: shape checks done by the
// callers, p filled except the launch geometry.
static int launch_verify(VerifyParams &p, int dtype, int es, specdec_stream_t stream) {
    static int exp = -1, cta_mult = 4, vpt = 0, split_eq = kSplitEqSpec, split_pool = kSplitPool;
    if (exp < 0) {
        const char *e = getenv("SPECDEC_K1_EXP");
        exp = e ? atoi(e) : 0;
        // completion mode override "E[,P]" (EqSpec verify, pool verify): 0 grid-wide
        // arrival, 1 epilogue kernel, 2 per-row arrival
        if (const char *sp = getenv("SPECDEC_K1_SPLIT")) {
            split_eq = atoi(sp);
            const char *c2 = strchr(sp, ',');
            split_pool = c2 ? atoi(c2 + 1) : split_eq;
        }
        const char *c = getenv("SPECDEC_K1_CTAS");  // tuning override: target CTAs per SM
        if (c && atoi(c) > 0) cta_mult = atoi(c);
        const char *v = getenv("SPECDEC_K1_VPT");   // tuning override: 16-B vectors per thread
        if (v && atoi(v) > 0) vpt = std::min(atoi(v), kVPT);
    }
    p.exp = exp;
    const int64_t B = p.B, k = p.k, V = p.V;
    const int VE = 16 / es;
    const int64_t rows = B * (k + 1);
    const int64_t quantum = static_cast<int64_t>(kVerifyThreads) * VE;
    const int64_t sms = device_sm_count();
    int64_t chunk;
    if (es == 2) {
        // 16-bit logits, register-resident: as many 16-B vectors per thread as possible (fewer
        // CTAs = fewer merges and arrivals on the latency-bound path) while the grid still
        // covers >= 3/4 of the SMs.  Sweep (profiles/r01/k1_sweep.txt): best or within 3 %
        // of best at B = 1, 2, 4, 8, 16.
        int v = kVPT;
        for (const int c : {8, 6, 4, 3, 2, 1}) {
            v = c;
            if (rows * ((V + quantum * c - 1) / (quantum * c)) * 4 >= 3 * sms) break;
        }
        if (vpt > 0) v = vpt;
        chunk = quantum * v;
    } else {
        // fp32 (strided loop): about cta_mult CTAs per SM in one wave, no tail wave
        const int64_t per_row = std::max<int64_t>(1, cta_mult * sms / rows);  // CTAs per (row, slot)
        chunk = (V + per_row - 1) / per_row;
        chunk = std::max<int64_t>(quantum, (chunk + quantum - 1) / quantum * quantum);
    }
    p.chunk = chunk;
    const int64_t n_chunks = (V + chunk - 1) / chunk;
    dim3 grid(static_cast<unsigned>(n_chunks), static_cast<unsigned>(rows));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    p.split = exp ? 0 : (p.wb_members ? split_pool : split_eq);  // the probes: grid arrival
    if (p.split == 1) {
        int rc;
        switch (dtype) {
            case SPECDEC_F32: rc = launch_k(verify_kernel_f32, grid, dim3(kVerifyThreads), 0, s, p); break;
            case SPECDEC_F16: rc = launch_k(verify_kernel16<false>, grid, dim3(kVerifyThreads), 0, s, p); break;
            default: rc = launch_k(verify_kernel16<true>, grid, dim3(kVerifyThreads), 0, s, p);
        }
        if (rc) return rc;
        return launch_k(verify_epilogue_kernel, dim3(1), dim3(kVerifyThreads), 0, s, p);
    }
    switch (dtype) {
        case SPECDEC_F32: return launch_k(verify_kernel_f32, grid, dim3(kVerifyThreads), 0, s, p);
        case SPECDEC_F16: return launch_k(verify_kernel16<false>, grid, dim3(kVerifyThreads), 0, s, p);
        default: return launch_k(verify_kernel16<true>, grid, dim3(kVerifyThreads), 0, s, p);
    }
}

}  // namespace specdec

extern "C" int specdec_verify_kernels(int pool) {
    static int split_eq = -1, split_pool = -1;
    if (split_eq < 0) {
        split_eq = kSplitEqSpec;
        split_pool = kSplitPool;
        if (const char *sp = getenv("SPECDEC_K1_SPLIT")) {
            split_eq = atoi(sp);
            const char *c2 = strchr(sp, ',');
            split_pool = c2 ? atoi(c2 + 1) : split_eq;
        }
    }
    return (pool ? split_pool : split_eq) == 1 ? 2 : 1;
}

namespace specdec {

// shape / pointer checks shared by both entry points
static int check_verify(const void *d_logits, int es, int64_t B, int64_t k, int64_t V,
                        int64_t row_stride, void *d_ws, size_t ws_bytes) {
    if (es == 0) return SPECDEC_ERR_DTYPE;
    if (k < 1 || k > kMaxK) return SPECDEC_ERR_ARG;
    if (B < 1 || V < 1 || row_stride < V || V > 0x7FFFFFFFll) return SPECDEC_ERR_SHAPE;
    if (B * (k + 1) > 65535) return SPECDEC_ERR_SHAPE;  // gridDim.y
    if (!d_logits || !d_ws) return SPECDEC_ERR_ARG;
    if (!aligned16(d_logits) || (row_stride * es) % 16 != 0 || (reinterpret_cast<uintptr_t>(d_ws) & 7u))
        return SPECDEC_ERR_ARG;
    if (ws_bytes < specdec_verify_workspace_size(B, k)) return SPECDEC_ERR_ARG;
    return SPECDEC_OK;
}

}  // namespace specdec

extern "C" int specdec_verify(const void *d_logits, int dtype, int64_t B, int64_t k, int64_t V,
                              int64_t row_stride, const int64_t *d_draft, const int32_t *d_n,
                              uint8_t *d_active, int64_t eos_id, int64_t pad_id,
                              int32_t *d_budget, int32_t *d_accept, int64_t *d_bonus,
                              int32_t *d_emit, uint8_t *d_finished, int64_t *d_pred,
                              int32_t *d_plan_L, int32_t *d_n_new, int32_t *d_pad_new,
                              int32_t *d_kept, int32_t *d_kept_draft, int32_t *d_anchor,
                              int64_t anchor_cap, int32_t *d_phys_old, int32_t *d_phys_new,
                              uint32_t *d_status, void *d_ws, size_t ws_bytes,
                              specdec_stream_t stream) {
    const int es = dtype_size(dtype);
    if (d_anchor && (!d_phys_old || !d_phys_new || anchor_cap < k + 2)) return SPECDEC_ERR_ARG;
    const int rc = check_verify(d_logits, es, B, k, V, row_stride, d_ws, ws_bytes);
    if (rc) return rc;
    if (!d_draft || !d_n || !d_active || !d_accept || !d_bonus || !d_emit || !d_finished ||
        !d_plan_L || !d_n_new || !d_pad_new || !d_kept)
        return SPECDEC_ERR_ARG;
    VerifyParams p{};
    p.logits = d_logits;
    p.B = B; p.k = k; p.V = V; p.row_stride = row_stride;
    p.draft = d_draft; p.n = d_n; p.active = d_active;
    p.eos_id = eos_id; p.pad_id = pad_id; p.budget = d_budget;
    p.accept = d_accept; p.bonus = d_bonus; p.emit = d_emit; p.finished = d_finished;
    p.pred = d_pred; p.plan_L = d_plan_L; p.n_new = d_n_new; p.pad_new = d_pad_new; p.kept = d_kept;
    p.kept_draft = d_kept_draft;
    p.anchor = d_anchor; p.anchor_cap = anchor_cap; p.phys_old = d_phys_old; p.phys_new = d_phys_new;
    p.status = d_status;
    set_ws(p, d_ws);
    return launch_verify(p, dtype, es, stream);
}

extern "C" int specdec_pool_verify(const void *d_logits, int dtype, int64_t B, int64_t k,
                                   int64_t V, int64_t row_stride, const int64_t *d_draft,
                                   const int32_t *d_members, const int32_t *d_mlen,
                                   uint8_t *d_mactive, int64_t eos_id, int64_t pad_id,
                                   int32_t *d_accept, int64_t *d_bonus, int32_t *d_emit,
                                   uint8_t *d_finished, int32_t *d_pool_len, int32_t *d_pool_gen,
                                   uint8_t *d_pool_active, int64_t *d_pool_tokens, int64_t cap_tok,
                                   int64_t *d_out_buf, int64_t max_new, uint32_t *d_status,
                                   void *d_ws, size_t ws_bytes, specdec_stream_t stream) {
    const int es = dtype_size(dtype);
    const int rc = check_verify(d_logits, es, B, k, V, row_stride, d_ws, ws_bytes);
    if (rc) return rc;
    if (!d_draft || !d_members || !d_mlen || !d_mactive || !d_accept || !d_bonus || !d_emit ||
        !d_finished || !d_pool_len || !d_pool_gen || !d_pool_active)
        return SPECDEC_ERR_ARG;
    if (d_pool_tokens && cap_tok < 1) return SPECDEC_ERR_SHAPE;
    if (max_new < 1) return SPECDEC_ERR_SHAPE;
    VerifyParams p{};
    p.logits = d_logits;
    p.B = B; p.k = k; p.V = V; p.row_stride = row_stride;
    p.draft = d_draft; p.n = d_mlen; p.active = d_mactive;
    p.eos_id = eos_id; p.pad_id = pad_id;
    p.accept = d_accept; p.bonus = d_bonus; p.emit = d_emit; p.finished = d_finished;
    p.wb_members = d_members; p.wb_len = d_pool_len; p.wb_gen = d_pool_gen; p.wb_active = d_pool_active;
    p.wb_tokens = d_pool_tokens; p.wb_cap_tok = cap_tok; p.wb_out_buf = d_out_buf; p.wb_max_new = max_new;
    p.status = d_status;
    set_ws(p, d_ws);
    return launch_verify(p, dtype, es, stream);
}

extern "C" int specdec_pool_verify_group(int32_t n_batches, const void *const *h_logits,
                                         const int64_t *const *h_draft, const int32_t *h_offset,
                                         const int32_t *h_rows, int dtype, int64_t k, int64_t V,
                                         int64_t row_stride, const int32_t *d_members,
                                         const int32_t *d_mlen, uint8_t *d_mactive, int64_t eos_id,
                                         int64_t pad_id, int32_t *d_accept, int64_t *d_bonus,
                                         int32_t *d_emit, uint8_t *d_finished, int32_t *d_pool_len,
                                         int32_t *d_pool_gen, uint8_t *d_pool_active,
                                         int64_t *d_pool_tokens, int64_t cap_tok, int64_t *d_out_buf,
                                         int64_t max_new, uint32_t *d_status, void *d_ws,
                                         size_t ws_bytes, specdec_stream_t stream) {
    if (n_batches < 1 || n_batches > kMaxGroup || !h_logits || !h_draft || !h_offset || !h_rows)
        return SPECDEC_ERR_ARG;
    const int es = dtype_size(dtype);
    int64_t R = 0;
    for (int32_t g = 0; g < n_batches; ++g) {
        if (h_rows[g] < 1 || h_offset[g] < 0) return SPECDEC_ERR_SHAPE;
        if (!h_logits[g] || !h_draft[g] || !aligned16(h_logits[g])) return SPECDEC_ERR_ARG;
        R += h_rows[g];
    }
    // the shape checks of one launch over R flat rows (logits pointer: the first batch's)
    const int rc = check_verify(h_logits[0], es, R, k, V, row_stride, d_ws, ws_bytes);
    if (rc) return rc;
    if (!d_members || !d_mlen || !d_mactive || !d_accept || !d_bonus || !d_emit || !d_finished ||
        !d_pool_len || !d_pool_gen || !d_pool_active)
        return SPECDEC_ERR_ARG;
    if (d_pool_tokens && cap_tok < 1) return SPECDEC_ERR_SHAPE;
    if (max_new < 1) return SPECDEC_ERR_SHAPE;
    VerifyParams p{};
    p.logits = h_logits[0];
    p.B = R; p.k = k; p.V = V; p.row_stride = row_stride;
    p.draft = h_draft[0]; p.n = d_mlen; p.active = d_mactive;
    p.eos_id = eos_id; p.pad_id = pad_id;
    p.accept = d_accept; p.bonus = d_bonus; p.emit = d_emit; p.finished = d_finished;
    p.wb_members = d_members; p.wb_len = d_pool_len; p.wb_gen = d_pool_gen; p.wb_active = d_pool_active;
    p.wb_tokens = d_pool_tokens; p.wb_cap_tok = cap_tok; p.wb_out_buf = d_out_buf; p.wb_max_new = max_new;
    p.status = d_status;
    p.ngroup = n_batches;
    int32_t r0 = 0;
    for (int32_t g = 0; g < n_batches; ++g) {
        p.g_row0[g] = r0;
        p.g_off[g] = h_offset[g];
        p.g_logits[g] = h_logits[g];
        p.g_draft[g] = h_draft[g];
        r0 += h_rows[g];
    }
    p.g_row0[n_batches] = r0;
    set_ws(p, d_ws);
    return launch_verify(p, dtype, es, stream);
}
