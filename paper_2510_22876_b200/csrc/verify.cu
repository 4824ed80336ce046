// verify.cu -- K1: Alg. 1 BatchVerify fused with the BatchRepad plan
// (§3.1).
//
// One pass over the logits tail [B][k+1][V]: every CTA scans one vocab chunk of one
// (row, slot) with 128-bit streaming loads, reduces to a packed (key, ~index) 64-bit
// maximum and merges it with one atomicMax (order-independent => bit-exact argmax with
// lowest-index ties, first-NaN rule).  The last CTA to arrive (acq/rel counter) runs the
// epilogue: first-mismatch scan (PAPER.md:304-306 with R1), bonus (R2), EOS/budget
// trim (R10) and the repad plan (L', p', kept) -- no host round trip, no second launch.
// The workspace is left zeroed for the next call.
#include <cuda_runtime.h>

#include <algorithm>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "host_util.h"

namespace specdec {

constexpr int kVerifyThreads = 256;

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
    int32_t *plan_L, *n_new, *pad_new, *kept;
    uint32_t *status;
    unsigned long long *ws_keys;  // [B*(k+1)]
    unsigned int *ws_counter;      // [1]
};

// Elements per 16-byte vector and key function per dtype.
template <int DT>
struct Lane;
template <>
struct Lane<SPECDEC_F32> {
    static constexpr int VE = 4;
    __device__ static void scan(const uint4 &w, uint32_t base, uint32_t &bk, uint32_t &bi) {
        const uint32_t e[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t kk = key32(e[q]);
            if (kk > bk) { bk = kk; bi = base + q; }
        }
    }
    __device__ static uint32_t key_at(const void *row, int64_t v) {
        return key32(reinterpret_cast<const uint32_t *>(row)[v]);
    }
};
template <uint32_t EXP1>
struct Lane16 {
    static constexpr int VE = 8;
    __device__ static void scan(const uint4 &w, uint32_t base, uint32_t &bk, uint32_t &bi) {
        const uint32_t e[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t lo = key16(e[q] & 0xFFFFu, EXP1);
            if (lo > bk) { bk = lo; bi = base + 2 * q; }
            const uint32_t hi = key16(e[q] >> 16, EXP1);
            if (hi > bk) { bk = hi; bi = base + 2 * q + 1; }
        }
    }
    __device__ static uint32_t key_at(const void *row, int64_t v) {
        return key16(reinterpret_cast<const uint16_t *>(row)[v], EXP1);
    }
};
template <>
struct Lane<SPECDEC_F16> : Lane16<0x7C00u> {};
template <>
struct Lane<SPECDEC_BF16> : Lane16<0x7F80u> {};

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

__device__ void verify_epilogue(const VerifyParams &p) {
    __shared__ int s_red[kVerifyThreads / kWarp];
    const int tid = threadIdx.x;
    const int64_t K1 = p.k + 1;
    int local_max = 0;
    for (int64_t i = tid; i < p.B; i += blockDim.x) {
        int32_t a = 0, m = 0, nn = 1, kp = 0;
        int64_t b = p.pad_id;
        uint8_t fin = 1;
        if (p.active[i]) {
            const int64_t *d = p.draft + i * p.k;
            int64_t pr_a = -1;
            a = static_cast<int32_t>(p.k);
            // first mismatch; R1: all k match -> a = k
            for (int64_t j = 0; j <= p.k; ++j) {
                const int64_t pr = unpack_idx(__ldcg(p.ws_keys + i * K1 + j));
                if (p.pred) p.pred[i * K1 + j] = pr;
                if (j < p.k && a == p.k && pr != d[j]) a = static_cast<int32_t>(j);
            }
            pr_a = unpack_idx(__ldcg(p.ws_keys + i * K1 + a));
            b = pr_a;  // bonus = pred at the first mismatch (R2)
            // E = D[:a] ++ [b]; cut after the first EOS, then to the budget (R10)
            m = a + 1;
            fin = 0;
            if (p.eos_id >= 0) {
                for (int32_t t = 0; t <= a; ++t) {
                    const int64_t tok = t < a ? d[t] : b;
                    if (tok == p.eos_id) { m = t + 1; fin = 1; break; }
                }
            }
            if (p.budget) {
                const int32_t bud = max(p.budget[i], 0);
                if (m >= bud) { m = bud; fin = 1; }
                p.budget[i] = bud - m;  // in/out: remaining budget after this round
            }
            if (!fin) {
                nn = p.n[i] + a + 1;
                kp = p.n[i] + a;
                local_max = max(local_max, nn);
            }
        } else if (p.pred) {
            for (int64_t j = 0; j <= p.k; ++j) p.pred[i * K1 + j] = -1;
        }
        for (int64_t j = 0; j <= p.k; ++j) p.ws_keys[i * K1 + j] = 0ull;  // self-clean
        p.accept[i] = a;
        p.bonus[i] = b;
        p.emit[i] = m;
        p.finished[i] = fin;
        p.active[i] = fin ? 0 : 1;  // in/out: rows still active after this round
        p.n_new[i] = nn;
        p.kept[i] = kp;
    }
    // L' = max n' over still-active rows (R6 minimal padding)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local_max = max(local_max, __shfl_xor_sync(0xFFFFFFFFu, local_max, o));
    if ((tid & 31) == 0) s_red[tid >> 5] = local_max;
    __syncthreads();
    if (tid < kWarp) {
        int v = tid < blockDim.x / kWarp ? s_red[tid] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
        if (tid == 0) s_red[0] = v;
    }
    __syncthreads();
    const int Lnew = s_red[0];
    for (int64_t i = tid; i < p.B; i += blockDim.x) p.pad_new[i] = Lnew > 0 ? Lnew - p.n_new[i] : 0;
    if (tid == 0) {
        *p.plan_L = Lnew;
        *p.ws_counter = 0u;  // self-clean
    }
}

// Arrival on the grid-wide counter; the last CTA runs the epilogue.
__device__ __forceinline__ void arrive_and_maybe_finish(const VerifyParams &p, int *s_last) {
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int total = gridDim.x * gridDim.y;
        const unsigned int prev = atomicAdd(p.ws_counter, 1u);
        *s_last = (prev == total - 1);
    }
    __syncthreads();
    if (!*s_last) return;
    __threadfence();
    verify_epilogue(p);
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

// fp32 logits (toy config): per-element keys, strict '>' in ascending index order.
__global__ void __launch_bounds__(kVerifyThreads) verify_kernel_f32(VerifyParams p) {
    using L = Lane<SPECDEC_F32>;
    constexpr int VE = L::VE;
    __shared__ unsigned long long s_red[kVerifyThreads / kWarp];
    __shared__ int s_last;
    const int tid = threadIdx.x;
    const int64_t row = blockIdx.y;
    const int64_t i = row / (p.k + 1);
    if (p.active[i]) {
        const char *rowp = static_cast<const char *>(p.logits) + row * p.row_stride * 4;
        const int64_t v0 = static_cast<int64_t>(blockIdx.x) * p.chunk;
        const int64_t v1 = min(p.V, v0 + p.chunk);
        const int64_t vec_end = v1 / VE;
        uint32_t bk = 0, bi = 0;
        for (int64_t vb = v0 / VE + tid; vb < vec_end; vb += kVerifyThreads)
            L::scan(ld_stream_v4(rowp + vb * 16), static_cast<uint32_t>(vb * VE), bk, bi);
        for (int64_t v = max(vec_end * VE, v0) + tid; v < v1; v += kVerifyThreads) {
            const uint32_t kk = L::key_at(rowp, v);
            if (kk > bk || (kk == bk && static_cast<uint32_t>(v) < bi)) { bk = kk; bi = static_cast<uint32_t>(v); }
        }
        cta_merge(p, row, bk ? pack_key(bk, bi) : 0ull, s_red);
    }
    arrive_and_maybe_finish(p, &s_last);
}

// 16-bit logits (fp16 / bf16): two passes over registers.
//  pass 1: packed max with NaN propagation (HMNMX2, one instruction per 2 logits), reduced
//          over the CTA -> M;
//  pass 2: only threads whose own max equals M look for their first element whose key
//          equals key(M) (keys make +0 == -0 and NaN == NaN); CTA min-index -> winner.
// The CTA's (key(M), ~first index) joins the grid-wide atomicMax like every other path.
template <bool BF16>
struct H16 {
    __device__ static uint32_t max2(uint32_t a, uint32_t b) {
        if constexpr (BF16) {
            __nv_bfloat162 r = __hmax2_nan(*reinterpret_cast<__nv_bfloat162 *>(&a), *reinterpret_cast<__nv_bfloat162 *>(&b));
            return *reinterpret_cast<uint32_t *>(&r);
        } else {
            __half2 r = __hmax2_nan(*reinterpret_cast<__half2 *>(&a), *reinterpret_cast<__half2 *>(&b));
            return *reinterpret_cast<uint32_t *>(&r);
        }
    }
    static constexpr uint32_t kExp = BF16 ? 0x7F80u : 0x7C00u;
    static constexpr uint32_t kNegInf2 = BF16 ? 0xFF80FF80u : 0xFC00FC00u;
};

constexpr int kMaxVPT = 8;  // 16-byte vectors per thread

template <bool BF16>
__global__ void __launch_bounds__(kVerifyThreads) verify_kernel16(VerifyParams p) {
    using T = H16<BF16>;
    __shared__ unsigned long long s_red[kVerifyThreads / kWarp];
    __shared__ uint32_t s_m[kVerifyThreads / kWarp];
    __shared__ int s_last;
    const int tid = threadIdx.x;
    const int64_t row = blockIdx.y;
    const int64_t i = row / (p.k + 1);
    if (p.active[i]) {
        const char *rowp = static_cast<const char *>(p.logits) + row * p.row_stride * 2;
        const int64_t v0 = static_cast<int64_t>(blockIdx.x) * p.chunk;
        const int64_t v1 = min(p.V, v0 + p.chunk);
        const int64_t vec0 = v0 / 8, vec_end = v1 / 8;
        uint4 w[kMaxVPT];
#pragma unroll
        for (int u = 0; u < kMaxVPT; ++u) {
            const int64_t vv = vec0 + u * kVerifyThreads + tid;
            w[u] = vv < vec_end ? ld_stream_v4(rowp + vv * 16)
                                : make_uint4(T::kNegInf2, T::kNegInf2, T::kNegInf2, T::kNegInf2);
        }
        uint32_t m2 = T::kNegInf2;
#pragma unroll
        for (int u = 0; u < kMaxVPT; ++u)
            m2 = T::max2(T::max2(m2, T::max2(w[u].x, w[u].y)), T::max2(w[u].z, w[u].w));
        // ragged tail (V % 8): scalar elements folded into the pair max
        const int64_t tail0 = max(vec_end * 8, v0);
        for (int64_t v = tail0 + tid; v < v1; v += kVerifyThreads) {
            const uint32_t x = reinterpret_cast<const uint16_t *>(rowp)[v];
            m2 = T::max2(m2, x | (x << 16));
        }
        uint32_t m = T::max2(m2, (m2 >> 16) | (m2 << 16)) & 0xFFFFu;
        const uint32_t my_m = m;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, m, o);
            m = T::max2(m | (m << 16), y | (y << 16)) & 0xFFFFu;
        }
        if ((tid & 31) == 0) s_m[tid >> 5] = m;
        __syncthreads();
        m = s_m[0];
#pragma unroll
        for (int q = 1; q < kVerifyThreads / kWarp; ++q) m = T::max2(m | (m << 16), s_m[q] | (s_m[q] << 16)) & 0xFFFFu;
        const uint32_t kM = key16(m, T::kExp);
        uint32_t first = 0xFFFFFFFFu;
        if (key16(my_m, T::kExp) == kM) {
#pragma unroll
            for (int u = 0; u < kMaxVPT; ++u) {
                const int64_t vv = vec0 + u * kVerifyThreads + tid;
                if (vv >= vec_end || first != 0xFFFFFFFFu) break;
                const uint32_t e[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (first == 0xFFFFFFFFu && key16(e[q] & 0xFFFFu, T::kExp) == kM) first = static_cast<uint32_t>(vv * 8 + 2 * q);
                    if (first == 0xFFFFFFFFu && key16(e[q] >> 16, T::kExp) == kM) first = static_cast<uint32_t>(vv * 8 + 2 * q + 1);
                }
            }
            if (first == 0xFFFFFFFFu) {
                for (int64_t v = tail0 + tid; v < v1; v += kVerifyThreads)
                    if (key16(reinterpret_cast<const uint16_t *>(rowp)[v], T::kExp) == kM) { first = static_cast<uint32_t>(v); break; }
            }
        }
        // every thread holding M contributes (key(M), ~first); max -> lowest index
        cta_merge(p, row, first != 0xFFFFFFFFu ? pack_key(kM, first) : 0ull, s_red);
    }
    arrive_and_maybe_finish(p, &s_last);
}

}  // namespace specdec

using namespace specdec;

extern "C" size_t specdec_verify_workspace_size(int64_t B, int64_t k) {
    if (B < 1 || k < 1) return 0;
    return static_cast<size_t>(B * (k + 1)) * sizeof(unsigned long long) + 16;
}

extern "C" int specdec_verify(const void *d_logits, int dtype, int64_t B, int64_t k, int64_t V,
                              int64_t row_stride, const int64_t *d_draft, const int32_t *d_n,
                              uint8_t *d_active, int64_t eos_id, int64_t pad_id,
                              int32_t *d_budget, int32_t *d_accept, int64_t *d_bonus,
                              int32_t *d_emit, uint8_t *d_finished, int64_t *d_pred,
                              int32_t *d_plan_L, int32_t *d_n_new, int32_t *d_pad_new,
                              int32_t *d_kept, uint32_t *d_status, void *d_ws, size_t ws_bytes,
                              specdec_stream_t stream) {
    const int es = dtype_size(dtype);
    if (es == 0) return SPECDEC_ERR_DTYPE;
    if (B < 1 || k < 1 || V < 1 || row_stride < V || V > 0x7FFFFFFFll) return k < 1 ? SPECDEC_ERR_ARG : SPECDEC_ERR_SHAPE;
    if (B > 65535 / (k + 1) + 0) return SPECDEC_ERR_SHAPE;  // gridDim.y limit
    if (!d_logits || !d_draft || !d_n || !d_active || !d_accept || !d_bonus || !d_emit ||
        !d_finished || !d_plan_L || !d_n_new || !d_pad_new || !d_kept || !d_ws)
        return SPECDEC_ERR_ARG;
    if (!aligned16(d_logits) || (row_stride * es) % 16 != 0 || (reinterpret_cast<uintptr_t>(d_ws) & 7u))
        return SPECDEC_ERR_ARG;
    if (ws_bytes < specdec_verify_workspace_size(B, k)) return SPECDEC_ERR_ARG;

    VerifyParams p;
    p.logits = d_logits;
    p.B = B; p.k = k; p.V = V; p.row_stride = row_stride;
    p.draft = d_draft; p.n = d_n; p.active = d_active;
    p.eos_id = eos_id; p.pad_id = pad_id; p.budget = d_budget;
    p.accept = d_accept; p.bonus = d_bonus; p.emit = d_emit; p.finished = d_finished;
    p.pred = d_pred; p.plan_L = d_plan_L; p.n_new = d_n_new; p.pad_new = d_pad_new; p.kept = d_kept;
    p.status = d_status;
    p.ws_keys = static_cast<unsigned long long *>(d_ws);
    p.ws_counter = reinterpret_cast<unsigned int *>(static_cast<char *>(d_ws) + B * (k + 1) * 8);

    // chunk: 16-bit paths hold up to kMaxVPT vectors per thread in registers; aim for
    // >= 4 CTAs per SM over the whole tail.  fp32 (toy) uses one vector per step.
    const int VE = 16 / es;
    const int64_t rows = B * (k + 1);
    const int64_t quantum = static_cast<int64_t>(kVerifyThreads) * VE;
    const int64_t target_ctas = 4ll * device_sm_count();
    int64_t chunk = (V * rows + target_ctas - 1) / target_ctas;
    chunk = (chunk + quantum - 1) / quantum * quantum;
    chunk = std::max<int64_t>(quantum, std::min<int64_t>(chunk, quantum * (es == 2 ? kMaxVPT : 8)));
    p.chunk = chunk;
    const int64_t n_chunks = (V + chunk - 1) / chunk;
    dim3 grid(static_cast<unsigned>(n_chunks), static_cast<unsigned>(rows));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    switch (dtype) {
        case SPECDEC_F32: verify_kernel_f32<<<grid, kVerifyThreads, 0, s>>>(p); break;
        case SPECDEC_F16: verify_kernel16<false><<<grid, kVerifyThreads, 0, s>>>(p); break;
        default: verify_kernel16<true><<<grid, kVerifyThreads, 0, s>>>(p); break;
    }
    return check_launch();
}
