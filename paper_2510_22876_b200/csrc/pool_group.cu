// pool_group.cu -- K4: EXSpec GetBatch over a sliding window (Alg. 3, PAPER.md:488-494,
// 508; §3.2; readings R11-R14).
//
// One CTA of 1024 threads plans the whole window on device:
//   1. RefillWindow: stable compaction of d_order by d_active (block scan), first W ids;
//   2. per member: group count and rank among equal lengths (the length histogram,
//      computed by all-pairs comparison of the <= 2048 window lengths held in smem);
//   3. groups ordered by (-count, length); each group yields same-length batches of
//      min(B, remaining) while remaining >= min_group; group offsets by an ordered sum;
//   4. leftovers keep window order (block scan) and fill fallback batches of B.
// Every step is a deterministic function of the inputs, so the plan is bit-identical to
// the oracle's (tests/test_gpu_pool.py).
#include <cuda_runtime.h>

#include "common.cuh"
#include "host_util.h"

namespace specdec {

constexpr int kPoolThreads = 1024;
constexpr int kPoolMaxW = 2048;

__device__ int block_exclusive_scan(int v, int *s_warp, int &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int w = lane < (blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, w, o);
            if (lane >= o) w += y;
        }
        s_warp[lane] = w;  // inclusive warp prefix
    }
    __syncthreads();
    const int before = (wid > 0 ? s_warp[wid - 1] : 0) + x - v;
    total = s_warp[(blockDim.x >> 5) - 1];
    __syncthreads();
    return before;
}

struct PoolSmem {
    int wid[kPoolMaxW];     // window member ids
    int wlen[kPoolMaxW];    // their lengths
    int cnt[kPoolMaxW];     // group size of the member's length
    int rank[kPoolMaxW];    // rank within its group (window order)
    int lead[kPoolMaxW];    // window index of the group's first member
    int gbase[kPoolMaxW];   // (leaders) first batch index of the group
    int nsb[kPoolMaxW];     // (leaders) number of same-length batches
    int matched[kPoolMaxW]; // (leaders) members placed in same-length batches
    int bmax[kPoolMaxW];    // per batch: max length
    int bmin[kPoolMaxW];    // per batch: min length
    int bcnt[kPoolMaxW];    // per batch: member count
    int warp[32];
    int scalars[8];
};

__global__ void __launch_bounds__(kPoolThreads) pool_group_kernel(
    const int32_t *len, const uint8_t *active, const int32_t *order, int32_t N, int32_t W,
    int32_t B, int32_t min_group, int32_t *window, int32_t *window_size, int32_t *batch_of,
    int32_t *slot_of, int32_t *members, int32_t *mlen, int32_t *mpad, uint8_t *mactive,
    int32_t *bsize, uint8_t *bkind, int32_t *blen, int32_t *n_batches, int64_t *counters) {
    pdl_wait();
    pdl_launch_dependents();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PoolSmem &sm = *reinterpret_cast<PoolSmem *>(smem_raw);
    const int tid = threadIdx.x;
    const int T = blockDim.x;

    for (int s = tid; s < N; s += T) {
        batch_of[s] = -1;
        slot_of[s] = -1;
    }
    // ---- 1. RefillWindow: first W active ids in admission order
    int filled = 0;
    for (int base = 0; base < N && filled < W; base += T) {
        const int t = base + tid;
        int s = -1, f = 0;
        if (t < N) {
            s = order[t];
            f = active[s] ? 1 : 0;
        }
        int tot;
        const int pos = filled + block_exclusive_scan(f, sm.warp, tot);
        if (f && pos < W) {
            sm.wid[pos] = s;
            sm.wlen[pos] = len[s];
        }
        filled += tot;
    }
    const int Wn = min(filled, W);
    __syncthreads();
    // ---- 2. group counts / ranks / leaders (length histogram over the window)
    for (int w = tid; w < Wn; w += T) {
        const int l = sm.wlen[w];
        int c = 0, r = 0, first = w;
        for (int u = 0; u < Wn; ++u) {
            if (sm.wlen[u] == l) {
                ++c;
                if (u < w) ++r;
                first = min(first, u);
            }
        }
        sm.cnt[w] = c;
        sm.rank[w] = r;
        sm.lead[w] = first;
    }
    __syncthreads();
    // ---- 3. same-length batches per group (leaders), groups ordered by (-count, length)
    const int mg = B == 1 ? 1 : min_group;
    for (int w = tid; w < Wn; w += T) {
        if (sm.rank[w] != 0) continue;
        const int c = sm.cnt[w];
        int nb = 0, m = 0;
        if (c >= mg) {
            const int full = c / B, rem = c % B;
            nb = full + (rem >= mg ? 1 : 0);
            m = full * B + (rem >= mg ? rem : 0);
        }
        sm.nsb[w] = nb;
        sm.matched[w] = m;
    }
    __syncthreads();
    int local_same = 0, local_groups = 0;
    for (int w = tid; w < Wn; w += T) {
        if (sm.rank[w] != 0) continue;
        ++local_groups;
        local_same += sm.nsb[w];
        const int c = sm.cnt[w], l = sm.wlen[w];
        int base = 0;
        for (int u = 0; u < Wn; ++u) {
            if (sm.rank[u] != 0) continue;
            const int cu = sm.cnt[u], lu = sm.wlen[u];
            if (cu > c || (cu == c && lu < l)) base += sm.nsb[u];
        }
        sm.gbase[w] = base;
    }
    int tot_same, n_groups;
    block_exclusive_scan(local_same, sm.warp, tot_same);
    block_exclusive_scan(local_groups, sm.warp, n_groups);
    // ---- 4. place members: same-length slots, then leftovers in window order
    int n_left = 0;
    for (int base = 0; base < Wn; base += T) {
        const int w = base + tid;
        int unmatched = 0, bi = -1, sl = -1;
        if (w < Wn) {
            const int ld = sm.lead[w], r = sm.rank[w];
            if (r < sm.matched[ld]) {
                bi = sm.gbase[ld] + r / B;
                sl = r % B;
            } else {
                unmatched = 1;
            }
        }
        int tot;
        const int ui = n_left + block_exclusive_scan(unmatched, sm.warp, tot);
        if (unmatched) {
            bi = tot_same + ui / B;
            sl = ui % B;
        }
        if (w < Wn) sm.rank[w] = bi * B + sl;  // reuse: flat slot index
        n_left += tot;
    }
    const int nb_total = tot_same + (n_left + B - 1) / B;
    for (int b = tid; b < nb_total; b += T) {
        sm.bmax[b] = 0;
        sm.bmin[b] = 0x7FFFFFFF;
        sm.bcnt[b] = 0;
    }
    for (int x = tid; x < nb_total * B; x += T) {
        members[x] = -1;
        mlen[x] = 0;
        mpad[x] = 0;
        mactive[x] = 0;
    }
    __syncthreads();
    for (int w = tid; w < Wn; w += T) {
        const int flat = sm.rank[w], b = flat / B, l = sm.wlen[w], s = sm.wid[w];
        atomicMax(&sm.bmax[b], l);
        atomicMin(&sm.bmin[b], l);
        atomicAdd(&sm.bcnt[b], 1);
        members[flat] = s;
        mlen[flat] = l;
        mactive[flat] = 1;
        batch_of[s] = b;
        slot_of[s] = flat % B;
        window[w] = s;
    }
    __syncthreads();
    long long lsame = 0, lsame_m = 0, lfb_m = 0, lfb_tok = 0;
    for (int w = tid; w < Wn; w += T) {
        const int flat = sm.rank[w], b = flat / B;
        mpad[flat] = sm.bmax[b] - sm.wlen[w];
        if (sm.bmax[b] == sm.bmin[b]) {
            ++lsame_m;
        } else {
            ++lfb_m;
            lfb_tok += sm.wlen[w];
        }
    }
    for (int b = tid; b < nb_total; b += T) {
        const int same = sm.bmax[b] == sm.bmin[b];
        bsize[b] = sm.bcnt[b];
        bkind[b] = static_cast<uint8_t>(same);
        blen[b] = sm.bmax[b];
        lsame += same;
    }
    // counters (accumulated): batches, same-length batches, members in same-length
    // batches, members in fallback batches, fallback member tokens, window size, groups
    if (lsame) atomicAdd(reinterpret_cast<unsigned long long *>(counters + 1), static_cast<unsigned long long>(lsame));
    if (lsame_m) atomicAdd(reinterpret_cast<unsigned long long *>(counters + 2), static_cast<unsigned long long>(lsame_m));
    if (lfb_m) atomicAdd(reinterpret_cast<unsigned long long *>(counters + 3), static_cast<unsigned long long>(lfb_m));
    if (lfb_tok) atomicAdd(reinterpret_cast<unsigned long long *>(counters + 4), static_cast<unsigned long long>(lfb_tok));
    if (tid == 0) {
        *window_size = Wn;
        *n_batches = nb_total;
        atomicAdd(reinterpret_cast<unsigned long long *>(counters + 0), static_cast<unsigned long long>(nb_total));
        atomicAdd(reinterpret_cast<unsigned long long *>(counters + 5), static_cast<unsigned long long>(Wn));
        atomicAdd(reinterpret_cast<unsigned long long *>(counters + 6), static_cast<unsigned long long>(n_groups));
    }
}

}  // namespace specdec

using namespace specdec;

extern "C" int specdec_pool_group(const int32_t *d_len, const uint8_t *d_active,
                                  const int32_t *d_order, int32_t N, int32_t W, int32_t B,
                                  int32_t min_group, int32_t *d_window, int32_t *d_window_size,
                                  int32_t *d_batch_of, int32_t *d_slot_of, int32_t *d_members,
                                  int32_t *d_mlen, int32_t *d_mpad, uint8_t *d_mactive,
                                  int32_t *d_bsize, uint8_t *d_bkind, int32_t *d_blen,
                                  int32_t *d_n_batches, int64_t *d_counters,
                                  specdec_stream_t stream) {
    if (N < 1 || W < 1 || W > kPoolMaxW || B < 1 || B > W) return SPECDEC_ERR_SHAPE;
    if (min_group < 1) return SPECDEC_ERR_ARG;
    if (!d_len || !d_active || !d_order || !d_window || !d_window_size || !d_batch_of ||
        !d_slot_of || !d_members || !d_mlen || !d_mpad || !d_mactive || !d_bsize || !d_bkind ||
        !d_blen || !d_n_batches || !d_counters)
        return SPECDEC_ERR_ARG;
    if (reinterpret_cast<uintptr_t>(d_counters) & 7u) return SPECDEC_ERR_ARG;
    static bool attr_done = false;
    const int smem = static_cast<int>(sizeof(PoolSmem));
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(pool_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return record_cuda_error(e);
        attr_done = true;
    }
    return launch_k(pool_group_kernel, dim3(1), dim3(kPoolThreads), smem,
                    reinterpret_cast<cudaStream_t>(stream), d_len, d_active, d_order, N, W, B,
                    min_group, d_window, d_window_size, d_batch_of, d_slot_of, d_members, d_mlen,
                    d_mpad, d_mactive, d_bsize, d_bkind, d_blen, d_n_batches, d_counters);
}
