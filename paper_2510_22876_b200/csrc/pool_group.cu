// pool_group.cu -- K4: EXSpec GetBatch over a sliding window (Alg. 3, PAPER.md:488-494,
// 508; §3.2; readings R11-R14).
//
// One CTA (up to 1024 threads: half the window rounded up to a power of two, >= 64) plans
// the whole window on device:
//   1. RefillWindow: stable compaction of d_order by d_active (block scan), first W ids;
//   2. the length histogram: a block-wide bitonic sort of the (length, window position)
//      keys puts every group contiguous and in window order, so a member's group is a
//      scan over segment heads and its rank its offset in the segment;
//   3. groups ordered by (-count, length) -- a second bitonic sort over the group keys;
//      each group yields same-length batches of min(B, remaining) while remaining >=
//      min_group; group offsets by an exclusive scan in that order;
//   4. leftovers keep window order (block scan) and fill fallback batches of B -- with
//      deferred fallback (R27, specdec_pool_group_deferred) only those whose wait reached
//      the patience, when step 3 formed any same-length batch; the others sit out.
// Every step is a deterministic function of the inputs, so the plan is bit-identical to
// the oracle's (tests/test_gpu_pool.py).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "host_util.h"
#include "pool_gate.h"

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
    unsigned long long key[kPoolMaxW];  // sort buffer (member keys, then group keys)
    int wid[kPoolMaxW];     // window member ids
    int wlen[kPoolMaxW];    // their lengths
    int grp[kPoolMaxW];     // member -> group (groups numbered by ascending length)
    int rank[kPoolMaxW];    // member -> rank within its group (window order); later: flat slot
    int gstart[kPoolMaxW + 1];  // group -> first position in the sorted member order
    int nsb[kPoolMaxW];     // group -> number of same-length batches
    int matched[kPoolMaxW]; // group -> members placed in same-length batches
    union {
        struct {
            int gbase[kPoolMaxW];   // group -> first batch index
            int bmax[kPoolMaxW];    // per batch: max length
            int bmin[kPoolMaxW];    // per batch: min length
            int bcnt[kPoolMaxW];    // per batch: member count
        };
        int hist[4 * kPoolMaxW];    // GetBatch (batch 0 only): window length histogram
    };
    int warp[32];
    int red[4];
};
constexpr int kHistBins = 4 * kPoolMaxW;  // length range the one-batch GetBatch histograms directly

// Ascending bitonic sort of key[0, n) (n a power of two <= 2 * blockDim.x, padded with ~0).
// Keys are unique (or equal padding), so the result is unique whatever the thread
// schedule.  Register resident: thread t < P = n / 2 holds elements t and t + P.  A substep with j < 32 pairs lanes of one warp (shuffle), j == P pairs the
// thread's own two elements, and only 32 <= j < P goes through shared memory (two block
// barriers) -- 14 of the 55 substeps at n = 1024.  (The former all-shared-memory version,
// with an integer division per pair, took 11.5 us at n = 1024; profiles/r01/k4bench.txt.)
// Generic (64-bit keys: window lengths >= 2^20 only).
template <typename K>
__device__ __forceinline__ K keep(K x, K y, bool lo) {
    return lo ? (x < y ? x : y) : (x > y ? x : y);
}

template <typename K>
__device__ void block_bitonic_sort_generic(K *key, int n) {
    const int tid = threadIdx.x;
    const int P = n >> 1;
    const bool on = tid < P;
    const bool wact = tid < ((P + 31) & ~31);  // whole warps for the shuffles (P < 32: warp 0)
    K x0 = on ? key[tid] : K(0), x1 = on ? key[tid + P] : K(0);
    const int i0 = tid, i1 = tid + P;
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == P) {  // only at k == n: every pair ascending, i0 the lower
                if (on) {
                    const K lo = x0 < x1 ? x0 : x1, hi = x0 < x1 ? x1 : x0;
                    x0 = lo;
                    x1 = hi;
                }
            } else if (j >= 32) {
                __syncthreads();  // the previous exchange's reads are done
                if (on) {
                    key[i0] = x0;
                    key[i1] = x1;
                }
                __syncthreads();
                if (on) {
                    const K y0 = key[i0 ^ j], y1 = key[i1 ^ j];
                    x0 = keep(x0, y0, ((i0 & j) == 0) == ((i0 & k) == 0));
                    x1 = keep(x1, y1, ((i1 & j) == 0) == ((i1 & k) == 0));
                }
            } else if (wact) {  // j < min(P, 32): lane ^ j < P for every lane < P
                const K y0 = __shfl_xor_sync(0xFFFFFFFFu, x0, j);
                const K y1 = __shfl_xor_sync(0xFFFFFFFFu, x1, j);
                if (on) {
                    x0 = keep(x0, y0, ((i0 & j) == 0) == ((i0 & k) == 0));
                    x1 = keep(x1, y1, ((i1 & j) == 0) == ((i1 & k) == 0));
                }
            }
        }
    }
    __syncthreads();
    if (on) {
        key[i0] = x0;
        key[i1] = x1;
    }
    __syncthreads();
}

// The 32-bit keys' sort, unrolled for a fixed n = 2^LOGN: thread t < n / E holds the E
// consecutive elements t*E .. t*E + E - 1, so substeps with j < E are register
// compare-exchanges, E <= j < 32 E warp shuffles (lane ^ j / E) and only larger j go
// through shared memory; every direction and partner is a compile-time constant or a
// bit test on t.
template <int LOGN>
__device__ void block_bitonic_sort_fixed(uint32_t *key) {
    constexpr int n = 1 << LOGN;
    constexpr int E = n >= 128 ? 4 : 2;
    constexpr int NT = n / E > 0 ? n / E : 1;
    const int t = threadIdx.x;
    const bool on = t < NT;
    const bool wact = t < ((NT + 31) & ~31);
    uint32_t x[E];
#pragma unroll
    for (int r = 0; r < E; ++r) x[r] = (on && t * E + r < n) ? key[t * E + r] : 0xFFFFFFFFu;
#pragma unroll
    for (int k = 2; k <= n; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < E) {
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    if ((r & j) == 0) {
                        const bool up = ((t * E + r) & k) == 0;
                        const uint32_t a = x[r], b = x[r | j];
                        const uint32_t lo = min(a, b), hi = max(a, b);
                        x[r] = up ? lo : hi;
                        x[r | j] = up ? hi : lo;
                    }
                }
            } else if (j < 32 * E) {
                if (wact) {
#pragma unroll
                    for (int r = 0; r < E; ++r) {
                        const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x[r], j / E);
                        const int i = t * E + r;
                        x[r] = (((i & j) == 0) == ((i & k) == 0)) ? min(x[r], y) : max(x[r], y);
                    }
                }
            } else {
                __syncthreads();  // the previous exchange's reads are done
                if (on) {
#pragma unroll
                    for (int r = 0; r < E; ++r) key[t * E + r] = x[r];
                }
                __syncthreads();
                if (on) {
#pragma unroll
                    for (int r = 0; r < E; ++r) {
                        const int i = t * E + r;
                        const uint32_t y = key[i ^ j];
                        x[r] = (((i & j) == 0) == ((i & k) == 0)) ? min(x[r], y) : max(x[r], y);
                    }
                }
            }
        }
    }
    __syncthreads();
    if (on) {
#pragma unroll
        for (int r = 0; r < E; ++r)
            if (t * E + r < n) key[t * E + r] = x[r];
    }
    __syncthreads();
}

__device__ void block_bitonic_sort(uint32_t *key, int n) {
    switch (n) {
        case 1: break;
        case 2: block_bitonic_sort_fixed<1>(key); break;
        case 4: block_bitonic_sort_fixed<2>(key); break;
        case 8: block_bitonic_sort_fixed<3>(key); break;
        case 16: block_bitonic_sort_fixed<4>(key); break;
        case 32: block_bitonic_sort_fixed<5>(key); break;
        case 64: block_bitonic_sort_fixed<6>(key); break;
        case 128: block_bitonic_sort_fixed<7>(key); break;
        case 256: block_bitonic_sort_fixed<8>(key); break;
        case 512: block_bitonic_sort_fixed<9>(key); break;
        case 1024: block_bitonic_sort_fixed<10>(key); break;
        default: block_bitonic_sort_fixed<11>(key); break;
    }
}

// ---- RefillWindow: the first W active ids in admission order, into
// sm.wid / sm.wlen; returns the window size.
__device__ int refill_window(PoolSmem &sm, const int32_t *len, const uint8_t *active, const int32_t *order,
                             int32_t N, int32_t W, const int32_t *fb_epoch = nullptr, int32_t prev_epoch = 0) {
    const int tid = threadIdx.x, T = blockDim.x;
    int filled = 0;
    for (int base = 0; base < N && filled < W; base += T) {
        const int t = base + tid;
        int s = -1, f = 0;
        if (t < N) {
            s = order[t];
            // R28: a member of the previous plan's mixed batches is still in flight
            f = active[s] && !(fb_epoch && fb_epoch[s] == prev_epoch) ? 1 : 0;
        }
        int tot;
        const int pos = filled + block_exclusive_scan(f, sm.warp, tot);
        if (f && pos < W) {
            sm.wid[pos] = s;
            sm.wlen[pos] = len[s];
        }
        filled += tot;
    }
    __syncthreads();
    return min(filled, W);
}

// The whole-window plan (steps 2-4 above) after RefillWindow, plus the Alg. 3 gate.
__device__ void plan_full(PoolSmem &sm, int Wn, int32_t B, int32_t min_group, int32_t *window,
                          int32_t *window_size, int32_t *batch_of, int32_t *slot_of, int32_t *members,
                          int32_t *mlen, int32_t *mpad, uint8_t *mactive, int32_t *bsize, uint8_t *bkind,
                          int32_t *blen, int32_t *n_batches, int64_t *counters, const Alg3Gate &gate, int exp,
                          const PoolDefer &defer) {
    const int tid = threadIdx.x;
    const int T = blockDim.x;
    if (exp == 1) return;  // timing probe only (SPECDEC_K4_EXP): up to RefillWindow
    // ---- 2. length histogram: sort (length, window position), groups = equal-length runs.
    // Keys are 32-bit, (length << 11) | position, when every window length is in [0, 2^20)
    // (position < W <= 2048), else 64-bit (length << 32) | position.
    int n2 = 1;
    while (n2 < Wn) n2 <<= 1;
    int big = 0;
    for (int i = tid; i < Wn; i += T) big |= (sm.wlen[i] < 0 || sm.wlen[i] >= (1 << 20)) ? 1 : 0;
    const bool wide = __syncthreads_or(big) != 0;
    uint32_t *key32 = reinterpret_cast<uint32_t *>(sm.key);
    if (wide) {
        for (int i = tid; i < n2; i += T)
            sm.key[i] = i < Wn ? (static_cast<unsigned long long>(static_cast<uint32_t>(sm.wlen[i])) << 32) |
                                     static_cast<uint32_t>(i)
                               : ~0ull;
        __syncthreads();
        block_bitonic_sort_generic(sm.key, n2);
    } else {
        for (int i = tid; i < n2; i += T)
            key32[i] = i < Wn ? (static_cast<uint32_t>(sm.wlen[i]) << 11) | static_cast<uint32_t>(i) : ~0u;
        __syncthreads();
        block_bitonic_sort(key32, n2);
    }
    // the i-th sorted member's length class and window position
    auto klen = [&](int i) -> uint32_t { return wide ? static_cast<uint32_t>(sm.key[i] >> 32) : key32[i] >> 11; };
    auto kpos = [&](int i) -> int {
        return wide ? static_cast<int>(sm.key[i] & 0xFFFFFFFFull) : static_cast<int>(key32[i] & 0x7FFu);
    };
    if (exp == 2) return;  // probe: + the member sort
    int n_groups = 0;
    for (int base = 0; base < Wn; base += T) {  // group id = number of run heads before
        const int i = base + tid;
        int head = 0;
        if (i < Wn) head = (i == 0 || klen(i) != klen(i - 1)) ? 1 : 0;
        int tot;
        const int g = n_groups + block_exclusive_scan(head, sm.warp, tot);
        if (head) sm.gstart[g] = i;
        n_groups += tot;
    }
    if (tid == 0) sm.gstart[n_groups] = Wn;
    __syncthreads();
    // member -> (group, rank): binary search of its sorted position among the group starts
    for (int i = tid; i < Wn; i += T) {
        int lo = 0, hi = n_groups - 1;  // last g with gstart[g] <= i
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (sm.gstart[mid] <= i) lo = mid; else hi = mid - 1;
        }
        const int w = kpos(i);
        sm.grp[w] = lo;
        sm.rank[w] = i - sm.gstart[lo];
    }
    // ---- 3. same-length batches per group; groups ordered by (-count, length)
    const int mg = B == 1 ? 1 : min_group;
    for (int g = tid; g < n_groups; g += T) {
        const int c = sm.gstart[g + 1] - sm.gstart[g];
        int nb = 0, m = 0;
        // batches of min(B, remaining) while remaining >= mg (R11), in closed form
        if (c >= mg && mg <= B) {
            const int full = c / B, rem = c % B;  // every full batch starts with >= B >= mg left
            nb = full + (rem >= mg ? 1 : 0);
            m = full * B + (rem >= mg ? rem : 0);
        } else if (c >= mg) {                     // mg > B: only full batches, while >= mg left
            nb = (c - mg) / B + 1;
            m = nb * B;
        }
        sm.nsb[g] = nb;
        sm.matched[g] = m;
    }
    __syncthreads();
    int g2 = 1;
    while (g2 < n_groups) g2 <<= 1;
    // key: (-count, length) ascending, 32-bit: (2048 - count) << 11 | group id (ids ascend
    // with the length; count in [1, 2048], id < 2048)
    for (int g = tid; g < g2; g += T)
        key32[g] = g < n_groups
            ? (static_cast<uint32_t>(kPoolMaxW - (sm.gstart[g + 1] - sm.gstart[g])) << 11) | static_cast<uint32_t>(g)
            : ~0u;
    __syncthreads();
    block_bitonic_sort(key32, g2);
    if (exp == 3) return;  // probe: + groups and the group sort
    int run = 0;
    for (int base = 0; base < n_groups; base += T) {  // gbase: exclusive scan of nsb in that order
        const int q = base + tid;
        const int g = q < n_groups ? static_cast<int>(key32[q] & 0x7FFu) : 0;
        const int v = q < n_groups ? sm.nsb[g] : 0;
        int tot;
        const int before = run + block_exclusive_scan(v, sm.warp, tot);
        if (q < n_groups) sm.gbase[g] = before;
        run += tot;
    }
    const int tot_same = run;
    __syncthreads();
    // ---- 4. place members: same-length slots, then leftovers in window order.  R27: when
    // step 3 formed a same-length batch, a leftover whose wait is below the patience sits
    // this epoch out (flat slot -1); the waits are updated here (one CTA: no race).
    const bool deferring = defer.wait != nullptr && defer.patience > 0 && tot_same > 0;
    int n_left = 0, n_deferred = 0;
    for (int base = 0; base < Wn; base += T) {
        const int w = base + tid;
        int unmatched = 0, bi = -1, sl = -1, deferred = 0;
        if (w < Wn) {
            const int g = sm.grp[w], r = sm.rank[w];
            if (r < sm.matched[g]) {
                bi = sm.gbase[g] + r / B;
                sl = r % B;
            } else if (deferring && defer.wait[sm.wid[w]] < defer.patience) {
                deferred = 1;
            } else {
                unmatched = 1;
            }
            if (defer.wait) defer.wait[sm.wid[w]] = deferred ? defer.wait[sm.wid[w]] + 1 : 0;
        }
        int tot;
        const int ui = n_left + block_exclusive_scan(unmatched, sm.warp, tot);
        if (unmatched) {
            bi = tot_same + ui / B;
            sl = ui % B;
        }
        if (w < Wn) sm.rank[w] = deferred ? -1 : bi * B + sl;  // reuse: flat slot index
        n_left += tot;
        n_deferred += __syncthreads_count(deferred);
    }
    const int nb_total = tot_same + (n_left + B - 1) / B;
    if (exp == 4) return;  // probe: + member placement scans
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
        window[w] = s;
        if (flat < 0) continue;  // deferred (R27): in the window, in no batch
        atomicMax(&sm.bmax[b], l);
        atomicMin(&sm.bmin[b], l);
        atomicAdd(&sm.bcnt[b], 1);
        members[flat] = s;
        mlen[flat] = l;
        mactive[flat] = 1;
        batch_of[s] = b;
        slot_of[s] = flat % B;
    }
    __syncthreads();
    long long lsame = 0, lsame_m = 0, lfb_m = 0, lfb_tok = 0;
    const int32_t ep = defer.fb_epoch ? *defer.epoch : 0;  // read before thread 0 advances it
    for (int w = tid; w < Wn; w += T) {
        const int flat = sm.rank[w], b = flat / B;
        if (flat < 0) continue;
        mpad[flat] = sm.bmax[b] - sm.wlen[w];
        if (sm.bmax[b] == sm.bmin[b]) {
            ++lsame_m;
        } else {
            ++lfb_m;
            lfb_tok += sm.wlen[w];
            if (defer.fb_epoch) defer.fb_epoch[sm.wid[w]] = ep;  // R28: in flight next plan
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
    // batches, members in fallback batches, fallback member tokens, window size, groups,
    // deferred members (R27)
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
        if (n_deferred)
            atomicAdd(reinterpret_cast<unsigned long long *>(counters + 7), static_cast<unsigned long long>(n_deferred));
    }
    if (defer.fb_epoch) {
        __syncthreads();  // every thread has read the epoch
        if (tid == 0) *defer.epoch = ep + 1;
    }
    if (gate.members) {
        // Alg. 3 device loop: batch 0 as the row maps of this iteration's gather / verify /
        // scatter (one launch fewer than a separate gate kernel).  The barrier makes this
        // block's stores of batch 0's members / mactive visible to every thread.
        __syncthreads();
        const bool valid = nb_total > 0;
        const bool same = valid && sm.bmax[0] == sm.bmin[0];
        // batch 0 goes through the staging: a mixed batch (dense rectangle consumer) or every
        // batch (dense = 1); never with the slot-indexed consumer (dense = 2)
        const bool moves = valid && gate.dense != 2 && (!same || gate.dense == 1);
        if (gate.cond && tid == 0) {
            cudaGraphSetConditional(gate.cond, moves ? 1u : 0u);
            if (gate.cond2) cudaGraphSetConditional(gate.cond2, moves ? 1u : 0u);
        }
        for (int j = tid; j < B; j += T) {
            const int32_t m = valid ? members[j] : -1;
            gate.members[j] = m;
            gate.active[j] = valid ? mactive[j] : 0;
            gate.kv[j] = moves ? m : -1;
            gate.scol[j] = (valid ? sm.bmax[0] : 0) - 1;
        }
        if (tid == 0 && gate.exec && valid) {
            atomicAdd(gate.exec, 1ull);
            if (same) {
                atomicAdd(gate.exec + 1, 1ull);
                atomicAdd(gate.exec + 2, static_cast<unsigned long long>(sm.bcnt[0]));
            } else {
                atomicAdd(gate.exec + 3, static_cast<unsigned long long>(sm.bcnt[0]));
            }
        }
    }
}

__global__ void __launch_bounds__(kPoolThreads) pool_group_kernel(
    const int32_t *len, const uint8_t *active, const int32_t *order, int32_t N, int32_t W,
    int32_t B, int32_t min_group, int32_t *window, int32_t *window_size, int32_t *batch_of,
    int32_t *slot_of, int32_t *members, int32_t *mlen, int32_t *mpad, uint8_t *mactive,
    int32_t *bsize, uint8_t *bkind, int32_t *blen, int32_t *n_batches, int64_t *counters, Alg3Gate gate,
    int exp, PoolDefer defer) {
    pdl_wait();
    pdl_launch_dependents();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PoolSmem &sm = *reinterpret_cast<PoolSmem *>(smem_raw);
    for (int s = threadIdx.x; s < N; s += blockDim.x) {
        batch_of[s] = -1;
        slot_of[s] = -1;
    }
    const int Wn = refill_window(sm, len, active, order, N, W, defer.fb_epoch,
                                 defer.fb_epoch ? *defer.epoch - 1 : 0);
    plan_full(sm, Wn, B, min_group, window, window_size, batch_of, slot_of, members, mlen, mpad, mactive, bsize,
              bkind, blen, n_batches, counters, gate, exp, defer);
}

// ---- Alg. 3's GetBatch as printed (one batch per iteration): batch 0 of the
// window plan above, without planning the rest.  Batch 0 is the first batch of the
// heaviest length group -- largest count, ties to the smaller length -- if its count
// reaches min_group (R11), i.e. min(B, count) of its members in window order; else no
// group qualifies and batch 0 is the first min(B, |window|) members of the window.  A
// length histogram (shared-memory atomics; counts are order-independent) and one block
// maximum find the group, one block scan in window order picks its members: no sort.
// Windows whose lengths span more than kHistBins values take the full plan instead.
__device__ __forceinline__ int block_reduce_max(int v, int *s_warp) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = __reduce_max_sync(0xFFFFFFFFu, v);
    __syncthreads();
    if (lane == 0) s_warp[wid] = v;
    __syncthreads();
    int m = s_warp[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = max(m, s_warp[w]);
    return m;
}
__device__ __forceinline__ int block_reduce_sum(int v, int *s_warp) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = __reduce_add_sync(0xFFFFFFFFu, v);
    __syncthreads();
    if (lane == 0) s_warp[wid] = v;
    __syncthreads();
    int m = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) m += s_warp[w];
    return m;
}

__global__ void __launch_bounds__(kPoolThreads) pool_getbatch_kernel(
    const int32_t *len, const uint8_t *active, const int32_t *order, int32_t N, int32_t W,
    int32_t B, int32_t min_group, int32_t *window, int32_t *window_size, int32_t *batch_of,
    int32_t *slot_of, int32_t *members, int32_t *mlen, int32_t *mpad, uint8_t *mactive,
    int32_t *bsize, uint8_t *bkind, int32_t *blen, int32_t *n_batches, int64_t *counters, Alg3Gate gate) {
    pdl_wait();
    pdl_launch_dependents();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PoolSmem &sm = *reinterpret_cast<PoolSmem *>(smem_raw);
    const int tid = threadIdx.x, T = blockDim.x;
    for (int s = tid; s < N; s += T) {
        batch_of[s] = -1;
        slot_of[s] = -1;
    }
    const int Wn = refill_window(sm, len, active, order, N, W);
    // the window's length range (lengths are >= 1)
    int lo = 0x7FFFFFFF, hi = 0;
    for (int w = tid; w < Wn; w += T) {
        lo = min(lo, sm.wlen[w]);
        hi = max(hi, sm.wlen[w]);
    }
    const int Lmax = block_reduce_max(hi, sm.warp);
    const int Lmin = -block_reduce_max(-lo, sm.warp);
    if (Wn > 0 && (Lmin < 0 || static_cast<int64_t>(Lmax) - Lmin >= kHistBins)) {
        plan_full(sm, Wn, B, min_group, window, window_size, batch_of, slot_of, members, mlen, mpad, mactive,
                  bsize, bkind, blen, n_batches, counters, gate, 0, PoolDefer{});
        return;
    }
    const int R = Wn > 0 ? Lmax - Lmin + 1 : 0;
    for (int b = tid; b < R; b += T) sm.hist[b] = 0;
    __syncthreads();
    for (int w = tid; w < Wn; w += T) atomicAdd(&sm.hist[sm.wlen[w] - Lmin], 1);
    __syncthreads();
    // the heaviest group: (count, then the smaller length) as one packed maximum over the
    // groups that reach min_group (>= 1 when B == 1)
    const int mg = B == 1 ? 1 : min_group;
    int best = 0, distinct = 0;
    for (int b = tid; b < R; b += T) {
        const int c = sm.hist[b];
        distinct += c > 0;
        if (c >= mg) best = max(best, (c << 13) | (kHistBins - 1 - b));  // c <= 2048: 25 bits
    }
    best = block_reduce_max(best, sm.warp);
    distinct = block_reduce_sum(distinct, sm.warp);
    const bool grouped = best > 0;
    const int Lsel = grouped ? Lmin + (kHistBins - 1 - (best & (kHistBins - 1))) : 0;
    const int take = grouped ? min(B, best >> 13) : min(B, Wn);
    // batch 0's members in window order: the first `take` of the chosen length (or of the
    // window); the scan stops once they are found
    for (int x = tid; x < B; x += T) {
        members[x] = -1;
        mlen[x] = 0;
        mpad[x] = 0;
        mactive[x] = 0;
    }
    __syncthreads();
    int found = 0;
    for (int base = 0; base < Wn && found < take; base += T) {
        const int w = base + tid;
        const int f = (w < Wn && (!grouped || sm.wlen[w] == Lsel)) ? 1 : 0;
        int tot;
        const int r = found + block_exclusive_scan(f, sm.warp, tot);
        if (f && r < take) {
            sm.rank[r] = w;  // slot r <- window position w
        }
        found += tot;
    }
    __syncthreads();
    // batch 0: width, kind (every member the same length), outputs
    int bmx = 0, bmn = 0x7FFFFFFF;
    for (int r = tid; r < take; r += T) {
        const int l = sm.wlen[sm.rank[r]];
        bmx = max(bmx, l);
        bmn = min(bmn, l);
    }
    bmx = block_reduce_max(bmx, sm.warp);
    bmn = -block_reduce_max(-bmn, sm.warp);
    const bool same = take > 0 && bmx == bmn;
    long long tok = 0;
    for (int r = tid; r < take; r += T) {
        const int w = sm.rank[r], s = sm.wid[w], l = sm.wlen[w];
        members[r] = s;
        mlen[r] = l;
        mpad[r] = bmx - l;
        mactive[r] = 1;
        batch_of[s] = 0;
        slot_of[s] = r;
        tok += l;
    }
    for (int w = tid; w < Wn; w += T) window[w] = sm.wid[w];
    if (tok && !same) atomicAdd(reinterpret_cast<unsigned long long *>(counters + 4), static_cast<unsigned long long>(tok));
    if (tid == 0) {
        *window_size = Wn;
        *n_batches = take > 0 ? 1 : 0;
        bsize[0] = take;
        bkind[0] = static_cast<uint8_t>(same);
        blen[0] = take > 0 ? bmx : 0;
        // counters (accumulated) of the batch planned: batches, same-length batches, their
        // members, fallback members, fallback tokens (above), window size, distinct lengths
        if (take > 0) {
            atomicAdd(reinterpret_cast<unsigned long long *>(counters + 0), 1ull);
            atomicAdd(reinterpret_cast<unsigned long long *>(counters + (same ? 1 : 3)),
                      same ? 1ull : static_cast<unsigned long long>(take));
            if (same) atomicAdd(reinterpret_cast<unsigned long long *>(counters + 2), static_cast<unsigned long long>(take));
        }
        atomicAdd(reinterpret_cast<unsigned long long *>(counters + 5), static_cast<unsigned long long>(Wn));
        atomicAdd(reinterpret_cast<unsigned long long *>(counters + 6), static_cast<unsigned long long>(distinct));
    }
    if (gate.members) {
        __syncthreads();  // batch 0's member / mactive stores visible to every thread
        const bool valid = take > 0;
        const bool moves = valid && gate.dense != 2 && (!same || gate.dense == 1);
        if (gate.cond && tid == 0) {
            cudaGraphSetConditional(gate.cond, moves ? 1u : 0u);
            if (gate.cond2) cudaGraphSetConditional(gate.cond2, moves ? 1u : 0u);
        }
        for (int j = tid; j < B; j += T) {
            const int32_t m = valid ? members[j] : -1;
            gate.members[j] = m;
            gate.active[j] = valid ? mactive[j] : 0;
            gate.kv[j] = moves ? m : -1;
            gate.scol[j] = (valid ? bmx : 0) - 1;
        }
        if (tid == 0 && gate.exec && valid) {
            atomicAdd(gate.exec, 1ull);
            if (same) {
                atomicAdd(gate.exec + 1, 1ull);
                atomicAdd(gate.exec + 2, static_cast<unsigned long long>(take));
            } else {
                atomicAdd(gate.exec + 3, static_cast<unsigned long long>(take));
            }
        }
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
    return pool_group_launch(d_len, d_active, d_order, N, W, B, min_group, d_window, d_window_size, d_batch_of,
                             d_slot_of, d_members, d_mlen, d_mpad, d_mactive, d_bsize, d_bkind, d_blen,
                             d_n_batches, d_counters, Alg3Gate{}, stream);
}

extern "C" int specdec_pool_group_deferred(const int32_t *d_len, const uint8_t *d_active,
                                           const int32_t *d_order, int32_t N, int32_t W, int32_t B,
                                           int32_t min_group, int32_t *d_wait, int32_t patience,
                                           int32_t *d_fb_epoch, int32_t *d_epoch,
                                           int32_t *d_window, int32_t *d_window_size,
                                           int32_t *d_batch_of, int32_t *d_slot_of, int32_t *d_members,
                                           int32_t *d_mlen, int32_t *d_mpad, uint8_t *d_mactive,
                                           int32_t *d_bsize, uint8_t *d_bkind, int32_t *d_blen,
                                           int32_t *d_n_batches, int64_t *d_counters,
                                           specdec_stream_t stream) {
    if (patience < 0 || (patience > 0 && !d_wait) || (!d_fb_epoch != !d_epoch)) return SPECDEC_ERR_ARG;
    PoolDefer defer;
    defer.wait = d_wait;
    defer.patience = patience;
    defer.fb_epoch = d_fb_epoch;
    defer.epoch = d_epoch;
    return pool_group_launch(d_len, d_active, d_order, N, W, B, min_group, d_window, d_window_size, d_batch_of,
                             d_slot_of, d_members, d_mlen, d_mpad, d_mactive, d_bsize, d_bkind, d_blen,
                             d_n_batches, d_counters, Alg3Gate{}, stream, false, defer);
}

extern "C" int specdec_pool_getbatch(const int32_t *d_len, const uint8_t *d_active,
                                     const int32_t *d_order, int32_t N, int32_t W, int32_t B,
                                     int32_t min_group, int32_t *d_window, int32_t *d_window_size,
                                     int32_t *d_batch_of, int32_t *d_slot_of, int32_t *d_members,
                                     int32_t *d_mlen, int32_t *d_mpad, uint8_t *d_mactive,
                                     int32_t *d_bsize, uint8_t *d_bkind, int32_t *d_blen,
                                     int32_t *d_n_batches, int64_t *d_counters,
                                     specdec_stream_t stream) {
    return pool_group_launch(d_len, d_active, d_order, N, W, B, min_group, d_window, d_window_size, d_batch_of,
                             d_slot_of, d_members, d_mlen, d_mpad, d_mactive, d_bsize, d_bkind, d_blen,
                             d_n_batches, d_counters, Alg3Gate{}, stream, true);
}

int specdec::pool_group_launch(const int32_t *d_len, const uint8_t *d_active, const int32_t *d_order, int32_t N,
                               int32_t W, int32_t B, int32_t min_group, int32_t *d_window,
                               int32_t *d_window_size, int32_t *d_batch_of, int32_t *d_slot_of,
                               int32_t *d_members, int32_t *d_mlen, int32_t *d_mpad, uint8_t *d_mactive,
                               int32_t *d_bsize, uint8_t *d_bkind, int32_t *d_blen, int32_t *d_n_batches,
                               int64_t *d_counters, const Alg3Gate &gate, specdec_stream_t stream,
                               bool one_batch, const PoolDefer &defer) {
    if (N < 1 || W < 1 || W > kPoolMaxW || B < 1 || B > W) return SPECDEC_ERR_SHAPE;
    if (min_group < 1) return SPECDEC_ERR_ARG;
    if (!d_len || !d_active || !d_order || !d_window || !d_window_size || !d_batch_of ||
        !d_slot_of || !d_members || !d_mlen || !d_mpad || !d_mactive || !d_bsize || !d_bkind ||
        !d_blen || !d_n_batches || !d_counters)
        return SPECDEC_ERR_ARG;
    if (reinterpret_cast<uintptr_t>(d_counters) & 7u) return SPECDEC_ERR_ARG;
    static bool attr_done = false;
    static const int exp = getenv("SPECDEC_K4_EXP") ? atoi(getenv("SPECDEC_K4_EXP")) : 0;
    const int smem = static_cast<int>(sizeof(PoolSmem));
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(pool_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(pool_getbatch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return record_cuda_error(e);
        attr_done = true;
    }
    // threads: enough for the bitonic sorts (n <= 2 * threads, n = the window rounded up to
    // a power of two) and no more -- a block barrier costs more with more warps
    int w2 = 1;
    while (w2 < W) w2 <<= 1;
    const int threads = std::min(kPoolThreads, std::max(64, w2 / 2));
    if (one_batch)
        return launch_k(pool_getbatch_kernel, dim3(1), dim3(threads), smem, reinterpret_cast<cudaStream_t>(stream),
                        d_len, d_active, d_order, N, W, B, min_group, d_window, d_window_size, d_batch_of,
                        d_slot_of, d_members, d_mlen, d_mpad, d_mactive, d_bsize, d_bkind, d_blen, d_n_batches,
                        d_counters, gate);
    return launch_k(pool_group_kernel, dim3(1), dim3(threads), smem,
                    reinterpret_cast<cudaStream_t>(stream), d_len, d_active, d_order, N, W, B,
                    min_group, d_window, d_window_size, d_batch_of, d_slot_of, d_members, d_mlen,
                    d_mpad, d_mactive, d_bsize, d_bkind, d_blen, d_n_batches, d_counters, gate, exp, defer);
}
