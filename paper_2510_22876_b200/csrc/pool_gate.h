// pool_gate.h -- internal (not part of the C ABI): K4 with the Alg. 3 device loop's gate
// fused into its tail (pool_group.cu, used by specdec_pool_alg3 in pool_exec.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "specdec.h"

namespace specdec {

// Batch 0 of the plan as the row maps of the iteration's gather / verify / scatter:
// members (or -1), active flags, the KV rows to move (-1 unless batch 0 goes through the
// staging) and the scatter column (width - 1); exec counts executed batches, same-length
// ones, their members and fallback members.  members == nullptr: no gate.
struct Alg3Gate {
    int32_t *members = nullptr, *kv = nullptr, *scol = nullptr;
    uint8_t *active = nullptr;
    unsigned long long *exec = nullptr;
    int dense = 0;  // specdec_pool_desc::dense_consumer
    // CUDA-graph conditional handles (cudaGraphConditionalHandle; one per conditional node)
    // set to "batch 0 moves KV" for the gather / scatter IF nodes of specdec_pool_alg3_graph;
    // 0 = none
    unsigned long long cond = 0, cond2 = 0;
};

// Deferred fallback (reading R27, specdec_pool_group_deferred): wait[N] epochs each sequence
// has sat out; patience <= 0 or wait == nullptr: the R11 plan.
struct PoolDefer {
    int32_t *wait = nullptr;
    int32_t patience = 0;
    // Pipelined fallback (reading R28): epoch[0] counts the plans; fb_epoch[s] is the plan
    // that last put s in a mixed-length batch.  A sequence with fb_epoch[s] == epoch - 1
    // is left out of the window (its batch runs beside this plan); members of this plan's
    // mixed batches get fb_epoch = epoch.  fb_epoch == nullptr: off.
    int32_t *fb_epoch = nullptr;
    int32_t *epoch = nullptr;
};

int pool_group_launch(const int32_t *d_len, const uint8_t *d_active, const int32_t *d_order, int32_t N,
                      int32_t W, int32_t B, int32_t min_group, int32_t *d_window, int32_t *d_window_size,
                      int32_t *d_batch_of, int32_t *d_slot_of, int32_t *d_members, int32_t *d_mlen,
                      int32_t *d_mpad, uint8_t *d_mactive, int32_t *d_bsize, uint8_t *d_bkind,
                      int32_t *d_blen, int32_t *d_n_batches, int64_t *d_counters, const Alg3Gate &gate,
                      specdec_stream_t stream, bool one_batch = false, const PoolDefer &defer = PoolDefer{});

}  // namespace specdec
