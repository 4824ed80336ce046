// common.cuh -- small sm_100a device helpers shared by the specdec kernels
// (mbarrier + cp.async.bulk PTX wrappers, cache-hinted loads, argmax keys).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "specdec.h"

namespace specdec {

constexpr int kWarp = 32;

// ----------------------------------------------------------------------------- argmax key
// A logit is mapped to an unsigned key whose order equals the argmax order of
// PAPER.md:303 under readings R4/R5: larger value -> larger key; +0 and -0 -> the same
// key; every NaN -> the top key (NaN ranks above +inf, all NaNs tie so the lowest index
// wins).  Packing (key << 32) | ~index into 64 bits turns "max value, then lowest index"
// into a plain unsigned max -- associative and commutative, so any split or atomic
// combine order gives the bit-exact same winner.
__device__ __forceinline__ uint32_t key16(uint32_t bits, uint32_t exp_all_ones) {
    const uint32_t mag = bits & 0x7FFFu;
    const uint32_t k = (bits & 0x8000u) ? (0x8000u - mag) : (0x8000u + mag);
    return mag > exp_all_ones ? 0xFFFFFFFFu : k;
}
// the same order in 16 bits (NaN -> 0xFFFF, above +inf's 0xFF80 / 0xFC00)
__device__ __forceinline__ uint32_t key16s(uint32_t bits, uint32_t exp_all_ones) {
    const uint32_t mag = bits & 0x7FFFu;
    const uint32_t k = (bits & 0x8000u) ? (0x8000u - mag) : (0x8000u + mag);
    return mag > exp_all_ones ? 0xFFFFu : k;
}
__device__ __forceinline__ uint32_t key32(uint32_t bits) {
    const uint32_t mag = bits & 0x7FFFFFFFu;
    const uint32_t k = (bits & 0x80000000u) ? (0x80000000u - mag) : (0x80000000u + mag);
    return mag > 0x7F800000u ? 0xFFFFFFFFu : k;
}
__device__ __forceinline__ unsigned long long pack_key(uint32_t key, uint32_t idx) {
    return (static_cast<unsigned long long>(key) << 32) | static_cast<uint32_t>(~idx);
}
__device__ __forceinline__ uint32_t unpack_idx(unsigned long long p) {
    return ~static_cast<uint32_t>(p & 0xFFFFFFFFull);
}

// ----------------------------------------------------------------------------- PDL
// Programmatic dependent launch: a kernel launched with the programmatic-serialization
// attribute may start while its predecessor drains; griddepcontrol.wait blocks until the
// predecessor has completed and its writes are visible (a no-op without the attribute).
// Every specdec kernel waits before touching any input, so ordering is unchanged; only the
// launch latency between consecutive kernels overlaps.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ----------------------------------------------------------------------------- loads
__device__ __forceinline__ uint4 ld_stream_v4(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ----------------------------------------------------------------------------- mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Bounded wait: a pipeline bug must surface as a trapped kernel (launch error), never
// as a hung GPU.  ~2^26 try_wait rounds is seconds, far above any legitimate wait.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++spins > (1u << 26)) __trap();
    }
}

// ----------------------------------------------------------------------------- bulk copies
// global -> shared, completion via the mbarrier's transaction count (TMA 1-D bulk copy).
__device__ __forceinline__ void bulk_load(void *smem_dst, const void *gmem_src, uint32_t bytes,
                                          uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// shared -> global, tracked by bulk async-groups.
__device__ __forceinline__ void bulk_store(void *gmem_dst, const void *smem_src, uint32_t bytes,
                                           uint64_t policy) {
    asm volatile(
        "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
            gmem_dst),
        "r"(smem_u32(smem_src)), "r"(bytes), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

}  // namespace specdec
