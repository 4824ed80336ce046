// k1_stream.cu -- design experiment for K1 (not part of libspecdec): how fast can a
// latency-bound reduction over the verify logits (Qwen3 B=8: 48 rows x 151936 bf16 =
// 14.6 MB, cold in HBM) run back to back inside a CUDA graph, for several grid shapes?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/exp/k1_stream.cu -o k1_stream
//   ./k1_stream [rows] [V]
// Every kernel reduces its share to a packed bf16 max and writes one word per CTA.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_go() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ uint4 ldnc(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t mx2(uint32_t a, uint32_t b) {
    __nv_bfloat162 r = __hmax2_nan(*reinterpret_cast<__nv_bfloat162 *>(&a), *reinterpret_cast<__nv_bfloat162 *>(&b));
    return *reinterpret_cast<uint32_t *>(&r);
}
__device__ __forceinline__ uint32_t vmax(uint4 w) { return mx2(mx2(w.x, w.y), mx2(w.z, w.w)); }

template <int T>
__device__ __forceinline__ uint32_t block_max(uint32_t m) {
    __shared__ uint32_t s[T / 32];
    for (int o = 16; o; o >>= 1) m = mx2(m, __shfl_xor_sync(~0u, m, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    m = s[0];
    for (int q = 1; q < T / 32; ++q) m = mx2(m, s[q]);
    return m;
}

// (a) the current K1 shape: grid (chunks, rows), 256 threads, VPT vectors per thread
template <int VPT>
__global__ void __launch_bounds__(256) k_grid(const char *base, long row_bytes, long vec_per_row, uint32_t *out) {
    pdl_wait();
    pdl_go();
    const long row = blockIdx.y;
    const uint4 *p = reinterpret_cast<const uint4 *>(base + row * row_bytes);
    const long v0 = (long)blockIdx.x * 256 * VPT;
    uint4 w[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
        const long v = v0 + threadIdx.x + u * 256;
        w[u] = v < vec_per_row ? ldnc(p + v) : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
    }
    uint32_t m = 0xFF80FF80u;
#pragma unroll
    for (int u = 0; u < VPT; ++u) m = mx2(m, vmax(w[u]));
    m = block_max<256>(m);
    if (threadIdx.x == 0) atomicMax(out + row, m & 0xFFFF);
}

// (b) flattened ranges: grid G, T threads, VPT vectors per thread (one wave)
template <int T, int VPT>
__global__ void __launch_bounds__(T) k_flat(const uint4 *base, long n_vec, uint32_t *out) {
    pdl_wait();
    pdl_go();
    const long per = (n_vec + gridDim.x - 1) / gridDim.x;
    const long v0 = blockIdx.x * per, v1 = min(n_vec, v0 + per);
    uint4 w[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
        const long v = v0 + threadIdx.x + (long)u * T;
        w[u] = v < v1 ? ldnc(base + v) : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
    }
    uint32_t m = 0xFF80FF80u;
#pragma unroll
    for (int u = 0; u < VPT; ++u) m = mx2(m, vmax(w[u]));
    for (long v = v0 + threadIdx.x + (long)VPT * T; v < v1; v += T) m = mx2(m, vmax(ldnc(base + v)));
    m = block_max<T>(m);
    if (threadIdx.x == 0) out[blockIdx.x] = m;
}

// (c) same as (b) inside clusters of CS CTAs, reduced to rank 0 through DSMEM
template <int T, int VPT>
__global__ void __launch_bounds__(T) k_cluster(const uint4 *base, long n_vec, uint32_t *out) {
    __shared__ uint32_t part[16];
    cg::cluster_group cl = cg::this_cluster();
    pdl_wait();
    pdl_go();
    const long per = (n_vec + gridDim.x - 1) / gridDim.x;
    const long v0 = blockIdx.x * per, v1 = min(n_vec, v0 + per);
    uint4 w[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
        const long v = v0 + threadIdx.x + (long)u * T;
        w[u] = v < v1 ? ldnc(base + v) : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
    }
    uint32_t m = 0xFF80FF80u;
#pragma unroll
    for (int u = 0; u < VPT; ++u) m = mx2(m, vmax(w[u]));
    for (long v = v0 + threadIdx.x + (long)VPT * T; v < v1; v += T) m = mx2(m, vmax(ldnc(base + v)));
    m = block_max<T>(m);
    const unsigned r = cl.block_rank();
    if (threadIdx.x == 0) {
        uint32_t *dst = cl.map_shared_rank(part, 0);
        dst[r] = m;
    }
    cl.sync();
    if (r == 0 && threadIdx.x == 0) {
        uint32_t x = part[0];
        for (unsigned q = 1; q < cl.num_blocks(); ++q) x = mx2(x, part[q]);
        out[blockIdx.x / cl.num_blocks()] = x;
    }
}

// (d) TMA bulk: one elected thread requests the CTA's whole range into shared memory in
// CHUNK-byte pieces (one mbarrier each), all threads reduce each piece as it lands
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int T, int CHUNK, int NCH>
__global__ void __launch_bounds__(T) k_tma(const char *base, long n_bytes, uint32_t *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (long)CHUNK * NCH);
    const long per = ((n_bytes + gridDim.x - 1) / gridDim.x + 15) / 16 * 16;
    const long b0 = blockIdx.x * per, b1 = min(n_bytes, b0 + per);
    const int nch = (int)((b1 - b0 + CHUNK - 1) / CHUNK);
    if (threadIdx.x == 0) {
        for (int c = 0; c < NCH; ++c) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + c)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();
    pdl_go();
    if (threadIdx.x == 0) {
        for (int c = 0; c < nch && c < NCH; ++c) {
            const long o = b0 + (long)c * CHUNK;
            const uint32_t nb = (uint32_t)min((long)CHUNK, b1 - o);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + c)), "r"(nb) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(sm + (long)c * CHUNK)), "l"(base + o), "r"(nb), "r"(su32(bar + c)) : "memory");
        }
    }
    uint32_t m = 0xFF80FF80u;
    for (int c = 0; c < nch && c < NCH; ++c) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n}"
                         : "=r"(ok) : "r"(su32(bar + c)) : "memory");
        const long o = b0 + (long)c * CHUNK;
        const int nv = (int)(min((long)CHUNK, b1 - o) / 16);
        const uint4 *s = reinterpret_cast<const uint4 *>(sm + (long)c * CHUNK);
        for (int v = threadIdx.x; v < nv; v += T) m = mx2(m, vmax(s[v]));
    }
    m = block_max<T>(m);
    if (threadIdx.x == 0) out[blockIdx.x] = m;
}

int main(int argc, char **argv) {
    const long rows = argc > 1 ? atol(argv[1]) : 48, V = argc > 2 ? atol(argv[2]) : 151936;
    const long row_bytes = V * 2, bytes = rows * row_bytes, n_vec = bytes / 16;
    const int RING = 16, N = 64;
    std::vector<char *> ring(RING);
    for (auto &p : ring) {
        CK(cudaMalloc(&p, bytes));
        CK(cudaMemset(p, 0x3F, bytes));
    }
    uint32_t *out;
    CK(cudaMalloc(&out, 1 << 20));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto run = [&](const char *name, auto launch_one) {
        for (int pdl = 0; pdl < 2; ++pdl) {
            for (int j = 0; j < 3; ++j) launch_one(ring[j], pdl);
            CK(cudaStreamSynchronize(s));
            cudaGraph_t g;
            cudaGraphExec_t ge;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
            for (int j = 0; j < N; ++j) launch_one(ring[j % RING], pdl);
            CK(cudaStreamEndCapture(s, &g));
            CK(cudaGraphInstantiate(&ge, g, 0));
            CK(cudaGraphLaunch(ge, s));
            CK(cudaStreamSynchronize(s));
            float best = 1e9;
            for (int rep = 0; rep < 7; ++rep) {
                CK(cudaEventRecord(e0, s));
                CK(cudaGraphLaunch(ge, s));
                CK(cudaEventRecord(e1, s));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                best = std::min(best, ms * 1e3f / N);
            }
            printf("%-44s pdl=%d  %7.2f us/launch  %7.1f GB/s\n", name, pdl, best, bytes / (best * 1e3));
            CK(cudaGraphExecDestroy(ge));
            CK(cudaGraphDestroy(g));
        }
    };
    auto cfg_launch = [&](auto kern, dim3 grid, dim3 block, size_t smem, int cluster, int pdl, auto... args) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = s;
        cudaLaunchAttribute at[2];
        int na = 0;
        if (pdl) { at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[na].val.programmaticStreamSerializationAllowed = 1; ++na; }
        if (cluster > 1) { at[na].id = cudaLaunchAttributeClusterDimension; at[na].val.clusterDim.x = cluster; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1; ++na; }
        cfg.attrs = at; cfg.numAttrs = na;
        CK(cudaLaunchKernelEx(&cfg, kern, args...));
    };
    char buf[128];
    printf("rows=%ld V=%ld bytes=%.2f MB sms=%d ring=%d (%.0f MB)\n", rows, V, bytes / 1e6, sms, RING, RING * bytes / 1e6);
    // (0) launch floor: empty-ish kernel of one CTA
    run("empty 1 CTA", [&](char *p, int pdl) { cfg_launch(k_flat<256, 1>, dim3(1), dim3(256), 0, 1, pdl, (const uint4 *)p, 0L, out); });
    // (a) current shape
    {
        const long vpr = row_bytes / 16, nch = (vpr + 2047) / 2048;
        snprintf(buf, sizeof buf, "grid %ldx%ld x256 vpt8 (current K1)", nch, rows);
        run(buf, [&](char *p, int pdl) { cfg_launch(k_grid<8>, dim3(nch, rows), dim3(256), 0, 1, pdl, (const char *)p, row_bytes, vpr, out); });
    }
    // (b) flattened one-wave shapes
    for (int G : {sms / 2, 96, 128, sms, 2 * sms, 4 * sms}) {
        const long per = (n_vec + G - 1) / G;
        if (per <= 256 * 4) {
            snprintf(buf, sizeof buf, "flat G=%d x256 vpt4 (%ld KB/CTA)", G, per * 16 / 1024);
            run(buf, [&](char *p, int pdl) { cfg_launch(k_flat<256, 4>, dim3(G), dim3(256), 0, 1, pdl, (const uint4 *)p, n_vec, out); });
        }
        if (per <= 512 * 8) {
            snprintf(buf, sizeof buf, "flat G=%d x512 vpt8 (%ld KB/CTA)", G, per * 16 / 1024);
            run(buf, [&](char *p, int pdl) { cfg_launch(k_flat<512, 8>, dim3(G), dim3(512), 0, 1, pdl, (const uint4 *)p, n_vec, out); });
        }
        if (per <= 512 * 16) {
            snprintf(buf, sizeof buf, "flat G=%d x512 vpt16 (%ld KB/CTA)", G, per * 16 / 1024);
            run(buf, [&](char *p, int pdl) { cfg_launch(k_flat<512, 16>, dim3(G), dim3(512), 0, 1, pdl, (const uint4 *)p, n_vec, out); });
        }
        if (per <= 1024 * 8) {
            snprintf(buf, sizeof buf, "flat G=%d x1024 vpt8 (%ld KB/CTA)", G, per * 16 / 1024);
            run(buf, [&](char *p, int pdl) { cfg_launch(k_flat<1024, 8>, dim3(G), dim3(1024), 0, 1, pdl, (const uint4 *)p, n_vec, out); });
        }
    }
    // (c) clusters
    for (int cs : {2, 4, 8, 16}) {
        if (cs == 16) CK(cudaFuncSetAttribute(k_cluster<512, 16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        const int G = 128;
        snprintf(buf, sizeof buf, "cluster%d G=%d x512 vpt16", cs, G);
        run(buf, [&](char *p, int pdl) { cfg_launch(k_cluster<512, 16>, dim3(G), dim3(512), 0, cs, pdl, (const uint4 *)p, n_vec, out); });
    }
    // (d) TMA bulk into shared memory
    {
        constexpr int CH = 16384, NCH = 12;
        const size_t smem = (size_t)CH * NCH + NCH * 8;
        CK(cudaFuncSetAttribute(k_tma<256, CH, NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_tma<512, CH, NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        for (int G : {96, 128, sms}) {
            if ((bytes + G - 1) / G > (long)CH * NCH) continue;
            snprintf(buf, sizeof buf, "tma G=%d x256 16KB chunks", G);
            run(buf, [&](char *p, int pdl) { cfg_launch(k_tma<256, CH, NCH>, dim3(G), dim3(256), smem, 1, pdl, (const char *)p, bytes, out); });
            snprintf(buf, sizeof buf, "tma G=%d x512 16KB chunks", G);
            run(buf, [&](char *p, int pdl) { cfg_launch(k_tma<512, CH, NCH>, dim3(G), dim3(512), smem, 1, pdl, (const char *)p, bytes, out); });
        }
    }
    return 0;
}
