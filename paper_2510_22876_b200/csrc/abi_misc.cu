// abi_misc.cu -- version, error reporting and device-property cache for libspecdec.so.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "host_util.h"

namespace specdec {

static thread_local std::string g_last_error;

int record_cuda_error(cudaError_t e) {
    g_last_error = cudaGetErrorString(e);
    return SPECDEC_ERR_CUDA;
}

int annotate_error(int rc, const char *where) {
    if (rc == SPECDEC_ERR_CUDA) g_last_error = std::string(where) + ": " + g_last_error;
    return rc;
}

static thread_local int g_pdl_suppress = 0;
void pdl_suppress(bool on) { g_pdl_suppress += on ? 1 : -1; }

int device_sm_count() {
    static std::mutex mu;
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    std::lock_guard<std::mutex> lk(mu);
    if (cache[dev] == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
        cache[dev] = n;
    }
    return cache[dev];
}

bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("SPECDEC_PDL");
        on = e ? atoi(e) != 0 : 1;
    }
    return on != 0 && g_pdl_suppress == 0;
}

// SPECDEC_CARVEOUT (percent of the unified L1 / shared-memory array given to shared memory,
// 0-100; unset or < 0: the driver's per-kernel default): every specdec kernel gets the same
// preferred carveout, so an SM switching between them (K1 -> K3 -> K2 of a round, K2's
// ~200 KB of shared memory) need not be reconfigured between kernels.
void ensure_carveout(const void *fn) {
    static int pct = -2;
    static std::mutex mu;
    static const void *done[128];
    static int n_done = 0;
    if (pct == -2) {
        const char *e = getenv("SPECDEC_CARVEOUT");
        pct = e ? atoi(e) : -1;
    }
    if (pct < 0) return;
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < n_done; ++i)
        if (done[i] == fn) return;
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
    cudaGetLastError();
    if (n_done < 128) done[n_done++] = fn;
}

}  // namespace specdec

extern "C" int specdec_version(void) { return 121; }  // 1.21: specdec_batch_init

extern "C" const char *specdec_last_cuda_error(void) { return specdec::g_last_error.c_str(); }
