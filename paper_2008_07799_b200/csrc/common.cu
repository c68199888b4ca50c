// Library state: error messages, launch counter, version.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace drg {

std::atomic<uint64_t> g_launches{0};
static thread_local char g_msg[1024] = "";

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_msg, sizeof(g_msg), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    int code = (e == cudaErrorMemoryAllocation) ? DRG_ERR_NOMEM : DRG_ERR_CUDA;
    return fail(code, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

void keep_pool_reserved() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_dev = dev;
}

}  // namespace drg

extern "C" int drg_abi_version(void) { return DRG_ABI_VERSION; }
extern "C" const char *drg_last_error(void) { return drg::g_msg; }
extern "C" uint64_t drg_launch_count(void) {
    return drg::g_launches.load(std::memory_order_relaxed);
}
