// Shared helpers for the sm_100a kernels of the DRGraph layout path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/drgraph_b200.h"

namespace drg {

extern std::atomic<uint64_t> g_launches;

int fail(int code, const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what);

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Keep freed stream-ordered allocations reserved in the device pool (no re-map
// of multi-GB scratch on every call).
void keep_pool_reserved();

// Stream-ordered scratch allocation (freed on the same stream at scope exit).
struct Scratch {
    void *p = nullptr;
    cudaStream_t s;
    explicit Scratch(cudaStream_t st) : s(st) {}
    Scratch(const Scratch &) = delete;
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
    cudaError_t alloc(size_t bytes) {
        if (p) {
            cudaFreeAsync(p, s);
            p = nullptr;
        }
        keep_pool_reserved();
        return cudaMallocAsync(&p, bytes ? bytes : 16, s);
    }
    template <class T>
    T *as() const { return reinterpret_cast<T *>(p); }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Sort 64-bit (row << 32 | col) keys (+ optional fp64 values), drop keys whose row
// is >= n_rows (sentinels), sum duplicate keys' values, emit a CSR with rows
// sorted.  *out_nnz (host) receives the unique count.  Defined in coarsen.cu.
int sort_unique_csr(uint64_t *keys, double *vals, int64_t nnz, int64_t n_rows,
                    int64_t *out_indptr, int32_t *out_cols, double *out_vals, int64_t *out_nnz,
                    cudaStream_t st);

// grid size for warp-per-item kernels: one warp per item, `wpb` warps per block
inline unsigned warp_grid(int64_t items, int wpb) {
    int64_t g = ceil_div(items, wpb);
    if (g < 1) g = 1;
    if (g > 0x7fffffffLL) g = 0x7fffffffLL;
    return (unsigned)g;
}

// SM count of the current device (cached per device; 148 on B200)
inline int sm_count() {
    static int cache[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (cache[dev] == 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 148;
    }
    return cache[dev];
}

// ---- Philox4x32-10 counter-based RNG ----------------------------------------
struct u32x4 {
    uint32_t x, y, z, w;
};

// Philox4x32-R (Salmon et al., SC'11); R = 10 is the standard safety margin, R = 7
// already passes BigCrush (used where the draw count per step is high).
template <int ROUNDS = 10>
__device__ __forceinline__ u32x4 philox4x32(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < ROUNDS; ++r) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ float u32_to_unit(uint32_t v) {  // [0, 1), 24 bits
    return (float)(v >> 8) * (1.0f / 16777216.0f);
}

}  // namespace drg

#define DRG_LAUNCHED(name)                                          \
    do {                                                            \
        drg::g_launches.fetch_add(1, std::memory_order_relaxed);   \
        cudaError_t _e = cudaGetLastError();                        \
        if (_e != cudaSuccess) return drg::cuda_fail(_e, name);     \
    } while (0)

#define DRG_CUDA(call)                                              \
    do {                                                            \
        cudaError_t _e = (call);                                    \
        if (_e != cudaSuccess) return drg::cuda_fail(_e, #call);    \
    } while (0)

#define DRG_TRY(call)                                               \
    do {                                                            \
        int _rc = (call);                                           \
        if (_rc != DRG_OK) return _rc;                              \
    } while (0)
