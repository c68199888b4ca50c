// Connected-component count (replaces connected_components, graph.py:369-388; the
// reference layout only logs it and reports stats["components"],
// optimizer.py:374-378).  Lock-free union-find: hook the larger root under the
// smaller with atomicCAS, path halving in find, then count roots.
#include <cub/cub.cuh>

#include "common.cuh"

namespace drg {
namespace {

__device__ __forceinline__ int32_t find_root(int32_t *parent_, int32_t x) {
    volatile int32_t *parent = parent_;
    int32_t p = parent[x];
    while (p != x) {
        const int32_t gp = parent[p];
        if (gp != p) parent[x] = gp;  // path halving (benign race)
        x = p;
        p = parent[x];
    }
    return x;
}

__global__ void cc_init_kernel(int32_t *parent, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        parent[i] = (int32_t)i;
}

__device__ __forceinline__ void hook(int32_t *parent, int32_t a, int32_t b) {
    while (true) {
        a = find_root(parent, a);
        b = find_root(parent, b);
        if (a == b) return;
        if (a < b) {
            int32_t t = a;
            a = b;
            b = t;
        }
        if (atomicCAS(parent + a, a, b) == a) return;
    }
}

constexpr int64_t kLongRow = 1024;   // rows above this go to the block-per-row pass

// Thread per node for rows up to kLongRow entries; longer rows (R-MAT hubs: a
// thread looping over a 10^5-entry row held the whole pass for 0.4 s) are queued.
__global__ void cc_hook_kernel(const int64_t *__restrict__ indptr,
                               const int32_t *__restrict__ indices, int64_t n, int32_t *parent,
                               int32_t *long_rows, int *n_long) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = indptr[v], hi = indptr[v + 1];
        if (hi - lo > kLongRow) {
            long_rows[atomicAdd(n_long, 1)] = (int32_t)v;
            continue;
        }
        for (int64_t e = lo; e < hi; ++e) {
            const int32_t u = __ldg(indices + e);
            if (u > v) hook(parent, (int32_t)v, u);
        }
    }
}

// Block per queued long row, threads striding over its entries.
__global__ void cc_hook_long_kernel(const int64_t *__restrict__ indptr,
                                    const int32_t *__restrict__ indices,
                                    const int32_t *__restrict__ long_rows,
                                    const int *__restrict__ n_long, int32_t *parent) {
    const int nl = *n_long;
    for (int r = blockIdx.x; r < nl; r += gridDim.x) {
        const int32_t v = long_rows[r];
        for (int64_t e = indptr[v] + threadIdx.x; e < indptr[v + 1]; e += blockDim.x) {
            const int32_t u = __ldg(indices + e);
            if (u > v) hook(parent, v, u);
        }
    }
}

__global__ void cc_count_kernel(int32_t *parent, int64_t n, unsigned long long *count) {
    unsigned long long local = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        local += (find_root(parent, (int32_t)i) == (int32_t)i);
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(kFull, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

__global__ void cc_flag_kernel(int32_t *parent, int64_t n, int32_t *is_root) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = find_root(parent, (int32_t)i);
        parent[i] = r;
        is_root[i] = (r == (int32_t)i) ? 1 : 0;
    }
}

// roots are component minima (hooks go larger -> smaller), so numbering roots in id
// order reproduces the reference's first-seen labels
__global__ void cc_label_kernel(const int32_t *__restrict__ parent,
                                const int32_t *__restrict__ root_rank, int64_t n,
                                int32_t *labels) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        labels[i] = root_rank[parent[i]];
}

}  // namespace
}  // namespace drg

using namespace drg;

extern "C" int drg_components(const int64_t *indptr, const int32_t *indices, int64_t n,
                              int32_t *out_labels, int64_t *out_count, void *stream) {
    if (n < 0 || n >= 0x7fffffffLL) return fail(DRG_ERR_INVALID, "bad node count");
    *out_count = 0;
    if (n == 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    Scratch parent(st), cnt(st);
    DRG_CUDA(parent.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(cnt.alloc(sizeof(unsigned long long)));
    DRG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(n, 256), sm_count() * 32);
    cc_init_kernel<<<g, 256, 0, st>>>(parent.as<int32_t>(), n);
    DRG_LAUNCHED("cc_init_kernel");
    Scratch lst(st), nl(st);
    DRG_CUDA(lst.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(nl.alloc(sizeof(int)));
    DRG_CUDA(cudaMemsetAsync(nl.p, 0, sizeof(int), st));
    cc_hook_kernel<<<g, 256, 0, st>>>(indptr, indices, n, parent.as<int32_t>(),
                                      lst.as<int32_t>(), nl.as<int>());
    DRG_LAUNCHED("cc_hook_kernel");
    cc_hook_long_kernel<<<sm_count() * 4, 256, 0, st>>>(indptr, indices, lst.as<int32_t>(),
                                                  nl.as<int>(), parent.as<int32_t>());
    DRG_LAUNCHED("cc_hook_long_kernel");
    cc_count_kernel<<<g, 256, 0, st>>>(parent.as<int32_t>(), n, cnt.as<unsigned long long>());
    DRG_LAUNCHED("cc_count_kernel");
    unsigned long long h = 0;
    DRG_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    *out_count = (int64_t)h;
    if (out_labels) {
        Scratch flags(st), rk(st), tmp(st);
        DRG_CUDA(flags.alloc(sizeof(int32_t) * (size_t)n));
        DRG_CUDA(rk.alloc(sizeof(int32_t) * (size_t)n));
        cc_flag_kernel<<<g, 256, 0, st>>>(parent.as<int32_t>(), n, flags.as<int32_t>());
        DRG_LAUNCHED("cc_flag_kernel");
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, flags.as<int32_t>(), rk.as<int32_t>(), n, st);
        DRG_CUDA(tmp.alloc(tb));
        DRG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flags.as<int32_t>(), rk.as<int32_t>(),
                                               n, st));
        g_launches.fetch_add(1, std::memory_order_relaxed);
        cc_label_kernel<<<g, 256, 0, st>>>(parent.as<int32_t>(), rk.as<int32_t>(), n, out_labels);
        DRG_LAUNCHED("cc_label_kernel");
    }
    return DRG_OK;
}
