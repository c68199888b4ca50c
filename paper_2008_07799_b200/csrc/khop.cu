// K1: bounded k-hop BFS from every source (replaces all_k_neighborhoods,
// graph.py:308-366).
//
// Tier 1 (warp per source): a 512-slot open-addressing hash set and a 256-entry
// BFS list live in shared memory.  A BFS level is expanded 32 frontier nodes at a
// time: lanes take the flattened (frontier node, edge) pairs (warp scan of the
// degrees + shuffle binary search), so neighbour-list loads are coalesced and no
// lane idles on low-degree frontiers.  New nodes are appended with a ballot-
// aggregated counter; the finished list is bitonic-sorted on the packed key
// (dist << 29 | id), which IS the reference's (dist, id) row order.
// Tier 2 (block per source, 1024 threads, 192 KB dynamic shared memory) re-runs
// the sources whose ball overflowed tier 1 (hubs, large k).  Both tiers run a
// count pass and a fill pass (two-phase ABI).
#include <cub/cub.cuh>

#include <climits>

#include "common.cuh"

namespace drg {
namespace {

constexpr uint32_t kEmpty = 0xffffffffu;
constexpr int kIdBits = 29;
constexpr uint32_t kIdMask = (1u << kIdBits) - 1;

constexpr int kWarpLog2Hash = 9;
constexpr int kWarpHash = 1 << kWarpLog2Hash;  // 512 slots
constexpr int kWarpList = 256;                  // BFS list entries incl. the source
constexpr int kWarpsPerBlock = 8;

constexpr int kBlockLog2Hash = 15;
constexpr int kBlockHash = 1 << kBlockLog2Hash;  // 32768 slots
constexpr int kBlockList = 16384;                 // entries incl. the source
constexpr int kBlockThreads = 1024;
constexpr size_t kBlockSmem = sizeof(uint32_t) * (kBlockHash + kBlockList + 1);

__device__ __forceinline__ uint32_t hslot(uint32_t key, int log2cap) {
    return (key * 2654435761u) >> (32 - log2cap);
}

__device__ __forceinline__ bool hash_insert(uint32_t *table, int log2cap, uint32_t key) {
    const uint32_t mask = (1u << log2cap) - 1;
    uint32_t s = hslot(key, log2cap);
    while (true) {
        uint32_t old = atomicCAS(&table[s], kEmpty, key);
        if (old == kEmpty) return true;
        if (old == key) return false;
        s = (s + 1) & mask;
    }
}

// Warp-cooperative: the calling warp expands frontier entries list[fb, fe)
// (fe - fb <= 32).  For every flattened (frontier node, edge) pair it inserts
// the neighbour; `emit(ins, w)` is called by all lanes (warp-uniform control).
template <class Emit>
__device__ __forceinline__ void expand_chunk(const int64_t *__restrict__ indptr,
                                             const int32_t *__restrict__ indices,
                                             const uint32_t *list, int fb, int fe,
                                             uint32_t *table, int log2cap, int lane,
                                             int64_t lim, Emit &&emit) {
    const int f = fb + lane;
    int64_t start = 0;
    int deg = 0;
    if (f < fe) {
        const uint32_t u = list[f] & kIdMask;
        start = indptr[u];
        deg = (int)min(indptr[u + 1] - start, lim);
    }
    int incl = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    const int excl = incl - deg;
    for (int base = 0; base < total; base += 32) {
        const int e = base + lane;
        int owner = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            int cand = owner + step;
            int ex = __shfl_sync(kFull, excl, cand);
            if (ex <= e) owner = cand;
        }
        const int64_t ostart = __shfl_sync(kFull, start, owner);
        const int oexcl = __shfl_sync(kFull, excl, owner);
        bool ins = false;
        uint32_t w = 0;
        if (e < total) {
            w = (uint32_t)__ldg(indices + ostart + (e - oexcl));
            ins = hash_insert(table, log2cap, w);
        }
        if (!emit(ins, w)) break;  // warp-uniform stop (overflow)
    }
}

__device__ __forceinline__ void bitonic_sort_warp(uint32_t *a, int P, int lane) {
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = lane; i < (P >> 1); i += 32) {
                int lo = 2 * i - (i & (stride - 1));
                int hi = lo + stride;
                bool up = (lo & size) == 0;
                uint32_t x = a[lo], y = a[hi];
                if ((x > y) == up) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
            __syncwarp();
        }
}

__device__ __forceinline__ void bitonic_sort_block(uint32_t *a, int P) {
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < (P >> 1); i += blockDim.x) {
                int lo = 2 * i - (i & (stride - 1));
                int hi = lo + stride;
                bool up = (lo & size) == 0;
                uint32_t x = a[lo], y = a[hi];
                if ((x > y) == up) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
            __syncthreads();
        }
}

// Neighbour cap (BASELINE C3): a capped row is the first `cap` entries of the full
// (dist, id)-sorted row.  The last hop (d == k-1) only starts when <= cap nodes
// (source included) are known, so at most r = cap + 1 - cnt entries come from it,
// the smallest ids not yet seen; each frontier node's row is sorted by id and fewer
// than cnt of its entries are already seen, so its first r + cnt = cap + 1 entries
// hold every candidate -- reading only those leaves the capped row unchanged (a
// Barabasi-Albert leaf next to a 5000-degree hub reads 257 entries, not 5000).
// `trunc` says the CSR rows are sorted (checked once on the device).
__device__ __forceinline__ int64_t last_hop_limit(int64_t cap, int d, int k, int trunc) {
    return (trunc && cap > 0 && d == k - 1) ? cap + 1 : INT64_MAX;
}

__global__ void rows_unsorted_kernel(const int64_t *__restrict__ indptr,
                                     const int32_t *__restrict__ indices, int64_t n, int *bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t e = indptr[i] + 1; e < indptr[i + 1]; ++e)
            if (indices[e - 1] >= indices[e]) {
                *bad = 1;
                break;
            }
}

// counts != nullptr: count pass.  Otherwise fill pass into out_ids/out_dists.
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    khop_warp_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                     int64_t n, int k, int64_t cap, int trunc, int64_t *counts,
                     const int64_t *__restrict__ out_indptr, int32_t *out_ids,
                     int32_t *out_dists, int32_t *ovf_list, unsigned long long *ovf_count) {
    __shared__ uint32_t s_table[kWarpsPerBlock][kWarpHash];
    __shared__ uint32_t s_list[kWarpsPerBlock][2 * kWarpList];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *table = s_table[warp];
    uint32_t *list = s_list[warp];
    for (int64_t s = (int64_t)blockIdx.x * kWarpsPerBlock + warp; s < n;
         s += (int64_t)gridDim.x * kWarpsPerBlock) {
        for (int i = lane; i < kWarpHash; i += 32) table[i] = kEmpty;
        __syncwarp();
        if (lane == 0) {
            hash_insert(table, kWarpLog2Hash, (uint32_t)s);
            list[0] = (uint32_t)s;
        }
        __syncwarp();
        int cnt = 1;
        bool overflow = false;
        int lb = 0, le = 1;
        for (int d = 0; d < k && !overflow; ++d) {
            const uint32_t tag = (uint32_t)(d + 1) << kIdBits;
            const int64_t lim = last_hop_limit(cap, d, k, trunc);
            for (int fb = lb; fb < le && !overflow; fb += 32) {
                expand_chunk(indptr, indices, list, fb, le, table, kWarpLog2Hash, lane, lim,
                             [&](bool ins, uint32_t w) {
                                 unsigned bal = __ballot_sync(kFull, ins);
                                 int pos = cnt + __popc(bal & ((1u << lane) - 1u));
                                 if (ins && pos < kWarpList) list[pos] = tag | w;
                                 cnt += __popc(bal);
                                 if (cnt > kWarpList) overflow = true;
                                 return !overflow;
                             });
            }
            __syncwarp();
            lb = le;
            le = cnt;
            if (cap > 0 && (int64_t)(cnt - 1) >= cap) break;  // later levels sort after the cap
        }
        if (overflow) {
            if (lane == 0) {
                unsigned long long i = atomicAdd(ovf_count, 1ull);
                ovf_list[i] = (int32_t)s;
                if (counts) counts[s] = 0;
            }
            __syncwarp();
            continue;
        }
        const int found = cnt - 1;
        int64_t row = found;
        if (cap > 0 && row > cap) row = cap;
        if (counts) {
            if (lane == 0) counts[s] = row;
        } else if (row > 0) {
            uint32_t *a = list + 1;
            int P = 1;
            while (P < found) P <<= 1;
            for (int i = found + lane; i < P; i += 32) a[i] = kEmpty;
            __syncwarp();
            bitonic_sort_warp(a, P, lane);
            const int64_t base = out_indptr[s];
            for (int q = lane; q < row; q += 32) {
                uint32_t v = a[q];
                out_ids[base + q] = (int32_t)(v & kIdMask);
                out_dists[base + q] = (int32_t)(v >> kIdBits);
            }
        }
        __syncwarp();
    }
}

// Tier 2: one 1024-thread block per overflowed source.
__global__ void __launch_bounds__(kBlockThreads)
    khop_block_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                      int k, int64_t cap, int trunc, const int32_t *__restrict__ sources,
                      int64_t n_sources, int64_t *counts, const int64_t *__restrict__ out_indptr,
                      int32_t *out_ids, int32_t *out_dists, int32_t *fail_source) {
    extern __shared__ uint32_t smem[];
    uint32_t *table = smem;
    uint32_t *list = smem + kBlockHash;
    __shared__ int s_cnt;
    __shared__ int s_ovf;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    for (int64_t idx = blockIdx.x; idx < n_sources; idx += gridDim.x) {
        const int32_t s = sources[idx];
        for (int i = threadIdx.x; i < kBlockHash; i += blockDim.x) table[i] = kEmpty;
        __syncthreads();
        if (threadIdx.x == 0) {
            hash_insert(table, kBlockLog2Hash, (uint32_t)s);
            list[0] = (uint32_t)s;
            s_cnt = 1;
            s_ovf = 0;
        }
        __syncthreads();
        int lb = 0, le = 1;
        for (int d = 0; d < k; ++d) {
            const uint32_t tag = (uint32_t)(d + 1) << kIdBits;
            const int64_t lim = last_hop_limit(cap, d, k, trunc);
            for (int fb = lb + warp * 32; fb < le; fb += nwarps * 32) {
                int fe = min(fb + 32, le);
                expand_chunk(indptr, indices, list, fb, fe, table, kBlockLog2Hash, lane, lim,
                             [&](bool ins, uint32_t w) {
                                 unsigned bal = __ballot_sync(kFull, ins);
                                 int base = 0;
                                 if (lane == 0 && bal) base = atomicAdd(&s_cnt, __popc(bal));
                                 base = __shfl_sync(kFull, base, 0);
                                 int pos = base + __popc(bal & ((1u << lane) - 1u));
                                 if (ins) {
                                     if (pos < kBlockList) list[pos] = tag | w;
                                     else s_ovf = 1;
                                 }
                                 int o = __shfl_sync(kFull, *(volatile int *)&s_ovf, 0);
                                 return o == 0;
                             });
                if (__shfl_sync(kFull, *(volatile int *)&s_ovf, 0)) break;
            }
            __syncthreads();
            const int cnt = s_cnt;
            const int ovf = s_ovf;
            __syncthreads();
            if (ovf) break;
            lb = le;
            le = cnt;
            if (cap > 0 && (int64_t)(cnt - 1) >= cap) break;
        }
        const int ovf = s_ovf;
        const int found = s_cnt - 1;
        __syncthreads();
        if (ovf) {
            if (threadIdx.x == 0) atomicCAS(fail_source, -1, s);
            continue;
        }
        int64_t row = found;
        if (cap > 0 && row > cap) row = cap;
        if (counts) {
            if (threadIdx.x == 0) counts[s] = row;
        } else if (row > 0) {
            uint32_t *a = list + 1;
            int P = 1;
            while (P < found) P <<= 1;
            for (int i = found + threadIdx.x; i < P; i += blockDim.x) a[i] = kEmpty;
            __syncthreads();
            bitonic_sort_block(a, P);
            const int64_t base = out_indptr[s];
            for (int q = threadIdx.x; q < row; q += blockDim.x) {
                uint32_t v = a[q];
                out_ids[base + q] = (int32_t)(v & kIdMask);
                out_dists[base + q] = (int32_t)(v >> kIdBits);
            }
        }
        __syncthreads();
    }
}

__global__ void k1_copy_kernel(const int32_t *__restrict__ indices, int64_t nnz, int32_t *ids,
                               int32_t *dists) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        ids[e] = indices[e];
        dists[e] = 1;
    }
}

int run_khop(const int64_t *indptr, const int32_t *indices, int64_t n, int k, int64_t cap,
             int64_t *counts, const int64_t *out_indptr, int32_t *out_ids, int32_t *out_dists,
             cudaStream_t st) {
    Scratch ovf(st), ovf_cnt(st), failbuf(st);
    DRG_CUDA(ovf.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(ovf_cnt.alloc(sizeof(unsigned long long)));
    DRG_CUDA(failbuf.alloc(sizeof(int32_t)));
    DRG_CUDA(cudaMemsetAsync(ovf_cnt.p, 0, sizeof(unsigned long long), st));
    DRG_CUDA(cudaMemsetAsync(failbuf.p, 0xff, sizeof(int32_t), st));
    int trunc = 0;
    if (cap > 0) {   // the last-hop truncation needs id-sorted rows
        Scratch bad(st);
        DRG_CUDA(bad.alloc(sizeof(int)));
        DRG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
        rows_unsorted_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), kSMs * 16), 256, 0,
                               st>>>(indptr, indices, n, bad.as<int>());
        DRG_LAUNCHED("rows_unsorted_kernel");
        int h_bad = 1;
        DRG_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        DRG_CUDA(cudaStreamSynchronize(st));
        trunc = h_bad == 0;
    }
    unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n, kWarpsPerBlock), kSMs * 32);
    khop_warp_kernel<<<blocks, kWarpsPerBlock * 32, 0, st>>>(
        indptr, indices, n, k, cap, trunc, counts, out_indptr, out_ids, out_dists,
        ovf.as<int32_t>(), ovf_cnt.as<unsigned long long>());
    DRG_LAUNCHED("khop_warp_kernel");
    unsigned long long h_ovf = 0;
    DRG_CUDA(cudaMemcpyAsync(&h_ovf, ovf_cnt.p, sizeof(h_ovf), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (h_ovf > 0) {
        DRG_CUDA(cudaFuncSetAttribute(khop_block_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kBlockSmem));
        unsigned b2 = (unsigned)std::min<unsigned long long>(h_ovf, kSMs);
        khop_block_kernel<<<b2, kBlockThreads, kBlockSmem, st>>>(
            indptr, indices, k, cap, trunc, ovf.as<int32_t>(), (int64_t)h_ovf, counts, out_indptr,
            out_ids, out_dists, failbuf.as<int32_t>());
        DRG_LAUNCHED("khop_block_kernel");
        int32_t h_fail = -1;
        DRG_CUDA(cudaMemcpyAsync(&h_fail, failbuf.p, sizeof(h_fail), cudaMemcpyDeviceToHost, st));
        DRG_CUDA(cudaStreamSynchronize(st));
        if (h_fail >= 0)
            return fail(DRG_ERR_UNSUPPORTED,
                        "k-hop ball of node %d exceeds %d entries (block tier capacity); "
                        "use a smaller k or a neighbour cap",
                        h_fail, kBlockList - 1);
    }
    return DRG_OK;
}

__global__ void degree_kernel(const int64_t *__restrict__ indptr, int64_t n, int64_t *counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        counts[i] = indptr[i + 1] - indptr[i];
}

}  // namespace
}  // namespace drg

using namespace drg;

extern "C" int drg_khop_count(const int64_t *indptr, const int32_t *indices, int64_t n, int k,
                              int64_t cap, int64_t *out_indptr, int64_t *out_nnz,
                              void *stream) {
    if (k < 1 || k > 6) return fail(DRG_ERR_INVALID, "k must be in [1, 6], got %d", k);
    if (n < 0 || n >= (1LL << kIdBits))
        return fail(DRG_ERR_INVALID, "node count %lld outside [0, 2^29)", (long long)n);
    if (!out_indptr || !out_nnz) return fail(DRG_ERR_INVALID, "null output");
    cudaStream_t st = as_stream(stream);
    if (n == 0) {
        DRG_CUDA(cudaMemsetAsync(out_indptr, 0, sizeof(int64_t), st));
        *out_nnz = 0;
        return DRG_OK;
    }
    Scratch counts(st), tmp(st);
    DRG_CUDA(counts.alloc(sizeof(int64_t) * (size_t)n));
    if (k == 1 && cap <= 0) {
        degree_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), kSMs * 16), 256, 0, st>>>(
            indptr, n, counts.as<int64_t>());
        DRG_LAUNCHED("degree_kernel");
    } else {
        DRG_TRY(run_khop(indptr, indices, n, k, cap, counts.as<int64_t>(), nullptr, nullptr,
                         nullptr, st));
    }
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, counts.as<int64_t>(), out_indptr + 1, n, st);
    DRG_CUDA(tmp.alloc(tb));
    DRG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, counts.as<int64_t>(), out_indptr + 1, n,
                                           st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    DRG_CUDA(cudaMemsetAsync(out_indptr, 0, sizeof(int64_t), st));
    DRG_CUDA(cudaMemcpyAsync(out_nnz, out_indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    return DRG_OK;
}

extern "C" int drg_khop_fill(const int64_t *indptr, const int32_t *indices, int64_t n, int k,
                             int64_t cap, const int64_t *out_indptr, int32_t *out_ids,
                             int32_t *out_dists, void *stream) {
    if (k < 1 || k > 6) return fail(DRG_ERR_INVALID, "k must be in [1, 6], got %d", k);
    if (n < 0 || n >= (1LL << kIdBits))
        return fail(DRG_ERR_INVALID, "node count %lld outside [0, 2^29)", (long long)n);
    cudaStream_t st = as_stream(stream);
    if (n == 0) return DRG_OK;
    if (k == 1 && cap <= 0) {
        int64_t nnz = 0;
        DRG_CUDA(cudaMemcpyAsync(&nnz, indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        DRG_CUDA(cudaStreamSynchronize(st));
        if (nnz > 0) {
            k1_copy_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nnz, 256), kSMs * 16), 256, 0,
                             st>>>(indices, nnz, out_ids, out_dists);
            DRG_LAUNCHED("k1_copy_kernel");
        }
        return DRG_OK;
    }
    return run_khop(indptr, indices, n, k, cap, nullptr, out_indptr, out_ids, out_dists, st);
}
