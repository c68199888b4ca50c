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
// the sources whose ball overflowed tier 1 (hubs, large k).  Tier 3 (block per
// source, global memory) takes the balls of any size that overflow tier 2 (BA / R-MAT
// hubs at k >= 2, every source when k > 7): a visited-stamp array and a BFS list of n
// entries per resident block, level bounds per source, rows finished by a segmented
// sort of each level by id.  All tiers run a count pass and a fill pass (two-phase
// ABI); bfs_k_neighborhood (graph.py:280-305) is tier 3 on one source.
#include <cub/cub.cuh>

#include <algorithm>
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
constexpr int kMaxPackedK = (1 << (32 - kIdBits)) - 1;   // dist bits of the packed keys

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
                      int32_t *out_ids, int32_t *out_dists, int32_t *t3_list, int *t3_count) {
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
        if (ovf) {   // the global-memory tier takes it
            if (threadIdx.x == 0) t3_list[atomicAdd(t3_count, 1)] = s;
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

// ---- tier 3: global memory ---------------------------------------------------
// One block per source, any ball size.  Per resident block: stamp[n] (int32; a node
// is visited iff stamp == the source's tag, so nothing is cleared between sources)
// and list[n] (the BFS list, source first, levels contiguous in BFS order).  The
// count pass records found[idx]; the fill pass copies the list after the source to
// tmp[tmp_off[idx] ...] and the level starts to lvl[idx * (k + 1) + d] (list
// positions, d = 0..k; lvl[.. + k] = end), so that a segmented sort of every
// (source, level) run by id yields the reference's (dist, id) rows.
constexpr int kT3Threads = 1024;

__global__ void __launch_bounds__(kT3Threads)
    khop_global_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                       int64_t n, int k, int64_t cap, int trunc,
                       const int32_t *__restrict__ sources, int64_t n_sources, int tag_base,
                       int32_t *stamp_all, uint32_t *list_all, int64_t *found,
                       const int64_t *__restrict__ tmp_off, uint32_t *tmp, int64_t *lvl) {
    __shared__ unsigned long long s_cnt;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    int32_t *stamp = stamp_all + (size_t)blockIdx.x * n;
    uint32_t *list = list_all + (size_t)blockIdx.x * n;
    for (int64_t idx = blockIdx.x; idx < n_sources; idx += gridDim.x) {
        const int32_t s = sources[idx];
        const int32_t tag = tag_base + (int32_t)idx + 1;
        if (threadIdx.x == 0) {
            stamp[s] = tag;
            list[0] = (uint32_t)s;
            s_cnt = 1;
        }
        __syncthreads();
        int64_t lb = 0, le = 1;
        int d = 0;
        if (lvl && threadIdx.x == 0) lvl[idx * (k + 1)] = 1;
        for (; d < k; ++d) {
            const int64_t lim = last_hop_limit(cap, d, k, trunc);
            for (int64_t fb = lb + warp * 32; fb < le; fb += (int64_t)nwarps * 32) {
                const int64_t f = fb + lane;
                int64_t start = 0;
                int64_t deg = 0;
                if (f < le) {
                    const uint32_t u = list[f];
                    start = indptr[u];
                    deg = min(indptr[u + 1] - start, lim);
                }
                int64_t incl = deg;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int64_t t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += t;
                }
                const int64_t total = __shfl_sync(kFull, incl, 31);
                const int64_t excl = incl - deg;
                for (int64_t base = 0; base < total; base += 32) {
                    const int64_t e = base + lane;
                    int owner = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const int cand = owner + step;
                        if (__shfl_sync(kFull, excl, cand) <= e) owner = cand;
                    }
                    const int64_t ostart = __shfl_sync(kFull, start, owner);
                    const int64_t oexcl = __shfl_sync(kFull, excl, owner);
                    bool ins = false;
                    uint32_t w = 0;
                    if (e < total) {
                        w = (uint32_t)__ldg(indices + ostart + (e - oexcl));
                        ins = atomicExch(stamp + w, tag) != tag;
                    }
                    const unsigned bal = __ballot_sync(kFull, ins);
                    unsigned long long b0 = 0;
                    if (lane == 0 && bal) b0 = atomicAdd(&s_cnt, (unsigned long long)__popc(bal));
                    b0 = __shfl_sync(kFull, b0, 0);
                    if (ins) list[b0 + __popc(bal & ((1u << lane) - 1u))] = w;
                }
            }
            __syncthreads();
            const int64_t cnt = (int64_t)s_cnt;
            __syncthreads();
            lb = le;
            le = cnt;
            if (lvl && threadIdx.x == 0) lvl[idx * (k + 1) + d + 1] = cnt;
            if (cnt == lb) { ++d; break; }                    // no new level
            if (cap > 0 && cnt - 1 >= cap) { ++d; break; }    // later levels sort after the cap
        }
        if (lvl && threadIdx.x == 0)
            for (int q = d + 1; q <= k; ++q) lvl[idx * (k + 1) + q] = le;
        const int64_t nf = le - 1;
        if (found && threadIdx.x == 0) found[idx] = nf;
        if (tmp) {
            uint32_t *dst = tmp + tmp_off[idx];
            for (int64_t q = threadIdx.x; q < nf; q += blockDim.x) dst[q] = list[1 + q];
        }
        __syncthreads();
    }
}

// segment bounds of the (source, level) runs in tmp coordinates
__global__ void t3_segments_kernel(const int64_t *__restrict__ lvl, const int64_t *__restrict__ tmp_off,
                                   int64_t n_sources, int k, int64_t *beg, int64_t *end) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_sources * k;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = g / k, d = g - idx * k;
        beg[g] = tmp_off[idx] + lvl[idx * (k + 1) + d] - 1;
        end[g] = tmp_off[idx] + lvl[idx * (k + 1) + d + 1] - 1;
    }
}

// count pass: counts[s] = row length; fill pass: the first row entries of the sorted
// runs into the output rows (dist from the level bounds)
__global__ void t3_emit_kernel(const int32_t *__restrict__ sources, int64_t n_sources, int k,
                               int64_t cap, const int64_t *__restrict__ found,
                               const int64_t *__restrict__ lvl, const int64_t *__restrict__ tmp_off,
                               const uint32_t *__restrict__ sorted, int64_t *counts,
                               const int64_t *__restrict__ out_indptr, int32_t *out_ids,
                               int32_t *out_dists) {
    for (int64_t idx = blockIdx.x; idx < n_sources; idx += gridDim.x) {
        const int32_t s = sources[idx];
        int64_t row = found[idx];
        if (cap > 0 && row > cap) row = cap;
        if (counts) {
            if (threadIdx.x == 0) counts[s] = row;
            continue;
        }
        const int64_t base = out_indptr[s];
        const int64_t *L = lvl + idx * (k + 1);
        for (int64_t q = threadIdx.x; q < row; q += blockDim.x) {
            int d = 0;
            while (d + 1 < k && L[d + 1] - 1 <= q) ++d;
            out_ids[base + q] = (int32_t)sorted[tmp_off[idx] + q];
            out_dists[base + q] = d + 1;
        }
    }
}

// Tier 3 over `sources` (device int32[n_sources]).  counts != NULL: count pass.
// found_out (optional, device int64[n_sources]) receives the full ball sizes.
int run_tier3(const int64_t *indptr, const int32_t *indices, int64_t n, int k, int64_t cap,
              int trunc, const int32_t *sources, int64_t n_sources, int64_t *counts,
              const int64_t *out_indptr, int32_t *out_ids, int32_t *out_dists,
              int64_t *found_out, cudaStream_t st) {
    if (n_sources <= 0) return DRG_OK;
    // resident blocks: one per SM, bounded by a 2 GB budget of stamp + list arrays
    const int64_t per_block = 8 * std::max<int64_t>(n, 1);
    const int64_t G = std::max<int64_t>(1, std::min<int64_t>({n_sources, (int64_t)sm_count(),
                                                              (int64_t(2) << 30) / per_block}));
    Scratch stamp(st), list(st), found(st);
    DRG_CUDA(stamp.alloc(sizeof(int32_t) * (size_t)(G * n)));
    DRG_CUDA(list.alloc(sizeof(uint32_t) * (size_t)(G * n)));
    DRG_CUDA(found.alloc(sizeof(int64_t) * (size_t)n_sources));
    DRG_CUDA(cudaMemsetAsync(stamp.p, 0, sizeof(int32_t) * (size_t)(G * n), st));
    khop_global_kernel<<<(unsigned)G, kT3Threads, 0, st>>>(
        indptr, indices, n, k, cap, trunc, sources, n_sources, 0, stamp.as<int32_t>(),
        list.as<uint32_t>(), found.as<int64_t>(), nullptr, nullptr, nullptr);
    DRG_LAUNCHED("khop_global_kernel");
    if (found_out)
        DRG_CUDA(cudaMemcpyAsync(found_out, found.p, sizeof(int64_t) * (size_t)n_sources,
                                 cudaMemcpyDeviceToDevice, st));
    if (counts) {
        t3_emit_kernel<<<(unsigned)std::min<int64_t>(n_sources, 4096), 32, 0, st>>>(
            sources, n_sources, k, cap, found.as<int64_t>(), nullptr, nullptr, nullptr, counts,
            nullptr, nullptr, nullptr);
        DRG_LAUNCHED("t3_emit_kernel");
        return DRG_OK;
    }
    if (!out_ids) return DRG_OK;
    // fill: offsets of every source's ball in tmp, the BFS again (tags past the
    // count pass's), a segmented sort per (source, level), then the row prefixes
    Scratch off(st), tb(st), tmp(st), sorted(st), lvl(st), beg(st), endb(st);
    DRG_CUDA(off.alloc(sizeof(int64_t) * (size_t)(n_sources + 1)));
    DRG_CUDA(cudaMemsetAsync(off.p, 0, sizeof(int64_t), st));
    size_t tbytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tbytes, found.as<int64_t>(), off.as<int64_t>() + 1,
                                  n_sources, st);
    DRG_CUDA(tb.alloc(tbytes));
    DRG_CUDA(cub::DeviceScan::InclusiveSum(tb.p, tbytes, found.as<int64_t>(),
                                           off.as<int64_t>() + 1, n_sources, st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    int64_t total = 0;
    DRG_CUDA(cudaMemcpyAsync(&total, off.as<int64_t>() + n_sources, sizeof(int64_t),
                             cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    DRG_CUDA(tmp.alloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(total, 1)));
    DRG_CUDA(sorted.alloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(total, 1)));
    DRG_CUDA(lvl.alloc(sizeof(int64_t) * (size_t)(n_sources * (k + 1))));
    if (n_sources + 1 >= 0x7fffffff) return fail(DRG_ERR_UNSUPPORTED, "too many tier-3 sources");
    khop_global_kernel<<<(unsigned)G, kT3Threads, 0, st>>>(
        indptr, indices, n, k, cap, trunc, sources, n_sources, (int)n_sources,
        stamp.as<int32_t>(), list.as<uint32_t>(), nullptr, off.as<int64_t>(),
        tmp.as<uint32_t>(), lvl.as<int64_t>());
    DRG_LAUNCHED("khop_global_kernel");
    const int64_t nseg = n_sources * k;
    DRG_CUDA(beg.alloc(sizeof(int64_t) * (size_t)nseg));
    DRG_CUDA(endb.alloc(sizeof(int64_t) * (size_t)nseg));
    t3_segments_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nseg, 256), 4096), 256, 0, st>>>(
        lvl.as<int64_t>(), off.as<int64_t>(), n_sources, k, beg.as<int64_t>(), endb.as<int64_t>());
    DRG_LAUNCHED("t3_segments_kernel");
    if (total > 0) {
        size_t sb = 0;
        cub::DeviceSegmentedSort::SortKeys(nullptr, sb, tmp.as<uint32_t>(), sorted.as<uint32_t>(),
                                           total, nseg, beg.as<int64_t>(), endb.as<int64_t>(), st);
        Scratch sbuf(st);
        DRG_CUDA(sbuf.alloc(sb));
        DRG_CUDA(cub::DeviceSegmentedSort::SortKeys(sbuf.p, sb, tmp.as<uint32_t>(),
                                                    sorted.as<uint32_t>(), total, nseg,
                                                    beg.as<int64_t>(), endb.as<int64_t>(), st));
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    t3_emit_kernel<<<(unsigned)std::min<int64_t>(n_sources, 4096), 256, 0, st>>>(
        sources, n_sources, k, cap, found.as<int64_t>(), lvl.as<int64_t>(), off.as<int64_t>(),
        sorted.as<uint32_t>(), nullptr, out_indptr, out_ids, out_dists);
    DRG_LAUNCHED("t3_emit_kernel");
    DRG_CUDA(cudaStreamSynchronize(st));   // scratch lifetimes end with the call
    return DRG_OK;
}

__global__ void iota_kernel(int32_t *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)i;
}

int rows_sorted_flag(const int64_t *indptr, const int32_t *indices, int64_t n, int64_t cap,
                     cudaStream_t st, int *trunc) {
    *trunc = 0;
    if (cap <= 0) return DRG_OK;   // the last-hop truncation needs id-sorted rows
    Scratch bad(st);
    DRG_CUDA(bad.alloc(sizeof(int)));
    DRG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    rows_unsorted_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), sm_count() * 16), 256, 0,
                           st>>>(indptr, indices, n, bad.as<int>());
    DRG_LAUNCHED("rows_unsorted_kernel");
    int h_bad = 1;
    DRG_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    *trunc = h_bad == 0;
    return DRG_OK;
}

int run_khop(const int64_t *indptr, const int32_t *indices, int64_t n, int k, int64_t cap,
             int64_t *counts, const int64_t *out_indptr, int32_t *out_ids, int32_t *out_dists,
             cudaStream_t st) {
    int trunc = 0;
    DRG_TRY(rows_sorted_flag(indptr, indices, n, cap, st, &trunc));
    if (k > kMaxPackedK) {   // (dist << 29 | id) keys hold dist <= 7: tier 3 only
        Scratch all(st);
        DRG_CUDA(all.alloc(sizeof(int32_t) * (size_t)n));
        iota_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), sm_count() * 16), 256, 0, st>>>(
            all.as<int32_t>(), n);
        DRG_LAUNCHED("iota_kernel");
        return run_tier3(indptr, indices, n, k, cap, trunc, all.as<int32_t>(), n, counts,
                         out_indptr, out_ids, out_dists, nullptr, st);
    }
    Scratch ovf(st), ovf_cnt(st), t3(st), t3_cnt(st);
    DRG_CUDA(ovf.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(ovf_cnt.alloc(sizeof(unsigned long long)));
    DRG_CUDA(cudaMemsetAsync(ovf_cnt.p, 0, sizeof(unsigned long long), st));
    unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n, kWarpsPerBlock), sm_count() * 32);
    khop_warp_kernel<<<blocks, kWarpsPerBlock * 32, 0, st>>>(
        indptr, indices, n, k, cap, trunc, counts, out_indptr, out_ids, out_dists,
        ovf.as<int32_t>(), ovf_cnt.as<unsigned long long>());
    DRG_LAUNCHED("khop_warp_kernel");
    unsigned long long h_ovf = 0;
    DRG_CUDA(cudaMemcpyAsync(&h_ovf, ovf_cnt.p, sizeof(h_ovf), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (h_ovf > 0) {
        DRG_CUDA(t3.alloc(sizeof(int32_t) * (size_t)h_ovf));
        DRG_CUDA(t3_cnt.alloc(sizeof(int)));
        DRG_CUDA(cudaMemsetAsync(t3_cnt.p, 0, sizeof(int), st));
        DRG_CUDA(cudaFuncSetAttribute(khop_block_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kBlockSmem));
        unsigned b2 = (unsigned)std::min<unsigned long long>(h_ovf, sm_count());
        khop_block_kernel<<<b2, kBlockThreads, kBlockSmem, st>>>(
            indptr, indices, k, cap, trunc, ovf.as<int32_t>(), (int64_t)h_ovf, counts, out_indptr,
            out_ids, out_dists, t3.as<int32_t>(), t3_cnt.as<int>());
        DRG_LAUNCHED("khop_block_kernel");
        int h_t3 = 0;
        DRG_CUDA(cudaMemcpyAsync(&h_t3, t3_cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        DRG_CUDA(cudaStreamSynchronize(st));
        if (h_t3 > 0)
            DRG_TRY(run_tier3(indptr, indices, n, k, cap, trunc, t3.as<int32_t>(), h_t3, counts,
                              out_indptr, out_ids, out_dists, nullptr, st));
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
    if (k < 1) return fail(DRG_ERR_INVALID, "k must be >= 1, got %d", k);
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
        degree_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), sm_count() * 16), 256, 0, st>>>(
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
    if (k < 1) return fail(DRG_ERR_INVALID, "k must be >= 1, got %d", k);
    if (n < 0 || n >= (1LL << kIdBits))
        return fail(DRG_ERR_INVALID, "node count %lld outside [0, 2^29)", (long long)n);
    cudaStream_t st = as_stream(stream);
    if (n == 0) return DRG_OK;
    if (k == 1 && cap <= 0) {
        int64_t nnz = 0;
        DRG_CUDA(cudaMemcpyAsync(&nnz, indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        DRG_CUDA(cudaStreamSynchronize(st));
        if (nnz > 0) {
            k1_copy_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nnz, 256), sm_count() * 16), 256, 0,
                             st>>>(indices, nnz, out_ids, out_dists);
            DRG_LAUNCHED("k1_copy_kernel");
        }
        return DRG_OK;
    }
    return run_khop(indptr, indices, n, k, cap, nullptr, out_indptr, out_ids, out_dists, st);
}

/* bfs_k_neighborhood (graph.py:280-305): tier 3 on one source. */
extern "C" int drg_khop_source(const int64_t *indptr, const int32_t *indices, int64_t n, int k,
                               int64_t source, int32_t *out_ids, int32_t *out_dists,
                               int64_t capacity, int64_t *out_count, void *stream) {
    if (k < 1) return fail(DRG_ERR_INVALID, "k must be >= 1, got %d", k);
    if (n <= 0 || n >= (1LL << kIdBits))
        return fail(DRG_ERR_INVALID, "node count %lld outside [1, 2^29)", (long long)n);
    if (source < 0 || source >= n)
        return fail(DRG_ERR_INVALID, "source %lld out of range for %lld nodes", (long long)source,
                    (long long)n);
    if (!out_count) return fail(DRG_ERR_INVALID, "null output");
    cudaStream_t st = as_stream(stream);
    Scratch src(st), found(st), cnt(st), ip(st);
    DRG_CUDA(src.alloc(sizeof(int32_t)));
    DRG_CUDA(found.alloc(sizeof(int64_t)));
    const int32_t s32 = (int32_t)source;
    DRG_CUDA(cudaMemcpyAsync(src.p, &s32, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    DRG_TRY(run_tier3(indptr, indices, n, k, 0, 0, src.as<int32_t>(), 1, nullptr, nullptr, nullptr,
                      nullptr, found.as<int64_t>(), st));
    int64_t h_found = 0;
    DRG_CUDA(cudaMemcpyAsync(&h_found, found.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    *out_count = h_found;
    if (!out_ids || h_found == 0) return DRG_OK;
    if (capacity < h_found) return fail(DRG_ERR_INVALID, "output capacity %lld < %lld entries",
                                        (long long)capacity, (long long)h_found);
    // the fill path writes at out_indptr[source]: a one-entry offset array
    DRG_CUDA(ip.alloc(sizeof(int64_t) * (size_t)(n + 1)));
    DRG_CUDA(cudaMemsetAsync(ip.p, 0, sizeof(int64_t) * (size_t)(n + 1), st));
    return run_tier3(indptr, indices, n, k, 0, 0, src.as<int32_t>(), 1, nullptr, ip.as<int64_t>(),
                     out_ids, out_dists, nullptr, st);
}
