// K4: greedy coarsening as a lexicographically-first MIS (replaces
// coarsen_with_order, multilevel.py:48-79), coarse CSR, map composition, and the
// A10 level aggregation.
//
// The reference visits nodes in order pi; an unassigned node becomes a seed and
// absorbs its unassigned neighbours.  Equivalently (SURVEY §7 hard part 4): with
// rank(v) = position of v in pi, v is a seed iff no lower-ranked neighbour is a
// seed (the greedy MIS under rank), a non-seed's parent is its minimum-rank seed
// neighbour, and coarse ids are dense in seed-rank order.  The MIS is resolved in
// rounds: an undecided node turns NONSEED as soon as a lower-ranked neighbour is a
// SEED and turns SEED once all lower-ranked neighbours are decided NONSEED.
// Decisions are monotone, so in-place (chaotic) updates inside a round are safe.
#include <cub/cub.cuh>

#include "common.cuh"

namespace drg {
namespace {

constexpr int8_t kUndecided = 0, kSeed = 1, kNonSeed = 2;
constexpr int kWpb = 8;

__global__ void rank_kernel(const int64_t *__restrict__ order, int64_t n, int32_t *rank,
                            int *bad) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = order[r];
        if (v < 0 || v >= n) {
            atomicExch(bad, 1);
            continue;
        }
        rank[v] = (int32_t)r;
    }
}

// warp per undecided node
__global__ void __launch_bounds__(kWpb * 32)
    mis_round_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                     int64_t n, const int32_t *__restrict__ rank, int8_t *status,
                     unsigned long long *undecided) {
    const int lane = threadIdx.x & 31;
    unsigned long long local = 0;
    for (int64_t v = (int64_t)blockIdx.x * kWpb + (threadIdx.x >> 5); v < n;
         v += (int64_t)gridDim.x * kWpb) {
        if (((volatile int8_t *)status)[v] != kUndecided) continue;
        const int32_t rv = rank[v];
        bool seed_lower = false, pending = false;
        for (int64_t e = indptr[v] + lane; e < indptr[v + 1]; e += 32) {
            const int32_t u = __ldg(indices + e);
            if (__ldg(rank + u) < rv) {
                const int8_t s = ((volatile int8_t *)status)[u];
                seed_lower |= (s == kSeed);
                pending |= (s == kUndecided);
            }
        }
        seed_lower = __any_sync(kFull, seed_lower);
        pending = __any_sync(kFull, pending);
        if (lane == 0) {
            if (seed_lower) status[v] = kNonSeed;
            else if (!pending) status[v] = kSeed;
            else local++;
        }
    }
    if (lane == 0 && local) atomicAdd(undecided, local);
}

__global__ void seed_flag_kernel(const int64_t *__restrict__ order, int64_t n,
                                 const int8_t *__restrict__ status, int32_t *flag_by_rank) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        flag_by_rank[r] = status[order[r]] == kSeed ? 1 : 0;
}

__global__ void __launch_bounds__(kWpb * 32)
    parent_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                  int64_t n, const int32_t *__restrict__ rank, const int8_t *__restrict__ status,
                  const int32_t *__restrict__ id_by_rank, int32_t *parent) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = (int64_t)blockIdx.x * kWpb + (threadIdx.x >> 5); v < n;
         v += (int64_t)gridDim.x * kWpb) {
        if (status[v] == kSeed) {
            if (lane == 0) parent[v] = id_by_rank[rank[v]];
            continue;
        }
        int32_t best = 0x7fffffff;
        for (int64_t e = indptr[v] + lane; e < indptr[v + 1]; e += 32) {
            const int32_t u = __ldg(indices + e);
            if (status[u] == kSeed) best = min(best, __ldg(rank + u));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(kFull, best, o));
        if (lane == 0) parent[v] = id_by_rank[best];
    }
}

// keys (parent[src] << 32 | parent[dst]) for every directed entry; entries whose
// endpoints share a parent get the sentinel (n_coarse << 32), which sorts last.
template <class V>
__global__ void __launch_bounds__(kWpb * 32)
    pair_keys_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ targets,
                     const V *__restrict__ vals, int64_t n, const int32_t *__restrict__ parent,
                     int64_t n_coarse, uint64_t *keys, V *vals_out) {
    const int lane = threadIdx.x & 31;
    const uint64_t sentinel = (uint64_t)n_coarse << 32;
    for (int64_t v = (int64_t)blockIdx.x * kWpb + (threadIdx.x >> 5); v < n;
         v += (int64_t)gridDim.x * kWpb) {
        const uint64_t a = (uint32_t)parent[v];
        for (int64_t e = indptr[v] + lane; e < indptr[v + 1]; e += 32) {
            const uint32_t b = (uint32_t)__ldg(parent + __ldg(targets + e));
            keys[e] = (a == b) ? sentinel : ((a << 32) | b);
            if (vals) vals_out[e] = vals[e];
        }
    }
}

// CSR from sorted unique keys: indptr[a] = first key index with row >= a.
__global__ void csr_from_keys_kernel(const uint64_t *__restrict__ keys, int64_t nnz,
                                     int64_t n_rows, int64_t *indptr, int32_t *cols) {
    for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a <= n_rows;
         a += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t probe = (uint64_t)a << 32;
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < probe) lo = mid + 1;
            else hi = mid;
        }
        indptr[a] = lo;
    }
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x)
        cols[e] = (int32_t)(keys[e] & 0xffffffffu);
}

// from_edges keys: both directions of every non-loop pair (graph.py:101-110)
__global__ void edge_keys_kernel(const int64_t *__restrict__ pairs, int64_t m, int64_t n,
                                 uint64_t *keys, int *bad) {
    const uint64_t sentinel = (uint64_t)n << 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = pairs[2 * i], v = pairs[2 * i + 1];
        if (u < 0 || v < 0 || u >= n || v >= n) {
            atomicExch(bad, 1);
            keys[2 * i] = keys[2 * i + 1] = sentinel;
            continue;
        }
        if (u == v) {
            keys[2 * i] = keys[2 * i + 1] = sentinel;
        } else {
            keys[2 * i] = ((uint64_t)u << 32) | (uint64_t)v;
            keys[2 * i + 1] = ((uint64_t)v << 32) | (uint64_t)u;
        }
    }
}

__global__ void compose_kernel(const int32_t *__restrict__ first,
                               const int32_t *__restrict__ second, int64_t n, int32_t *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = second[first[i]];
}

__global__ void iota_kernel(int32_t *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)i;
}

inline unsigned flat_grid(int64_t n, int threads = 256) {
    return (unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(n, threads), 1), sm_count() * 32);
}

inline int bits_for(uint64_t v) {
    int b = 0;
    while (b < 64 && (v >> b) != 0) ++b;
    return b;
}

}  // namespace

// Sort keys (and optional fp64 values), drop the sentinel tail, reduce duplicates
// (values summed), and emit a CSR.  Returns the unique count in *out_nnz.
int sort_unique_csr(uint64_t *keys, double *vals, int64_t nnz, int64_t n_coarse,
                    int64_t *out_indptr, int32_t *out_cols, double *out_vals, int64_t *out_nnz,
                    cudaStream_t st) {
    Scratch k2(st), v2(st), uk(st), uv(st), cnt(st), tmp(st);
    const int end_bit = 32 + bits_for((uint64_t)n_coarse);
    DRG_CUDA(k2.alloc(sizeof(uint64_t) * (size_t)nnz));
    if (vals) DRG_CUDA(v2.alloc(sizeof(double) * (size_t)nnz));
    size_t tb = 0;
    if (vals)
        cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, k2.as<uint64_t>(), vals,
                                        v2.as<double>(), nnz, 0, end_bit, st);
    else
        cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, k2.as<uint64_t>(), nnz, 0, end_bit, st);
    size_t tb2 = 0;
    DRG_CUDA(uk.alloc(sizeof(uint64_t) * (size_t)nnz));
    DRG_CUDA(cnt.alloc(sizeof(int64_t)));
    if (vals) {
        DRG_CUDA(uv.alloc(sizeof(double) * (size_t)nnz));
        cub::DeviceReduce::ReduceByKey(nullptr, tb2, k2.as<uint64_t>(), uk.as<uint64_t>(),
                                       v2.as<double>(), uv.as<double>(), cnt.as<int64_t>(),
                                       cuda::std::plus<double>{}, nnz, st);
    } else {
        cub::DeviceSelect::Unique(nullptr, tb2, k2.as<uint64_t>(), uk.as<uint64_t>(),
                                  cnt.as<int64_t>(), nnz, st);
    }
    DRG_CUDA(tmp.alloc(std::max(tb, tb2)));
    if (vals)
        DRG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys, k2.as<uint64_t>(), vals,
                                                 v2.as<double>(), nnz, 0, end_bit, st));
    else
        DRG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys, k2.as<uint64_t>(), nnz, 0,
                                                end_bit, st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (vals)
        DRG_CUDA(cub::DeviceReduce::ReduceByKey(tmp.p, tb2, k2.as<uint64_t>(), uk.as<uint64_t>(),
                                                v2.as<double>(), uv.as<double>(),
                                                cnt.as<int64_t>(), cuda::std::plus<double>{},
                                                nnz, st));
    else
        DRG_CUDA(cub::DeviceSelect::Unique(tmp.p, tb2, k2.as<uint64_t>(), uk.as<uint64_t>(),
                                           cnt.as<int64_t>(), nnz, st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    int64_t n_unique = 0;
    DRG_CUDA(cudaMemcpyAsync(&n_unique, cnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (n_unique > 0) {  // drop the sentinel (always the largest key)
        uint64_t last = 0;
        DRG_CUDA(cudaMemcpyAsync(&last, uk.as<uint64_t>() + n_unique - 1, sizeof(uint64_t),
                                 cudaMemcpyDeviceToHost, st));
        DRG_CUDA(cudaStreamSynchronize(st));
        if ((last >> 32) >= (uint64_t)n_coarse) n_unique--;
    }
    csr_from_keys_kernel<<<flat_grid(std::max<int64_t>(n_unique, n_coarse + 1)), 256, 0, st>>>(
        uk.as<uint64_t>(), n_unique, n_coarse, out_indptr, out_cols);
    DRG_LAUNCHED("csr_from_keys_kernel");
    if (vals && n_unique > 0)
        DRG_CUDA(cudaMemcpyAsync(out_vals, uv.p, sizeof(double) * (size_t)n_unique,
                                 cudaMemcpyDeviceToDevice, st));
    *out_nnz = n_unique;
    return DRG_OK;
}

}  // namespace drg

using namespace drg;

extern "C" int drg_coarsen(const int64_t *indptr, const int32_t *indices, int64_t n,
                           const int64_t *order, int32_t *out_parent, int64_t *out_n_coarse,
                           int32_t *out_rounds, void *stream) {
    if (n < 1) return fail(DRG_ERR_INVALID, "cannot coarsen an empty graph");
    if (n >= 0x7fffffffLL) return fail(DRG_ERR_INVALID, "node count exceeds int32");
    cudaStream_t st = as_stream(stream);
    Scratch rank(st), status(st), ctr(st), flag(st), ids(st), tmp(st);
    DRG_CUDA(rank.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(status.alloc((size_t)n));
    DRG_CUDA(ctr.alloc(16));
    DRG_CUDA(cudaMemsetAsync(status.p, 0, (size_t)n, st));
    DRG_CUDA(cudaMemsetAsync(ctr.p, 0, 16, st));
    int *d_bad = reinterpret_cast<int *>(ctr.as<char>() + 8);
    unsigned long long *d_und = ctr.as<unsigned long long>();
    rank_kernel<<<flat_grid(n), 256, 0, st>>>(order, n, rank.as<int32_t>(), d_bad);
    DRG_LAUNCHED("rank_kernel");
    const unsigned wg = (unsigned)std::min<int64_t>(ceil_div(n, kWpb), sm_count() * 64);
    int rounds = 0;
    for (;;) {
        DRG_CUDA(cudaMemsetAsync(d_und, 0, sizeof(unsigned long long), st));
        mis_round_kernel<<<wg, kWpb * 32, 0, st>>>(indptr, indices, n, rank.as<int32_t>(),
                                                   status.as<int8_t>(), d_und);
        DRG_LAUNCHED("mis_round_kernel");
        ++rounds;
        unsigned long long h[2] = {0, 0};
        DRG_CUDA(cudaMemcpyAsync(h, ctr.p, 16, cudaMemcpyDeviceToHost, st));
        DRG_CUDA(cudaStreamSynchronize(st));
        if ((int)(h[1] & 0xffffffffu)) return fail(DRG_ERR_INVALID, "order is not a permutation");
        if (h[0] == 0) break;
        if (rounds > 100000) return fail(DRG_ERR_CUDA, "MIS did not converge");
    }
    DRG_CUDA(flag.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(ids.alloc(sizeof(int32_t) * (size_t)(n + 1)));
    seed_flag_kernel<<<flat_grid(n), 256, 0, st>>>(order, n, status.as<int8_t>(),
                                                    flag.as<int32_t>());
    DRG_LAUNCHED("seed_flag_kernel");
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.as<int32_t>(), ids.as<int32_t>(), n, st);
    DRG_CUDA(tmp.alloc(tb));
    DRG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag.as<int32_t>(), ids.as<int32_t>(), n,
                                           st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    parent_kernel<<<wg, kWpb * 32, 0, st>>>(indptr, indices, n, rank.as<int32_t>(),
                                            status.as<int8_t>(), ids.as<int32_t>(), out_parent);
    DRG_LAUNCHED("parent_kernel");
    int32_t last_id = 0, last_flag = 0;
    DRG_CUDA(cudaMemcpyAsync(&last_id, ids.as<int32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaMemcpyAsync(&last_flag, flag.as<int32_t>() + n - 1, 4, cudaMemcpyDeviceToHost,
                             st));
    DRG_CUDA(cudaStreamSynchronize(st));
    *out_n_coarse = (int64_t)last_id + last_flag;
    if (out_rounds) *out_rounds = rounds;
    return DRG_OK;
}

extern "C" int drg_coarse_graph(const int64_t *indptr, const int32_t *indices, int64_t n,
                                const int32_t *parent, int64_t n_coarse, int64_t *out_indptr,
                                int32_t *out_indices, int64_t *out_nnz, void *stream) {
    if (n < 0 || n_coarse < 0) return fail(DRG_ERR_INVALID, "negative size");
    cudaStream_t st = as_stream(stream);
    int64_t nnz = 0;
    if (n > 0) {
        DRG_CUDA(cudaMemcpyAsync(&nnz, indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        DRG_CUDA(cudaStreamSynchronize(st));
    }
    if (nnz == 0) {
        DRG_CUDA(cudaMemsetAsync(out_indptr, 0, sizeof(int64_t) * (size_t)(n_coarse + 1), st));
        *out_nnz = 0;
        return DRG_OK;
    }
    Scratch keys(st);
    DRG_CUDA(keys.alloc(sizeof(uint64_t) * (size_t)nnz));
    const unsigned wg = (unsigned)std::min<int64_t>(ceil_div(n, kWpb), sm_count() * 64);
    pair_keys_kernel<double><<<wg, kWpb * 32, 0, st>>>(indptr, indices, nullptr, n, parent,
                                                       n_coarse, keys.as<uint64_t>(), nullptr);
    DRG_LAUNCHED("pair_keys_kernel");
    return sort_unique_csr(keys.as<uint64_t>(), nullptr, nnz, n_coarse, out_indptr, out_indices,
                           nullptr, out_nnz, st);
}

extern "C" int drg_compose_maps(const int32_t *first, const int32_t *second, int64_t n,
                                int32_t *out, void *stream) {
    if (n <= 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    if (!first) {
        iota_kernel<<<flat_grid(n), 256, 0, st>>>(out, n);
        DRG_LAUNCHED("iota_kernel");
        return DRG_OK;
    }
    compose_kernel<<<flat_grid(n), 256, 0, st>>>(first, second, n, out);
    DRG_LAUNCHED("compose_kernel");
    return DRG_OK;
}

extern "C" int drg_aggregate_pairs(const int64_t *indptr, const int32_t *targets,
                                   const double *weights, int64_t n, int64_t nnz,
                                   const int32_t *parent, int64_t n_coarse, int64_t *out_indptr,
                                   int32_t *out_targets, double *out_weights, int64_t *out_nnz,
                                   void *stream) {
    if (n < 0 || nnz < 0 || n_coarse < 0) return fail(DRG_ERR_INVALID, "negative size");
    cudaStream_t st = as_stream(stream);
    if (nnz == 0) {
        DRG_CUDA(cudaMemsetAsync(out_indptr, 0, sizeof(int64_t) * (size_t)(n_coarse + 1), st));
        *out_nnz = 0;
        return DRG_OK;
    }
    Scratch keys(st), vals(st);
    DRG_CUDA(keys.alloc(sizeof(uint64_t) * (size_t)nnz));
    DRG_CUDA(vals.alloc(sizeof(double) * (size_t)nnz));
    const unsigned wg = (unsigned)std::min<int64_t>(ceil_div(n, kWpb), sm_count() * 64);
    pair_keys_kernel<double><<<wg, kWpb * 32, 0, st>>>(indptr, targets, weights, n, parent,
                                                       n_coarse, keys.as<uint64_t>(),
                                                       vals.as<double>());
    DRG_LAUNCHED("pair_keys_kernel");
    return sort_unique_csr(keys.as<uint64_t>(), vals.as<double>(), nnz, n_coarse, out_indptr,
                           out_targets, out_weights, out_nnz, st);
}

extern "C" int drg_aggregate_nodes(const double *values, const int32_t *parent, int64_t n,
                                   int64_t n_coarse, double *out, void *stream) {
    if (n <= 0 || n_coarse <= 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    Scratch k2(st), v2(st), uk(st), cnt(st), tmp(st);
    DRG_CUDA(k2.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(v2.alloc(sizeof(double) * (size_t)n));
    DRG_CUDA(uk.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(cnt.alloc(sizeof(int64_t)));
    const int end_bit = bits_for((uint64_t)n_coarse);
    size_t tb = 0, tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, parent, k2.as<int32_t>(), values,
                                    v2.as<double>(), n, 0, std::max(end_bit, 1), st);
    cub::DeviceReduce::ReduceByKey(nullptr, tb2, k2.as<int32_t>(), uk.as<int32_t>(),
                                   v2.as<double>(), out, cnt.as<int64_t>(),
                                   cuda::std::plus<double>{}, n, st);
    DRG_CUDA(tmp.alloc(std::max(tb, tb2)));
    DRG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, parent, k2.as<int32_t>(), values,
                                             v2.as<double>(), n, 0, std::max(end_bit, 1), st));
    DRG_CUDA(cub::DeviceReduce::ReduceByKey(tmp.p, tb2, k2.as<int32_t>(), uk.as<int32_t>(),
                                            v2.as<double>(), out, cnt.as<int64_t>(),
                                            cuda::std::plus<double>{}, n, st));
    g_launches.fetch_add(2, std::memory_order_relaxed);
    return DRG_OK;
}

extern "C" int drg_from_edges(const int64_t *pairs, int64_t m, int64_t n, int64_t *out_indptr,
                              int32_t *out_indices, int64_t *out_nnz, void *stream) {
    if (m < 0 || n < 0 || n >= 0x7fffffffLL) return fail(DRG_ERR_INVALID, "bad sizes");
    cudaStream_t st = as_stream(stream);
    if (m == 0) {
        DRG_CUDA(cudaMemsetAsync(out_indptr, 0, sizeof(int64_t) * (size_t)(n + 1), st));
        *out_nnz = 0;
        return DRG_OK;
    }
    Scratch keys(st), bad(st);
    DRG_CUDA(keys.alloc(sizeof(uint64_t) * (size_t)(2 * m)));
    DRG_CUDA(bad.alloc(sizeof(int)));
    DRG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    edge_keys_kernel<<<flat_grid(m), 256, 0, st>>>(pairs, m, n, keys.as<uint64_t>(), bad.as<int>());
    DRG_LAUNCHED("edge_keys_kernel");
    int h_bad = 0;
    DRG_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (h_bad) return fail(DRG_ERR_INVALID, "node id outside [0, %lld)", (long long)n);
    return sort_unique_csr(keys.as<uint64_t>(), nullptr, 2 * m, n, out_indptr, out_indices,
                           nullptr, out_nnz, st);
}
