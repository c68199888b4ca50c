// K2 + K3: Gaussian similarity over k-hop rows (replaces build_sparse_similarity,
// similarity.py:216-278).
//
//  hist_kernel   warp per row: per-distance multiplicities c_i(d) (rows are
//                (dist,id)-sorted, so the row's entropy only depends on them),
//                non-isolated count, max distance.
//  sigma_kernel  thread per row, fp64: the reference's geometric bisection
//                (search_sigma, similarity.py:167-199) over <= 6 histogram bins
//                with _row_perplexity's shift-stabilised entropy (148-164); then the
//                unshifted conditional table p_{j|i} = table_i[d] / Z_i with the
//                underflow fallback (122-145).  Stored per node and distance:
//                pcond[i*k + d-1].
//  symm_kernel   warp per row: P_ij = (pcond[i][d_ij] + pcond[j][d_ij]) / (2 N_ne).
//                BFS distances are symmetric (d_ij = d_ji), so the mirror value is a
//                gather from the L2-resident pcond table -- no transpose, no sort,
//                and the two stored entries are bitwise equal (a+b == b+a).  The
//                warp reduction of the row gives row_mass (similarity.py:84-91).
#include <cub/cub.cuh>

#include "common.cuh"

namespace drg {
namespace {

constexpr int kMaxK = 6;
constexpr int kWpb = 8;

__global__ void __launch_bounds__(kWpb * 32)
    hist_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ dists, int64_t n,
                int k, int32_t *__restrict__ hist, int *max_dist,
                unsigned long long *n_nonisolated) {
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = (int64_t)blockIdx.x * kWpb + (threadIdx.x >> 5);
    int local_max = 0;
    unsigned long long local_ne = 0;
    for (int64_t i = warp0; i < n; i += (int64_t)gridDim.x * kWpb) {
        const int64_t lo = indptr[i], hi = indptr[i + 1];
        int c[kMaxK];
#pragma unroll
        for (int d = 0; d < kMaxK; ++d) c[d] = 0;
        for (int64_t e = lo + lane; e < hi; e += 32) {
            int d = __ldg(dists + e);
#pragma unroll
            for (int q = 0; q < kMaxK; ++q) c[q] += (d == q + 1);
            local_max = max(local_max, d);
        }
#pragma unroll
        for (int q = 0; q < kMaxK; ++q) {
            int v = c[q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane == 0 && q < k) hist[i * k + q] = v;
        }
        if (lane == 0 && hi > lo) local_ne++;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local_max = max(local_max, __shfl_xor_sync(kFull, local_max, o));
    if (lane == 0) {
        if (local_max) atomicMax(max_dist, local_max);
        if (local_ne) atomicAdd(n_nonisolated, local_ne);
    }
}

// 2**H of a row from its histogram (similarity.py:148-164).
__device__ double row_perplexity(const double *cnt, const double *dval, int nb, double sigma) {
    const double inv = 1.0 / (2.0 * sigma * sigma);
    double expo[kMaxK], vals[kMaxK];
    double mx = -INFINITY;
    for (int b = 0; b < nb; ++b) {
        expo[b] = -(dval[b] * dval[b]) * inv;
        mx = fmax(mx, expo[b]);
    }
    double total = 0.0;
    for (int b = 0; b < nb; ++b) {
        vals[b] = exp(expo[b] - mx);
        total += cnt[b] * vals[b];
    }
    double h = 0.0;
    for (int b = 0; b < nb; ++b) {
        double p = vals[b] / total;
        h += cnt[b] * (p > 0.0 ? p * log2(p) : 0.0);
    }
    return exp2(-h);
}

__global__ void sigma_kernel(const int32_t *__restrict__ hist, int64_t n, int k, int uniform,
                             double perplexity, double tol, int max_iter, double smin,
                             double smax, double *__restrict__ sigma_out,
                             double *__restrict__ pcond) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int h[kMaxK];
        int64_t n_row = 0;
        for (int d = 0; d < k; ++d) {
            h[d] = hist[i * k + d];
            n_row += h[d];
        }
        double *pc = pcond + i * k;
        for (int d = 0; d < k; ++d) pc[d] = 0.0;
        sigma_out[i] = 1.0;
        if (n_row == 0) continue;
        if (uniform) {  // closed form, similarity.py:202-213 (inv = 1/deg)
            pc[0] = 1.0 / (double)n_row;
            continue;
        }
        double cnt[kMaxK], dval[kMaxK];
        int nb = 0;
        for (int d = 0; d < k; ++d)
            if (h[d] > 0) {
                cnt[nb] = (double)h[d];
                dval[nb] = (double)(d + 1);
                nb++;
            }
        // target: "auto" = min(row size, max(degree, 1)) (similarity.py:253-256), clamped
        // to [1, row size] inside search_sigma (similarity.py:181)
        double target;
        if (perplexity <= 0.0) {
            int64_t deg = h[0] > 1 ? h[0] : 1;
            target = (double)(n_row < deg ? n_row : deg);
        } else {
            target = perplexity;
        }
        double s = 1.0;
        if (n_row > 1) {
            target = fmin(fmax(target, 1.0), (double)n_row);
            double lo = smin, hi = smax, best_err = INFINITY;
            for (int it = 0; it < max_iter; ++it) {
                const double mid = sqrt(lo * hi);
                const double perp = row_perplexity(cnt, dval, nb, mid);
                const double err = fabs(perp - target);
                if (err < best_err) {
                    best_err = err;
                    s = mid;
                }
                if (err <= tol) break;
                if (perp > target) hi = mid;
                else lo = mid;
            }
        }
        sigma_out[i] = s;
        // conditional row (similarity.py:122-145): unshifted Gaussian table
        const double inv = 1.0 / (2.0 * s * s);
        const int dmax = (int)dval[nb - 1];
        double table[kMaxK];
        double Z = 0.0;
        for (int d = 1; d <= dmax; ++d) {
            table[d - 1] = exp((double)(-(d * d)) * inv);
            Z += (double)h[d - 1] * table[d - 1];
        }
        if (Z == 0.0) {  // vanishing bandwidth: uniform over the nearest entries
            const int dmin = (int)dval[0];
            pc[dmin - 1] = 1.0 / (double)h[dmin - 1];
        } else {
            for (int d = 0; d < dmax; ++d) pc[d] = h[d] > 0 ? table[d] / Z : 0.0;
        }
    }
}

__global__ void __launch_bounds__(kWpb * 32)
    symm_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ ids,
                const int32_t *__restrict__ dists, int64_t n, int k,
                const double *__restrict__ pcond, double denom, double *__restrict__ weights,
                double *__restrict__ row_mass) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * kWpb + (threadIdx.x >> 5); i < n;
         i += (int64_t)gridDim.x * kWpb) {
        const int64_t lo = indptr[i], hi = indptr[i + 1];
        const double *pi = pcond + i * k;
        double acc = 0.0;
        for (int64_t e = lo + lane; e < hi; e += 32) {
            const int j = __ldg(ids + e);
            const int d = __ldg(dists + e) - 1;
            const double w = (pi[d] + __ldg(pcond + (int64_t)j * k + d)) / denom;
            weights[e] = w;
            acc += w;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (lane == 0) row_mass[i] = acc;
    }
}

// Last (dist, id) key of every row: membership of i in a capped row j is then
// key(d_ij, i) <= lastkey[j] (rows are (dist,id)-sorted prefixes of the ball).
__global__ void lastkey_kernel(const int64_t *__restrict__ indptr,
                               const int32_t *__restrict__ ids,
                               const int32_t *__restrict__ dists, int64_t n,
                               uint32_t *lastkey) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = indptr[i], hi = indptr[i + 1];
        lastkey[i] = hi > lo ? (((uint32_t)dists[hi - 1] << 29) | (uint32_t)ids[hi - 1]) : 0u;
    }
}

// Union symmetrisation of capped rows (BASELINE C3; the reference itself
// mis-symmetrises capped rows): every stored (i, j, d) emits
// key (i, j) with P = (p_{j|i} + [i in row j] p_{i|j}) / (2 N_ne); when i is not in
// j's capped row it also emits the missing mirror (j, i) with the same value.
__global__ void __launch_bounds__(kWpb * 32)
    union_emit_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ ids,
                      const int32_t *__restrict__ dists, int64_t n, int k,
                      const double *__restrict__ pcond, const uint32_t *__restrict__ lastkey,
                      double denom, uint64_t *keys, double *vals) {
    const int lane = threadIdx.x & 31;
    const uint64_t sentinel = (uint64_t)n << 32;
    for (int64_t i = (int64_t)blockIdx.x * kWpb + (threadIdx.x >> 5); i < n;
         i += (int64_t)gridDim.x * kWpb) {
        const int64_t lo = indptr[i], hi = indptr[i + 1];
        const double *pi = pcond + i * k;
        for (int64_t e = lo + lane; e < hi; e += 32) {
            const int j = __ldg(ids + e);
            const int d = __ldg(dists + e);
            const bool mirror = (((uint32_t)d << 29) | (uint32_t)i) <= __ldg(lastkey + j);
            const double w =
                (pi[d - 1] + (mirror ? __ldg(pcond + (int64_t)j * k + d - 1) : 0.0)) / denom;
            keys[2 * e] = ((uint64_t)i << 32) | (uint32_t)j;
            vals[2 * e] = w;
            keys[2 * e + 1] = mirror ? sentinel : (((uint64_t)j << 32) | (uint32_t)i);
            vals[2 * e + 1] = w;
        }
    }
}

__global__ void __launch_bounds__(kWpb * 32)
    row_sum_kernel(const int64_t *__restrict__ indptr, const double *__restrict__ w, int64_t n,
                   double *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * kWpb + (threadIdx.x >> 5); i < n;
         i += (int64_t)gridDim.x * kWpb) {
        double acc = 0.0;
        for (int64_t e = indptr[i] + lane; e < indptr[i + 1]; e += 32) acc += w[e];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (lane == 0) out[i] = acc;
    }
}

}  // namespace
}  // namespace drg

using namespace drg;

extern "C" int drg_similarity_union(const int64_t *nd_indptr, const int32_t *nd_ids,
                                    const int32_t *nd_dists, int64_t n, int64_t nnz, int k,
                                    double perplexity, double tol, int max_iter,
                                    double sigma_min, double sigma_max, double *out_sigma,
                                    int64_t *out_indptr, int32_t *out_targets,
                                    double *out_weights, double *out_row_mass, int64_t *out_nnz,
                                    double *out_total_mass, int64_t *out_n_nonisolated,
                                    void *stream) {
    if (k < 1 || k > kMaxK) return fail(DRG_ERR_INVALID, "k must be in [1, 6], got %d", k);
    if (n < 0 || nnz < 0 || n >= (1LL << 29)) return fail(DRG_ERR_INVALID, "bad sizes");
    if (perplexity > 0.0 && perplexity < 1.0)
        return fail(DRG_ERR_INVALID, "perplexity must be >= 1 or 'auto'");
    if (!(sigma_min > 0.0) || !(sigma_max > sigma_min))
        return fail(DRG_ERR_INVALID, "need 0 < sigma_min < sigma_max");
    cudaStream_t st = as_stream(stream);
    *out_nnz = 0;
    if (out_total_mass) *out_total_mass = 0.0;
    if (out_n_nonisolated) *out_n_nonisolated = 0;
    if (n == 0) return DRG_OK;
    Scratch hist(st), pcond(st), flags(st), lastkey(st), keys(st), vals(st), tmp(st), total(st);
    DRG_CUDA(hist.alloc(sizeof(int32_t) * (size_t)n * k));
    DRG_CUDA(pcond.alloc(sizeof(double) * (size_t)n * k));
    DRG_CUDA(flags.alloc(16));
    DRG_CUDA(cudaMemsetAsync(flags.p, 0, 16, st));
    int *d_maxd = flags.as<int>();
    unsigned long long *d_ne = reinterpret_cast<unsigned long long *>(flags.as<char>() + 8);
    const unsigned wg = (unsigned)std::min<int64_t>(ceil_div(n, kWpb), sm_count() * 64);
    hist_kernel<<<wg, kWpb * 32, 0, st>>>(nd_indptr, nd_dists, n, k, hist.as<int32_t>(), d_maxd,
                                          d_ne);
    DRG_LAUNCHED("hist_kernel");
    int h_flags[4] = {0, 0, 0, 0};
    DRG_CUDA(cudaMemcpyAsync(h_flags, flags.p, 16, cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    unsigned long long n_ne = 0;
    memcpy(&n_ne, &h_flags[2], sizeof(n_ne));
    if (out_n_nonisolated) *out_n_nonisolated = (int64_t)n_ne;
    const int uniform = (k == 1 || h_flags[0] <= 1) ? 1 : 0;
    sigma_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 128), sm_count() * 64), 128, 0, st>>>(
        hist.as<int32_t>(), n, k, uniform, perplexity, tol, max_iter, sigma_min, sigma_max,
        out_sigma, pcond.as<double>());
    DRG_LAUNCHED("sigma_kernel");
    if (nnz == 0) {
        DRG_CUDA(cudaMemsetAsync(out_indptr, 0, sizeof(int64_t) * (size_t)(n + 1), st));
        DRG_CUDA(cudaMemsetAsync(out_row_mass, 0, sizeof(double) * (size_t)n, st));
        return DRG_OK;
    }
    DRG_CUDA(lastkey.alloc(sizeof(uint32_t) * (size_t)n));
    lastkey_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), sm_count() * 32), 256, 0, st>>>(
        nd_indptr, nd_ids, nd_dists, n, lastkey.as<uint32_t>());
    DRG_LAUNCHED("lastkey_kernel");
    DRG_CUDA(keys.alloc(sizeof(uint64_t) * (size_t)(2 * nnz)));
    DRG_CUDA(vals.alloc(sizeof(double) * (size_t)(2 * nnz)));
    const double denom = 2.0 * (double)(n_ne > 0 ? n_ne : 1);
    union_emit_kernel<<<wg, kWpb * 32, 0, st>>>(nd_indptr, nd_ids, nd_dists, n, k,
                                                pcond.as<double>(), lastkey.as<uint32_t>(), denom,
                                                keys.as<uint64_t>(), vals.as<double>());
    DRG_LAUNCHED("union_emit_kernel");
    DRG_TRY(sort_unique_csr(keys.as<uint64_t>(), vals.as<double>(), 2 * nnz, n, out_indptr,
                            out_targets, out_weights, out_nnz, st));
    row_sum_kernel<<<wg, kWpb * 32, 0, st>>>(out_indptr, out_weights, n, out_row_mass);
    DRG_LAUNCHED("row_sum_kernel");
    size_t tb = 0;
    DRG_CUDA(total.alloc(sizeof(double)));
    cub::DeviceReduce::Sum(nullptr, tb, out_row_mass, total.as<double>(), n, st);
    DRG_CUDA(tmp.alloc(tb));
    DRG_CUDA(cub::DeviceReduce::Sum(tmp.p, tb, out_row_mass, total.as<double>(), n, st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    double h_total = 0.0;
    DRG_CUDA(cudaMemcpyAsync(&h_total, total.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (out_total_mass) *out_total_mass = h_total;
    return DRG_OK;
}

extern "C" int drg_similarity(const int64_t *nd_indptr, const int32_t *nd_ids,
                              const int32_t *nd_dists, int64_t n, int64_t nnz, int k,
                              double perplexity, double tol, int max_iter, double sigma_min,
                              double sigma_max, double *out_sigma, double *out_weights,
                              double *out_row_mass, double *out_total_mass,
                              int64_t *out_n_nonisolated, void *stream) {
    if (k < 1 || k > kMaxK) return fail(DRG_ERR_INVALID, "k must be in [1, 6], got %d", k);
    if (n < 0 || nnz < 0) return fail(DRG_ERR_INVALID, "negative size");
    if (perplexity > 0.0 && perplexity < 1.0)
        return fail(DRG_ERR_INVALID, "perplexity must be >= 1 or 'auto'");
    if (!(sigma_min > 0.0) || !(sigma_max > sigma_min))
        return fail(DRG_ERR_INVALID, "need 0 < sigma_min < sigma_max");
    cudaStream_t st = as_stream(stream);
    if (out_total_mass) *out_total_mass = 0.0;
    if (out_n_nonisolated) *out_n_nonisolated = 0;
    if (n == 0) return DRG_OK;
    Scratch hist(st), pcond(st), flags(st), tmp(st), total(st);
    DRG_CUDA(hist.alloc(sizeof(int32_t) * (size_t)n * k));
    DRG_CUDA(pcond.alloc(sizeof(double) * (size_t)n * k));
    DRG_CUDA(flags.alloc(16));
    DRG_CUDA(cudaMemsetAsync(flags.p, 0, 16, st));
    int *d_maxd = flags.as<int>();
    unsigned long long *d_ne = reinterpret_cast<unsigned long long *>(flags.as<char>() + 8);
    const unsigned wg = (unsigned)std::min<int64_t>(ceil_div(n, kWpb), sm_count() * 64);
    hist_kernel<<<wg, kWpb * 32, 0, st>>>(nd_indptr, nd_dists, n, k, hist.as<int32_t>(), d_maxd,
                                          d_ne);
    DRG_LAUNCHED("hist_kernel");
    int h_flags[4] = {0, 0, 0, 0};
    DRG_CUDA(cudaMemcpyAsync(h_flags, flags.p, 16, cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    const int maxd = h_flags[0];
    unsigned long long n_ne = 0;
    memcpy(&n_ne, &h_flags[2], sizeof(n_ne));
    if (out_n_nonisolated) *out_n_nonisolated = (int64_t)n_ne;
    const int uniform = (k == 1 || maxd <= 1) ? 1 : 0;  // similarity.py:236-237
    sigma_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 128), sm_count() * 64), 128, 0, st>>>(
        hist.as<int32_t>(), n, k, uniform, perplexity, tol, max_iter, sigma_min, sigma_max,
        out_sigma, pcond.as<double>());
    DRG_LAUNCHED("sigma_kernel");
    if (nnz == 0) {
        DRG_CUDA(cudaMemsetAsync(out_row_mass, 0, sizeof(double) * (size_t)n, st));
        return DRG_OK;
    }
    const double denom = 2.0 * (double)(n_ne > 0 ? n_ne : 1);
    symm_kernel<<<wg, kWpb * 32, 0, st>>>(nd_indptr, nd_ids, nd_dists, n, k, pcond.as<double>(),
                                          denom, out_weights, out_row_mass);
    DRG_LAUNCHED("symm_kernel");
    size_t tb = 0;
    DRG_CUDA(total.alloc(sizeof(double)));
    cub::DeviceReduce::Sum(nullptr, tb, out_row_mass, total.as<double>(), n, st);
    DRG_CUDA(tmp.alloc(tb));
    DRG_CUDA(cub::DeviceReduce::Sum(tmp.p, tb, out_row_mass, total.as<double>(), n, st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    double h_total = 0.0;
    DRG_CUDA(cudaMemcpyAsync(&h_total, total.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (out_total_mass) *out_total_mass = h_total;
    return DRG_OK;
}
