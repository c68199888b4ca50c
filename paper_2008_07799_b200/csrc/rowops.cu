// Per-row and per-interaction drop-ins of the reference's public helpers, on the
// device (the package has no CPU path):
//
//  drg_gaussian_table   precompute_gaussian_table (similarity.py:110-119)
//  drg_rows_sigma       search_sigma (similarity.py:167-199) over _row_perplexity
//                       (148-164), one thread per row
//  drg_rows_conditional conditional_similarity_row (similarity.py:122-145): unshifted
//                       table, fsum-normalised, underflow -> uniform over the nearest
//  drg_gradients        attractive_gradient / repulsive_gradient (optimizer.py:174-203)
//
// exp is evaluated in double-double and rounded once (exp_cr), and the row sum is
// Shewchuk's exact summation rounded like math.fsum, so a conditional row is the
// reference's value bit for bit (its own test compares them with ==).
#include <math.h>

#include <algorithm>
#include <climits>

#include "common.cuh"

namespace drg {
namespace {

// ---- double-double helpers -------------------------------------------------
struct dd {
    double h, l;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}

__device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}

__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.h, b.h);
    s.l = __dadd_rn(s.l, __dadd_rn(a.l, b.l));
    return two_sum(s.h, s.l);
}

__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.h, b.h);
    p.l = __fma_rn(a.h, b.l, __fma_rn(a.l, b.h, p.l));
    return two_sum(p.h, p.l);
}

// exp(x) to ~100 bits, rounded once: x = k ln2 + r (ln2 in three parts, r as a
// double-double), exp(r) by its Taylor series in double-double (|r| <= 0.35: 27
// terms reach 2^-110), then 2^k.
__device__ double exp_cr(double x) {
    if (x != x) return x;
    if (x > 709.8) return INFINITY;
    if (x < -745.2) return 0.0;
    const double ln2_hi = 6.93147180369123816490e-01;   // 0x3fe62e42fee00000: 32 bits
    const double ln2_mid = 1.9082149292705877e-10;      // ln2 - ln2_hi, rounded
    const double ln2_lo = 1.1612227229362532e-26;       // the remainder
    const double kd = rint(x * 1.44269504088896338700e+00);
    const int k = (int)kd;
    // r = x - k ln2 (k ln2_hi is exact: ln2_hi has 32 significant bits)
    dd r = two_sum(x, -kd * ln2_hi);
    r = dd_add(r, two_prod(-kd, ln2_mid));
    r = dd_add(r, two_prod(-kd, ln2_lo));
    // Taylor series, Horner from the top in double-double
    dd acc = {1.0, 0.0};
    for (int i = 27; i >= 1; --i) {
        acc = dd_mul(acc, r);
        // acc = 1 + acc / i
        const double q = acc.h / (double)i;
        dd qi = two_prod(q, (double)i);
        const double rem = ((acc.h - qi.h) - qi.l + acc.l) / (double)i;
        acc = dd_add({1.0, 0.0}, two_sum(q, rem));
    }
    const double m = __dadd_rn(acc.h, acc.l);
    if (k > -1000) return ldexp(m, k);
    // deep subnormal range: scale in two steps from the double-double value
    return ldexp(__dadd_rn(ldexp(acc.h, 60), ldexp(acc.l, 60)), k - 60);
}

// ---- math.fsum: Shewchuk partials, correctly rounded (Python's msum) ---------
constexpr int kMaxPartials = 64;

struct FSum {
    double p[kMaxPartials];
    int n = 0;
    bool ok = true;
    __device__ void add(double x) {
        int i = 0;
        for (int j = 0; j < n; ++j) {
            double y = p[j];
            if (fabs(x) < fabs(y)) {
                const double t = x;
                x = y;
                y = t;
            }
            const double hi = __dadd_rn(x, y);
            const double lo = __dsub_rn(y, __dsub_rn(hi, x));
            if (lo != 0.0) p[i++] = lo;
            x = hi;
        }
        if (i >= kMaxPartials) {
            ok = false;
            return;
        }
        p[i++] = x;
        n = i;
    }
    __device__ double result() const {
        if (n == 0) return 0.0;
        int i = n - 1;
        double hi = p[i], lo = 0.0;
        while (i > 0) {
            const double x = hi;
            const double y = p[--i];
            hi = __dadd_rn(x, y);
            const double yr = __dsub_rn(hi, x);
            lo = __dsub_rn(y, yr);
            if (lo != 0.0) break;
        }
        // half-way case: make the rounding of hi + lo agree with the exact sum
        if (i > 0 && ((lo < 0.0 && p[i - 1] < 0.0) || (lo > 0.0 && p[i - 1] > 0.0))) {
            const double y = lo * 2.0;
            const double x = __dadd_rn(hi, y);
            const double yr = __dsub_rn(x, hi);
            if (y == yr) hi = x;
        }
        return hi;
    }
};

// table value of distance d at bandwidth sigma, exactly as the reference computes it
__device__ __forceinline__ double gauss(int d, double inv) {
    return exp_cr(__dmul_rn((double)(-(d * d)), inv));
}

__global__ void gaussian_table_kernel(int k, double sigma, double *out) {
    const double inv = 1.0 / (2.0 * sigma * sigma);
    for (int d = 1 + (int)threadIdx.x; d <= k; d += blockDim.x) out[d - 1] = gauss(d, inv);
}

constexpr int kMaxBins = 64;   // distinct distances of one row (rows hold d <= k <= 6)

// 2**H of a row from its distinct distances and multiplicities (similarity.py:148-164)
__device__ double row_perp(const double *cnt, const double *dv, int nb, double sigma) {
    const double inv = 1.0 / (2.0 * sigma * sigma);
    double mx = -INFINITY;
    for (int b = 0; b < nb; ++b) mx = fmax(mx, -(dv[b] * dv[b]) * inv);
    double total = 0.0;
    for (int b = 0; b < nb; ++b) total += cnt[b] * exp(-(dv[b] * dv[b]) * inv - mx);
    double h = 0.0;
    for (int b = 0; b < nb; ++b) {
        const double p = exp(-(dv[b] * dv[b]) * inv - mx) / total;
        h += cnt[b] * (p > 0.0 ? p * log2(p) : 0.0);
    }
    return exp2(-h);
}

__global__ void rows_sigma_kernel(const int64_t *__restrict__ indptr,
                                  const int32_t *__restrict__ dists, int64_t nrows,
                                  double perplexity, double tol, int max_iter, double smin,
                                  double smax, double *sigma, int *bad) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = indptr[r], hi = indptr[r + 1], len = hi - lo;
        if (len == 0) continue;
        if (len == 1) {
            sigma[r] = 1.0;
            continue;
        }
        // np.unique: distinct distances in increasing order with their counts
        double dv[kMaxBins], cnt[kMaxBins];
        int nb = 0;
        int prev = INT_MIN;
        while (true) {
            int nxt = INT_MAX, c = 0;
            for (int64_t e = lo; e < hi; ++e) {
                const int d = dists[e];
                if (d > prev && d < nxt) {
                    nxt = d;
                    c = 1;
                } else if (d == nxt) {
                    ++c;
                }
            }
            if (nxt == INT_MAX) break;
            if (nb == kMaxBins) {
                atomicExch(bad, 1);
                break;
            }
            dv[nb] = (double)nxt;
            cnt[nb] = (double)c;
            ++nb;
            prev = nxt;
        }
        const double target = fmin(fmax(perplexity, 1.0), (double)len);
        double lo_s = smin, hi_s = smax, best = 1.0, best_err = INFINITY;
        for (int it = 0; it < max_iter; ++it) {
            const double mid = sqrt(lo_s * hi_s);
            const double perp = row_perp(cnt, dv, nb, mid);
            const double err = fabs(perp - target);
            if (err < best_err) {
                best_err = err;
                best = mid;
            }
            if (err <= tol) break;
            if (perp > target) hi_s = mid;
            else lo_s = mid;
        }
        sigma[r] = best;
    }
}

__global__ void rows_conditional_kernel(const int64_t *__restrict__ indptr,
                                        const int32_t *__restrict__ dists, int64_t nrows,
                                        const double *__restrict__ sigma, double *p, int *bad) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = indptr[r], hi = indptr[r + 1];
        if (hi == lo) continue;
        const double s = sigma[r];
        const double inv = 1.0 / (2.0 * s * s);
        FSum acc;
        int dmin = INT_MAX;
        for (int64_t e = lo; e < hi; ++e) {
            const int d = dists[e];
            acc.add(gauss(d, inv));
            dmin = min(dmin, d);
        }
        if (!acc.ok) atomicExch(bad, 1);
        const double total = acc.result();
        if (total == 0.0) {   // every kernel value underflowed: uniform over the nearest
            int64_t nn = 0;
            for (int64_t e = lo; e < hi; ++e) nn += dists[e] == dmin;
            const double q = 1.0 / (double)nn;
            for (int64_t e = lo; e < hi; ++e) p[e] = dists[e] == dmin ? q : 0.0;
        } else {
            for (int64_t e = lo; e < hi; ++e) p[e] = gauss(dists[e], inv) / total;
        }
    }
}

// attractive (kind 0, optimizer.py:174-186, no clip) or repulsive (kind 1, 189-203)
__global__ void gradients_kernel(const double *__restrict__ yi, const double *__restrict__ yj,
                                 int64_t n, int b, double gamma, double eps, double clip, int kind,
                                 double *out) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const double dx = yi[2 * q] - yj[2 * q], dy = yi[2 * q + 1] - yj[2 * q + 1];
        const double ld2 = dx * dx + dy * dy;
        double gx = 0.0, gy = 0.0;
        double pw = 1.0;
        for (int i = 0; i < b - 1; ++i) pw *= ld2;
        if (kind == 0) {
            if (ld2 != 0.0) {
                const double coef = -2.0 * (double)b * pw / (1.0 + pw * ld2);
                gx = coef * dx;
                gy = coef * dy;
            }
        } else if (ld2 + eps > 0.0) {
            const double coef = gamma * 2.0 * (double)b / ((ld2 + eps) * (1.0 + pw * ld2));
            gx = fmin(fmax(coef * dx, -clip), clip);
            gy = fmin(fmax(coef * dy, -clip), clip);
        }
        out[2 * q] = gx;
        out[2 * q + 1] = gy;
    }
}

unsigned grid_for(int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 128), sm_count() * 16));
}

}  // namespace
}  // namespace drg

using namespace drg;

extern "C" int drg_gaussian_table(int k, double sigma, double *out, void *stream) {
    if (k < 1) return fail(DRG_ERR_INVALID, "k must be >= 1");
    gaussian_table_kernel<<<1, 128, 0, as_stream(stream)>>>(k, sigma, out);
    DRG_LAUNCHED("gaussian_table_kernel");
    return DRG_OK;
}

extern "C" int drg_rows_sigma(const int64_t *indptr, const int32_t *dists, int64_t nrows,
                              double perplexity, double tol, int max_iter, double sigma_min,
                              double sigma_max, double *out_sigma, void *stream) {
    if (nrows <= 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    Scratch bad(st);
    DRG_CUDA(bad.alloc(sizeof(int)));
    DRG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    rows_sigma_kernel<<<grid_for(nrows), 128, 0, st>>>(indptr, dists, nrows, perplexity, tol,
                                                       max_iter, sigma_min, sigma_max, out_sigma,
                                                       bad.as<int>());
    DRG_LAUNCHED("rows_sigma_kernel");
    int h = 0;
    DRG_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (h) return fail(DRG_ERR_UNSUPPORTED, "a row holds more than %d distinct distances", kMaxBins);
    return DRG_OK;
}

extern "C" int drg_rows_conditional(const int64_t *indptr, const int32_t *dists, int64_t nrows,
                                    const double *sigma, double *out_p, void *stream) {
    if (nrows <= 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    Scratch bad(st);
    DRG_CUDA(bad.alloc(sizeof(int)));
    DRG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    rows_conditional_kernel<<<grid_for(nrows), 128, 0, st>>>(indptr, dists, nrows, sigma, out_p,
                                                             bad.as<int>());
    DRG_LAUNCHED("rows_conditional_kernel");
    int h = 0;
    DRG_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (h) return fail(DRG_ERR_UNSUPPORTED, "row sum needs more than %d partials", kMaxPartials);
    return DRG_OK;
}

extern "C" int drg_gradients(const double *yi, const double *yj, int64_t n, int b, double gamma,
                             double eps, double clip, int kind, double *out, void *stream) {
    if (n <= 0) return DRG_OK;
    if (b < 1) return fail(DRG_ERR_INVALID, "b must be >= 1");
    gradients_kernel<<<grid_for(n), 128, 0, as_stream(stream)>>>(yi, yj, n, b, gamma, eps, clip,
                                                                 kind, out);
    DRG_LAUNCHED("gradients_kernel");
    return DRG_OK;
}
