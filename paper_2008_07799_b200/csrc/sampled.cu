// Reference-faithful sampled epochs (update="sampled").
//
// K7 (layout.cu) applies one epoch's EXPECTED displacement with a CSR gather.  This
// kernel instead replays the reference step itself (_kernels.py:65-140), Hogwild
// style like sgd_epoch with threads > 1 (optimizer.py:325-345): every thread runs
// steps s of the epoch; a step draws a directed pair (i0, j0) ~ P at level 0 (the
// source by a Vose table over the row masses, then the target by binary search in
// the row's cumulative weights -- the same law as the reference's canonical-pair
// table plus direction coin, optimizer.py:206-229), maps both ends to the current
// level, applies the clipped attractive update to both ends if they differ, then M
// negatives ~ Q at level 0, mapped and redrawn (<= 9 attempts) while they hit i or
// j, each moving both ends.  Updates are float2 atomic adds on y; the source
// position is tracked locally through the step as in the sequential kernel.
#include "common.cuh"

namespace drg {
namespace {

struct SArgs {
    const int64_t *indptr0;
    const int32_t *targets0;
    const float *cum0;
    const uint2 *src_alias;
    const uint2 *neg_alias;
    int64_t n0;
    const int32_t *map;
    int64_t n_steps;
    float lr, gamma, eps, clip;
    int b, M;
    uint32_t key0, key1, level;
    int t;
};

__device__ __forceinline__ float clampf(float g, float c) { return fminf(fmaxf(g, -c), c); }

__device__ __forceinline__ float ipowf(float x, int n) {
    float r = 1.0f;
    for (int i = 0; i < n; ++i) r *= x;
    return r;
}

__device__ __forceinline__ int64_t alias_pick(const uint2 *table, int64_t n, uint32_t hi,
                                              uint32_t lo, uint32_t coin) {
    const int64_t idx = (int64_t)__umul64hi(((uint64_t)hi << 32) | lo, (uint64_t)n);
    const uint2 rec = __ldg(table + idx);
    return (u32_to_unit(coin) < __uint_as_float(rec.x)) ? idx : (int64_t)rec.y;
}

__device__ __forceinline__ float2 ld_y(const float2 *y, int64_t i) { return __ldcg(y + i); }

__device__ __forceinline__ void add_y(float2 *y, int64_t i, float dx, float dy) {
    atomicAdd(y + i, make_float2(dx, dy));
}

__global__ void __launch_bounds__(256) sampled_kernel(SArgs A, float2 *y) {
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const float two_b = 2.0f * (float)A.b;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < A.n_steps;
         s += nthreads) {
        const uint32_t c1 = (uint32_t)(s >> 32) ^ ((uint32_t)A.t << 1);
        u32x4 r = philox4x32(u32x4{(uint32_t)s, c1, (A.level << 24) | 0xff00u, 0x5a3d1e55u},
                             A.key0, A.key1);
        // directed pair ~ P at level 0
        const int64_t i0 = alias_pick(A.src_alias, A.n0, r.x, r.y, r.z);
        int64_t lo = A.indptr0[i0], hi = A.indptr0[i0 + 1];
        if (hi <= lo) continue;
        const float u = u32_to_unit(r.w);
        int64_t a = lo, bnd = hi - 1;  // first e with cum[e] > u (last entry is 1)
        while (a < bnd) {
            const int64_t mid = (a + bnd) >> 1;
            if (__ldg(A.cum0 + mid) > u) bnd = mid;
            else a = mid + 1;
        }
        const int64_t j0 = A.targets0[a];
        const int64_t i = A.map ? (int64_t)A.map[i0] : i0;
        const int64_t j = A.map ? (int64_t)A.map[j0] : j0;
        float2 yi = ld_y(y, i);
        if (i != j) {  // _kernels.py:82-105
            const float2 yj = ld_y(y, j);
            const float dx = yi.x - yj.x, dy = yi.y - yj.y;
            const float ld2 = dx * dx + dy * dy;
            if (ld2 > 0.f) {
                const float pw = ipowf(ld2, A.b - 1);
                const float coef = -two_b * pw / (1.0f + pw * ld2);
                const float gx = A.lr * clampf(coef * dx, A.clip);
                const float gy = A.lr * clampf(coef * dy, A.clip);
                add_y(y, i, gx, gy);
                add_y(y, j, -gx, -gy);
                yi.x += gx;
                yi.y += gy;
            }
        }
        for (int m = 0; m < A.M; ++m) {  // _kernels.py:106-140
            int64_t target = -1;
            for (int attempt = 0; attempt < 9; ++attempt) {
                const u32x4 q = philox4x32(
                    u32x4{(uint32_t)s, c1, (A.level << 24) | ((uint32_t)m << 8) | (uint32_t)attempt,
                          0x9e6a7e11u},
                    A.key0, A.key1);
                const int64_t c0 = alias_pick(A.neg_alias, A.n0, q.x, q.y, q.z);
                const int64_t cm = A.map ? (int64_t)A.map[c0] : c0;
                if (cm != i && cm != j) {
                    target = cm;
                    break;
                }
            }
            if (target < 0) continue;
            const float2 yc = ld_y(y, target);
            const float dx = yi.x - yc.x, dy = yi.y - yc.y;
            const float ld2 = dx * dx + dy * dy;
            if (ld2 + A.eps > 0.f) {
                const float pw = ipowf(ld2, A.b - 1);
                const float coef = A.gamma * two_b / ((ld2 + A.eps) * (1.0f + pw * ld2));
                const float gx = A.lr * clampf(coef * dx, A.clip);
                const float gy = A.lr * clampf(coef * dy, A.clip);
                add_y(y, i, gx, gy);
                add_y(y, target, -gx, -gy);
                yi.x += gx;
                yi.y += gy;
            }
        }
    }
}

// warp per row: inclusive prefix of P normalised by the row sum (last entry 1)
__global__ void row_cum_kernel(const int64_t *__restrict__ indptr, const double *__restrict__ P,
                               int64_t n, float *cum) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t lo = indptr[i], hi = indptr[i + 1];
        double total = 0.0;
        for (int64_t e = lo + lane; e < hi; e += 32) total += P[e];
        for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(kFull, total, o);
        double carry = 0.0;
        for (int64_t base = lo; base < hi; base += 32) {
            const int64_t e = base + lane;
            double v = e < hi ? P[e] : 0.0;
            for (int o = 1; o < 32; o <<= 1) {
                double t = __shfl_up_sync(kFull, v, o);
                if (lane >= o) v += t;
            }
            if (e < hi) cum[e] = (e == hi - 1 || total <= 0.0) ? 1.0f : (float)((carry + v) / total);
            carry += __shfl_sync(kFull, v, 31);
        }
    }
}

}  // namespace
}  // namespace drg

using namespace drg;

extern "C" int drg_row_cumulative(const int64_t *indptr, const double *P, int64_t n,
                                  float *out_cum, void *stream) {
    if (n <= 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(n * 32, 256), kSMs * 64);
    row_cum_kernel<<<g, 256, 0, st>>>(indptr, P, n, out_cum);
    DRG_LAUNCHED("row_cum_kernel");
    return DRG_OK;
}

extern "C" int drg_layout_sampled(const int64_t *indptr0, const int32_t *targets0,
                                  const float *cum0, const uint64_t *src_alias,
                                  const uint64_t *neg_alias, int64_t n0, const int32_t *map,
                                  float *y, int64_t n_l, int64_t n_steps, int t0, int n_iter,
                                  int iters, double lr0, double gamma, double eps, double clip,
                                  int b, int M, uint64_t seed, int level, int64_t max_threads,
                                  void *stream) {
    if (n0 <= 0 || n_l <= 0 || n_steps < 0 || n_iter < 0) return DRG_OK;
    if (b < 1 || M < 0 || iters < 1) return fail(DRG_ERR_INVALID, "bad optimizer parameters");
    cudaStream_t st = as_stream(stream);
    SArgs A;
    A.indptr0 = indptr0;
    A.targets0 = targets0;
    A.cum0 = cum0;
    A.src_alias = reinterpret_cast<const uint2 *>(src_alias);
    A.neg_alias = reinterpret_cast<const uint2 *>(neg_alias);
    A.n0 = n0;
    A.map = map;
    A.n_steps = n_steps;
    A.gamma = (float)gamma;
    A.eps = (float)eps;
    A.clip = (float)clip;
    A.b = b;
    A.M = M;
    A.key0 = (uint32_t)seed;
    A.key1 = (uint32_t)(seed >> 32);
    A.level = (uint32_t)level;
    int64_t threads = std::max<int64_t>(256, std::min<int64_t>(n_steps, max_threads));
    const unsigned grid = (unsigned)ceil_div(threads, 256);
    for (int j = 0; j < n_iter; ++j) {
        A.t = t0 + j;
        A.lr = (float)std::max(lr0 * (1.0 - (double)A.t / (double)iters), 0.0);
        sampled_kernel<<<grid, 256, 0, st>>>(A, reinterpret_cast<float2 *>(y));
        DRG_LAUNCHED("sampled_kernel");
    }
    return DRG_OK;
}
