// Reference-faithful sampled epochs (update="sampled").
//
// K7 (layout.cu) applies one epoch's EXPECTED displacement with a CSR gather.  This
// kernel instead replays the reference step itself (_kernels.py:65-140), Hogwild
// style like sgd_epoch with threads > 1 (optimizer.py:325-345): every thread runs
// steps s of the epoch; a step draws a directed pair (i0, j0) ~ P at level 0 (the
// source by a Vose table over the row masses, then the target by the row's own Vose
// table -- the same law as the reference's canonical-pair table plus direction
// coin, optimizer.py:206-229), maps both ends to the current level, applies the
// clipped attractive update to both ends if they differ, then M negatives ~ Q at
// level 0, mapped and redrawn (<= 9 attempts) while they hit i or j, each moving
// both ends.  Updates are float2 atomic adds on y; the source position is tracked
// locally through the step as in the sequential kernel.
//
// Latency: all first-attempt draws (pair + M negatives) are made up front and
// their table loads issued together; the dependent chain of a step is then
// source alias -> row bounds -> row alias record + target -> (map) -> y.
#include "common.cuh"

namespace drg {
namespace {

constexpr int kMaxNeg = 6;  // negatives whose first draw is issued early

struct SArgs {
    const int64_t *indptr0;
    const int32_t *targets0;
    const uint2 *row_alias;  // per entry {fp32 threshold, int32 alias target}
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

__device__ __forceinline__ int64_t bucket(int64_t n, uint32_t hi, uint32_t lo) {
    return (int64_t)__umul64hi(((uint64_t)hi << 32) | lo, (uint64_t)n);
}

__device__ __forceinline__ int64_t accept(const uint2 rec, int64_t idx, uint32_t coin) {
    return (u32_to_unit(coin) < __uint_as_float(rec.x)) ? idx : (int64_t)rec.y;
}

__device__ __forceinline__ u32x4 neg_draw(const SArgs &A, int64_t s, uint32_t c1, int m,
                                          int attempt) {
    return philox4x32(
        u32x4{(uint32_t)s, c1, (A.level << 24) | ((uint32_t)m << 8) | (uint32_t)attempt,
              0x9e6a7e11u},
        A.key0, A.key1);
}

__device__ __forceinline__ float2 ld_y(const float2 *y, int64_t i) { return __ldcg(y + i); }

__device__ __forceinline__ void add_y(float2 *y, int64_t i, float dx, float dy) {
    atomicAdd(y + i, make_float2(dx, dy));
}

__global__ void __launch_bounds__(256, 4) sampled_kernel(SArgs A, float2 *y) {
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const float two_b = 2.0f * (float)A.b;
    const int Me = min(A.M, kMaxNeg);
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < A.n_steps;
         s += nthreads) {
        const uint32_t c1 = (uint32_t)(s >> 32) ^ ((uint32_t)A.t << 1);
        // ---- all first-attempt draws, table loads in flight together
        const u32x4 r = philox4x32(u32x4{(uint32_t)s, c1, (A.level << 24) | 0xff00u, 0x5a3d1e55u},
                                   A.key0, A.key1);
        const int64_t sb = bucket(A.n0, r.x, r.y);
        const uint2 srec = __ldg(A.src_alias + sb);
        int32_t nbk[kMaxNeg];   // level-0 ids < 2^31
        uint2 nrec[kMaxNeg];
        uint32_t ncoin[kMaxNeg];
#pragma unroll
        for (int m = 0; m < kMaxNeg; ++m) {
            if (m < Me) {
                const u32x4 q = neg_draw(A, s, c1, m, 0);
                nbk[m] = (int32_t)bucket(A.n0, q.x, q.y);
                ncoin[m] = q.z;
                nrec[m] = __ldg(A.neg_alias + nbk[m]);
            }
        }
        // ---- directed pair ~ P at level 0: source alias, then the row's alias
        const int64_t i0 = accept(srec, sb, r.z);
        const int64_t lo = __ldg(A.indptr0 + i0), hi = __ldg(A.indptr0 + i0 + 1);
        if (hi <= lo) continue;
        const u32x4 r2 = philox4x32(u32x4{(uint32_t)s, c1, (A.level << 24) | 0xfe00u, 0x3c6ef372u},
                                    A.key0, A.key1);
        const int64_t e = lo + bucket(hi - lo, r2.x, r2.y);
        const uint2 rrec = __ldg(A.row_alias + e);
        const int32_t tj = __ldg(A.targets0 + e);
        const int64_t j0 = (u32_to_unit(r2.z) < __uint_as_float(rrec.x)) ? (int64_t)tj
                                                                          : (int64_t)rrec.y;
        const int64_t i = A.map ? (int64_t)__ldg(A.map + i0) : i0;
        const int64_t j = A.map ? (int64_t)__ldg(A.map + j0) : j0;
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
                int64_t c0;
                if (attempt == 0 && m < Me) {
                    int32_t bk = 0;
                    uint2 rc = make_uint2(0, 0);
                    uint32_t cn = 0;
#pragma unroll
                    for (int q = 0; q < kMaxNeg; ++q)
                        if (q == m) {
                            bk = nbk[q];
                            rc = nrec[q];
                            cn = ncoin[q];
                        }
                    c0 = accept(rc, bk, cn);
                } else {
                    const u32x4 q = neg_draw(A, s, c1, m, attempt);
                    const int64_t bk = bucket(A.n0, q.x, q.y);
                    c0 = accept(__ldg(A.neg_alias + bk), bk, q.z);
                }
                const int64_t cm = A.map ? (int64_t)__ldg(A.map + c0) : c0;
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

// Thread per row: Vose's construction over the row's entries (optimizer.py:111-139,
// same stack discipline: small / large lists in index order, popped from the back),
// fp64 scaled weights in scratch, stacks in the caller's int32 scratch (the small
// stack grows up from the row start, the large one down from the row end).
// rec[e] = {fp32 threshold of bucket e, target of its alias entry}.
__global__ void row_alias_kernel(const int64_t *__restrict__ indptr,
                                 const int32_t *__restrict__ targets,
                                 const double *__restrict__ P, int64_t n, int32_t *stack,
                                 double *w, uint2 *rec) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = indptr[i], hi = indptr[i + 1];
        const int64_t len = hi - lo;
        if (len <= 0) continue;
        double total = 0.0;
        for (int64_t e = lo; e < hi; ++e) total += P[e];
        for (int64_t e = lo; e < hi; ++e) rec[e] = make_uint2(__float_as_uint(1.0f), targets[e]);
        if (!(total > 0.0)) continue;  // massless row: uniform
        const double f = (double)len / total;
        int64_t ns = 0, nl = 0;
        for (int64_t e = lo; e < hi; ++e) {
            w[e] = P[e] * f;
            if (w[e] < 1.0) stack[lo + ns++] = (int32_t)(e - lo);
            else stack[hi - 1 - nl++] = (int32_t)(e - lo);
        }
        while (ns > 0 && nl > 0) {
            const int64_t sm = lo + stack[lo + --ns];
            const int64_t lg = lo + stack[hi - 1 - --nl];
            rec[sm] = make_uint2(__float_as_uint((float)w[sm]), targets[lg]);
            w[lg] = (w[lg] + w[sm]) - 1.0;
            if (w[lg] < 1.0) stack[lo + ns++] = (int32_t)(lg - lo);
            else stack[hi - 1 - nl++] = (int32_t)(lg - lo);
        }
        // leftovers keep threshold 1 (optimizer.py:137-138)
    }
}

}  // namespace
}  // namespace drg

using namespace drg;

extern "C" int drg_row_alias(const int64_t *indptr, const int32_t *targets, const double *P,
                             int64_t n, int64_t nnz, uint64_t *out_rec, void *stream) {
    if (n <= 0 || nnz <= 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    Scratch stack(st), w(st);
    DRG_CUDA(stack.alloc(sizeof(int32_t) * (size_t)nnz));
    DRG_CUDA(w.alloc(sizeof(double) * (size_t)nnz));
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(n, 128), kSMs * 64);
    row_alias_kernel<<<g, 128, 0, st>>>(indptr, targets, P, n, stack.as<int32_t>(),
                                        w.as<double>(), reinterpret_cast<uint2 *>(out_rec));
    DRG_LAUNCHED("row_alias_kernel");
    return DRG_OK;
}

extern "C" int drg_layout_sampled(const int64_t *indptr0, const int32_t *targets0,
                                  const uint64_t *row_alias, const uint64_t *src_alias,
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
    A.row_alias = reinterpret_cast<const uint2 *>(row_alias);
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
