// Parity instrument on the device: the KL
// divergence of a layout with the unnormalised t-kernel lp_kernel
// (optimizer.py:150-152),
//     KL(P || Q) = sum P log P + sum P log(1 + d^(2b)) + log Z,
//     Z = sum_{i != j} 1 / (1 + d_ij^(2b)),
// with Z exact (tiled all-pairs, fp32 inner sums over 2048-point shared-memory
// tiles, fp64 across tiles) or Monte-Carlo over uniform ordered pairs (Philox).
#include <cub/cub.cuh>

#include "common.cuh"

namespace drg {
namespace {

constexpr int kTile = 2048;
constexpr int kThreads = 256;

__device__ __forceinline__ float tkernel(float ld2, int b) {
    float pw = 1.0f;
    for (int i = 0; i < b; ++i) pw *= ld2;
    return 1.0f / (1.0f + pw);
}

__global__ void __launch_bounds__(kThreads)
    z_exact_kernel(const float2 *__restrict__ y, int64_t n, int b, double *acc) {
    __shared__ float2 tile[kTile];
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const float2 yi = i < n ? y[i] : make_float2(0.f, 0.f);
    double total = 0.0;
    for (int64_t jt = 0; jt < n; jt += kTile) {
        const int64_t cnt = min((int64_t)kTile, n - jt);
        for (int q = threadIdx.x; q < kTile; q += kThreads)
            tile[q] = q < cnt ? y[jt + q] : make_float2(3e18f, 3e18f);
        __syncthreads();
        float s = 0.f;
        if (b == 2) {
#pragma unroll 8
            for (int q = 0; q < kTile; ++q) {
                const float dx = yi.x - tile[q].x, dy = yi.y - tile[q].y;
                const float ld2 = fmaf(dx, dx, dy * dy);
                s += __frcp_rn(fmaf(ld2, ld2, 1.0f));
            }
        } else {
            for (int q = 0; q < kTile; ++q) {
                const float dx = yi.x - tile[q].x, dy = yi.y - tile[q].y;
                s += tkernel(fmaf(dx, dx, dy * dy), b);
            }
        }
        total += (double)s;
        __syncthreads();
    }
    if (i < n) total -= 1.0;  // the i == j term
    else total = 0.0;
    typedef cub::BlockReduce<double, kThreads> BR;
    __shared__ typename BR::TempStorage tmp;
    const double bsum = BR(tmp).Sum(total);
    if (threadIdx.x == 0) atomicAdd(acc, bsum);
}

__global__ void __launch_bounds__(kThreads)
    z_mc_kernel(const float2 *__restrict__ y, int64_t n, int b, int64_t pairs, uint32_t k0,
                uint32_t k1, double *acc) {
    double total = 0.0;
    for (int64_t p = (int64_t)blockIdx.x * kThreads + threadIdx.x; p < pairs;
         p += (int64_t)gridDim.x * kThreads) {
        const u32x4 r = philox4x32(u32x4{(uint32_t)p, (uint32_t)(p >> 32), 0x2a11u, 0x7e57u}, k0, k1);
        const int64_t i = (int64_t)__umul64hi(((uint64_t)r.x << 32) | r.y, (uint64_t)n);
        int64_t j = (int64_t)__umul64hi(((uint64_t)r.z << 32) | r.w, (uint64_t)(n - 1));
        j += (j >= i);
        const float2 a = y[i], c = y[j];
        const float dx = a.x - c.x, dy = a.y - c.y;
        total += (double)tkernel(fmaf(dx, dx, dy * dy), b);
    }
    typedef cub::BlockReduce<double, kThreads> BR;
    __shared__ typename BR::TempStorage tmp;
    const double bsum = BR(tmp).Sum(total);
    if (threadIdx.x == 0) atomicAdd(acc, bsum);
}

// warp per row: sum P log P, sum P log(1 + d^(2b)), sum P
__global__ void __launch_bounds__(kThreads)
    p_terms_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ targets,
                   const double *__restrict__ P, const float2 *__restrict__ y, int64_t n, int b,
                   double *acc) {
    const int lane = threadIdx.x & 31;
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int64_t i = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * kThreads) >> 5) {
        const float2 yi = y[i];
        for (int64_t e = indptr[i] + lane; e < indptr[i + 1]; e += 32) {
            const double w = P[e];
            if (!(w > 0.0)) continue;
            const float2 yj = y[targets[e]];
            const double dx = (double)yi.x - yj.x, dy = (double)yi.y - yj.y;
            double pw = 1.0;
            const double ld2 = dx * dx + dy * dy;
            for (int q = 0; q < b; ++q) pw *= ld2;
            t0 += w * log(w);
            t1 += w * log1p(pw);
            t2 += w;
        }
    }
    typedef cub::BlockReduce<double, kThreads> BR;
    __shared__ typename BR::TempStorage tmp;
    double s0 = BR(tmp).Sum(t0);
    __syncthreads();
    double s1 = BR(tmp).Sum(t1);
    __syncthreads();
    double s2 = BR(tmp).Sum(t2);
    if (threadIdx.x == 0) {
        atomicAdd(acc, s0);
        atomicAdd(acc + 1, s1);
        atomicAdd(acc + 2, s2);
    }
}

}  // namespace
}  // namespace drg

using namespace drg;

extern "C" int drg_kl_terms(const int64_t *indptr, const int32_t *targets, const double *P,
                            int64_t n, const float *y, int b, int64_t z_pairs, uint64_t seed,
                            double *out4, void *stream) {
    if (n < 2 || b < 1) return fail(DRG_ERR_INVALID, "need n >= 2 and b >= 1");
    cudaStream_t st = as_stream(stream);
    Scratch acc(st);
    DRG_CUDA(acc.alloc(4 * sizeof(double)));
    DRG_CUDA(cudaMemsetAsync(acc.p, 0, 4 * sizeof(double), st));
    double *d = acc.as<double>();
    const float2 *yy = reinterpret_cast<const float2 *>(y);
    p_terms_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n * 32, kThreads), kSMs * 16), kThreads,
                     0, st>>>(indptr, targets, P, yy, n, b, d);
    DRG_LAUNCHED("p_terms_kernel");
    if (z_pairs <= 0) {
        z_exact_kernel<<<(unsigned)ceil_div(n, kThreads), kThreads, 0, st>>>(yy, n, b, d + 3);
        DRG_LAUNCHED("z_exact_kernel");
    } else {
        z_mc_kernel<<<(unsigned)std::min<int64_t>(ceil_div(z_pairs, kThreads), kSMs * 32), kThreads,
                      0, st>>>(yy, n, b, z_pairs, (uint32_t)seed, (uint32_t)(seed >> 32), d + 3);
        DRG_LAUNCHED("z_mc_kernel");
    }
    DRG_CUDA(cudaMemcpyAsync(out4, d, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (z_pairs > 0) out4[3] = out4[3] / (double)z_pairs * (double)n * (double)(n - 1);
    return DRG_OK;
}
