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
    p_terms_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n * 32, kThreads), sm_count() * 16), kThreads,
                     0, st>>>(indptr, targets, P, yy, n, b, d);
    DRG_LAUNCHED("p_terms_kernel");
    if (z_pairs <= 0) {
        z_exact_kernel<<<(unsigned)ceil_div(n, kThreads), kThreads, 0, st>>>(yy, n, b, d + 3);
        DRG_LAUNCHED("z_exact_kernel");
    } else {
        z_mc_kernel<<<(unsigned)std::min<int64_t>(ceil_div(z_pairs, kThreads), sm_count() * 32), kThreads,
                      0, st>>>(yy, n, b, z_pairs, (uint32_t)seed, (uint32_t)(seed >> 32), d + 3);
        DRG_LAUNCHED("z_mc_kernel");
    }
    DRG_CUDA(cudaMemcpyAsync(out4, d, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (z_pairs > 0) out4[3] = out4[3] / (double)z_pairs * (double)n * (double)(n - 1);
    return DRG_OK;
}

// ---------------------------------------------------------------------------------
// Neighbourhood preservation (metrics.py:114-145): for each query node i with
// k_i = |H_i| (its k_eval-hop set, from K1), the k_i nearest OTHER nodes of the
// layout with ties broken by lower id (the reference's exact mode, stable argsort
// metrics.py:77-95), then Jaccard |H_i & L_i| / |H_i | L_i|; empty H_i counts 1.
// k-NN: uniform grid over the layout, ring search around the query cell; a ring
// is complete once the k-th distance is < r * cell (strict: ties cannot hide in
// unsearched cells).  Distances in fp64 from the fp32 positions, computed like
// numpy ((dx*dx) + (dy*dy), no FMA).  Warp tier for k <= 448, block tier for
// k <= 3584.
namespace drg {
namespace {

struct Grid {
    double x0, y0, cs;
    int gx, gy;
    const int32_t *cell_start;  // [gx*gy + 1]
    const int32_t *cell_nodes;  // nodes sorted by cell
};

__device__ __forceinline__ double d2_of(float2 a, float2 b) {
    const double dx = (double)a.x - (double)b.x, dy = (double)a.y - (double)b.y;
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

__device__ __forceinline__ bool key_less(uint64_t da, uint32_t ia, uint64_t db, uint32_t ib) {
    return da < db || (da == db && ia < ib);
}

// bitonic sort of (d, id) pairs over P (power of two) entries, `nt` cooperating threads
__device__ void pair_sort(uint64_t *d, uint32_t *id, int P, int tid, int nt, bool block) {
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < (P >> 1); i += nt) {
                const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                if (key_less(d[hi], id[hi], d[lo], id[lo]) == up) {
                    const uint64_t td = d[lo];
                    d[lo] = d[hi];
                    d[hi] = td;
                    const uint32_t ti = id[lo];
                    id[lo] = id[hi];
                    id[hi] = ti;
                }
            }
            if (block) __syncthreads();
            else __syncwarp();
        }
}

__device__ void u32_sort(uint32_t *a, int P, int tid, int nt, bool block) {
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < (P >> 1); i += nt) {
                const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                if ((a[lo] > a[hi]) == up) {
                    const uint32_t t = a[lo];
                    a[lo] = a[hi];
                    a[hi] = t;
                }
            }
            if (block) __syncthreads();
            else __syncwarp();
        }
}

__device__ __forceinline__ int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

// One query, cooperatively by `nt` threads (a warp or a block) with candidate
// buffers of capacity CAP in shared memory.  Returns the intersection count (all
// threads), or -1 if the candidate set overflowed.
template <int CAP, bool BLOCK>
__device__ int np_query(const Grid &G, const float2 *__restrict__ y, int64_t n, int32_t q,
                        int k, const int32_t *__restrict__ hop_ids, int64_t hop_lo,
                        uint64_t *cd, uint32_t *cid, int *s_cnt, int tid, int nt) {
    const float2 yq = y[q];
    const int cx = min(max((int)floor(((double)yq.x - G.x0) / G.cs), 0), G.gx - 1);
    const int cy = min(max((int)floor(((double)yq.y - G.y0) / G.cs), 0), G.gy - 1);
    int cnt = 0;
    if (BLOCK) {
        if (tid == 0) *s_cnt = 0;
        __syncthreads();
    }
    const int rmax = max(G.gx, G.gy);
    for (int r = 0; r <= rmax; ++r) {
        // cells of ring r: iterate the (2r+1)^2 square border
        const int side = 2 * r + 1;
        const int ncell = (r == 0) ? 1 : 4 * (side - 1);
        for (int c = 0; c < ncell; ++c) {
            int dx, dy;
            if (r == 0) {
                dx = 0;
                dy = 0;
            } else {
                const int edge = c / (side - 1), off = c % (side - 1);
                if (edge == 0) { dx = -r + off; dy = -r; }
                else if (edge == 1) { dx = r; dy = -r + off; }
                else if (edge == 2) { dx = r - off; dy = r; }
                else { dx = -r; dy = r - off; }
            }
            const int x = cx + dx, yy = cy + dy;
            if (x < 0 || yy < 0 || x >= G.gx || yy >= G.gy) continue;
            const int cell = yy * G.gx + x;
            const int a = G.cell_start[cell], b = G.cell_start[cell + 1];
            for (int base = a; base < b; base += nt) {
                const int p = base + tid;
                bool take = false;
                uint32_t v = 0;
                uint64_t dv = 0;
                if (p < b) {
                    v = (uint32_t)G.cell_nodes[p];
                    if ((int32_t)v != q) {
                        take = true;
                        dv = (uint64_t)__double_as_longlong(d2_of(yq, y[v]));
                    }
                }
                int pos;
                if (BLOCK) {
                    pos = take ? atomicAdd(s_cnt, 1) : 0;
                } else {
                    const unsigned bal = __ballot_sync(kFull, take);
                    pos = cnt + __popc(bal & ((1u << tid) - 1u));
                    cnt += __popc(bal);
                }
                if (take && pos < CAP) {
                    cd[pos] = dv;
                    cid[pos] = v;
                }
                if (BLOCK) {
                    __syncthreads();
                    cnt = *s_cnt;
                    __syncthreads();
                }
                if (cnt > CAP - nt) {  // prune to the k best so far
                    if (cnt > CAP) return -1;
                    const int P = next_pow2(cnt);
                    for (int i = cnt + tid; i < P; i += nt) {
                        cd[i] = ~0ull;
                        cid[i] = 0xffffffffu;
                    }
                    if (BLOCK) __syncthreads();
                    else __syncwarp();
                    pair_sort(cd, cid, P, tid, nt, BLOCK);
                    cnt = min(cnt, k);
                    if (BLOCK) {
                        if (tid == 0) *s_cnt = cnt;
                        __syncthreads();
                    }
                }
            }
        }
        if (cnt >= k) {
            // k-th smallest distance among candidates; stop if < r * cs
            const int P = next_pow2(cnt);
            for (int i = cnt + tid; i < P; i += nt) {
                cd[i] = ~0ull;
                cid[i] = 0xffffffffu;
            }
            if (BLOCK) __syncthreads();
            else __syncwarp();
            pair_sort(cd, cid, P, tid, nt, BLOCK);
            cnt = min(cnt, k);  // keep the k best
            if (BLOCK) {
                if (tid == 0) *s_cnt = cnt;
                __syncthreads();
            }
            const double dk = __longlong_as_double((long long)cd[k - 1]);
            const double reach = (double)r * G.cs;
            if (dk < reach * reach || r == rmax) break;
        }
    }
    if (cnt < k) {  // fewer than k other nodes exist at all (k <= n - 1 by construction)
        return -1;
    }
    // L ids sorted, then count hop ids present (binary search)
    const int P = next_pow2(k);
    for (int i = k + tid; i < P; i += nt) cid[i] = 0xffffffffu;
    if (BLOCK) __syncthreads();
    else __syncwarp();
    u32_sort(cid, P, tid, nt, BLOCK);
    int inter = 0;
    for (int e = tid; e < k; e += nt) {
        const uint32_t h = (uint32_t)hop_ids[hop_lo + e];
        int lo = 0, hi = k;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cid[mid] < h) lo = mid + 1;
            else hi = mid;
        }
        inter += (lo < k && cid[lo] == h);
    }
    if (BLOCK) {
        __syncthreads();
        if (tid == 0) *s_cnt = 0;
        __syncthreads();
        atomicAdd(s_cnt, inter);
        __syncthreads();
        inter = *s_cnt;
        __syncthreads();
    } else {
        for (int o = 16; o > 0; o >>= 1) inter += __shfl_xor_sync(kFull, inter, o);
    }
    return inter;
}

constexpr int kNpWarpCap = 512;
constexpr int kNpWarps = 4;
constexpr int kNpBlockCap = 4096;

__global__ void __launch_bounds__(kNpWarps * 32)
    np_warp_kernel(Grid G, const float2 *__restrict__ y, int64_t n,
                   const int64_t *__restrict__ hop_indptr, const int32_t *__restrict__ hop_ids,
                   const int32_t *__restrict__ queries, int64_t nq, double *score,
                   int32_t *big_list, unsigned long long *big_count) {
    __shared__ uint64_t s_d[kNpWarps][kNpWarpCap];
    __shared__ uint32_t s_id[kNpWarps][kNpWarpCap];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t t = (int64_t)blockIdx.x * kNpWarps + w; t < nq; t += (int64_t)gridDim.x * kNpWarps) {
        const int32_t q = queries ? queries[t] : (int32_t)t;
        const int64_t lo = hop_indptr[q], hi = hop_indptr[q + 1];
        const int k = (int)(hi - lo);
        if (k == 0) {
            if (lane == 0) score[t] = 1.0;
            continue;
        }
        if (k > kNpWarpCap - 64) {
            if (lane == 0) big_list[atomicAdd(big_count, 1ull)] = (int32_t)t;
            continue;
        }
        const int inter = np_query<kNpWarpCap, false>(G, y, n, q, k, hop_ids, lo, s_d[w], s_id[w],
                                                      nullptr, lane, 32);
        if (lane == 0) score[t] = inter < 0 ? -1.0 : (double)inter / (double)(2 * k - inter);
        __syncwarp();
    }
}

__global__ void __launch_bounds__(256)
    np_block_kernel(Grid G, const float2 *__restrict__ y, int64_t n,
                    const int64_t *__restrict__ hop_indptr, const int32_t *__restrict__ hop_ids,
                    const int32_t *__restrict__ queries, const int32_t *__restrict__ list,
                    int64_t nl, double *score) {
    extern __shared__ uint64_t smem64[];
    uint64_t *cd = smem64;
    uint32_t *cid = reinterpret_cast<uint32_t *>(smem64 + kNpBlockCap);
    __shared__ int s_cnt;
    for (int64_t b = blockIdx.x; b < nl; b += gridDim.x) {
        const int64_t t = list[b];
        const int32_t q = queries ? queries[t] : (int32_t)t;
        const int64_t lo = hop_indptr[q], hi = hop_indptr[q + 1];
        const int k = (int)(hi - lo);
        int inter = -1;
        if (k <= kNpBlockCap - 512)
            inter = np_query<kNpBlockCap, true>(G, y, n, q, k, hop_ids, lo, cd, cid, &s_cnt,
                                                threadIdx.x, blockDim.x);
        if (threadIdx.x == 0) score[t] = inter < 0 ? -1.0 : (double)inter / (double)(2 * k - inter);
        __syncthreads();
    }
}

__global__ void bbox_kernel(const float2 *__restrict__ y, int64_t n, float *out4) {
    float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float2 v = y[i];
        mnx = fminf(mnx, v.x);
        mny = fminf(mny, v.y);
        mxx = fmaxf(mxx, v.x);
        mxy = fmaxf(mxy, v.y);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mnx = fminf(mnx, __shfl_xor_sync(kFull, mnx, o));
        mny = fminf(mny, __shfl_xor_sync(kFull, mny, o));
        mxx = fmaxf(mxx, __shfl_xor_sync(kFull, mxx, o));
        mxy = fmaxf(mxy, __shfl_xor_sync(kFull, mxy, o));
    }
    if ((threadIdx.x & 31) == 0) {
        // order-preserving integer maps for float atomics
        auto enc = [](float f) {
            unsigned u = __float_as_uint(f);
            return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
        };
        atomicMin(reinterpret_cast<unsigned *>(out4) + 0, enc(mnx));
        atomicMin(reinterpret_cast<unsigned *>(out4) + 1, enc(mny));
        atomicMax(reinterpret_cast<unsigned *>(out4) + 2, enc(mxx));
        atomicMax(reinterpret_cast<unsigned *>(out4) + 3, enc(mxy));
    }
}

__global__ void cell_kernel(const float2 *__restrict__ y, int64_t n, double x0, double y0,
                            double cs, int gx, int gy, int32_t *cell_of, int32_t *counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float2 v = y[i];
        const int cx = min(max((int)floor(((double)v.x - x0) / cs), 0), gx - 1);
        const int cy = min(max((int)floor(((double)v.y - y0) / cs), 0), gy - 1);
        const int c = cy * gx + cx;
        cell_of[i] = c;
        atomicAdd(counts + c, 1);
    }
}

__global__ void iota32_kernel(int32_t *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)i;
}

}  // namespace
}  // namespace drg

using namespace drg;

static inline float dec_f(unsigned u) {
    u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

extern "C" int drg_neighborhood_preservation(const float *y, int64_t n,
                                             const int64_t *hop_indptr, const int32_t *hop_ids,
                                             const int32_t *queries, int64_t n_queries,
                                             double *out_score, void *stream) {
    if (n < 2) return fail(DRG_ERR_INVALID, "need at least 2 nodes");
    if (n >= 0x7fffffffLL) return fail(DRG_ERR_INVALID, "node count exceeds int32");
    cudaStream_t st = as_stream(stream);
    const float2 *yy = reinterpret_cast<const float2 *>(y);
    const int64_t nq = queries ? n_queries : n;
    Scratch bb(st), cell_of(st), counts(st), start(st), nodes(st), keys2(st), iota(st), tmp(st),
        big(st), bigc(st), scores(st);
    DRG_CUDA(bb.alloc(16));
    const unsigned init[4] = {0xffffffffu, 0xffffffffu, 0u, 0u};
    DRG_CUDA(cudaMemcpyAsync(bb.p, init, 16, cudaMemcpyHostToDevice, st));
    bbox_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), sm_count() * 8), 256, 0, st>>>(
        yy, n, bb.as<float>());
    DRG_LAUNCHED("bbox_kernel");
    unsigned hb[4];
    DRG_CUDA(cudaMemcpyAsync(hb, bb.p, 16, cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    const double x0 = dec_f(hb[0]), y0 = dec_f(hb[1]), x1 = dec_f(hb[2]), y1 = dec_f(hb[3]);
    if (!std::isfinite(x0) || !std::isfinite(x1) || !std::isfinite(y0) || !std::isfinite(y1))
        return fail(DRG_ERR_NONFINITE, "non-finite layout");
    const double span = std::max(std::max(x1 - x0, y1 - y0), 1e-30);
    const int g = (int)std::max(1.0, std::ceil(std::sqrt((double)n / 2.0)));
    const double cs = span / g * (1.0 + 1e-9);
    const int gx = std::max(1, (int)std::ceil((x1 - x0) / cs + 1e-12));
    const int gy = std::max(1, (int)std::ceil((y1 - y0) / cs + 1e-12));
    const int64_t ncell = (int64_t)gx * gy;
    DRG_CUDA(cell_of.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(counts.alloc(sizeof(int32_t) * (size_t)(ncell + 1)));
    DRG_CUDA(start.alloc(sizeof(int32_t) * (size_t)(ncell + 1)));
    DRG_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(int32_t) * (size_t)(ncell + 1), st));
    const unsigned fg = (unsigned)std::min<int64_t>(ceil_div(n, 256), sm_count() * 16);
    cell_kernel<<<fg, 256, 0, st>>>(yy, n, x0, y0, cs, gx, gy, cell_of.as<int32_t>(),
                                    counts.as<int32_t>());
    DRG_LAUNCHED("cell_kernel");
    size_t tb = 0, tb2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, counts.as<int32_t>(), start.as<int32_t>(),
                                  ncell + 1, st);
    DRG_CUDA(nodes.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(keys2.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(iota.alloc(sizeof(int32_t) * (size_t)n));
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, cell_of.as<int32_t>(), keys2.as<int32_t>(),
                                    iota.as<int32_t>(), nodes.as<int32_t>(), n, 0, 32, st);
    DRG_CUDA(tmp.alloc(std::max(tb, tb2)));
    DRG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, counts.as<int32_t>(), start.as<int32_t>(),
                                           ncell + 1, st));
    iota32_kernel<<<fg, 256, 0, st>>>(iota.as<int32_t>(), n);
    DRG_LAUNCHED("iota32_kernel");
    DRG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb2, cell_of.as<int32_t>(),
                                             keys2.as<int32_t>(), iota.as<int32_t>(),
                                             nodes.as<int32_t>(), n, 0, 32, st));
    g_launches.fetch_add(2, std::memory_order_relaxed);
    Grid G{x0, y0, cs, gx, gy, start.as<int32_t>(), nodes.as<int32_t>()};
    DRG_CUDA(big.alloc(sizeof(int32_t) * (size_t)std::max<int64_t>(nq, 1)));
    DRG_CUDA(bigc.alloc(sizeof(unsigned long long)));
    DRG_CUDA(cudaMemsetAsync(bigc.p, 0, sizeof(unsigned long long), st));
    np_warp_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nq, kNpWarps), sm_count() * 64),
                     kNpWarps * 32, 0, st>>>(G, yy, n, hop_indptr, hop_ids, queries, nq,
                                             out_score, big.as<int32_t>(),
                                             bigc.as<unsigned long long>());
    DRG_LAUNCHED("np_warp_kernel");
    unsigned long long h_big = 0;
    DRG_CUDA(cudaMemcpyAsync(&h_big, bigc.p, sizeof(h_big), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (h_big > 0) {
        const size_t smem = (size_t)kNpBlockCap * (8 + 4);
        DRG_CUDA(cudaFuncSetAttribute(np_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        np_block_kernel<<<(unsigned)std::min<unsigned long long>(h_big, sm_count() * 2), 256, smem, st>>>(
            G, yy, n, hop_indptr, hop_ids, queries, big.as<int32_t>(), (int64_t)h_big, out_score);
        DRG_LAUNCHED("np_block_kernel");
    }
    return DRG_OK;
}
