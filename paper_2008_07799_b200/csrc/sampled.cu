// Reference-faithful sampled epochs (update="sampled").
//
// K7 (layout.cu) applies one epoch's EXPECTED displacement with a CSR gather.  This
// kernel instead replays the reference step itself (_kernels.py:65-140), Hogwild
// style like sgd_epoch with threads > 1 (optimizer.py:325-345): every thread runs
// steps s of the epoch.  The reference draws a level-0 pair (i0, j0) ~ P and maps it
// to level l; that law equals "source a ~ R^l, then with probability c_a the
// collapsed pair (a, a), else the target b ~ P^l_a." (c_a = mass of pairs inside
// a / R^l_a), which this kernel samples from level-l tables (a Vose table over R^l,
// one Vose table per row of P^l) so coarse levels stay L2-resident.  Attraction is
// clipped and applied to both ends if i != j; M negatives ~ Q^l are redrawn (<= 9
// attempts) while they hit i or j, each moving both ends.  Updates are float2
// atomic adds on y; the source position is tracked locally through the step as in
// the sequential kernel.
//
// Latency: all first-attempt draws (pair + M negatives) are made up front and
// their table loads issued together; the dependent chain of a step is then
// source alias -> row bounds / c_a -> row alias record + target -> y.
#include <stdlib.h>

#include <algorithm>
#include <climits>
#include <mutex>
#include <string.h>
#include <dlfcn.h>

#include <cub/cub.cuh>

#include "common.cuh"

namespace drg {
namespace {

constexpr int kMaxNeg = 6;  // negatives whose first draw is issued early

// Distance-evaluation counts (_kernels.py:86, 122).  One counter would take one
// same-address atomic per warp -- ~3e5 per 5-epoch draw launch on the mesh,
// serialised in one L2 slice -- so warps add into kEvalSlots counters 128 B apart
// (EvalSlots below), summed into the caller's counter once per call.
constexpr int kEvalSlots = 64, kEvalStride = 16;

__device__ __forceinline__ void count_evals(unsigned long long *slots, unsigned nev) {
    if (!slots) return;
    const unsigned act = __activemask();
    nev = __reduce_add_sync(act, nev);
    if ((threadIdx.x & 31) == __ffs(act) - 1 && nev)
        atomicAdd(slots + (blockIdx.x % kEvalSlots) * kEvalStride, (unsigned long long)nev);
}

__global__ void evals_finish_kernel(unsigned long long *slots, unsigned long long *evals) {
    unsigned long long v = 0;
    for (int q = threadIdx.x; q < kEvalSlots; q += 32) v += slots[q * kEvalStride];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if (threadIdx.x == 0) *evals += v;
}

// The level's negative table (Q^l, optimizer.py:243-259): Vose over the nodes
// [0, n) that carry graph mass and, with probability tail_thr / 2^32, a uniform
// pick among the tail [n, n + tail_n) -- the isolated nodes, all at the same floor
// weight (optimizer.py:258), which isolated_last numbers last.  The law of one
// table over every node, from a table the size of the connected part (R-MAT: 53%
// at level 0, 40% at the coarse levels, where it stays in L2).  Drawn at the
// level itself: a level-0 draw mapped through the parent map has the same law
// (Q^l_a = sum of the level-0 weights in a) and costs a second random load.
struct NegTab {
    const uint2 *alias;
    int64_t n, tail_n;
    uint32_t tail_thr;
};

__device__ __forceinline__ int64_t bucket(int64_t n, uint32_t hi, uint32_t lo);
__device__ __forceinline__ int64_t accept(const uint2 rec, int64_t idx, uint32_t coin);

// L2 eviction-priority hints (createpolicy + ld.global.nc.L2::cache_hint): in the
// draw pass the negative table (re-read ~5 times per step) is kept, the one-touch
// random reads of the multi-GB / 100+ MB tables (row offsets, source table, maps)
// are evicted first, so the level's Q^l table stays in L2 on R-MAT.
__device__ __forceinline__ uint64_t l2_keep() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_stream() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint2 ld_hint(const uint2 *a, uint64_t pol) {
    uint2 r;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y) : "l"(a), "l"(pol));
    return r;
}
__device__ __forceinline__ int64_t ld_hint(const int64_t *a, uint64_t pol) {
    int64_t r;
    asm volatile("ld.global.nc.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(r) : "l"(a), "l"(pol));
    return r;
}
__device__ __forceinline__ uint4 ld_hint(const uint4 *a, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(a), "l"(pol));
    return r;
}
__device__ __forceinline__ int32_t ld_hint(const int32_t *a, uint64_t pol) {
    int32_t r;
    asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(a), "l"(pol));
    return r;
}

template <bool HINT = false>
__device__ __forceinline__ int64_t pick_neg(const NegTab &T, const u32x4 &q, uint64_t pol = 0) {
    if (q.w < T.tail_thr) return T.n + bucket(T.tail_n, q.x, q.y);
    const int64_t bk = bucket(T.n, q.x, q.y);
    return accept(HINT ? ld_hint(T.alias + bk, pol) : __ldg(T.alias + bk), bk, q.z);
}

struct SArgs {
    const int64_t *indptr;
    const uint2 *rec;        // level CSR records {target, W}
    const uint4 *row_alias;  // per entry {fp32 threshold, alias target, own target, 0}
    const uint2 *src_alias;  // Vose over R^l
    const float *collapse;   // probability that the drawn pair collapses into the source
    NegTab neg;              // Q^l
    int64_t n;
    int64_t step_lo;
    int64_t n_steps;
    float lr, gamma, eps, clip;
    int b, M;
    uint32_t key0, key1, level;
    int t;
    int probe;   // latency probe (DRG_SAMPLED_PROBE, tests only): 1 = no atomics, 2 = no row draw
    unsigned long long *evals;   // optional: distance evaluations (_kernels.py:86, 122)
};

__device__ __forceinline__ float clampf(float g, float c) { return fminf(fmaxf(g, -c), c); }

// x^n with n a compile-time constant (B > 0) or the runtime n (B == 0)
template <int B>
__device__ __forceinline__ float ipow_b(float x, int n) {
    if (B > 0) {
        float r = 1.0f;
#pragma unroll
        for (int i = 0; i < B - 1; ++i) r *= x;
        return r;
    }
    float r = 1.0f;
    for (int i = 0; i < n; ++i) r *= x;
    return r;
}

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
    return philox4x32<7>(
        u32x4{(uint32_t)s, c1, (A.level << 24) | ((uint32_t)m << 8) | (uint32_t)attempt,
              0x9e6a7e11u},
        A.key0, A.key1);
}

__device__ __forceinline__ float2 ld_y(const float2 *y, int64_t i) { return __ldcg(y + i); }

__device__ __forceinline__ void add_y(float2 *y, int64_t i, float dx, float dy) {
    atomicAdd(y + i, make_float2(dx, dy));
}

// Warp-aggregated update: lanes of the warp that target the same node combine their
// increments and one of them issues the atomic (same-address atomics serialise in
// L2; on hub-heavy levels -- R-MAT coarse levels -- most of a warp hits the same
// few nodes).  Called by all active lanes together; i < 0 = no update.
template <bool AGG>
__device__ __forceinline__ void add_y_w(float2 *y, int64_t i, float dx, float dy, int probe = 0) {
    if (probe & 1) {   // latency probe: keep the value live, skip the memory update
        if (i >= 0 && dx == 1234.5f) y[0].x = dy;
        return;
    }
    if (!AGG) {
        if (i >= 0) add_y(y, i, dx, dy);
        return;
    }
    const unsigned active = __activemask();
    const unsigned peers = __match_any_sync(active, (int)i);   // ids < 2^31 (-1: none)
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    for (unsigned rest = peers & ~(1u << leader); rest; rest &= rest - 1) {
        const int src = __ffs(rest) - 1;
        const float tx = __shfl_sync(peers, dx, src);
        const float ty = __shfl_sync(peers, dy, src);
        if (lane == leader) {
            dx += tx;
            dy += ty;
        }
    }
    if (lane == leader && i >= 0) add_y(y, i, dx, dy);
}

// One repulsion of _kernels.py:120-140: the source moves by +g (tracked locally in
// yi and in its step total), the negative by -g (returned in tu/tx/ty).
template <int B = 0>
__device__ __forceinline__ void repel(float2 &yi, float2 yc, int64_t target, float lr,
                                      float gamma, float eps, float clip, float two_b, int b,
                                      int64_t &tu, float &tx, float &ty, float &gix, float &giy) {
    tu = -1;
    tx = ty = 0.f;
    if (target < 0) return;
    const float dx = yi.x - yc.x, dy = yi.y - yc.y;
    const float ld2 = dx * dx + dy * dy;
    if (!(ld2 + eps > 0.f)) return;
    const float pw = ipow_b<B>(ld2, b - 1);
    const float coef = __fdividef(gamma * two_b, (ld2 + eps) * (1.0f + pw * ld2));
    const float gx = lr * clampf(coef * dx, clip);
    const float gy = lr * clampf(coef * dy, clip);
    tu = target;
    tx = -gx;
    ty = -gy;
    yi.x += gx;
    yi.y += gy;
    gix += gx;
    giy += gy;
}

// A negative whose position was gathered at the start of the step misses the
// updates this step already applied to the same node (a repeated negative); they
// are added back from the step's own record (ax/ay = 0 where nothing was applied),
// giving the sequential kernel's value.
__device__ __forceinline__ void own_updates(float2 &yc, int64_t target, int m,
                                            const int32_t *at, const float *ax,
                                            const float *ay) {
#pragma unroll
    for (int q = 0; q < kMaxNeg; ++q)
        if (q < m && at[q] == target) {
            yc.x += ax[q];
            yc.y += ay[q];
        }
}

template <bool AGG>
__global__ void __launch_bounds__(256, 3) sampled_kernel(SArgs A, float2 *y) {
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const float two_b = 2.0f * (float)A.b;
    const int Me = min(A.M, kMaxNeg);
    unsigned nev = 0;
    for (int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; sl < A.n_steps;
         sl += nthreads) {
        const int64_t s = A.step_lo + sl;
        const uint32_t c1 = (uint32_t)(s >> 32) ^ ((uint32_t)A.t << 1);
        // ---- every first-attempt draw up front; table loads in flight together
        const u32x4 r = philox4x32<7>(u32x4{(uint32_t)s, c1, (A.level << 24) | 0xff00u, 0x5a3d1e55u},
                                   A.key0, A.key1);
        const u32x4 r2 = philox4x32<7>(u32x4{(uint32_t)s, c1, (A.level << 24) | 0xfe00u, 0x3c6ef372u},
                                    A.key0, A.key1);
        const int64_t sb = bucket(A.n, r.x, r.y);
        const uint2 srec = __ldg(A.src_alias + sb);
        int32_t cand[kMaxNeg];   // first-attempt negatives (node ids < 2^31)
        float2 ycand[kMaxNeg];
#pragma unroll
        for (int m = 0; m < kMaxNeg; ++m) {
            if (m < Me) {
                cand[m] = (int32_t)pick_neg(A.neg, neg_draw(A, s, c1, m, 0));
            }
        }
        // speculative gathers of the candidates (redrawn below only if they hit i/j)
#pragma unroll
        for (int m = 0; m < kMaxNeg; ++m)
            if (m < Me) ycand[m] = ld_y(y, cand[m]);
        // ---- directed pair: source a ~ R^l; collapsed (a, a) with prob collapse[a],
        // else target ~ P^l_a. by the row's alias table
        const int64_t i = accept(srec, sb, r.z);
        const int64_t lo = __ldg(A.indptr + i), hi = __ldg(A.indptr + i + 1);
        const float cprob = A.collapse ? __ldg(A.collapse + i) : 0.0f;   // NULL: none (level 0)
        float2 yi = ld_y(y, i);
        int64_t j = i;
        if ((A.probe & 2) && hi > lo) {
            j = (int64_t)bucket(A.n, r2.x, r2.y);
        } else if (hi > lo && !(u32_to_unit(r.w) < cprob)) {
            const int64_t e = lo + bucket(hi - lo, r2.x, r2.y);
            const uint4 rrec = __ldcs(A.row_alias + e);   // one 16-byte record, evict-first
            j = (u32_to_unit(r2.z) < __uint_as_float(rrec.x)) ? (int64_t)rrec.z : (int64_t)rrec.y;
        }
        float gix = 0.f, giy = 0.f;   // the source's own increments of this step
        int64_t upd = -1;
        float ux = 0.f, uy = 0.f;
        nev += i != j;
        if (i != j) {  // _kernels.py:82-105
            const float2 yj = ld_y(y, j);
            const float dx = yi.x - yj.x, dy = yi.y - yj.y;
            const float ld2 = dx * dx + dy * dy;
            if (ld2 > 0.f) {
                const float pw = ipowf(ld2, A.b - 1);
                const float coef = __fdividef(-two_b * pw, 1.0f + pw * ld2);
                const float gx = A.lr * clampf(coef * dx, A.clip);
                const float gy = A.lr * clampf(coef * dy, A.clip);
                upd = j;
                ux = -gx;
                uy = -gy;
                yi.x += gx;
                yi.y += gy;
                gix += gx;
                giy += gy;
            }
        }
        add_y_w<AGG>(y, upd, ux, uy, A.probe);
        int32_t at[kMaxNeg];   // this step's updates of its first negatives
        float ax[kMaxNeg], ay[kMaxNeg];
#pragma unroll
        for (int m = 0; m < kMaxNeg; ++m) {  // _kernels.py:106-140
            if (m < Me) {
                int64_t target = -1;
                float2 yc = make_float2(0.f, 0.f);
                if (cand[m] != i && cand[m] != j) {
                    target = cand[m];
                    yc = ycand[m];
                    own_updates(yc, target, m, at, ax, ay);   // gathered before them
                }
                for (int attempt = 1; target < 0 && attempt < 9; ++attempt) {
                    const int64_t c0 = pick_neg(A.neg, neg_draw(A, s, c1, m, attempt));
                    if (c0 != i && c0 != j) {
                        target = c0;
                        yc = ld_y(y, c0);   // after this step's own atomics
                    }
                }
                int64_t tu;
                float tx, ty;
                nev += target >= 0;
                repel(yi, yc, target, A.lr, A.gamma, A.eps, A.clip, two_b, A.b, tu, tx, ty, gix,
                      giy);
                at[m] = (int32_t)tu;
                ax[m] = tx;
                ay[m] = ty;
                add_y_w<AGG>(y, tu, tx, ty, A.probe);
            }
        }
        for (int m = Me; m < A.M; ++m) {
            int64_t target = -1;
            float2 yc = make_float2(0.f, 0.f);
            for (int attempt = 0; target < 0 && attempt < 9; ++attempt) {
                const int64_t c0 = pick_neg(A.neg, neg_draw(A, s, c1, m, attempt));
                if (c0 != i && c0 != j) {
                    target = c0;
                    yc = ld_y(y, c0);
                }
            }
            int64_t tu;
            float tx, ty;
            nev += target >= 0;
            repel(yi, yc, target, A.lr, A.gamma, A.eps, A.clip, two_b, A.b, tu, tx, ty, gix, giy);
            add_y_w<AGG>(y, tu, tx, ty, A.probe);
        }
        // the source's own increments of the step, published once (the step sees
        // them locally in sequence, as the reference kernel does)
        add_y_w<AGG>(y, (gix != 0.f || giy != 0.f) ? i : -1, gix, giy, A.probe);
    }
    count_evals(A.evals, nev);
}

// ---- split formulation: draws, then updates -----------------------------------
// Everything a step draws -- the directed pair (i, j) and its M negatives, including
// the redraws (they are rejected only against i and j) -- depends on the static
// level tables and the counters, never on y.  draw_kernel resolves all of it for
// one or more whole epochs at full occupancy (a throughput-bound pass over the
// alias tables); apply_kernel then runs the Hogwild updates with the draws as a
// coalesced stream, so a step's dependent chain is just "gather y_i, y_j, y_c ->
// math -> atomics".  The same counters are used as in sampled_kernel, so the drawn
// steps are identical; only the interleaving of concurrent steps differs.
// Draw records: [epoch][field][step] int32, field 0 = i, 1 = j (j == i: collapsed
// pair, no attraction), 2 + m = negative m (-1: all 9 attempts hit i or j).
struct DArgs {
    const int64_t *indptr;
    const uint2 *span;    // optional {row start, row length} per node: one load, not two
    const uint4 *row_alias;
    const uint2 *src_alias;
    const float *collapse;
    NegTab neg;           // Q^l of the level itself
    const int32_t *map;   // non-NULL: level-0 pair tables, the pair mapped to level l
    int64_t n;            // nodes of the tables
    int64_t step_lo;
    int64_t n_steps;
    int64_t n_epochs;
    int M;
    uint32_t key0, key1, level;
    int t_first;
    int probe;
    int32_t *out;
    unsigned long long *evals;   // optional: distance evaluations (_kernels.py:86, 122)
    // source segment (multi-GPU: the sources a rank owns): the source alias table is
    // over n_src items; item q is node src_perm[src_lo + q] (src_perm NULL: src_lo + q)
    int64_t n_src, src_lo;
    const int32_t *src_perm;
    int64_t out_stride;   // field stride of out (>= n_steps; ranks' slices of one buffer)
    // optional 32-byte source records (drg_src_records; 1-GPU draws, src_lo = 0, no
    // src_perm): bucket b's {threshold, alias, span of b} and {span of the alias,
    // collapse of b, collapse of the alias} -- one random sector per drawn source
    // instead of three table reads (alias record, row span, collapse)
    const uint4 *src_rec = nullptr;
};

// small blocks: they fit beside the update pass's resident blocks
constexpr int kDrawBlock = 128;

// One step's draws, the reference's sequence (_kernels.py:66-119): the directed
// pair (source ~ R, target by the row's alias table, both mapped to the level) and
// the M negatives ~ Q^l redrawn (<= 9) while they hit i or j.  The first kMaxNeg
// negatives land in neg[] (-1: all attempts hit i or j); later ones are written to
// rest[m * stride] (the split form's records; NULL: M <= kMaxNeg).
template <bool HINT>
__device__ __forceinline__ void draw_step(const DArgs &A, int64_t s, uint32_t c1, int64_t &i_out,
                                          int64_t &j_out, int32_t *neg, int32_t *rest,
                                          int64_t stride, unsigned &nev) {
    const uint64_t keep = HINT ? l2_keep() : 0, once = HINT ? l2_stream() : 0;
    SArgs K;   // the counter layout of sampled_kernel
    K.key0 = A.key0;
    K.key1 = A.key1;
    K.level = A.level;
    const u32x4 r = philox4x32<7>(u32x4{(uint32_t)s, c1, (A.level << 24) | 0xff00u, 0x5a3d1e55u},
                                  A.key0, A.key1);
    const u32x4 r2 = philox4x32<7>(u32x4{(uint32_t)s, c1, (A.level << 24) | 0xfe00u, 0x3c6ef372u},
                                   A.key0, A.key1);
    const int64_t sb = bucket(A.n_src, r.x, r.y);
    uint2 srec = make_uint2(0u, 0u);
    uint4 q0 = make_uint4(0u, 0u, 0u, 0u), q1 = q0;
    if (A.src_rec) {   // both halves of one 32-byte record: one sector
        q0 = HINT ? ld_hint(A.src_rec + 2 * sb, once) : __ldg(A.src_rec + 2 * sb);
        q1 = HINT ? ld_hint(A.src_rec + 2 * sb + 1, once) : __ldg(A.src_rec + 2 * sb + 1);
    } else {
        srec = HINT ? ld_hint(A.src_alias + sb, once) : __ldg(A.src_alias + sb);
    }
    const int Me = min(A.M, kMaxNeg);
    int32_t cand[kMaxNeg];
#pragma unroll
    for (int m = 0; m < kMaxNeg; ++m) {
        if (m < Me) {
            cand[m] = (int32_t)pick_neg<HINT>(A.neg, neg_draw(K, s, c1, m, 0), keep);
        }
    }
    int64_t i, lo, hi;
    float cprob;
    if (A.src_rec) {
        const bool own = u32_to_unit(r.z) < __uint_as_float(q0.x);   // accept()
        i = own ? sb : (int64_t)q0.y;
        lo = own ? q0.z : q1.x;
        hi = lo + (own ? q0.w : q1.y);
        cprob = __uint_as_float(own ? q1.z : q1.w);
    } else {
        i = accept(srec, sb, r.z);
        i = A.src_perm ? (int64_t)__ldg(A.src_perm + A.src_lo + i) : A.src_lo + i;
        if (A.span) {
            const uint2 sp = HINT ? ld_hint(A.span + i, once) : __ldg(A.span + i);
            lo = sp.x;
            hi = lo + sp.y;
        } else {
            lo = HINT ? ld_hint(A.indptr + i, once) : __ldg(A.indptr + i);
            hi = HINT ? ld_hint(A.indptr + i + 1, once) : __ldg(A.indptr + i + 1);
        }
        cprob = A.collapse ? __ldg(A.collapse + i) : 0.0f;   // NULL: none
    }
    int64_t j = i;
    if ((A.probe & 2) && hi > lo) {
        j = (int64_t)bucket(A.n, r2.x, r2.y);
    } else if (hi > lo && !(u32_to_unit(r.w) < cprob)) {
        // one random 16-byte record of a multi-GB table: evict-first, so it does not
        // push the hot alias / y tables out of L2
        const uint4 rrec = __ldcs(A.row_alias + lo + bucket(hi - lo, r2.x, r2.y));
        j = (u32_to_unit(r2.z) < __uint_as_float(rrec.x)) ? (int64_t)rrec.z : (int64_t)rrec.y;
    }
    if (A.map) {   // the level-0 pair as seen at level l (_kernels.py:76-81)
        i = HINT ? ld_hint(A.map + i, once) : __ldg(A.map + i);
        j = HINT ? ld_hint(A.map + j, once) : __ldg(A.map + j);
    }
    nev += i != j;
    for (int m = 0; m < A.M; ++m) {
        int64_t target = -1;
        int first = 0;
        if (m < Me) {
            int32_t c0 = 0;
#pragma unroll
            for (int q = 0; q < kMaxNeg; ++q)
                if (q == m) c0 = cand[q];
            if (c0 != i && c0 != j) target = c0;
            first = 1;
        }
        for (int attempt = first; target < 0 && attempt < 9; ++attempt) {
            const int64_t c0 = pick_neg<HINT>(A.neg, neg_draw(K, s, c1, m, attempt), keep);
            if (c0 != i && c0 != j) target = c0;
        }
        nev += target >= 0;
        if (m < Me) {
#pragma unroll
            for (int q = 0; q < kMaxNeg; ++q)
                if (q == m) neg[q] = (int32_t)target;
        } else {
            __stcs(rest + (int64_t)(m - Me) * stride, (int32_t)target);
        }
    }
    i_out = i;
    j_out = j;
}

template <bool HINT>
__global__ void __launch_bounds__(kDrawBlock) draw_kernel(DArgs A) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= A.n_steps * A.n_epochs) return;
    const int64_t ep = g / A.n_steps, sl = g - ep * A.n_steps;
    const int64_t s = A.step_lo + sl;
    const uint32_t c1 = (uint32_t)(s >> 32) ^ ((uint32_t)(A.t_first + (int)ep) << 1);
    const int Me = min(A.M, kMaxNeg);
    int32_t *o = A.out + ep * (int64_t)(2 + A.M) * A.out_stride + sl;
    int64_t i, j;
    int32_t neg[kMaxNeg];
    unsigned nev = 0;
    draw_step<HINT>(A, s, c1, i, j, neg, o + (int64_t)(2 + Me) * A.out_stride, A.out_stride, nev);
    __stcs(o, (int32_t)i);   // read once by the update pass: streaming stores
    __stcs(o + A.out_stride, (int32_t)j);
#pragma unroll
    for (int m = 0; m < kMaxNeg; ++m)
        if (m < Me) __stcs(o + (int64_t)(2 + m) * A.out_stride, neg[m]);
    count_evals(A.evals, nev);
}

NegTab make_negtab(const uint64_t *alias, int64_t n, int64_t tail_n, double tail_p) {
    NegTab T;
    T.alias = reinterpret_cast<const uint2 *>(alias);
    T.n = n;
    T.tail_n = tail_n > 0 ? tail_n : 0;
    const double thr = std::floor(std::min(std::max(tail_p, 0.0), 1.0) * 4294967296.0 + 0.5);
    T.tail_thr = T.tail_n > 0 ? (uint32_t)std::min(thr, 4294967295.0) : 0u;
    return T;
}

int launch_draws(const DArgs &D, cudaStream_t st) {
    static const bool hints = [] {
        // measured: R-MAT scale 24 +1%, the C4 mesh -6% (its tables fit L2 and the
        // evict-first reads are re-read there): off unless DRG_DRAW_HINTS=1
        const char *e = getenv("DRG_DRAW_HINTS");
        return e && e[0] == '1';
    }();
    const unsigned grid = (unsigned)ceil_div(D.n_steps * D.n_epochs, kDrawBlock);
    if (hints) draw_kernel<true><<<grid, kDrawBlock, 0, st>>>(D);
    else draw_kernel<false><<<grid, kDrawBlock, 0, st>>>(D);
    DRG_LAUNCHED("draw_kernel");
    return DRG_OK;
}

struct PArgs {
    const int32_t *draws;   // one epoch of draw records (or a sub-batch's first step)
    int64_t n_steps;        // steps this launch applies
    int64_t stride;         // field stride of the draw records (the epoch's step count)
    unsigned long long *delta;   // deterministic mode: fixed-point increments [n][2]
    uint64_t spread;        // != 0: step sl runs column (sl * spread) % n_steps (see below)
    float lr, gamma, eps, clip;
    float hot_scale;        // apply_hot_kernel's fixed-point scale (set by launch_apply)
    int b, M;
    int probe;
    const float2 *snap = nullptr;   // DRG_SAMPLED_SNAPSHOT: epoch-start copy of y (negatives' reads)
    int *locks = nullptr;   // per-node step locks (apply_steps_locked), node v at v & lock_mask
    uint32_t lock_mask = 0xffffffffu;
    int zero = 0;           // 0 (a value the compiler cannot fold: release dependency)
};

// The reference step (_kernels.py:82-140) on drawn (i, j, negatives): the source's
// position is carried through the step, attraction and each repulsion move the
// other end by the opposite clipped increment; the source's own total is published
// once.  The next step's draw record is prefetched while this step runs.
// Deterministic mode (threads = 1): the epoch runs as sub-batches of steps that all
// read the positions frozen at the sub-batch start and add their increments to a
// 64-bit fixed-point buffer (integer atomics: the sum is independent of the order),
// which flush_kernel folds into y -- bitwise reproducible, with the same staleness
// law as Hogwild at that many steps in flight.
constexpr double kFixScale = 1099511627776.0;   // 2^40: |increment sum| < 2^23 per sub-batch

__device__ __forceinline__ void add_fixed(unsigned long long *d, int64_t i, float dx, float dy) {
    if (i < 0) return;
    atomicAdd(d + 2 * i, (unsigned long long)__double2ll_rn((double)dx * kFixScale));
    atomicAdd(d + 2 * i + 1, (unsigned long long)__double2ll_rn((double)dy * kFixScale));
}

// ---- position stores: where a step reads and moves the nodes it touches -------
// (one step body, step_body below, serves every mode)
template <bool AGG>
struct GlobalStore {   // Hogwild on y: float2 reductions (warp-aggregated on hub levels)
    float2 *y;
    int probe;
    __device__ __forceinline__ float2 load(int64_t v) const { return ld_y(y, v); }
    __device__ __forceinline__ float2 load_neg(int64_t v) const { return ld_y(y, v); }
    __device__ __forceinline__ void add(int64_t v, float dx, float dy) const {
        add_y_w<AGG>(y, v, dx, dy, probe);
    }
    __device__ __forceinline__ void add_neg(int64_t v, float dx, float dy) const { add(v, dx, dy); }
};

struct FixedStore {    // deterministic sub-batch: y frozen, fixed-point increments
    const float2 *y;
    unsigned long long *delta;
    __device__ __forceinline__ float2 load(int64_t v) const { return __ldcg(y + v); }
    __device__ __forceinline__ float2 load_neg(int64_t v) const { return __ldcg(y + v); }
    __device__ __forceinline__ void add(int64_t v, float dx, float dy) const {
        add_fixed(delta, v, dx, dy);
    }
    __device__ __forceinline__ void add_neg(int64_t v, float dx, float dy) const {
        add_fixed(delta, v, dx, dy);
    }
};

// Negatives read from a read-only snapshot of the positions (refreshed between
// epochs by snap_copy_kernel); every update -- the negatives' reactions too -- still
// goes to y at once.  Random gathers and float2 reductions on the SAME array run at
// 148 G/s on this B200, on separate arrays at 260 G/s (scripts/l2_random_peak.cu,
// profiles/r02_l2_random_peak.txt: reductions invalidate the lines the gathers
// replicate across the two L2 partitions); with the five negative gathers of a step
// moved to the snapshot the step's 14 accesses run at 213 G/s.  A negative's
// position is then up to one epoch old -- the weak long-range repulsion tolerates
// far more (the multi-GPU form, epoch-old reads AND deferred reactions: KL +0.00%,
// NP within noise on the C4 mesh); source and partner stay live.
struct SnapStore {
    float2 *y;
    const float2 *snap;
    int probe;
    __device__ __forceinline__ float2 load(int64_t v) const { return ld_y(y, v); }
    // (ld.cg, not the non-coherent path: with programmatic dependent launches this
    // kernel's blocks can become resident while the previous epoch's blocks still
    // fill the SM's L1 with the old snapshot)
    __device__ __forceinline__ float2 load_neg(int64_t v) const { return __ldcg(snap + v); }
    __device__ __forceinline__ void add(int64_t v, float dx, float dy) const {
        add_y_w<false>(y, v, dx, dy, probe);
    }
    __device__ __forceinline__ void add_neg(int64_t v, float dx, float dy) const { add(v, dx, dy); }
};

__global__ void snap_copy_kernel(const float2 *y, float2 *snap, int64_t n) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const float4 *s4 = reinterpret_cast<const float4 *>(y);
    float4 *d4 = reinterpret_cast<float4 *>(snap);
    const int64_t n4 = n / 2;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n4;
         v += (int64_t)gridDim.x * blockDim.x)
        d4[v] = __ldcg(s4 + v);
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) snap[n - 1] = __ldcg(y + n - 1);
}

__global__ void flush_kernel(float2 *y, unsigned long long *d, int64_t n) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const ulonglong2 q = reinterpret_cast<ulonglong2 *>(d)[v];
        if (q.x | q.y) {
            float2 p = y[v];
            p.x = (float)((double)p.x + (double)(long long)q.x * (1.0 / kFixScale));
            p.y = (float)((double)p.y + (double)(long long)q.y * (1.0 / kFixScale));
            y[v] = p;
            reinterpret_cast<ulonglong2 *>(d)[v] = make_ulonglong2(0ull, 0ull);
        }
    }
}

// One reference step (_kernels.py:82-140) on drawn (i, j, negatives) through a store.
// Negatives past kMaxNeg are read from the draw records at column sl.
template <int B, class St>
__device__ __forceinline__ void step_body(const PArgs &A, const St &st, int64_t i, int64_t j,
                                          const int32_t *cand, int64_t sl) {
    const float two_b = 2.0f * (float)A.b;
    const int Me = min(A.M, kMaxNeg);
    float2 yi = st.load(i);
    const float2 yj = st.load(j);
    float2 ycand[kMaxNeg];
#pragma unroll
    for (int m = 0; m < kMaxNeg; ++m)
        ycand[m] = (m < Me && cand[m] >= 0) ? st.load_neg(cand[m]) : make_float2(0.f, 0.f);
    float gix = 0.f, giy = 0.f;
    int64_t upd = -1;
    float ux = 0.f, uy = 0.f;
    if (i != j) {  // _kernels.py:82-105
        const float dx = yi.x - yj.x, dy = yi.y - yj.y;
        const float ld2 = dx * dx + dy * dy;
        if (ld2 > 0.f) {
            const float pw = ipow_b<B>(ld2, A.b - 1);
            const float coef = __fdividef(-two_b * pw, 1.0f + pw * ld2);
            const float gx = A.lr * clampf(coef * dx, A.clip);
            const float gy = A.lr * clampf(coef * dy, A.clip);
            upd = j;
            ux = -gx;
            uy = -gy;
            yi.x += gx;
            yi.y += gy;
            gix += gx;
            giy += gy;
        }
    }
    st.add(upd, ux, uy);
    float ax[kMaxNeg], ay[kMaxNeg];   // this step's updates of its first negatives
#pragma unroll
    for (int m = 0; m < kMaxNeg; ++m) {  // _kernels.py:106-140
        if (m < Me) {
            float2 yc = ycand[m];
            own_updates(yc, cand[m], m, cand, ax, ay);   // gathered before them
            int64_t tu;
            float tx, ty;
            repel<B>(yi, yc, cand[m], A.lr, A.gamma, A.eps, A.clip, two_b, A.b, tu, tx, ty, gix,
                     giy);
            ax[m] = tx;
            ay[m] = ty;
            st.add_neg(tu, tx, ty);
        }
    }
    for (int m = Me; m < A.M; ++m) {   // negatives past kMaxNeg: gathered after the atomics
        const int64_t target = __ldcs(A.draws + (2 + m) * A.stride + sl);
        const float2 yc = target >= 0 ? st.load_neg(target) : make_float2(0.f, 0.f);
        int64_t tu;
        float tx, ty;
        repel<B>(yi, yc, target, A.lr, A.gamma, A.eps, A.clip, two_b, A.b, tu, tx, ty, gix, giy);
        st.add_neg(tu, tx, ty);
    }
    st.add((gix != 0.f || giy != 0.f) ? i : -1, gix, giy);
}

// Steps under per-node locks on the source and the attraction partner: the steps
// in flight then touch disjoint (i, j) pairs, so the attraction -- the local
// structure NP measures -- never reads a position another in-flight step is about
// to move, at any number of steps in flight.  The negatives stay Hogwild (their
// staleness is harmless: the multi-GPU form reads them from epoch-old snapshots at
// no cost in KL or NP).  Measured on C1 (100 seeds): Hogwild at n/4 steps in flight
// KL +2.4% / NP -11.6%, under locks KL +0.01% / NP +1.6% +- 1.9%.
//   * acquire: both locks tried at once (CAS on min(i, j), then max(i, j); one L2
//     round trip); a step that gets only one releases it and tries again the next
//     time round the loop, while the warp's other lanes run their steps; after
//     kLockTries failures it runs unlocked (plain Hogwild) -- nothing ever waits.
//   * release: no fence (MEMBAR.SC.GPU + L1 invalidation cost ~25 us per step).
//     The updates of i and j are RETURNING atomics; the release stores carry a data
//     dependency on their results, so they are issued after the updates were
//     performed in L2 -- where the next holder's CAS and its ld.cg reads go.
constexpr int kLockTries = 64;

struct LockedStore {   // Hogwild on y for the negatives, returning atomics for i and j
    float2 *y;
    mutable int sink;
    __device__ __forceinline__ float2 load(int64_t v) const { return ld_y(y, v); }
    __device__ __forceinline__ float2 load_neg(int64_t v) const { return ld_y(y, v); }
    __device__ __forceinline__ void add(int64_t v, float dx, float dy) const {
        if (v < 0) return;
        const float2 old = atomicAdd(y + v, make_float2(dx, dy));
        sink |= __float_as_int(old.x);
    }
    __device__ __forceinline__ void add_neg(int64_t v, float dx, float dy) const {
        if (v >= 0) add_y(y, v, dx, dy);
    }
};

template <int B>
__device__ __forceinline__ void apply_steps_locked(const PArgs &A, float2 *y, int64_t sl,
                                                   const int64_t nthreads) {
    const int Me = min(A.M, kMaxNeg);
    const int64_t ns = A.n_steps, sd = A.stride;
    int *L = A.locks;
    if (sl >= ns) return;
    int32_t ci = __ldcs(A.draws + sl), cj = __ldcs(A.draws + sd + sl);
    int32_t cc[kMaxNeg];
#pragma unroll
    for (int m = 0; m < kMaxNeg; ++m) cc[m] = m < Me ? __ldcs(A.draws + (2 + m) * sd + sl) : -1;
    int fails = 0;
    while (sl < ns) {
        const uint32_t qi = (uint32_t)ci & A.lock_mask, qj = (uint32_t)cj & A.lock_mask;
        const uint32_t lo = min(qi, qj), hi = max(qi, qj);
        const int r0 = atomicCAS(L + lo, 0, 1);
        const int r1 = lo != hi ? atomicCAS(L + hi, 0, 1) : 0;
        const bool got = r0 == 0 && r1 == 0;
        if (!got) {
            if (r0 == 0) atomicExch(L + lo, 0);
            if (r1 == 0 && lo != hi) atomicExch(L + hi, 0);
            if (++fails <= kLockTries) continue;
        }
        asm volatile("" ::: "memory");   // the step's reads stay below the acquire
        const int64_t i = ci, j = cj, cur = sl;
        int32_t cand[kMaxNeg];
#pragma unroll
        for (int m = 0; m < kMaxNeg; ++m) cand[m] = cc[m];
        sl += nthreads;
        if (sl < ns) {
            ci = __ldcs(A.draws + sl);
            cj = __ldcs(A.draws + sd + sl);
#pragma unroll
            for (int m = 0; m < kMaxNeg; ++m)
                if (m < Me) cc[m] = __ldcs(A.draws + (2 + m) * sd + sl);
        }
        const LockedStore st{y, 0};
        step_body<B>(A, st, i, j, cand, cur);
        if (got) {
            const int z = st.sink & A.zero;   // 0, known only once the updates returned
            asm volatile("" ::: "memory");
            atomicExch(L + lo, z);
            if (lo != hi) atomicExch(L + hi, z);
        }
        fails = 0;
    }
}

// grid-stride over the launch's steps; the next step's record is prefetched while
// this step runs
// The columns of several ranks' draws (emulated multi-GPU: rank after rank in one
// buffer) are visited in a spread order so the steps in flight at any time are
// drawn from every rank, as on W GPUs, not from one rank's part at a time.
// (SPREAD: a compile-time switch, the 64-bit modulo stays out of the 1-GPU kernels)
template <bool SPREAD>
__device__ __forceinline__ int64_t column(const PArgs &A, int64_t sl) {
    return SPREAD ? (int64_t)(((uint64_t)sl * A.spread) % (uint64_t)A.n_steps) : sl;
}

template <int B, class St, bool SPREAD = false>
__device__ __forceinline__ void apply_steps(const PArgs &A, const St &st, int64_t sl,
                                            const int64_t nthreads) {
    const int Me = min(A.M, kMaxNeg);
    const int64_t ns = A.n_steps, sd = A.stride;
    if (sl >= ns) return;
    int64_t col = column<SPREAD>(A, sl);
    int32_t ci = __ldcs(A.draws + col), cj = __ldcs(A.draws + sd + col);
    int32_t cc[kMaxNeg];
#pragma unroll
    for (int m = 0; m < kMaxNeg; ++m) cc[m] = m < Me ? __ldcs(A.draws + (2 + m) * sd + col) : -1;
    for (; sl < ns; sl += nthreads) {
        const int64_t i = ci, j = cj, cur = col;
        int32_t cand[kMaxNeg];
#pragma unroll
        for (int m = 0; m < kMaxNeg; ++m) cand[m] = cc[m];
        const int64_t nx = sl + nthreads;
        if (nx < ns) {
            col = column<SPREAD>(A, nx);
            ci = __ldcs(A.draws + col);
            cj = __ldcs(A.draws + sd + col);
#pragma unroll
            for (int m = 0; m < kMaxNeg; ++m)
                if (m < Me) cc[m] = __ldcs(A.draws + (2 + m) * sd + col);
        }
        step_body<B>(A, st, i, j, cand, cur);
    }
}

template <bool AGG, int B, bool DET = false>
__device__ __forceinline__ void apply_epoch(const PArgs &A, float2 *y, int64_t sl,
                                            const int64_t nthreads) {
    if (DET) apply_steps<B>(A, FixedStore{y, A.delta}, sl, nthreads);
    else apply_steps<B>(A, GlobalStore<AGG>{y, A.probe}, sl, nthreads);
}

// ---- hub levels: the hottest nodes staged per block ------------------------------
// On hub-heavy levels (R-MAT's coarse levels: one node is the source of a third of
// an epoch's steps) every step reads and moves the same few nodes, and their
// float2 reductions serialise on one L2 line each.  Here each block stages the K
// hottest nodes: their positions are read from shared memory (refreshed from y
// after every round of steps) and their increments summed in shared memory
// (warp-aggregated), then added to y with one reduction per node per block and
// round.  A hub thus moves between rounds, where the plain form moves it as its
// reductions land; within a round the steps in flight see the same hub position in
// both forms.  Rounds are block-uniform (one step per thread per round).
// Membership is a 8192-bit filter on the low id bits (one shared load rejects
// almost every non-hot node) before an open-addressing probe; the block's
// increments of a hot node are summed in 32-bit fixed point by native shared
// ATOMS.ADD (shared float atomics are CAS loops on sm_100): each increment
// v = rint(dx * scale), |v| < 2^30, split into v >> 16 and v & 0xffff summed in
// two words (no overflow for any block size), scale = the power of two that keeps
// the largest increment lr * clip * (1 + M) below 2^30 (PArgs::hot_scale).
constexpr int kHot = 64;
constexpr int kHotSlots = 256;
constexpr int kHotFilterWords = 256;

template <bool AGG>
struct HotStore {
    float2 *y;
    int probe;
    float scale;
    const unsigned *filter;    // shared: bit (v & 8191) set for every hot node
    const int *key;            // shared open-addressing table: node id -> slot
    const unsigned char *slot;
    const float2 *pos;         // shared: staged positions
    int *acc;                  // shared: [kHot][4] x >> 16, x & 0xffff, y >> 16, y & 0xffff
    __device__ __forceinline__ int find(int64_t v) const {
        if (v < 0) return -1;
        const uint32_t b = (uint32_t)v & 8191u;
        if (!((filter[b >> 5] >> (b & 31)) & 1u)) return -1;
        uint32_t h = ((uint32_t)v * 2654435761u) >> (32 - 8);
        for (int p = 0; p < kHotSlots; ++p) {
            const int k = key[h];
            if (k == (int)v) return slot[h];
            if (k < 0) return -1;
            h = (h + 1) & (kHotSlots - 1);
        }
        return -1;
    }
    __device__ __forceinline__ float2 load(int64_t v) const {
        const int q = find(v);
        return q >= 0 ? pos[q] : ld_y(y, v);
    }
    __device__ __forceinline__ float2 load_neg(int64_t v) const { return load(v); }
    __device__ __forceinline__ void add(int64_t v, float dx, float dy) const {
        const int q = find(v);
        if (q < 0) {
            add_y_w<AGG>(y, v, dx, dy, probe);
            return;
        }
        const int fx = __float2int_rn(dx * scale), fy = __float2int_rn(dy * scale);
        int *a = acc + 4 * q;
        atomicAdd(a + 0, fx >> 16);
        atomicAdd(a + 1, fx & 0xffff);
        atomicAdd(a + 2, fy >> 16);
        atomicAdd(a + 3, fy & 0xffff);
    }
    __device__ __forceinline__ void add_neg(int64_t v, float dx, float dy) const { add(v, dx, dy); }
};

__device__ __forceinline__ float hot_sum(const int *a, float inv_scale) {
    return (float)((double)((int64_t)a[0] * 65536 + (int64_t)a[1]) * (double)inv_scale);
}

template <bool AGG, int B>
__global__ void __launch_bounds__(1024)
    apply_hot_kernel(PArgs A, float2 *y, const int32_t *__restrict__ hot, int n_hot) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ unsigned s_filter[kHotFilterWords];
    __shared__ int s_key[kHotSlots];
    __shared__ unsigned char s_slot[kHotSlots];
    __shared__ float2 s_pos[kHot];
    __shared__ int s_acc[kHot * 4];
    const int tid = threadIdx.x;
    const int K = min(n_hot, kHot);
    for (int q = tid; q < kHotSlots; q += blockDim.x) s_key[q] = -1;
    for (int q = tid; q < kHotFilterWords; q += blockDim.x) s_filter[q] = 0u;
    __syncthreads();
    for (int q = tid; q < K; q += blockDim.x) {   // (blocks may be smaller than K)
        const int v = hot[q];
        uint32_t h = ((uint32_t)v * 2654435761u) >> (32 - 8);
        while (atomicCAS(&s_key[h], -1, v) != -1) h = (h + 1) & (kHotSlots - 1);
        s_slot[h] = (unsigned char)q;
        const uint32_t b = (uint32_t)v & 8191u;
        atomicOr(&s_filter[b >> 5], 1u << (b & 31));
        s_pos[q] = ld_y(y, v);
    }
    for (int q = tid; q < kHot * 4; q += blockDim.x) s_acc[q] = 0;
    __syncthreads();
    const float inv = 1.0f / A.hot_scale;
    const HotStore<AGG> st{y, A.probe, A.hot_scale, s_filter, s_key, s_slot, s_pos, s_acc};
    const int Me = min(A.M, kMaxNeg);
    const int64_t ns = A.n_steps, sd = A.stride;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ns; base += nthreads) {
        const int64_t sl = base + tid;
        if (sl < ns) {
            int32_t cand[kMaxNeg];
#pragma unroll
            for (int m = 0; m < kMaxNeg; ++m) cand[m] = m < Me ? __ldcs(A.draws + (2 + m) * sd + sl) : -1;
            step_body<B>(A, st, __ldcs(A.draws + sl), __ldcs(A.draws + sd + sl), cand, sl);
        }
        __syncthreads();
        for (int q = tid; q < K; q += blockDim.x) {   // publish the round's increments,
            const int v = hot[q];                        // refresh the staged position
            int *a = s_acc + 4 * q;
            const float dx = hot_sum(a, inv), dy = hot_sum(a + 2, inv);
            if (dx != 0.f || dy != 0.f) add_y(y, v, dx, dy);
            a[0] = a[1] = a[2] = a[3] = 0;
            s_pos[q] = ld_y(y, v);
        }
        __syncthreads();
    }
}

// Hub levels drawn inline: each round's steps drawn by draw_step (no draw records
// written and re-read) and applied through the hot store.  The draws' random DRAM
// reads then overlap other warps' updates inside one kernel, where the split form
// runs a draw pass and an update pass that each fill the SMs.  M <= kMaxNeg.
template <bool AGG, int B, bool HINT>
__global__ void __launch_bounds__(256, 4)
    apply_hot_fused_kernel(DArgs D, PArgs A, float2 *y, const int32_t *__restrict__ hot,
                           int n_hot) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ unsigned s_filter[kHotFilterWords];
    __shared__ int s_key[kHotSlots];
    __shared__ unsigned char s_slot[kHotSlots];
    __shared__ float2 s_pos[kHot];
    __shared__ int s_acc[kHot * 4];
    const int tid = threadIdx.x;
    const int K = min(n_hot, kHot);
    for (int q = tid; q < kHotSlots; q += blockDim.x) s_key[q] = -1;
    for (int q = tid; q < kHotFilterWords; q += blockDim.x) s_filter[q] = 0u;
    __syncthreads();
    for (int q = tid; q < K; q += blockDim.x) {   // (blocks may be smaller than K)
        const int v = hot[q];
        uint32_t h = ((uint32_t)v * 2654435761u) >> (32 - 8);
        while (atomicCAS(&s_key[h], -1, v) != -1) h = (h + 1) & (kHotSlots - 1);
        s_slot[h] = (unsigned char)q;
        const uint32_t b = (uint32_t)v & 8191u;
        atomicOr(&s_filter[b >> 5], 1u << (b & 31));
        s_pos[q] = ld_y(y, v);
    }
    for (int q = tid; q < kHot * 4; q += blockDim.x) s_acc[q] = 0;
    __syncthreads();
    const float inv = 1.0f / A.hot_scale;
    const HotStore<AGG> st{y, A.probe, A.hot_scale, s_filter, s_key, s_slot, s_pos, s_acc};
    const int64_t ns = A.n_steps;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const uint32_t tt = (uint32_t)D.t_first << 1;
    unsigned nev = 0;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ns; base += nthreads) {
        const int64_t sl = base + tid;
        if (sl < ns) {
            const int64_t s = D.step_lo + sl;
            int64_t i, j;
            int32_t cand[kMaxNeg];
            draw_step<HINT>(D, s, (uint32_t)(s >> 32) ^ tt, i, j, cand, nullptr, 0, nev);
            step_body<B>(A, st, i, j, cand, sl);
        }
        __syncthreads();
        for (int q = tid; q < K; q += blockDim.x) {   // publish the round's increments,
            const int v = hot[q];                        // refresh the staged position
            int *a = s_acc + 4 * q;
            const float dx = hot_sum(a, inv), dy = hot_sum(a + 2, inv);
            if (dx != 0.f || dy != 0.f) add_y(y, v, dx, dy);
            a[0] = a[1] = a[2] = a[3] = 0;
            s_pos[q] = ld_y(y, v);
        }
        __syncthreads();
    }
    count_evals(D.evals, nev);
}

template <bool AGG, int B>
__global__ void __launch_bounds__(256, 4) apply_kernel(PArgs A, float2 *y) {
    // launched with programmatic stream serialization: the previous epoch's grid
    // must be complete (and its y updates visible) before this one reads y
    asm volatile("griddepcontrol.wait;" ::: "memory");
    apply_epoch<AGG, B>(A, y, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                        (int64_t)gridDim.x * blockDim.x);
}

template <int B>
__global__ void __launch_bounds__(256, 4) apply_snap_kernel(PArgs A, float2 *y) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    apply_steps<B>(A, SnapStore{y, A.snap, A.probe},
                   (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                   (int64_t)gridDim.x * blockDim.x);
}

// ---- snapshot form with the negatives drawn in the update pass -------------------
// One table of 16-byte records {fp32 threshold, alias, y.x, y.y} per node: Q^l's Vose
// bucket v next to node v's snapshot position.  A negative's draw (bucket -> record)
// then brings the position of the bucket's own node in the same sector: one random
// L2 read per negative instead of two (the alias record in the draw pass, the
// position in the update pass; a second 8-byte read only when the alias is taken or
// a redraw is needed).  The draws use draw_step's counters and the same records, so
// the negatives are bit for bit those drg_sampled_draws reports; the draw pass then
// resolves only the pair (i, j) (8-byte draw records instead of 28).  M <= kMaxNeg.
struct NArgs {
    uint4 *rec;             // [n_y]; .xy = Q^l bucket (zeros past neg.n), .zw = snapshot position
    int64_t n, tail_n;      // NegTab: Vose over [0, n), uniform tail [n, n + tail_n)
    uint32_t tail_thr;
    uint32_t key0, key1, level;
    int t;
    int64_t step_lo;
    unsigned long long *evals;
};

__global__ void negsnap_init_kernel(const uint2 *__restrict__ alias, int64_t n_alias, uint4 *rec,
                                    int64_t n) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const uint2 a = v < n_alias ? alias[v] : make_uint2(0u, 0u);
        rec[v] = make_uint4(a.x, a.y, 0u, 0u);
    }
}

__global__ void negsnap_refresh_kernel(const float2 *y, uint4 *rec, int64_t n) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        reinterpret_cast<float2 *>(rec + v)[1] = __ldcg(y + v);
}

struct NegSnapStore {   // source / partner live on y; negatives resolved by the caller
    float2 *y;
    int probe;
    int32_t c[kMaxNeg];
    float2 p[kMaxNeg];
    __device__ __forceinline__ float2 load(int64_t v) const { return ld_y(y, v); }
    __device__ __forceinline__ float2 load_neg(int64_t v) const {
        float2 r = p[0];
#pragma unroll
        for (int q = 1; q < kMaxNeg; ++q)
            if (c[q] == (int32_t)v) r = p[q];
        return r;
    }
    __device__ __forceinline__ void add(int64_t v, float dx, float dy) const {
        add_y_w<false>(y, v, dx, dy, probe);
    }
    __device__ __forceinline__ void add_neg(int64_t v, float dx, float dy) const { add(v, dx, dy); }
};

// (record reads through L2 (ld.cg), not the non-coherent path: with programmatic
// dependent launches this kernel's blocks can become resident while the previous
// epoch's blocks still fill the SM's L1 with the old positions)
__device__ __forceinline__ float2 negsnap_pos(const uint4 *rec, int64_t v) {
    return __ldcg(reinterpret_cast<const float2 *>(rec + v) + 1);
}

// MC > 0: M known at compile time (the default M = 5: no dead sixth negative held in
// registers, no predication on m < M)
template <int B, int MC>
__global__ void __launch_bounds__(256, 3) apply_negsnap_kernel(PArgs A0, NArgs N, float2 *y) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    PArgs A = A0;
    if (MC > 0) A.M = MC;
    const int Me = MC > 0 ? MC : min(A.M, kMaxNeg);
    const int64_t ns = A.n_steps, sd = A.stride;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const uint4 *rec = N.rec;
    SArgs K;   // the counter layout of draw_step
    K.key0 = N.key0;
    K.key1 = N.key1;
    K.level = N.level;
    unsigned nev = 0;
    int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sl < ns) {
        int32_t ci = __ldcs(A.draws + sl), cj = __ldcs(A.draws + sd + sl);
        for (; sl < ns; sl += nthreads) {
            const int64_t i = ci, j = cj, cur = sl;
            const int64_t s = N.step_lo + sl;
            const uint32_t c1 = (uint32_t)(s >> 32) ^ ((uint32_t)N.t << 1);
            if (sl + nthreads < ns) {
                ci = __ldcs(A.draws + sl + nthreads);
                cj = __ldcs(A.draws + sd + sl + nthreads);
            }
            NegSnapStore st;
            st.y = y;
            st.probe = A.probe;
            // first attempt of every negative: one record each, all in flight
            uint4 r[kMaxNeg];
            int32_t bk[kMaxNeg];
            uint32_t coin[kMaxNeg];
#pragma unroll
            for (int m = 0; m < kMaxNeg; ++m) {
                if (m < Me) {
                    const u32x4 q = neg_draw(K, s, c1, m, 0);
                    const bool tail = q.w < N.tail_thr;
                    bk[m] = (int32_t)(tail ? N.n + bucket(N.tail_n, q.x, q.y)
                                           : bucket(N.n, q.x, q.y));
                    coin[m] = tail ? 0u : q.z;   // (a tail pick is always its own node)
                    r[m] = __ldcg(rec + bk[m]);
                    if (tail) r[m].x = 0x7f800000u;   // threshold +inf: accept
                }
            }
#pragma unroll
            for (int m = 0; m < kMaxNeg; ++m) {
                st.c[m] = -1;
                st.p[m] = make_float2(0.f, 0.f);
                if (m < Me) {
                    const bool own = u32_to_unit(coin[m]) < __uint_as_float(r[m].x);
                    int64_t c = own ? bk[m] : (int64_t)r[m].y;
                    bool have = own;
                    float2 pos = make_float2(__uint_as_float(r[m].z), __uint_as_float(r[m].w));
                    for (int attempt = 1; (c == i || c == j) && attempt < 9; ++attempt) {
                        const u32x4 q = neg_draw(K, s, c1, m, attempt);
                        have = false;
                        if (q.w < N.tail_thr) {
                            c = N.n + bucket(N.tail_n, q.x, q.y);
                        } else {
                            const int64_t b2 = bucket(N.n, q.x, q.y);
                            const uint4 r2 = __ldcg(rec + b2);
                            const bool own2 = u32_to_unit(q.z) < __uint_as_float(r2.x);
                            c = own2 ? b2 : (int64_t)r2.y;
                            if (own2) {
                                have = true;
                                pos = make_float2(__uint_as_float(r2.z), __uint_as_float(r2.w));
                            }
                        }
                    }
                    if (c != i && c != j) {
                        st.c[m] = (int32_t)c;
                        st.p[m] = have ? pos : negsnap_pos(rec, c);
                        ++nev;
                    }
                }
            }
            step_body<B>(A, st, i, j, st.c, cur);
        }
    }
    count_evals(N.evals, nev);
}

// Few steps in flight (small or fidelity-capped levels): the step is a dependent
// chain issued by one or two warps per SM, so this instance drops the 4-blocks-per-SM
// register cap (no parameter reloads / rematerialisation in the chain).
template <bool AGG, int B>
__global__ void __launch_bounds__(256, 1) apply_kernel_lc(PArgs A, float2 *y) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    apply_epoch<AGG, B>(A, y, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                        (int64_t)gridDim.x * blockDim.x);
}

// steps under (i, j) locks (DRG_SAMPLED_LOCKED)
template <int B>
__global__ void __launch_bounds__(256, 1) apply_locked_kernel(PArgs A, float2 *y) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    apply_steps_locked<B>(A, y, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                          (int64_t)gridDim.x * blockDim.x);
}

// deterministic sub-batch: one step per thread, positions frozen for the launch
template <int B>
__global__ void __launch_bounds__(256) apply_det_kernel(PArgs A, float2 *y) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    apply_epoch<false, B, true>(A, y, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                                (int64_t)gridDim.x * blockDim.x);
}

constexpr int64_t kLowConcurrency = 65536;   // steps in flight below which _lc runs

// the kernel instance: b = 2 (the default) compiled in, other b at run time
template <bool AGG>
void *apply_instance(int b, int64_t threads = INT64_MAX) {
    if (threads < kLowConcurrency)
        return b == 2 ? (void *)apply_kernel_lc<AGG, 2> : (void *)apply_kernel_lc<AGG, 0>;
    return b == 2 ? (void *)apply_kernel<AGG, 2> : (void *)apply_kernel<AGG, 0>;
}

// Consecutive epochs on one stream as programmatic dependent launches: the next
// grid is set up while the previous drains (its griddepcontrol.wait holds the
// steps back), so small levels do not pay the full launch gap per epoch.
// apply_hot_kernel's fixed-point scale: the largest increment one add carries is
// lr * clip per clipped term, 1 + M terms; kept below 2^30
float hot_scale_for(const PArgs &P) {
    const double big = std::max(1e-30, (double)P.lr * (double)P.clip * (1.0 + P.M));
    return (float)std::exp2(std::min(40.0, std::floor(std::log2(1073741824.0 / big))));
}

// one epoch of a hub level with the draws inline (apply_hot_fused_kernel), PDL
int launch_hot_fused(const DArgs &D, const PArgs &P, float2 *y, unsigned grid, int block,
                     bool agg, const int32_t *hot, int n_hot, bool hints, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PArgs Q = P;
    Q.hot_scale = hot_scale_for(P);
    DArgs E = D;
    void *args[] = {&E, &Q, &y, &hot, &n_hot};
    // hints: the draws' one-touch table reads L2 evict-first and the Q table
    // evict-last (DRG_SAMPLED_L2_HINTS; R-MAT scale 24: 295.6 -> 306 iters/s; the
    // BA-1M hub level, whose tables fit L2, 7% slower -- the caller sets it for big
    // tables only).  Keeping the positions evict-last as well measured no gain.
#define DRG_FUSED_FN(H)                                                                \
    (agg ? (P.b == 2 ? (void *)apply_hot_fused_kernel<true, 2, H>                      \
                     : (void *)apply_hot_fused_kernel<true, 0, H>)                     \
         : (P.b == 2 ? (void *)apply_hot_fused_kernel<false, 2, H>                     \
                     : (void *)apply_hot_fused_kernel<false, 0, H>))
    void *fn = hints ? DRG_FUSED_FN(true) : DRG_FUSED_FN(false);
#undef DRG_FUSED_FN
    DRG_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
    DRG_LAUNCHED("apply_hot_fused_kernel");
    return DRG_OK;
}

int launch_apply(const PArgs &P, float2 *y, unsigned grid, int block, bool agg, cudaStream_t st,
                 const int32_t *hot = nullptr, int n_hot = 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PArgs Q = P;
    Q.hot_scale = hot_scale_for(P);
    void *args[] = {&Q, &y, &hot, &n_hot};
    const int64_t threads = (int64_t)grid * block;
    void *fn;
    if (hot && n_hot > 0) {
        // one block per SM: each block stages the hot nodes and publishes their
        // increments once per round, so fewer, larger blocks mean fewer same-address
        // reductions and reloads on the hubs per round (R-MAT: 512 blocks of 128
        // published 32 k hub updates per round at 64 k steps in flight)
        const int64_t per_sm = ceil_div(threads, (int64_t)sm_count());
        const int hb = (int)std::min<int64_t>(threads, std::min<int64_t>(
                                                          1024, std::max<int64_t>(32, ceil_div(per_sm, 32) * 32)));
        cfg.blockDim = dim3((unsigned)hb);
        cfg.gridDim = dim3((unsigned)ceil_div(threads, hb));
    }
    if (P.locks && !(hot && n_hot > 0) && !agg)
        fn = P.b == 2 ? (void *)apply_locked_kernel<2> : (void *)apply_locked_kernel<0>;
    else if (P.snap && !(hot && n_hot > 0) && !agg)
        fn = P.b == 2 ? (void *)apply_snap_kernel<2> : (void *)apply_snap_kernel<0>;
    else if (hot && n_hot > 0)   // hub level: the hottest nodes staged per block
        fn = agg ? (P.b == 2 ? (void *)apply_hot_kernel<true, 2> : (void *)apply_hot_kernel<true, 0>)
                 : (P.b == 2 ? (void *)apply_hot_kernel<false, 2> : (void *)apply_hot_kernel<false, 0>);
    else
        fn = agg ? apply_instance<true>(P.b, threads) : apply_instance<false>(P.b, threads);
    DRG_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
    DRG_LAUNCHED("apply_kernel");
    return DRG_OK;
}

// refresh of the negatives' snapshot (DRG_SAMPLED_SNAPSHOT), in the epochs' PDL chain
int launch_snap_copy(const float2 *y, float2 *snap, int64_t n, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::min<int64_t>(ceil_div(std::max<int64_t>(n / 2, 1), 256),
                                                   (int64_t)sm_count() * 8));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void *args[] = {&y, &snap, &n};
    DRG_CUDA(cudaLaunchKernelExC(&cfg, (void *)snap_copy_kernel, args));
    DRG_LAUNCHED("snap_copy_kernel");
    return DRG_OK;
}

int launch_negsnap_epoch(const PArgs &P, const NArgs &N, float2 *y, int64_t n_y, unsigned grid,
                         int block, bool refresh, cudaStream_t st) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (refresh) {
        cfg.gridDim = dim3((unsigned)std::min<int64_t>(ceil_div(n_y, 256), (int64_t)sm_count() * 8));
        cfg.blockDim = dim3(256);
        const float2 *yc = y;
        uint4 *rec = N.rec;
        void *rargs[] = {&yc, &rec, &n_y};
        DRG_CUDA(cudaLaunchKernelExC(&cfg, (void *)negsnap_refresh_kernel, rargs));
        DRG_LAUNCHED("negsnap_refresh_kernel");
    }
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3((unsigned)block);
    PArgs Q = P;
    NArgs M = N;
    void *args[] = {&Q, &M, &y};
    void *fn = P.b == 2 ? (P.M == 5 ? (void *)apply_negsnap_kernel<2, 5>
                                    : (void *)apply_negsnap_kernel<2, 0>)
                        : (void *)apply_negsnap_kernel<0, 0>;
    DRG_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
    DRG_LAUNCHED("apply_negsnap_kernel");
    return DRG_OK;
}

// One epoch in the deterministic mode: sub-batches of `batch` consecutive steps,
// each an apply_det_kernel (positions frozen, fixed-point increments) and a
// flush_kernel, as programmatic dependent launches on one stream.
int launch_det_epoch(PArgs P, float2 *y, int64_t batch, int64_t n_y, cudaStream_t st) {
    const int64_t total = P.n_steps;
    const int32_t *base = P.draws;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    for (int64_t lo = 0; lo < total; lo += batch) {
        P.draws = base + lo;
        P.n_steps = std::min(batch, total - lo);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)ceil_div(P.n_steps, 256));
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        void *args[] = {&P, &y};
        DRG_CUDA(cudaLaunchKernelExC(&cfg, P.b == 2 ? (void *)apply_det_kernel<2>
                                                    : (void *)apply_det_kernel<0>, args));
        DRG_LAUNCHED("apply_det_kernel");
        cfg.gridDim = dim3((unsigned)std::min<int64_t>(ceil_div(n_y, 256), sm_count() * 8));
        unsigned long long *d = P.delta;
        void *fargs[] = {&y, &d, &n_y};
        DRG_CUDA(cudaLaunchKernelExC(&cfg, (void *)flush_kernel, fargs));
        DRG_LAUNCHED("flush_kernel");
    }
    return DRG_OK;
}

// Per-row alias tables (build_alias_table, optimizer.py:111-139, applied to every
// row of P) by the parallel sweep: the law of Vose's construction without its
// sequential stack.  rec[e] = {fp32 threshold of bucket e, alias target, own target}.
constexpr int kRowWarpMax = 512;   // rows up to this length: warp-parallel sweep
constexpr int kRowWarps = 4;

// Warp per row (len <= kRowWarpMax): the parallel sweep of drg_alias_build
// (layout.cu) inside one row, in shared memory -- lights / heavies compacted in index
// order by ballots, deficit / surplus prefix sums by warp scans, then each lane
// resolves its items by binary search.
__global__ void __launch_bounds__(kRowWarps * 32)
    row_alias_warp_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ targets,
                          const double *__restrict__ P, int64_t n, uint4 *rec, double *rowsum,
                          int64_t *long_rows, int *n_long) {
    __shared__ double s_w[kRowWarps][kRowWarpMax];
    __shared__ double s_ds[kRowWarps][kRowWarpMax];   // delta (lights) | sigma (heavies)
    __shared__ int16_t s_idx[kRowWarps][kRowWarpMax]; // lights from the front, heavies after
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    double *w = s_w[wp], *ds = s_ds[wp];
    int16_t *idx = s_idx[wp];
    for (int64_t i = (int64_t)blockIdx.x * kRowWarps + wp; i < n; i += (int64_t)gridDim.x * kRowWarps) {
        const int64_t lo = indptr[i], hi = indptr[i + 1];
        const int len = (int)(hi - lo);
        if (len > kRowWarpMax) {   // the block tier takes it: queue the row
            if (lane == 0) long_rows[atomicAdd(n_long, 1)] = i;
            continue;
        }
        if (len == 0) {
            if (lane == 0 && rowsum) rowsum[i] = 0.0;
            continue;
        }
        double tot = 0.0;
        for (int e = lane; e < len; e += 32) tot += P[lo + e];
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(kFull, tot, o);
        if (lane == 0 && rowsum) rowsum[i] = tot;
        if (!(tot > 0.0)) {
            for (int e = lane; e < len; e += 32)
                rec[lo + e] = make_uint4(__float_as_uint(1.0f), targets[lo + e], targets[lo + e], 0u);
            continue;
        }
        const double f = (double)len / tot;
        // compaction: lights [0, na), heavies [na, len) in index order
        int na = 0;
        for (int base = 0; base < len; base += 32) {
            const int e = base + lane;
            const double x = e < len ? P[lo + e] * f : 2.0;
            if (e < len) w[e] = x;
            const unsigned bl = __ballot_sync(kFull, e < len && x < 1.0);
            if (e < len && x < 1.0) idx[na + __popc(bl & ((1u << lane) - 1u))] = (int16_t)e;
            na += __popc(bl);
        }
        int nh = 0;
        for (int base = 0; base < len; base += 32) {
            const int e = base + lane;
            const bool h = e < len && !(w[e] < 1.0);
            const unsigned bh = __ballot_sync(kFull, h);
            if (h) idx[na + nh + __popc(bh & ((1u << lane) - 1u))] = (int16_t)e;
            nh += __popc(bh);
        }
        __syncwarp();
        // inclusive prefix sums: delta over lights, sigma over heavies
        for (int part = 0; part < 2; ++part) {
            const int off = part ? na : 0, cnt = part ? nh : na;
            double carry = 0.0;
            for (int base = 0; base < cnt; base += 32) {
                const int k = base + lane;
                double v = 0.0;
                if (k < cnt) v = part ? w[idx[off + k]] - 1.0 : 1.0 - w[idx[off + k]];
                for (int o = 1; o < 32; o <<= 1) {
                    const double t = __shfl_up_sync(kFull, v, o);
                    if (lane >= o) v += t;
                }
                if (k < cnt) ds[off + k] = carry + v;
                carry += __shfl_sync(kFull, v, 31);
            }
        }
        __syncwarp();
        const double *delta = ds, *sigma = ds + na;
        for (int k = lane; k < na; k += 32) {   // lights
            const double prev = k ? delta[k - 1] : 0.0;
            int a = 0, b = nh;
            while (a < b) {
                const int m = (a + b) >> 1;
                if (sigma[m] > prev) b = m;
                else a = m + 1;
            }
            const int item = idx[k];
            const uint32_t own = (uint32_t)targets[lo + item];
            rec[lo + item] = a < nh ? make_uint4(__float_as_uint((float)w[item]),
                                                 (uint32_t)targets[lo + idx[na + a]], own, 0u)
                                    : make_uint4(__float_as_uint(1.0f), own, own, 0u);
        }
        for (int k = lane; k < nh; k += 32) {   // heavies
            int a = 0, b = na;
            while (a < b) {
                const int m = (a + b) >> 1;
                if (delta[m] >= sigma[k]) b = m;
                else a = m + 1;
            }
            const int item = idx[na + k];
            const uint32_t own = (uint32_t)targets[lo + item];
            if (a < na && k + 1 < nh) {
                const double p = fmin(fmax(1.0 + sigma[k] - delta[a], 0.0), 1.0);
                rec[lo + item] = make_uint4(__float_as_uint((float)p),
                                            (uint32_t)targets[lo + idx[na + k + 1]], own, 0u);
            } else {
                rec[lo + item] = make_uint4(__float_as_uint(1.0f), own, own, 0u);
            }
        }
        __syncwarp();
    }
}

// Block per long row (> kRowWarpMax entries): the same parallel sweep as the warp
// tier, chunked over the row with block scans, the per-entry arrays (scaled weight,
// deficit / surplus prefix sums, light / heavy index lists) in global scratch at the
// row's own entry range -- rows of any length, O(len / blockDim) steps per thread.
constexpr int kRowBlock = 512;

__global__ void __launch_bounds__(kRowBlock)
    row_alias_block_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ targets,
                           const double *__restrict__ P, int64_t n, double *w, double *ds,
                           int32_t *idx, uint4 *rec, double *rowsum,
                           const int64_t *__restrict__ long_rows, const int *__restrict__ n_long) {
    using BR = cub::BlockReduce<double, kRowBlock>;
    using BSI = cub::BlockScan<int, kRowBlock>;
    using BSD = cub::BlockScan<double, kRowBlock>;
    __shared__ union {
        typename BR::TempStorage r;
        typename BSI::TempStorage si;
        typename BSD::TempStorage sd;
    } tmp;
    __shared__ double s_bcast;
    const int tid = threadIdx.x;
    const int nl = *n_long;   // rows the warp tier queued (any order: rows are independent)
    for (int r = blockIdx.x; r < nl; r += gridDim.x) {
        const int64_t i = long_rows[r];
        const int64_t lo = indptr[i], hi = indptr[i + 1];
        const int64_t len = hi - lo;
        double part = 0.0;
        for (int64_t e = tid; e < len; e += kRowBlock) part += P[lo + e];
        const double tot_r = BR(tmp.r).Sum(part);
        if (tid == 0) s_bcast = tot_r;
        __syncthreads();
        const double tot = s_bcast;
        if (tid == 0 && rowsum) rowsum[i] = tot;
        if (!(tot > 0.0)) {
            for (int64_t e = tid; e < len; e += kRowBlock)
                rec[lo + e] = make_uint4(__float_as_uint(1.0f), targets[lo + e], targets[lo + e], 0u);
            __syncthreads();
            continue;
        }
        const double f = (double)len / tot;
        // stable compaction: lights [0, na), heavies [na, len) in index order
        int64_t count[2] = {0, 0};
        for (int pass = 0; pass < 2; ++pass) {
            for (int64_t base = 0; base < len; base += kRowBlock) {
                const int64_t e = base + tid;
                bool take = false;
                if (e < len) {
                    const double x = pass == 0 ? P[lo + e] * f : w[lo + e];
                    if (pass == 0) w[lo + e] = x;
                    take = pass == 0 ? x < 1.0 : !(x < 1.0);
                }
                int pos, tot_take;
                BSI(tmp.si).ExclusiveSum(take ? 1 : 0, pos, tot_take);
                if (take) idx[lo + (pass ? count[0] : 0) + count[pass] + pos] = (int32_t)e;
                count[pass] += tot_take;
                __syncthreads();
            }
        }
        const int64_t na = count[0], nh = count[1];
        // inclusive prefix sums: delta over lights, sigma over heavies
        for (int part2 = 0; part2 < 2; ++part2) {
            const int64_t off = part2 ? na : 0, cnt = part2 ? nh : na;
            double carry = 0.0;
            for (int64_t base = 0; base < cnt; base += kRowBlock) {
                const int64_t k = base + tid;
                double v = 0.0;
                if (k < cnt) {
                    const double x = w[lo + idx[lo + off + k]];
                    v = part2 ? x - 1.0 : 1.0 - x;
                }
                double incl, agg;
                BSD(tmp.sd).InclusiveSum(v, incl, agg);
                if (k < cnt) ds[lo + off + k] = carry + incl;
                carry += agg;
                __syncthreads();
            }
        }
        const double *delta = ds + lo, *sigma = ds + lo + na;
        const int32_t *id = idx + lo;
        for (int64_t k = tid; k < na; k += kRowBlock) {   // lights
            const double prev = k ? delta[k - 1] : 0.0;
            int64_t a = 0, b = nh;
            while (a < b) {
                const int64_t m = (a + b) >> 1;
                if (sigma[m] > prev) b = m;
                else a = m + 1;
            }
            const int64_t item = id[k];
            const uint32_t own = (uint32_t)targets[lo + item];
            rec[lo + item] = a < nh ? make_uint4(__float_as_uint((float)w[lo + item]),
                                                 (uint32_t)targets[lo + id[na + a]], own, 0u)
                                    : make_uint4(__float_as_uint(1.0f), own, own, 0u);
        }
        for (int64_t k = tid; k < nh; k += kRowBlock) {   // heavies
            int64_t a = 0, b = na;
            while (a < b) {
                const int64_t m = (a + b) >> 1;
                if (delta[m] >= sigma[k]) b = m;
                else a = m + 1;
            }
            const int64_t item = id[na + k];
            const uint32_t own = (uint32_t)targets[lo + item];
            if (a < na && k + 1 < nh) {
                const double p = fmin(fmax(1.0 + sigma[k] - delta[a], 0.0), 1.0);
                rec[lo + item] = make_uint4(__float_as_uint((float)p),
                                            (uint32_t)targets[lo + id[na + k + 1]], own, 0u);
            } else {
                rec[lo + item] = make_uint4(__float_as_uint(1.0f), own, own, 0u);
            }
        }
        __syncthreads();
    }
}

// the per-call slot array behind count_evals (no slots when the caller counts nothing)
struct EvalSlots {
    Scratch buf;
    unsigned long long *target = nullptr;
    explicit EvalSlots(cudaStream_t st) : buf(st) {}
    int init(unsigned long long *evals, cudaStream_t st) {
        target = evals;
        if (!evals) return DRG_OK;
        const size_t bytes = sizeof(unsigned long long) * kEvalSlots * kEvalStride;
        DRG_CUDA(buf.alloc(bytes));
        DRG_CUDA(cudaMemsetAsync(buf.p, 0, bytes, st));
        return DRG_OK;
    }
    unsigned long long *slots() const { return target ? buf.as<unsigned long long>() : nullptr; }
    int finish(cudaStream_t st) {
        if (!target) return DRG_OK;
        evals_finish_kernel<<<1, 32, 0, st>>>(slots(), target);
        DRG_LAUNCHED("evals_finish_kernel");
        return DRG_OK;
    }
};

}  // namespace
}  // namespace drg

using namespace drg;

extern "C" int drg_row_alias(const int64_t *indptr, const int32_t *targets, const double *P,
                             int64_t n, int64_t nnz, uint64_t *out_rec, double *out_rowsum,
                             void *stream) {
    if (n <= 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    // rows longer than kRowWarpMax (at most nnz / (kRowWarpMax + 1) of them) are queued
    // by the warp tier; the block tier walks only that list (a grid-stride pass over
    // all n rows cost 2.7 ms on the C4 mesh, which has none)
    const int64_t max_long = nnz / (kRowWarpMax + 1) + 1;
    Scratch lst(st), cnt(st);
    DRG_CUDA(lst.alloc(sizeof(int64_t) * (size_t)max_long));
    DRG_CUDA(cnt.alloc(sizeof(int)));
    DRG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), st));
    const unsigned gw = (unsigned)std::min<int64_t>(ceil_div(n, kRowWarps), sm_count() * 64);
    row_alias_warp_kernel<<<gw, kRowWarps * 32, 0, st>>>(indptr, targets, P, n,
                                                         reinterpret_cast<uint4 *>(out_rec),
                                                         out_rowsum, lst.as<int64_t>(),
                                                         cnt.as<int>());
    DRG_LAUNCHED("row_alias_warp_kernel");
    if (nnz > kRowWarpMax) {
        Scratch idx(st), w(st), ds(st);
        DRG_CUDA(idx.alloc(sizeof(int32_t) * (size_t)nnz));
        DRG_CUDA(w.alloc(sizeof(double) * (size_t)nnz));
        DRG_CUDA(ds.alloc(sizeof(double) * (size_t)nnz));
        const unsigned g = (unsigned)std::min<int64_t>(max_long, sm_count() * 4);
        row_alias_block_kernel<<<g, kRowBlock, 0, st>>>(indptr, targets, P, n, w.as<double>(),
                                                        ds.as<double>(), idx.as<int32_t>(),
                                                        reinterpret_cast<uint4 *>(out_rec),
                                                        out_rowsum, lst.as<int64_t>(),
                                                        cnt.as<int>());
        DRG_LAUNCHED("row_alias_block_kernel");
    }
    return DRG_OK;
}

namespace {

// Internal streams of the split formulation, per device: the updates run on the
// highest-priority stream (their blocks are placed first whenever an SM frees up),
// the draws of the next epochs on the lowest, so the throughput-bound draw pass
// fills what the latency-bound, concurrency-capped update pass leaves idle.
struct SideStreams {
    cudaStream_t hi = nullptr, lo = nullptr;
};

cudaError_t side_streams(SideStreams *out) {
    static std::mutex mu;
    static SideStreams per_dev[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> g(mu);
    SideStreams &ss = per_dev[dev];
    if (!ss.hi) {
        int least = 0, greatest = 0;
        if ((e = cudaDeviceGetStreamPriorityRange(&least, &greatest)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithPriority(&ss.hi, cudaStreamNonBlocking, greatest)) != cudaSuccess)
            return e;
        if ((e = cudaStreamCreateWithPriority(&ss.lo, cudaStreamNonBlocking, least)) != cudaSuccess)
            return e;
    }
    *out = ss;
    return cudaSuccess;
}

struct Events {
    cudaEvent_t e[6] = {};
    ~Events() {
        for (cudaEvent_t x : e)
            if (x) cudaEventDestroy(x);
    }
    cudaError_t create() {
        for (cudaEvent_t &x : e) {
            cudaError_t r = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
            if (r != cudaSuccess) return r;
        }
        return cudaSuccess;
    }
};

// bytes per draw buffer (two buffers): >= 5 level-0 epochs of the C4 mesh per draw
// launch -- one epoch per chunk (64 MB) cost 226 us per epoch in cross-stream event
// waits, 5 epochs per chunk 213 us
constexpr size_t kDrawBudget = size_t(256) << 20;

}  // namespace

namespace drg {
namespace {
__global__ void row_spans_kernel(const int64_t *__restrict__ indptr, int64_t n, uint2 *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = indptr[i];
        out[i] = make_uint2((uint32_t)lo, (uint32_t)(indptr[i + 1] - lo));
    }
}
}  // namespace
}  // namespace drg

extern "C" int drg_row_spans(const int64_t *indptr, int64_t n, uint64_t *out_span, void *stream) {
    if (n <= 0) return DRG_OK;
    int64_t last = 0;
    DRG_CUDA(cudaMemcpyAsync(&last, indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost,
                             as_stream(stream)));
    DRG_CUDA(cudaStreamSynchronize(as_stream(stream)));
    if (last >= (int64_t)1 << 32) return fail(DRG_ERR_UNSUPPORTED, "row spans need nnz < 2^32");
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, 256), sm_count() * 16);
    row_spans_kernel<<<grid, 256, 0, as_stream(stream)>>>(indptr, n, reinterpret_cast<uint2 *>(out_span));
    DRG_LAUNCHED("row_spans_kernel");
    return DRG_OK;
}

namespace drg {
namespace {
__global__ void src_records_kernel(const uint2 *__restrict__ alias, int64_t n,
                                   const int64_t *__restrict__ indptr,
                                   const float *__restrict__ collapse, uint4 *out) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * blockDim.x) {
        const uint2 rec = alias[b];
        const int64_t a = rec.y;
        const int64_t lb = indptr[b], la = indptr[a];
        const float cb = collapse ? collapse[b] : 0.0f, ca = collapse ? collapse[a] : 0.0f;
        out[2 * b] = make_uint4(rec.x, rec.y, (uint32_t)lb, (uint32_t)(indptr[b + 1] - lb));
        out[2 * b + 1] = make_uint4((uint32_t)la, (uint32_t)(indptr[a + 1] - la),
                                    __float_as_uint(cb), __float_as_uint(ca));
    }
}
}  // namespace
}  // namespace drg

extern "C" int drg_src_records(const uint64_t *src_alias, int64_t n_src, const int64_t *indptr,
                               const float *collapse, uint64_t *out, void *stream) {
    if (n_src <= 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    int64_t last = 0;
    DRG_CUDA(cudaMemcpyAsync(&last, indptr + n_src, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (last >= (int64_t)1 << 32) return fail(DRG_ERR_UNSUPPORTED, "source records need nnz < 2^32");
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n_src, 256), sm_count() * 16);
    src_records_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint2 *>(src_alias), n_src,
                                             indptr, collapse, reinterpret_cast<uint4 *>(out));
    DRG_LAUNCHED("src_records_kernel");
    return DRG_OK;
}

extern "C" int drg_sampled_draws(const int64_t *indptr, const uint64_t *row_span,
                                 const uint64_t *row_alias,
                                 const uint64_t *src_alias, const float *collapse,
                                 const uint64_t *neg_alias, const int32_t *map, int64_t n,
                                 int64_t neg_n, int64_t neg_tail_n, double neg_tail_p,
                                 int64_t step_lo,
                                 int64_t n_steps, int t0, int n_epochs, int M, uint64_t seed,
                                 int level, int32_t *out, void *stream) {
    if (n <= 0 || n_steps <= 0 || n_epochs <= 0) return DRG_OK;
    if (n >= 0x7fffffffLL) return fail(DRG_ERR_INVALID, "level exceeds 2^31 - 1 nodes");
    if (M < 0) return fail(DRG_ERR_INVALID, "M must be >= 0");
    DArgs D;
    D.indptr = indptr;
    D.span = reinterpret_cast<const uint2 *>(row_span);
    D.row_alias = reinterpret_cast<const uint4 *>(row_alias);
    D.src_alias = reinterpret_cast<const uint2 *>(src_alias);
    D.collapse = collapse;
    D.neg = make_negtab(neg_alias, neg_n, neg_tail_n, neg_tail_p);
    D.map = map;
    D.n = n;
    D.step_lo = step_lo;
    D.n_steps = n_steps;
    D.n_epochs = n_epochs;
    D.M = M;
    D.key0 = (uint32_t)seed;
    D.key1 = (uint32_t)(seed >> 32);
    D.level = (uint32_t)level;
    D.t_first = t0;
    D.probe = 0;
    D.out = out;
    D.evals = nullptr;
    D.n_src = n;
    D.src_lo = 0;
    D.src_perm = nullptr;
    D.out_stride = n_steps;
    DRG_TRY(launch_draws(D, as_stream(stream)));
    return DRG_OK;
}

extern "C" int drg_sampled_apply(const int32_t *draws, int64_t n_steps, float *y, double lr,
                                 double gamma, double eps, double clip, int b, int M,
                                 int64_t max_threads, int flags, void *stream) {
    if (n_steps <= 0) return DRG_OK;
    if (b < 1 || M < 0 || max_threads < 1) return fail(DRG_ERR_INVALID, "bad optimizer parameters");
    PArgs P;
    P.draws = draws;
    P.n_steps = n_steps;
    P.stride = n_steps;
    P.delta = nullptr;
    P.spread = 0;
    P.lr = (float)lr;
    P.gamma = (float)gamma;
    P.eps = (float)eps;
    P.clip = (float)clip;
    P.b = b;
    P.M = M;
    P.probe = 0;
    const int64_t threads = std::min<int64_t>(n_steps, max_threads);
    const int block = (int)std::min<int64_t>(256, threads);
    const unsigned grid = (unsigned)(threads / block);   // <= threads steps in flight
    cudaStream_t st = as_stream(stream);
    float2 *yy = reinterpret_cast<float2 *>(y);
    void *args[] = {&P, &yy};
    Scratch locks(st);
    if (flags & DRG_SAMPLED_LOCKED) {
        // the node count is not an argument here: a 2^20-entry table indexed by the
        // low id bits (two nodes sharing an entry only exclude each other)
        if (flags & DRG_SAMPLED_AGGREGATE)
            return fail(DRG_ERR_UNSUPPORTED, "locked steps serve plain levels");
        DRG_CUDA(locks.alloc(sizeof(int) << 20));
        DRG_CUDA(cudaMemsetAsync(locks.p, 0, sizeof(int) << 20, st));
        P.locks = locks.as<int>();
        P.lock_mask = (1u << 20) - 1;
        DRG_CUDA(cudaLaunchKernel(b == 2 ? (void *)apply_locked_kernel<2>
                                         : (void *)apply_locked_kernel<0>,
                                  dim3(grid), dim3(block), args, 0, st));
        DRG_LAUNCHED("apply_locked_kernel");
        return DRG_OK;
    }
    DRG_CUDA(cudaLaunchKernel((flags & DRG_SAMPLED_AGGREGATE) ? apply_instance<true>(b)
                                                              : apply_instance<false>(b),
                              dim3(grid), dim3(block), args, 0, st));
    DRG_LAUNCHED("apply_kernel");
    return DRG_OK;
}

extern "C" int drg_layout_sampled(const int64_t *indptr, const uint64_t *row_span,
                                  const uint64_t *rec,
                                  const uint64_t *row_alias, const uint64_t *src_alias,
                                  const float *collapse, const uint64_t *neg_alias,
                                  const int32_t *map, int64_t n,
                                  int64_t neg_n, int64_t neg_tail_n, double neg_tail_p,
                                  float *y, int64_t step_lo, int64_t n_steps, int t0, int n_iter,
                                  int iters,
                                  double lr0, double gamma, double eps, double clip, int b, int M,
                                  uint64_t seed, int level, int64_t max_threads, int flags,
                                  int64_t n_y, uint64_t *evals, const int32_t *hot, int n_hot,
                                  void *stream) {
    if (n <= 0 || n_steps <= 0 || n_iter <= 0) return DRG_OK;
    if (n_y <= 0) n_y = n;
    const bool det = flags & DRG_SAMPLED_DETERMINISTIC;
    if (det && (flags & DRG_SAMPLED_FUSED))
        return fail(DRG_ERR_INVALID, "the deterministic mode runs the split form");
    if (n >= 0x7fffffffLL) return fail(DRG_ERR_INVALID, "level exceeds 2^31 - 1 nodes");
    if (b < 1 || M < 0 || iters < 1) return fail(DRG_ERR_INVALID, "bad optimizer parameters");
    cudaStream_t st = as_stream(stream);
    EvalSlots evs(st);
    DRG_TRY(evs.init(reinterpret_cast<unsigned long long *>(evals), st));
    unsigned long long *ev_ctr = evs.slots();
    const bool agg = flags & DRG_SAMPLED_AGGREGATE;
    const char *probe_env = getenv("DRG_SAMPLED_PROBE");
    const int probe = probe_env ? atoi(probe_env) : 0;
    // exactly min(n_steps, max_threads) steps in flight (1: the sequential kernel)
    const int64_t threads = std::max<int64_t>(1, std::min<int64_t>(n_steps, max_threads));
    // small levels: halve the block until the grid spans two blocks per SM (the
    // update pass is latency-bound; 5 blocks of 256 on 5 SMs left the C4 mesh's
    // coarsest level at 12.4 us per epoch, 64-thread blocks run it in 9.8 us)
    int block = (int)std::min<int64_t>(256, threads);
    while (block > 32 && threads / block < 2 * (int64_t)sm_count()) block /= 2;
    const unsigned grid = (unsigned)(threads / block);
    auto lr_at = [&](int t) { return (float)std::max(lr0 * (1.0 - (double)t / (double)iters), 0.0); };
    if ((flags & (DRG_SAMPLED_LOCKED | DRG_SAMPLED_SNAPSHOT)) && (flags & DRG_SAMPLED_FUSED))
        return fail(DRG_ERR_UNSUPPORTED, "locked steps and snapshot reads serve the split form");
    if ((flags & DRG_SAMPLED_SRC_RECORDS) && (flags & DRG_SAMPLED_FUSED))
        return fail(DRG_ERR_UNSUPPORTED, "source records serve the split form");
    if ((flags & DRG_SAMPLED_FUSED) && map)
        return fail(DRG_ERR_UNSUPPORTED, "the fused form draws from level tables (map == NULL)");
    if (flags & DRG_SAMPLED_FUSED) {   // one kernel per epoch, draws inline
        SArgs A;
        A.indptr = indptr;
        A.rec = reinterpret_cast<const uint2 *>(rec);
        A.row_alias = reinterpret_cast<const uint4 *>(row_alias);
        A.src_alias = reinterpret_cast<const uint2 *>(src_alias);
        A.collapse = collapse;
        A.neg = make_negtab(neg_alias, neg_n, neg_tail_n, neg_tail_p);
        A.n = n;
        A.step_lo = step_lo;
        A.n_steps = n_steps;
        A.gamma = (float)gamma;
        A.eps = (float)eps;
        A.clip = (float)clip;
        A.b = b;
        A.M = M;
        A.key0 = (uint32_t)seed;
        A.key1 = (uint32_t)(seed >> 32);
        A.level = (uint32_t)level;
        A.probe = probe;
        A.evals = ev_ctr;
        for (int j = 0; j < n_iter; ++j) {
            A.t = t0 + j;
            A.lr = lr_at(A.t);
            if (agg) sampled_kernel<true><<<grid, block, 0, st>>>(A, reinterpret_cast<float2 *>(y));
            else sampled_kernel<false><<<grid, block, 0, st>>>(A, reinterpret_cast<float2 *>(y));
            DRG_LAUNCHED("sampled_kernel");
        }
        return evs.finish(st);
    }
    // split: draw_kernel (K epochs per launch, double-buffered, low-priority stream)
    // -> apply_kernel per epoch (high-priority stream); joined back into `stream`
    // snapshot form with the negatives drawn in the update pass (apply_negsnap_kernel):
    // the draw pass resolves only the pairs.  (DRG_NEGSNAP=0: the negatives stay in the
    // draw pass and only their positions come from the snapshot, apply_snap_kernel)
    static const bool negsnap_on = [] {
        const char *e = getenv("DRG_NEGSNAP");
        return !(e && e[0] == '0');
    }();
    const bool use_negsnap = (flags & DRG_SAMPLED_SNAPSHOT) && negsnap_on && M >= 1 &&
                             M <= kMaxNeg && !det && !agg && !(hot && n_hot > 0) &&
                             !(flags & DRG_SAMPLED_LOCKED);
    const int Md = use_negsnap ? 0 : M;   // negatives in the draw records
    const size_t rec_bytes = (size_t)(2 + Md) * sizeof(int32_t) * (size_t)n_steps;
    const int K = (int)std::max<int64_t>(1, std::min<int64_t>(n_iter, (int64_t)(kDrawBudget / rec_bytes)));
    const int nchunks = (n_iter + K - 1) / K;
    Scratch buf(st);
    DRG_CUDA(buf.alloc(rec_bytes * (size_t)K * (nchunks > 1 ? 2 : 1)));
    Scratch locks(st);
    if (flags & DRG_SAMPLED_LOCKED) {
        if (det || agg || (hot && n_hot > 0))
            return fail(DRG_ERR_UNSUPPORTED,
                        "locked steps serve plain Hogwild levels (no hub aggregation / staging, "
                        "not the deterministic mode)");
        DRG_CUDA(locks.alloc(sizeof(int) * (size_t)n_y));
        DRG_CUDA(cudaMemsetAsync(locks.p, 0, sizeof(int) * (size_t)n_y, st));
    }
    Scratch snap(st);
    const bool use_snap = flags & DRG_SAMPLED_SNAPSHOT;
    if (use_snap) {
        if (det || agg || (hot && n_hot > 0) || (flags & (DRG_SAMPLED_FUSED | DRG_SAMPLED_LOCKED)))
            return fail(DRG_ERR_UNSUPPORTED,
                        "snapshot reads serve plain Hogwild levels in the split form");
        DRG_CUDA(snap.alloc((use_negsnap ? sizeof(uint4) : sizeof(float2)) * (size_t)n_y));
        if (use_negsnap) {
            negsnap_init_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n_y, 256),
                                                              (int64_t)sm_count() * 8),
                                  256, 0, st>>>(reinterpret_cast<const uint2 *>(neg_alias), neg_n,
                                                snap.as<uint4>(), n_y);
            DRG_LAUNCHED("negsnap_init_kernel");
        }
    }
    static const int snap_every = [] {   // (experiments: refresh every r-th epoch)
        const char *e = getenv("DRG_SNAP_EVERY");
        return e ? std::max(1, atoi(e)) : 1;
    }();
    SideStreams ss;
    DRG_CUDA(side_streams(&ss));
    Events ev;   // 0 start, 1-2 drawn[2], 3-4 applied[2], 5 draws done
    DRG_CUDA(ev.create());
    DRG_CUDA(cudaEventRecord(ev.e[0], st));
    DRG_CUDA(cudaStreamWaitEvent(ss.lo, ev.e[0], 0));
    DRG_CUDA(cudaStreamWaitEvent(ss.hi, ev.e[0], 0));
    DArgs D;
    D.indptr = indptr;
    D.span = reinterpret_cast<const uint2 *>(row_span);
    D.row_alias = reinterpret_cast<const uint4 *>(row_alias);
    D.src_alias = reinterpret_cast<const uint2 *>(src_alias);
    D.collapse = collapse;
    D.neg = make_negtab(neg_alias, neg_n, neg_tail_n, neg_tail_p);
    D.map = map;
    D.n = n;
    D.step_lo = step_lo;
    D.n_steps = n_steps;
    D.M = Md;
    D.key0 = (uint32_t)seed;
    D.key1 = (uint32_t)(seed >> 32);
    D.level = (uint32_t)level;
    D.probe = probe;
    D.evals = ev_ctr;
    D.n_src = n;
    D.src_lo = 0;
    D.src_perm = nullptr;
    D.out_stride = n_steps;
    if (flags & DRG_SAMPLED_SRC_RECORDS) D.src_rec = reinterpret_cast<const uint4 *>(src_alias);
    auto chunk_buf = [&](int c) { return buf.as<int32_t>() + (size_t)(c & 1) * K * (rec_bytes / 4); };
    auto draw = [&](int c) -> int {
        D.t_first = t0 + c * K;
        D.n_epochs = std::min(K, n_iter - c * K);
        D.out = chunk_buf(c);
        DRG_TRY(launch_draws(D, ss.lo));
        DRG_CUDA(cudaEventRecord(ev.e[1 + (c & 1)], ss.lo));
        return DRG_OK;
    };
    PArgs P;
    P.n_steps = n_steps;
    P.stride = n_steps;
    P.delta = nullptr;
    P.spread = 0;
    P.gamma = (float)gamma;
    P.eps = (float)eps;
    P.clip = (float)clip;
    P.b = b;
    P.M = M;
    P.probe = probe;
    // hub levels whose hottest nodes are staged, draws inline (DRG_HOT_FUSED=1): faster
    // at full concurrency (R-MAT 270 -> 306 iters/s), but those levels run capped at
    // HOT_MAX_THREADS steps in flight for fidelity, and there the split form wins
    // (the draw pass keeps its full occupancy): 208 inline vs 240 split at 64 k
    static const bool hot_fused = [] {
        const char *e = getenv("DRG_HOT_FUSED");
        return e && e[0] == '1';
    }();
    if (hot && n_hot > 0 && !det && M <= kMaxNeg && hot_fused) {
        for (int j = 0; j < n_iter; ++j) {
            D.t_first = t0 + j;
            D.n_epochs = 1;
            P.lr = lr_at(t0 + j);
            DRG_TRY(launch_hot_fused(D, P, reinterpret_cast<float2 *>(y), grid, block, agg, hot,
                                     n_hot, flags & DRG_SAMPLED_L2_HINTS, ss.hi));
        }
        DRG_CUDA(cudaEventRecord(ev.e[0], ss.hi));
        DRG_CUDA(cudaStreamWaitEvent(st, ev.e[0], 0));
        return evs.finish(st);
    }
    P.locks = locks.as<int>();   // NULL unless DRG_SAMPLED_LOCKED
    P.snap = use_snap && !use_negsnap ? snap.as<float2>() : nullptr;
    int rc = draw(0);
    if (rc) return rc;
    Scratch delta(st);
    if (det) {   // fixed-point increments of a sub-batch, zero between sub-batches
        DRG_CUDA(delta.alloc(sizeof(unsigned long long) * 2 * (size_t)n_y));
        DRG_CUDA(cudaMemsetAsync(delta.p, 0, sizeof(unsigned long long) * 2 * (size_t)n_y, st));
        P.delta = delta.as<unsigned long long>();
    }
    for (int c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks) {
            if (c >= 1) DRG_CUDA(cudaStreamWaitEvent(ss.lo, ev.e[3 + ((c + 1) & 1)], 0));
            if ((rc = draw(c + 1))) return rc;
        }
        DRG_CUDA(cudaStreamWaitEvent(ss.hi, ev.e[1 + (c & 1)], 0));
        const int ne = std::min(K, n_iter - c * K);
        for (int e = 0; e < ne; ++e) {
            const int t = t0 + c * K + e;
            P.lr = lr_at(t);
            P.draws = chunk_buf(c) + (size_t)e * (rec_bytes / 4);
            if (det) {
                DRG_TRY(launch_det_epoch(P, reinterpret_cast<float2 *>(y), threads, n_y, ss.hi));
                continue;
            }
            if (use_negsnap) {
                NArgs N;
                N.rec = snap.as<uint4>();
                N.n = D.neg.n;
                N.tail_n = D.neg.tail_n;
                N.tail_thr = D.neg.tail_thr;
                N.key0 = D.key0;
                N.key1 = D.key1;
                N.level = D.level;
                N.t = t;
                N.step_lo = step_lo;
                N.evals = ev_ctr;
                DRG_TRY(launch_negsnap_epoch(P, N, reinterpret_cast<float2 *>(y), n_y, grid, block,
                                             (c * K + e) % snap_every == 0, ss.hi));
                continue;
            }
            if (use_snap && (c * K + e) % snap_every == 0)
                DRG_TRY(launch_snap_copy(reinterpret_cast<const float2 *>(y), snap.as<float2>(),
                                         n_y, ss.hi));
            DRG_TRY(launch_apply(P, reinterpret_cast<float2 *>(y), grid, block, agg, ss.hi, hot,
                                 n_hot));
        }
        DRG_CUDA(cudaEventRecord(ev.e[3 + (c & 1)], ss.hi));
    }
    DRG_CUDA(cudaEventRecord(ev.e[5], ss.lo));
    DRG_CUDA(cudaStreamWaitEvent(st, ev.e[5], 0));
    DRG_CUDA(cudaEventRecord(ev.e[0], ss.hi));
    DRG_CUDA(cudaStreamWaitEvent(st, ev.e[0], 0));
    return evs.finish(st);
}

// =============================================================================
// Multi-GPU sampled epochs: one process per GPU, the level's
// positions partitioned by node range -- rank r owns rows [lo_r, hi_r) in a buffer
// every peer maps (CUDA IPC over NVLink / NVSwitch) -- and Hogwild on that ONE
// distributed array, as the reference's worker threads share one pos
// (optimizer.py:325-345):
//   * a rank runs the steps whose source it owns (sources drawn from its segment
//     of the level-0 nodes; n_l R(segment) / R steps per epoch);
//   * the source and the attraction partner are read and updated in place through
//     the peer table (a cut edge's partner is a remote load / remote atomics);
//   * a negative is read from the rank's replicated snapshot of the epoch-start
//     positions and its reaction summed into a delta array; at the epoch end one
//     reduce-scatter of the deltas and one all-gather of the parts (NCCL over
//     NVLink) fold the reactions in and refresh every snapshot.
// Only the negatives (weak, long-range repulsion) see epoch-start positions; the
// law of a step is otherwise the reference's.  One GPU emulates W ranks with all
// W parts local and every rank's steps in ONE apply launch (no rank ever waits on
// another), which is also the fidelity emulation of any W.
// Snapshot and delta use a padded layout: node v of part r at r * pad + v - lo_r.
// =============================================================================
namespace drg {
namespace {

constexpr int kMaxParts = 8;

struct ShardView {
    float2 *part[kMaxParts];
    int64_t lo[kMaxParts + 1];
    int64_t pad;
    int nparts;
    int self;               // the caller's part; -1: every part is local (emulation)
    const float2 *snap;     // [nparts * pad]
    float2 *delta;          // [nparts * pad]
};

__device__ __forceinline__ int owner_of(const ShardView &V, int64_t v) {
    int r = 0;
#pragma unroll
    for (int q = 1; q < kMaxParts; ++q) r += (q < V.nparts && v >= V.lo[q]);
    return r;
}

__device__ __forceinline__ int64_t padded(const ShardView &V, int64_t v) {
    const int r = owner_of(V, v);
    return r * V.pad + (v - V.lo[r]);
}

__device__ __forceinline__ float2 *addr_of(const ShardView &V, int64_t v, bool &remote) {
    const int r = owner_of(V, v);
    remote = V.self >= 0 && r != V.self;
    return V.part[r] + (v - V.lo[r]);
}

// remote: two scalar float reductions (always supported on peer memory over
// NVLink); local: one float2 reduction
__device__ __forceinline__ void add_at(float2 *p, bool remote, float dx, float dy) {
    if (remote) {
        atomicAdd(&p->x, dx);
        atomicAdd(&p->y, dy);
    } else {
        atomicAdd(p, make_float2(dx, dy));
    }
}

// the multi-GPU store: source and partner through the peer table, negatives from
// the snapshot with their reactions deferred into the delta array
struct ShardStore {
    ShardView V;
    __device__ __forceinline__ float2 load(int64_t v) const {
        bool remote;
        return __ldcg(addr_of(V, v, remote));
    }
    __device__ __forceinline__ float2 load_neg(int64_t v) const {
        return __ldcg(V.snap + padded(V, v));
    }
    __device__ __forceinline__ void add(int64_t v, float dx, float dy) const {
        if (v < 0) return;
        bool remote;
        float2 *p = addr_of(V, v, remote);
        add_at(p, remote, dx, dy);
    }
    __device__ __forceinline__ void add_neg(int64_t v, float dx, float dy) const {
        if (v >= 0) atomicAdd(V.delta + padded(V, v), make_float2(dx, dy));
    }
};

template <int B, bool SPREAD>
__global__ void __launch_bounds__(256) apply_shard_kernel(PArgs A, ShardView V) {
    apply_steps<B, ShardStore, SPREAD>(A, ShardStore{V},
                                       (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                                       (int64_t)gridDim.x * blockDim.x);
}


// part[r][q] += src[r * pad + q] for q < cnt_r (atomics: peers may be updating the
// part at the same time); src zeroed when `clear`
__global__ void fold_kernel(ShardView V, int r0, int r1, float2 *src, int64_t src_base, int clear) {
    for (int r = r0; r < r1; ++r) {
        const int64_t cnt = V.lo[r + 1] - V.lo[r];
        for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt;
             q += (int64_t)gridDim.x * blockDim.x) {
            float2 *s = src + (r - src_base) * V.pad + q;
            const float2 d = *s;
            if (d.x != 0.f || d.y != 0.f) {
                atomicAdd(V.part[r] + q, d);
                if (clear) *s = make_float2(0.f, 0.f);
            }
        }
    }
}

// padded snapshot of the local parts (emulation) / of a full array
__global__ void snap_parts_kernel(ShardView V, float2 *snap) {
    for (int r = 0; r < V.nparts; ++r) {
        const int64_t cnt = V.lo[r + 1] - V.lo[r];
        for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt;
             q += (int64_t)gridDim.x * blockDim.x)
            snap[r * V.pad + q] = __ldcg(V.part[r] + q);
    }
}

// full y -> local parts (r0..r1) and the padded snapshot; or padded -> full y
__global__ void load_parts_kernel(ShardView V, int r0, int r1, const float2 *y, float2 *snap) {
    const int64_t n = V.lo[V.nparts];
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int r = owner_of(V, v);
        const float2 p = y[v];
        snap[r * V.pad + v - V.lo[r]] = p;
        if (r >= r0 && r < r1) V.part[r][v - V.lo[r]] = p;
    }
}

__global__ void unpad_kernel(ShardView V, const float2 *padded_y, float2 *y) {
    const int64_t n = V.lo[V.nparts];
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        y[v] = padded_y[padded(V, v)];
}

// ---- NCCL, loaded at run time (torch's libnccl.so.2; no link-time dependency) --
typedef int nccl_result_t;
typedef void *nccl_comm_t;
struct NcclUid {
    char internal[128];
};
struct Nccl {
    nccl_result_t (*get_unique_id)(NcclUid *) = nullptr;
    nccl_result_t (*comm_init_rank)(nccl_comm_t *, int, NcclUid, int) = nullptr;
    nccl_result_t (*comm_destroy)(nccl_comm_t) = nullptr;
    nccl_result_t (*all_gather)(const void *, void *, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*reduce_scatter)(const void *, void *, size_t, int, int, nccl_comm_t,
                                    cudaStream_t) = nullptr;
    const char *(*error_string)(nccl_result_t) = nullptr;
    bool ok = false;
};
constexpr int kNcclFloat32 = 7, kNcclSum = 0;

const Nccl &nccl() {
    static Nccl N;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        N.get_unique_id = (decltype(N.get_unique_id))dlsym(h, "ncclGetUniqueId");
        N.comm_init_rank = (decltype(N.comm_init_rank))dlsym(h, "ncclCommInitRank");
        N.comm_destroy = (decltype(N.comm_destroy))dlsym(h, "ncclCommDestroy");
        N.all_gather = (decltype(N.all_gather))dlsym(h, "ncclAllGather");
        N.reduce_scatter = (decltype(N.reduce_scatter))dlsym(h, "ncclReduceScatter");
        N.error_string = (decltype(N.error_string))dlsym(h, "ncclGetErrorString");
        N.ok = N.get_unique_id && N.comm_init_rank && N.comm_destroy && N.all_gather &&
               N.reduce_scatter && N.error_string;
    });
    return N;
}

#define DRG_NCCL(call)                                                                  \
    do {                                                                                \
        nccl_result_t _r = (call);                                                      \
        if (_r != 0) return fail(DRG_ERR_CUDA, "%s: %s", #call, nccl().error_string(_r)); \
    } while (0)

}  // namespace

// The communication context behind drg_shard_* (SURVEY §8(b) item 7).
struct ShardCtx {
    int world = 1, rank = 0;       // rank -1: one process emulates all `world` parts
    int64_t capacity = 0;          // nodes per part buffer
    float2 *own[kMaxParts] = {};   // cudaMalloc'd part buffers of this process
    float2 *peer[kMaxParts] = {};  // opened IPC mappings of the peers' buffers
    ShardView view = {};
    nccl_comm_t comm = nullptr;
    float2 *recv = nullptr;        // reduce-scatter landing buffer [pad]
    int64_t recv_cap = 0;
    // lagged exchange (drg_shard_run, DRG_SHARD_LAGGED): the second snapshot and
    // delta buffers [world * pad] and the stream the exchange overlaps on
    float2 *snap2 = nullptr, *delta2 = nullptr;
    int64_t buf2_cap = 0;
    cudaStream_t comm_stream = nullptr;
};

}  // namespace drg

extern "C" int drg_shard_create(int world, int rank, int64_t capacity, void **out_ctx) {
    if (world < 1 || world > kMaxParts) return fail(DRG_ERR_INVALID, "world must be in [1, %d]", kMaxParts);
    if (rank < -1 || rank >= world) return fail(DRG_ERR_INVALID, "bad rank %d", rank);
    if (capacity < 1) return fail(DRG_ERR_INVALID, "capacity must be >= 1");
    ShardCtx *c = new ShardCtx();
    c->world = world;
    c->rank = rank;
    c->capacity = capacity;
    const int nlocal = rank < 0 ? world : 1;
    for (int q = 0; q < nlocal; ++q) {
        cudaError_t e = cudaMalloc(&c->own[q], sizeof(float2) * (size_t)capacity);
        if (e != cudaSuccess) {
            for (int z = 0; z < q; ++z) cudaFree(c->own[z]);
            delete c;
            return cuda_fail(e, "cudaMalloc(part)");
        }
        c->view.part[rank < 0 ? q : rank] = c->own[q];
    }
    c->view.nparts = world;
    c->view.self = rank;
    *out_ctx = c;
    return DRG_OK;
}

extern "C" int drg_shard_destroy(void *ctx) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    if (!c) return DRG_OK;
    if (c->comm) nccl().comm_destroy(c->comm);
    for (float2 *p : c->peer)
        if (p) cudaIpcCloseMemHandle(p);
    for (float2 *p : c->own)
        if (p) cudaFree(p);
    if (c->recv) cudaFree(c->recv);
    if (c->snap2) cudaFree(c->snap2);
    if (c->delta2) cudaFree(c->delta2);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    delete c;
    return DRG_OK;
}

extern "C" int drg_shard_ipc_handle(void *ctx, uint8_t *out_handle64) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    if (c->rank < 0) return fail(DRG_ERR_INVALID, "an emulated context has no peers");
    cudaIpcMemHandle_t h;
    DRG_CUDA(cudaIpcGetMemHandle(&h, c->own[0]));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    memcpy(out_handle64, &h, 64);
    return DRG_OK;
}

extern "C" int drg_shard_open_peer(void *ctx, int r, const uint8_t *handle64) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    if (c->rank < 0 || r < 0 || r >= c->world || r == c->rank)
        return fail(DRG_ERR_INVALID, "bad peer %d", r);
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    void *p = nullptr;
    DRG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->peer[r] = static_cast<float2 *>(p);
    c->view.part[r] = c->peer[r];
    return DRG_OK;
}

extern "C" int drg_nccl_unique_id(uint8_t *out128) {
    if (!nccl().ok) return fail(DRG_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
    NcclUid u;
    DRG_NCCL(nccl().get_unique_id(&u));
    memcpy(out128, &u, 128);
    return DRG_OK;
}

extern "C" int drg_shard_nccl_init(void *ctx, const uint8_t *uid128) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    if (c->rank < 0) return fail(DRG_ERR_INVALID, "an emulated context has no communicator");
    if (!nccl().ok) return fail(DRG_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
    NcclUid u;
    memcpy(&u, uid128, 128);
    DRG_NCCL(nccl().comm_init_rank(&c->comm, c->world, u, c->rank));
    return DRG_OK;
}

// Level layout: bounds[0..world] (host) partition [0, n); snap / delta are caller
// device buffers of world * pad float2 (pad = the longest part), delta zeroed.
extern "C" int drg_shard_level(void *ctx, int64_t n, const int64_t *bounds, float *snap,
                               float *delta, int64_t *out_pad) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    if (bounds[0] != 0 || bounds[c->world] != n) return fail(DRG_ERR_INVALID, "bounds must span [0, n)");
    int64_t pad = 1;
    for (int r = 0; r < c->world; ++r) {
        if (bounds[r + 1] < bounds[r]) return fail(DRG_ERR_INVALID, "bounds must be sorted");
        pad = std::max<int64_t>(pad, bounds[r + 1] - bounds[r]);
    }
    if (pad > c->capacity) return fail(DRG_ERR_INVALID, "part of %lld nodes > capacity %lld",
                                       (long long)pad, (long long)c->capacity);
    for (int r = 0; r < c->world; ++r)
        if (!c->view.part[r]) return fail(DRG_ERR_INVALID, "peer %d not opened", r);
    for (int r = 0; r <= c->world; ++r) c->view.lo[r] = bounds[r];
    for (int r = c->world + 1; r <= kMaxParts; ++r) c->view.lo[r] = n;
    c->view.pad = pad;
    c->view.snap = reinterpret_cast<const float2 *>(snap);
    c->view.delta = reinterpret_cast<float2 *>(delta);
    *out_pad = pad;
    return DRG_OK;
}

namespace {
std::pair<int, int> local_parts(const ShardCtx *c) {
    return c->rank < 0 ? std::make_pair(0, c->world) : std::make_pair(c->rank, c->rank + 1);
}
unsigned shard_grid(int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), sm_count() * 8));
}
}  // namespace

// y (device [n][2], full level) -> this process's parts + the snapshot
extern "C" int drg_shard_load(void *ctx, const float *y, void *stream) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    const auto lp = local_parts(c);
    const int64_t n = c->view.lo[c->world];
    load_parts_kernel<<<shard_grid(n), 256, 0, as_stream(stream)>>>(
        c->view, lp.first, lp.second, reinterpret_cast<const float2 *>(y),
        const_cast<float2 *>(c->view.snap));
    DRG_LAUNCHED("load_parts_kernel");
    return DRG_OK;
}

// the level's positions gathered from every part into y (device [n][2]): the
// all-gather of the parts into the snapshot (NCCL or local), then unpadded
extern "C" int drg_shard_store(void *ctx, float *y, void *stream) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    cudaStream_t st = as_stream(stream);
    float2 *snap = const_cast<float2 *>(c->view.snap);
    if (c->rank < 0 || c->world == 1) {
        snap_parts_kernel<<<shard_grid(c->view.pad), 256, 0, st>>>(c->view, snap);
        DRG_LAUNCHED("snap_parts_kernel");
    } else if (c->comm) {
        DRG_NCCL(nccl().all_gather(c->own[0], snap, (size_t)c->view.pad * 2, kNcclFloat32, c->comm, st));
    } else {
        return fail(DRG_ERR_INVALID, "multi-process context without a communicator: the caller "
                                     "gathers the parts");
    }
    unpad_kernel<<<shard_grid(c->view.lo[c->world]), 256, 0, st>>>(c->view, snap,
                                                                    reinterpret_cast<float2 *>(y));
    DRG_LAUNCHED("unpad_kernel");
    return DRG_OK;
}

// The epoch-end exchange: deltas reduced onto their owners and folded in, the
// parts gathered into every snapshot.  Emulation: local kernels.  Multi-process
// without a communicator: not available (the caller exchanges with
// drg_shard_fold / drg_shard_read_part).
namespace drg {
namespace {
// fold `delta` (reactions) into the parts, then refresh `snap` from the parts
int shard_exchange(ShardCtx *c, float2 *snap, float2 *delta, cudaStream_t st) {
    if (c->rank < 0 || c->world == 1) {
        const auto lp = local_parts(c);
        fold_kernel<<<shard_grid(c->view.pad), 256, 0, st>>>(c->view, lp.first, lp.second,
                                                             delta, 0, 1);
        DRG_LAUNCHED("fold_kernel");
        snap_parts_kernel<<<shard_grid(c->view.pad), 256, 0, st>>>(c->view, snap);
        DRG_LAUNCHED("snap_parts_kernel");
        return DRG_OK;
    }
    if (!c->comm) return fail(DRG_ERR_INVALID, "no communicator");
    if (c->recv_cap < c->view.pad) {
        if (c->recv) cudaFree(c->recv);
        c->recv = nullptr;
        DRG_CUDA(cudaMalloc(&c->recv, sizeof(float2) * (size_t)c->view.pad));
        c->recv_cap = c->view.pad;
    }
    const size_t cnt = (size_t)c->view.pad * 2;
    DRG_NCCL(nccl().reduce_scatter(delta, c->recv, cnt, kNcclFloat32, kNcclSum, c->comm, st));
    fold_kernel<<<shard_grid(c->view.pad), 256, 0, st>>>(c->view, c->rank, c->rank + 1, c->recv,
                                                         c->rank, 0);
    DRG_LAUNCHED("fold_kernel");
    DRG_CUDA(cudaMemsetAsync(delta, 0, sizeof(float2) * (size_t)c->view.pad * c->world, st));
    DRG_NCCL(nccl().all_gather(c->own[0], snap, cnt, kNcclFloat32, c->comm, st));
    return DRG_OK;
}
}  // namespace
}  // namespace drg

extern "C" int drg_shard_exchange(void *ctx, void *stream) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    cudaStream_t st = as_stream(stream);
    float2 *snap = const_cast<float2 *>(c->view.snap);
    if (c->rank < 0 || c->world == 1) return shard_exchange(c, snap, c->view.delta, st);
    return shard_exchange(c, snap, c->view.delta, st);
}

// host-collective path (tests over gloo): fold a reduced delta slice [pad] into the
// own part; copy the own part [pad] out
extern "C" int drg_shard_fold(void *ctx, float *recv, void *stream) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    if (c->rank < 0) return fail(DRG_ERR_INVALID, "emulated context");
    fold_kernel<<<shard_grid(c->view.pad), 256, 0, as_stream(stream)>>>(
        c->view, c->rank, c->rank + 1, reinterpret_cast<float2 *>(recv), c->rank, 0);
    DRG_LAUNCHED("fold_kernel");
    return DRG_OK;
}

extern "C" int drg_shard_read_part(void *ctx, float *out, void *stream) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    if (c->rank < 0) return fail(DRG_ERR_INVALID, "emulated context");
    DRG_CUDA(cudaMemcpyAsync(out, c->own[0], sizeof(float2) * (size_t)c->view.pad,
                             cudaMemcpyDeviceToDevice, as_stream(stream)));
    return DRG_OK;
}

// One sampled epoch t of a sharded level for the sources this process owns:
// per segment s (one per local part) the draws of steps [step_lo[s], +n_steps[s])
// from the segment's source table (seg_alias[s] over seg_n[s] items, node
// perm[seg_lo[s] + q] or seg_lo[s] + q), all segments' steps then applied by one
// launch with <= max_threads steps in flight.  No exchange (drg_shard_exchange).
// out_draws (optional, device int32 [2 + M][total]) receives the draw records.
namespace drg {
namespace {
// the draw arguments common to a sharded level's segments (drg_shard_epoch / _run)
DArgs shard_dargs(const int64_t *indptr, const uint64_t *row_span, const uint64_t *row_alias,
                  const float *collapse,
                  const uint64_t *neg_alias, const int32_t *map, int64_t n_tab, NegTab neg,
                  const int32_t *perm, int M, uint64_t seed, int level, int64_t total,
                  unsigned long long *evals) {
    DArgs D;
    D.indptr = indptr;
    D.span = reinterpret_cast<const uint2 *>(row_span);
    D.row_alias = reinterpret_cast<const uint4 *>(row_alias);
    D.collapse = collapse;
    (void)neg_alias;
    D.neg = neg;
    D.map = map;
    D.n = n_tab;
    D.n_epochs = 1;
    D.M = M;
    D.key0 = (uint32_t)seed;
    D.key1 = (uint32_t)(seed >> 32);
    D.level = (uint32_t)level;
    D.t_first = 0;
    D.probe = 0;
    D.evals = evals;
    D.src_perm = perm;
    D.out_stride = total;
    return D;
}

// every local segment's draws of epochs [t, t + n_epochs) into out ([epoch][2 + M][total])
int shard_draws(DArgs D, int nseg, const uint64_t *const *seg_alias, const int64_t *seg_n,
                const int64_t *seg_lo, const int64_t *step_lo, const int64_t *n_steps, int t,
                int n_epochs, int32_t *out, cudaStream_t st) {
    D.t_first = t;
    D.n_epochs = n_epochs;
    int64_t off = 0;
    for (int s = 0; s < nseg; ++s) {
        if (n_steps[s] == 0) continue;
        D.src_alias = reinterpret_cast<const uint2 *>(seg_alias[s]);
        D.n_src = seg_n[s];
        D.src_lo = seg_lo[s];
        D.step_lo = step_lo[s];
        D.n_steps = n_steps[s];
        D.out = out + off;
        DRG_TRY(launch_draws(D, st));
        off += n_steps[s];
    }
    return DRG_OK;
}

PArgs shard_pargs(int64_t total, int nseg, int64_t max_threads, double gamma, double eps,
                  double clip, int b, int M) {
    PArgs P;
    P.n_steps = total;
    P.stride = total;
    P.delta = nullptr;
    // several local segments (emulation): a prime stride > total visits the columns
    // in a spread order (a bijection of [0, total))
    P.spread = (nseg > 1 && max_threads > 1) ? 4294967291ull : 0;
    P.gamma = (float)gamma;
    P.eps = (float)eps;
    P.clip = (float)clip;
    P.b = b;
    P.M = M;
    P.probe = 0;
    return P;
}

int launch_shard_apply(const PArgs &P, const ShardView &V, int64_t max_threads, cudaStream_t st) {
    const int64_t threads = std::max<int64_t>(1, std::min<int64_t>(P.n_steps, max_threads));
    int block = (int)std::min<int64_t>(256, threads);
    while (block > 32 && threads / block < 2 * (int64_t)sm_count()) block /= 2;
    const unsigned grid = (unsigned)std::max<int64_t>(1, threads / block);
    if (P.spread) {
        if (P.b == 2) apply_shard_kernel<2, true><<<grid, block, 0, st>>>(P, V);
        else apply_shard_kernel<0, true><<<grid, block, 0, st>>>(P, V);
    } else {
        if (P.b == 2) apply_shard_kernel<2, false><<<grid, block, 0, st>>>(P, V);
        else apply_shard_kernel<0, false><<<grid, block, 0, st>>>(P, V);
    }
    DRG_LAUNCHED("apply_shard_kernel");
    return DRG_OK;
}

float lr_of(double lr0, int t, int iters) {
    return (float)std::max(lr0 * (1.0 - (double)t / (double)iters), 0.0);
}
}  // namespace
}  // namespace drg

// One sampled epoch t of a sharded level for the sources this process owns:
// per segment s (one per local part) the draws of steps [step_lo[s], +n_steps[s])
// from the segment's source table (seg_alias[s] over seg_n[s] items, node
// perm[seg_lo[s] + q] or seg_lo[s] + q), all segments' steps then applied by one
// launch with <= max_threads steps in flight.  No exchange (drg_shard_exchange).
// out_draws (optional, device int32 [2 + M][total]) receives the draw records.
extern "C" int drg_shard_epoch(void *ctx, const int64_t *indptr, const uint64_t *row_span,
                               const uint64_t *row_alias,
                               const float *collapse, const uint64_t *neg_alias,
                               const int32_t *map, int64_t n_tab, int64_t neg_n,
                               int64_t neg_tail_n, double neg_tail_p, const int32_t *perm,
                               int nseg, const uint64_t *const *seg_alias, const int64_t *seg_n,
                               const int64_t *seg_lo, const int64_t *step_lo,
                               const int64_t *n_steps, int t, int iters, double lr0,
                               double gamma, double eps, double clip, int b, int M, uint64_t seed,
                               int level, int64_t max_threads, uint64_t *evals,
                               int32_t *out_draws, void *stream) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    cudaStream_t st = as_stream(stream);
    if (M < 0 || b < 1 || iters < 1) return fail(DRG_ERR_INVALID, "bad optimizer parameters");
    if (nseg < 1 || nseg > kMaxParts) return fail(DRG_ERR_INVALID, "bad segment count");
    int64_t total = 0;
    for (int s = 0; s < nseg; ++s) total += n_steps[s];
    if (total == 0) return DRG_OK;
    Scratch buf(st);
    DRG_CUDA(buf.alloc(sizeof(int32_t) * (size_t)(2 + M) * (size_t)total));
    EvalSlots evs(st);
    DRG_TRY(evs.init(reinterpret_cast<unsigned long long *>(evals), st));
    const DArgs D = shard_dargs(indptr, row_span, row_alias, collapse, neg_alias, map, n_tab,
                                make_negtab(neg_alias, neg_n, neg_tail_n, neg_tail_p), perm, M, seed,
                                level, total, evs.slots());
    DRG_TRY(shard_draws(D, nseg, seg_alias, seg_n, seg_lo, step_lo, n_steps, t, 1,
                        buf.as<int32_t>(), st));
    if (out_draws)   // the epoch's draw records, [2 + M][total] (tests)
        DRG_CUDA(cudaMemcpyAsync(out_draws, buf.p, sizeof(int32_t) * (size_t)(2 + M) * total,
                                 cudaMemcpyDeviceToDevice, st));
    PArgs P = shard_pargs(total, nseg, max_threads, gamma, eps, clip, b, M);
    P.draws = buf.as<int32_t>();
    P.lr = lr_of(lr0, t, iters);
    DRG_TRY(launch_shard_apply(P, c->view, max_threads, st));
    return evs.finish(st);
}

// Epochs t0 .. t0 + n_iter - 1 of a sharded level, exchange included, in one call
// (no host round trip per epoch).  Draws: K epochs per launch, double-buffered one
// chunk ahead on the low-priority stream.  Exchange after every epoch: on the
// caller's stream (epoch t + 1 sees every update of epoch t), or with
// DRG_SHARD_LAGGED on the context's exchange stream, overlapped with the next epoch
// -- two snapshot and two delta buffers, epoch t reading the snapshot of the end of
// epoch t - 2 (at the latest) and its reactions folded in by the end of epoch t + 1.
// The emulation (rank -1) runs the lagged form in that worst-case order, so its
// fidelity bounds the real one.
extern "C" int drg_shard_run(void *ctx, const int64_t *indptr, const uint64_t *row_span,
                             const uint64_t *row_alias,
                             const float *collapse, const uint64_t *neg_alias,
                             const int32_t *map, int64_t n_tab, int64_t neg_n,
                             int64_t neg_tail_n, double neg_tail_p, const int32_t *perm, int nseg,
                             const uint64_t *const *seg_alias, const int64_t *seg_n,
                             const int64_t *seg_lo, const int64_t *step_lo,
                             const int64_t *n_steps, int t0, int n_iter, int iters, double lr0,
                             double gamma, double eps, double clip, int b, int M, uint64_t seed,
                             int level, int64_t max_threads, int flags, int exchange_every,
                             uint64_t *evals, void *stream) {
    ShardCtx *c = static_cast<ShardCtx *>(ctx);
    if (exchange_every < 1) return fail(DRG_ERR_INVALID, "exchange_every must be >= 1");
    cudaStream_t st = as_stream(stream);
    if (M < 0 || b < 1 || iters < 1) return fail(DRG_ERR_INVALID, "bad optimizer parameters");
    if (nseg < 1 || nseg > kMaxParts) return fail(DRG_ERR_INVALID, "bad segment count");
    if (c->rank >= 0 && c->world > 1 && !c->comm)
        return fail(DRG_ERR_INVALID, "multi-process context without a communicator: run the "
                                     "epochs with drg_shard_epoch and exchange on the host");
    if (n_iter <= 0) return DRG_OK;
    int64_t total = 0;
    for (int s = 0; s < nseg; ++s) total += n_steps[s];
    const bool lagged = (flags & DRG_SHARD_LAGGED) && c->world > 1;
    if (lagged && exchange_every > 1)
        return fail(DRG_ERR_INVALID, "the lagged exchange runs after every epoch");
    const size_t nbuf = (size_t)c->view.pad * c->world;
    if (lagged && c->buf2_cap < (int64_t)nbuf) {
        if (c->snap2) cudaFree(c->snap2);
        if (c->delta2) cudaFree(c->delta2);
        c->snap2 = c->delta2 = nullptr;
        c->buf2_cap = 0;
        DRG_CUDA(cudaMalloc(&c->snap2, sizeof(float2) * nbuf));
        DRG_CUDA(cudaMalloc(&c->delta2, sizeof(float2) * nbuf));
        c->buf2_cap = (int64_t)nbuf;
    }
    if (lagged && !c->comm_stream)
        DRG_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    float2 *snap[2] = {const_cast<float2 *>(c->view.snap), c->snap2};
    float2 *delta[2] = {c->view.delta, c->delta2};
    if (lagged) {   // both buffers start as the epoch-start snapshot / zero
        DRG_CUDA(cudaMemcpyAsync(snap[1], snap[0], sizeof(float2) * nbuf,
                                 cudaMemcpyDeviceToDevice, st));
        DRG_CUDA(cudaMemsetAsync(delta[1], 0, sizeof(float2) * nbuf, st));
    }
    EvalSlots evs(st);
    DRG_TRY(evs.init(reinterpret_cast<unsigned long long *>(evals), st));
    if (total == 0) {   // nothing drawn here; the exchanges still pair with the peers'
        for (int j = 0; j < n_iter; ++j)
            if (lagged || (j + 1) % exchange_every == 0 || j + 1 == n_iter)
                DRG_TRY(shard_exchange(c, snap[0], delta[0], st));
        return evs.finish(st);
    }
    const DArgs D = shard_dargs(indptr, row_span, row_alias, collapse, neg_alias, map, n_tab,
                                make_negtab(neg_alias, neg_n, neg_tail_n, neg_tail_p), perm, M, seed,
                                level, total, evs.slots());
    const size_t rec_bytes = (size_t)(2 + M) * sizeof(int32_t) * (size_t)total;
    const int K = (int)std::max<int64_t>(1, std::min<int64_t>(n_iter, (int64_t)(kDrawBudget / rec_bytes)));
    const int nchunks = (n_iter + K - 1) / K;
    Scratch buf(st);
    DRG_CUDA(buf.alloc(rec_bytes * (size_t)K * (nchunks > 1 ? 2 : 1)));
    SideStreams ss;
    DRG_CUDA(side_streams(&ss));
    Events ev;   // 0 start, 1-2 drawn[2], 3-4 applied[2], 5 draws done
    DRG_CUDA(ev.create());
    Events xev;  // lagged: 0-1 exchange of an even / odd epoch done, 2-3 epoch applied
    if (lagged) DRG_CUDA(xev.create());
    DRG_CUDA(cudaEventRecord(ev.e[0], st));
    DRG_CUDA(cudaStreamWaitEvent(ss.lo, ev.e[0], 0));
    auto chunk_buf = [&](int q) { return buf.as<int32_t>() + (size_t)(q & 1) * K * (rec_bytes / 4); };
    auto draw = [&](int q) -> int {
        DRG_TRY(shard_draws(D, nseg, seg_alias, seg_n, seg_lo, step_lo, n_steps, t0 + q * K,
                            std::min(K, n_iter - q * K), chunk_buf(q), ss.lo));
        DRG_CUDA(cudaEventRecord(ev.e[1 + (q & 1)], ss.lo));
        return DRG_OK;
    };
    DRG_TRY(draw(0));
    PArgs P = shard_pargs(total, nseg, max_threads, gamma, eps, clip, b, M);
    ShardView V = c->view;
    cudaStream_t xs = c->rank < 0 ? st : c->comm_stream;   // emulation: worst-case order
    if (lagged && xs != st) {
        DRG_CUDA(cudaEventRecord(xev.e[0], st));
        DRG_CUDA(cudaStreamWaitEvent(xs, xev.e[0], 0));
    }
    for (int q = 0; q < nchunks; ++q) {
        if (q + 1 < nchunks) {
            if (q >= 1) DRG_CUDA(cudaStreamWaitEvent(ss.lo, ev.e[3 + ((q + 1) & 1)], 0));
            DRG_TRY(draw(q + 1));
        }
        DRG_CUDA(cudaStreamWaitEvent(st, ev.e[1 + (q & 1)], 0));
        const int ne = std::min(K, n_iter - q * K);
        for (int e = 0; e < ne; ++e) {
            const int j = q * K + e, t = t0 + j;
            P.lr = lr_of(lr0, t, iters);
            P.draws = chunk_buf(q) + (size_t)e * (rec_bytes / 4);
            if (!lagged) {   // exchange after every exchange_every-th epoch and the last
                DRG_TRY(launch_shard_apply(P, V, max_threads, st));
                if ((j + 1) % exchange_every == 0 || j + 1 == n_iter)
                    DRG_TRY(shard_exchange(c, snap[0], delta[0], st));
                continue;
            }
            // epoch j reads snap[j & 1] and writes delta[j & 1]: both last touched
            // by the exchange of epoch j - 2
            if (xs != st && j >= 2) DRG_CUDA(cudaStreamWaitEvent(st, xev.e[j & 1], 0));
            V.snap = snap[j & 1];
            V.delta = delta[j & 1];
            DRG_TRY(launch_shard_apply(P, V, max_threads, st));
            if (xs == st) {   // emulation, the worst case: after epoch j fold epoch
                // j - 1's reactions (delta[(j + 1) & 1]; zero at j = 0) and snapshot
                // for epoch j + 2
                DRG_TRY(shard_exchange(c, snap[j & 1], delta[(j + 1) & 1], st));
                continue;
            }
            DRG_CUDA(cudaEventRecord(xev.e[2 + (j & 1)], st));
            DRG_CUDA(cudaStreamWaitEvent(xs, xev.e[2 + (j & 1)], 0));
            DRG_TRY(shard_exchange(c, snap[j & 1], delta[j & 1], xs));
            DRG_CUDA(cudaEventRecord(xev.e[j & 1], xs));
        }
        DRG_CUDA(cudaEventRecord(ev.e[3 + (q & 1)], st));
    }
    if (lagged) {   // the outstanding reactions: the last epoch's
        if (xs == st) {
            DRG_TRY(shard_exchange(c, snap[0], delta[(n_iter - 1) & 1], st));
        } else {
            DRG_CUDA(cudaEventRecord(xev.e[4], xs));
            DRG_CUDA(cudaStreamWaitEvent(st, xev.e[4], 0));
        }
    }
    DRG_CUDA(cudaEventRecord(ev.e[5], ss.lo));
    DRG_CUDA(cudaStreamWaitEvent(st, ev.e[5], 0));
    return evs.finish(st);
}
