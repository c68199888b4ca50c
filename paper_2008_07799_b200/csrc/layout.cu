// K7/K8: the node-parallel layout iteration and its level scheduler, K6
// prolongation + radius, and the negative-sampler tables (A8).
//
// K7 replaces the sgd_steps loop (_kernels.py:48-141) driven by sgd_epoch
// (optimizer.py:310-353).  One reference epoch at level l draws n_l positive
// pairs ~ P and M negatives ~ Q per pair; its expected displacement of node a is
//
//     lr * [ sum_b 2 n_l P^l_ab clip(g_att(a,b)) + M n_l (R_a + Q_a) E_c clip(g_rep(a,c)) ]
// The kernel applies exactly that, gathering: one warp per node streams the
// node's CSR row as packed 8-byte records {int32 target, fp32 W_ab = 2 n_l P_ab}
// (one coalesced LDG.64 per entry) and gathers y_b (8 bytes, L2-resident for
// every config here), then lanes 0..M-1 draw one negative each (Philox keyed by
// seed/level/t/node/m/attempt -> alias pick, redraw if c == a, <= 9 attempts like
// _kernels.py:108-117) and add V_a clip(g_rep).  Warp-shuffle reduction, lane 0
// writes y_a.  fp32 throughout; per-interaction math follows
// attractive_gradient / repulsive_gradient (optimizer.py:174-203) with the
// kernel's clip (_kernels.py:94-101, 126-135).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <climits>
#include <vector>

#include "common.cuh"

namespace drg {
namespace {

constexpr int kWpb = 8;  // warps per block of the layout kernel

__device__ __forceinline__ float ipowf(float x, int n) {
    float r = 1.0f;
    for (int i = 0; i < n; ++i) r *= x;
    return r;
}

__device__ __forceinline__ float clampf(float g, float c) { return fminf(fmaxf(g, -c), c); }

// 1/x with one MUFU.RCP (x >= 1 here: no denormal fix-up needed), ~1 ulp.
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

struct IterArgs {
    const int64_t *indptr;
    const uint2 *rec;     // {target, W bits}
    const float *V;
    const uint2 *alias;   // {prob bits, alias}
    int64_t n, row_lo, row_hi;
    float lr, gamma, eps, clip;
    int b, M;
    uint32_t key0, key1;
    uint32_t level;
    int t;
    const int32_t *neg_idx;
    int32_t *nonfinite;
    // heavy-row split (may be null)
    const int32_t *hslot;
    const int32_t *hptr;
    const int32_t *hrow;
    const int64_t *hbegin;
    float2 *hpart;
    int64_t hchunks;
};

__device__ __forceinline__ u32x4 neg_bits(const IterArgs &A, int64_t a, int m, int attempt) {
    return philox4x32(u32x4{(uint32_t)a, (uint32_t)(a >> 32) ^ ((uint32_t)A.t << 1),
                            (A.level << 24) | ((uint32_t)m << 8) | (uint32_t)attempt,
                            0x5eed1e55u},
                      A.key0, A.key1);
}

__device__ __forceinline__ int64_t alias_index(const IterArgs &A, const u32x4 &r) {
    const uint64_t r64 = ((uint64_t)r.x << 32) | r.y;
    return (int64_t)__umul64hi(r64, (uint64_t)A.n);
}

// y gathers: read-only path when the kernel never writes y_in (Jacobi); L2-coherent
// loads in the in-place mode, where other warps update y while it is read.
template <bool INPLACE>
__device__ __forceinline__ float2 load_y(const float2 *y, int64_t i) {
    if (INPLACE) return __ldcg(y + i);
    return __ldg(y + i);
}

// (ld2)^(b-1) by repeated multiply (optimizer.py:142-147); B > 0 is compile-time.
template <int B>
__device__ __forceinline__ float powbm1(float ld2, int b) {
    if (B > 0) {
        float r = 1.0f;
#pragma unroll
        for (int i = 0; i < B - 1; ++i) r *= ld2;
        return r;
    }
    return ipowf(ld2, b - 1);
}

constexpr int kDepth = 4;   // row entries in flight per lane (4 x 32 = 128 per warp pass)

// One negative draw: Philox word pair -> alias bucket, coin -> accept / alias.
__device__ __forceinline__ int64_t resolve_draw(const IterArgs &A, const u32x4 &r, uint2 rec,
                                                int64_t idx) {
    return (u32_to_unit(r.z) < __uint_as_float(rec.x)) ? idx : (int64_t)rec.y;
}

// A warp owns `npw` consecutive nodes (npw = 32 / M): the M negative draws of all
// of them are made at once (one Philox pass for the whole warp, alias records
// loaded before the row streams start), then each node's row is streamed with
// kDepth records + kDepth y-gathers in flight per lane.
//  CLAMP_ATT: clip the attractive gradient.  For b <= 3 and the default clip 5 it
//             is provably inactive (|g_att| <= (2b-1)^((2b-1)/2b) < 5), so the
//             host drops it.
//  PARTNER:   also reject a negative equal to the node's sampled positive partner
//             j ~ W_a. (the reference redraws c in {i, j}, _kernels.py:108-117);
//             only visible when Q_j is not negligible, so enabled on small levels.
template <bool INPLACE, int B, bool CLAMP_ATT, bool PARTNER>
__global__ void __launch_bounds__(kWpb * 32, 5)
    layout_iter_kernel(IterArgs A, int npw, const float2 *y_in, float2 *y_out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t a0 = A.row_lo + ((int64_t)blockIdx.x * kWpb + warp) * npw;
    if (a0 >= A.row_hi) return;
    const int nodes = (int)min((int64_t)npw, A.row_hi - a0);
    const int b = B > 0 ? B : A.b;
    const float two_b = 2.0f * (float)b;
    const int M = A.M;

    // ---- negative draws, first attempt (lane q -> node q / M, sample q % M).
    // Only the coin, the spare word and the alias record stay live across the rows.
    const int nq = nodes * M;
    const int my_node = (npw == 1) ? 0 : (M > 0 ? lane / M : 0);
    const bool neg_lane = (npw == 1) ? (lane < M) : (lane < nq);
    int32_t cand = -1;
    uint32_t coin = 0, spare = 0;
    uint2 arec = make_uint2(0, 0);
    int32_t aidx = 0;
    if (neg_lane) {
        const int64_t an = a0 + my_node;
        const int m = (npw == 1) ? lane : lane - my_node * M;
        if (A.neg_idx) {
            cand = A.neg_idx[an * M + m];
        } else {
            const u32x4 nb = neg_bits(A, an, m, 0);
            aidx = (int32_t)alias_index(A, nb);
            arec = __ldg(A.alias + aidx);
            coin = nb.z;
            spare = nb.w;
        }
    }

    // ---- attractive rows, node by node
    float att_x = 0.f, att_y = 0.f;  // kept by lane i for node i
    int64_t partner = -1;            // kept by lane i for node i
    for (int i = 0; i < nodes; ++i) {
        const int64_t a = a0 + i;
        const int64_t lo = __ldg(A.indptr + a), hi = __ldg(A.indptr + a + 1);
        const int hs = A.hslot ? __ldg(A.hslot + a) : -1;
        const int cnt = hs >= 0 ? 0 : (int)(hi - lo);   // heavy rows: chunk partials
        const uint2 *row = A.rec + lo;
        const float2 ya = load_y<INPLACE>(y_in, a);
        float ax = 0.f, ay = 0.f, wsum = 0.f;
        // one entry's attraction; padding slots (w = 0, y_b = y_a: ld2 == 0) add an
        // exact zero for every b >= 1
        auto add_entry = [&](uint2 r, float2 yb) {
            const float dx = ya.x - yb.x, dy = ya.y - yb.y;
            const float ld2 = fmaf(dx, dx, dy * dy);
            const float pw = powbm1<B>(ld2, b);
            const float w = __uint_as_float(r.y);
            const float inv = rcp_approx(fmaf(pw, ld2, 1.0f));
            if (CLAMP_ATT) {
                const float coef = -two_b * pw * inv;
                ax = fmaf(w, clampf(coef * dx, A.clip), ax);
                ay = fmaf(w, clampf(coef * dy, A.clip), ay);
            } else {
                // the constant -2b is applied once per node below
                const float wc = (B == 1 ? w : w * pw) * inv;
                ax = fmaf(wc, dx, ax);
                ay = fmaf(wc, dy, ay);
            }
            if (PARTNER) wsum += w;
        };
        if (cnt <= 32) {
            // short row (power-law levels: most rows): one slot per lane instead of a
            // kDepth-deep pass -- the same sums, the deep pass's extra slots being
            // exact zeros
            const uint2 r = lane < cnt ? __ldcs(row + lane) : make_uint2((uint32_t)a, 0u);
            add_entry(r, load_y<INPLACE>(y_in, r.x));
        } else {
            for (int base = 0; base < cnt; base += 32 * kDepth) {
                uint2 r[kDepth];
#pragma unroll
                for (int j = 0; j < kDepth; ++j) {
                    const int e = base + j * 32 + lane;
                    r[j] = e < cnt ? __ldcs(row + e) : make_uint2((uint32_t)a, 0u);
                }
                float2 yb[kDepth];
#pragma unroll
                for (int j = 0; j < kDepth; ++j) yb[j] = load_y<INPLACE>(y_in, r[j].x);
#pragma unroll
                for (int j = 0; j < kDepth; ++j) add_entry(r[j], yb[j]);
            }
        }
        if (!CLAMP_ATT) {
            ax *= -two_b;
            ay *= -two_b;
        }
        if (hs >= 0)   // chunk sums of the heavy-row kernel (already scaled)
            for (int c = __ldg(A.hptr + hs) + lane; c < __ldg(A.hptr + hs + 1); c += 32) {
                const float2 p = A.hpart[c];
                ax += p.x;
                ay += p.y;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ax += __shfl_xor_sync(kFull, ax, o);
            ay += __shfl_xor_sync(kFull, ay, o);
        }
        if (lane == i) {
            att_x = ax;
            att_y = ay;
        }
        if (PARTNER && M > 0) {
            // sample j ~ W_a. with the node's spare Philox word: second pass over the
            // (short) row, lane-major cumulative order
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(kFull, wsum, o);
            const uint32_t ubits = __shfl_sync(kFull, spare, (npw == 1) ? 0 : i * M);
            float tau = u32_to_unit(ubits) * wsum;
            int64_t found = -1;
            for (int base = 0; base < cnt && wsum > 0.f; base += 32) {
                const int e = base + lane;
                const uint2 rr = e < cnt ? row[e] : make_uint2(0u, 0u);
                const float w = __uint_as_float(rr.y);
                float incl = w;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    float t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += t;
                }
                const unsigned hit = __ballot_sync(kFull, e < cnt && w > 0.f && incl > tau);
                if (hit) {
                    const int src = __ffs(hit) - 1;
                    found = (int64_t)__shfl_sync(kFull, rr.x, src);
                    break;
                }
                tau -= __shfl_sync(kFull, incl, 31);
            }
            if (lane == i) partner = found;
        }
    }

    // ---- repulsive: finish the draws (redraw while c == a or c == partner, <= 9
    // attempts, _kernels.py:108-117), gather y_c, clip(g_rep)
    const int64_t part = PARTNER ? __shfl_sync(kFull, partner, min(my_node, 31)) : -1;
    float rx = 0.f, ry = 0.f;
    if (neg_lane) {
        const int64_t an = a0 + my_node;
        const int m = (npw == 1) ? lane : lane - my_node * M;
        int64_t c = cand;
        if (!A.neg_idx) {
            c = (u32_to_unit(coin) < __uint_as_float(arec.x)) ? aidx : (int64_t)arec.y;
            for (int attempt = 1; (c == an || c == part) && attempt < 9; ++attempt) {
                const u32x4 nb = neg_bits(A, an, m, attempt);
                const int64_t qi = alias_index(A, nb);
                c = resolve_draw(A, nb, __ldg(A.alias + qi), qi);
            }
            if (c == an || c == part) c = -1;
        }
        if (c >= 0) {
            const float2 ya = load_y<INPLACE>(y_in, an);
            const float2 yc = load_y<INPLACE>(y_in, c);
            const float dx = ya.x - yc.x, dy = ya.y - yc.y;
            const float ld2 = fmaf(dx, dx, dy * dy);
            const float pw = powbm1<B>(ld2, b);
            if (ld2 + A.eps > 0.f) {   // repulsive_gradient's guard (optimizer.py:197)
                const float den = fmaxf((ld2 + A.eps) * fmaf(pw, ld2, 1.0f), 1.17549435e-38f);
                const float coef = A.gamma * two_b * rcp_approx(den);
                rx = clampf(coef * dx, A.clip);
                ry = clampf(coef * dy, A.clip);
            }
        }
    }
    if (npw == 1) {
        // M > 32 tail (serial), then a whole-warp reduction
        for (int m = lane + 32; m < M; m += 32) {
            int64_t c = -1;
            if (A.neg_idx) {
                c = A.neg_idx[a0 * M + m];
            } else {
                for (int attempt = 0; attempt < 9; ++attempt) {
                    u32x4 q = neg_bits(A, a0, m, attempt);
                    int64_t qi = alias_index(A, q);
                    c = resolve_draw(A, q, __ldg(A.alias + qi), qi);
                    if (c != a0 && c != part) break;
                    c = -1;
                }
            }
            if (c >= 0) {
                const float2 ya = load_y<INPLACE>(y_in, a0);
                const float2 yc = load_y<INPLACE>(y_in, c);
                const float dx = ya.x - yc.x, dy = ya.y - yc.y;
                const float ld2 = fmaf(dx, dx, dy * dy);
                const float pw = powbm1<B>(ld2, b);
                if (ld2 + A.eps > 0.f) {
                    const float den =
                        fmaxf((ld2 + A.eps) * fmaf(pw, ld2, 1.0f), 1.17549435e-38f);
                    const float coef = A.gamma * two_b * rcp_approx(den);
                    rx += clampf(coef * dx, A.clip);
                    ry += clampf(coef * dy, A.clip);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            rx += __shfl_xor_sync(kFull, rx, o);
            ry += __shfl_xor_sync(kFull, ry, o);
        }
    } else {
        // segmented sum over the M consecutive lanes of each node (shuffles), then
        // lane i fetches node i's total from lane i*M
        const int sub = lane - my_node * M;
        for (int o = 1; o < M; o <<= 1) {
            const float tx = __shfl_down_sync(kFull, rx, o);
            const float ty = __shfl_down_sync(kFull, ry, o);
            if (sub + o < M && lane + o < 32) {
                rx += tx;
                ry += ty;
            }
        }
        const int src = min(lane * M, 31);
        rx = __shfl_sync(kFull, rx, src);
        ry = __shfl_sync(kFull, ry, src);
    }

    // ---- update (lane i writes node i)
    if (lane < nodes) {
        const int64_t a = a0 + lane;
        const float2 ya = load_y<INPLACE>(y_in, a);
        const float Va = __ldg(A.V + a);
        const float gx = fmaf(Va, rx, att_x), gy = fmaf(Va, ry, att_y);
        const float2 out = make_float2(fmaf(A.lr, gx, ya.x), fmaf(A.lr, gy, ya.y));
        if (!isfinite(out.x) || !isfinite(out.y)) {
            if (A.nonfinite) atomicMin(A.nonfinite, A.t);
        }
        y_out[a] = out;
    }
}

// One warp per chunk of a heavy row: the same attraction math as the row loop,
// the chunk's sum to A.hpart[c].
template <bool INPLACE, int B, bool CLAMP_ATT>
__global__ void __launch_bounds__(kWpb * 32)
    heavy_chunk_kernel(IterArgs A, const float2 *y_in) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * kWpb + (threadIdx.x >> 5);
    if (c >= A.hchunks) return;
    const int b = B > 0 ? B : A.b;
    const float two_b = 2.0f * (float)b;
    const int64_t a = A.hrow[c];
    const int64_t lo = A.hbegin[c];
    const int cnt = (int)min((int64_t)DRG_HEAVY_CHUNK, __ldg(A.indptr + a + 1) - lo);
    const uint2 *row = A.rec + lo;
    const float2 ya = load_y<INPLACE>(y_in, a);
    float ax = 0.f, ay = 0.f;
    for (int base = 0; base < cnt; base += 32 * kDepth) {
        uint2 r[kDepth];
#pragma unroll
        for (int j = 0; j < kDepth; ++j) {
            const int e = base + j * 32 + lane;
            r[j] = e < cnt ? __ldcs(row + e) : make_uint2((uint32_t)a, 0u);
        }
        float2 yb[kDepth];
#pragma unroll
        for (int j = 0; j < kDepth; ++j) yb[j] = load_y<INPLACE>(y_in, r[j].x);
#pragma unroll
        for (int j = 0; j < kDepth; ++j) {
            const float dx = ya.x - yb[j].x, dy = ya.y - yb[j].y;
            const float ld2 = fmaf(dx, dx, dy * dy);
            const float pw = powbm1<B>(ld2, b);
            const float w = __uint_as_float(r[j].y);
            const float inv = rcp_approx(fmaf(pw, ld2, 1.0f));
            if (CLAMP_ATT) {
                const float coef = -two_b * pw * inv;
                ax = fmaf(w, clampf(coef * dx, A.clip), ax);
                ay = fmaf(w, clampf(coef * dy, A.clip), ay);
            } else {
                const float wc = (B == 1 ? w : w * pw) * inv;
                ax = fmaf(wc, dx, ax);
                ay = fmaf(wc, dy, ay);
            }
        }
    }
    if (!CLAMP_ATT) {
        ax *= -two_b;
        ay *= -two_b;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ax += __shfl_xor_sync(kFull, ax, o);
        ay += __shfl_xor_sync(kFull, ay, o);
    }
    if (lane == 0) A.hpart[c] = make_float2(ax, ay);
}

// ---------------------------------------------------------------------------------
// Stochastic gather (update="sgather"): the node-parallel Jacobi iteration with the
// attraction SAMPLED instead of summed over the whole row -- each node draws S
// partners b ~ W_a. from its row's Vose table and applies (sum_b W_ab / S) clip(g_att)
// per draw (unbiased for the A12 expectation, with the reference's per-epoch
// sampling noise: a node takes part in ~2 attractive interactions per epoch), plus
// the M negatives of K7 (redrawn if they hit the node or its first partner, like
// _kernels.py:108-117).  Deterministic (Philox per node), gather-only (no atomics),
// node-range shardable like K7.  A warp owns npw = 32 / (S + M) nodes; each lane
// makes one draw and one y gather, then a segmented shuffle sum per node.
struct SGArgs {
    const uint4 *row_alias;  // per entry {threshold, alias target, own target, 0}
    const float *wsum;       // per node sum_b W_ab
    int S;
};

template <bool INPLACE, int B, bool CLAMP_ATT>
__global__ void __launch_bounds__(kWpb * 32)
    sgather_kernel(IterArgs A, SGArgs G, int npw, const float2 *y_in, float2 *y_out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t a0 = A.row_lo + ((int64_t)blockIdx.x * kWpb + warp) * npw;
    if (a0 >= A.row_hi) return;
    const int nodes = (int)min((int64_t)npw, A.row_hi - a0);
    const int b = B > 0 ? B : A.b;
    const float two_b = 2.0f * (float)b;
    const int K = G.S + A.M;
    const int my = K > 0 ? lane / K : 0;
    const int r = lane - my * K;
    const bool active = lane < nodes * K;
    const bool att = active && r < G.S;
    const int64_t a = a0 + min(my, nodes - 1);
    // 1. attraction draws
    int64_t pb = -1;
    if (att) {
        const int64_t lo = __ldg(A.indptr + a), hi = __ldg(A.indptr + a + 1);
        if (hi > lo) {
            const u32x4 q = philox4x32(u32x4{(uint32_t)a, (uint32_t)(a >> 32) ^ ((uint32_t)A.t << 1),
                                             (A.level << 24) | 0xA00000u | (uint32_t)r, 0x71d3a5c1u},
                                       A.key0, A.key1);
            const int64_t e = lo + (int64_t)__umul64hi(((uint64_t)q.x << 32) | q.y,
                                                        (uint64_t)(hi - lo));
            const uint4 rr = __ldg(G.row_alias + e);
            pb = (u32_to_unit(q.z) < __uint_as_float(rr.x)) ? (int64_t)rr.z : (int64_t)rr.y;
        }
    }
    // 2. the node's first partner, for the negatives' rejection
    const int64_t partner = __shfl_sync(kFull, pb, min(my * K, 31));
    // 3. negatives
    int64_t c = -1;
    if (active && !att) {
        const int m = r - G.S;
        if (A.neg_idx) {
            c = A.neg_idx[a * A.M + m];
        } else {
            for (int attempt = 0; attempt < 9; ++attempt) {
                const u32x4 nb = neg_bits(A, a, m, attempt);
                const int64_t idx = alias_index(A, nb);
                c = resolve_draw(A, nb, __ldg(A.alias + idx), idx);
                if (c != a && c != partner) break;
                c = -1;
            }
        }
    }
    // 4. one interaction per lane
    float gx = 0.f, gy = 0.f;
    const int64_t other = att ? pb : c;
    if (active && other >= 0) {
        const float2 ya = load_y<INPLACE>(y_in, a);
        const float2 yo = load_y<INPLACE>(y_in, other);
        const float dx = ya.x - yo.x, dy = ya.y - yo.y;
        const float ld2 = fmaf(dx, dx, dy * dy);
        const float pw = powbm1<B>(ld2, b);
        if (att) {
            const float wS = __ldg(G.wsum + a) / (float)G.S;
            const float coef = -two_b * pw * rcp_approx(fmaf(pw, ld2, 1.0f));
            gx = wS * (CLAMP_ATT ? clampf(coef * dx, A.clip) : coef * dx);
            gy = wS * (CLAMP_ATT ? clampf(coef * dy, A.clip) : coef * dy);
        } else if (ld2 + A.eps > 0.f) {
            const float Va = __ldg(A.V + a);
            const float den = fmaxf((ld2 + A.eps) * fmaf(pw, ld2, 1.0f), 1.17549435e-38f);
            const float coef = A.gamma * two_b * rcp_approx(den);
            gx = Va * clampf(coef * dx, A.clip);
            gy = Va * clampf(coef * dy, A.clip);
        }
    }
    // 5. segmented sum over the K lanes of each node; lane i writes node i
    for (int o = 1; o < K; o <<= 1) {
        const float tx = __shfl_down_sync(kFull, gx, o);
        const float ty = __shfl_down_sync(kFull, gy, o);
        if (r + o < K && lane + o < 32) {
            gx += tx;
            gy += ty;
        }
    }
    const int src = min(lane * K, 31);
    gx = __shfl_sync(kFull, gx, src);
    gy = __shfl_sync(kFull, gy, src);
    if (lane < nodes) {
        const int64_t an = a0 + lane;
        const float2 ya = load_y<INPLACE>(y_in, an);
        const float2 out = make_float2(fmaf(A.lr, gx, ya.x), fmaf(A.lr, gy, ya.y));
        if (!isfinite(out.x) || !isfinite(out.y)) {
            if (A.nonfinite) atomicMin(A.nonfinite, A.t);
        }
        y_out[an] = out;
    }
}

template <bool INPLACE>
void launch_sgather(unsigned grid, cudaStream_t st, const IterArgs &A, const SGArgs &G, int npw,
                    bool clamp, const float2 *src, float2 *dst) {
#define DRG_SG(BB, CC) sgather_kernel<INPLACE, BB, CC><<<grid, kWpb * 32, 0, st>>>(A, G, npw, src, dst)
    switch (A.b) {
        case 1: if (clamp) DRG_SG(1, true); else DRG_SG(1, false); break;
        case 2: if (clamp) DRG_SG(2, true); else DRG_SG(2, false); break;
        case 3: if (clamp) DRG_SG(3, true); else DRG_SG(3, false); break;
        default: if (clamp) DRG_SG(0, true); else DRG_SG(0, false); break;
    }
#undef DRG_SG
}

template <bool INPLACE, int B>
void launch_iter_b(unsigned grid, cudaStream_t st, const IterArgs &A, int npw, bool clamp,
                   bool partner, const float2 *src, float2 *dst) {
    if (A.hchunks > 0) {
        const unsigned hg = (unsigned)ceil_div(A.hchunks, kWpb);
        if (clamp) heavy_chunk_kernel<INPLACE, B, true><<<hg, kWpb * 32, 0, st>>>(A, src);
        else heavy_chunk_kernel<INPLACE, B, false><<<hg, kWpb * 32, 0, st>>>(A, src);
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    if (clamp) {
        if (partner) layout_iter_kernel<INPLACE, B, true, true><<<grid, kWpb * 32, 0, st>>>(A, npw, src, dst);
        else layout_iter_kernel<INPLACE, B, true, false><<<grid, kWpb * 32, 0, st>>>(A, npw, src, dst);
    } else {
        if (partner) layout_iter_kernel<INPLACE, B, false, true><<<grid, kWpb * 32, 0, st>>>(A, npw, src, dst);
        else layout_iter_kernel<INPLACE, B, false, false><<<grid, kWpb * 32, 0, st>>>(A, npw, src, dst);
    }
}

template <bool INPLACE>
void launch_iter(unsigned grid, cudaStream_t st, const IterArgs &A, int npw, bool clamp,
                 bool partner, const float2 *src, float2 *dst) {
    switch (A.b) {
        case 1: launch_iter_b<INPLACE, 1>(grid, st, A, npw, clamp, partner, src, dst); break;
        case 2: launch_iter_b<INPLACE, 2>(grid, st, A, npw, clamp, partner, src, dst); break;
        case 3: launch_iter_b<INPLACE, 3>(grid, st, A, npw, clamp, partner, src, dst); break;
        default: launch_iter_b<INPLACE, 0>(grid, st, A, npw, clamp, partner, src, dst); break;
    }
}

// Largest |component| the attractive gradient can reach: max_d 2b d^(2b-1)/(1+d^(2b))
// = (2b-1)^((2b-1)/(2b)) (at d^(2b) = 2b-1).
inline bool attractive_clip_active(int b, double clip) {
    const double gmax = std::pow(2.0 * b - 1.0, (2.0 * b - 1.0) / (2.0 * b));
    return !(clip >= gmax * (1.0 + 1e-4));
}

constexpr int64_t kPartnerMaxNodes = 65536;  // partner rejection on levels up to this size

__global__ void level_pack_kernel(const int32_t *__restrict__ targets, const double *__restrict__ P,
                                  int64_t nnz, double scale, uint2 *rec) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x)
        rec[e] = make_uint2((uint32_t)targets[e], __float_as_uint((float)(scale * P[e])));
}

__global__ void node_pack_kernel(const double *__restrict__ R, const double *__restrict__ Q,
                                 double q_scale, int64_t n, double scale, float *V) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        V[i] = (float)(scale * (R[i] + q_scale * Q[i]));
}

// w = mass^power (zero -> 0), block max into *top (optimizer.py:249-255)
__global__ void neg_pow_kernel(const double *__restrict__ mass, int64_t n, double power, double *w,
                               unsigned long long *top_bits) {
    double local = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double m = mass[i];
        double v = (power == 0.0) ? 1.0 : (m > 0.0 ? pow(m, power) : 0.0);
        w[i] = v;
        local = fmax(local, v);
    }
    for (int o = 16; o > 0; o >>= 1) local = fmax(local, __shfl_xor_sync(kFull, local, o));
    if ((threadIdx.x & 31) == 0 && local > 0.0)
        atomicMax(top_bits, (unsigned long long)__double_as_longlong(local));
}

// zero -> 1e-8 * top (optimizer.py:256-258); top == 0 -> all ones
__global__ void neg_floor_kernel(double *w, int64_t n, const unsigned long long *top_bits) {
    const double top = __longlong_as_double((long long)*top_bits);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (top <= 0.0) w[i] = 1.0;
        else if (!(w[i] > 0.0)) w[i] = 1e-8 * top;
    }
}

__global__ void centroid_kernel(const float2 *__restrict__ y, int64_t n, double *partial) {
    double sx = 0.0, sy = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float2 v = y[i];
        sx += v.x;
        sy += v.y;
    }
    typedef cub::BlockReduce<double, 256> BR;
    __shared__ typename BR::TempStorage t1, t2;
    double bx = BR(t1).Sum(sx);
    double by = BR(t2).Sum(sy);
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = bx;
        partial[2 * blockIdx.x + 1] = by;
    }
}

__global__ void radius_kernel(const float2 *__restrict__ y, int64_t n, const double *partial,
                              int nparts, unsigned long long *rmax_bits) {
    double cx = 0.0, cy = 0.0;
    for (int p = 0; p < nparts; ++p) {  // fixed order: deterministic centroid
        cx += partial[2 * p];
        cy += partial[2 * p + 1];
    }
    cx /= (double)n;
    cy /= (double)n;
    double local = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float2 v = y[i];
        double dx = (double)v.x - cx, dy = (double)v.y - cy;
        local = fmax(local, sqrt(dx * dx + dy * dy));
    }
    for (int o = 16; o > 0; o >>= 1) local = fmax(local, __shfl_xor_sync(kFull, local, o));
    if ((threadIdx.x & 31) == 0) atomicMax(rmax_bits, (unsigned long long)__double_as_longlong(local));
}

__global__ void prolong_kernel(const float2 *__restrict__ yc, const int32_t *__restrict__ parent,
                               int64_t n, float jitter, uint32_t k0, uint32_t k1, float2 *yf) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float2 v = yc[parent[i]];
        if (jitter > 0.f) {
            u32x4 r = philox4x32(u32x4{(uint32_t)i, (uint32_t)(i >> 32), 0x9a55u, 0x1e7u}, k0, k1);
            // Box-Muller: two independent N(0,1)
            const float u1 = ((float)(r.x >> 8) + 1.0f) * (1.0f / 16777216.0f);  // (0, 1]
            const float u2 = u32_to_unit(r.y);
            const float rad = sqrtf(-2.0f * logf(u1));
            float s, c;
            sincospif(2.0f * u2, &s, &c);
            v.x += jitter * rad * c;
            v.y += jitter * rad * s;
        }
        yf[i] = v;
    }
}

inline unsigned flat_grid(int64_t n, int threads = 256) {
    return (unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(n, threads), 1), sm_count() * 32);
}

}  // namespace
}  // namespace drg

using namespace drg;

__global__ void weight_kernel(const double *__restrict__ P, int64_t nnz, double scale, float *w) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x)
        w[e] = (float)(scale * P[e]);
}

__global__ void interleave_kernel(const int32_t *__restrict__ tg, const float *__restrict__ w,
                                  int64_t nnz, uint2 *rec) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x)
        rec[e] = make_uint2((uint32_t)tg[e], __float_as_uint(w[e]));
}

extern "C" int drg_level_pack(const int64_t *indptr, const int32_t *targets, const double *P,
                              const double *R, const double *Q, double q_scale, int64_t n,
                              int64_t nnz, int sort_rows, uint64_t *out_rec, float *out_V,
                              void *stream) {
    if (n < 0 || nnz < 0) return fail(DRG_ERR_INVALID, "negative size");
    cudaStream_t st = as_stream(stream);
    const double scale = 2.0 * (double)n;
    if (nnz > 0 && sort_rows && nnz < 0x7fffffffLL && n < 0x7fffffffLL) {
        // rows re-ordered by target id: neighbouring lanes then gather neighbouring
        // y's (fewer L1 sectors per warp load); the pair masses are unchanged
        Scratch w(st), tg2(st), w2(st), tmp(st);
        DRG_CUDA(w.alloc(sizeof(float) * (size_t)nnz));
        DRG_CUDA(tg2.alloc(sizeof(int32_t) * (size_t)nnz));
        DRG_CUDA(w2.alloc(sizeof(float) * (size_t)nnz));
        weight_kernel<<<flat_grid(nnz), 256, 0, st>>>(P, nnz, scale, w.as<float>());
        DRG_LAUNCHED("weight_kernel");
        size_t tb = 0;
        cub::DeviceSegmentedSort::SortPairs(nullptr, tb, targets, tg2.as<int32_t>(), w.as<float>(),
                                            w2.as<float>(), (int)nnz, (int)n, indptr, indptr + 1,
                                            st);
        DRG_CUDA(tmp.alloc(tb));
        DRG_CUDA(cub::DeviceSegmentedSort::SortPairs(tmp.p, tb, targets, tg2.as<int32_t>(),
                                                     w.as<float>(), w2.as<float>(), (int)nnz,
                                                     (int)n, indptr, indptr + 1, st));
        g_launches.fetch_add(1, std::memory_order_relaxed);
        interleave_kernel<<<flat_grid(nnz), 256, 0, st>>>(tg2.as<int32_t>(), w2.as<float>(), nnz,
                                                          reinterpret_cast<uint2 *>(out_rec));
        DRG_LAUNCHED("interleave_kernel");
    } else if (nnz > 0) {
        level_pack_kernel<<<flat_grid(nnz), 256, 0, st>>>(targets, P, nnz, scale,
                                                          reinterpret_cast<uint2 *>(out_rec));
        DRG_LAUNCHED("level_pack_kernel");
    }
    if (n > 0) {
        node_pack_kernel<<<flat_grid(n), 256, 0, st>>>(R, Q, q_scale, n, (double)n, out_V);
        DRG_LAUNCHED("node_pack_kernel");
    }
    return DRG_OK;
}

extern "C" int drg_layout_iters(const int64_t *indptr, const uint64_t *rec, const float *V,
                                const uint64_t *alias, int64_t n, int64_t row_lo, int64_t row_hi,
                                float *y_in, float *y_out, int t0, int n_iter, int iters,
                                double lr0, double gamma, double eps, double clip, int b, int M,
                                uint64_t seed, int level, const int32_t *neg_idx,
                                int32_t *nonfinite, const drg_heavy_split *heavy,
                                unsigned flags, void *stream) {
    if (n <= 0 || n_iter < 0) return DRG_OK;
    if (row_lo < 0 || row_hi > n || row_lo > row_hi)
        return fail(DRG_ERR_INVALID, "row range [%lld, %lld) outside [0, %lld)",
                    (long long)row_lo, (long long)row_hi, (long long)n);
    if (b < 1 || M < 0 || iters < 1) return fail(DRG_ERR_INVALID, "bad optimizer parameters");
    if (n >= 0x7fffffffLL) return fail(DRG_ERR_INVALID, "level exceeds 2^31 - 1 nodes");
    if (neg_idx && n_iter != 1) return fail(DRG_ERR_INVALID, "neg_idx needs n_iter == 1");
    const bool inplace = (flags & DRG_FLAG_INPLACE) != 0;
    if (inplace && y_in != y_out) return fail(DRG_ERR_INVALID, "in-place needs y_in == y_out");
    if (!inplace && y_in == y_out) return fail(DRG_ERR_INVALID, "Jacobi needs two buffers");
    cudaStream_t st = as_stream(stream);
    IterArgs A;
    A.indptr = indptr;
    A.rec = reinterpret_cast<const uint2 *>(rec);
    A.V = V;
    A.alias = reinterpret_cast<const uint2 *>(alias);
    A.n = n;
    A.row_lo = row_lo;
    A.row_hi = row_hi;
    A.gamma = (float)gamma;
    A.eps = (float)eps;
    A.clip = (float)clip;
    A.b = b;
    A.M = M;
    A.key0 = (uint32_t)seed;
    A.key1 = (uint32_t)(seed >> 32);
    A.level = (uint32_t)level;
    A.neg_idx = neg_idx;
    A.nonfinite = nonfinite;
    A.hslot = nullptr;
    A.hptr = nullptr;
    A.hrow = nullptr;
    A.hbegin = nullptr;
    A.hpart = nullptr;
    A.hchunks = 0;
    if (heavy && heavy->n_chunks > 0) {
        A.hslot = heavy->slot;
        A.hptr = heavy->chunk_ptr;
        A.hrow = heavy->chunk_row;
        A.hbegin = heavy->chunk_begin;
        A.hpart = reinterpret_cast<float2 *>(heavy->partial);
        A.hchunks = heavy->n_chunks;
    }
    const int64_t rows = row_hi - row_lo;
    if (rows == 0) return DRG_OK;
    const int npw = (M == 0) ? 8 : (M <= 32 ? std::min(8, 32 / M) : 1);
    const unsigned grid = (unsigned)ceil_div(ceil_div(rows, npw), kWpb);
    const bool clamp = attractive_clip_active(b, clip);
    const bool partner = n <= kPartnerMaxNodes;
    // several iterations ping-pong the two buffers: only a prefix [0, row_hi) may be
    // updated (rows past it -- a frozen isolated tail -- are never written, so the
    // caller keeps them equal in both buffers)
    if (n_iter > 1 && row_lo != 0)
        return fail(DRG_ERR_INVALID, "n_iter > 1 needs a prefix row range [0, row_hi)");
    float2 *src = reinterpret_cast<float2 *>(y_in);
    float2 *dst = reinterpret_cast<float2 *>(y_out);
    if (!inplace && n_iter > 1 && n_iter % 2 == 0) {
        // Jacobi ping-pong with the last write landing in y_out: an even count
        // starts from a copy of the input in y_out (y_in becomes scratch).
        DRG_CUDA(cudaMemcpyAsync(dst, src, sizeof(float2) * (size_t)n, cudaMemcpyDeviceToDevice,
                                 st));
        std::swap(src, dst);
    }
    for (int j = 0; j < n_iter; ++j) {
        const int t = t0 + j;
        A.t = t;
        A.lr = (float)std::max(lr0 * (1.0 - (double)t / (double)iters), 0.0);  // optimizer.py:322
        if (inplace) {
            launch_iter<true>(grid, st, A, npw, clamp, partner, src, src);
        } else {
            launch_iter<false>(grid, st, A, npw, clamp, partner, src, dst);
            std::swap(src, dst);
        }
        DRG_LAUNCHED("layout_iter_kernel");
    }
    return DRG_OK;
}

extern "C" int drg_layout_radius(const float *y, int64_t n, double *out_radius, void *stream) {
    if (n <= 0) return fail(DRG_ERR_INVALID, "empty layout");
    cudaStream_t st = as_stream(stream);
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(n, 256), 256);
    Scratch partial(st), rmax(st);
    DRG_CUDA(partial.alloc(sizeof(double) * 2 * g));
    DRG_CUDA(rmax.alloc(sizeof(unsigned long long)));
    DRG_CUDA(cudaMemsetAsync(rmax.p, 0, sizeof(unsigned long long), st));
    centroid_kernel<<<g, 256, 0, st>>>(reinterpret_cast<const float2 *>(y), n, partial.as<double>());
    DRG_LAUNCHED("centroid_kernel");
    radius_kernel<<<flat_grid(n), 256, 0, st>>>(reinterpret_cast<const float2 *>(y), n,
                                                partial.as<double>(), (int)g,
                                                rmax.as<unsigned long long>());
    DRG_LAUNCHED("radius_kernel");
    unsigned long long bits = 0;
    DRG_CUDA(cudaMemcpyAsync(&bits, rmax.p, sizeof(bits), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    double r;
    memcpy(&r, &bits, sizeof(r));
    *out_radius = r;
    return DRG_OK;
}

extern "C" int drg_prolong(const float *y_coarse, const int32_t *parent, int64_t n_fine,
                           double jitter, uint64_t seed, float *y_fine, void *stream) {
    if (n_fine <= 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    prolong_kernel<<<flat_grid(n_fine), 256, 0, st>>>(
        reinterpret_cast<const float2 *>(y_coarse), parent, n_fine, (float)jitter, (uint32_t)seed,
        (uint32_t)(seed >> 32), reinterpret_cast<float2 *>(y_fine));
    DRG_LAUNCHED("prolong_kernel");
    return DRG_OK;
}

extern "C" int drg_negative_weights(const double *row_mass, int64_t n, double power,
                                    double *out_w, void *stream) {
    if (n <= 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    Scratch top(st);
    DRG_CUDA(top.alloc(sizeof(unsigned long long)));
    DRG_CUDA(cudaMemsetAsync(top.p, 0, sizeof(unsigned long long), st));
    neg_pow_kernel<<<flat_grid(n), 256, 0, st>>>(row_mass, n, power, out_w,
                                                 top.as<unsigned long long>());
    DRG_LAUNCHED("neg_pow_kernel");
    neg_floor_kernel<<<flat_grid(n), 256, 0, st>>>(out_w, n, top.as<unsigned long long>());
    DRG_LAUNCHED("neg_floor_kernel");
    return DRG_OK;
}

// Alias table on the device (replaces the host Vose loop of build_alias_table,
// optimizer.py:111-139).  Parallel "sweep" construction: with normalised weights
// (mean 1), light items l_1..l_a (w < 1) and heavy items h_1..h_b in index order,
// deficits delta_i = sum_{k<=i} (1 - w_lk) and surpluses sigma_j = sum_{k<=j}
// (w_hk - 1), the sequential sweep (a heavy absorbs lights until its residual drops
// to <= 1, then is itself topped up by the next heavy) assigns
//   light i  -> alias h_j, j = first j with sigma_j > delta_{i-1},  prob w_li;
//   heavy j  -> alias h_{j+1}, prob 1 + sigma_j - delta_i', i' = first i with
//               delta_i >= sigma_j (prob 1 if it never retires).
// Every bucket holds exactly mass 1 and every item its weight: the same law as
// Vose's table (a different but equally valid table).
namespace drg {
namespace {

__global__ void alias_norm_kernel(const double *__restrict__ w, int64_t n, const double *total,
                                  double *wn, uint8_t *light, uint8_t *heavy, int *bad) {
    const double f = (double)n / *total;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = w[i];
        if (v < 0.0 || !(v == v)) atomicExch(bad, 1);
        const double x = v * f;
        wn[i] = x;
        light[i] = x < 1.0;
        heavy[i] = !(x < 1.0);
    }
}

__global__ void alias_gap_kernel(const double *__restrict__ wn, const int32_t *__restrict__ idx,
                                 const int64_t *cnt, int heavy, double *out) {
    const int64_t m = *cnt;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double x = wn[idx[k]];
        out[k] = heavy ? x - 1.0 : 1.0 - x;
    }
}

__device__ __forceinline__ int64_t upper_bound_d(const double *a, int64_t m, double v) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] > v) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

__device__ __forceinline__ int64_t lower_bound_d(const double *a, int64_t m, double v) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] >= v) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

__global__ void alias_light_kernel(const double *__restrict__ wn, const int32_t *__restrict__ L,
                                   const int64_t *na, const double *__restrict__ delta,
                                   const int32_t *__restrict__ H, const int64_t *nb,
                                   const double *__restrict__ sigma, uint2 *table) {
    const int64_t a = *na, b = *nb;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double prev = k == 0 ? 0.0 : delta[k - 1];
        const int64_t j = upper_bound_d(sigma, b, prev);
        const int32_t item = L[k];
        if (j < b) table[item] = make_uint2(__float_as_uint((float)wn[item]), (uint32_t)H[j]);
        else table[item] = make_uint2(__float_as_uint(1.0f), (uint32_t)item);
    }
}

__global__ void alias_heavy_kernel(const int32_t *__restrict__ H, const int64_t *nb,
                                   const double *__restrict__ sigma, const int64_t *na,
                                   const double *__restrict__ delta, uint2 *table) {
    const int64_t a = *na, b = *nb;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < b;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t item = H[k];
        const int64_t i = lower_bound_d(delta, a, sigma[k]);
        if (i < a && k + 1 < b) {
            const double p = fmin(fmax(1.0 + sigma[k] - delta[i], 0.0), 1.0);
            table[item] = make_uint2(__float_as_uint((float)p), (uint32_t)H[k + 1]);
        } else {
            table[item] = make_uint2(__float_as_uint(1.0f), (uint32_t)item);
        }
    }
}

__global__ void iota_i32_kernel(int32_t *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)i;
}

}  // namespace
}  // namespace drg

extern "C" int drg_alias_build(const double *weights, int64_t n, uint64_t *out_table,
                               double *out_total, void *stream) {
    if (n <= 0) return fail(DRG_ERR_INVALID, "cannot build an alias table over zero items");
    if (n >= 0x7fffffffLL) return fail(DRG_ERR_INVALID, "alias table over >= 2^31 items");
    cudaStream_t st = as_stream(stream);
    Scratch tot(st), wn(st), lf(st), hf(st), idx(st), L(st), H(st), cnt(st), dl(st), sg(st),
        dls(st), sgs(st), tmp(st), bad(st);
    DRG_CUDA(tot.alloc(sizeof(double)));
    DRG_CUDA(wn.alloc(sizeof(double) * (size_t)n));
    DRG_CUDA(lf.alloc((size_t)n));
    DRG_CUDA(hf.alloc((size_t)n));
    DRG_CUDA(idx.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(L.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(H.alloc(sizeof(int32_t) * (size_t)n));
    DRG_CUDA(cnt.alloc(2 * sizeof(int64_t)));
    DRG_CUDA(dl.alloc(sizeof(double) * (size_t)n));
    DRG_CUDA(sg.alloc(sizeof(double) * (size_t)n));
    DRG_CUDA(dls.alloc(sizeof(double) * (size_t)n));
    DRG_CUDA(sgs.alloc(sizeof(double) * (size_t)n));
    DRG_CUDA(bad.alloc(sizeof(int)));
    DRG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceReduce::Sum(nullptr, t1, weights, tot.as<double>(), n, st);
    cub::DeviceSelect::Flagged(nullptr, t2, idx.as<int32_t>(), lf.as<uint8_t>(), L.as<int32_t>(),
                               cnt.as<int64_t>(), n, st);
    cub::DeviceScan::InclusiveSum(nullptr, t3, dl.as<double>(), dls.as<double>(), n, st);
    DRG_CUDA(tmp.alloc(std::max(t1, std::max(t2, t3))));
    DRG_CUDA(cub::DeviceReduce::Sum(tmp.p, t1, weights, tot.as<double>(), n, st));
    double total = 0.0;
    DRG_CUDA(cudaMemcpyAsync(&total, tot.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (!(total > 0.0)) return fail(DRG_ERR_INVALID, "all weights are zero");
    if (out_total) *out_total = total;
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(n, 256), sm_count() * 16);
    alias_norm_kernel<<<g, 256, 0, st>>>(weights, n, tot.as<double>(), wn.as<double>(),
                                         lf.as<uint8_t>(), hf.as<uint8_t>(), bad.as<int>());
    DRG_LAUNCHED("alias_norm_kernel");
    iota_i32_kernel<<<g, 256, 0, st>>>(idx.as<int32_t>(), n);
    DRG_LAUNCHED("iota_i32_kernel");
    int64_t *na = cnt.as<int64_t>(), *nb = cnt.as<int64_t>() + 1;
    DRG_CUDA(cub::DeviceSelect::Flagged(tmp.p, t2, idx.as<int32_t>(), lf.as<uint8_t>(),
                                        L.as<int32_t>(), na, n, st));
    DRG_CUDA(cub::DeviceSelect::Flagged(tmp.p, t2, idx.as<int32_t>(), hf.as<uint8_t>(),
                                        H.as<int32_t>(), nb, n, st));
    alias_gap_kernel<<<g, 256, 0, st>>>(wn.as<double>(), L.as<int32_t>(), na, 0, dl.as<double>());
    DRG_LAUNCHED("alias_gap_kernel");
    alias_gap_kernel<<<g, 256, 0, st>>>(wn.as<double>(), H.as<int32_t>(), nb, 1, sg.as<double>());
    DRG_LAUNCHED("alias_gap_kernel");
    // prefix sums over the full length (entries past the counts are never read)
    DRG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, t3, dl.as<double>(), dls.as<double>(), n, st));
    DRG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, t3, sg.as<double>(), sgs.as<double>(), n, st));
    g_launches.fetch_add(5, std::memory_order_relaxed);
    uint2 *table = reinterpret_cast<uint2 *>(out_table);
    alias_light_kernel<<<g, 256, 0, st>>>(wn.as<double>(), L.as<int32_t>(), na, dls.as<double>(),
                                          H.as<int32_t>(), nb, sgs.as<double>(), table);
    DRG_LAUNCHED("alias_light_kernel");
    alias_heavy_kernel<<<g, 256, 0, st>>>(H.as<int32_t>(), nb, sgs.as<double>(), na,
                                          dls.as<double>(), table);
    DRG_LAUNCHED("alias_heavy_kernel");
    int h_bad = 0;
    DRG_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (h_bad) return fail(DRG_ERR_INVALID, "negative weight");
    return DRG_OK;
}

extern "C" int drg_layout_sgather(const int64_t *indptr, const uint64_t *rec,
                                  const uint64_t *row_alias, const float *wsum, const float *V,
                                  const uint64_t *alias, int64_t n, int64_t row_lo,
                                  int64_t row_hi, float *y_in, float *y_out, int t0, int n_iter,
                                  int iters, double lr0, double gamma, double eps, double clip,
                                  int b, int M, int S, uint64_t seed, int level,
                                  const int32_t *neg_idx, int32_t *nonfinite, unsigned flags,
                                  void *stream) {
    if (n <= 0 || n_iter < 0) return DRG_OK;
    if (n >= 0x7fffffffLL) return fail(DRG_ERR_INVALID, "level exceeds 2^31 - 1 nodes");
    if (row_lo < 0 || row_hi > n || row_lo > row_hi) return fail(DRG_ERR_INVALID, "bad row range");
    if (b < 1 || M < 0 || S < 1 || S + M > 32 || iters < 1)
        return fail(DRG_ERR_INVALID, "need b >= 1, S >= 1, S + M <= 32");
    if (neg_idx && n_iter != 1) return fail(DRG_ERR_INVALID, "neg_idx needs n_iter == 1");
    const bool inplace = (flags & DRG_FLAG_INPLACE) != 0;
    if (inplace != (y_in == y_out)) return fail(DRG_ERR_INVALID, "buffer / flag mismatch");
    if (n_iter > 1 && row_lo != 0)   // as drg_layout_iters: a prefix, the tail frozen
        return fail(DRG_ERR_INVALID, "n_iter > 1 needs a prefix row range [0, row_hi)");
    cudaStream_t st = as_stream(stream);
    IterArgs A = {};
    A.indptr = indptr;
    A.rec = reinterpret_cast<const uint2 *>(rec);
    A.V = V;
    A.alias = reinterpret_cast<const uint2 *>(alias);
    A.n = n;
    A.row_lo = row_lo;
    A.row_hi = row_hi;
    A.gamma = (float)gamma;
    A.eps = (float)eps;
    A.clip = (float)clip;
    A.b = b;
    A.M = M;
    A.key0 = (uint32_t)seed;
    A.key1 = (uint32_t)(seed >> 32);
    A.level = (uint32_t)level;
    A.neg_idx = neg_idx;
    A.nonfinite = nonfinite;
    SGArgs G{reinterpret_cast<const uint4 *>(row_alias), wsum, S};
    const int64_t rows = row_hi - row_lo;
    if (rows == 0) return DRG_OK;
    const int npw = std::max(1, 32 / (S + M));
    const unsigned grid = (unsigned)ceil_div(ceil_div(rows, npw), kWpb);
    const bool clamp = attractive_clip_active(b, clip);
    float2 *src = reinterpret_cast<float2 *>(y_in);
    float2 *dst = reinterpret_cast<float2 *>(y_out);
    if (!inplace && n_iter > 1 && n_iter % 2 == 0) {
        DRG_CUDA(cudaMemcpyAsync(dst, src, sizeof(float2) * (size_t)n, cudaMemcpyDeviceToDevice,
                                 st));
        std::swap(src, dst);
    }
    for (int j = 0; j < n_iter; ++j) {
        A.t = t0 + j;
        A.lr = (float)std::max(lr0 * (1.0 - (double)A.t / (double)iters), 0.0);
        if (inplace) {
            launch_sgather<true>(grid, st, A, G, npw, clamp, src, src);
        } else {
            launch_sgather<false>(grid, st, A, G, npw, clamp, src, dst);
            std::swap(src, dst);
        }
        DRG_LAUNCHED("sgather_kernel");
    }
    return DRG_OK;
}
