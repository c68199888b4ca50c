// Host-side visiting order of a coarsening level: numpy's
// Generator(PCG64).permutation(n) reproduced bit for bit (multilevel.py:91 draws
// it; the reference's coarsening maps depend on it, so the bit stream must match).
// numpy's own routine shuffles an int64 arange in place (Fisher-Yates from the top,
// bounded draws by masked rejection on the buffered 32-bit half-words of PCG64-XSL-RR)
// and takes ~40 ms for the C4 mesh's 1.73 M nodes -- on the critical path of
// layout_graph's hierarchy stage.  Here the raw PCG64 words are generated in parallel
// slices (LCG jump-ahead), the bounded draws (numpy's random_interval: masked
// rejection on buffered 32-bit half-words; n < 2^31 so always the 32-bit branch)
// consume them on one thread, ahead of the int32 swaps on another.
#include <stdint.h>
#include <stdlib.h>
#include <sys/mman.h>

#include <atomic>
#include <memory>
#include <thread>
#include <vector>

#include "common.cuh"

namespace {

struct Pcg64 {
    __uint128_t state, inc;
    bool has32;
    uint32_t u32;

    uint64_t next64() {
        const __uint128_t mult =
            ((__uint128_t)0x2360ED051FC65DA4ULL << 64) | (__uint128_t)0x4385DF649FCCF645ULL;
        state = state * mult + inc;
        const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
        const unsigned rot = (unsigned)(state >> 122);
        return (x >> rot) | (x << ((64 - rot) & 63));
    }
};

struct HugeBuf {
    void *p = nullptr;
    explicit HugeBuf(size_t bytes) {
        const size_t align = size_t(2) << 20;
        const size_t sz = (bytes + align - 1) / align * align;
        p = aligned_alloc(align, sz ? sz : align);
        if (p) madvise(p, sz ? sz : align, MADV_HUGEPAGE);
    }
    ~HugeBuf() { free(p); }
};

}  // namespace

// state after `delta` steps of the LCG (Brown's jump-ahead)
__uint128_t lcg_advance(__uint128_t state, __uint128_t inc, uint64_t delta) {
    const __uint128_t mult =
        ((__uint128_t)0x2360ED051FC65DA4ULL << 64) | (__uint128_t)0x4385DF649FCCF645ULL;
    __uint128_t acc_mult = 1, acc_plus = 0, cur_mult = mult, cur_plus = inc;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

extern "C" int drg_pcg64_permutation(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                                     uint64_t inc_lo, int has_uint32, uint32_t uinteger,
                                     int64_t n, int32_t *out) {
    using namespace drg;
    if (n < 0 || n >= 0x7fffffffLL) return fail(DRG_ERR_INVALID, "permutation size %lld", (long long)n);
    if (n > 0 && !out) return fail(DRG_ERR_INVALID, "null output");
    const __uint128_t st0 = ((__uint128_t)state_hi << 64) | state_lo;
    const __uint128_t inc = ((__uint128_t)inc_hi << 64) | inc_lo;
    if (n < 2) {
        for (int64_t i = 0; i < n; ++i) out[i] = (int32_t)i;
        return DRG_OK;
    }
    // 1. the raw 64-bit outputs, in parallel slices from jumped-ahead states (each
    //    thread first-touches its own pages): n words = 2n half-words, ~1.4x what the
    //    masked rejection consumes (more are generated on the fly if ever needed)
    const int64_t R = n;
    // scratch on transparent huge pages where the kernel allows it (4 KiB-page faults
    // on fresh memory cost more than the arithmetic here)
    HugeBuf rawb(sizeof(uint64_t) * (size_t)R), jsb(sizeof(int32_t) * (size_t)(n - 1));
    if (!rawb.p || !jsb.p) return fail(DRG_ERR_NOMEM, "permutation scratch");
    uint64_t *raw = static_cast<uint64_t *>(rawb.p);
    int32_t *js = static_cast<int32_t *>(jsb.p);
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>(8, R / (1 << 16)));
    {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                const int64_t lo = R * t / T, hi = R * (t + 1) / T;
                Pcg64 g{lcg_advance(st0, inc, (uint64_t)lo), inc, false, 0};
                for (int64_t k = lo; k < hi; ++k) raw[(size_t)k] = g.next64();
                for (int64_t k = (n - 1) * t / T; k < (n - 1) * (t + 1) / T; ++k) js[k] = 0;
                for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i) out[i] = (int32_t)i;
            });
        for (auto &x : th) x.join();
    }
    // 2. the bounded draws j_k in [0, n-1-k] (i = n-1-k): numpy takes the half-words
    //    in order (low half of a word first, the high half buffered), masks each to
    //    the next power of two and rejects values above the bound.  Branch-free: every
    //    half-word is tried, k advances on acceptance.  On a producer thread; 3. the
    //    swaps follow block by block on this one.
    constexpr int64_t kBlock = 1 << 16;
    const int64_t total = n - 1;
    const int64_t nblocks = (total + kBlock - 1) / kBlock;
    std::atomic<int64_t> ready{0};
    std::thread producer([&] {
        const uint32_t *hw = reinterpret_cast<const uint32_t *>(raw);   // little-endian
        int32_t *jo = js;
        int64_t k = 0;
        auto take = [&](uint32_t h) {
            const uint32_t mx = (uint32_t)(n - 1 - k);   // >= 1
            const uint32_t mask = (uint32_t)((2ull << (31 - __builtin_clz(mx))) - 1);
            const uint32_t v = h & mask;
            jo[k] = (int32_t)v;
            k += v <= mx;
        };
        if (has_uint32) take(uinteger);
        const int64_t H = 2 * R;
        int64_t p = 0;
        for (int64_t b = 0; b < nblocks; ++b) {
            const int64_t end = std::min(total, (b + 1) * kBlock);
            while (k < end && p < H) {
                // within a power-of-two band of the bound m = n-1-k the mask is fixed,
                // so the loop-carried chain is just compare + decrement (~1 ns per
                // half-word instead of re-deriving the mask from k every time)
                const uint32_t mx0 = (uint32_t)(n - 1 - k);
                const uint32_t lowb = 1u << (31 - __builtin_clz(mx0));
                const uint32_t mask = (uint32_t)(2ull * lowb - 1);
                const int64_t kend = std::min<int64_t>(end, (int64_t)n - lowb);   // m >= lowb
                uint32_t m = mx0;
                int64_t kk = k;
                while (kk < kend && p < H) {
                    const uint32_t v = hw[p++] & mask;
                    jo[kk] = (int32_t)v;
                    const uint32_t d = v <= m;
                    kk += d;
                    m -= d;
                }
                k = kk;
            }
            if (k < end) {   // past the generated words (not reached in practice)
                Pcg64 tail{lcg_advance(st0, inc, (uint64_t)R), inc, false, 0};
                while (k < total) {
                    const uint64_t w = tail.next64();
                    take((uint32_t)w);
                    if (k < total) take((uint32_t)(w >> 32));
                }
            }
            ready.store(b + 1, std::memory_order_release);
        }
    });
    for (int64_t b = 0; b < nblocks; ++b) {
        while (ready.load(std::memory_order_acquire) <= b) std::this_thread::yield();
        const int64_t end = std::min(total, (b + 1) * kBlock);
        // j is uniform on [0, i]: on large levels every swap misses the caches, so the
        // swap kPrefetch steps ahead is prefetched (its j is already drawn)
        constexpr int64_t kPrefetch = 64;
        for (int64_t k = b * kBlock; k < end; ++k) {
            if (k + kPrefetch < end) __builtin_prefetch(out + js[k + kPrefetch], 1);
            const int64_t i = n - 1 - k, j = js[k];
            const int32_t t = out[i];
            out[i] = out[j];
            out[j] = t;
        }
    }
    producer.join();
    return DRG_OK;
}
