// Text ingestion on the device: the edge-list and MatrixMarket parsers of
// graph.py:128-243 over the raw UTF-8 bytes of a file.
//
// The reference reads a file as text (cli.py:194, universal newlines) and parses
// the string: str.splitlines() (graph.py:128-131) splits at \n, \r, \r\n, \v, \f,
// \x1c-\x1e, U+0085, U+2028, U+2029; every line is stripped and split on Unicode
// whitespace; ids go through int() (sign, Unicode decimal digits, single
// underscores between digits).  Here:
//   1. utf8_check_kernel: strict UTF-8 validation (what open(..., encoding="utf-8")
//      enforces), first bad byte by atomicMin;
//   2. line starts: a tile pass counts the line starts in 4 KiB tiles, CUB scans the
//      tile counts, a second tile pass writes the starts in order (block scan);
//   3. parse_lines_kernel: one thread per line decodes code points and runs the
//      token / int() state machine of the reference's loop; per-line status and
//      the two ids;
//   4. the first failing line (atomicMin) and the accepted pairs (CUB select, line
//      order) go back to the host, which only formats the reference's message for
//      that one line.
// Line breaks are whitespace to str.split(), so a line's segment [start_l,
// start_{l+1}) can be tokenised without trimming its break.
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include "common.cuh"
#include "unicode_tables.cuh"

namespace drg {
namespace {

constexpr int kTileBytes = 4096;
constexpr int kTileThreads = 256;
constexpr int kBytesPerThread = kTileBytes / kTileThreads;   // 16

// ---- UTF-8 -------------------------------------------------------------------------
__device__ __forceinline__ bool is_cont(uint8_t b) { return (b & 0xC0) == 0x80; }

__device__ __forceinline__ int lead_len(uint8_t b) {
    if (b < 0x80) return 1;
    if (b >= 0xC2 && b <= 0xDF) return 2;
    if (b >= 0xE0 && b <= 0xEF) return 3;
    if (b >= 0xF0 && b <= 0xF4) return 4;
    return 0;   // continuation byte or never valid (C0, C1, F5..FF)
}

// Strict decoder rules (Python's utf-8 codec): shortest form, no surrogates, <= U+10FFFF.
__device__ bool valid_at(const uint8_t *t, int64_t n, int64_t p) {
    const uint8_t b = t[p];
    if (b < 0x80) return true;
    if (is_cont(b)) {   // must continue a lead at p-1..p-3 whose sequence covers p
        for (int back = 1; back <= 3 && p - back >= 0; ++back) {
            const uint8_t c = t[p - back];
            if (!is_cont(c)) return lead_len(c) > back;
        }
        return false;
    }
    const int len = lead_len(b);
    if (len == 0 || p + len > n) return false;
    const uint8_t b1 = t[p + 1];
    if (!is_cont(b1)) return false;
    if (b == 0xE0 && b1 < 0xA0) return false;
    if (b == 0xED && b1 > 0x9F) return false;
    if (b == 0xF0 && b1 < 0x90) return false;
    if (b == 0xF4 && b1 > 0x8F) return false;
    for (int k = 2; k < len; ++k)
        if (!is_cont(t[p + k])) return false;
    return true;
}

__global__ void utf8_check_kernel(const uint8_t *__restrict__ t, int64_t n,
                                  unsigned long long *first_bad) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x)
        if (!valid_at(t, n, p)) atomicMin(first_bad, (unsigned long long)p);
}

// ---- line starts ---------------------------------------------------------------------
// Does a line break END at byte e?  mode 0: str.splitlines (\r\n is one break, ending
// at the \n); mode 1: "\n" only (text already read through universal newlines, or
// io.StringIO iteration).
__device__ __forceinline__ bool break_ends(const uint8_t *t, int64_t n, int64_t e, int mode) {
    const uint8_t b = t[e];
    if (b == '\n') return true;
    if (mode == 1) return false;
    switch (b) {
        case '\r': return !(e + 1 < n && t[e + 1] == '\n');
        case 0x0B: case 0x0C: case 0x1C: case 0x1D: case 0x1E: return true;
        case 0x85: return e >= 1 && t[e - 1] == 0xC2;                               // U+0085
        case 0xA8: case 0xA9: return e >= 2 && t[e - 1] == 0x80 && t[e - 2] == 0xE2;   // U+2028/9
        default: return false;
    }
}

// line starts in [q0, q0 + kBytesPerThread): q == 0, or a break ended at q - 1
__device__ __forceinline__ unsigned starts_mask(const uint8_t *t, int64_t n, int64_t q0, int mode) {
    unsigned mask = 0;
#pragma unroll
    for (int k = 0; k < kBytesPerThread; ++k) {
        const int64_t q = q0 + k;
        if (q < n && (q == 0 || break_ends(t, n, q - 1, mode))) mask |= 1u << k;
    }
    return mask;
}

__global__ void __launch_bounds__(kTileThreads)
    line_count_kernel(const uint8_t *__restrict__ t, int64_t n, int mode, int64_t *tile_count) {
    using BR = cub::BlockReduce<int, kTileThreads>;
    __shared__ typename BR::TempStorage tmp;
    const int64_t q0 = (int64_t)blockIdx.x * kTileBytes + (int64_t)threadIdx.x * kBytesPerThread;
    const int c = __popc(starts_mask(t, n, q0, mode));
    const int tot = BR(tmp).Sum(c);
    if (threadIdx.x == 0) tile_count[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kTileThreads)
    line_fill_kernel(const uint8_t *__restrict__ t, int64_t n, int mode,
                     const int64_t *__restrict__ tile_off, int64_t *starts) {
    using BS = cub::BlockScan<int, kTileThreads>;
    __shared__ typename BS::TempStorage tmp;
    const int64_t q0 = (int64_t)blockIdx.x * kTileBytes + (int64_t)threadIdx.x * kBytesPerThread;
    unsigned mask = starts_mask(t, n, q0, mode);
    int off;
    BS(tmp).ExclusiveSum(__popc(mask), off);
    int64_t o = tile_off[blockIdx.x] + off;
    while (mask) {
        const int k = __ffs(mask) - 1;
        mask &= mask - 1;
        starts[o++] = q0 + k;
    }
}

// ---- per-line parse ------------------------------------------------------------------
__device__ __forceinline__ uint32_t decode(const uint8_t *t, int64_t p, int *len) {
    const uint8_t b = t[p];
    if (b < 0x80) {
        *len = 1;
        return b;
    }
    if (b < 0xE0) {
        *len = 2;
        return ((b & 0x1Fu) << 6) | (t[p + 1] & 0x3Fu);
    }
    if (b < 0xF0) {
        *len = 3;
        return ((b & 0x0Fu) << 12) | ((t[p + 1] & 0x3Fu) << 6) | (t[p + 2] & 0x3Fu);
    }
    *len = 4;
    return ((b & 0x07u) << 18) | ((t[p + 1] & 0x3Fu) << 12) | ((t[p + 2] & 0x3Fu) << 6) |
           (t[p + 3] & 0x3Fu);
}

__device__ __forceinline__ bool is_space(uint32_t c) {
    if (c < 0x80) return (c >= 0x09 && c <= 0x0D) || (c >= 0x1C && c <= 0x20);
    int lo = 0, hi = kNumSpace;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (kSpace[m] < c) lo = m + 1;
        else hi = m;
    }
    return lo < kNumSpace && kSpace[lo] == c;
}

// decimal value of an Nd digit, -1 otherwise
__device__ __forceinline__ int digit_value(uint32_t c) {
    if (c < 0x80) return (c >= '0' && c <= '9') ? (int)(c - '0') : -1;
    int lo = 0, hi = kNumDigitRuns;   // last run start <= c
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (kDigitZero[m] <= c) lo = m + 1;
        else hi = m;
    }
    if (lo == 0) return -1;
    const uint32_t d = c - kDigitZero[lo - 1];
    return d < 10 ? (int)d : -1;
}

// int(token) (Python's grammar: [sign] digit (["_"] digit)*), fed one code point at a
// time.  Magnitudes beyond 2^63 - 1 set `big` (Python keeps them exact; the callers
// then raise what the reference raises for such ids).
struct IntParse {
    uint64_t mag = 0;
    bool neg = false, big = false, bad = false, digit_last = false, any_digit = false,
         us_last = false;
    int pos = 0;
    __device__ void feed(uint32_t c) {
        const int d = digit_value(c);
        if (pos++ == 0 && (c == '+' || c == '-')) {
            neg = c == '-';
            return;
        }
        if (d >= 0) {
            if (mag > (0x7fffffffffffffffull - (uint64_t)d) / 10) big = true;
            else mag = mag * 10 + (uint64_t)d;
            digit_last = any_digit = true;
            us_last = false;
        } else if (c == '_' && digit_last) {
            digit_last = false;
            us_last = true;
        } else {
            bad = true;
        }
    }
    __device__ bool ok() const { return !bad && any_digit && !us_last; }
    __device__ bool negative() const { return neg && (mag != 0 || big); }
};

enum LineStatus : int8_t {
    kSkip = 0,       // blank or comment
    kPair = 1,       // two ids parsed
    kTokens = 2,     // edge list: not exactly two tokens / MatrixMarket: fewer than two
    kMalformed = 3,  // int() fails on one of the first two tokens
    kNegative = 4,   // edge list: negative id
    kRange = 5,      // MatrixMarket: index outside 1..rows
};

struct ParseArgs {
    const uint8_t *t;
    int64_t n;
    const int64_t *starts;
    int64_t n_lines;
    int kind;          // 0 edge list (graph.py:134-167), 1 MatrixMarket entries (227-241)
    int64_t rows;      // MatrixMarket: declared rows (= cols)
    int8_t *status;
    int64_t *pairs;    // [n_lines][2] raw ids (0-based for MatrixMarket)
    unsigned long long *first_err;   // min line index with an error status
    int *overflow;     // an accepted edge-list id exceeds int64
};

__global__ void parse_lines_kernel(ParseArgs A) {
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < A.n_lines;
         l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = A.starts[l];
        const int64_t hi = l + 1 < A.n_lines ? A.starts[l + 1] : A.n;
        IntParse tok[2];
        int ntok = 0;
        bool in_tok = false;
        uint32_t first = 0;   // first non-space code point of the line
        for (int64_t p = lo; p < hi;) {
            int len;
            const uint32_t c = decode(A.t, p, &len);
            p += len;
            if (is_space(c)) {
                in_tok = false;
                continue;
            }
            if (!in_tok) {
                in_tok = true;
                if (ntok == 0) first = c;
                ++ntok;
                // a comment line (graph.py:143 / 195,224) needs no further tokens
                if (ntok == 1 && (c == '%' || (A.kind == 0 && c == '#'))) break;
                // MatrixMarket reads the first two parts only (graph.py:227-232)
                if (A.kind == 1 && ntok > 2) break;
            }
            if (ntok <= 2) tok[ntok - 1].feed(c);
        }
        int8_t st;
        int64_t u = 0, v = 0;
        if (ntok == 0 || first == '%' || (A.kind == 0 && first == '#')) {
            st = kSkip;
        } else if (A.kind == 0 ? ntok != 2 : ntok < 2) {
            st = kTokens;
        } else if (!tok[0].ok() || !tok[1].ok()) {
            st = kMalformed;
        } else if (A.kind == 0) {
            if (tok[0].negative() || tok[1].negative()) {
                st = kNegative;
            } else {
                st = kPair;
                if (tok[0].big || tok[1].big) atomicOr(A.overflow, 1);
                u = (int64_t)tok[0].mag;
                v = (int64_t)tok[1].mag;
            }
        } else {
            bool in = true;
            for (int k = 0; k < 2; ++k)
                in = in && !tok[k].big && !tok[k].negative() && tok[k].mag >= 1 &&
                     (int64_t)tok[k].mag <= A.rows;
            st = in ? kPair : kRange;
            u = (int64_t)tok[0].mag - 1;
            v = (int64_t)tok[1].mag - 1;
        }
        A.status[l] = st;
        A.pairs[2 * l] = u;
        A.pairs[2 * l + 1] = v;
        if (st >= kTokens) atomicMin(A.first_err, (unsigned long long)l);
    }
}

// MatrixMarket "more than the declared entries" (graph.py:225-226): the first
// non-skipped line whose rank among non-skipped lines is `declared`.
__global__ void mm_excess_kernel(const int8_t *status, const int64_t *rank, int64_t n_lines,
                                 int64_t declared, unsigned long long *first_excess) {
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n_lines;
         l += (int64_t)gridDim.x * blockDim.x)
        if (status[l] != kSkip && rank[l] == declared)
            atomicMin(first_excess, (unsigned long long)l);
}

struct NotSkip {
    __host__ __device__ int64_t operator()(int8_t s) const { return s != kSkip ? 1 : 0; }
};

// ---- sparse-id remap (graph.py:94-100) -----------------------------------------------
__global__ void lower_bound_kernel(int64_t *ids, int64_t m, const int64_t *sorted, int64_t d) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = ids[k];
        int64_t lo = 0, hi = d;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (sorted[mid] < x) lo = mid + 1;
            else hi = mid;
        }
        ids[k] = lo;
    }
}

unsigned grid_for(int64_t items, int block = 256) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, block), sm_count() * 32));
}

}  // namespace
}  // namespace drg

using namespace drg;

extern "C" int drg_text_lines(const uint8_t *text, int64_t nbytes, int mode, int64_t *out_starts,
                              int64_t *out_count, int64_t *out_bad_byte, void *stream) {
    if (nbytes < 0 || (mode != 0 && mode != 1)) return fail(DRG_ERR_INVALID, "bad text arguments");
    if (out_count) *out_count = 0;
    if (out_bad_byte) *out_bad_byte = -1;
    if (nbytes == 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    const int64_t tiles = ceil_div(nbytes, kTileBytes);
    Scratch cnt(st), off(st), tmp(st), bad(st);
    DRG_CUDA(cnt.alloc(sizeof(int64_t) * (size_t)tiles));
    DRG_CUDA(off.alloc(sizeof(int64_t) * (size_t)tiles));
    DRG_CUDA(bad.alloc(sizeof(unsigned long long)));
    if (out_bad_byte) {
        DRG_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
        utf8_check_kernel<<<grid_for(nbytes), 256, 0, st>>>(text, nbytes, bad.as<unsigned long long>());
        DRG_LAUNCHED("utf8_check_kernel");
        unsigned long long b = 0;
        DRG_CUDA(cudaMemcpyAsync(&b, bad.p, sizeof(b), cudaMemcpyDeviceToHost, st));
        DRG_CUDA(cudaStreamSynchronize(st));
        if (b != ~0ull) {
            *out_bad_byte = (int64_t)b;
            return DRG_OK;
        }
    }
    line_count_kernel<<<(unsigned)tiles, kTileThreads, 0, st>>>(text, nbytes, mode, cnt.as<int64_t>());
    DRG_LAUNCHED("line_count_kernel");
    size_t tb = 0;
    DRG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.as<int64_t>(), off.as<int64_t>(), tiles, st));
    DRG_CUDA(tmp.alloc(tb));
    DRG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.as<int64_t>(), off.as<int64_t>(), tiles, st));
    int64_t last[2] = {0, 0};
    DRG_CUDA(cudaMemcpyAsync(&last[0], off.as<int64_t>() + (tiles - 1), sizeof(int64_t),
                             cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaMemcpyAsync(&last[1], cnt.as<int64_t>() + (tiles - 1), sizeof(int64_t),
                             cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    const int64_t total = last[0] + last[1];
    if (out_count) *out_count = total;
    if (out_starts) {
        line_fill_kernel<<<(unsigned)tiles, kTileThreads, 0, st>>>(text, nbytes, mode,
                                                                   off.as<int64_t>(), out_starts);
        DRG_LAUNCHED("line_fill_kernel");
    }
    return DRG_OK;
}

extern "C" int drg_parse_lines(const uint8_t *text, int64_t nbytes, const int64_t *starts,
                               int64_t n_lines, int kind, int64_t rows, int64_t declared,
                               int64_t *out_pairs, int64_t *out_m, int64_t *out_err_line,
                               int32_t *out_err_status, int32_t *out_overflow, void *stream) {
    if (nbytes < 0 || n_lines < 0 || (kind != 0 && kind != 1))
        return fail(DRG_ERR_INVALID, "bad parse arguments");
    *out_m = 0;
    *out_err_line = -1;
    *out_err_status = 0;
    *out_overflow = 0;
    if (n_lines == 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    Scratch status(st), raw(st), flags(st), tmp(st), cnt(st);
    DRG_CUDA(status.alloc((size_t)n_lines));
    DRG_CUDA(raw.alloc(sizeof(int64_t) * 2 * (size_t)n_lines));
    DRG_CUDA(flags.alloc(2 * sizeof(unsigned long long) + sizeof(int) + sizeof(int64_t)));
    unsigned long long *first_err = flags.as<unsigned long long>();
    int *overflow = reinterpret_cast<int *>(first_err + 2);
    DRG_CUDA(cudaMemsetAsync(first_err, 0xff, 2 * sizeof(unsigned long long), st));
    DRG_CUDA(cudaMemsetAsync(overflow, 0, sizeof(int), st));
    ParseArgs A{text, nbytes, starts, n_lines, kind, rows, status.as<int8_t>(), raw.as<int64_t>(),
                first_err, overflow};
    parse_lines_kernel<<<grid_for(n_lines), 256, 0, st>>>(A);
    DRG_LAUNCHED("parse_lines_kernel");
    if (kind == 1) {   // entries beyond the declared count
        Scratch rank(st);
        DRG_CUDA(rank.alloc(sizeof(int64_t) * (size_t)n_lines));
        auto it = thrust::make_transform_iterator(status.as<int8_t>(), NotSkip());
        size_t tb = 0;
        DRG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, it, rank.as<int64_t>(), n_lines, st));
        DRG_CUDA(tmp.alloc(tb));
        DRG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, it, rank.as<int64_t>(), n_lines, st));
        mm_excess_kernel<<<grid_for(n_lines), 256, 0, st>>>(status.as<int8_t>(), rank.as<int64_t>(),
                                                            n_lines, declared, first_err + 1);
        DRG_LAUNCHED("mm_excess_kernel");
    }
    unsigned long long fe[2];
    int ov = 0;
    DRG_CUDA(cudaMemcpyAsync(fe, first_err, sizeof(fe), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaMemcpyAsync(&ov, overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (kind == 1 && fe[1] != ~0ull && fe[1] <= fe[0]) {   // checked before the entry's parts
        *out_err_line = (int64_t)fe[1];
        *out_err_status = 6;
        return DRG_OK;
    }
    if (fe[0] != ~0ull) {
        *out_err_line = (int64_t)fe[0];
        int8_t s = 0;
        DRG_CUDA(cudaMemcpyAsync(&s, status.as<int8_t>() + fe[0], 1, cudaMemcpyDeviceToHost, st));
        DRG_CUDA(cudaStreamSynchronize(st));
        *out_err_status = s;
        return DRG_OK;
    }
    *out_overflow = ov;
    // accepted pairs in line order
    const int64_t *src = raw.as<int64_t>();
    DRG_CUDA(cnt.alloc(sizeof(int64_t)));
    size_t tb = 0;
    // status is kPair or kSkip here: select the 16-byte pairs whose flag is set
    const int4 *pairs16 = reinterpret_cast<const int4 *>(src);
    DRG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, pairs16, status.as<int8_t>(),
                                        reinterpret_cast<int4 *>(out_pairs), cnt.as<int64_t>(),
                                        n_lines, st));
    Scratch tmp2(st);
    DRG_CUDA(tmp2.alloc(tb));
    DRG_CUDA(cub::DeviceSelect::Flagged(tmp2.p, tb, pairs16, status.as<int8_t>(),
                                        reinterpret_cast<int4 *>(out_pairs), cnt.as<int64_t>(),
                                        n_lines, st));
    DRG_CUDA(cudaMemcpyAsync(out_m, cnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    return DRG_OK;
}

extern "C" int drg_id_remap(int64_t *pairs, int64_t m, int remap_sparse, int64_t *out_n,
                            void *stream) {
    *out_n = 0;
    if (m <= 0) return DRG_OK;
    cudaStream_t st = as_stream(stream);
    const int64_t k = 2 * m;
    Scratch sorted(st), uniq(st), cnt(st), tmp(st);
    DRG_CUDA(sorted.alloc(sizeof(int64_t) * (size_t)k));
    DRG_CUDA(uniq.alloc(sizeof(int64_t) * (size_t)k));
    DRG_CUDA(cnt.alloc(sizeof(int64_t)));
    size_t tb1 = 0, tb2 = 0;
    // ids are non-negative: sort as unsigned keys
    const uint64_t *keys = reinterpret_cast<const uint64_t *>(pairs);
    DRG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb1, keys, sorted.as<uint64_t>(), k, 0, 64, st));
    DRG_CUDA(cub::DeviceSelect::Unique(nullptr, tb2, sorted.as<int64_t>(), uniq.as<int64_t>(),
                                       cnt.as<int64_t>(), k, st));
    DRG_CUDA(tmp.alloc(std::max(tb1, tb2)));
    DRG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb1, keys, sorted.as<uint64_t>(), k, 0, 64, st));
    DRG_CUDA(cub::DeviceSelect::Unique(tmp.p, tb2, sorted.as<int64_t>(), uniq.as<int64_t>(),
                                       cnt.as<int64_t>(), k, st));
    int64_t d = 0, mx = 0;
    DRG_CUDA(cudaMemcpyAsync(&d, cnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaMemcpyAsync(&mx, sorted.as<int64_t>() + (k - 1), sizeof(int64_t),
                             cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    if (mx < 0) return fail(DRG_ERR_INVALID, "negative node id");   // sign bit sorts last
    // the reference's lookup table of max id + 1 entries (graph.py:97) cannot exist
    if (remap_sparse && mx > 2 * d && mx == INT64_MAX)
        return fail(DRG_ERR_INVALID, "Maximum allowed dimension exceeded");
    if (remap_sparse && mx > 2 * d) {
        lower_bound_kernel<<<grid_for(k), 256, 0, st>>>(pairs, k, uniq.as<int64_t>(), d);
        DRG_LAUNCHED("lower_bound_kernel");
        *out_n = d;
    } else {
        *out_n = mx + 1;
    }
    return DRG_OK;
}
