// Output formats after the layout: the coordinate file
// (output.py:12-17), the edge-list serialisation (graph.py:246-250) and the SVG
// rendering (output.py:56-108), formatted on the device.
//
// Every record is produced twice by the same device function -- once for its length
// (pass 1, then a CUB scan gives the offsets), once into the output text (pass 2) --
// so the result is one contiguous byte string equal to Python's "\n".join(...).
// Numbers follow Python's formatting exactly:
//   * f"{x:.Nf}": the exact binary value rounded half-to-even at N decimals.  v * 10^N
//     is split exactly into p + e (p = fl(v * 10^N), e = fma(v, 10^N, -p)), and the
//     tie test compares frac(p) - 1/2 with -e, both exact; valid while v * 10^N <
//     2^50 (records outside, never seen in layouts, are flagged for the caller);
//     nan / inf / -inf and the sign of negative zeros as Python prints them;
//   * int(round(255 * c)) colour channels: round-half-even (rint);
//   * the SVG geometry (output.py:70-81, 94-99) with the same IEEE operation order
//     (explicit _rn intrinsics, no contraction), so every coordinate is bitwise the
//     reference's before it is printed.
#include <string.h>

#include <cub/cub.cuh>

#include "common.cuh"

namespace drg {
namespace {

struct Out {
    char *p;
    int n = 0;
    __device__ void ch(char c) {
        if (p) p[n] = c;
        ++n;
    }
    __device__ void str(const char *s) {
        while (*s) ch(*s++);
    }
    __device__ void u64(uint64_t v, int min_digits = 1) {
        char d[20];
        int k = 0;
        do {
            d[k++] = (char)('0' + v % 10);
            v /= 10;
        } while (v);
        while (k < min_digits) d[k++] = '0';
        while (k) ch(d[--k]);
    }
};

// f"{v:.{prec}f}"; returns false when |v| * 10^prec >= 2^50 (not formatted exactly here)
__device__ bool fixed(Out &o, double v, int prec) {
    if (isnan(v)) {
        o.str("nan");
        return true;
    }
    if (isinf(v)) {
        o.str(v < 0 ? "-inf" : "inf");
        return true;
    }
    double scale = 1.0;
    uint64_t div = 1;
    for (int k = 0; k < prec; ++k) {
        scale *= 10.0;
        div *= 10;
    }
    const bool neg = signbit(v);
    const double a = fabs(v);
    const double p = __dmul_rn(a, scale);
    if (!(p < 1125899906842624.0)) return false;   // 2^50
    const double e = fma(a, scale, -p);              // a * scale == p + e exactly
    const double q = floor(p);
    const double d = (p - q) - 0.5;                  // exact where it matters (see above)
    uint64_t N = (uint64_t)q;
    if (d > -e || (d == -e && (N & 1))) ++N;
    if (neg) o.ch('-');
    o.u64(N / div);
    if (prec) {
        o.ch('.');
        o.u64(N % div, prec);
    }
    return true;
}

// ---- coordinate rows: "x y" (output.py:16)
__device__ bool coord_row(Out &o, const double *pos, int64_t i) {
    bool ok = fixed(o, pos[2 * i], 6);
    o.ch(' ');
    ok = fixed(o, pos[2 * i + 1], 6) && ok;
    o.ch('\n');
    return ok;
}

// ---- SVG
struct SvgArgs {
    const double *xs, *ys;
    const int32_t *edges;   // [m][2]
    int64_t m, n;
    double lmin, lrange;
    char line_tail[64];     // '" stroke-width="{edge_width}"/>' ... (host formatted)
    char circle_tail[64];   // '" r="{node_radius}" fill="black"/>'
};

__device__ __forceinline__ double edge_length(const SvgArgs &A, int64_t k) {
    const int32_t u = A.edges[2 * k], v = A.edges[2 * k + 1];
    const double du = __dsub_rn(A.xs[u], A.xs[v]);
    const double dv = __dsub_rn(A.ys[u], A.ys[v]);
    return __dsqrt_rn(__dadd_rn(__dmul_rn(du, du), __dmul_rn(dv, dv)));   // output.py:94-96
}

__device__ void hex2(Out &o, int v) {
    const char *h = "0123456789abcdef";
    o.ch(h[(v >> 4) & 15]);
    o.ch(h[v & 15]);
}

__device__ bool svg_line(Out &o, const SvgArgs &A, int64_t k) {
    const int32_t u = A.edges[2 * k], v = A.edges[2 * k + 1];
    const double len = edge_length(A, k);
    const double t = A.lrange > 0 ? __ddiv_rn(__dsub_rn(len, A.lmin), A.lrange) : 0.0;
    double r, g, b;   // _edge_color (output.py:44-51)
    if (t <= 0.5) {
        const double s = __dmul_rn(2.0, t);
        r = __dsub_rn(1.0, s);
        g = s;
        b = 0.0;
    } else {
        const double s = __dsub_rn(__dmul_rn(2.0, t), 1.0);
        r = 0.0;
        g = __dsub_rn(1.0, s);
        b = s;
    }
    bool ok = true;
    o.str("<line x1=\"");
    ok = fixed(o, A.xs[u], 2) && ok;
    o.str("\" y1=\"");
    ok = fixed(o, A.ys[u], 2) && ok;
    o.str("\" x2=\"");
    ok = fixed(o, A.xs[v], 2) && ok;
    o.str("\" y2=\"");
    ok = fixed(o, A.ys[v], 2) && ok;
    o.str("\" stroke=\"#");
    hex2(o, (int)rint(__dmul_rn(255.0, r)));
    hex2(o, (int)rint(__dmul_rn(255.0, g)));
    hex2(o, (int)rint(__dmul_rn(255.0, b)));
    o.str(A.line_tail);
    o.ch('\n');
    return ok;
}

__device__ bool svg_circle(Out &o, const SvgArgs &A, int64_t i) {
    bool ok = true;
    o.str("<circle cx=\"");
    ok = fixed(o, A.xs[i], 2) && ok;
    o.str("\" cy=\"");
    ok = fixed(o, A.ys[i], 2) && ok;
    o.str(A.circle_tail);
    o.ch('\n');
    return ok;
}

// ---- record kinds
enum Kind { kCoords = 0, kEdges = 1, kSvgLines = 2, kSvgCircles = 3 };

struct RecArgs {
    int kind;
    int64_t count;
    const double *pos;                 // kCoords
    const int64_t *indptr;             // kEdges: CSR, one record per entry with u < v
    const int32_t *indices;
    int64_t n_rows;
    SvgArgs svg;
};

// kEdges: entry e of row u is a record iff u < indices[e]; the row of e by binary search
__device__ int64_t row_of(const int64_t *indptr, int64_t n_rows, int64_t e) {
    int64_t lo = 0, hi = n_rows;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (indptr[mid] <= e) lo = mid;
        else hi = mid;
    }
    return lo;
}

__device__ bool record(Out &o, const RecArgs &A, int64_t r) {
    switch (A.kind) {
        case kCoords: return coord_row(o, A.pos, r);
        case kEdges: {
            const int64_t u = row_of(A.indptr, A.n_rows, r);
            const int32_t v = A.indices[r];
            if (u >= v) return true;   // each edge once, u < v (graph.py:58-63)
            o.u64((uint64_t)u);
            o.ch(' ');
            o.u64((uint64_t)v);
            o.ch('\n');
            return true;
        }
        case kSvgLines: return svg_line(o, A.svg, r);
        default: return svg_circle(o, A.svg, r);
    }
}

__global__ void rec_len_kernel(RecArgs A, int64_t *len, unsigned long long *first_bad) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < A.count;
         r += (int64_t)gridDim.x * blockDim.x) {
        Out o{nullptr};
        if (!record(o, A, r)) atomicMin(first_bad, (unsigned long long)r);
        len[r] = o.n;
    }
}

__global__ void rec_write_kernel(RecArgs A, const int64_t *off, char *out) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < A.count;
         r += (int64_t)gridDim.x * blockDim.x) {
        Out o{out + off[r]};
        record(o, A, r);
    }
}

// SVG geometry: xs, ys of output.py:79-80 and the min / max edge length
__global__ void svg_xy_kernel(const double *pos, int64_t n, double min0, double min1,
                              double off0, double off1, double scale, double size, double *xs,
                              double *ys) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        xs[i] = __dadd_rn(off0, __dmul_rn(__dsub_rn(pos[2 * i], min0), scale));
        ys[i] = __dsub_rn(size, __dadd_rn(off1, __dmul_rn(__dsub_rn(pos[2 * i + 1], min1), scale)));
    }
}

__global__ void svg_len_range_kernel(SvgArgs A, unsigned long long *mn, unsigned long long *mx) {
    // non-negative doubles order like their bit patterns
    unsigned long long lo = ~0ull, hi = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < A.m;
         k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(edge_length(A, k));
        lo = min(lo, b);
        hi = max(hi, b);
    }
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(kFull, lo, o));
        hi = max(hi, __shfl_xor_sync(kFull, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mn, lo);
        atomicMax(mx, hi);
    }
}

__global__ void minmax2_kernel(const double *pos, int64_t n, double *out) {
    // out = {min x, min y, max x, max y} via ordered-int encodings
    __shared__ double s[4][32];
    double v[4] = {INFINITY, INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        v[0] = fmin(v[0], pos[2 * i]);
        v[1] = fmin(v[1], pos[2 * i + 1]);
        v[2] = fmax(v[2], pos[2 * i]);
        v[3] = fmax(v[3], pos[2 * i + 1]);
    }
    for (int o = 16; o; o >>= 1) {
        v[0] = fmin(v[0], __shfl_xor_sync(kFull, v[0], o));
        v[1] = fmin(v[1], __shfl_xor_sync(kFull, v[1], o));
        v[2] = fmax(v[2], __shfl_xor_sync(kFull, v[2], o));
        v[3] = fmax(v[3], __shfl_xor_sync(kFull, v[3], o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0)
        for (int k = 0; k < 4; ++k) s[k][w] = v[k];
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 0; k < 4; ++k)
            for (int j = 1; j < (int)(blockDim.x >> 5); ++j)
                s[k][0] = k < 2 ? fmin(s[k][0], s[k][j]) : fmax(s[k][0], s[k][j]);
        // block results combined by the ordered-int trick
        for (int k = 0; k < 4; ++k) {
            long long b = __double_as_longlong(s[k][0]);
            long long key = b >= 0 ? b : (b ^ 0x7fffffffffffffffLL);   // monotone in the value
            if (k < 2) atomicMin(reinterpret_cast<long long *>(out) + k, key);
            else atomicMax(reinterpret_cast<long long *>(out) + k, key);
        }
    }
}

unsigned grid_for(int64_t items) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, 256), sm_count() * 32));
}

// pass 1 -> scan -> pass 2; *out_len = total bytes; out == NULL: size only
int emit(const RecArgs &A, char *out, int64_t *out_len, int64_t *out_bad, cudaStream_t st) {
    *out_len = 0;
    if (out_bad) *out_bad = -1;
    if (A.count <= 0) return DRG_OK;
    Scratch len(st), off(st), tmp(st), bad(st);
    DRG_CUDA(len.alloc(sizeof(int64_t) * (size_t)A.count));
    DRG_CUDA(off.alloc(sizeof(int64_t) * (size_t)A.count));
    DRG_CUDA(bad.alloc(sizeof(unsigned long long)));
    DRG_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
    rec_len_kernel<<<grid_for(A.count), 256, 0, st>>>(A, len.as<int64_t>(), bad.as<unsigned long long>());
    DRG_LAUNCHED("rec_len_kernel");
    size_t tb = 0;
    DRG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.as<int64_t>(), off.as<int64_t>(), A.count, st));
    DRG_CUDA(tmp.alloc(tb));
    DRG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len.as<int64_t>(), off.as<int64_t>(), A.count, st));
    int64_t last[2];
    unsigned long long b = 0;
    DRG_CUDA(cudaMemcpyAsync(&last[0], off.as<int64_t>() + A.count - 1, 8, cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaMemcpyAsync(&last[1], len.as<int64_t>() + A.count - 1, 8, cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaMemcpyAsync(&b, bad.p, 8, cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    *out_len = last[0] + last[1];
    if (out_bad && b != ~0ull) *out_bad = (int64_t)b;
    if (out) {
        rec_write_kernel<<<grid_for(A.count), 256, 0, st>>>(A, off.as<int64_t>(), out);
        DRG_LAUNCHED("rec_write_kernel");
    }
    return DRG_OK;
}

}  // namespace
}  // namespace drg

using namespace drg;

extern "C" int drg_format_coords(const double *pos, int64_t n, char *out, int64_t *out_len,
                                 int64_t *out_bad_row, void *stream) {
    if (n < 0) return fail(DRG_ERR_INVALID, "n must be >= 0");
    RecArgs A{};
    A.kind = kCoords;
    A.count = n;
    A.pos = pos;
    return emit(A, out, out_len, out_bad_row, as_stream(stream));
}

extern "C" int drg_format_edge_list(const int64_t *indptr, const int32_t *indices, int64_t n,
                                    int64_t nnz, char *out, int64_t *out_len, void *stream) {
    if (n < 0 || nnz < 0) return fail(DRG_ERR_INVALID, "bad graph size");
    RecArgs A{};
    A.kind = kEdges;
    A.count = nnz;
    A.indptr = indptr;
    A.indices = indices;
    A.n_rows = n;
    return emit(A, out, out_len, nullptr, as_stream(stream));
}

extern "C" int drg_bbox2(const double *pos, int64_t n, double *out_bbox, void *stream) {
    if (n <= 0) return fail(DRG_ERR_INVALID, "empty layout");
    cudaStream_t st = as_stream(stream);
    Scratch buf(st);
    DRG_CUDA(buf.alloc(4 * sizeof(double)));
    const long long init[4] = {0x7fffffffffffffffLL, 0x7fffffffffffffffLL,
                               (long long)0x8000000000000000ULL, (long long)0x8000000000000000ULL};
    DRG_CUDA(cudaMemcpyAsync(buf.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    minmax2_kernel<<<grid_for(n), 256, 0, st>>>(pos, n, buf.as<double>());
    DRG_LAUNCHED("minmax2_kernel");
    long long keys[4];
    DRG_CUDA(cudaMemcpyAsync(keys, buf.p, sizeof(keys), cudaMemcpyDeviceToHost, st));
    DRG_CUDA(cudaStreamSynchronize(st));
    for (int k = 0; k < 4; ++k) {
        const long long b = keys[k] >= 0 ? keys[k] : (keys[k] ^ 0x7fffffffffffffffLL);
        double d;
        memcpy(&d, &b, sizeof(d));
        out_bbox[k] = d;
    }
    return DRG_OK;
}

extern "C" int drg_format_svg(const double *pos, int64_t n, const int32_t *edges, int64_t m,
                              double min_x, double min_y, double off_x, double off_y, double scale,
                              double size, const char *line_tail, const char *circle_tail,
                              char *out_lines, int64_t *out_lines_len, char *out_circles,
                              int64_t *out_circles_len, int64_t *out_bad, void *stream) {
    if (n < 0 || m < 0) return fail(DRG_ERR_INVALID, "bad sizes");
    if (strlen(line_tail) >= 64 || strlen(circle_tail) >= 64)
        return fail(DRG_ERR_INVALID, "style strings too long");
    cudaStream_t st = as_stream(stream);
    *out_lines_len = *out_circles_len = 0;
    *out_bad = -1;
    if (n == 0) return DRG_OK;
    Scratch xy(st), rng(st);
    DRG_CUDA(xy.alloc(2 * sizeof(double) * (size_t)n));
    double *xs = xy.as<double>(), *ys = xs + n;
    svg_xy_kernel<<<grid_for(n), 256, 0, st>>>(pos, n, min_x, min_y, off_x, off_y, scale, size, xs, ys);
    DRG_LAUNCHED("svg_xy_kernel");
    RecArgs A{};
    A.svg.xs = xs;
    A.svg.ys = ys;
    A.svg.edges = edges;
    A.svg.m = m;
    A.svg.n = n;
    strcpy(A.svg.line_tail, line_tail);
    strcpy(A.svg.circle_tail, circle_tail);
    if (m > 0) {
        DRG_CUDA(rng.alloc(2 * sizeof(unsigned long long)));
        const unsigned long long init[2] = {~0ull, 0ull};
        DRG_CUDA(cudaMemcpyAsync(rng.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
        svg_len_range_kernel<<<grid_for(m), 256, 0, st>>>(A.svg, rng.as<unsigned long long>(),
                                                          rng.as<unsigned long long>() + 1);
        DRG_LAUNCHED("svg_len_range_kernel");
        unsigned long long mm[2];
        DRG_CUDA(cudaMemcpyAsync(mm, rng.p, sizeof(mm), cudaMemcpyDeviceToHost, st));
        DRG_CUDA(cudaStreamSynchronize(st));
        double lo, hi;
        memcpy(&lo, &mm[0], 8);
        memcpy(&hi, &mm[1], 8);
        A.svg.lmin = lo;
        A.svg.lrange = hi - lo;
        A.kind = kSvgLines;
        A.count = m;
        int64_t bad = -1;
        int rc = emit(A, out_lines, out_lines_len, &bad, st);
        if (rc) return rc;
        if (bad >= 0) *out_bad = bad;
    }
    A.kind = kSvgCircles;
    A.count = n;
    int64_t bad = -1;
    int rc = emit(A, out_circles, out_circles_len, &bad, st);
    if (rc) return rc;
    if (bad >= 0 && *out_bad < 0) *out_bad = m + bad;
    return DRG_OK;
}
