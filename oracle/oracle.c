/*
 * oracle.c -- CPU restatement of the DRGraph layout path (TEST INFRASTRUCTURE).
 *
 * This file is the checker, not the product.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  Every function
 * restates one function of the reference package (drgraph, /root/reference/pkg/src)
 * and cites the file:line it follows.  It is pinned against golden vectors produced
 * by the reference itself (tests/golden/make_golden.py).
 *
 * Build: make -C oracle   (gcc -O2 -ffp-contract=off: no FMA contraction, so the
 * fp64 update sequence of sgd_steps is reproduced bit for bit).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* k-hop neighbourhoods: graph.py:308-366 (per-source deque BFS with a stamp   */
/* array, rows sorted by (dist, id)).  `cap` > 0 is the BASELINE C3 extension: */
/* the row is the (dist,id)-sorted prefix of length cap.                       */
/* ------------------------------------------------------------------------- */

typedef struct {
    const int64_t *indptr; const int32_t *indices; int64_t n; int k; int64_t cap;
    int64_t lo, hi;
    int64_t *counts;            /* count pass output (may be NULL in fill pass) */
    const int64_t *out_indptr;  /* fill pass */
    int32_t *out_ids, *out_dists;
} khop_job;

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

static void *khop_worker(void *arg) {
    khop_job *J = (khop_job *)arg;
    int64_t n = J->n;
    int64_t *stamp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int32_t *depth = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int64_t qcap = 1024;
    int32_t *queue = (int32_t *)malloc(sizeof(int32_t) * qcap);
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * qcap);
    for (int64_t i = 0; i < n; ++i) stamp[i] = -1;
    for (int64_t s = J->lo; s < J->hi; ++s) {
        int64_t qh = 0, qt = 0;
        stamp[s] = s; depth[s] = 0;
        queue[qt++] = (int32_t)s;
        while (qh < qt) {
            int32_t v = queue[qh++];
            int32_t d = depth[v];
            if (d == J->k) break;                      /* graph.py:343-344 */
            for (int64_t e = J->indptr[v]; e < J->indptr[v + 1]; ++e) {
                int32_t u = J->indices[e];
                if (stamp[u] != s) {
                    stamp[u] = s; depth[u] = d + 1;
                    if (qt == qcap) {
                        qcap *= 2;
                        queue = (int32_t *)realloc(queue, sizeof(int32_t) * qcap);
                        keys = (uint64_t *)realloc(keys, sizeof(uint64_t) * qcap);
                    }
                    queue[qt++] = u;
                }
            }
        }
        int64_t found = qt - 1;                         /* the source is queue[0] */
        int64_t row = found;
        if (J->cap > 0 && row > J->cap) row = J->cap;
        if (J->counts) J->counts[s] = row;
        if (J->out_ids && row > 0) {
            for (int64_t q = 1; q < qt; ++q)
                keys[q - 1] = ((uint64_t)(uint32_t)depth[queue[q]] << 32) | (uint32_t)queue[q];
            qsort(keys, (size_t)found, sizeof(uint64_t), cmp_u64);  /* lexsort((ids, ds)) */
            int64_t base = J->out_indptr[s];
            for (int64_t q = 0; q < row; ++q) {
                J->out_ids[base + q] = (int32_t)(keys[q] & 0xffffffffu);
                J->out_dists[base + q] = (int32_t)(keys[q] >> 32);
            }
        }
    }
    free(stamp); free(depth); free(queue); free(keys);
    return NULL;
}

static void run_khop(khop_job *proto, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    khop_job jobs[256];
    int64_t n = proto->n;
    for (int t = 0; t < threads; ++t) {
        jobs[t] = *proto;
        jobs[t].lo = n * t / threads;
        jobs[t].hi = n * (t + 1) / threads;
        pthread_create(&th[t], NULL, khop_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

int orc_khop_count(const int64_t *indptr, const int32_t *indices, int64_t n, int k,
                   int64_t cap, int64_t *counts, int threads) {
    khop_job J = {indptr, indices, n, k, cap, 0, n, counts, NULL, NULL, NULL};
    run_khop(&J, threads);
    return 0;
}

int orc_khop_fill(const int64_t *indptr, const int32_t *indices, int64_t n, int k,
                  int64_t cap, const int64_t *out_indptr, int32_t *out_ids,
                  int32_t *out_dists, int threads) {
    khop_job J = {indptr, indices, n, k, cap, 0, n, NULL, out_indptr, out_ids, out_dists};
    run_khop(&J, threads);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Perplexity bisection: similarity.py:148-199 (_row_perplexity, search_sigma) */
/* and the conditional row similarity.py:110-145 (unshifted table, fsum, the   */
/* underflow fallback).  Rows are given as their per-distance histogram        */
/* hist[i*k + d-1] (BFS rows are sorted by distance, so this is exact).        */
/* ------------------------------------------------------------------------- */

/* Shewchuk exact partial sums, as math.fsum (similarity.py:136, 272). */
static double fsum_add(double *partials, int *np_, double x) {
    int i = 0;
    for (int j = 0; j < *np_; ++j) {
        double y = partials[j];
        if (fabs(x) < fabs(y)) { double t = x; x = y; y = t; }
        double hi = x + y;
        double lo = y - (hi - x);
        if (lo != 0.0) partials[i++] = lo;
        x = hi;
    }
    if (x != 0.0) partials[i++] = x;
    *np_ = i;
    return 0.0;
}

static double fsum_result(const double *partials, int np_) {
    /* round-half-even correction as CPython's math.fsum */
    if (np_ == 0) return 0.0;
    int n = np_;
    double hi = partials[--n];
    double lo = 0.0;
    while (n > 0) {
        double x = hi;
        double y = partials[--n];
        hi = x + y;
        double yr = hi - x;
        lo = y - yr;
        if (lo != 0.0) break;
    }
    if (n > 0 && ((lo < 0.0 && partials[n - 1] < 0.0) || (lo > 0.0 && partials[n - 1] > 0.0))) {
        double y = lo * 2.0;
        double x = hi + y;
        double yr = x - hi;
        if (y == yr) hi = x;
    }
    return hi;
}

/* sum of c copies of v for each (c, v), exactly rounded */
static double fsum_hist(const int64_t *c, const double *v, int k) {
    double partials[256];
    int np_ = 0;
    for (int d = 0; d < k; ++d) {
        for (int64_t r = 0; r < c[d]; ++r) {
            fsum_add(partials, &np_, v[d]);   /* partial count stays < 64 for doubles */
        }
    }
    return fsum_result(partials, np_);
}

static double row_perplexity(const int64_t *counts, const double *dvals, int nb, double sigma) {
    /* similarity.py:148-164 over the nb distinct distances present */
    double inv = 1.0 / (2.0 * sigma * sigma);
    double expo[8], vals[8], terms[8];
    double mx = -INFINITY;
    for (int b = 0; b < nb; ++b) {
        expo[b] = -(dvals[b] * dvals[b]) * inv;
        if (expo[b] > mx) mx = expo[b];
    }
    for (int b = 0; b < nb; ++b) vals[b] = exp(expo[b] - mx);
    double total = 0.0;
    for (int b = 0; b < nb; ++b) total += (double)counts[b] * vals[b];
    for (int b = 0; b < nb; ++b) {
        double p = vals[b] / total;
        terms[b] = p > 0 ? p * log2(p) : 0.0;
    }
    double h = 0.0;
    for (int b = 0; b < nb; ++b) h += (double)counts[b] * terms[b];
    h = -h;
    return pow(2.0, h);
}

/* math.fsum over an array (the total_mass of similarity.py:272, long P arrays). */
double orc_fsum(const double *x, int64_t n) {
    double partials[128];
    int np_ = 0;
    for (int64_t i = 0; i < n; ++i) fsum_add(partials, &np_, x[i]);
    return fsum_result(partials, np_);
}

double orc_search_sigma(const int64_t *counts, const double *dvals, int nb, int64_t n_row,
                        double target_in, double tol, int max_iter, double smin, double smax) {
    if (n_row == 1) return 1.0;                                   /* similarity.py:179-180 */
    double target = target_in < 1.0 ? 1.0 : target_in;
    if (target > (double)n_row) target = (double)n_row;           /* similarity.py:181 */
    double lo = smin, hi = smax, best_sigma = 1.0, best_err = INFINITY;
    for (int it = 0; it < max_iter; ++it) {
        double mid = sqrt(lo * hi);
        double perp = row_perplexity(counts, dvals, nb, mid);
        double err = fabs(perp - target);
        if (err < best_err) { best_err = err; best_sigma = mid; }
        if (err <= tol) break;
        if (perp > target) hi = mid; else lo = mid;
    }
    return best_sigma;
}

typedef struct {
    const int64_t *hist; int64_t n; int k; double perplexity; double tol; int max_iter;
    double smin, smax; int64_t lo, hi; double *sigma; double *pcond;
} sigma_job;

static void *sigma_worker(void *arg) {
    sigma_job *J = (sigma_job *)arg;
    int k = J->k;
    for (int64_t i = J->lo; i < J->hi; ++i) {
        const int64_t *h = J->hist + i * k;
        double *pc = J->pcond + i * k;
        int64_t n_row = 0;
        for (int d = 0; d < k; ++d) n_row += h[d];
        for (int d = 0; d < k; ++d) pc[d] = 0.0;
        J->sigma[i] = 1.0;
        if (n_row == 0) continue;
        int64_t counts[8]; double dvals[8]; int nb = 0;
        for (int d = 0; d < k; ++d) if (h[d] > 0) { counts[nb] = h[d]; dvals[nb] = (double)(d + 1); nb++; }
        double target;
        if (J->perplexity <= 0.0) {                               /* "auto": similarity.py:253-254 */
            int64_t deg = h[0] > 1 ? h[0] : 1;
            target = (double)(n_row < deg ? n_row : deg);
        } else {
            target = J->perplexity;
        }
        double s = orc_search_sigma(counts, dvals, nb, n_row, target, J->tol, J->max_iter,
                                    J->smin, J->smax);
        J->sigma[i] = s;
        /* conditional row, similarity.py:122-145 */
        int dmax = (int)dvals[nb - 1];
        double inv = 1.0 / (2.0 * s * s);
        double table[8];
        for (int d = 1; d <= dmax; ++d) table[d - 1] = exp((double)(-(d * d)) * inv);
        double tv[8]; int64_t tc[8];
        for (int d = 0; d < k; ++d) { tc[d] = h[d]; tv[d] = d < dmax ? table[d] : 0.0; }
        double total = fsum_hist(tc, tv, dmax);
        if (total == 0.0) {
            int dmin = (int)dvals[0];
            pc[dmin - 1] = 1.0 / (double)h[dmin - 1];
        } else {
            for (int d = 0; d < dmax; ++d) pc[d] = h[d] > 0 ? table[d] / total : 0.0;
        }
    }
    return NULL;
}

/* Per-row sigma and per-distance conditional probability pcond[i*k + d-1]
 * (= p_{j|i} for any j at hop distance d from i). */
int orc_sigma_rows(const int64_t *hist, int64_t n, int k, double perplexity, double tol,
                   int max_iter, double smin, double smax, double *sigma, double *pcond,
                   int threads) {
    if (k < 1 || k > 8) return -1;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    sigma_job jobs[256];
    for (int t = 0; t < threads; ++t) {
        sigma_job J = {hist, n, k, perplexity, tol, max_iter, smin, smax,
                       n * t / threads, n * (t + 1) / threads, sigma, pcond};
        jobs[t] = J;
        pthread_create(&th[t], NULL, sigma_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Greedy coarsening with an explicit order: multilevel.py:48-68.             */
/* ------------------------------------------------------------------------- */
int64_t orc_coarsen_with_order(const int64_t *indptr, const int32_t *indices, int64_t n,
                               const int64_t *order, int32_t *parent) {
    for (int64_t i = 0; i < n; ++i) parent[i] = -1;
    int32_t next_id = 0;
    for (int64_t r = 0; r < n; ++r) {
        int64_t v = order[r];
        if (parent[v] != -1) continue;
        parent[v] = next_id;
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
            int32_t u = indices[e];
            if (parent[u] == -1) parent[u] = next_id;
        }
        next_id++;
    }
    return next_id;
}

/* ------------------------------------------------------------------------- */
/* Vose alias construction: optimizer.py:111-139 (stack order reproduced).    */
/* `total` is numpy's weights.sum() passed in so the scaling is identical.    */
/* ------------------------------------------------------------------------- */
int orc_build_alias(const double *weights, int64_t n, double total, double *prob, int32_t *alias) {
    if (n <= 0 || total <= 0) return -1;
    double *scaled = (double *)malloc(sizeof(double) * n);
    int64_t *small = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *large = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t ns = 0, nl = 0;
    double f = (double)n / total;
    for (int64_t i = 0; i < n; ++i) {
        scaled[i] = weights[i] * f;
        prob[i] = 1.0;
        alias[i] = (int32_t)i;
    }
    for (int64_t i = 0; i < n; ++i) if (scaled[i] < 1.0) small[ns++] = i;
    for (int64_t i = 0; i < n; ++i) if (scaled[i] >= 1.0) large[nl++] = i;
    while (ns > 0 && nl > 0) {
        int64_t s = small[--ns];
        int64_t l = large[--nl];
        prob[s] = scaled[s];
        alias[s] = (int32_t)l;
        scaled[l] = (scaled[l] + scaled[s]) - 1.0;
        if (scaled[l] < 1.0) small[ns++] = l; else large[nl++] = l;
    }
    for (int64_t i = 0; i < ns; ++i) prob[small[i]] = 1.0;
    free(scaled); free(small); free(large);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* The SGD step loop: _kernels.py:24-141 (splitmix64 stream, alias picks,      */
/* clipped attractive + repulsive updates on fp64 positions, in place).        */
/* ------------------------------------------------------------------------- */
static inline double next_uniform(uint64_t *state) {
    *state += 0x9E3779B97F4A7C15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z = z ^ (z >> 31);
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

static inline int64_t alias_pick(const double *rec, int64_t n, double u1, double u2) {
    int64_t idx = (int64_t)(u1 * (double)n);
    if (idx >= n) idx = n - 1;
    if (u2 < rec[2 * idx]) return idx;
    return (int64_t)rec[2 * idx + 1];
}

static inline double clipd(double g, double c) {
    if (g > c) return c;
    if (g < -c) return -c;
    return g;
}

int64_t orc_sgd_steps(double *pos, const double *pos_rec, int64_t n_pairs,
                      const int32_t *pair_rec, const double *neg_rec, int64_t n_neg,
                      const int32_t *node_map, int mapped, int64_t n_steps, int neg_count,
                      int b, double gamma, double eps, double clip, double lr, uint64_t seed) {
    uint64_t state = seed;
    int64_t dist_evals = 0;
    double bf = (double)b;
    for (int64_t step = 0; step < n_steps; ++step) {
        double u1 = next_uniform(&state);
        double u2 = next_uniform(&state);
        int64_t e = alias_pick(pos_rec, n_pairs, u1, u2);
        double u3 = next_uniform(&state);
        int64_t i0, j0;
        if (u3 < 0.5) { i0 = pair_rec[2 * e]; j0 = pair_rec[2 * e + 1]; }
        else          { i0 = pair_rec[2 * e + 1]; j0 = pair_rec[2 * e]; }
        int64_t i = mapped ? node_map[i0] : i0;
        int64_t j = mapped ? node_map[j0] : j0;
        if (i != j) {
            double dx = pos[2 * i] - pos[2 * j];
            double dy = pos[2 * i + 1] - pos[2 * j + 1];
            double ld2 = dx * dx + dy * dy;
            dist_evals++;
            if (ld2 > 0.0) {
                double pw = 1.0;
                for (int p = 0; p < b - 1; ++p) pw *= ld2;
                double coef = -2.0 * bf * pw / (1.0 + pw * ld2);
                double gx = clipd(coef * dx, clip);
                double gy = clipd(coef * dy, clip);
                pos[2 * i] += lr * gx;
                pos[2 * i + 1] += lr * gy;
                pos[2 * j] -= lr * gx;
                pos[2 * j + 1] -= lr * gy;
            }
        }
        for (int m = 0; m < neg_count; ++m) {
            int64_t target = -1;
            for (int attempt = 0; attempt < 9; ++attempt) {
                u1 = next_uniform(&state);
                u2 = next_uniform(&state);
                int64_t c = alias_pick(neg_rec, n_neg, u1, u2);
                int64_t cm = mapped ? node_map[c] : c;
                if (cm != i && cm != j) { target = cm; break; }
            }
            if (target < 0) continue;
            double dx = pos[2 * i] - pos[2 * target];
            double dy = pos[2 * i + 1] - pos[2 * target + 1];
            double ld2 = dx * dx + dy * dy;
            dist_evals++;
            if (ld2 + eps > 0.0) {
                double pw = 1.0;
                for (int p = 0; p < b - 1; ++p) pw *= ld2;
                double coef = gamma * 2.0 * bf / ((ld2 + eps) * (1.0 + pw * ld2));
                double gx = clipd(coef * dx, clip);
                double gy = clipd(coef * dy, clip);
                pos[2 * i] += lr * gx;
                pos[2 * i + 1] += lr * gy;
                pos[2 * target] -= lr * gx;
                pos[2 * target + 1] -= lr * gy;
            }
        }
    }
    return dist_evals;
}

/* Hogwild epoch over `workers` threads, optimizer.py:325-345: worker w runs
 * counts[w] steps from seeds[w] on the shared position array (lost updates are
 * accepted). */
typedef struct {
    double *pos; const double *pos_rec; int64_t n_pairs; const int32_t *pair_rec;
    const double *neg_rec; int64_t n_neg; const int32_t *node_map; int mapped;
    int64_t n_steps; int neg_count; int b; double gamma, eps, clip, lr; uint64_t seed;
    int64_t evals;
} sgd_job;

static void *sgd_worker(void *arg) {
    sgd_job *J = (sgd_job *)arg;
    J->evals = orc_sgd_steps(J->pos, J->pos_rec, J->n_pairs, J->pair_rec, J->neg_rec, J->n_neg,
                             J->node_map, J->mapped, J->n_steps, J->neg_count, J->b, J->gamma,
                             J->eps, J->clip, J->lr, J->seed);
    return NULL;
}

int64_t orc_sgd_epoch_threads(double *pos, const double *pos_rec, int64_t n_pairs,
                              const int32_t *pair_rec, const double *neg_rec, int64_t n_neg,
                              const int32_t *node_map, int mapped, const int64_t *counts,
                              const uint64_t *seeds, int workers, int neg_count, int b,
                              double gamma, double eps, double clip, double lr) {
    if (workers < 1) workers = 1;
    if (workers > 256) workers = 256;
    pthread_t th[256];
    sgd_job jobs[256];
    for (int w = 0; w < workers; ++w) {
        sgd_job J = {pos, pos_rec, n_pairs, pair_rec, neg_rec, n_neg, node_map, mapped,
                     counts[w], neg_count, b, gamma, eps, clip, lr, seeds[w], 0};
        jobs[w] = J;
    }
    if (workers == 1) {
        sgd_worker(&jobs[0]);
        return jobs[0].evals;
    }
    for (int w = 0; w < workers; ++w) pthread_create(&th[w], NULL, sgd_worker, &jobs[w]);
    int64_t total = 0;
    for (int w = 0; w < workers; ++w) { pthread_join(th[w], NULL); total += jobs[w].evals; }
    return total;
}
