/*
 * drgraph_b200.h -- C ABI of the B200-native DRGraph layout path.
 *
 * One shared library (paper_2008_07799_b200/libdrgraph_b200.so, sm_100a) exports
 * every entry point below.  The ABI is plain C: raw DEVICE pointers the caller
 * allocates and owns, sizes as int64_t, and a cudaStream_t passed as `void *`
 * (NULL = legacy default stream).  Every call returns an int status:
 *
 *     DRG_OK (0)            success
 *     DRG_ERR_INVALID (-1)  bad argument             -> Python ValueError
 *     DRG_ERR_CUDA (-2)     CUDA runtime error       -> RuntimeError
 *     DRG_ERR_NONFINITE(-3) non-finite coordinate    -> FloatingPointError
 *     DRG_ERR_UNSUPPORTED(-4) input outside a kernel tier (e.g. a k-hop ball
 *                           larger than the block tier holds) -> RuntimeError
 *     DRG_ERR_NOMEM (-5)    device allocation failed -> MemoryError
 *
 * drg_last_error() returns a thread-local message for the last failure.  No C++
 * exception crosses the ABI.  Variable-size outputs are two-phase (a count call,
 * then a fill into caller-allocated buffers) or take a documented upper bound.
 * Calls that return a host scalar synchronise `stream`; all others are
 * asynchronous on it.  All calls release nothing they did not allocate.
 *
 * Each entry point names the reference function it replaces
 * (/root/reference/pkg/src/drgraph/<file>:<line>).
 */
#ifndef DRGRAPH_B200_H
#define DRGRAPH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DRG_OK 0
#define DRG_ERR_INVALID (-1)
#define DRG_ERR_CUDA (-2)
#define DRG_ERR_NONFINITE (-3)
#define DRG_ERR_UNSUPPORTED (-4)
#define DRG_ERR_NOMEM (-5)

#define DRG_ABI_VERSION 1

/* --- library --------------------------------------------------------------- */
int drg_abi_version(void);
const char *drg_last_error(void);
/* Number of kernels this library has launched since it was loaded. */
uint64_t drg_launch_count(void);

/* --- K1: k-hop neighbourhoods ----------------------------------------------
 * Replaces all_k_neighborhoods (graph.py:308-366) / bfs_k_neighborhood
 * (graph.py:280-305).  Input: canonical CSR (graph.py:27-36): indptr int64[n+1],
 * indices int32[2E], rows sorted.  Output rows hold every node within k hops
 * (excluding the source) sorted by (dist, id); `cap` > 0 keeps the sorted prefix
 * of length cap (BASELINE config C3 extension; cap <= 0 = reference behaviour).
 * Phase 1 writes out_indptr[n+1] (device) and *out_nnz (host); phase 2 fills
 * out_ids[nnz] / out_dists[nnz].  1 <= k <= 6, n < 2^29. */
int drg_khop_count(const int64_t *indptr, const int32_t *indices, int64_t n, int k,
                   int64_t cap, int64_t *out_indptr, int64_t *out_nnz, void *stream);
int drg_khop_fill(const int64_t *indptr, const int32_t *indices, int64_t n, int k,
                  int64_t cap, const int64_t *out_indptr, int32_t *out_ids,
                  int32_t *out_dists, void *stream);
/* bfs_k_neighborhood (graph.py:280-305): one source's row, (dist, id)-sorted, by the
 * global-memory tier (any ball size, any k >= 1).  out_ids == NULL: *out_count (host)
 * only; else out_ids/out_dists (device, capacity entries) receive the row. */
int drg_khop_source(const int64_t *indptr, const int32_t *indices, int64_t n, int k,
                    int64_t source, int32_t *out_ids, int32_t *out_dists, int64_t capacity,
                    int64_t *out_count, void *stream);

/* --- K2 + K3: Gaussian similarity --------------------------------------------
 * Replaces build_sparse_similarity (similarity.py:216-278) with search_sigma
 * (similarity.py:167-199), _row_perplexity (148-164), conditional_similarity_row
 * (122-145), the k=1 / all-ones closed form (202-213) and
 * SparseSimilarity.row_masses (84-91).  Input: a NeighborDistances CSR
 * (graph.py:252-263, mirror-complete rows).  perplexity <= 0 means "auto".
 * Outputs (device): sigma[n], weights[nnz] (pair masses, bitwise symmetric),
 * row_mass[n]; host: *out_total_mass (sum of weights), *out_n_nonisolated. */
int drg_similarity(const int64_t *nd_indptr, const int32_t *nd_ids, const int32_t *nd_dists,
                   int64_t n, int64_t nnz, int k, double perplexity, double tol,
                   int max_iter, double sigma_min, double sigma_max, double *out_sigma,
                   double *out_weights, double *out_row_mass, double *out_total_mass,
                   int64_t *out_n_nonisolated, void *stream);

/* Capped rows (BASELINE C3, k-hop rows truncated to their (dist,id)-sorted prefix):
 * the same per-row bisection and conditional rows, then UNION symmetrisation
 * P_ij = (p_{j|i} + p_{i|j}) / (2 N_ne) with a missing mirror counting 0 (SURVEY
 * §8(a) A6; the reference mis-symmetrises such rows).  The output CSR has rows
 * sorted by target id; out_targets / out_weights must hold 2*nnz entries;
 * *out_nnz (host) is the union size. */
int drg_similarity_union(const int64_t *nd_indptr, const int32_t *nd_ids,
                         const int32_t *nd_dists, int64_t n, int64_t nnz, int k,
                         double perplexity, double tol, int max_iter, double sigma_min,
                         double sigma_max, double *out_sigma, int64_t *out_indptr,
                         int32_t *out_targets, double *out_weights, double *out_row_mass,
                         int64_t *out_nnz, double *out_total_mass, int64_t *out_n_nonisolated,
                         void *stream);

/* --- K4: coarsening ------------------------------------------------------------
 * Replaces coarsen_with_order (multilevel.py:48-79).  `order` (device int64[n])
 * is the visiting permutation (multilevel.py:91 draws it with numpy PCG64; the
 * caller passes the same array).  out_parent[n] = coarse id, dense in seed
 * creation order; *out_n_coarse (host).  Bit-exact with the greedy pass. */
int drg_coarsen(const int64_t *indptr, const int32_t *indices, int64_t n,
                const int64_t *order, int32_t *out_parent, int64_t *out_n_coarse,
                int32_t *out_rounds, void *stream);
/* Coarse CSR (multilevel.py:70-78 + from_edges graph.py:80-125): deduplicated
 * images of the fine edges with different parents, rows sorted.  out_indices
 * must hold nnz(fine) entries (upper bound); *out_nnz (host) is the used size. */
int drg_coarse_graph(const int64_t *indptr, const int32_t *indices, int64_t n,
                     const int32_t *parent, int64_t n_coarse, int64_t *out_indptr,
                     int32_t *out_indices, int64_t *out_nnz, void *stream);
/* compose_maps step (multilevel.py:116-123): out[i] = second[first[i]]. */
int drg_compose_maps(const int32_t *first, const int32_t *second, int64_t n, int32_t *out,
                     void *stream);

/* --- A10: level aggregation ----------------------------
 * P^l from P^{l-1}: sum of pair masses over (parent[i], parent[j]) with
 * parent[i] != parent[j].  Output capacity = nnz (upper bound). */
int drg_aggregate_pairs(const int64_t *indptr, const int32_t *targets, const double *weights,
                        int64_t n, int64_t nnz, const int32_t *parent, int64_t n_coarse,
                        int64_t *out_indptr, int32_t *out_targets, double *out_weights,
                        int64_t *out_nnz, void *stream);
/* out[c] = sum of values[v] over parent[v] == c (every c has >= 1 child). */
int drg_aggregate_nodes(const double *values, const int32_t *parent, int64_t n,
                        int64_t n_coarse, double *out, void *stream);

/* --- A8: negative sampler ------------------------------------------------------
 * Node weights of build_negative_sampler (optimizer.py:243-259): mass^power,
 * zero -> 1e-8 * max, power 0 -> uniform.  out_w[n] device. */
int drg_negative_weights(const double *row_mass, int64_t n, double power, double *out_w,
                         void *stream);
/* Alias table (replaces build_alias_table, optimizer.py:111-139) over weights[n]
 * (device), built on the device by a parallel sweep (prefix sums of light deficits
 * and heavy surpluses + binary search; the same law as Vose's table), packed as
 * uint64 records {float32 threshold (low word), int32 alias (high word)};
 * *out_total (host, may be NULL) receives the weight sum.  n < 2^31. */
int drg_alias_build(const double *weights, int64_t n, uint64_t *out_table, double *out_total,
                    void *stream);

/* --- K7 / K8: layout iterations --------------------------------------------------
 * Pack a level for the gradient kernel: rec[e] = {int32 target, float32 2*n*P[e]},
 * V[a] = n * (R[a] + q_scale * Q[a])  (SURVEY §8(a) A12 expectation-matching
 * weights; Q may be unnormalised negative weights with q_scale = 1 / sum).
 * sort_rows != 0 re-orders each row by target id (locality of the y gathers;
 * needed for (dist,id)-ordered level-0 rows). */
int drg_level_pack(const int64_t *indptr, const int32_t *targets, const double *P,
                   const double *R, const double *Q, double q_scale, int64_t n, int64_t nnz,
                   int sort_rows, uint64_t *out_rec, float *out_V, void *stream);

#define DRG_FLAG_INPLACE 1u   /* Hogwild-style in-place update (y_out == y_in) */

/* Heavy-row split for drg_layout_iters (heavy-tailed rows, e.g. R-MAT hubs): rows
 * listed here are streamed by several warps in chunks of DRG_HEAVY_CHUNK entries
 * whose partial sums the row's warp then adds (deterministic order). */
#define DRG_HEAVY_CHUNK 2048
typedef struct drg_heavy_split {
    const int32_t *slot;        /* [n] heavy index of each row, -1 for normal rows */
    const int32_t *chunk_ptr;   /* [n_heavy + 1] first chunk of each heavy row */
    const int32_t *chunk_row;   /* [n_chunks] row of each chunk */
    const int64_t *chunk_begin; /* [n_chunks] first entry of each chunk */
    int64_t n_chunks;
    float *partial;             /* [2 * n_chunks] scratch for the chunk sums */
} drg_heavy_split;

/* n_iter node-parallel iterations t = t0 .. t0+n_iter-1 of level `level`
 * (replaces the sgd_epoch loop of layout_graph, optimizer.py:310-353, 405-407,
 * and the step kernel _kernels.py:48-141):
 *   y_a += lr_t * ( sum_b W_ab clip(g_att(y_a, y_b)) + V_a sum_m clip(g_rep(y_a, y_cm)) )
 * lr_t = lr0 * max(1 - t/iters, 0); negatives c_m ~ alias table, Philox keyed by
 * (seed, level, t, node, m, attempt), redrawn up to 9 times if c_m == a.
 * Only rows [row_lo, row_hi) are updated (node-range sharding; with n_iter > 1 the
 * range must be a prefix [0, row_hi) and rows past it, never written, must agree in
 * both buffers -- the frozen isolated tail).  Jacobi: reads
 * y_in, writes y_out (ping-pong; the result is in y_out).  With
 * DRG_FLAG_INPLACE, y_in must equal y_out.  neg_idx (optional, n*M int32, -1 =
 * skip) replaces the sampled negatives (parity mode, n_iter must be 1).
 * nonfinite (optional device int, init INT_MAX) receives the first t whose
 * update produced a non-finite coordinate.  heavy (optional) splits long rows. */
int drg_layout_iters(const int64_t *indptr, const uint64_t *rec, const float *V,
                     const uint64_t *alias, int64_t n, int64_t row_lo, int64_t row_hi,
                     float *y_in, float *y_out, int t0, int n_iter, int iters, double lr0,
                     double gamma, double eps, double clip, int b, int M, uint64_t seed,
                     int level, const int32_t *neg_idx, int32_t *nonfinite,
                     const drg_heavy_split *heavy, unsigned flags, void *stream);

/* Host routine (no device work): the visiting order of one coarsening level,
 * numpy's Generator(PCG64).permutation(n) bit for bit (multilevel.py:91), from the
 * bit generator's state (128-bit state and increment, buffered 32-bit half-word) into
 * out[n] (host int32).  Replaces the numpy call on layout_graph's critical path. */
int drg_pcg64_permutation(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                          uint64_t inc_lo, int has_uint32, uint32_t uinteger, int64_t n,
                          int32_t *out);

/* --- reference-faithful sampled epochs (update = "sampled") ----------------------
 * Per-row alias tables over P (optimizer.py:111-139 applied to each row):
 * out_rec[e] = 16-byte {fp32 threshold of bucket e, int32 target of its alias
 * entry, int32 target[e], 0} (out_rec holds 2*nnz uint64); a row sample is
 * e = lo + bucket, then target[e] if coin < threshold else the alias target.  out_rowsum[n] (optional) = row sums of P.  With a Vose table over
 * the row masses this draws a directed pair with probability P_ij, the law of the
 * reference's canonical-pair table plus direction coin (optimizer.py:206-240). */
int drg_row_alias(const int64_t *indptr, const int32_t *targets, const double *P, int64_t n,
                  int64_t nnz, uint64_t *out_rec, double *out_rowsum, void *stream);
/* out_span[i] = {indptr[i], indptr[i+1] - indptr[i]} as two uint32 (requires
 * indptr[n] < 2^32): the sampled draws' per-node row record. */
int drg_row_spans(const int64_t *indptr, int64_t n, uint64_t *out_span, void *stream);
/* n_iter epochs t = t0.. of n_steps steps each, every step being the reference
 * step (_kernels.py:65-140) on the level's positions y (in place, Hogwild):
 * source a ~ src_alias (R^l), collapsed pair (a, a) with probability collapse[a]
 * (collapse = NULL: no collapsed pairs, as at level 0)
 * (pairs inside a coarse node, which the reference draws at level 0 and maps),
 * else b from the row's alias table (targets from rec = the level's {target, W}
 * records); clipped attraction on both ends if i != j; M negatives ~ Q^l redrawn
 * (<= 9) while they hit i or j, both ends moved (float2 atomics).  Q^l is the
 * level's own table: neg_alias (Vose records) over the level's nodes [0, neg_n)
 * and, with probability neg_tail_p, a uniform pick in [neg_n, neg_n + neg_tail_n)
 * (isolated nodes at equal floor weight, numbered last; neg_tail_n = 0: none).
 * Steps step_lo .. step_lo + n_steps - 1 of each epoch run here (a rank's share of
 * the epoch in the multi-GPU mode); at most max_threads steps run concurrently.
 * n: entries of src_alias.  row_span (device uint64 per node, may be NULL): {row start,
 * row length} as two uint32 (drg_row_spans; nnz < 2^32) -- one load per drawn
 * source instead of the two row offsets.  map (device int32, may be NULL): the pair tables are
 * level 0's and the drawn source and target are mapped to level l through map
 * (composed parent maps), the reference's own draw-then-map (_kernels.py:76-81);
 * the negatives drawn from Q^l directly have the law of its draw-then-map (115).
 * flags: DRG_SAMPLED_AGGREGATE combines the updates of a warp's lanes that hit the
 * same node before the atomic (hub-heavy levels); DRG_SAMPLED_FUSED draws inline in
 * the update kernel (one launch per epoch) instead of the default split -- every
 * draw of whole epochs resolved first by a full-occupancy pass on an internal
 * low-priority stream, the updates then replaying them on a high-priority stream,
 * double-buffered so the next epochs' draws overlap the current updates; the work
 * is joined back into `stream`.  Both forms draw identical steps.
 * DRG_SAMPLED_DETERMINISTIC (the reference's threads = 1 contract): each
 * epoch runs as sub-batches of max_threads consecutive steps that read the positions
 * frozen at the sub-batch start and sum their increments in 64-bit fixed point
 * (integer atomics), folded into y after the sub-batch -- bitwise reproducible.
 * n_y: nodes of y (<= 0: n).  evals (device uint64, may be NULL) accumulates the
 * distance evaluations of the reference's counter (_kernels.py:86, 122): steps with
 * i != j plus negatives that found a target.  hot (device int32 [n_hot], may be
 * NULL): hub levels -- up to 32 nodes whose positions each block stages in shared
 * memory (read from there, increments summed there and added to y once per block
 * per round of steps) instead of serialising every step's reduction on their L2
 * lines. */
#define DRG_SAMPLED_AGGREGATE 1
#define DRG_SAMPLED_FUSED 2
#define DRG_SAMPLED_DETERMINISTIC 4
/* hub levels drawn inline: L2 eviction-priority hints on the draws' table reads (for
 * tables far above L2: R-MAT scale 24 +3.5%, BA-1M -7% on its hub level) */
#define DRG_SAMPLED_L2_HINTS 8
/* src_alias points at 32-byte source records (drg_src_records): each source draw
 * reads the Vose bucket, the row span and the collapse probability of both of the
 * bucket's outcomes from one sector (split form only) */
#define DRG_SAMPLED_SRC_RECORDS 16
/* steps under per-node locks on the source i and the attraction partner j: the
 * steps in flight touch disjoint (i, j) pairs, so attraction never reads a position
 * another in-flight step is about to move -- the reference's sequential semantics
 * for the pair (_kernels.py:82-105) at any number of steps in flight; the negatives
 * stay Hogwild.  Try-locks (CAS) released without a fence: the updates of i and j
 * are returning atomics and the release depends on their results.  A step that
 * cannot get both locks retries while the warp's other lanes run, and after 64
 * failures runs unlocked.  Plain levels only (not with AGGREGATE, hot nodes, FUSED
 * or DETERMINISTIC: DRG_ERR_UNSUPPORTED).  Also accepted by drg_sampled_apply. */
#define DRG_SAMPLED_LOCKED 32
/* the negatives' positions are read from a read-only copy of y refreshed before
 * every epoch (their reactions, like every other update, still go to y at once):
 * random gathers and reductions on separate arrays run 1.8x faster than on one
 * (the two L2 partitions keep replicas of read-only lines).  A negative's position
 * is up to one epoch old.  Plain Hogwild levels in the split form only.  For M <= 6
 * the copy is a table of 16-byte records {Q^l bucket v, position of v} and the
 * update pass draws the negatives itself (same counters and records as the draw
 * pass: the same negatives), so a negative costs one random read instead of two
 * and the draw pass resolves only the pairs. */
#define DRG_SAMPLED_SNAPSHOT 64

int drg_layout_sampled(const int64_t *indptr, const uint64_t *row_span, const uint64_t *rec,
                       const uint64_t *row_alias,
                       const uint64_t *src_alias, const float *collapse,
                       const uint64_t *neg_alias, const int32_t *map, int64_t n,
                       int64_t neg_n, int64_t neg_tail_n, double neg_tail_p, float *y,
                       int64_t step_lo,
                       int64_t n_steps, int t0,
                       int n_iter, int iters, double lr0, double gamma, double eps, double clip,
                       int b, int M, uint64_t seed, int level, int64_t max_threads,
                       int flags, int64_t n_y, uint64_t *evals, const int32_t *hot,
                       int n_hot, void *stream);

/* The two halves of the split form, exposed for callers that keep the draws (and
 * for the parity tests).  drg_sampled_draws: out[(e * (2 + M) + f) * n_steps + s]
 * for epochs t0 + e (e < n_epochs) and steps step_lo + s: f = 0 the source i, f = 1
 * the target j (j == i: collapsed pair), f = 2 + m negative m (-1 when all 9
 * attempts hit i or j) -- exactly the steps drg_layout_sampled runs.
 * drg_sampled_apply: one epoch of those steps on y, at most max_threads steps in
 * flight (max_threads = 1: sequential, the reference kernel's order). */
/* 32-byte source records of a source Vose table over nodes [0, n_src) (src_alias
 * as drg_alias_build writes it) for DRG_SAMPLED_SRC_RECORDS: per bucket b,
 * out[4b..4b+3] = {threshold | alias << 32, row start of b | row length of b << 32,
 * row start | row length of the alias, collapse of b | collapse of the alias << 32}
 * (fp32 bits; collapse NULL: 0).  Needs nnz < 2^32.  Replaces the separate
 * alias / drg_row_spans / collapse reads of the reference's source draw
 * (_kernels.py:66-75; optimizer.py:111-139). */
int drg_src_records(const uint64_t *src_alias, int64_t n_src, const int64_t *indptr,
                    const float *collapse, uint64_t *out, void *stream);

int drg_sampled_draws(const int64_t *indptr, const uint64_t *row_span, const uint64_t *row_alias,
                      const uint64_t *src_alias, const float *collapse,
                      const uint64_t *neg_alias, const int32_t *map, int64_t n,
                      int64_t neg_n, int64_t neg_tail_n, double neg_tail_p, int64_t step_lo,
                      int64_t n_steps,
                      int t0, int n_epochs, int M, uint64_t seed, int level, int32_t *out,
                      void *stream);
int drg_sampled_apply(const int32_t *draws, int64_t n_steps, float *y, double lr, double gamma,
                      double eps, double clip, int b, int M, int64_t max_threads, int flags,
                      void *stream);

/* Stochastic gather (update = "sgather"): drg_layout_iters with the attraction
 * SAMPLED -- every node draws S partners b ~ W_a. from its row's alias table
 * (row_alias, from drg_row_alias) and applies wsum[a]/S * clip(g_att) per draw
 * (wsum[a] = sum_b W_ab), plus M negatives as in drg_layout_iters, redrawn if they
 * hit the node or its first partner.  Same buffers, flags and determinism as
 * drg_layout_iters; S + M <= 32. */
int drg_layout_sgather(const int64_t *indptr, const uint64_t *rec, const uint64_t *row_alias,
                       const float *wsum, const float *V, const uint64_t *alias, int64_t n,
                       int64_t row_lo, int64_t row_hi, float *y_in, float *y_out, int t0,
                       int n_iter, int iters, double lr0, double gamma, double eps, double clip,
                       int b, int M, int S, uint64_t seed, int level, const int32_t *neg_idx,
                       int32_t *nonfinite, unsigned flags, void *stream);

/* --- K6: prolongation ---------------------------------------------------------------
 * _layout_radius (optimizer.py:356-358): max distance to the centroid (host). */
int drg_layout_radius(const float *y, int64_t n, double *out_radius, void *stream);
/* prolong (multilevel.py:126-138): y_fine[i] = y_coarse[parent[i]] + N(0, jitter)
 * (Philox Box-Muller keyed by (seed, i); jitter <= 0 copies). */
int drg_prolong(const float *y_coarse, const int32_t *parent, int64_t n_fine, double jitter,
                uint64_t seed, float *y_fine, void *stream);

/* --- multi-GPU sampled epochs ----------------------------
 * One process per GPU; the level's positions partitioned by node range, rank r's
 * rows [bounds[r], bounds[r+1]) in a part buffer every peer maps through CUDA IPC
 * (NVLink / NVSwitch).  Hogwild on that one distributed array, as the reference's
 * workers share one pos (optimizer.py:325-345): a rank runs the steps whose source
 * it owns; source and attraction partner are read and updated in place through
 * the peer table; negatives are read from a replicated snapshot of the epoch-start
 * positions and their reactions summed into a delta array, folded in at the epoch
 * end by a reduce-scatter + all-gather (NCCL, loaded at run time).  rank = -1: one
 * process emulates all `world` parts locally (every rank's steps in one launch).
 * Snapshot / delta layout: node v of part r at r * pad + v - bounds[r]. */
int drg_shard_create(int world, int rank, int64_t capacity, void **out_ctx);
int drg_shard_destroy(void *ctx);
int drg_shard_ipc_handle(void *ctx, uint8_t *out_handle64);
int drg_shard_open_peer(void *ctx, int peer, const uint8_t *handle64);
int drg_nccl_unique_id(uint8_t *out128);
int drg_shard_nccl_init(void *ctx, const uint8_t *uid128);
int drg_shard_level(void *ctx, int64_t n, const int64_t *bounds, float *snap, float *delta,
                    int64_t *out_pad);
int drg_shard_load(void *ctx, const float *y, void *stream);
/* drg_allgather_Y of the survey: every part gathered into y (device [n][2]). */
int drg_shard_store(void *ctx, float *y, void *stream);
int drg_shard_exchange(void *ctx, void *stream);
int drg_shard_fold(void *ctx, float *recv, void *stream);
int drg_shard_read_part(void *ctx, float *out, void *stream);
int drg_shard_epoch(void *ctx, const int64_t *indptr, const uint64_t *row_span,
                    const uint64_t *row_alias,
                    const float *collapse, const uint64_t *neg_alias, const int32_t *map,
                    int64_t n_tab, int64_t neg_n, int64_t neg_tail_n, double neg_tail_p,
                    const int32_t *perm, int nseg,
                    const uint64_t *const *seg_alias, const int64_t *seg_n, const int64_t *seg_lo,
                    const int64_t *step_lo, const int64_t *n_steps, int t, int iters, double lr0,
                    double gamma, double eps, double clip, int b, int M, uint64_t seed, int level,
                    int64_t max_threads, uint64_t *evals, int32_t *out_draws, void *stream);
/* Epochs t0 .. t0 + n_iter - 1 of a sharded level with the exchange after each, in one
 * call (drg_shard_epoch + drg_shard_exchange per epoch, no host round trip): draws K
 * epochs per launch one chunk ahead.  DRG_SHARD_LAGGED overlaps epoch t's exchange with
 * epoch t + 1 (two snapshot / delta buffers): epoch t reads the snapshot of the end of
 * epoch t - 2 at the latest, its reactions are folded in by the end of epoch t + 1 (the
 * emulation, rank -1, runs exactly that worst case).  exchange_every = r > 1 (not
 * lagged): the exchange after every r-th epoch (and the last) only -- negatives read
 * a snapshot up to r epochs old, reactions fold in after up to r epochs.  Needs the
 * NCCL communicator (or rank -1). */
#define DRG_SHARD_LAGGED 1
int drg_shard_run(void *ctx, const int64_t *indptr, const uint64_t *row_span,
                  const uint64_t *row_alias,
                  const float *collapse, const uint64_t *neg_alias, const int32_t *map,
                  int64_t n_tab, int64_t neg_n, int64_t neg_tail_n, double neg_tail_p,
                  const int32_t *perm, int nseg, const uint64_t *const *seg_alias,
                  const int64_t *seg_n, const int64_t *seg_lo, const int64_t *step_lo,
                  const int64_t *n_steps, int t0, int n_iter, int iters, double lr0, double gamma,
                  double eps, double clip, int b, int M, uint64_t seed, int level,
                  int64_t max_threads, int flags, int exchange_every, uint64_t *evals,
                  void *stream);

/* --- single-row / single-interaction drop-ins -----------------------------------
 * precompute_gaussian_table (similarity.py:110-119): out[d-1] = exp(-d^2 / (2 sigma^2)),
 * d = 1..k (device fp64; exp evaluated in double-double and rounded once). */
int drg_gaussian_table(int k, double sigma, double *out, void *stream);
/* search_sigma (similarity.py:167-199) for every row of a (row offsets, hop distances)
 * CSR (device): out_sigma[r] (rows of one entry: 1.0; empty rows untouched). */
int drg_rows_sigma(const int64_t *indptr, const int32_t *dists, int64_t nrows, double perplexity,
                   double tol, int max_iter, double sigma_min, double sigma_max,
                   double *out_sigma, void *stream);
/* conditional_similarity_row (similarity.py:122-145) for every row at bandwidth
 * sigma[r]: out_p[e] = table[d_e] / fsum(row) (math.fsum's correctly rounded sum),
 * uniform over the minimum-distance entries when every value underflows. */
int drg_rows_conditional(const int64_t *indptr, const int32_t *dists, int64_t nrows,
                         const double *sigma, double *out_p, void *stream);
/* attractive_gradient (kind 0, optimizer.py:174-186) / repulsive_gradient (kind 1,
 * 189-203) of n interactions y_i[q] -> y_j[q] (device fp64 [n][2]) into out. */
int drg_gradients(const double *yi, const double *yj, int64_t n, int b, double gamma, double eps,
                  double clip, int kind, double *out, void *stream);

/* --- parity instruments -----------------------------
 * KL(P || Q) terms of a layout y (device fp32 [n][2]) with the unnormalised
 * t-kernel lp_kernel (optimizer.py:150-152): out4 (host) = {sum P log P,
 * sum P log(1 + d^(2b)), sum P, Z = sum_{i != j} 1/(1 + d_ij^(2b))}; Z is exact
 * (tiled all-pairs) when z_pairs <= 0, else a Monte-Carlo estimate over z_pairs
 * uniform ordered pairs.  KL = (out4[0] + out4[1]) / out4[2] + log(out4[3]). */
int drg_kl_terms(const int64_t *indptr, const int32_t *targets, const double *P, int64_t n,
                 const float *y, int b, int64_t z_pairs, uint64_t seed, double *out4,
                 void *stream);

/* Neighbourhood preservation per query node (metrics.py:114-145): Jaccard of the
 * node's k_eval-hop set (hop_indptr/hop_ids, e.g. from drg_khop_*) and its k
 * nearest other layout nodes (k = hop-set size; exact, ties to the lower id, the
 * reference's exact mode metrics.py:77-95); empty hop sets score 1.
 * queries (device int32, NULL = all nodes); out_score (device fp64 [n_queries]),
 * -1 marks a node whose hop set exceeds 3584 entries. */
int drg_neighborhood_preservation(const float *y, int64_t n, const int64_t *hop_indptr,
                                  const int32_t *hop_ids, const int32_t *queries,
                                  int64_t n_queries, double *out_score, void *stream);

/* --- graph construction and diagnostics ---------------------------------------------
 * from_edges (graph.py:80-125): canonical CSR from m (u, v) pairs (device int64
 * [m][2]), self-loops dropped, duplicates and reversed pairs merged, rows sorted.
 * out_indices must hold 2*m entries; *out_nnz (host) = 2 * edge_count.  Ids must
 * lie in [0, n). */
int drg_from_edges(const int64_t *pairs, int64_t m, int64_t n, int64_t *out_indptr,
                   int32_t *out_indices, int64_t *out_nnz, void *stream);
/* --- text ingestion (graph.py:128-243) -----------------------------
 * drg_text_lines: line starts of UTF-8 text (device bytes).  mode 0 = str.splitlines
 * (graph.py:128-131 on the text cli.py:194 reads: \n, \r, \r\n, \v, \f, \x1c-\x1e,
 * U+0085, U+2028, U+2029), mode 1 = "\n" only (text-stream iteration).  *out_count
 * (host) = number of lines (a final break opens no line); out_starts (device int64
 * [*out_count], NULL: count only).  out_bad_byte (host, NULL: no check) = offset of
 * the first byte that is not strict UTF-8 (-1: valid; else nothing else is done). */
int drg_text_lines(const uint8_t *text, int64_t nbytes, int mode, int64_t *out_starts,
                   int64_t *out_count, int64_t *out_bad_byte, void *stream);
/* drg_parse_lines: lines [starts[l], starts[l+1]) (the last ends at nbytes) parsed as
 * kind 0 = edge list (graph.py:134-167: blank and '#'/'%' lines skipped, exactly two
 * int() ids, none negative) or kind 1 = MatrixMarket entry lines (graph.py:218-241:
 * blank and '%' lines skipped, >= 2 parts, 1 <= i, j <= rows, at most `declared`).
 * int() = Python's grammar over Unicode decimal digits with single underscores.
 * out_pairs (device int64 [n_lines][2]) receives the accepted ids in line order
 * (0-based for kind 1), *out_m (host) their count.  The first failing line (index,
 * host *out_err_line, -1 if none) and its status (*out_err_status: 2 token count,
 * 3 malformed integer, 4 negative id, 5 index out of range, 6 beyond the declared
 * entries) let the caller raise the reference's ParseError; *out_overflow (host) = an
 * accepted edge-list id exceeds 2^63 - 1. */
int drg_parse_lines(const uint8_t *text, int64_t nbytes, const int64_t *starts, int64_t n_lines,
                    int kind, int64_t rows, int64_t declared, int64_t *out_pairs, int64_t *out_m,
                    int64_t *out_err_line, int32_t *out_err_status, int32_t *out_overflow,
                    void *stream);
/* drg_id_remap: node count of from_edges without an explicit count (graph.py:90-103)
 * for m device pairs: *out_n (host) = max id + 1, or -- remap_sparse != 0 and max id
 * > 2 * distinct ids -- the distinct count, the ids then compacted in place to their
 * rank among the distinct ids.  A negative id returns DRG_ERR_INVALID. */
int drg_id_remap(int64_t *pairs, int64_t m, int remap_sparse, int64_t *out_n, void *stream);

/* --- output formats (output.py:12-108, graph.py:246-250) -------
 * Each entry is called twice: out == NULL returns the byte count in *out_len (host),
 * then out (device, *out_len bytes) receives the text.  Numbers are formatted as
 * Python formats them (f"{x:.6f}" / f"{x:.2f}": exact round-half-even; nan, inf).
 * drg_format_coords: "x y\n" per node of pos (device fp64 [n][2]) -- write_coords
 * without its "#nodes N" header line.  *out_bad_row (host): first row with a
 * coordinate >= 2^50 / 10^6 in magnitude (not formatted exactly), -1 if none. */
int drg_format_coords(const double *pos, int64_t n, char *out, int64_t *out_len,
                      int64_t *out_bad_row, void *stream);
/* drg_format_edge_list: "u v\n" for every CSR entry with u < v, in CSR order. */
int drg_format_edge_list(const int64_t *indptr, const int32_t *indices, int64_t n, int64_t nnz,
                         char *out, int64_t *out_len, void *stream);
/* drg_bbox2: out_bbox (host) = {min x, min y, max x, max y} of pos (device fp64 [n][2]). */
int drg_bbox2(const double *pos, int64_t n, double *out_bbox, void *stream);
/* drg_format_svg: the <line> records of the m edges (device int32 [m][2], the drawn
 * sample) and the <circle> records of the n nodes of write_svg (output.py:56-108),
 * node positions fitted with the host-computed min / offset / scale / canvas size
 * exactly as output.py:70-80 does; edge colours from the edge length range.
 * line_tail / circle_tail (host strings < 64 bytes): the text after the colour /
 * after cy (the style's formatted widths).  Two outputs as above; *out_bad (host)
 * = first record with an out-of-range number, -1 if none. */
int drg_format_svg(const double *pos, int64_t n, const int32_t *edges, int64_t m, double min_x,
                   double min_y, double off_x, double off_y, double scale, double size,
                   const char *line_tail, const char *circle_tail, char *out_lines,
                   int64_t *out_lines_len, char *out_circles, int64_t *out_circles_len,
                   int64_t *out_bad, void *stream);

/* connected_components (graph.py:369-388): out_labels[n] (device, may be NULL)
 * numbered 0..C-1 in first-seen order (component of the smallest unlabelled id),
 * *out_count (host) = C.  layout_graph uses it for a warning and
 * stats["components"] (optimizer.py:374-378). */
int drg_components(const int64_t *indptr, const int32_t *indices, int64_t n,
                   int32_t *out_labels, int64_t *out_count, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DRGRAPH_B200_H */
