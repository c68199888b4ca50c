"""Final-layout parity (north star: KL and k-NN neighbourhood preservation of the
final layout within 2% of the reference's; SURVEY §8(d) parity protocol).

Same graph, P, hierarchy and initial Y per seed for both arms; the reference arm
is the oracle port of the reference's step loop (oracle.c, pinned bit for bit to
the reference's own layouts by tests/test_oracle_golden.py) on this box's host
cores; KL with the reference's unnormalised t-kernel and exact Z, NP =
metrics.py:114-145 with k_eval = 2.

The reference's own seed-to-seed spread of NP is ~13% per layout;
the paired per-seed gap between two layouts of the same seed is as wide (-30% ..
+40% on the reduced C2, for every GPU form AND between two runs of the reference's
own Hogwild: scripts/diag_c2_locks.py).  So the NP gap is asserted as "consistent
with |gap| <= 2%": the paired mean relative gap over the seeds must lie within 2% +
3 standard errors (a 2-sigma bar fails a faithful run about once in 100; 40 seeds
keep the bar near 8%, below the -11.6% a Hogwild run without the locks shows).  KL
(spread ~0.3%) is asserted within 2% directly.
"""

from __future__ import annotations

import os
import statistics

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2008_07799_b200")


def _arms(og, bg, k, perplexity, iters, max_levels, init, seeds, threads_ours):
    from paper_2008_07799_b200 import quality as Q
    nd = O.all_k_neighborhoods(og, k)
    ns = O.build_sparse_similarity(nd, perplexity)
    bns = B.SparseSimilarity(ns.indptr, ns.targets, ns.weights, ns.total_mass, ns.sigma, ns.k)
    host_threads = os.cpu_count() if og.node_count > 20_000 else 1
    rows = []
    for seed in seeds:
        h = O.build_hierarchy(og, 0.8, 16, O.derive_seed(seed, O.HIERARCHY_TAG),
                              max_levels=max_levels)
        rng = np.random.default_rng(O.derive_seed(seed, O.INIT_TAG))
        n_top = h.levels[-1].node_count
        y0 = (rng.uniform(-1e-4, 1e-4, (n_top, 2)) if init == "uniform"
              else rng.normal(0.0, 1e-4, (n_top, 2))).astype(np.float32).astype(np.float64)
        ref, _, _, _ = O.layout_graph(og, k=k, perplexity=perplexity,
                                      params=O.OptimizerParams(iters=iters, seed=seed,
                                                               threads=host_threads),
                                      max_levels=max_levels, init=y0)
        ours = B.layout_graph(bg, B.SimilarityParams(k=k, perplexity=perplexity),
                              B.OptimizerParams(iters=iters, seed=seed, init=init,
                                                threads=threads_ours),
                              max_levels=max_levels, init_positions=y0).positions
        rows.append([Q.kl_divergence(bns, y, 2) for y in (ref, ours)]
                    + [Q.neighborhood_preservation(bg, y, 2) for y in (ref, ours)])
    return np.array(rows)


def _check(rows):
    kl_ref, kl_ours, np_ref, np_ours = rows.T
    kl_gap = float(np.median(kl_ours) / np.median(kl_ref) - 1)
    d = np_ours / np_ref - 1
    np_gap, np_se = float(d.mean()), float(d.std(ddof=1) / np.sqrt(len(d)))
    assert abs(kl_gap) <= 0.02, kl_gap
    assert abs(np_gap) <= 0.02 + 3 * np_se, (np_gap, np_se, kl_gap)
    return kl_gap, np_gap, np_se


@pytest.mark.parametrize("threads", [1, 16])
def test_c1_grid_final_layout_parity(threads):
    """BASELINE C1: 100 x 100 grid, k=2, perplexity 30, 300 iterations, single level,
    uniform init; 40 seeds; threads = 1 (deterministic sub-batches, the default) and
    threads = 16 (steps under (i, j) locks, n/2 in flight)."""
    from paper_2008_07799_b200 import synthetic
    g = synthetic.grid(100, 100, device="host")
    og, bg = O.Graph(g.indptr, g.indices), B.Graph(g.indptr, g.indices)
    rows = _arms(og, bg, 2, 30.0, 300, 1, "uniform", range(5000, 5040), threads)
    print("C1, threads", threads, _check(rows))


@pytest.mark.parametrize("threads", [1, 16])
def test_c2_reduced_rgg_final_layout_parity(threads):
    """BASELINE C2 reduced to 50 000 points (mean degree 10), k=3, perplexity 30,
    500 iterations, 3 levels; 40 seeds; threads = 1 (the default, deterministic) and
    threads = 16 (steps under (i, j) locks on every level)."""
    from paper_2008_07799_b200 import synthetic
    g = synthetic.rgg(50_000, seed=0, device="host")
    og, bg = O.Graph(g.indptr, g.indices), B.Graph(g.indptr, g.indices)
    rows = _arms(og, bg, 3, 30.0, 500, 3, "normal", range(700, 740), threads)
    print("reduced C2, threads", threads, _check(rows))
