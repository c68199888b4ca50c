"""Repeatability of the reduced-C2 locked layouts (tests/test_gpu_quality.py's setup):
per-seed NP of the reference and of several GPU variants, repeated."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
import paper_2008_07799_b200 as B
from paper_2008_07799_b200 import quality as Q, synthetic

g = synthetic.rgg(50_000, seed=0, device="host")
og, bg = O.Graph(g.indptr, g.indices), B.Graph(g.indptr, g.indices)
nd = O.all_k_neighborhoods(og, 3)
ns = O.build_sparse_similarity(nd, 30.0)
bns = B.SparseSimilarity(ns.indptr, ns.targets, ns.weights, ns.total_mass, ns.sigma, ns.k)
seeds = list(range(700, 700 + int(sys.argv[1]) if len(sys.argv) > 1 else 710))
variants = {"locked n/1": dict(threads=16),
            "locked n/1 (again)": dict(threads=16),
            "locked n/4,n/1": dict(threads=16, sampled_concurrency=4, sampled_concurrency_coarse=1),
            "locked n/16,n/4": dict(threads=16, sampled_concurrency=16, sampled_concurrency_coarse=4),
            "hogwild n/256": dict(threads=16, sampled_locks=False),
            "deterministic": dict(threads=1)}
out = {k: [] for k in variants}
ref = []
for seed in seeds:
    h = O.build_hierarchy(og, 0.8, 16, O.derive_seed(seed, O.HIERARCHY_TAG), max_levels=3)
    rng = np.random.default_rng(O.derive_seed(seed, O.INIT_TAG))
    y0 = rng.normal(0.0, 1e-4, (h.levels[-1].node_count, 2)).astype(np.float32).astype(np.float64)
    r, _, _, _ = O.layout_graph(og, k=3, perplexity=30.0,
                                params=O.OptimizerParams(iters=500, seed=seed, threads=16),
                                max_levels=3, init=y0)
    ref.append((Q.kl_divergence(bns, r, 2), Q.neighborhood_preservation(bg, r, 2)))
    for name, kw in variants.items():
        y = B.layout_graph(bg, B.SimilarityParams(k=3, perplexity=30.0),
                           B.OptimizerParams(iters=500, seed=seed, **kw), max_levels=3,
                           init_positions=y0).positions
        out[name].append((Q.kl_divergence(bns, y, 2), Q.neighborhood_preservation(bg, y, 2)))
    print(seed, "ref np %.4f" % ref[-1][1], {k: round(v[-1][1], 4) for k, v in out.items()}, flush=True)
ref = np.array(ref)
for name, rows in out.items():
    rows = np.array(rows)
    d = rows[:, 1] / ref[:, 1] - 1
    print(json.dumps({"variant": name, "seeds": len(seeds),
                      "kl_gap_median": float(np.median(rows[:, 0]) / np.median(ref[:, 0]) - 1),
                      "np_gap_mean": float(d.mean()), "np_gap_sem": float(d.std(ddof=1) / np.sqrt(len(d))),
                      "np_gap_min": float(d.min()), "np_gap_max": float(d.max())}), flush=True)
