"""Generate golden vectors by running the REFERENCE package (drgraph) here.

Run in the build container only (it needs /root/reference, read-only):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  The fixtures pin oracle/ (tests/test_oracle_golden.py)
and, through the oracle, the GPU path.  Nothing at test/bench time reads
/root/reference: the vectors travel in the repo.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, REF)

import drgraph  # noqa: E402
from drgraph import optimizer as ropt  # noqa: E402
from drgraph.graph import all_k_neighborhoods, from_edges  # noqa: E402
from drgraph.multilevel import build_hierarchy, coarsen_once  # noqa: E402
from drgraph.optimizer import (OptimizerParams, build_samplers, layout_graph,  # noqa: E402
                               sgd_epoch)
from drgraph.similarity import SimilarityParams, build_sparse_similarity  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def rand_graph(n, m, seed, connect=False):
    rng = np.random.default_rng(seed)
    pairs = set()
    if connect:
        perm = rng.permutation(n)
        for a, b in zip(perm[:-1], perm[1:]):
            pairs.add((min(int(a), int(b)), max(int(a), int(b))))
    while len(pairs) < m:
        u, v = int(rng.integers(0, n)), int(rng.integers(0, n))
        if u != v:
            pairs.add((min(u, v), max(u, v)))
    return from_edges(np.array(sorted(pairs)), node_count=n)


def grid(w, h):
    idx = np.arange(w * h).reshape(h, w)
    e = np.concatenate([np.column_stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()]),
                        np.column_stack([idx[:-1, :].ravel(), idx[1:, :].ravel()])])
    return from_edges(e, node_count=w * h)


def graphs():
    g = {}
    g["p5"] = from_edges(np.column_stack([np.arange(4), np.arange(1, 5)]), node_count=5)
    g["star4"] = from_edges(np.column_stack([np.zeros(4, dtype=int), np.arange(1, 5)]),
                            node_count=5)
    g["iso"] = from_edges(np.array([[0, 1], [1, 2], [3, 4]]), node_count=7)
    g["grid17"] = grid(17, 17)
    g["r60"] = rand_graph(60, 120, seed=1, connect=True)
    g["r200"] = rand_graph(200, 420, seed=11)
    g["r500"] = rand_graph(500, 1100, seed=42, connect=True)
    g["dense80"] = rand_graph(80, 900, seed=5, connect=True)
    return g


def main():
    out = {}
    gs = graphs()
    for name, g in gs.items():
        out[f"g/{name}/indptr"] = g.indptr
        out[f"g/{name}/indices"] = g.indices
        for k in (1, 2, 3):
            nd = all_k_neighborhoods(g, k)
            out[f"nd/{name}/{k}/indptr"] = nd.indptr
            out[f"nd/{name}/{k}/ids"] = nd.ids
            out[f"nd/{name}/{k}/dists"] = nd.dists
            for perp in ("auto", 2.0, 5.0, 30.0):
                if k == 1 and perp != "auto":
                    continue
                ns = build_sparse_similarity(nd, SimilarityParams(k=k, perplexity=perp))
                tag = f"sim/{name}/{k}/{perp}"
                out[tag + "/weights"] = ns.weights
                out[tag + "/sigma"] = ns.sigma
                out[tag + "/total"] = np.array([ns.total_mass])
                out[tag + "/row_masses"] = ns.row_masses()
        # hierarchy maps for a few seeds
        for seed in (0, 7, 123):
            h = build_hierarchy(g, rho=0.8, min_size=4, seed=seed)
            out[f"h/{name}/{seed}/sizes"] = np.array([lv.node_count for lv in h.levels])
            for li, m in enumerate(h.maps):
                out[f"h/{name}/{seed}/map{li}"] = m
            for li, lv in enumerate(h.levels[1:], start=1):
                out[f"h/{name}/{seed}/lvl{li}/indptr"] = lv.indptr
                out[f"h/{name}/{seed}/lvl{li}/indices"] = lv.indices
        # single coarsen with an explicit seed
        coarse, parent = coarsen_once(g, 99)
        out[f"c/{name}/parent"] = parent
        out[f"c/{name}/indptr"] = coarse.indptr
        out[f"c/{name}/indices"] = coarse.indices

    # samplers + bitwise SGD epochs (the reference kernel) on r60 and r500
    for name in ("r60", "r500", "grid17"):
        g = gs[name]
        for k in (1, 2):
            ns = build_sparse_similarity(all_k_neighborhoods(g, k), SimilarityParams(k=k))
            s = build_samplers(ns)
            tag = f"smp/{name}/{k}"
            out[tag + "/pos_rec"] = s.pos_rec
            out[tag + "/pair_rec"] = s.pair_rec
            out[tag + "/neg_rec"] = s.neg_rec
            h = build_hierarchy(g, min_size=8, seed=ropt._derive_seed(3, 1))
            params = OptimizerParams(seed=3, iters=10, neg_samples=5, b=2)
            for level in sorted({0, h.depth}):
                n = h.levels[level].node_count
                pos = np.random.default_rng(20 + level).normal(size=(n, 2))
                out[f"{tag}/sgd/{level}/pos0"] = pos.copy()
                stats = {}
                for t in range(3):
                    sgd_epoch(pos, h, s, params, t, stats)
                out[f"{tag}/sgd/{level}/pos3"] = pos.copy()
                out[f"{tag}/sgd/{level}/evals"] = np.array([stats["distance_evals"]])
                out[f"{tag}/sgd/{level}/depth"] = np.array([h.depth])

    # full layouts, bitwise (threads=1, fixed seed)
    for name, k, iters, seed in (("p5", 1, 20, 7), ("iso", 1, 30, 7), ("r60", 2, 30, 5),
                                 ("grid17", 1, 40, 0), ("r500", 2, 15, 1)):
        g = gs[name]
        lay = layout_graph(g, SimilarityParams(k=k), OptimizerParams(seed=seed, iters=iters))
        tag = f"lay/{name}/{k}/{iters}/{seed}"
        out[tag + "/pos"] = lay.positions
        out[tag + "/levels"] = np.array(lay.stats["levels"])
        out[tag + "/steps"] = np.array([lay.stats["gradient_steps"]])
        out[tag + "/evals"] = np.array([lay.stats["distance_evals"]])

    # derived seeds (SeedSequence chain, optimizer.py:32-34)
    i = 0
    for s in (0, 1, 3, 7, 12345):
        for tags in ((1,), (2,), (3, 1), (4, 0, 0, 0), (4, 2, 5, 1)):
            out[f"ds/{i}/args"] = np.array([s, *tags], dtype=np.int64)
            out[f"ds/{i}/val"] = np.array([ropt._derive_seed(s, *tags)], dtype=np.uint64)
            i += 1
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB "
          f"(drgraph {drgraph.__version__})")


if __name__ == "__main__":
    main()
