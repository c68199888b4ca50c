"""BASELINE C5 final-layout parity at full scale (R-MAT scale 24, 16.8 M nodes, k=1,
M=5, 500 iterations per level, 5 forced levels): the reference arm and the GPU arm
on the same graph (synthetic.rmat_edges: a counter-based generator, identical from
numpy and from the device), P, hierarchy and Y0 per seed, each evaluated with the
oracle's evaluators: KL with a Monte-Carlo Z over a fixed seeded
sample of ordered pairs, NP (metrics.py:114-145, k_eval = 1) on a fixed seeded sample
of nodes of degree 1..2048.

    python scripts/quality_c5.py ref  SEED [THREADS]   # CPU container: oracle layout
    python scripts/quality_c5.py ours SEED [SEED ...]  # GPU box: layout_graph

One JSON line per (arm, seed); the reference run takes ~1.5 h per seed on 8 cores.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402

SCALE = int(os.environ.get("C5_SCALE", 24))
EF, ITERS, LEVELS = 16, int(os.environ.get("C5_ITERS", 500)), 5
Z_PAIRS, NP_NODES, NP_MAXDEG = int(os.environ.get("C5_Z", 100_000_000)), 20_000, 2048


def host_graph():
    from paper_2008_07799_b200 import synthetic
    n = 1 << SCALE
    chunk = 1 << 24
    parts = [synthetic.rmat_edges(SCALE, EF, seed=0, lo=lo, hi=lo + chunk, device="numpy")
             for lo in range(0, EF * n, chunk)]
    return O.from_edges(np.concatenate(parts), n)


def device_graph():
    from paper_2008_07799_b200 import synthetic
    g = synthetic.rmat(SCALE, EF, seed=0, device="host")
    return O.Graph(g.indptr, g.indices), g


def checksum(g) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(g.indptr).tobytes())
    h.update(np.ascontiguousarray(g.indices).tobytes())
    return h.hexdigest()[:16]


def evaluate(og, ns, y):
    deg = np.diff(og.indptr)
    pool = np.flatnonzero((deg >= 1) & (deg <= NP_MAXDEG))
    sample = np.sort(np.random.default_rng(7).choice(pool, min(NP_NODES, len(pool)),
                                                     replace=False))
    kl = O.kl_divergence(ns, y, 2, z_pairs=Z_PAIRS, seed=11)
    npv = O.neighborhood_preservation(og, y, 1, sample=sample)
    return kl, npv


def init_for(n_top, seed):
    rng = np.random.default_rng(O.derive_seed(seed, O.INIT_TAG))
    return rng.normal(0.0, 1e-4, size=(n_top, 2)).astype(np.float32).astype(np.float64)


def main():
    arm = sys.argv[1]
    t0 = time.perf_counter()
    if arm == "ref":
        seeds = [int(sys.argv[2])]
        threads = int(sys.argv[3]) if len(sys.argv) > 3 else (os.cpu_count() or 1)
        og = host_graph()
    else:
        seeds = [int(s) for s in sys.argv[2:]]
        og, bg = device_graph()
    ns = O.build_sparse_similarity(O.all_k_neighborhoods(og, 1), "auto")
    t_graph = time.perf_counter() - t0
    for seed in seeds:
        t1 = time.perf_counter()
        if arm == "ref":
            y, _, _, _ = O.layout_graph(og, k=1, perplexity="auto",
                                        params=O.OptimizerParams(iters=ITERS, seed=seed,
                                                                 threads=threads),
                                        max_levels=LEVELS, force_levels=LEVELS,
                                        init=lambda n_top: init_for(n_top, seed))
        else:
            import paper_2008_07799_b200 as B
            from paper_2008_07799_b200.optimizer import _HIERARCHY_TAG, _derive_seed
            h = B.build_hierarchy(bg, 0.8, 16, _derive_seed(seed, _HIERARCHY_TAG),
                                  max_levels=LEVELS, force_levels=LEVELS)
            y0 = init_for(h.levels[-1].node_count, seed)
            del h
            threads = 16
            y = B.layout_graph(bg, B.SimilarityParams(k=1, perplexity="auto"),
                               B.OptimizerParams(iters=ITERS, seed=seed, threads=threads),
                               max_levels=LEVELS, force_levels=LEVELS,
                               init_positions=y0).positions
        t_layout = time.perf_counter() - t1
        kl, npv = evaluate(og, ns, y)
        print(json.dumps({"workload": "rmat24", "impl": "reference" if arm == "ref" else "sampled",
                          "seed": seed, "kl": kl, "np": npv, "layout_s": t_layout,
                          "threads": threads, "graph_s": t_graph, "graph_sha": checksum(og),
                          "z_pairs": Z_PAIRS, "np_nodes": NP_NODES}), flush=True)


if __name__ == "__main__":
    main()
