"""Final-layout quality parity: GPU layouts vs the reference algorithm (oracle port)
on the same graph, P, hierarchy and initial Y, over many seeds.

    python scripts/quality.py grid 20        # C1, 20 seeds
    python scripts/quality.py rgg 5          # C2, 5 seeds (KL by Monte-Carlo Z, sampled NP)

Prints one JSON line per (workload, impl) with KL / NP medians and spreads
(SURVEY §8(c) evaluators: KL with the unnormalised t-kernel of lp_kernel,
optimizer.py:150-152; NP = metrics.py:114-145).
"""

from __future__ import annotations

import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402

CONFIGS = {
    "grid": dict(k=2, perplexity=30.0, iters=300, max_levels=1, init="uniform", z_pairs=None,
                 np_sample=None),
    "rgg": dict(k=3, perplexity=30.0, iters=500, max_levels=3, init="normal", z_pairs=None,
                np_sample=None),
    "rgg1": dict(k=3, perplexity=30.0, iters=500, max_levels=1, init="normal", z_pairs=None,
                 np_sample=None),
    "mesh_small": dict(k=2, perplexity=50.0, iters=800, max_levels=4, init="normal",
                       z_pairs=None, np_sample=None),
    # BASELINE C3: Barabasi-Albert 1M, k=2 with the neighbour cap 256 (union P)
    "ba": dict(k=2, perplexity=50.0, iters=500, max_levels=None, init="normal", z_pairs=None,
               np_sample=20_000, np_max_degree=2048, cap=256, np_k=1),
    # (NP over 20k sampled nodes of degree <= 2048: a hub's hop set exceeds the device
    # k-NN instrument, and a hub's 2-hop ball is most of the graph)
    # BASELINE C5 at a reduced scale (R-MAT scale 18, 262k nodes): level 0 sampled,
    # the hub-heavy coarse levels gathered -- the mixed plan C5 runs
    "rmat18": dict(k=1, perplexity="auto", iters=500, max_levels=5, force_levels=5,
                   init="normal", z_pairs=None, np_sample=20_000, np_max_degree=2048, np_k=1,
                   np_min_degree=1),   # (isolated nodes score 1 in both arms)
    # C5 at scale 20 (1 M nodes, 5 forced levels)
    "rmat20": dict(k=1, perplexity="auto", iters=500, max_levels=5, force_levels=5,
                   init="normal", z_pairs=None, np_sample=20_000, np_max_degree=2048, np_k=1,
                   np_min_degree=1),
    # BASELINE C4 itself: 120^3 mesh, 1.73 M nodes (the bench workload)
    "mesh": dict(k=2, perplexity=50.0, iters=800, max_levels=4, init="normal",
                 z_pairs=None, np_sample=None),
}


def graph_for(name):
    import paper_2008_07799_b200 as B
    from paper_2008_07799_b200 import synthetic
    if name == "grid":
        g = synthetic.grid(100, 100, device="host")
    elif name in ("rgg", "rgg1"):
        g = synthetic.rgg(200_000, seed=0, device="host")
    elif name == "mesh":
        g = synthetic.mesh3d(120, device="host")
    elif name in ("rmat18", "rmat20"):
        g = synthetic.rmat(int(name[4:]), 16, seed=0, device="host")
    elif name == "ba":
        g = synthetic.barabasi_albert(1_000_000, 4, seed=0, device="host")
    else:
        g = synthetic.mesh3d(40, device="host")
    return O.Graph(g.indptr, g.indices), B.Graph(g.indptr, g.indices)


def init_for(cfg, n, seed):
    rng = np.random.default_rng(O.derive_seed(seed, O.INIT_TAG))
    if cfg["init"] == "uniform":
        return rng.uniform(-1e-4, 1e-4, size=(n, 2)).astype(np.float32).astype(np.float64)
    return rng.normal(0.0, 1e-4, size=(n, 2)).astype(np.float32).astype(np.float64)


def main(name="grid", n_seeds=10, modes=("jacobi", "inplace", "sampled"), evaluator="gpu",
         seed0=0):
    import paper_2008_07799_b200 as B
    from paper_2008_07799_b200 import quality as Q
    cfg = CONFIGS[name]
    og, bg = graph_for(name)
    cap = cfg.get("cap", 0)
    nd = O.all_k_neighborhoods(og, cfg["k"], cap=cap)
    ns = (O.build_capped_similarity(nd, cfg["perplexity"]) if cap
          else O.build_sparse_similarity(nd, cfg["perplexity"]))
    bns = B.SparseSimilarity(ns.indptr, ns.targets, ns.weights, ns.total_mass, ns.sigma, ns.k)
    del nd
    sample = None
    if cfg["np_sample"]:
        deg = np.diff(og.indptr)
        pool = np.flatnonzero((deg <= cfg.get("np_max_degree", deg.max()))
                              & (deg >= cfg.get("np_min_degree", 0)))
        sample = np.sort(np.random.default_rng(7).choice(pool, cfg["np_sample"], replace=False))
    results = {"reference": [], **{m: [] for m in modes}}
    threads = os.cpu_count() if og.node_count > 50_000 else 1
    for seed in range(seed0, seed0 + n_seeds):
        h = O.build_hierarchy(og, 0.8, 16, O.derive_seed(seed, O.HIERARCHY_TAG),
                              max_levels=cfg["max_levels"], force_levels=cfg.get("force_levels"))
        y0 = init_for(cfg, h.levels[-1].node_count, seed)
        t0 = time.perf_counter()
        opt = O.OptimizerParams(iters=cfg["iters"], seed=seed, threads=threads)
        pos, _, _, _ = O.layout_graph(og, k=cfg["k"], perplexity=cfg["perplexity"], params=opt,
                                      max_levels=cfg["max_levels"], init=y0, neighbor_cap=cap,
                                      force_levels=cfg.get("force_levels"))
        t_ref = time.perf_counter() - t0
        runs = {"reference": (pos, t_ref)}
        for m in modes:
            t0 = time.perf_counter()
            upd, _, div = m.partition(":")
            extra = {}
            if upd == "sampledf":   # the fused one-kernel form of "sampled"
                upd, extra = "sampled", {"sampled_fused": True}
            if upd == "sampledL":   # steps under (i, j) locks on plain levels
                upd, extra = "sampled", {"sampled_locks": True}
            if upd == "sampledS":   # negatives from a per-epoch snapshot on every plain level
                upd, extra = "sampled", {"sampled_snapshot": True}
            if upd == "sampledN":   # negatives read live (no snapshot)
                upd, extra = "sampled", {"sampled_snapshot": False}
            if upd == "sampledH":   # plain Hogwild (no locks) on every level
                upd, extra = "sampled", {"sampled_locks": False}
            if upd == "sampledh":   # "sampled" on every level, hub-heavy ones included
                upd, extra = "sampled", {"hub_levels": "sampled"}
            if div and upd == "sampled":
                fine, _, coarse = div.partition(":")
                extra = {**extra, "sampled_concurrency": int(fine)}
                if coarse:
                    extra["sampled_concurrency_coarse"] = int(coarse)
            elif div and upd == "sgather":
                extra = {"att_samples": int(div)}
            if upd == "sampledv":   # the multi-GPU path on W ranks emulated on this GPU
                upd, extra = "sampled", {"virtual_ranks": int(div), "threads": 16,
                                         "shard_min_nodes": 65536}
            elif upd.startswith("sampledvr"):   # ... exchanging every r epochs: sampledvrR:W
                r = int(upd[len("sampledvr"):])
                upd, extra = "sampled", {"virtual_ranks": int(div), "threads": 16,
                                         "shard_exchange_every": r, "shard_min_nodes": 65536}
            elif upd == "sampledvl":   # ... with the lagged (overlapped) exchange
                upd, extra = "sampled", {"virtual_ranks": int(div), "threads": 16,
                                         "shard_lagged": True, "shard_min_nodes": 65536}
            elif upd == "sampledd":   # threads = 1: the deterministic sub-batch form
                upd, extra = "sampled", {"threads": 1}
            elif upd == "sampled":
                extra = {**extra, "threads": 16}
            lay = B.layout_graph(bg, B.SimilarityParams(k=cfg["k"], perplexity=cfg["perplexity"],
                                                        neighbor_cap=cap or None),
                                 B.OptimizerParams(iters=cfg["iters"], seed=seed, update=upd,
                                                   init=cfg["init"], **extra),
                                 max_levels=cfg["max_levels"], init_positions=y0,
                                 force_levels=cfg.get("force_levels"))
            runs[m] = (lay.positions, time.perf_counter() - t0)
        for key, (y, t) in runs.items():
            if evaluator == "gpu":   # device instruments (exact Z, exact-mode k-NN)
                kl = Q.kl_divergence(bns, y, 2, z_pairs=cfg["z_pairs"], seed=11)
                npv = Q.neighborhood_preservation(bg, y, cfg.get("np_k", 2), sample=sample)
            else:
                kl = O.kl_divergence(ns, y, 2, z_pairs=cfg["z_pairs"], seed=11)
                npv = O.neighborhood_preservation(og, y, cfg.get("np_k", 2), sample=sample)
            results[key].append({"seed": seed, "kl": kl, "np": npv, "s": t})
    for key, rs in results.items():
        kls = [r["kl"] for r in rs]
        nps = [r["np"] for r in rs]
        line = {"workload": name, "impl": key, "seeds": len(rs),
                "kl_median": statistics.median(kls), "kl_min": min(kls), "kl_max": max(kls),
                "np_median": statistics.median(nps), "np_min": min(nps), "np_max": max(nps),
                "kl_mean": statistics.fmean(kls), "np_mean": statistics.fmean(nps),
                "kl_sem": statistics.stdev(kls) / len(kls) ** 0.5 if len(kls) > 1 else None,
                "np_sem": statistics.stdev(nps) / len(nps) ** 0.5 if len(nps) > 1 else None,
                "seconds_median": statistics.median(r["s"] for r in rs)}
        if key != "reference":
            ref = results["reference"]
            # paired per-seed differences (same graph, P, hierarchy and Y0 per seed):
            # mean relative gap and its standard error
            for q in ("kl", "np"):
                d = [a[q] / b[q] - 1 for a, b in zip(rs, ref) if b[q] != 0]
                if len(d) > 1:
                    line[f"{q}_paired_rel_mean"] = statistics.fmean(d)
                    line[f"{q}_paired_rel_sem"] = statistics.stdev(d) / len(d) ** 0.5
            line["kl_rel_vs_ref"] = line["kl_median"] / statistics.median(r["kl"] for r in ref) - 1
            line["np_rel_vs_ref"] = line["np_median"] / statistics.median(r["np"] for r in ref) - 1
            line["kl_mean_rel_vs_ref"] = line["kl_mean"] / statistics.fmean(r["kl"] for r in ref) - 1
            line["np_mean_rel_vs_ref"] = line["np_mean"] / statistics.fmean(r["np"] for r in ref) - 1
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "grid", int(a[1]) if len(a) > 1 else 10,
         tuple(a[2].split(",")) if len(a) > 2 else ("jacobi", "inplace", "sampled"),
         a[3] if len(a) > 3 else "gpu", int(a[4]) if len(a) > 4 else 0)
