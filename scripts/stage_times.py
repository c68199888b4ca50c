"""Wall time of every stage of the device pipeline (synchronised), for profiling."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2008_07799_b200 as B  # noqa: E402
from paper_2008_07799_b200 import optimizer as OPT, synthetic  # noqa: E402
from paper_2008_07799_b200.graph import device_components, device_k_neighborhoods  # noqa: E402
from paper_2008_07799_b200.multilevel import device_build_hierarchy  # noqa: E402
from paper_2008_07799_b200.similarity import device_similarity  # noqa: E402

T = {}


def tick(name, t0):
    torch.cuda.synchronize()
    T[name] = round((time.perf_counter() - t0) * 1e3, 2)
    return time.perf_counter()


def main(name="mesh"):
    import bench
    sim, opt, hier = bench.params_for(name, 100)
    for rep in range(2):
        t = time.perf_counter()
        dg = bench.build_workload(name)
        t = tick("generate", t)
        gh = dg.to_host()
        t = tick("d2h_graph", t)
        dg = B.DeviceGraph.from_host(gh)
        t = tick("h2d_graph_pageable", t)
        device_components(dg)
        t = tick("components", t)
        nd = device_k_neighborhoods(dg, sim.k)
        t = tick("khop", t)
        ds = device_similarity(nd, sim)
        t = tick("similarity", t)
        dh = device_build_hierarchy(dg, 0.8, 16, 123, hier.get("max_levels"),
                                    hier.get("force_levels"))
        t = tick("hierarchy", t)
        R = ds.row_mass
        Wn = OPT.device_negative_weights(R, 0.75)
        t = tick("neg_weights", t)
        ip, tg, P = ds.indptr, ds.targets, ds.weights
        for level in range(dh.depth + 1):
            n_l = dh.levels[level].node_count
            if level > 0:
                parent = dh.maps[level - 1]
                ip, tg, P = OPT._aggregate_pairs(ip, tg, P, parent, n_l)
                t = tick(f"agg_pairs_{level}", t)
                R = OPT._aggregate_nodes(R, parent, n_l)
                Wn = OPT._aggregate_nodes(Wn, parent, n_l)
                t = tick(f"agg_nodes_{level}", t)
            alias, total = OPT._alias_device(Wn)
            t = tick(f"alias_{level}", t)
            OPT.pack_level(ip, tg, P, R, Wn, 1.0 / total, n_l, sort_rows=False)
            t = tick(f"pack_{level}", t)
        print(rep, T, flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:]))
