"""Per-stage device time of build_level_data (gather plans: P^l aggregation, packing,
alias tables, heavy-row split, sampled tables) for a bench workload.  Diagnostics."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2008_07799_b200 import optimizer as OPT  # noqa: E402


def main(name="rmat"):
    sim, opt, hier = bench.params_for(name, 20)
    dg = bench.build_workload(name)
    prep = OPT.prepare_layout(dg, sim, opt, max_levels=hier.get("max_levels"),
                              force_levels=hier.get("force_levels"))
    ds, dh = prep.similarity, prep.hierarchy
    T = {}

    def tick(k, t0):
        torch.cuda.synchronize()
        T[k] = T.get(k, 0.0) + (time.perf_counter() - t0) * 1e3
        return time.perf_counter()

    for rep in range(2):
        T.clear()
        t = time.perf_counter()
        ip, tg, P, R = ds.indptr, ds.targets, ds.weights, ds.row_mass
        Wn = OPT.device_negative_weights(R, opt.neg_power)
        t = tick("neg_weights", t)
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
            OPT.pack_level(ip, tg, P, R, Wn, 1.0 / total, n_l)
            t = tick(f"pack_{level}", t)
            OPT.heavy_split(ip)
            t = tick(f"heavy_{level}", t)
            OPT.build_sampled_tables(ip, tg, P, R)
            t = tick(f"sampled_{level}", t)
            deg = (ip[1:] - ip[:-1])
            T[f"maxrow_{level}"] = int(deg.max())
            T[f"rows_over_512_{level}"] = int((deg > 512).sum())
        print(rep, {k: round(v, 2) if isinstance(v, float) else v for k, v in T.items()}, flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:]))
