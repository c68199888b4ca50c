"""Stage breakdown of one layout_graph call (the bench's e2e) on a workload:
host->device copy, each preprocessing stage (device events), the layout stage,
device->host copy.  Diagnostics only."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2008_07799_b200 as B  # noqa: E402
from paper_2008_07799_b200.graph import DeviceGraph  # noqa: E402
from paper_2008_07799_b200.optimizer import prepare_layout, start_first_order  # noqa: E402


def main(name="mesh"):
    sim, opt, hier = bench.params_for(name, None)
    gh = bench.build_workload(name).to_host()
    ip = torch.from_numpy(gh.indptr).pin_memory()
    ix = torch.from_numpy(gh.indices).pin_memory()
    g = B.Graph(ip.numpy(), ix.numpy())
    kw = dict(max_levels=hier.get("max_levels"), force_levels=hier.get("force_levels"))
    for rep in range(3):
        torch.cuda.synchronize()
        T = {}
        t0 = time.perf_counter()
        order = start_first_order(g.node_count, opt, 16, kw["max_levels"])
        dg = DeviceGraph.from_host(g)
        torch.cuda.synchronize()
        T["h2d_ms"] = (time.perf_counter() - t0) * 1e3
        t1 = time.perf_counter()
        prep = prepare_layout(dg, sim, opt, timed=True, first_order=order, **kw)
        torch.cuda.synchronize()
        T["prepare_wall_ms"] = (time.perf_counter() - t1) * 1e3
        T.update({k: round(v, 2) for k, v in prep.timings.items()})
        t2 = time.perf_counter()
        y = prep.plan.run()
        torch.cuda.synchronize()
        T["layout_ms"] = (time.perf_counter() - t2) * 1e3
        t3 = time.perf_counter()
        out = prep.to_original(y).cpu().numpy().astype(np.float64)
        T["d2h_ms"] = (time.perf_counter() - t3) * 1e3
        T["total_ms"] = (time.perf_counter() - t0) * 1e3
        del prep, out
    print(json.dumps({k: round(v, 2) for k, v in T.items()}))


if __name__ == "__main__":
    main(*sys.argv[1:2])
