"""Coarse-level sampled epochs of the C4 mesh: host enqueue time vs device time of
drg_layout_sampled over T epochs, and the same launches replayed from a CUDA graph.
Diagnostics only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2008_07799_b200.optimizer import prepare_layout  # noqa: E402


def main(name="mesh", T=800):
    sim, opt, hier = bench.params_for(name, T)
    dg = bench.build_workload(name)
    prep = prepare_layout(dg, sim, opt, max_levels=hier.get("max_levels"))
    plan = prep.plan
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for level in range(plan.depth, -1, -1):
        L = plan.levels[level]
        y = torch.randn(L.n, 2, device="cuda") * 10
        plan.sampled_steps(level, y, 0, L.n, 0, T)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.record()
        plan.sampled_steps(level, y, 0, L.n, 0, T)
        t1 = time.perf_counter()
        e.record()
        torch.cuda.synchronize()
        dev = s.elapsed_time(e) * 1e3 / T
        host = (t1 - t0) * 1e6 / T
        side = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                plan.sampled_steps(level, y, 0, L.n, 0, T)
        g.replay()
        torch.cuda.synchronize()
        s.record()
        for _ in range(3):
            g.replay()
        e.record()
        torch.cuda.synchronize()
        gr = s.elapsed_time(e) * 1e3 / (3 * T)
        print(f'{{"level": {level}, "n": {L.n}, "us_per_epoch_device": {dev:.2f}, '
              f'"us_per_epoch_host_enqueue": {host:.2f}, "us_per_epoch_graph": {gr:.2f}}}',
              flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:2])
