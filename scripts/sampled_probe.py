"""Latency probe of the sampled kernel: time level-0 epochs of the mesh with parts of
the step disabled (DRG_SAMPLED_PROBE: 1 = no atomics, 2 = target uniform instead of
the row draw, 3 = both) and at several concurrencies.  Diagnostics only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2008_07799_b200.optimizer import prepare_layout  # noqa: E402


def main(name="mesh"):
    sim, opt, hier = bench.params_for(name, 20)
    dg = bench.build_workload(name)
    prep = prepare_layout(dg, sim, opt, max_levels=hier.get("max_levels"))
    plan = prep.plan
    L = plan.levels[0]
    y = plan.init_positions()
    y = torch.randn(L.n, 2, device="cuda")
    for fused, probe in ((True, "0"), (True, "1"), (False, "0"), (False, "1"), (False, "2")):
        os.environ["DRG_SAMPLED_PROBE"] = probe
        plan.opt.sampled_fused = fused
        for div in (4, 16, 64):
            plan.opt.sampled_concurrency = div
            plan.sampled_steps(0, y, 0, L.n, 5, 2)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            plan.sampled_steps(0, y, 0, L.n, 5, 10)
            e.record()
            torch.cuda.synchronize()
            print(f"{'fused' if fused else 'split'} probe={probe} concurrency=n/{div}: {s.elapsed_time(e) / 10 * 1e3:.1f} us/epoch",
                  flush=True)
    os.environ["DRG_SAMPLED_PROBE"] = "0"


if __name__ == "__main__":
    main(*(sys.argv[1:]))
