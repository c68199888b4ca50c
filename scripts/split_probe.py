"""Split-form timing of the level-0 sampled epoch: the draw pass alone, the update
pass alone (on resident draws), and the overlapped pair as drg_layout_sampled runs
it.  Diagnostics only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2008_07799_b200.optimizer import prepare_layout  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main(name="mesh"):
    sim, opt, hier = bench.params_for(name, 20)
    dg = bench.build_workload(name)
    prep = prepare_layout(dg, sim, opt, max_levels=hier.get("max_levels"))
    plan = prep.plan
    for level in range(plan.depth + 1):
        L = plan.levels[level]
        y = torch.randn(L.n, 2, device="cuda")
        div = opt.sampled_concurrency if level == 0 else opt.sampled_concurrency_coarse
        mt = max(256, L.n // div)
        d = plan.sampled_draws(level, 0, L.n, 5)
        t_draw = timed(lambda: plan.sampled_draws(level, 0, L.n, 5))
        t_apply = timed(lambda: plan.sampled_apply(level, d[0], y, 5, max_threads=mt))
        t_both = timed(lambda: plan.sampled_steps(level, y, 0, L.n, 5, 1))
        t_ten = timed(lambda: plan.sampled_steps(level, y, 0, L.n, 5, 10), 3) / 10
        print(f"level {level} n={L.n}: draws {t_draw:.1f} us, apply {t_apply:.1f} us, "
              f"split epoch (1/call) {t_both:.1f} us, (10/call) {t_ten:.1f} us", flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:]))
