"""Per-level hub share of an R-MAT hierarchy (busiest node's R^l / sum R^l) and the
steps in flight the plan gives each level.

    python scripts/level_shares.py [scale] [levels]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2008_07799_b200 as B  # noqa: E402
from paper_2008_07799_b200 import synthetic  # noqa: E402
from paper_2008_07799_b200.optimizer import prepare_layout, sampled_divisors  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nlev = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dg = synthetic.rmat(scale, 16, seed=0)
opt = B.OptimizerParams(neg_samples=5, iters=1, seed=0, threads=16)
plan = prepare_layout(dg, B.SimilarityParams(k=1, perplexity="auto"), opt, max_levels=nlev,
                      force_levels=nlev).plan
fine, coarse = sampled_divisors(plan.levels[0].n, opt)
for lv, L in enumerate(plan.levels):
    R = L.sampled.mass
    share = float(R.max()) / float(R.sum())
    print(f"scale {scale} level {lv}: n {L.n} share {share:.3e} busiest {share * L.n:.0f} "
          f"hot {L.sampled.hot is not None} threads {plan._steps_in_flight(lv, fine if lv == 0 else coarse)}",
          flush=True)
