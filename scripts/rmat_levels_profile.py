"""C5 R-MAT scale 24: a short layout (``iters`` epochs per level) for an ncu capture of
the draw / apply kernels of every level (the launch order is coarsest level first:
per level one draw launch, then ``iters`` applies).

    python scripts/rmat_levels_profile.py [scale] [iters]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2008_07799_b200 as B  # noqa: E402
from paper_2008_07799_b200 import synthetic  # noqa: E402
from paper_2008_07799_b200.optimizer import prepare_layout  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dg = synthetic.rmat(scale, 16, seed=0)
opt = B.OptimizerParams(neg_samples=5, iters=iters, seed=0, threads=16)
prep = prepare_layout(dg, B.SimilarityParams(k=1, perplexity="auto"), opt, max_levels=5,
                      force_levels=5)
plan = prep.plan
torch.cuda.synchronize()
for lv, L in enumerate(plan.levels):
    S = L.sampled
    print(f"level {lv}: n {L.n} hubs {S.hubs} hot {None if S.hot is None else S.hot.numel()}",
          flush=True)
t = time.perf_counter()
y = plan.run()
torch.cuda.synchronize()
print(f"layout {time.perf_counter() - t:.3f} s for {iters} epochs per level", flush=True)
