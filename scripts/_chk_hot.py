import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2008_07799_b200 as B
from oracle import oracle as O
from paper_2008_07799_b200.graph import DeviceGraph
from paper_2008_07799_b200.optimizer import prepare_layout
rng = np.random.default_rng(8)
n = 20_001
hub = np.column_stack([np.zeros(n - 1, dtype=np.int64), np.arange(1, n)])
g = O.from_edges(np.concatenate([hub, rng.integers(1, n, size=(4000, 2))]), n)
gg = B.Graph(np.asarray(g.indptr, dtype=np.int64), np.asarray(g.indices, dtype=np.int32))
prep = prepare_layout(DeviceGraph.from_host(gg), B.SimilarityParams(k=1),
                      B.OptimizerParams(seed=1, iters=10, threads=4), min_size=16)
plan = prep.plan
S = plan.levels[0].sampled
hot = S.hot
y = rng.normal(0, 1.0, size=(n, 2)).astype(np.float32)
t = 2
_, gamma, _ = plan._level_args(0)
d = plan.sampled_draws(0, 0, n, t)[0]
for lr0 in (1.0, 0.02):
    plan.opt.lr0 = lr0
    want = O.drawn_steps(y.astype(np.float64), d.cpu().numpy(), lr0 * (1.0 - t / 10), gamma, 1e-3, 5.0, plan.opt.b)
    for label, h in (("hot", hot), ("plain", None)):
        S.hot = h
        yd = torch.from_numpy(y).cuda()
        plan.sampled_steps(0, yd, 0, n, t, 1, max_threads=1)
        got = yd.cpu().numpy()
        print(lr0, label, float(np.abs(got - want).max()), float(np.median(np.abs(got - want))))
