import os, sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_2008_07799_b200 as B
from conftest import golden_graph
from paper_2008_07799_b200.graph import DeviceGraph
from paper_2008_07799_b200.optimizer import prepare_layout
golden = dict(np.load("tests/golden/golden.npz"))
g = golden_graph(golden, "r500")
gg = B.Graph(np.asarray(g.indptr, dtype=np.int64), np.asarray(g.indices, dtype=np.int32))
prep = prepare_layout(DeviceGraph.from_host(gg), B.SimilarityParams(k=2),
                      B.OptimizerParams(seed=0, neg_samples=5, iters=10), min_size=8)
plan = prep.plan
n = plan.levels[0].n
rng = np.random.default_rng(12)
y0 = torch.from_numpy(rng.normal(0, 1.0, size=(n, 2)).astype(np.float32)).cuda()
def run(fused, steps, t=2):
    plan.opt.sampled_fused = fused
    y = y0.clone()
    plan.sampled_steps(0, y, 0, steps, t, 1, max_threads=1)
    return y
lo, hi = 1, n
for k in [1, 2, 4, 8, 16, 32, 64, 128, 256, 500]:
    a, b = run(False, k), run(True, k)
    d = float((a - b).abs().max())
    print(k, d)
    if d > 1e-5:
        break
# find first diverging step
prev_ok = 0
for k in range(1, n + 1):
    a, b = run(False, k), run(True, k)
    if float((a - b).abs().max()) > 1e-5:
        print("first diverging n_steps", k)
        d = plan.sampled_draws(0, 0, n, 2)[0].cpu().numpy()
        print("split draws of step", k - 1, d[:, k - 1])
        a0, b0 = run(False, k - 1), run(True, k - 1)
        moved_split = torch.nonzero((a - a0).abs().sum(1) > 0).flatten().tolist()
        moved_fused = torch.nonzero((b - b0).abs().sum(1) > 0).flatten().tolist()
        print("moved split", moved_split, "moved fused", moved_fused)
        break
