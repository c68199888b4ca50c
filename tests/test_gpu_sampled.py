"""Parity of the default update="sampled" path (split form: drg_sampled_draws ->
drg_sampled_apply) against the oracle.

* the drawn directed pairs follow the level's pair law -- the reference's level-0
  pair draw mapped to level l (_kernels.py:66-81) -- chi-square against the
  oracle's level data (P^l, R^l);
* the drawn negatives follow Q^l with the reference's <= 9 redraws while they hit
  i or j (_kernels.py:106-119), exact per-step law, chi-square;
* given the draws, one step == the reference step (_kernels.py:82-140, oracle
  drawn_steps, fp64) within 1e-5 * max(1, |g|); a whole epoch run sequentially
  (one step in flight) == the oracle's sequential replay;
* the fused kernel (draws inline) runs the same steps as the split form.
"""
import numpy as np
import pytest
import torch
from scipy import stats

import paper_2008_07799_b200 as B
from oracle import oracle as O
from conftest import golden_graph

pytestmark = pytest.mark.gpu

LEVELS = ["finest", "middle", "coarsest"]


def _setup(golden, name="r500", k=2, M=5):
    from paper_2008_07799_b200.graph import DeviceGraph
    from paper_2008_07799_b200.optimizer import prepare_layout
    g = golden_graph(golden, name)
    gg = B.Graph(np.asarray(g.indptr, dtype=np.int64), np.asarray(g.indices, dtype=np.int32))
    prep = prepare_layout(DeviceGraph.from_host(gg), B.SimilarityParams(k=k),
                          B.OptimizerParams(seed=0, neg_samples=M, iters=10), min_size=8)
    assert prep.relabel[0] is None          # oracle level data is in the same ids
    ns = O.build_sparse_similarity(O.all_k_neighborhoods(g, k))
    dh = prep.hierarchy
    oh = O.Hierarchy([lv.to_host() for lv in dh.levels], [m.cpu().numpy() for m in dh.maps],
                     0.8, 8)
    return prep.plan, ns, oh


def _level(plan, pick):
    return {"finest": 0, "middle": plan.depth // 2, "coarsest": plan.depth}[pick]


def _chi2(counts, expected):
    keep = expected > 0
    assert counts[~keep].sum() == 0, "draws outside the support"
    e = expected[keep]
    c = counts[keep]
    e = e * (c.sum() / e.sum())
    return stats.chisquare(c, e).pvalue


@pytest.mark.parametrize("pick", LEVELS)
def test_sampled_pair_law(golden, pick):
    plan, ns, oh = _setup(golden)
    level = _level(plan, pick)
    n = plan.levels[level].n
    ip, tg, P, R, Q = O.level_data(ns, oh, level)
    epochs = max(1, 3_000_000 // n)
    d = plan.sampled_draws(level, 0, n, 2, epochs).cpu().numpy()
    i = d[:, 0, :].ravel().astype(np.int64)
    j = d[:, 1, :].ravel().astype(np.int64)
    counts = np.bincount(i * n + j, minlength=n * n).astype(np.float64)
    expected = np.zeros(n * n)
    rows = np.repeat(np.arange(n), np.diff(ip))
    np.add.at(expected, rows * n + tg, P)
    inner = R - np.bincount(rows, weights=P, minlength=n)          # collapsed pairs (a, a)
    expected[np.arange(n) * n + np.arange(n)] += np.maximum(inner, 0.0)
    if level == 0:
        assert counts[np.arange(n) * n + np.arange(n)].sum() == 0
    assert _chi2(counts, expected) > 1e-6


@pytest.mark.parametrize("pick", LEVELS)
def test_sampled_negative_law(golden, pick):
    plan, ns, oh = _setup(golden)
    level = _level(plan, pick)
    n = plan.levels[level].n
    M = plan.opt.neg_samples
    _, _, _, _, Q = O.level_data(ns, oh, level)
    Q = Q / Q.sum()
    epochs = max(1, 600_000 // n)
    d = plan.sampled_draws(level, 0, n, 5, epochs).cpu().numpy()
    i = d[:, 0, :].ravel().astype(np.int64)
    j = d[:, 1, :].ravel().astype(np.int64)
    q = Q[i] + np.where(j != i, Q[j], 0.0)         # a draw is rejected with prob q
    f = np.where(q < 1, (1 - q ** 9) / np.maximum(1 - q, 1e-300), 9.0)
    exp = Q * f.sum() - np.bincount(i, weights=f * Q[i], minlength=n) \
        - np.bincount(j, weights=np.where(j != i, f * Q[j], 0.0), minlength=n)
    expected = np.concatenate([[np.sum(q ** 9)], exp]) * M
    negs = d[:, 2:, :].transpose(1, 0, 2).reshape(M, -1)
    assert not np.any((negs == i) | (negs == j))
    counts = np.bincount(negs.ravel().astype(np.int64) + 1, minlength=n + 1).astype(np.float64)
    assert _chi2(counts, expected) > 1e-6


def _negative_law_expected(Q, i, j, M, n):
    """Per-step law of the negatives: Q redrawn (<= 9) while it hits i or j."""
    q = Q[i] + np.where(j != i, Q[j], 0.0)
    f = np.where(q < 1, (1 - q ** 9) / np.maximum(1 - q, 1e-300), 9.0)
    exp = Q * f.sum() - np.bincount(i, weights=f * Q[i], minlength=n) \
        - np.bincount(j, weights=np.where(j != i, f * Q[j], 0.0), minlength=n)
    return np.concatenate([[np.sum(q ** 9)], exp]) * M


def test_negative_table_with_isolated_tail():
    """Q^l drawn as NegTable -- Vose over the connected prefix plus a uniform pick in
    the isolated tail (isolated_last numbers the isolated nodes last) -- has the law
    of one table over every node.  The reference's tail weight is a 1e-8 floor; a
    heavy uniform tail (half the top weight) makes the split visible to chi-square."""
    from paper_2008_07799_b200.graph import DeviceGraph
    from paper_2008_07799_b200.optimizer import build_neg_table, prepare_layout
    rng = np.random.default_rng(4)
    n_conn, n_iso = 300, 200
    g = B.from_edges(rng.integers(0, n_conn, size=(900, 2)), n_conn + n_iso)
    prep = prepare_layout(DeviceGraph.from_host(g), B.SimilarityParams(k=1),
                          B.OptimizerParams(seed=1, iters=5, threads=4), max_levels=1)
    plan = prep.plan
    S = plan.levels[0].sampled
    R = S.mass
    n, M = R.numel(), plan.opt.neg_samples
    w = R.pow(0.75)
    W = torch.where(R > 0, w, torch.full_like(w, 0.5 * float(w.max())))
    S.neg = build_neg_table(W, R)
    assert S.neg.tail_n == int((R == 0).sum()) >= n_iso and S.neg.tail_p > 0.1
    assert bool((R[:S.neg.n] > 0).any()) and bool((R[S.neg.n:] == 0).all())
    d = plan.sampled_draws(0, 0, n, 2, 4000).cpu().numpy()
    i = d[:, 0, :].ravel().astype(np.int64)
    j = d[:, 1, :].ravel().astype(np.int64)
    Q = W.cpu().numpy() / float(W.sum())
    expected = _negative_law_expected(Q, i, j, M, n)
    negs = d[:, 2:, :].transpose(1, 0, 2).reshape(M, -1)
    counts = np.bincount(negs.ravel().astype(np.int64) + 1, minlength=n + 1).astype(np.float64)
    assert _chi2(counts, expected) > 1e-6
    # the tail as a whole: its share of the first-attempt draws is tail_p
    tail = (negs >= S.neg.n).mean()
    assert abs(tail - S.neg.tail_p) < 5 * np.sqrt(S.neg.tail_p / negs.size) + 0.01


@pytest.mark.parametrize("b", [1, 2, 3])
@pytest.mark.parametrize("pick", ["finest", "coarsest"])
def test_sampled_drawn_step_parity(golden, b, pick):
    """One step from identical Y and identical draws: |d| <= 1e-5 max(1, |g|)."""
    plan, _, _ = _setup(golden)
    plan.opt = B.OptimizerParams(seed=0, neg_samples=5, iters=10, b=b)
    level = _level(plan, pick)
    n = plan.levels[level].n
    t = 3
    lr = 1.0 - t / 10
    _, gamma, _ = plan._level_args(level)
    d = plan.sampled_draws(level, 0, n, t)[0]
    rng = np.random.default_rng(b)
    y = rng.normal(0, 1.0, size=(n, 2)).astype(np.float32)
    yd = torch.from_numpy(y).cuda()
    for s in range(min(n, 48)):
        out = yd.clone()
        plan.sampled_apply(level, d[:, s:s + 1], out, t)
        got = out.cpu().numpy().astype(np.float64)
        want = O.drawn_steps(y.astype(np.float64), d[:, s:s + 1].cpu().numpy(), lr, gamma,
                             1e-3, 5.0, b)
        g_got, g_want = (got - y) / lr, (want - y) / lr
        assert np.all(np.abs(g_got - g_want) <= 1e-5 * np.maximum(1.0, np.abs(g_want))), s


@pytest.mark.parametrize("pick", ["finest", "coarsest"])
def test_sampled_sequential_epoch_parity(golden, pick):
    """A whole epoch with one step in flight == the oracle's sequential replay."""
    plan, _, _ = _setup(golden)
    level = _level(plan, pick)
    n = plan.levels[level].n
    t = 8
    _, gamma, _ = plan._level_args(level)
    d = plan.sampled_draws(level, 0, n, t)[0]
    rng = np.random.default_rng(7)
    y = rng.normal(0, 1.0, size=(n, 2)).astype(np.float32)
    yd = torch.from_numpy(y).cuda()
    plan.sampled_apply(level, d, yd, t, max_threads=1)
    want = O.drawn_steps(y.astype(np.float64), d.cpu().numpy(), 1.0 - t / 10, gamma, 1e-3, 5.0,
                         plan.opt.b)
    np.testing.assert_allclose(yd.cpu().numpy(), want, rtol=0, atol=1e-4)


def test_split_and_fused_run_the_same_steps(golden):
    plan, _, _ = _setup(golden)
    L = plan.levels[0]
    rng = np.random.default_rng(3)
    y = torch.from_numpy(rng.normal(0, 1.0, size=(L.n, 2)).astype(np.float32)).cuda()
    for s in (0, 1, 17, 250, L.n - 1):
        outs = []
        for fused in (False, True):
            plan.opt.sampled_fused = fused
            out = y.clone()
            plan.sampled_steps(0, out, s, 1, 4, 1)
            outs.append(out)
        plan.opt.sampled_fused = False
        assert not torch.equal(outs[0], y)
        torch.testing.assert_close(outs[0], outs[1], rtol=0, atol=1e-6)
    # a whole split epoch through drg_layout_sampled stays finite and moves y
    a = y.clone()
    plan.sampled_steps(0, a, 0, L.n, 5, 1)
    assert torch.isfinite(a).all() and not torch.equal(a, y)



def test_fused_and_split_epochs_agree_sequentially(golden):
    """With one step in flight the fused kernel and the split draw/apply passes run
    the same steps: over a whole late epoch (small learning rate) the positions
    agree to fp32 round-off amplified by the dynamics (the two kernels contract
    their arithmetic differently), and every node moves in both or in neither."""
    plan, _, _ = _setup(golden)
    n = plan.levels[0].n
    rng = np.random.default_rng(12)
    y0 = torch.from_numpy(rng.normal(0, 1.0, size=(n, 2)).astype(np.float32)).cuda()
    outs = []
    for fused in (False, True):
        plan.opt.sampled_fused = fused
        y = y0.clone()
        plan.sampled_steps(0, y, 0, n, 9, 1, max_threads=1)
        outs.append(y)
    plan.opt.sampled_fused = False
    moved = [(o - y0).abs().sum(1) > 0 for o in outs]
    assert torch.equal(moved[0], moved[1]) and bool(moved[0].any())
    torch.testing.assert_close(outs[0], outs[1], rtol=0, atol=1e-3)


@pytest.mark.parametrize("threads", [1, 256])
def test_hub_level_inline_draws_run_the_drawn_steps(threads):
    """Hub levels (hot nodes staged per block) draw inline (apply_hot_fused_kernel):
    one step in flight, the epoch equals the oracle's sequential replay of exactly
    the steps drg_sampled_draws reports; many in flight, it stays finite and moves
    the hub."""
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
    assert S.hot is not None and S.hubs
    # every step moves the hub: at lr ~ 1 the star's sequential dynamics amplify
    # fp32-vs-fp64 rounding chaotically; at lr0 = 0.02 they stay near-linear
    plan.opt.lr0 = 0.02
    t = 2
    _, gamma, _ = plan._level_args(0)
    d = plan.sampled_draws(0, 0, n, t)[0]
    y = rng.normal(0, 1.0, size=(n, 2)).astype(np.float32)
    yd = torch.from_numpy(y).cuda()
    plan.sampled_steps(0, yd, 0, n, t, 1, max_threads=threads)
    got = yd.cpu().numpy()
    assert np.isfinite(got).all()
    hub_id = int(S.hot[0])
    assert not np.array_equal(got[hub_id], y[hub_id])
    if threads == 1:
        want = O.drawn_steps(y.astype(np.float64), d.cpu().numpy(), 0.02 * (1.0 - t / 10),
                             gamma, 1e-3, 5.0, plan.opt.b)
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-4)


def _setup_level_tables(golden, mode="all"):
    """_setup with the coarse levels drawing from their own aggregated pair tables
    (build_mapped_level_data(level_tables=mode)): the level-l form of the law."""
    from paper_2008_07799_b200.optimizer import build_mapped_level_data
    from paper_2008_07799_b200.graph import DeviceGraph
    from paper_2008_07799_b200.optimizer import prepare_layout
    g = golden_graph(golden, "r500")
    gg = B.Graph(np.asarray(g.indptr, dtype=np.int64), np.asarray(g.indices, dtype=np.int32))
    prep = prepare_layout(DeviceGraph.from_host(gg), B.SimilarityParams(k=2),
                          B.OptimizerParams(seed=0, neg_samples=5, iters=10), min_size=8)
    plan = prep.plan
    plan.levels = build_mapped_level_data(prep.similarity, prep.hierarchy, plan.opt.neg_power,
                                          level_tables=mode)
    ns = O.build_sparse_similarity(O.all_k_neighborhoods(g, 2))
    dh = prep.hierarchy
    oh = O.Hierarchy([lv.to_host() for lv in dh.levels], [m.cpu().numpy() for m in dh.maps],
                     0.8, 8)
    return plan, ns, oh


@pytest.mark.parametrize("pick", ["middle", "coarsest"])
def test_level_tables_pair_law(golden, pick):
    """Coarse levels drawing from their own tables (source ~ R^l, collapse c_a,
    target ~ P^l_a.) follow the reference's draw-at-level-0-then-map law."""
    plan, ns, oh = _setup_level_tables(golden)
    level = _level(plan, pick)
    S = plan.levels[level].sampled
    assert S.map is None and S.collapse is not None
    n = plan.levels[level].n
    ip, tg, P, R, Q = O.level_data(ns, oh, level)
    epochs = max(1, 3_000_000 // n)
    d = plan.sampled_draws(level, 0, n, 2, epochs).cpu().numpy()
    i = d[:, 0, :].ravel().astype(np.int64)
    j = d[:, 1, :].ravel().astype(np.int64)
    counts = np.bincount(i * n + j, minlength=n * n).astype(np.float64)
    expected = np.zeros(n * n)
    rows = np.repeat(np.arange(n), np.diff(ip))
    np.add.at(expected, rows * n + tg, P)
    inner = R - np.bincount(rows, weights=P, minlength=n)
    expected[np.arange(n) * n + np.arange(n)] += np.maximum(inner, 0.0)
    assert _chi2(counts, expected) > 1e-6


@pytest.mark.parametrize("mode", ["none", "all"])
def test_source_records_draw_the_same_steps(golden, mode):
    """32-byte source records (drg_src_records, DRG_SAMPLED_SRC_RECORDS) make the same
    source, span and collapse decisions as the separate tables: with one step in
    flight a whole epoch is bitwise identical, at every level, for the mapped
    (level-0 tables) and the level-table plans."""
    from paper_2008_07799_b200.optimizer import src_records
    plan, _, _ = _setup_level_tables(golden, mode)
    rng = np.random.default_rng(21)
    for level in range(plan.depth + 1):
        L = plan.levels[level]
        S = L.sampled
        y0 = torch.from_numpy(rng.normal(0, 1.0, size=(L.n, 2)).astype(np.float32)).cuda()
        outs = []
        for use in (False, True):
            S.src_rec = (src_records(S, S.indptr if S.map is not None else L.indptr,
                                     S.collapse if level > 0 else None) if use else None)
            y = y0.clone()
            plan.sampled_steps(level, y, 0, L.n, 3, 1, max_threads=1)
            outs.append(y)
        S.src_rec = None
        assert not torch.equal(outs[0], y0)
        assert torch.equal(outs[0], outs[1])


# ---- steps under (i, j) locks (DRG_SAMPLED_LOCKED) ---------------------------------

@pytest.mark.parametrize("pick", ["finest", "coarsest"])
def test_locked_step_and_sequential_epoch_parity(golden, pick):
    """The locked form runs the reference step: single steps within 1e-5 max(1, |g|)
    of the oracle's drawn_steps, a whole epoch with one step in flight equal to the
    oracle's sequential replay."""
    plan, _, _ = _setup(golden)
    level = _level(plan, pick)
    n = plan.levels[level].n
    t = 3
    lr = 1.0 - t / 10
    _, gamma, _ = plan._level_args(level)
    d = plan.sampled_draws(level, 0, n, t)[0]
    y = np.random.default_rng(5).normal(0, 1.0, size=(n, 2)).astype(np.float32)
    yd = torch.from_numpy(y).cuda()
    for s in range(min(n, 24)):
        out = yd.clone()
        plan.sampled_apply(level, d[:, s:s + 1], out, t, locked=True)
        got = out.cpu().numpy().astype(np.float64)
        want = O.drawn_steps(y.astype(np.float64), d[:, s:s + 1].cpu().numpy(), lr, gamma,
                             1e-3, 5.0, plan.opt.b)
        g_got, g_want = (got - y) / lr, (want - y) / lr
        assert np.all(np.abs(g_got - g_want) <= 1e-5 * np.maximum(1.0, np.abs(g_want))), s
    # one step in flight: the same fp32 operations in the same order as the plain
    # form (bit for bit), and the oracle's sequential replay at the late-epoch
    # learning rate of test_sampled_sequential_epoch_parity
    for t2 in (3, 8):
        out, plain = yd.clone(), yd.clone()
        plan.sampled_apply(level, d, out, t2, max_threads=1, locked=True)
        plan.sampled_apply(level, d, plain, t2, max_threads=1)
        assert torch.equal(out, plain)
    want = O.drawn_steps(y.astype(np.float64), d.cpu().numpy(), 1.0 - 8 / 10, gamma, 1e-3, 5.0,
                         plan.opt.b)
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=0, atol=1e-4)


def test_locked_steps_on_one_pair_serialise():
    """Mutual exclusion and visibility of the locks: 8192 attraction-only steps over
    128 disjoint pairs, 256 in flight (every pair contended).  Steps on one pair all
    apply the same map to (y_i, y_j) and the pairs are disjoint, so ANY serial order
    gives bit for bit the sequential result -- the locked run must equal it; plain
    Hogwild at the same concurrency (stale reads, same-address increments from old
    positions) does not."""
    from paper_2008_07799_b200.graph import DeviceGraph
    from paper_2008_07799_b200.optimizer import prepare_layout
    from paper_2008_07799_b200 import synthetic
    g = synthetic.grid(16, 16, device="host")
    prep = prepare_layout(DeviceGraph.from_host(B.Graph(g.indptr, g.indices)),
                          B.SimilarityParams(k=1),
                          B.OptimizerParams(seed=0, neg_samples=0, iters=10, threads=4),
                          max_levels=1)
    plan = prep.plan
    n, pairs, steps = 256, 128, 8192
    rng = np.random.default_rng(3)
    p = rng.integers(0, pairs, size=steps)
    d = torch.from_numpy(np.stack([2 * p, 2 * p + 1]).astype(np.int32)).cuda()
    y = rng.normal(0, 1.0, size=(n, 2)).astype(np.float32)
    seq = torch.from_numpy(y).cuda()
    plan.sampled_apply(0, d, seq, 2, max_threads=1)
    locked = torch.from_numpy(y).cuda()
    plan.sampled_apply(0, d, locked, 2, max_threads=256, locked=True)
    assert torch.equal(locked, seq)
    hog = torch.from_numpy(y).cuda()
    plan.sampled_apply(0, d, hog, 2, max_threads=256)
    assert not torch.equal(hog, seq)


def test_locked_levels_policy(golden):
    """Auto policy: plain levels of small graphs run locked at threads > 1; threads = 1
    (deterministic), the fused form and sampled_locks=False do not."""
    plan, _, _ = _setup(golden)
    for kw, want in (({"threads": 8}, True), ({"threads": 1}, False),
                     ({"threads": 8, "sampled_fused": True}, False),
                     ({"threads": 8, "sampled_locks": False}, False)):
        plan.opt = B.OptimizerParams(seed=0, neg_samples=5, iters=10, **kw)
        hubs = plan.levels[0].sampled.hubs or plan.levels[0].sampled.hot is not None
        assert plan.locked_level(0) == (want and not hubs), kw
    plan.opt = B.OptimizerParams(seed=0, neg_samples=5, iters=10, threads=8)
    y = torch.from_numpy(np.random.default_rng(1).normal(0, 1, (plan.levels[0].n, 2))
                         .astype(np.float32)).cuda()
    y0 = y.clone()
    plan.sampled_steps(0, y, 0, plan.levels[0].n, 0, 2)      # two locked epochs run
    assert torch.isfinite(y).all() and not torch.equal(y, y0)


# ---- negatives read from a per-epoch snapshot (DRG_SAMPLED_SNAPSHOT) ----------------

@pytest.mark.parametrize("pick", ["finest", "coarsest"])
def test_snapshot_epoch_matches_its_sequential_restatement(golden, pick):
    """One step in flight: source and partner live, the negatives read from the
    epoch-start copy (plus the step's own earlier reactions), every update applied at
    once == the oracle's deferred_drawn_epoch(defer=False); and it differs from the
    live-negatives epoch (the flag does something)."""
    plan, _, _ = _setup(golden)
    plan.opt = B.OptimizerParams(seed=0, neg_samples=5, iters=10, threads=4,
                                 sampled_locks=False, sampled_snapshot=True)
    level = _level(plan, pick)
    n = plan.levels[level].n
    t = 8
    _, gamma, _ = plan._level_args(level)
    d = plan.sampled_draws(level, 0, n, t)[0]
    y = np.random.default_rng(11).normal(0, 1.0, size=(n, 2)).astype(np.float32)
    yd = torch.from_numpy(y).cuda()
    plan.evals = None
    plan.sampled_steps(level, yd, 0, n, t, 1, max_threads=1)
    want = O.deferred_drawn_epoch(y.astype(np.float64), d.cpu().numpy(), 1.0 - t / 10, gamma,
                                  1e-3, 5.0, plan.opt.b, defer=False)
    np.testing.assert_allclose(yd.cpu().numpy(), want, rtol=0, atol=1e-4)
    # the update pass draws the negatives itself here (apply_negsnap_kernel): the same
    # ones as the draw pass reports, counted by the distance-evaluation counter
    dn = d.cpu().numpy()
    assert int(plan.evals) == int((dn[0] != dn[1]).sum() + (dn[2:] >= 0).sum())
    # ... and with 64 steps in flight (Hogwild): the same steps, counted the same
    yc = torch.from_numpy(y).cuda()
    plan.evals = None
    plan.sampled_steps(level, yc, 0, n, t, 1, max_threads=64)
    assert torch.isfinite(yc).all() and not torch.equal(yc, torch.from_numpy(y).cuda())
    assert int(plan.evals) == int((dn[0] != dn[1]).sum() + (dn[2:] >= 0).sum())
    live = O.drawn_steps(y.astype(np.float64), d.cpu().numpy(), 1.0 - t / 10, gamma, 1e-3, 5.0,
                         plan.opt.b)
    assert np.abs(want - live).max() > 1e-3


def test_sampled_flag_combinations_are_rejected(golden):
    """DRG_SAMPLED_LOCKED / DRG_SAMPLED_SNAPSHOT serve plain Hogwild levels in the split
    form: with the deterministic mode, the fused form or each other the library
    answers DRG_ERR_UNSUPPORTED (NotImplementedError), never a silent fallback."""
    from paper_2008_07799_b200 import _lib
    plan, _, _ = _setup(golden)
    L = plan.levels[0]
    S = L.sampled
    ip, n_tab, mp, neg = plan._tables(0)
    y = torch.zeros((L.n, 2), dtype=torch.float32, device="cuda")

    def run(flags):
        _lib.call("drg_layout_sampled", _lib.ptr(ip), _lib.ptr(S.span), None,
                  _lib.ptr(S.row_alias), _lib.ptr(S.src_alias), None, _lib.ptr(neg.alias),
                  _lib.ptr(mp), n_tab, neg.n, neg.tail_n, float(neg.tail_p), _lib.ptr(y), 0, L.n,
                  0, 1, 10, 1.0, 0.1, 1e-3, 5.0, 2, 5, 1, 0, 64, flags, L.n, None, None, 0,
                  _lib.stream_ptr())

    run(_lib.DRG_SAMPLED_LOCKED)
    run(_lib.DRG_SAMPLED_SNAPSHOT)
    for bad in (_lib.DRG_SAMPLED_LOCKED | _lib.DRG_SAMPLED_DETERMINISTIC,
                _lib.DRG_SAMPLED_LOCKED | _lib.DRG_SAMPLED_FUSED,
                _lib.DRG_SAMPLED_LOCKED | _lib.DRG_SAMPLED_AGGREGATE,
                _lib.DRG_SAMPLED_SNAPSHOT | _lib.DRG_SAMPLED_LOCKED,
                _lib.DRG_SAMPLED_SNAPSHOT | _lib.DRG_SAMPLED_DETERMINISTIC,
                _lib.DRG_SAMPLED_SNAPSHOT | _lib.DRG_SAMPLED_FUSED):
        with pytest.raises((NotImplementedError, RuntimeError, ValueError)):
            run(bad)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
