"""The rest of the reference's public API on the device: the single-source BFS, K1's
global-memory tier (balls of any size, any k), the single-row similarity helpers,
the per-interaction gradients, the positive sampler, the threads = 1 determinism
contract and the distance-evaluation counter.  Checked against the oracle, the
reference's own hand values and pure-Python restatements (math.exp / math.fsum).
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from conftest import golden_graph
from oracle import oracle as O

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2008_07799_b200")


def as_gpu_graph(g):
    return B.Graph(np.asarray(g.indptr, dtype=np.int64), np.asarray(g.indices, dtype=np.int32))


def assert_nd_equal(got, want):
    assert np.array_equal(got.indptr, want.indptr)
    assert np.array_equal(got.ids, want.ids)
    assert np.array_equal(got.dists, want.dists)


# ------------------------------------------------------------- bfs_k_neighborhood
def test_bfs_k_neighborhood_hand_values():
    """test_graph.py:140-146: P5 from the middle at k=2."""
    g = B.from_edges(np.array([[0, 1], [1, 2], [2, 3], [3, 4]]), 5)
    assert B.bfs_k_neighborhood(g, 2, 2) == [(1, 1), (3, 1), (0, 2), (4, 2)]
    tri = B.from_edges(np.array([[0, 1], [1, 2], [0, 2]]), 3)
    assert B.bfs_k_neighborhood(tri, 0, 5) == [(1, 1), (2, 1)]
    with pytest.raises(ValueError):
        B.bfs_k_neighborhood(g, 5, 1)
    with pytest.raises(ValueError):
        B.bfs_k_neighborhood(g, 0, 0)


@pytest.mark.parametrize("k", [1, 2, 3, 5, 9])
def test_bfs_k_neighborhood_vs_oracle(golden, k):
    g = golden_graph(golden, "r200")
    bg = as_gpu_graph(g)
    for s in (0, 7, 55, 199):
        assert B.bfs_k_neighborhood(bg, s, k) == O.bfs_k_neighborhood(g, s, k)


# ------------------------------------------------------------- K1 global tier
def test_khop_global_tier_star_ball():
    """A leaf of a 20 000-leaf star has a 2-hop ball of 20 000 > 16 383 entries
    (past the block tier): the global-memory tier, bit-exact."""
    n = 20_001
    g = O.from_edges(np.column_stack([np.zeros(n - 1, dtype=np.int64), np.arange(1, n)]), n)
    want = O.all_k_neighborhoods(g, 2)
    assert_nd_equal(B.all_k_neighborhoods(as_gpu_graph(g), 2), want)
    for cap in (100, 16_500):
        assert_nd_equal(B.all_k_neighborhoods(as_gpu_graph(g), 2, cap=cap),
                        O.all_k_neighborhoods(g, 2, cap=cap))


def test_khop_global_tier_ba_100k_uncapped():
    """Uncapped BA-100k at k=2: hub balls of ~19k entries (SURVEY §7 hard part 3),
    bit-exact against the oracle (graph.py:308-366)."""
    from paper_2008_07799_b200 import synthetic
    gh = synthetic.barabasi_albert(100_000, 4, seed=0, device="host")
    g = O.Graph(gh.indptr, gh.indices)
    want = O.all_k_neighborhoods(g, 2)
    assert int(np.diff(want.indptr).max()) > 16_383   # some rows need the global tier
    assert_nd_equal(B.all_k_neighborhoods(as_gpu_graph(g), 2), want)


@pytest.mark.parametrize("k", [8, 11])
def test_khop_large_k_vs_oracle(k):
    """k > 7 (past the packed (dist, id) keys): every source on the global tier."""
    rng = np.random.default_rng(k)
    pairs = rng.integers(0, 300, size=(330, 2))
    g = O.from_edges(pairs, 300)
    nd = B.all_k_neighborhoods(as_gpu_graph(g), k)
    for s in range(300):
        row = O.bfs_k_neighborhood(g, s, k)
        lo, hi = nd.indptr[s], nd.indptr[s + 1]
        assert list(zip(nd.ids[lo:hi].tolist(), nd.dists[lo:hi].tolist())) == row


# ------------------------------------------------------------- similarity helpers
def test_gaussian_table_is_math_exp():
    """test_similarity.py:65-74: exact equality with math.exp."""
    for k, sigma in [(1, 0.9), (3, 1.0), (6, 0.37), (6, 2.5), (12, 3.3)]:
        inv = 1.0 / (2.0 * sigma * sigma)
        want = [math.exp(-(d * d) * inv) for d in range(1, k + 1)]
        assert B.precompute_gaussian_table(k, sigma).tolist() == want
    with pytest.raises(ValueError):
        B.precompute_gaussian_table(0, 1.0)


def test_exp_is_correctly_rounded_over_a_sweep():
    """exp_cr is correctly rounded (checked against 50-digit Decimal.exp) on 5 000
    arguments of the kernel's range; math.exp (glibc) itself is not always: it
    differs from the rounded value in ~1 of 5 000 here, so equality with the
    reference holds except at those arguments."""
    from decimal import Decimal, getcontext
    getcontext().prec = 50
    rng = np.random.default_rng(0)
    sig = np.exp(rng.uniform(np.log(1e-3), np.log(1e3), 1000))
    bad = glibc_off = 0
    for s in sig:
        t = B.precompute_gaussian_table(5, float(s))
        inv = 1.0 / (2.0 * s * s)
        for d, a in zip(range(1, 6), t.tolist()):
            x = -(d * d) * inv
            bad += a != float(Decimal(x).exp())
            glibc_off += a != math.exp(x)
    assert bad == 0
    assert glibc_off <= 5


def test_conditional_row_hand_values():
    """test_similarity.py:26-58."""
    for sigma in (0.3, 1.0, 42.0):
        assert B.conditional_similarity_row([(5, 1), (9, 1)], sigma) == [(5, 0.5), (9, 0.5)]
    row = dict(B.conditional_similarity_row([(0, 1), (1, 2)], 1.0))
    want = math.exp(-0.5) / (math.exp(-0.5) + math.exp(-2.0))
    assert abs(row[0] - want) <= 1e-12
    assert B.conditional_similarity_row([], 1.0) == []
    under = dict(B.conditional_similarity_row([(0, 1), (1, 2)], 1e-5))
    assert under[0] == 1.0 and under[1] == 0.0
    with pytest.raises(ValueError):
        B.conditional_similarity_row([(0, 1)], 0.0)


def test_conditional_row_bitwise_equals_fsum_form():
    """p = table[d] / math.fsum(values), bit for bit (test_similarity.py:76-84), with
    the table's correctly rounded exp (50-digit Decimal, see the sweep above)."""
    from decimal import Decimal, getcontext
    getcontext().prec = 50
    rng = np.random.default_rng(1)
    for _ in range(200):
        m = int(rng.integers(1, 40))
        row = [(j, int(d)) for j, d in enumerate(rng.integers(1, 7, m))]
        sigma = float(np.exp(rng.uniform(-2, 2)))
        inv = 1.0 / (2.0 * sigma * sigma)
        vals = [float(Decimal(-(d * d) * inv).exp()) for _, d in row]
        total = math.fsum(vals)
        want = [v / total for v in vals]
        assert [p for _, p in B.conditional_similarity_row(row, sigma)] == want


def test_search_sigma_vs_oracle():
    rng = np.random.default_rng(2)
    for _ in range(100):
        m = int(rng.integers(2, 60))
        d = rng.integers(1, 5, m)
        row = [(j, int(x)) for j, x in enumerate(d)]
        target = float(rng.uniform(1.0, m + 5))
        dv, cnt = np.unique(d, return_counts=True)
        want = O.search_sigma(cnt, dv, m, min(max(target, 1.0), float(m)))
        assert B.search_sigma(row, target) == pytest.approx(want, rel=1e-12)
    assert B.search_sigma([(3, 1)], 2.0) == 1.0
    row = [(j, 2) for j in range(4)]
    sigma = B.search_sigma(row, 4.0)
    h = -sum(p * math.log2(p) for _, p in B.conditional_similarity_row(row, sigma))
    assert h == 2.0
    with pytest.raises(ValueError):
        B.search_sigma([], 2.0)


# ------------------------------------------------------------- gradients, samplers
def test_gradient_hand_values_and_fd():
    """test_optimizer.py:79-141 (hand values; central differences b = 1..3)."""
    assert np.allclose(B.attractive_gradient((1.0, 0.0), (0.0, 0.0), 1), [-1.0, 0.0])
    assert np.array_equal(B.attractive_gradient((2.0, 3.0), (2.0, 3.0), 2), [0.0, 0.0])
    g = B.repulsive_gradient((1.0, 0.0), (0.0, 0.0), 2, 0.1, 0.0)
    assert g == pytest.approx([0.1 * 4.0 / 2.0, 0.0], rel=1e-12)
    assert np.all(np.abs(B.repulsive_gradient((1e-3, 0.0), (0.0, 0.0), 2, 0.1, 1e-9, 5.0))
                  <= 5.0)
    rng = np.random.default_rng(3)
    h = 1e-6
    for b in (1, 2, 3):
        for _ in range(20):
            yi, yj = rng.normal(size=2), rng.normal(size=2)

            def f(y):
                d2 = float(((y - yj) ** 2).sum())
                return math.log(1.0 / (1.0 + d2 ** b))
            grad = B.attractive_gradient(yi, yj, b)
            for ax in range(2):
                e = np.zeros(2)
                e[ax] = h
                fd = (f(yi + e) - f(yi - e)) / (2 * h)
                assert abs(fd - grad[ax]) <= 1e-4 * max(1.0, abs(grad[ax]))


def test_positive_sampler_and_alias_validation(golden):
    g = as_gpu_graph(golden_graph(golden, "p5"))
    ns = B.build_sparse_similarity(B.all_k_neighborhoods(g, 1), B.SimilarityParams(k=1))
    smp = B.build_positive_sampler(ns)
    src, dst = smp.sample_many(np.random.default_rng(4), 200_000)
    pairs = {(int(a), int(b)) for a, b in zip(src[:2000], dst[:2000])}
    assert pairs == {(0, 1), (1, 0), (1, 2), (2, 1), (2, 3), (3, 2), (3, 4), (4, 3)}
    w = ns.weights[ns.sources() < ns.targets]
    freq = np.bincount(np.minimum(src, dst), minlength=4)[:4] / len(src)
    assert np.abs(freq - w / w.sum()).max() < 0.01
    with pytest.raises(ValueError):
        B.build_alias_table(np.zeros(3))
    with pytest.raises(ValueError):
        B.build_alias_table(np.array([0.5, -0.1]))
    empty = B.build_sparse_similarity(
        B.all_k_neighborhoods(B.from_edges(np.empty((0, 2), dtype=np.int64), 2), 1))
    with pytest.raises(ValueError):
        B.build_positive_sampler(empty)


# ------------------------------------------------------------- determinism, counters
@pytest.mark.parametrize("name", ["p5", "grid17", "r500"])
def test_threads_one_is_bitwise_deterministic(golden, name):
    """SPEC.md:347 / test_acceptance.py:291-306: threads = 1 (the default) gives the
    same coordinates bit for bit; threads > 1 (Hogwild) still runs."""
    g = as_gpu_graph(golden_graph(golden, name))
    for k in (1, 2):
        opt = B.OptimizerParams(seed=5, iters=60)
        sim = B.SimilarityParams(k=k)
        a = B.layout_graph(g, sim, opt)
        b = B.layout_graph(g, sim, opt)
        assert np.array_equal(a.positions, b.positions)
    c = B.layout_graph(g, B.SimilarityParams(k=1), B.OptimizerParams(seed=5, iters=60, threads=4))
    assert np.isfinite(c.positions).all()


def test_distance_eval_counter():
    """test_optimizer.py:289-296 plus the exact count: on K2 every negative hits the
    positive pair (no target), so each step evaluates exactly one distance."""
    rng = np.random.default_rng(4)
    g = B.from_edges(rng.integers(0, 120, size=(240, 2)), 120)
    for threads in (1, 8):
        opt = B.OptimizerParams(seed=2, iters=7, neg_samples=5, threads=threads)
        lay = B.layout_graph(g, opt_params=opt)
        steps = opt.iters * sum(lay.stats["levels"])
        assert lay.stats["gradient_steps"] == steps
        assert 0 < lay.stats["distance_evals"] <= steps * (opt.neg_samples + 1)
    k2 = B.from_edges(np.array([[0, 1]]), 2)
    lay = B.layout_graph(k2, opt_params=B.OptimizerParams(seed=9, iters=50))
    assert lay.stats["distance_evals"] == lay.stats["gradient_steps"] == 100


def test_distance_eval_counter_matches_draws():
    """The device counter equals (i != j) + drawn negatives over the epoch's draws."""
    from paper_2008_07799_b200.graph import DeviceGraph
    from paper_2008_07799_b200.optimizer import prepare_layout
    rng = np.random.default_rng(6)
    g = B.from_edges(rng.integers(0, 3000, size=(9000, 2)), 3000)
    prep = prepare_layout(DeviceGraph.from_host(g), B.SimilarityParams(k=2),
                          B.OptimizerParams(seed=1, iters=10, threads=4))
    plan = prep.plan
    for level in range(plan.depth + 1):
        n = plan.levels[level].n
        y = torch.randn((n, 2), device="cuda")
        before = plan.distance_evals()
        plan.sampled_steps(level, y, 0, n, 3, 1)
        got = plan.distance_evals() - before
        d = plan.sampled_draws(level, 0, n, 3, 1)[0]
        want = int((d[0] != d[1]).sum()) + int((d[2:] >= 0).sum())
        assert got == want


def test_default_start_is_the_reference_draw_in_relabelled_order():
    """With isolated nodes the coarsest level is relabelled (isolated_last); the
    default Y0 must still be the reference's draw (optimizer.py:393-395) of each
    node, i.e. the same as passing that draw explicitly."""
    from paper_2008_07799_b200.optimizer import _INIT_TAG, _derive_seed
    rng = np.random.default_rng(8)
    pairs = rng.integers(0, 150, size=(300, 2))
    g = B.from_edges(pairs, 200)   # 50+ isolated nodes
    opt = B.OptimizerParams(seed=3, iters=20)
    a = B.layout_graph(g, B.SimilarityParams(k=1), opt, max_levels=1)
    y0 = np.random.default_rng(_derive_seed(3, _INIT_TAG)).normal(0.0, opt.init_scale, (200, 2))
    b = B.layout_graph(g, B.SimilarityParams(k=1), opt, max_levels=1, init_positions=y0)
    assert np.array_equal(a.positions, b.positions)
